"""B200-native (sm_100a) exact-projection IPG hot path of CoverBLIP (arXiv 1810.01967).

Drop-in for the reference package's reconstruction API on the north-star path
(``coverblip.projection.project_cone_exact``, ``ForwardOperator.apply/adjoint``,
``step_shrinkage``, ``solve`` / ``solve_compressed``).  Compute runs in
``libcoverblip_b200.so`` (hand-written CUDA for sm_100a + cuFFT); PyTorch is
used only for device memory, streams and ``torch.distributed``.
"""

from .dictionary import (CompressedDictionary, DeviceDictionary, Dictionary, ParameterGrid,
                         device_dictionary, generate_fingerprints, svd_compress)
from .projection import ConeProjection, project_cone_exact, project_device

__version__ = "0.1.0"

__all__ = [
    "CompressedDictionary", "ConeProjection", "DeviceDictionary", "Dictionary", "ParameterGrid",
    "device_dictionary", "generate_fingerprints", "project_cone_exact", "project_device",
    "svd_compress",
]


_LAZY = ("forward_model", "solver", "distributed", "workloads", "containers")


def __getattr__(name):  # lazy: operator / solver / distributed pull in more modules
    import importlib
    if name in _LAZY:
        return importlib.import_module(f".{name}", __name__)
    for mod in _LAZY:
        try:
            m = importlib.import_module(f".{mod}", __name__)
        except ModuleNotFoundError:
            continue
        if hasattr(m, name):
            return getattr(m, name)
    raise AttributeError(name)
