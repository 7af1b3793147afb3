"""Development aid: projection time per algorithm at cfg0 size (n=4096, D=2242, s=10)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1810_01967_b200 as cb
from paper_1810_01967_b200 import _lib, workloads
from paper_1810_01967_b200.forward_model import SamplingPattern, make_cartesian_operator
from paper_1810_01967_b200.projection import project_device, overflow_counts
cfg = workloads.make_cfg0()
A = make_cartesian_operator(SamplingPattern(cfg.pattern, cfg.spatial_shape))
V = torch.from_numpy(np.ascontiguousarray(cfg.cdict.basis, dtype=np.complex64)).cuda()
Yt = torch.from_numpy(np.ascontiguousarray(cfg.Y.T).astype(np.complex64)).cuda()
Z = (A.n / A.m) * A.fm_adjoint_compressed(Yt, V)
dd = cb.device_dictionary(cfg.cdict)
for algo in ("tcgen05", "ffma"):
    for rep in range(20):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        project_device(Z, dd, algo=algo)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(algo, f"{1e6*dt:.1f} us", overflow_counts(A.n, 10), flush=True)
