"""IPG probe for cfg2 / cfg4: timing of K iterations through solve_compressed, the per-trial
tile-pruning statistics, and (under ncu) a launch list of the loop.

    python scripts/probe_ipg.py cfg2|cfg4 [iters]
"""
import ctypes
import sys
import time

import torch

from paper_1810_01967_b200 import _lib, workloads
from paper_1810_01967_b200.forward_model import SamplingPattern, make_cartesian_operator
from paper_1810_01967_b200.solver import SolverConfig, solve_compressed

which = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 4
if "nograph" in sys.argv[3:]:
    # development: the host-driven iteration (every kernel visible to ncu's launch list)
    from paper_1810_01967_b200.solver import IpgState
    IpgState.graph_capable = lambda self, config: False
if "norephint" in sys.argv[3:]:
    from paper_1810_01967_b200.solver import IpgState
    IpgState.rep_hint_min_voxels = 1 << 62
dev = torch.device("cuda:0")
cfg = getattr(workloads, f"make_{which}")(device=dev)
s = cfg.cdict.s
A = make_cartesian_operator(SamplingPattern(cfg.pattern, cfg.spatial_shape), device=dev)
lib = _lib.load()
stats = []


def hook(k, st, mu, shrinks, fixed):
    listed, total = ctypes.c_int64(0), ctypes.c_int64(0)
    ws = st.project_workspace()
    lib.cbb_project_prune_stats(ws.data_ptr(), st.pws_bytes, st.n, ctypes.byref(st.dd.view),
                                ctypes.byref(listed), ctypes.byref(total), _lib.stream_ptr())
    det = None
    if "detail" in sys.argv[3:]:
        import numpy as np
        n_vt = (st.n + 127) // 128
        cnt = np.zeros(n_vt, dtype=np.int32)
        bkt = np.zeros(n_vt, dtype=np.int32)
        lib.cbb_project_prune_detail(ws.data_ptr(), st.pws_bytes, st.n, ctypes.byref(st.dd.view),
                                     cnt.ctypes.data, bkt.ctypes.data, _lib.stream_ptr())
        if cnt[0] >= 0:
            det = " ".join(f"b{b}: {int((bkt == b).sum())} vt x {cnt[bkt == b].mean() if (bkt == b).any() else 0:.0f}"
                           for b in range(4))
    stats.append((k, shrinks, listed.value / max(1, total.value) if listed.value >= 0 else None, det))


solve_compressed(cfg.Y, A, cfg.cdict, None, SolverConfig(mode="blip_exact", max_iters=2,
                                                          zeta=2.0, compressed=s))
torch.cuda.synchronize()
torch.cuda.profiler.start()
t0 = time.perf_counter()
X, maps, gam, trace = solve_compressed(cfg.Y, A, cfg.cdict, None,
                                       SolverConfig(mode="blip_exact", max_iters=iters, zeta=2.0,
                                                    compressed=s), on_iter=hook)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(f"{which}: {trace.iterations} iterations, loop {trace.total_time * 1e3 / trace.iterations:.2f} "
      f"ms/iter, fidelity {trace.fidelities()[-1]!r}")
for k, sh, fr, det in stats:
    print(f"  iter {k}: shrinks {sh}, listed tile fraction {fr}" + (f"  [{det}]" if det else ""))
