"""Pruned vs unpruned split screen on the same IPG trial (development aid): cfg4 / cfg2 state
after K iterations, one projection step timed with and without the pruning workspace."""
import ctypes
import sys

import torch

from paper_1810_01967_b200 import _lib, workloads
from paper_1810_01967_b200.forward_model import SamplingPattern, make_cartesian_operator
from paper_1810_01967_b200.solver import SolverConfig, _solve_core

which = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 5
dev = torch.device("cuda:0")
cfg = getattr(workloads, f"make_{which}")(device=dev)
s = cfg.cdict.s
A = make_cartesian_operator(SamplingPattern(cfg.pattern, cfg.spatial_shape), device=dev)
st, trace = _solve_core(cfg.Y, A, cfg.cdict, None,
                        SolverConfig(mode="blip_exact", max_iters=K, zeta=2.0, compressed=s),
                        None, cfg.cdict.basis, return_device=True)
lib = _lib.load()
mu = trace.records[-1]["mu"]
plain = lib.cbb_project_workspace_bytes(st.n, s)
full = st.pws_bytes
for label, wsb in (("pruned", full), ("unpruned", plain), ("pruned", full)):
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    times = []
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(lib.cbb_project_step_ex(
            st.X.data_ptr(), st.G.data_ptr(), float(mu), None, st.Z.data_ptr(), st.n,
            ctypes.byref(st.dd.view), st.idx.data_ptr(), st.idx.data_ptr(), st.idx_n.data_ptr(),
            st.gam_n.data_ptr(), st.Xn.data_ptr(), st.dX.data_ptr(), st.scal[1:2].data_ptr(),
            ws.data_ptr(), wsb, 0, _lib.stream_ptr()), "step")
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    listed, total = ctypes.c_int64(0), ctypes.c_int64(0)
    lib.cbb_project_prune_stats(ws.data_ptr(), wsb, st.n, ctypes.byref(st.dd.view),
                                ctypes.byref(listed), ctypes.byref(total), _lib.stream_ptr())
    frac = listed.value / total.value if listed.value >= 0 and total.value else None
    print(f"{which} after {K} it: {label:9s} step {min(times):7.2f} ms  listed {frac}", flush=True)
