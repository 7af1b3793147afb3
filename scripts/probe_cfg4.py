"""cfg4 (3-D IPG) probe: generation time, per-iteration time, map accuracy."""
import sys
import time

import numpy as np
import torch

from paper_1810_01967_b200 import workloads
from paper_1810_01967_b200.forward_model import SamplingPattern, make_cartesian_operator
from paper_1810_01967_b200.solver import SolverConfig, solve_compressed

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 3

# wall-time breakdown of the solve wrapper (state construction, output conversion)
import paper_1810_01967_b200.solver as _sv
_T = {}


def _timed(name, fn):
    def w(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn(*a, **k)
        torch.cuda.synchronize()
        _T[name] = _T.get(name, 0.0) + time.perf_counter() - t0
        return r
    return w


_sv.IpgState.__init__ = _timed("state_init", _sv.IpgState.__init__)
_sv._image_to_host = _timed("image_to_host", _sv._image_to_host)
_sv._maps_from = _timed("maps_from", _sv._maps_from)
dev = torch.device("cuda:0")
t = time.perf_counter()
cfg = workloads.make_cfg4(device=dev)
print("gen", time.perf_counter() - t, "d", cfg.d, "Y", cfg.Y.shape, flush=True)
t = time.perf_counter()
A = make_cartesian_operator(SamplingPattern(cfg.pattern, cfg.spatial_shape), device=dev)
print("op", time.perf_counter() - t, flush=True)
import os
prof = os.environ.get("PROBE_PROFILE") == "1"
for it in ((int(os.environ.get("PROBE_PROF_ITERS", "1")),) if prof else (1, iters)):
    if prof:
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
    conf = SolverConfig(mode="blip_exact", max_iters=it, zeta=2.0, compressed=10)
    torch.cuda.synchronize()
    t = time.perf_counter()
    X, maps, gam, trace = solve_compressed(cfg.Y, A, cfg.cdict, None, conf)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    if prof:
        torch.cuda.profiler.stop()
    trials = sum(r["shrinks"] + 1 for r in trace.records)
    print(f"iters {trace.iterations} trials {trials} wall {dt:.2f}s loop {trace.total_time:.2f}s "
          f"fid {trace.fidelities()[-1]:.4g}  breakdown {_T}", flush=True)
    _T.clear()
    from paper_1810_01967_b200.projection import overflow_counts
    print("   overflow_counts (exhaustive, warp-rescored) of last projection:",
          overflow_counts(A.n, 10), "of", A.n, flush=True)
    for r in trace.records:
        print("  ", {k: (round(v, 5) if isinstance(v, float) else v) for k, v in r.items()})
inside = cfg.labels > 0
true = cfg.cdict.parent.lookup_table[cfg.class_atoms[cfg.labels[inside]]]
ok = (np.asarray(maps.t1)[inside] == true[:, 0]) & (np.asarray(maps.t2)[inside] == true[:, 1]) \
    & (np.asarray(maps.b0)[inside] == true[:, 2])
print("map exact-atom fraction (inside)", float(ok.mean()),
      "T1 rel err median", float(np.median(np.abs(np.asarray(maps.t1)[inside] / true[:, 0] - 1))))
print("peak mem GB", torch.cuda.max_memory_allocated() / 1e9)
