"""Development aid: a short cfg2 IPG solve (for launch lists / timing breakdown)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1810_01967_b200 import workloads
from paper_1810_01967_b200.forward_model import SamplingPattern, make_cartesian_operator
from paper_1810_01967_b200.solver import SolverConfig, solve_compressed
from paper_1810_01967_b200.projection import overflow_count, overflow_counts
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = workloads.make_cfg2(device="cuda")
A = make_cartesian_operator(SamplingPattern(cfg.pattern, cfg.spatial_shape))
conf = SolverConfig(mode="blip_exact", max_iters=iters, zeta=2.0, compressed=20)
t0 = time.perf_counter()
X, maps, gam, trace = solve_compressed(cfg.Y, A, cfg.cdict, None, conf)
torch.cuda.synchronize()
print("iters", trace.iterations, "s/iter", (time.perf_counter() - t0) / trace.iterations,
      "overflow(last proj)", overflow_counts(A.n, 20), flush=True)
# single projections of the first IPG input under each algorithm
from paper_1810_01967_b200.projection import project_device
from paper_1810_01967_b200.dictionary import device_dictionary
V = torch.from_numpy(np.ascontiguousarray(cfg.cdict.basis, dtype=np.complex64)).cuda()
Yt = torch.from_numpy(np.ascontiguousarray(cfg.Y.T)).cuda()
Z = (A.n / A.m) * A.fm_adjoint_compressed(Yt, V)
dd = device_dictionary(cfg.cdict)
for algo in ("tcgen05", "ffma", "exhaustive"):
    for rep in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        idx, gam, proj = project_device(Z, dd, algo=algo)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(algo, f"{1e3*dt:.2f} ms", "overflows", overflow_counts(A.n, 20), flush=True)
    if algo == "tcgen05":
        ref_idx = idx.clone()
    else:
        print("  indices equal to tcgen05 path:", bool(torch.equal(idx, ref_idx)))
