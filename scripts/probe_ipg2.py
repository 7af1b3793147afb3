"""Development aid: one cfg2 IPG solve bracketed by cudaProfilerStart/Stop (for ncu
--profile-from-start off), after a warm-up solve."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1810_01967_b200 import workloads
from paper_1810_01967_b200.forward_model import SamplingPattern, make_cartesian_operator
from paper_1810_01967_b200.solver import SolverConfig, solve_compressed
cfg = workloads.make_cfg2(device="cuda")
A = make_cartesian_operator(SamplingPattern(cfg.pattern, cfg.spatial_shape))
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 3
solve_compressed(cfg.Y, A, cfg.cdict, None, SolverConfig(mode="blip_exact", max_iters=2, zeta=2.0, compressed=20))
torch.cuda.synchronize()
torch.cuda.profiler.start()
t0 = time.perf_counter()
X, maps, gam, tr = solve_compressed(cfg.Y, A, cfg.cdict, None, SolverConfig(mode="blip_exact", max_iters=iters, zeta=2.0, compressed=20))
torch.cuda.synchronize()
dt = time.perf_counter() - t0
torch.cuda.profiler.stop()
print(f"{tr.iterations} iters, {sum(r['shrinks'] + 1 for r in tr.records)} trials, {1e3*dt/tr.iterations:.2f} ms/iter, loop {1e3*tr.total_time/tr.iterations:.2f} ms/iter", flush=True)
