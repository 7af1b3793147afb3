"""Development aid: cfg0 IPG wall time per iteration (warm)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1810_01967_b200 import workloads
from paper_1810_01967_b200.forward_model import SamplingPattern, make_cartesian_operator
from paper_1810_01967_b200.solver import SolverConfig, solve_compressed
cfg = workloads.make_cfg0()
A = make_cartesian_operator(SamplingPattern(cfg.pattern, cfg.spatial_shape))
conf = SolverConfig(mode="blip_exact", max_iters=20, zeta=2.0, compressed=10)
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    X, maps, gam, tr = solve_compressed(cfg.Y, A, cfg.cdict, None, conf)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"solve {1e3*dt:.2f} ms, {tr.iterations} iters, {1e3*dt/tr.iterations:.3f} ms/iter, loop {1e3*tr.total_time:.2f} ms", flush=True)
