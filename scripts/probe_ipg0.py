"""cfg0 IPG timing probe: per-iteration loop time of repeated solves (cached state + graphs) and,
under ncu, the kernel launch list of one solve."""
import sys
import time

import torch

from paper_1810_01967_b200 import workloads
from paper_1810_01967_b200.forward_model import SamplingPattern, make_cartesian_operator
from paper_1810_01967_b200.solver import SolverConfig, solve_compressed

cfg = workloads.make_cfg0()
A = make_cartesian_operator(SamplingPattern(cfg.pattern, cfg.spatial_shape))
conf = SolverConfig(mode="blip_exact", max_iters=20, zeta=2.0, compressed=10)
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 4):
    if rep == 2:
        torch.cuda.profiler.start()
    X, maps, gam, trace = solve_compressed(cfg.Y, A, cfg.cdict, None, conf)
    if rep == 2:
        torch.cuda.profiler.stop()
    print(f"solve {rep}: {trace.iterations} it, loop {1e3 * trace.total_time / trace.iterations:.3f}"
          f" ms/iter, trials {sum(r['shrinks'] + 1 for r in trace.records)}", flush=True)
