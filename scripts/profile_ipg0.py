"""Development aid: cProfile of one warm cfg0 solve (host-side setup / loop overheads)."""
import cProfile, os, pstats, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1810_01967_b200 import workloads
from paper_1810_01967_b200.forward_model import SamplingPattern, make_cartesian_operator
from paper_1810_01967_b200.solver import SolverConfig, solve_compressed
cfg = workloads.make_cfg0()
A = make_cartesian_operator(SamplingPattern(cfg.pattern, cfg.spatial_shape))
conf = SolverConfig(mode="blip_exact", max_iters=20, zeta=2.0, compressed=10)
for _ in range(3):
    solve_compressed(cfg.Y, A, cfg.cdict, None, conf)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    solve_compressed(cfg.Y, A, cfg.cdict, None, conf)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
