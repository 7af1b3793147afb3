"""Operator timing probe (development aid): apply / adjoint / residual of the s-channel operator
at cfg2 or cfg4 through bench.operator_block.  CBB_LIB_PATH selects the library build.

    python scripts/probe_op.py cfg4|cfg2
"""
import json
import sys

import torch

import bench
from paper_1810_01967_b200 import workloads
from paper_1810_01967_b200.forward_model import SamplingPattern, make_cartesian_operator

which = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
dev = torch.device("cuda:0")
cfg = getattr(workloads, f"make_{which}")(device=dev)
A = make_cartesian_operator(SamplingPattern(cfg.pattern, cfg.spatial_shape), device=dev)
torch.cuda.synchronize()
torch.cuda.profiler.start()   # ncu --profile-from-start off: only the operator launches
res = bench.operator_block(A, cfg, dev, cfg.cdict.s)
torch.cuda.profiler.stop()
print(which, json.dumps({k: (round(v["ms"], 4), round(v["frac"], 3)) for k, v in res.items()
                         if isinstance(v, dict)}))
