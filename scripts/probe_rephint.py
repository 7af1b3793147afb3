"""Experiment (development aid): a third warm-start hint for the first trial of every IPG
iteration -- the best tile representative of Z = X - mu G, written into idx_n (which at a first
trial only repeats idx) -- and its effect on the pruned tile lists and the trial time.

    python scripts/probe_rephint.py cfg4 12 0|1
"""
import ctypes
import sys

import torch

from paper_1810_01967_b200 import _lib, workloads
from paper_1810_01967_b200.forward_model import SamplingPattern, make_cartesian_operator
from paper_1810_01967_b200.projection import project_device
from paper_1810_01967_b200.solver import IpgState, SolverConfig, solve_compressed

which, iters, use = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
IpgState.graph_capable = lambda self, config: False
dev = torch.device("cuda:0")
cfg = getattr(workloads, f"make_{which}")(device=dev)
s = cfg.cdict.s
A = make_cartesian_operator(SamplingPattern(cfg.pattern, cfg.spatial_shape), device=dev)
lib = _lib.load()
state = {"first": False, "grads": 0, "log": []}
orig_grad, orig_ps = IpgState.gradient, IpgState.project_step


def grad(self):
    orig_grad(self)
    state["first"] = True
    state["grads"] += 1


def ps(self, mu, slot, mu_dev=None):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record()
    first = state["first"] and state["grads"] >= 2
    if first and use:
        atoms_idx, rdd = self.dd.representatives()
        ridx, _, _ = project_device(self.X - float(mu) * self.G, rdd, idx_int64=True,
                                    proj_c128=False)
        self.idx_n.copy_(atoms_idx[ridx])
    ev[1].record()
    orig_ps(self, mu, slot, mu_dev)
    ev[2].record()
    torch.cuda.synchronize()
    listed, total = ctypes.c_int64(0), ctypes.c_int64(0)
    ws = self.project_workspace()
    lib.cbb_project_prune_stats(ws.data_ptr(), self.pws_bytes, self.n, ctypes.byref(self.dd.view),
                                ctypes.byref(listed), ctypes.byref(total), _lib.stream_ptr())
    state["log"].append((state["grads"], first, ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]),
                         listed.value / max(1, total.value)))
    state["first"] = False


IpgState.gradient, IpgState.project_step = grad, ps
X, maps, gam, trace = solve_compressed(cfg.Y, A, cfg.cdict, None,
                                       SolverConfig(mode="blip_exact", max_iters=iters, zeta=2.0,
                                                    compressed=s))
print(f"{which} use={use}: {trace.iterations} iterations, fidelity {trace.fidelities()[-1]!r}")
tot_h = tot_p = 0.0
for g, first, th, tp, fr in state["log"]:
    tot_h += th
    tot_p += tp
    print(f"  iter {g} {'first' if first else '     '} hint {th:6.2f} ms  project_step {tp:7.2f} ms  listed {fr:.3f}")
print(f"total hint {tot_h:.1f} ms, project_step {tot_p:.1f} ms over {len(state['log'])} trials")
