"""Development aid: matched-filter kernel time vs whole projection time (cfg1 and cfg2 input)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1810_01967_b200 as cb
from paper_1810_01967_b200 import _lib, workloads
from paper_1810_01967_b200.projection import project_device, overflow_counts
lib = _lib.load()
def run(label, Z, dd, algo="tcgen05", reps=3):
    lib.cbb_timing_enable(1)
    k = ctypes.c_float(0)
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        project_device(Z, dd, algo=algo)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        lib.cbb_timing_last_ms(ctypes.byref(k))
    lib.cbb_timing_enable(0)
    print(f"{label} {algo}: total {1e3*dt:.2f} ms, screening kernel {k.value:.2f} ms, overflows {overflow_counts(Z.shape[0], Z.shape[1])}", flush=True)
atoms = workloads.random_atoms(1 << 17 if "cfg2only" not in sys.argv else 1024, 10, seed=0)
Z, _ = workloads.cone_voxels(atoms, 1 << 20 if "cfg2only" not in sys.argv else 1024, seed=1, dtype=np.complex64)
if "cfg2only" not in sys.argv: run("cfg1", torch.from_numpy(Z).cuda(), cb.device_dictionary(atoms))
if len(sys.argv) > 1:
    from paper_1810_01967_b200.forward_model import SamplingPattern, make_cartesian_operator
    cfg = workloads.make_cfg2(device="cuda")
    A = make_cartesian_operator(SamplingPattern(cfg.pattern, cfg.spatial_shape))
    V = torch.from_numpy(np.ascontiguousarray(cfg.cdict.basis, dtype=np.complex64)).cuda()
    Yt = torch.from_numpy(np.ascontiguousarray(cfg.Y.T)).cuda()
    Z2 = (A.n / A.m) * A.fm_adjoint_compressed(Yt, V)
    dd2 = cb.device_dictionary(cfg.cdict)
    run("cfg2-iter1", Z2, dd2)
    run("cfg2-iter1", Z2, dd2, algo="ffma")
