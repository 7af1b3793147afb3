"""Matched-filter kernel time on cfg1 (library CUDA events around the mf launch; dev aid)."""
import ctypes, os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1810_01967_b200 as cb
from paper_1810_01967_b200 import _lib
from paper_1810_01967_b200.workloads import random_atoms, cone_voxels
from paper_1810_01967_b200.projection import project_device
N = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
D = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 17
atoms = random_atoms(D, 10, seed=0)
Z, gen = cone_voxels(atoms, N, seed=1, dtype=np.complex64)
dd = cb.device_dictionary(atoms); zt = torch.from_numpy(Z).cuda()
lib = _lib.load(); lib.cbb_timing_enable(1)
ks = []
for it in range(6):
    idx, gam, proj = project_device(zt, dd, algo="tcgen05", proj_c128=False)
    torch.cuda.synchronize()
    kms = ctypes.c_float(); _lib.check(lib.cbb_timing_last_ms(ctypes.byref(kms)), "timing")
    if it >= 2: ks.append(kms.value)
lib.cbb_timing_enable(0)
print(f"{os.environ.get('CBB_LIB_PATH','default')}: mf kernel median {statistics.median(ks):.3f} ms  min {min(ks):.3f}  agree={(idx.cpu().numpy()==gen).mean():.4f}")
