"""A/B timing of the cfg1 projection between two builds of the library (development aid).

    python scripts/ab_cfg1.py lib_a.so lib_b.so ...
Each library prepares the dictionary and projects 2^20 x 2^17 (s = 10) five times; the CUDA
events of the library bracket the screening kernel.
"""
import ctypes
import sys

import numpy as np
import torch

from paper_1810_01967_b200._lib import DictView
from paper_1810_01967_b200.workloads import cone_voxels, random_atoms

N, D, S = 1 << 20, 1 << 17, 10
atoms = random_atoms(D, S, seed=0)
Z, gen = cone_voxels(atoms, N, seed=1, dtype=np.complex64)
dev = torch.device("cuda")
zt = torch.from_numpy(Z).to(dev)
at = torch.from_numpy(atoms).to(dev)
idx = torch.empty(N, dtype=torch.int64, device=dev)
gam = torch.empty(N, dtype=torch.float64, device=dev)
proj = torch.empty((N, S), dtype=torch.complex64, device=dev)
libs = [ctypes.CDLL(p) for p in sys.argv[1:]]
res = {p: [] for p in sys.argv[1:]}
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
state = []
for p, lib in zip(sys.argv[1:], libs):
    lib.cbb_dict_storage_bytes.restype = ctypes.c_size_t
    lib.cbb_project_workspace_bytes.restype = ctypes.c_size_t
    nb = lib.cbb_dict_storage_bytes(ctypes.c_int64(D), ctypes.c_int32(S))
    store = torch.empty(nb, dtype=torch.uint8, device=dev)
    view = DictView()
    assert lib.cbb_dict_prepare(ctypes.c_void_p(at.data_ptr()), 1, ctypes.c_int64(D), S,
                                ctypes.c_void_p(store.data_ptr()), ctypes.byref(view), st) == 0
    wsb = lib.cbb_project_workspace_bytes(ctypes.c_int64(N), S)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    lib.cbb_timing_enable(1)
    state.append((store, view, ws, wsb))
ms = ctypes.c_float(0)
REPS = 24
# single projections of every library interleaved (A, B, C, A, B, C, ...): all builds see the same
# clock / power conditions
for it in range(REPS + 3):
    for p, lib, (store, view, ws, wsb) in zip(sys.argv[1:], libs, state):
        rc = lib.cbb_project_cone_exact(ctypes.c_void_p(zt.data_ptr()), 0, ctypes.c_int64(N),
                                        ctypes.byref(view), ctypes.c_void_p(idx.data_ptr()), 1,
                                        ctypes.c_void_p(gam.data_ptr()),
                                        ctypes.c_void_p(proj.data_ptr()), 0,
                                        ctypes.c_void_p(ws.data_ptr()), ctypes.c_size_t(wsb), 1, st)
        assert rc == 0
        lib.cbb_timing_last_ms(ctypes.byref(ms))
        if it >= 3:
            res[p].append(ms.value)
for p, v in res.items():
    print(f"{p}: screen kernel ms median {np.median(v):.3f} min {min(v):.3f} "
          f"p25 {np.percentile(v, 25):.3f} p75 {np.percentile(v, 75):.3f} ({len(v)} runs)")
