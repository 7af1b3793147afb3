"""Breakdown of the end-to-end projection path (development aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1810_01967_b200 as cb
from paper_1810_01967_b200.device import pinned_empty
from paper_1810_01967_b200.workloads import random_atoms, cone_voxels
N, D, S = 1 << 20, 1 << 17, 10
atoms = random_atoms(D, S, seed=0)
Z, _ = cone_voxels(atoms, N, seed=1, dtype=np.complex64)
dd = cb.device_dictionary(atoms)
Zp = pinned_empty((N, S), np.complex128); Zp[:] = Z
zh = torch.from_numpy(Zp); print("pinned:", zh.is_pinned())
dev = torch.device("cuda")
zt = torch.empty((N, S), dtype=torch.complex128, device=dev)
for name, f in [("H2D 168MB", lambda: zt.copy_(zh, non_blocking=True)),
                ("D2H 168MB", lambda: zh.copy_(zt, non_blocking=True))]:
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter(); f(); torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"{name}: {dt*1e3:.2f} ms  {zt.numel()*16/dt/1e9:.1f} GB/s")
t0 = time.perf_counter(); h = torch.empty((N, S), dtype=torch.complex128, pin_memory=True); print("pinned alloc ms", (time.perf_counter()-t0)*1e3)
del h
t0 = time.perf_counter(); h = torch.empty((N, S), dtype=torch.complex128, pin_memory=True); print("pinned alloc (cached) ms", (time.perf_counter()-t0)*1e3)
for i in range(4):
    t0 = time.perf_counter(); r = cb.project_cone_exact(Zp, dd); dt = time.perf_counter() - t0
    print(f"e2e call {i}: {dt*1e3:.2f} ms")
from paper_1810_01967_b200 import projection as P
for i in range(3):
    t0 = time.perf_counter(); out = P._project_pipelined(zh, dd, "auto", dev); dt = time.perf_counter() - t0
    print(f"pipelined only {i}: {dt*1e3:.2f} ms")
t0 = time.perf_counter(); a = out[0].numpy(); b = out[2].numpy(); print("numpy views ms", (time.perf_counter()-t0)*1e3)
