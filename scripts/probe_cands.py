"""Development aid: how many 32-atom chunks per voxel fall inside the tcgen05 window (cfg2)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1810_01967_b200 import workloads
from paper_1810_01967_b200.forward_model import SamplingPattern, make_cartesian_operator
cfg = workloads.make_cfg2(device="cuda")
A = make_cartesian_operator(SamplingPattern(cfg.pattern, cfg.spatial_shape))
V = torch.from_numpy(np.ascontiguousarray(cfg.cdict.basis, dtype=np.complex64)).cuda()
Y = torch.from_numpy(np.ascontiguousarray(cfg.Y.T)).cuda()
mu = A.n / A.m
Z = mu * A.fm_adjoint_compressed(Y, V)                       # first IPG projection input
D = torch.from_numpy(cfg.cdict.atoms_compressed.astype(np.complex64)).cuda()
d = D.shape[0]
nch = (d + 31) // 32
rel_win = 2 * (4 * 2.0 ** -11 + 2.0 ** -19 * 4)           # ~ fp16 window / ||z|| ||d||
for label, Zs in (("iter1 input", Z), ("noisy atoms", None)):
    if Zs is None:
        j = torch.randint(d, (8192,), device="cuda")
        Zs = D[j] * (0.5 + torch.rand(8192, 1, device="cuda"))
        Zs = Zs + 0.02 * torch.randn_like(Zs) * Zs.abs().mean()
    cnts, atoms_in = [], []
    for lo in range(0, min(Zs.shape[0], 16384), 2048):
        z = Zs[lo:lo + 2048]
        sc = (z @ D.conj().T).real                           # (b, d)
        smax = sc.max(1, keepdim=True).values
        win = rel_win * torch.linalg.vector_norm(z, dim=1, keepdim=True)
        inw = sc >= smax - win
        pad = nch * 32 - d
        inw = torch.nn.functional.pad(inw, (0, pad))
        ch = inw.view(inw.shape[0], nch, 32).any(2).sum(1)
        cnts.append(ch.cpu()); atoms_in.append(inw.sum(1).cpu())
    c = torch.cat(cnts).numpy(); a = torch.cat(atoms_in).numpy()
    print(label, "chunks in window: median", np.median(c), "p90", np.percentile(c, 90), "max", c.max(),
          "| atoms in window median", np.median(a), "p90", np.percentile(a, 90), "| >48 chunks", np.mean(c > 48))
