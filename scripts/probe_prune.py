"""Tile-pruning potential of the split screen on the coherent IPG dictionaries (cfg2 / cfg4).

For an atom ordering, every BT-atom tile t gets a centroid c_t and radius r_t = max ||d_j - c_t||.
Re<z, d_j> <= Re<z, c_t> + ||z|| r_t  (Cauchy-Schwarz), so a tile whose bound is below a voxel's
lower bound lb_v cannot hold that voxel's argmax.  Reports the fraction of (voxel, tile) pairs and
of (voxel tile, atom tile) pairs still needed, for several atom / voxel orders and lower bounds.

    python scripts/probe_prune.py cfg4|cfg2
"""
import sys
import time

import numpy as np
import torch

from paper_1810_01967_b200 import workloads
from paper_1810_01967_b200.forward_model import SamplingPattern, make_cartesian_operator
from paper_1810_01967_b200.solver import SolverConfig, solve_compressed

which = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
dev = torch.device("cuda:0")
cfg = getattr(workloads, f"make_{which}")(device=dev)
s = cfg.cdict.s
BT = 128 if s <= 10 else 64
VT = 128
A = make_cartesian_operator(SamplingPattern(cfg.pattern, cfg.spatial_shape), device=dev)
caps = {}
want = {1, 2, 5, 10, 20, 30}


def hook(k, st, mu, shrinks, fixed):
    if k in want:
        caps[k] = (st.Z.clone(), st.idx.clone(), st.idx_n.clone())


conf = SolverConfig(mode="blip_exact", max_iters=30 if which == "cfg2" else 20, zeta=2.0,
                    compressed=s)
solve_compressed(cfg.Y, A, cfg.cdict, None, conf, on_iter=hook)
atoms = torch.from_numpy(cfg.cdict.atoms_compressed).to(dev)            # (D, s) c128
D = atoms.shape[0]
table = np.asarray(cfg.cdict.parent.lookup_table)


def real2(x):
    return torch.cat([x.real, x.imag], dim=1)


def morton_order():
    ids = [np.unique(table[:, c], return_inverse=True)[1] for c in range(3)]
    code = np.zeros(D, dtype=np.int64)
    for b in range(8):
        for c in range(3):
            code |= ((ids[c] >> b) & 1).astype(np.int64) << (3 * b + c)
    return np.argsort(code, kind="stable")


def bisect_order():
    """Recursive split on the widest principal direction (kd-tree order of the real 2s rows)."""
    X = real2(atoms).cpu().numpy()
    order = np.arange(D)
    out = []
    stack = [order]
    while stack:
        ix = stack.pop()
        if len(ix) <= BT:
            out.append(ix)
            continue
        P = X[ix] - X[ix].mean(0)
        # top principal direction by a few power iterations
        v = P[np.argmax((P * P).sum(1))].copy()
        for _ in range(8):
            v = P.T @ (P @ v)
            v /= np.linalg.norm(v) + 1e-30
        proj = P @ v
        # split at a multiple of BT so tiles stay full
        half = ((len(ix) // BT + 1) // 2) * BT
        srt = ix[np.argsort(proj, kind="stable")]
        stack.append(srt[half:])
        stack.append(srt[:half])
    return np.concatenate(out)


orders = {"bisect": bisect_order()}


def tiles(order):
    a = atoms[torch.from_numpy(order).to(dev)]
    T = -(-D // BT)
    pad = T * BT - D
    ar = real2(a)
    c = torch.zeros((T, 2 * s), dtype=torch.float64, device=dev)
    r = torch.zeros(T, dtype=torch.float64, device=dev)
    for t in range(T):
        blk = ar[t * BT:min(D, (t + 1) * BT)]
        c[t] = blk.mean(0)
        r[t] = torch.linalg.vector_norm(blk - c[t], dim=1).max()
    return c, r, pad


for oname, order in orders.items():
    c, r, _ = tiles(order)
    pos = torch.empty(D, dtype=torch.int64, device=dev)
    pos[torch.from_numpy(order).to(dev)] = torch.arange(D, device=dev)
    rq = torch.quantile(r.float(), torch.tensor([0.1, 0.5, 0.9], device=dev)).tolist()
    print(f"[{which}] order={oname} tiles={c.shape[0]} radius p10/p50/p90 = "
          f"{rq[0]:.3f}/{rq[1]:.3f}/{rq[2]:.3f}", flush=True)
    for k, (Z, hint, new) in sorted(caps.items()):
        z = Z.to(torch.complex128)
        zr = real2(z)
        zn = torch.linalg.vector_norm(zr, dim=1)
        s_hint = (zr * real2(atoms[hint.long()])).sum(1)
        s_best = (zr * real2(atoms[new.long()])).sum(1)
        n = z.shape[0]
        res = {}
        for lbname, lb in (("hint", s_hint), ("best", s_best)):
            lb = lb - 1e-6 * zn                                  # rounding margin
            for vname in ("natural", "sort_hint"):
                if vname == "natural":
                    perm = torch.arange(n, device=dev)
                else:
                    perm = torch.argsort(pos[hint.long()], stable=True)
                need_pairs = 0
                need_tiles = 0
                nvt = -(-n // VT)
                for v0 in range(0, nvt, 4096):
                    v1 = min(nvt, v0 + 4096)
                    rows = perm[v0 * VT:min(n, v1 * VT)]
                    U = zr[rows] @ c.T + zn[rows, None] * r[None, :]
                    need = U >= lb[rows, None]
                    need_pairs += int(need.sum())
                    m = need.shape[0]
                    padr = (-m) % VT
                    if padr:
                        need = torch.cat([need, torch.zeros((padr, need.shape[1]), dtype=torch.bool,
                                                            device=dev)])
                    need_tiles += int(need.view(-1, VT, need.shape[1]).any(1).sum())
                res[(lbname, vname)] = (need_pairs / (n * c.shape[0]),
                                        need_tiles / (nvt * c.shape[0]))
        line = "  ".join(f"{lb}/{vn}: pairs {a:.3f} tiles {b:.3f}" for (lb, vn), (a, b) in res.items())
        print(f"   k={k:2d}  {line}", flush=True)


# ---- voxel order variants: (bucket of lb/||z||, hint position)
print(f"[{which}] voxel orders with lb/||z|| buckets (bisect order, per-voxel bounds, lb = hint)")
c, r, _ = tiles(orders["bisect"])
pos = torch.empty(D, dtype=torch.int64, device=dev)
pos[torch.from_numpy(orders["bisect"]).to(dev)] = torch.arange(D, device=dev)
schemes = {"pos": [], "b2(.5)": [0.5], "b4": [0.5, 0.8, 0.95], "b8": [0.3, 0.5, 0.7, 0.8, 0.9, 0.95, 0.98]}
for k, (Z, hint, new) in sorted(caps.items()):
    z = Z.to(torch.complex128)
    zr = real2(z)
    zn = torch.linalg.vector_norm(zr, dim=1)
    lb = (zr * real2(atoms[hint.long()])).sum(1)
    ratio = lb / zn.clamp_min(1e-300)
    n = z.shape[0]
    nvt = -(-n // VT)
    out = []
    for name, th in schemes.items():
        bucket = torch.zeros(n, dtype=torch.int64, device=dev)
        for t in th:
            bucket += (ratio < t).long()
        key = bucket * (D + 1) + pos[hint.long()]
        perm = torch.argsort(key, stable=True)
        need_tiles = 0
        for v0 in range(0, nvt, 4096):
            v1 = min(nvt, v0 + 4096)
            rows = perm[v0 * VT:min(n, v1 * VT)]
            U = zr[rows] @ c.T + zn[rows, None] * r[None, :]
            need = U >= (lb - 1e-6 * zn)[rows, None]
            m = need.shape[0]
            padr = (-m) % VT
            if padr:
                need = torch.cat([need, torch.zeros((padr, need.shape[1]), dtype=torch.bool, device=dev)])
            need_tiles += int(need.view(-1, VT, need.shape[1]).any(1).sum())
        out.append(f"{name}: {need_tiles / (nvt * c.shape[0]):.3f}")
    q = torch.quantile(ratio.float(), torch.tensor([0.05, 0.25, 0.5, 0.75], device=dev)).tolist()
    print(f"   k={k:2d}  " + "  ".join(out) + "   ratio q05/25/50/75 " + "/".join(f"{x:.2f}" for x in q), flush=True)
