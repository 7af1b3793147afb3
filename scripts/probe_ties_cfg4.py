"""How many atoms lie within a window of the fp64 max for the cfg4 IPG's projection inputs
(coherent off-resonance dictionary): windows relative to ||z|| max||d||."""
import numpy as np
import torch

from paper_1810_01967_b200 import workloads
from paper_1810_01967_b200.forward_model import SamplingPattern, make_cartesian_operator
from paper_1810_01967_b200.solver import SolverConfig, _solve_core

dev = torch.device("cuda:0")
cfg = workloads.make_cfg4(device=dev)
A = make_cartesian_operator(SamplingPattern(cfg.pattern, cfg.spatial_shape), device=dev)
D = torch.from_numpy(cfg.cdict.atoms_compressed).to(dev)            # (d, s) c128
dmax = float(torch.linalg.vector_norm(D, dim=1).max())
rng = np.random.default_rng(0)
for iters in (1, 5, 15):
    conf = SolverConfig(mode="blip_exact", max_iters=iters, zeta=2.0, compressed=10)
    st, tr = _solve_core(cfg.Y, A, cfg.cdict, None, conf, None, cfg.cdict.basis,
                         return_device=True)
    sel = torch.from_numpy(rng.choice(st.n, 4096, replace=False)).to(dev)
    Z = st.Z[sel].to(torch.complex128)
    S = (Z @ D.conj().T).real                                          # (4096, d)
    mx = S.max(dim=1).values
    nz = torch.linalg.vector_norm(Z, dim=1) * dmax
    inside = torch.from_numpy(cfg.labels > 0).to(dev)[sel]
    out = {}
    for name, rel in (("2^-8", 2.0 ** -8), ("2^-12", 2.0 ** -12), ("2^-16", 2.0 ** -16),
                      ("2.4e-5", 2.4e-5), ("2^-20", 2.0 ** -20)):
        cnt = (S >= (mx - rel * nz)[:, None]).sum(dim=1).float()
        out[name] = (float(cnt[inside].median()), float(cnt[~inside].median()),
                     float(cnt.mean()), float(cnt.max()))
    print(f"after {iters} iters: (median inside, median background, mean, max) atoms in window:",
          out, flush=True)
    # warm-start quality: the hint (idx of the last accepted iterate) vs the max for this Z
    hint = st.idx[sel].long()
    sh = S.gather(1, hint[:, None])[:, 0]
    gap = ((mx - sh) / nz).cpu().numpy()
    print("   hint gap (max - score(hint)) / |z||d| quantiles 10/50/90/99%:",
          np.quantile(gap, [0.1, 0.5, 0.9, 0.99]), " gap==0 fraction", float((gap == 0).mean()),
          flush=True)
    del st
    torch.cuda.empty_cache()
