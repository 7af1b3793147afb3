"""Seeded synthetic inputs for the BASELINE.json configurations (host numpy).

No public dataset is named by the benchmark; the paper's Brainweb phantom and
in-vivo scans are absent, so every config is generated from fixed seeds
(SURVEY 8d): seed 0 sequence / dictionary, 1 phantom / voxels, 2 masks, 3 noise.

* cfg0  64x64, 4 tissue classes, T=200 IR-bSSFP frames (flip/TR schedule of
        BASELINE configs[0]), T1 50 x T2 60 log grids (T2 < T1, D = 2242),
        Bloch-simulated atoms (``bloch_irbssfp``; the reference has only an
        analytic surrogate), unit-normalised, SVD s = 10; 8 of 64
        random lines per frame; 30 dB noise (reference ``harness.py:145-153`` rule).
* cfg1  N = 2^20 voxels x D = 2^17 random unit atoms, s = 10, voxel = atom x
        PD~U(0.2,1) x random phase + complex noise at 20 dB.
* cfg2  256x256, T=1000 frames (same sequence generator), T1 100 x T2 100 (T2 < T1) x
        dB0 21 values in -50..50 Hz (D = 120,624; SURVEY 8d grid proposal), SVD s = 20,
        multi-shot EPI 16 of 256 lines per frame (``make_epi_pattern``), 30 dB.  Large enough
        that the Bloch simulation, the Gram SVD and the measurement FFT run on the GPU
        (``make_cfg2(device=...)``; same recurrences as the host code, fp64).
* cfg4  256x256x64 ellipsoid phantom (6 shells), T=500, T1 100 x T2 100 x dB0 26 (D = 149,344),
        s = 10, per-frame random Cartesian masks at 1/16 of k-space, 30 dB (``make_cfg4``,
        GPU-generated frame chunk by frame chunk).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .dictionary import CompressedDictionary, Dictionary, svd_compress

__all__ = ["sequence_schedule", "bloch_irbssfp", "cfg0_dictionary", "Cfg0", "make_cfg0",
           "random_atoms", "cone_voxels", "make_cfg1", "random_line_pattern", "make_cfg2",
           "bloch_irbssfp_torch", "make_cfg4"]


def sequence_schedule(L: int, seed: int = 0):
    """alpha_t = 10 + 50 |sin(2 pi t / 250)| + N(0, 1) degrees; TR_t = 10 + U(0, 2) ms."""
    rng = np.random.default_rng(seed)
    t = np.arange(L)
    alpha = 10.0 + 50.0 * np.abs(np.sin(2 * np.pi * t / 250.0)) + rng.normal(0.0, 1.0, L)
    tr = 10.0 + rng.uniform(0.0, 2.0, L)
    return np.deg2rad(alpha), tr


def bloch_irbssfp(params, alpha, tr):
    """Single-isochromat Bloch simulation of an inversion-recovery bSSFP train.

    params (d, 3) = (T1 ms, T2 ms, B0 Hz).  Ideal 180 deg inversion, then per
    frame: RF rotation about x by alpha_t with alternating sign (0/180 phase
    cycling), relaxation + off-resonance precession for TR_t/2, readout
    (demodulated by the RF sign), another TR_t/2.  Returns (d, L) complex128.
    """
    p = np.atleast_2d(np.asarray(params, dtype=float))
    t1, t2, b0 = p[:, 0], p[:, 1], p[:, 2]
    d, L = p.shape[0], len(alpha)
    mx = np.zeros(d)
    my = np.zeros(d)
    mz = -np.ones(d)
    out = np.empty((d, L), dtype=complex)

    def relax(mx, my, mz, tau):
        e1 = np.exp(-tau / t1)
        e2 = np.exp(-tau / t2)
        phi = 2.0 * np.pi * b0 * tau / 1000.0
        c, s = np.cos(phi), np.sin(phi)
        mx, my = e2 * (c * mx - s * my), e2 * (s * mx + c * my)
        mz = e1 * mz + (1.0 - e1)
        return mx, my, mz

    for t in range(L):
        a = alpha[t] * (1.0 if t % 2 == 0 else -1.0)
        ca, sa = np.cos(a), np.sin(a)
        my, mz = ca * my + sa * mz, -sa * my + ca * mz
        mx, my, mz = relax(mx, my, mz, tr[t] / 2.0)
        sign = 1.0 if t % 2 == 0 else -1.0
        out[:, t] = sign * (mx + 1j * my)
        mx, my, mz = relax(mx, my, mz, tr[t] / 2.0)
    return out


def cfg0_dictionary(L: int = 200, n_t1: int = 50, n_t2: int = 60, seed: int = 0,
                    b0_values=(0.0,)) -> Dictionary:
    alpha, tr = sequence_schedule(L, seed)
    t1 = np.geomspace(100.0, 5000.0, n_t1)
    t2 = np.geomspace(20.0, 2000.0, n_t2)
    g1, g2, g3 = np.meshgrid(t1, t2, np.asarray(b0_values, float), indexing="ij")
    triples = np.stack([g1.ravel(), g2.ravel(), g3.ravel()], axis=1)
    triples = triples[triples[:, 1] < triples[:, 0]]
    raw = bloch_irbssfp(triples, alpha, tr)
    norms = np.linalg.norm(raw, axis=1)
    return Dictionary(atoms=raw / norms[:, None], norms=norms, lookup_table=triples,
                      tr_ms=float(np.mean(tr)), L=L)


def random_line_pattern(h: int, w: int, lines: int, L: int, seed: int = 2) -> np.ndarray:
    """Per-frame random Cartesian lines: `lines` of h rows without replacement, all columns.
    Returns (L, lines*w) int64 flat indices row*w + col (forward_model.py:138 order)."""
    rng = np.random.default_rng(seed)
    cols = np.arange(w)
    out = np.empty((L, lines * w), dtype=np.int64)
    for t in range(L):
        rows = np.sort(rng.choice(h, size=lines, replace=False))
        out[t] = (rows[:, None] * w + cols[None, :]).ravel()
    return out


@dataclass
class Cfg0:
    dictionary: Dictionary
    cdict: CompressedDictionary
    pattern: np.ndarray          # (L, m)
    spatial_shape: tuple
    gt: np.ndarray               # (n, L) ground-truth image
    gt_indices: np.ndarray
    pd: np.ndarray
    Y: np.ndarray                # (m, L) reference layout


def make_cfg0(h=64, w=64, L=200, s=10, lines=8, snr_db=30.0, n_t1=50, n_t2=60,
              classes=4) -> Cfg0:
    """BASELINE configs[0] (PR1): the CPU-runnable IPG reconstruction."""
    dct = cfg0_dictionary(L, n_t1, n_t2, seed=0)
    cd = svd_compress(dct, s)
    rng = np.random.default_rng(1)
    seg = np.zeros((h, w), dtype=np.int64)
    b = max(1, min(h, w) // 16)
    rr, cc = np.mgrid[0:h, 0:w]
    inside = (rr >= b) & (rr < h - b) & (cc >= b) & (cc < w - b)
    if classes == 4:
        lab = 1 + 2 * (rr >= h // 2) + (cc >= w // 2)
    else:
        lab = 1 + (rr * classes) // h
    seg[inside] = lab[inside]
    class_atoms = rng.integers(dct.d, size=classes + 1)
    pd = np.where(seg > 0, rng.uniform(0.5, 1.0, size=(h, w)), 0.0).ravel()
    idx = np.where(seg.ravel() > 0, class_atoms[seg.ravel()], 0)
    gt = pd[:, None] * dct.atoms[idx]
    pattern = random_line_pattern(h, w, lines, L, seed=2)
    # Y = A X0 + xi with ||xi|| = ||A X0|| 10^(-snr/20)  (harness.py:145-153)
    n = h * w
    F = np.fft.fft2(gt.reshape(h, w, L), axes=(0, 1), norm="ortho").reshape(n, L)
    Y0 = np.take_along_axis(F, pattern.T, axis=0)
    nrng = np.random.default_rng(3)
    xi = nrng.standard_normal(Y0.shape) + 1j * nrng.standard_normal(Y0.shape)
    xi *= np.linalg.norm(Y0) / np.linalg.norm(xi) * 10 ** (-snr_db / 20.0)
    return Cfg0(dictionary=dct, cdict=cd, pattern=pattern, spatial_shape=(h, w), gt=gt,
                gt_indices=np.where(seg.ravel() > 0, idx, -1), pd=pd, Y=Y0 + xi)


def random_atoms(D: int, s: int, seed: int = 0, dtype=np.complex128) -> np.ndarray:
    """i.i.d. CN(0, 1)^s atoms, unit-normalised (cfg1/cfg3)."""
    rng = np.random.default_rng(seed)
    out = np.empty((D, s), dtype=dtype)
    step = 1 << 18
    for lo in range(0, D, step):
        k = min(step, D - lo)
        a = rng.standard_normal((k, s)) + 1j * rng.standard_normal((k, s))
        a /= np.linalg.norm(a, axis=1)[:, None]
        out[lo:lo + k] = a
    return out


def cone_voxels(atoms: np.ndarray, N: int, seed: int = 1, snr_db: float = 20.0,
                pd_range=(0.2, 1.0), dtype=np.complex128):
    """Each voxel = atom_j x PD x e^{i phi} + complex noise at `snr_db` (per voxel)."""
    rng = np.random.default_rng(seed)
    D, s = atoms.shape
    out = np.empty((N, s), dtype=dtype)
    gen = np.empty(N, dtype=np.int64)
    step = 1 << 18
    for lo in range(0, N, step):
        k = min(step, N - lo)
        j = rng.integers(D, size=k)
        pd = rng.uniform(pd_range[0], pd_range[1], size=k)
        ph = np.exp(1j * rng.uniform(0.0, 2 * np.pi, size=k))
        x = (pd * ph)[:, None] * atoms[j]
        nz = (rng.standard_normal((k, s)) + 1j * rng.standard_normal((k, s))) / np.sqrt(2.0)
        sig = np.linalg.norm(x, axis=1) / np.sqrt(s) * 10 ** (-snr_db / 20.0)
        out[lo:lo + k] = x + nz * sig[:, None]
        gen[lo:lo + k] = j
    return out, gen


def make_cfg1(N: int = 1 << 20, D: int = 1 << 17, s: int = 10, dtype=np.complex64):
    """BASELINE configs[1]: standalone projection microbenchmark inputs."""
    atoms = random_atoms(D, s, seed=0)
    Z, gen = cone_voxels(atoms, N, seed=1, dtype=dtype)
    return atoms, Z, gen


# ---------------------------------------------------------------- cfg2 (GPU-generated)
def bloch_irbssfp_torch(params, alpha, tr, device):
    """``bloch_irbssfp`` on the GPU (torch fp64, identical recurrence).  Returns (d, L)
    complex128 device tensor."""
    import torch
    p = torch.as_tensor(np.atleast_2d(np.asarray(params, dtype=float)), device=device)
    t1, t2, b0 = p[:, 0], p[:, 1], p[:, 2]
    d, L = p.shape[0], len(alpha)
    mx = torch.zeros(d, dtype=torch.float64, device=device)
    my = torch.zeros_like(mx)
    mz = -torch.ones_like(mx)
    out = torch.empty((d, L), dtype=torch.complex128, device=device)
    for t in range(L):
        tau = float(tr[t]) / 2.0
        e1, e2 = torch.exp(-tau / t1), torch.exp(-tau / t2)
        phi = 2.0 * np.pi * b0 * tau / 1000.0
        c, sn = torch.cos(phi), torch.sin(phi)
        a = float(alpha[t]) * (1.0 if t % 2 == 0 else -1.0)
        ca, sa = np.cos(a), np.sin(a)
        my, mz = ca * my + sa * mz, -sa * my + ca * mz
        mx, my = e2 * (c * mx - sn * my), e2 * (sn * mx + c * my)
        mz = e1 * mz + (1.0 - e1)
        sign = 1.0 if t % 2 == 0 else -1.0
        out[:, t] = torch.complex(sign * mx, sign * my)
        mx, my = e2 * (c * mx - sn * my), e2 * (sn * mx + c * my)
        mz = e1 * mz + (1.0 - e1)
    return out


def _offres_dictionary(L, s, n_t1, n_t2, n_b0, dev):
    """T1 x T2 (T2 < T1) x dB0 Bloch IR-bSSFP dictionary simulated on the GPU, unit-normalised,
    compressed by the large-d route of ``dictionary.py:176-183`` (second-moment matrix, eigh,
    top-s, conjugated).  Returns (CompressedDictionary, raw (d, L) complex128 device atoms)."""
    import torch
    alpha, tr = sequence_schedule(L, seed=0)
    t1 = np.geomspace(100.0, 5000.0, n_t1)
    t2 = np.geomspace(50.0, 5000.0, n_t2)
    b0 = np.linspace(-50.0, 50.0, n_b0)
    g1, g2, g3 = np.meshgrid(t1, t2, b0, indexing="ij")
    triples = np.stack([g1.ravel(), g2.ravel(), g3.ravel()], axis=1)
    triples = triples[triples[:, 1] < triples[:, 0]]
    raw = bloch_irbssfp_torch(triples, alpha, tr, dev)
    raw /= torch.linalg.vector_norm(raw, dim=1, keepdim=True)
    gram = (raw.transpose(0, 1) @ raw.conj()).cpu().numpy()
    _, vecs = np.linalg.eigh(gram)
    basis = np.ascontiguousarray(vecs[:, ::-1][:, :s].conj())
    comp = raw @ torch.from_numpy(basis).to(dev)
    factors = torch.linalg.vector_norm(comp, dim=1)
    atoms_c = (comp / factors[:, None]).cpu().numpy()
    parent = Dictionary(atoms=np.zeros((len(triples), 1)), norms=None, lookup_table=triples,
                        tr_ms=float(np.mean(tr)), L=L)
    cd = CompressedDictionary(basis=basis, atoms_compressed=atoms_c,
                              renorm_factors=factors.cpu().numpy(), s=s, parent=parent)
    return cd, raw


@dataclass
class Cfg2:
    cdict: CompressedDictionary
    pattern: np.ndarray          # (L, m)
    spatial_shape: tuple
    Y: np.ndarray                # (m, L) reference layout, complex64
    d: int
    setup_seconds: float


def make_cfg2(h=256, w=256, L=1000, s=20, lines=16, snr_db=30.0, n_t1=100, n_t2=100,
              n_b0=21, classes=6, device=None) -> Cfg2:
    """BASELINE configs[2]: 2-D IPG with an off-resonance dictionary (GPU-generated)."""
    import time

    import torch

    from .forward_model import make_epi_pattern
    t0 = time.perf_counter()
    dev = torch.device(device) if device is not None else torch.device("cuda")
    cd, raw = _offres_dictionary(L, s, n_t1, n_t2, n_b0, dev)
    triples = cd.parent.lookup_table
    # phantom: `classes` horizontal bands inside a background border, one atom per class
    rng = np.random.default_rng(1)
    rr, cc = np.mgrid[0:h, 0:w]
    bd = max(1, min(h, w) // 16)
    inside = (rr >= bd) & (rr < h - bd) & (cc >= bd) & (cc < w - bd)
    lab = np.where(inside, 1 + (rr * classes) // h, 0).ravel()
    class_atoms = rng.integers(len(triples), size=classes + 1)
    pd = np.where(lab > 0, rng.uniform(0.5, 1.0, size=h * w), 0.0)
    idx = torch.as_tensor(class_atoms[lab], device=dev)
    gt = torch.as_tensor(pd, device=dev)[:, None] * raw[idx]          # (n, L) complex128
    del raw
    pat = make_epi_pattern((h, w), lines, L)
    pattern = np.asarray(pat.indices)
    F = torch.fft.fft2(gt.reshape(h, w, L), dim=(0, 1), norm="ortho").reshape(h * w, L)
    del gt
    Y0 = torch.gather(F, 0, torch.as_tensor(pattern.T, device=dev))
    del F
    nrng = np.random.default_rng(3)
    xi = nrng.standard_normal(Y0.shape) + 1j * nrng.standard_normal(Y0.shape)
    Y0 = Y0.cpu().numpy()
    xi *= np.linalg.norm(Y0) / np.linalg.norm(xi) * 10 ** (-snr_db / 20.0)
    Y = (Y0 + xi).astype(np.complex64)
    torch.cuda.empty_cache()
    return Cfg2(cdict=cd, pattern=pattern, spatial_shape=(h, w), Y=Y, d=len(triples),
                setup_seconds=time.perf_counter() - t0)


@dataclass
class Cfg4:
    cdict: CompressedDictionary
    pattern: np.ndarray          # (L, m) sorted flat k-space indices per frame
    spatial_shape: tuple
    Y: np.ndarray                # (m, L) reference layout, complex64
    labels: np.ndarray           # (n,) tissue class per voxel (0 = background)
    class_atoms: np.ndarray      # (classes + 1,) generating atom per class
    d: int
    setup_seconds: float


def make_cfg4(shape=(256, 256, 64), L=500, s=10, undersample=16, snr_db=30.0, n_t1=100,
              n_t2=100, n_b0=26, classes=6, device=None) -> Cfg4:
    """BASELINE configs[4]: 3-D IPG (GPU-generated).  256x256x64 phantom -- an ellipsoid split
    into `classes` concentric shells, PD~U(0.5, 1), zero background -- T=500 frames of the same
    sequence generator, T1 100 x T2 100 (T2 < T1) x dB0 26 atoms (D = 149,344 ~ 1.5e5), SVD s=10,
    per-frame random Cartesian masks of n/16 k-space locations (seed 2), 30 dB noise (seed 3).
    The (n, L) ground truth is never materialised: frames are synthesised, 3-D FFT'd and
    sampled in chunks."""
    import time

    import torch
    t0 = time.perf_counter()
    dev = torch.device(device) if device is not None else torch.device("cuda")
    cd, raw = _offres_dictionary(L, s, n_t1, n_t2, n_b0, dev)
    d = raw.shape[0]
    n = int(np.prod(shape))
    m = n // undersample
    rng = np.random.default_rng(1)
    g = np.meshgrid(*[(np.arange(k) + 0.5) / k * 2.0 - 1.0 for k in shape], indexing="ij")
    rad = np.sqrt(sum(x * x for x in g)).ravel() / 0.9
    lab = np.where(rad < 1.0, 1 + np.minimum((rad * classes).astype(np.int64), classes - 1), 0)
    class_atoms = rng.integers(d, size=classes + 1)
    pd = np.where(lab > 0, rng.uniform(0.5, 1.0, size=n), 0.0)
    pd_t = torch.as_tensor(pd, device=dev)
    idx_t = torch.as_tensor(class_atoms[lab], device=dev)
    gen = torch.Generator(device=dev)
    gen.manual_seed(2)
    pat_t = torch.empty((L, m), dtype=torch.int64, device=dev)
    for t in range(L):
        pat_t[t] = torch.sort(torch.randperm(n, generator=gen, device=dev)[:m]).values
    Yfm = torch.empty((L, m), dtype=torch.complex128, device=dev)
    chunk = 25
    for f0 in range(0, L, chunk):
        f1 = min(L, f0 + chunk)
        frames = (pd_t[None, :] * raw[idx_t, f0:f1].transpose(0, 1)).reshape((f1 - f0,) + shape)
        F = torch.fft.fftn(frames, dim=(1, 2, 3), norm="ortho").reshape(f1 - f0, n)
        Yfm[f0:f1] = torch.gather(F, 1, pat_t[f0:f1])
        del frames, F
    del raw
    gen.manual_seed(3)
    xi = torch.complex(torch.randn((L, m), generator=gen, device=dev, dtype=torch.float64),
                       torch.randn((L, m), generator=gen, device=dev, dtype=torch.float64))
    xi *= torch.linalg.vector_norm(Yfm) / torch.linalg.vector_norm(xi) * 10 ** (-snr_db / 20.0)
    Yfm += xi
    del xi
    Y = Yfm.to(torch.complex64).transpose(0, 1).contiguous().cpu().numpy()
    pattern = pat_t.cpu().numpy()
    del Yfm, pat_t
    torch.cuda.empty_cache()
    return Cfg4(cdict=cd, pattern=pattern, spatial_shape=tuple(shape), Y=Y, labels=lab,
                class_atoms=class_atoms, d=d, setup_seconds=time.perf_counter() - t0)
