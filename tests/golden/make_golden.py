"""Freeze golden vectors from the REAL reference (run in the build container only).

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

The reference cannot travel to the GPU box, so its outputs on seeded inputs are
committed here as small .npz fixtures; ``tests/test_oracle_golden.py`` pins the
oracle restatement to them and the GPU parity tests use them directly.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import coverblip  # noqa: E402  (the reference)
from coverblip import forward_model as ref_fm  # noqa: E402
from coverblip import projection as ref_proj  # noqa: E402
from coverblip import solver as ref_solver  # noqa: E402
from coverblip import dictionary as ref_dict  # noqa: E402

from paper_1810_01967_b200 import workloads  # noqa: E402  (input generators only)


class AtomDict:
    def __init__(self, atoms):
        self.atoms = atoms


def rand_atoms(rng, d, L):
    raw = rng.standard_normal((d, L)) + 1j * rng.standard_normal((d, L))
    return raw / np.linalg.norm(raw, axis=1)[:, None]


def projection_cases():
    out = {}
    cases = []
    rng = np.random.default_rng(72)
    a = rand_atoms(rng, 5, 6)
    z = rng.standard_normal((3, 6)) + 1j * rng.standard_normal((3, 6))
    cases.append(("tiny", z, a))
    rng = np.random.default_rng(70)
    a = rand_atoms(rng, 12, 8)
    z = np.zeros((2, 8), dtype=complex)
    z[0] = 2.5 * a[7]
    z[1] = -a[3]
    cases.append(("kat", z, a))
    rng = np.random.default_rng(9)
    base = rand_atoms(rng, 200, 10)
    a = np.concatenate([base, base[:50]])
    z = rng.standard_normal((300, 10)) + 1j * rng.standard_normal((300, 10))
    z[::7] = 0.0
    z[5] = 3.0 * a[210]
    cases.append(("ties", z, a))
    a = workloads.random_atoms(4096, 10, seed=0)
    z, _ = workloads.cone_voxels(a, 512, seed=1, dtype=np.complex64)
    cases.append(("cfg1sub", z.astype(np.complex128), a))
    dct = workloads.cfg0_dictionary(L=200)
    cd = ref_dict.svd_compress(ref_dict.Dictionary(atoms=dct.atoms, norms=dct.norms,
                                                   lookup_table=dct.lookup_table,
                                                   tr_ms=dct.tr_ms, L=dct.L), 10)
    rng = np.random.default_rng(11)
    j = rng.integers(cd.d, size=256)
    z = (0.5 + rng.random(256))[:, None] * cd.atoms_compressed[j]
    z = z + 0.01 * (rng.standard_normal(z.shape) + 1j * rng.standard_normal(z.shape))
    cases.append(("coherent", z, cd.atoms_compressed))
    for name, z, a in cases:
        r = ref_proj.project_cone_exact(z, AtomDict(a))
        out[f"{name}_Z"] = z
        out[f"{name}_atoms"] = a
        out[f"{name}_indices"] = r.indices
        out[f"{name}_gammas"] = r.gammas
        out[f"{name}_projected"] = r.projected
        out[f"{name}_cost"] = np.int64(r.cost)
    out["names"] = np.array([c[0] for c in cases])
    return out


def operator_cases():
    out = {}
    rng = np.random.default_rng(30)
    specs = [("epi8", ref_fm.make_epi_pattern((8, 8), 2, 5).indices, (8, 8)),
             ("full8", ref_fm.make_epi_pattern((8, 8), 8, 3).indices, (8, 8)),
             ("rand64", workloads.random_line_pattern(64, 64, 8, 12, seed=2), (64, 64)),
             ("epi_rect", ref_fm.make_epi_pattern((16, 8), 4, 6).indices, (16, 8))]
    for name, pat, shape in specs:
        P = ref_fm.SamplingPattern(indices=pat, spatial_shape=shape)
        A = ref_fm.make_cartesian_operator(P)
        X = rng.standard_normal((A.n, A.L)) + 1j * rng.standard_normal((A.n, A.L))
        Y = rng.standard_normal((A.m, A.L)) + 1j * rng.standard_normal((A.m, A.L))
        out[f"{name}_pattern"] = pat
        out[f"{name}_shape"] = np.array(shape)
        out[f"{name}_X"] = X
        out[f"{name}_Y"] = Y
        out[f"{name}_AX"] = A.apply(X)
        out[f"{name}_AHY"] = A.adjoint(Y)
    out["names"] = np.array([s[0] for s in specs])
    return out


def solver_small():
    """Compressed exact IPG on a reduced cfg0 through the reference solve_compressed."""
    cfg = workloads.make_cfg0(h=32, w=32, L=60, s=8, lines=6, snr_db=30.0, n_t1=20, n_t2=20)
    dct = cfg.dictionary
    rdict = ref_dict.Dictionary(atoms=dct.atoms, norms=dct.norms, lookup_table=dct.lookup_table,
                                tr_ms=dct.tr_ms, L=dct.L)
    cd = ref_dict.svd_compress(rdict, 8)
    P = ref_fm.SamplingPattern(indices=cfg.pattern, spatial_shape=cfg.spatial_shape)
    A = ref_fm.make_cartesian_operator(P)
    conf = ref_solver.SolverConfig(mode="blip_exact", max_iters=10, zeta=2.0, compressed=8)
    X, maps, gam, trace = ref_solver.solve_compressed(cfg.Y, A, cd, None, conf, gt=cfg.gt)
    rec = trace.records
    return dict(Y=cfg.Y, pattern=cfg.pattern, shape=np.array(cfg.spatial_shape),
                basis=cd.basis, atoms_c=cd.atoms_compressed, lookup=dct.lookup_table,
                X=X, gammas=gam, t1=maps.t1, t2=maps.t2,
                fidelity=np.array([r["fidelity"] for r in rec]),
                mu=np.array([r["mu"] for r in rec]),
                shrinks=np.array([r["shrinks"] for r in rec]),
                nmse=np.array([r["nmse"] for r in rec]))


def coil_maps(shape, c, seed):
    """Smooth complex receive profiles (Gaussian magnitude around c centres, linear phase)."""
    rng = np.random.default_rng(seed)
    h, w = shape
    yy, xx = np.meshgrid(np.arange(h) / h, np.arange(w) / w, indexing="ij")
    maps = []
    for _ in range(c):
        cy, cx = rng.uniform(0, 1, size=2)
        mag = np.exp(-((yy - cy) ** 2 + (xx - cx) ** 2) / 0.3)
        ph = 2 * np.pi * (rng.uniform(-1, 1) * yy + rng.uniform(-1, 1) * xx)
        maps.append((mag * np.exp(1j * ph)).ravel())
    return np.array(maps)


def coil_cases():
    """Multi-coil operator (forward_model.py:123-167 with c > 1), its compressed chain, and a
    small compressed IPG solve with coils through the reference."""
    out = {}
    rng = np.random.default_rng(40)
    shape, c, L, s = (16, 16), 3, 6, 3
    pat = ref_fm.make_epi_pattern(shape, 4, L).indices
    S = coil_maps(shape, c, 41)
    P = ref_fm.SamplingPattern(indices=pat, spatial_shape=shape)
    A = ref_fm.make_cartesian_operator(P, coil_maps=S)
    n = A.n
    X = rng.standard_normal((n, L)) + 1j * rng.standard_normal((n, L))
    Y = rng.standard_normal((c * A.m, L)) + 1j * rng.standard_normal((c * A.m, L))
    V, _ = np.linalg.qr(rng.standard_normal((L, s)) + 1j * rng.standard_normal((L, s)))
    Xc = rng.standard_normal((n, s)) + 1j * rng.standard_normal((n, s))
    out.update(op_pattern=pat, op_shape=np.array(shape), op_coils=S, op_X=X, op_Y=Y,
               op_AX=A.apply(X), op_AHY=A.adjoint(Y), op_V=V, op_Xc=Xc,
               op_AXc=A.apply(Xc @ V.conj().T), op_AHYV=A.adjoint(Y) @ V)
    # small IPG with 2 coils
    cfg = workloads.make_cfg0(h=32, w=32, L=60, s=8, lines=6, snr_db=30.0, n_t1=20, n_t2=20)
    dct = cfg.dictionary
    rdict = ref_dict.Dictionary(atoms=dct.atoms, norms=dct.norms, lookup_table=dct.lookup_table,
                                tr_ms=dct.tr_ms, L=dct.L)
    cd = ref_dict.svd_compress(rdict, 8)
    S2 = coil_maps(cfg.spatial_shape, 2, 42)
    P2 = ref_fm.SamplingPattern(indices=cfg.pattern, spatial_shape=cfg.spatial_shape)
    A2 = ref_fm.make_cartesian_operator(P2, coil_maps=S2)
    clean = A2.apply(cfg.gt)
    noise = rng.standard_normal(clean.shape) + 1j * rng.standard_normal(clean.shape)
    noise *= np.linalg.norm(clean) * 10 ** (-30 / 20) / np.linalg.norm(noise)
    Yc = clean + noise
    conf = ref_solver.SolverConfig(mode="blip_exact", max_iters=8, zeta=2.0, compressed=8)
    Xs, maps, gam, trace = ref_solver.solve_compressed(Yc, A2, cd, None, conf, gt=cfg.gt)
    rec = trace.records
    out.update(ipg_Y=Yc, ipg_pattern=cfg.pattern, ipg_shape=np.array(cfg.spatial_shape),
               ipg_coils=S2, ipg_basis=cd.basis, ipg_atoms_c=cd.atoms_compressed,
               ipg_lookup=dct.lookup_table, ipg_X=Xs, ipg_gammas=gam, ipg_t1=maps.t1,
               ipg_t2=maps.t2, ipg_fidelity=np.array([r["fidelity"] for r in rec]),
               ipg_mu=np.array([r["mu"] for r in rec]),
               ipg_shrinks=np.array([r["shrinks"] for r in rec]))
    return out


def container_files():
    """CBDICT01 / CBMEAS01 / EPI pattern JSON written by the reference's own savers."""
    dct = workloads.cfg0_dictionary(L=12, n_t1=5, n_t2=6, seed=0)
    rdict = ref_dict.Dictionary(atoms=dct.atoms, norms=dct.norms, lookup_table=dct.lookup_table,
                                tr_ms=dct.tr_ms, L=dct.L)
    ref_dict.save_dictionary(rdict, os.path.join(HERE, "small.cbdict"))
    rng = np.random.default_rng(50)
    Y = rng.standard_normal((24, 12)) + 1j * rng.standard_normal((24, 12))
    ref_fm.save_measurements(Y, os.path.join(HERE, "small.cbmeas"))
    ref_fm.save_pattern(ref_fm.make_epi_pattern((8, 8), 2, 12), os.path.join(HERE, "epi.json"))


def cfg0_reference():
    """BASELINE configs[0] through the reference (20 iterations, s = 10)."""
    cfg = workloads.make_cfg0()
    dct = cfg.dictionary
    rdict = ref_dict.Dictionary(atoms=dct.atoms, norms=dct.norms, lookup_table=dct.lookup_table,
                                tr_ms=dct.tr_ms, L=dct.L)
    cd = ref_dict.svd_compress(rdict, 10)
    P = ref_fm.SamplingPattern(indices=cfg.pattern, spatial_shape=cfg.spatial_shape)
    A = ref_fm.make_cartesian_operator(P)
    conf = ref_solver.SolverConfig(mode="blip_exact", max_iters=20, zeta=2.0, compressed=10)
    t0 = time.perf_counter()
    X, maps, gam, trace = ref_solver.solve_compressed(cfg.Y, A, cd, None, conf, gt=cfg.gt)
    secs = time.perf_counter() - t0
    rec = trace.records
    idx = None
    # recover indices from the maps (lookup rows are unique per atom)
    lut = {tuple(r): i for i, r in enumerate(dct.lookup_table)}
    idx = np.array([lut[(a, b, c)] for a, b, c in zip(maps.t1, maps.t2, maps.b0)])
    return dict(Y=cfg.Y, basis=cd.basis, atoms_c=cd.atoms_compressed, indices=idx,
                gammas=gam, fidelity=np.array([r["fidelity"] for r in rec]),
                mu=np.array([r["mu"] for r in rec]),
                shrinks=np.array([r["shrinks"] for r in rec]),
                nmse=np.array([r["nmse"] for r in rec]), seconds=np.float64(secs),
                X_checksum=np.array([np.sum(np.abs(X) ** 2), np.sum(X.real), np.sum(X.imag)]))


def main():
    meta = dict(reference_version=coverblip.__version__, numpy=np.__version__)
    print(meta)
    only = sys.argv[1:]   # e.g. "coils": regenerate just that fixture
    if only:
        if "coils" in only:
            np.savez_compressed(os.path.join(HERE, "coils.npz"), **coil_cases())
        if "containers" in only:
            container_files()
        print("golden fixtures written to", HERE, only)
        return
    np.savez_compressed(os.path.join(HERE, "projection.npz"), **projection_cases())
    np.savez_compressed(os.path.join(HERE, "operator.npz"), **operator_cases())
    np.savez_compressed(os.path.join(HERE, "solver_small.npz"), **solver_small())
    np.savez_compressed(os.path.join(HERE, "cfg0_reference.npz"), **cfg0_reference(),
                        numpy_version=np.array(np.__version__))
    np.savez_compressed(os.path.join(HERE, "coils.npz"), **coil_cases())
    container_files()
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
