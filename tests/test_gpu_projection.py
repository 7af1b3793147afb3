"""GPU parity of the exact cone projection against the CPU oracle (and golden vectors).

Gate: indices bit-exact vs the fp64 oracle on identical inputs except
documented near-ties ((s1 - s2) / |s1| < 1e-5); gammas / projected within 1e-4
relative (we assert far tighter: the winner is rescored in fp64 on the caller's
own data, so complex128 inputs match to ~1e-12).
"""

import numpy as np
import pytest

from oracle import projection as orc

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _pkg():
    import paper_1810_01967_b200 as p
    return p


def random_atoms(rng, d, L):
    raw = rng.standard_normal((d, L)) + 1j * rng.standard_normal((d, L))
    return raw / np.linalg.norm(raw, axis=1)[:, None]


def assert_parity(Z, atoms, res, gamma_rtol=1e-12, allow_ties=True):
    ref = orc.project_cone_exact(Z, atoms)
    i1, s1, s2 = orc.top2(np.asarray(Z, dtype=complex), atoms)
    idx = np.asarray(res.indices)
    diff = idx != ref.indices
    if allow_ties:
        ties = orc.near_tie_mask(s1, s2)
        bad = diff & ~ties
    else:
        bad = diff
    assert not bad.any(), f"{bad.sum()} non-near-tie index mismatches (of {len(idx)})"
    same = ~diff
    g = np.asarray(res.gammas)
    denom = max(np.linalg.norm(ref.gammas[same]), 1e-300)
    assert np.linalg.norm(g[same] - ref.gammas[same]) / denom <= gamma_rtol
    P = np.asarray(res.projected)
    pd = max(np.linalg.norm(ref.projected[same]), 1e-300)
    assert np.linalg.norm(P[same] - ref.projected[same]) / pd <= max(gamma_rtol, 1e-15)
    return diff.sum()


def _f16_mma_emulation(zh, ah, kp):
    """fp16 tcgen05 accumulation model: each K=16 block's sum is added to the fp16 accumulator
    with ONE round-to-nearest-even (scripts/probe_f16acc.cu); the hardware's internal sum is
    exact up to a finite-width alignment (covered by the 2^-19 slack of the window)."""
    acc = np.zeros((zh.shape[0], ah.shape[0]), dtype=np.float16)
    peak = np.zeros(acc.shape)
    for k0 in range(0, kp, 16):
        part = zh[:, k0:k0 + 16].astype(np.float64) @ ah[:, k0:k0 + 16].astype(np.float64).T
        acc = (acc.astype(np.float64) + part).astype(np.float16)
        peak = np.maximum(peak, np.abs(acc.astype(np.float64)))
    return acc.astype(np.float64), peak


def test_tc_debug_scores_match_f16_emulation():
    """Raw tcgen05 scores == bit-exact emulation of the fp16 MMA on the scaled fp16 operands
    (descriptors, swizzled tiles, TMEM A layout, .pack::16b read-back, accumulation model)."""
    import ctypes
    p = _pkg()
    from paper_1810_01967_b200 import _lib
    from paper_1810_01967_b200.device import workspace
    rng = np.random.default_rng(5)
    for s in (10, 16, 20):
        kp = 32 if 2 * s < 32 else 64
        atoms = random_atoms(rng, 300, s)
        Z = rng.standard_normal((300, s)) + 1j * rng.standard_normal((300, s))
        Z[:40] *= np.exp(rng.uniform(-30, 30, size=(40, 1)))   # wide dynamic range of voxels
        dd = p.device_dictionary(atoms)
        sd = dd.bounds()["scale_d"]
        assert sd == 2.0 ** -np.frexp(dd.bounds()["dmax"])[1]
        lib = _lib.load()
        zt = torch.from_numpy(Z).cuda()
        wsb = lib.cbb_project_workspace_bytes(300, s)
        ws = workspace(wsb, dd.device, "project")
        _lib.check(lib.cbb_project_prologue(zt.data_ptr(), 1, 300, ctypes.byref(dd.view),
                                            ws.data_ptr(), wsb, _lib.stream_ptr()), "prologue")
        out = torch.empty((128, 128), dtype=torch.float32, device="cuda")
        sv = 2.0 ** (13 - np.frexp(np.linalg.norm(Z, axis=1))[1])
        zr = np.zeros((384, kp))
        zr[:300, :2 * s] = np.concatenate([Z.real, Z.imag], 1) * sv[:, None]
        ar = np.zeros((384, kp))
        ar[:300, :2 * s] = np.concatenate([atoms.real, atoms.imag], 1) * sd
        zr[:300, 2 * s] = 1.0         # sentinel column right after the data: voxel rows 1,
        ar[300:, 2 * s] = -65504.0    # zero-padded atom rows of the last tile -65504
        zh, ah = zr.astype(np.float16), ar.astype(np.float16)
        assert np.all(np.isfinite(zh)) and np.abs(zh).max() < 2.0 ** 13
        for at, bt in ((0, 0), (1, 2), (2, 1)):
            _lib.check(lib.cbb_debug_tc_scores(ws.data_ptr(), ctypes.byref(dd.view), at, bt,
                                               out.data_ptr(), _lib.stream_ptr()), "dbg")
            got = out.cpu().numpy().astype(np.float64)
            exp, peak = _f16_mma_emulation(zh[at * 128:(at + 1) * 128],
                                           ah[bt * 128:(bt + 1) * 128], kp)
            # bit-exact except rare 1-ulp flips where the tensor core's internal (aligned,
            # finite-width) K=16 sum is not exact under heavy cancellation
            # (a flip in an intermediate accumulator propagates: compare with its ulp)
            ulp = (kp // 16) * 2.0 ** (np.floor(np.log2(np.maximum(peak, 2.0 ** -14))) - 10)
            flips = got != exp
            assert flips.mean() < 1e-3, (s, at, bt, flips.sum())
            assert np.all(np.abs(got - exp)[flips] <= ulp[flips]), (s, at, bt)
            # and the accumulation error stays inside the certified acc term
            z64 = zh[at * 128:(at + 1) * 128].astype(np.float64)
            a64 = ah[bt * 128:(bt + 1) * 128].astype(np.float64)
            nks = (2 * s + 1 + 15) // 16    # K-steps that carry data (the production kernel)
            bound = nks * 2.0 ** -11 * 1.002 * np.outer(np.linalg.norm(z64, axis=1),
                                                             np.linalg.norm(a64, axis=1))
            assert np.all(np.abs(got - z64 @ a64.T) <= bound + 2.0 ** -24)


@pytest.mark.parametrize("algo", ["tcgen05", "ffma", "exhaustive"])
@pytest.mark.parametrize("s", [2, 6, 10, 16, 20, 32])
def test_random_parity(algo, s):
    p = _pkg()
    rng = np.random.default_rng(100 + s)
    atoms = random_atoms(rng, 1000, s)
    Z = rng.standard_normal((777, s)) + 1j * rng.standard_normal((777, s))
    if algo == "tcgen05" and 2 * s >= 64:   # no spare sentinel column in K = 64
        from paper_1810_01967_b200._lib import NativeError
        with pytest.raises(NativeError, match="status 3"):
            p.project_cone_exact(Z, atoms, algo=algo)
        return
    res = p.project_cone_exact(Z, atoms, algo=algo)
    assert res.indices.dtype == np.int64 and res.gammas.dtype == np.float64
    assert res.projected.dtype == np.complex128 and res.cost == 777 * 1000
    assert_parity(Z, atoms, res)


def test_large_dim_uses_exhaustive():
    p = _pkg()
    rng = np.random.default_rng(7)
    atoms = random_atoms(rng, 300, 40)  # 2s = 80 > 64: no tensor-core path
    Z = rng.standard_normal((50, 40)) + 1j * rng.standard_normal((50, 40))
    assert_parity(Z, atoms, p.project_cone_exact(Z, atoms))


def test_reference_kats():
    """test_projection.py:34-81 known answers."""
    p = _pkg()
    rng = np.random.default_rng(70)
    atoms = random_atoms(rng, 12, 8)
    Z = np.zeros((1, 8), dtype=complex)
    Z[0] = 2.5 * atoms[7]
    r = p.project_cone_exact(Z, atoms)
    assert r.indices[0] == 7
    assert r.gammas[0] == pytest.approx(2.5, rel=1e-12)
    np.testing.assert_allclose(r.projected, Z, atol=1e-12)
    a1 = random_atoms(np.random.default_rng(71), 1, 8)
    r = p.project_cone_exact(-a1, a1)
    assert r.gammas[0] == 0.0 and np.all(r.projected == 0)
    atoms = random_atoms(np.random.default_rng(75), 5, 6)
    with pytest.raises(ValueError, match="dimension mismatch"):
        p.project_cone_exact(np.zeros((2, 7), dtype=complex), atoms)


def test_ties_zero_rows_and_duplicates():
    p = _pkg()
    rng = np.random.default_rng(9)
    base = random_atoms(rng, 400, 10)
    atoms = np.concatenate([base, base[:50]])      # exact duplicate atoms: ties -> lowest index
    Z = rng.standard_normal((300, 10)) + 1j * rng.standard_normal((300, 10))
    Z[::7] = 0.0                                   # all-zero rows -> index 0, gamma 0
    Z[5] = 3.0 * atoms[410]                        # duplicate of atom 10 -> must pick 10
    for algo in ("tcgen05", "ffma", "exhaustive"):
        r = p.project_cone_exact(Z, atoms, algo=algo)
        assert r.indices[5] == 10
        assert np.all(r.indices[::7] == 0) and np.all(r.gammas[::7] == 0.0)
        assert_parity(Z, atoms, r, allow_ties=False)


def test_cfg1_subsample_parity_and_complex64():
    p = _pkg()
    from paper_1810_01967_b200.workloads import cone_voxels, random_atoms as ra
    atoms = ra(1 << 15, 10, seed=0)
    Z, gen = cone_voxels(atoms, 5000, seed=1, dtype=np.complex64)
    for algo in ("tcgen05", "ffma"):
        r = p.project_cone_exact(Z, atoms, algo=algo)
        assert_parity(Z.astype(np.complex128), atoms, r, allow_ties=False)


def test_coherent_dictionary_overflow_path():
    """MRF-like coherent atoms: many candidates inside the fp16 window -> exhaustive rescans."""
    p = _pkg()
    from paper_1810_01967_b200.workloads import cfg0_dictionary
    from paper_1810_01967_b200 import svd_compress
    from paper_1810_01967_b200.projection import overflow_count
    dct = cfg0_dictionary(L=200, n_t1=30, n_t2=30)
    cd = svd_compress(dct, 10)
    rng = np.random.default_rng(11)
    j = rng.integers(cd.d, size=2000)
    Z = (0.5 + rng.random(2000))[:, None] * cd.atoms_compressed[j]
    Z = Z + 0.01 * (rng.standard_normal(Z.shape) + 1j * rng.standard_normal(Z.shape))
    r = p.project_cone_exact(Z, cd, algo="tcgen05")
    ov = overflow_count(2000, 10)
    assert_parity(Z, cd.atoms_compressed, r)
    print("overflowed voxels:", ov)


def test_device_tensor_roundtrip():
    p = _pkg()
    rng = np.random.default_rng(12)
    atoms = random_atoms(rng, 513, 10)
    Z = rng.standard_normal((1000, 10)) + 1j * rng.standard_normal((1000, 10))
    r = p.project_cone_exact(torch.from_numpy(Z).cuda(), atoms)
    assert r.indices.is_cuda and r.projected.is_cuda
    rh = p.project_cone_exact(Z, atoms)
    np.testing.assert_array_equal(r.indices.cpu().numpy(), rh.indices)
    np.testing.assert_array_equal(r.gammas.cpu().numpy(), rh.gammas)


def test_pinned_pipelined_path_matches_device_path():
    """numpy + pinned host buffers take the chunked H2D/compute/D2H pipeline."""
    p = _pkg()
    from paper_1810_01967_b200.device import pinned_empty
    from paper_1810_01967_b200.workloads import cone_voxels, random_atoms as ra
    atoms = ra(4096, 10, seed=3)
    Z, _ = cone_voxels(atoms, 300_000, seed=4)
    Zp = pinned_empty(Z.shape, np.complex128)
    Zp[:] = Z
    r_pipe = p.project_cone_exact(Zp, atoms)
    r_dev = p.project_cone_exact(torch.from_numpy(Z).cuda(), atoms)
    np.testing.assert_array_equal(r_pipe.indices, r_dev.indices.cpu().numpy())
    np.testing.assert_array_equal(r_pipe.gammas, r_dev.gammas.cpu().numpy())
    np.testing.assert_array_equal(r_pipe.projected, r_dev.projected.cpu().numpy())
    sub = slice(0, 2000)
    assert_parity(Z[sub], atoms, type(r_pipe)(r_pipe.indices[sub], r_pipe.gammas[sub],
                                               r_pipe.projected[sub], 0), allow_ties=False)
