"""The reference's solver known-answer tests, ported to the B200 solver (device IPG loop).

Ported from the reference's ``tests/test_solver.py`` (the classes and line ranges are cited per
test) with the reference's own problem generators restated through the package's public
types.  These exercise the device loop's branches: weights (``cbb_residual`` with w), the fixed
step, the carried step policy, the fixed point (||dX||^2 == 0), the zero denominator, the kappa
rescale, compressed / uncompressed equivalence and Gaussian recovery.  Also: non-finite voxels
follow ``np.argmax`` (first NaN wins) and the drop-in monkey patch of the reference's own solve
loop (``coverblip.solver.project_cone_exact``) when the reference package is installed.
"""

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def manifold_dictionary(L, n_t1=4, n_t2=3, n_b0=4):
    """test_solver.py:29-35."""
    from paper_1810_01967_b200.dictionary import ParameterGrid, generate_fingerprints
    grid = ParameterGrid(t1_values=np.linspace(300.0, 2000.0, n_t1),
                         t2_values=np.linspace(40.0, 250.0, n_t2),
                         b0_values=np.linspace(-60.0, 60.0, n_b0))
    return generate_fingerprints(grid, tr_ms=10.0, L=L)


def on_model_image(rng, dct, n):
    """test_solver.py:38-41."""
    idx = rng.integers(dct.d, size=n)
    pd = 0.5 + rng.random(n)
    return pd[:, None] * dct.atoms[idx], idx, pd


def assert_strictly_decreasing(trace, fp32_rel=1e-6):
    """test_solver.py:44-47; the complex64 device state can stall at convergence within
    fp32 rounding of the fidelity (the reference's fp64 loop stops at rel_tol = 1e-6)."""
    f = trace.fidelities()
    for a, b in zip(f, f[1:]):
        assert b < a * (1 + fp32_rel), (a, b)


def rank_two_dictionary(d, L, seed):
    """test_solver.py:218-229."""
    from paper_1810_01967_b200.dictionary import Dictionary
    rng = np.random.default_rng(seed)
    u = rng.standard_normal(L) + 1j * rng.standard_normal(L)
    v = rng.standard_normal(L) + 1j * rng.standard_normal(L)
    coeffs = rng.standard_normal((d, 2))
    raw = coeffs[:, 0:1] * u + coeffs[:, 1:2] * v
    norms = np.linalg.norm(raw, axis=1)
    lookup = np.column_stack([np.arange(d) + 100.0, np.arange(d) + 10.0, np.arange(d) * 1.0])
    return Dictionary(atoms=raw / norms[:, None], norms=norms, lookup_table=lookup, tr_ms=10.0,
                      L=L)


def _ops():
    from paper_1810_01967_b200 import forward_model as fm
    return fm


def test_gaussian_near_exact_recovery():
    """test_solver.py:87-102 (blip_exact: the B200 projection is exact)."""
    from paper_1810_01967_b200.solver import SolverConfig, solve
    fm = _ops()
    rng = np.random.default_rng(83)
    L, n, m = 32, 64, 32
    dct = manifold_dictionary(L, 8, 4, 8)
    assert dct.d == 256
    A = fm.make_gaussian_operator(n=n, m=m, L=L, seed=84)
    X0, _, _ = on_model_image(rng, dct, n)
    X, maps, gammas, trace = solve(A.apply(X0), A, dct, None, SolverConfig(mode="blip_exact"),
                                   gt=X0)
    assert_strictly_decreasing(trace)
    assert np.linalg.norm(X - X0) / np.linalg.norm(X0) < 1e-4
    assert trace.iterations <= 50


def test_monotone_with_noise():
    """test_solver.py:104-118."""
    from paper_1810_01967_b200.solver import SolverConfig, solve
    fm = _ops()
    rng = np.random.default_rng(85)
    L = 16
    dct = manifold_dictionary(L, 5, 3, 5)
    A = fm.make_gaussian_operator(n=24, m=12, L=L, seed=86)
    X0, _, _ = on_model_image(rng, dct, 24)
    Y = A.apply(X0)
    noise = rng.standard_normal(Y.shape) + 1j * rng.standard_normal(Y.shape)
    Y = Y + noise * (0.01 * np.linalg.norm(Y) / np.linalg.norm(noise))
    _, _, _, trace = solve(Y, A, dct, None, SolverConfig(mode="blip_exact"))
    assert_strictly_decreasing(trace)


def test_device_loop_fixed_point():
    """test_solver.py:144-160 through the device loop: basis-vector atoms and measurements whose
    only misfit is imaginary (invisible to Re<z, d>) make the second iteration's projection
    reproduce the iterate bit for bit: ||dX||^2 == 0 (fixed-point branch) ends the loop."""
    from paper_1810_01967_b200.dictionary import Dictionary
    from paper_1810_01967_b200.solver import SolverConfig, solve
    fm = _ops()
    rng = np.random.default_rng(110)
    A = fm.make_cartesian_operator(fm.make_epi_pattern((4, 4), 4, 8), identity_transform=True)
    eye = Dictionary(atoms=np.eye(8, dtype=complex), norms=np.ones(8),
                     lookup_table=np.column_stack([np.arange(8.0)] * 3), tr_ms=10.0, L=8)
    idx = rng.integers(8, size=16)
    pd = 1.0 + rng.integers(8, size=16) / 8.0          # exact in fp32
    X0 = pd[:, None] * eye.atoms[idx]
    Y = A.apply(X0) + 1j * 0.25 * rng.integers(-4, 5, size=(16, 8))
    seen = []
    X, maps, gam, trace = solve(Y, A, eye, None,
                                SolverConfig(mode="blip_exact", mu_init=1.0, max_iters=10),
                                on_iter=lambda k, st, mu, sh, fixed: seen.append((k, fixed)))
    assert seen[-1] == (2, True), seen               # iteration 2 hit nd == 0
    assert trace.iterations == 1                     # the fixed point is not a recorded step
    np.testing.assert_array_equal(X, X0)
    np.testing.assert_array_equal(maps.t1, idx.astype(float))


def test_zero_denominator_and_fixed_point_step_rule():
    """test_solver.py:144-171: the step rule (B200 projection) accepts mu on a zero
    denominator and reports the fixed point without shrinking."""
    from paper_1810_01967_b200.projection import project_cone_exact
    from paper_1810_01967_b200.solver import step_shrinkage
    fm = _ops()
    rng = np.random.default_rng(87)
    dct = manifold_dictionary(8)
    A = fm.make_cartesian_operator(fm.make_epi_pattern((4, 4), 4, 8), identity_transform=True)
    X0, _, _ = on_model_image(rng, dct, 16)
    Y = A.apply(X0)
    X = np.zeros_like(X0)
    G = A.adjoint(A.apply(X) - Y)
    mu, proj, shrinks, fixed = step_shrinkage(X, G, 4.0, lambda Z: project_cone_exact(Z, dct),
                                              lambda dX: np.zeros_like(dX), zeta=2.0,
                                              max_shrink=60)
    assert mu == 4.0 and shrinks == 0 and not fixed

    class BasisDict:
        atoms = np.eye(8, dtype=complex)

    idx = rng.integers(8, size=16)
    Xb = (0.5 + rng.random(16))[:, None] * BasisDict.atoms[idx]
    mu, proj, shrinks, fixed = step_shrinkage(Xb, np.zeros_like(Xb), 4.0,
                                              lambda Z: project_cone_exact(Z, BasisDict()),
                                              A.apply, zeta=2.0, max_shrink=60)
    assert fixed and shrinks == 0


def test_kappa_rescale_never_worsens_fidelity():
    """test_solver.py:200-212."""
    from paper_1810_01967_b200.solver import SolverConfig, solve
    fm = _ops()
    rng = np.random.default_rng(91)
    L = 16
    dct = manifold_dictionary(L, 5, 3, 5)
    A = fm.make_gaussian_operator(n=24, m=8, L=L, seed=92)
    X0, _, _ = on_model_image(rng, dct, 24)
    Y = A.apply(X0)
    _, _, _, trace = solve(Y, A, dct, None, SolverConfig(mode="blip_exact"))
    f = trace.fidelities()
    assert f[0] <= np.linalg.norm(Y)
    assert_strictly_decreasing(trace)


def test_compressed_exact_rank_equivalence():
    """test_solver.py:233-247."""
    from paper_1810_01967_b200.dictionary import svd_compress
    from paper_1810_01967_b200.solver import SolverConfig, solve, solve_compressed
    fm = _ops()
    rng = np.random.default_rng(93)
    dct = rank_two_dictionary(20, 12, 94)
    cdict = svd_compress(dct, 2)
    A = fm.make_gaussian_operator(n=10, m=6, L=12, seed=95)
    X0, _, _ = on_model_image(rng, dct, 10)
    Y = A.apply(X0)
    _, mu_maps, _, _ = solve(Y, A, dct, None, SolverConfig(mode="blip_exact"))
    _, c_maps, _, _ = solve_compressed(Y, A, cdict, None,
                                       SolverConfig(mode="blip_exact", compressed=2))
    np.testing.assert_array_equal(mu_maps.t1, c_maps.t1)
    np.testing.assert_array_equal(mu_maps.t2, c_maps.t2)
    np.testing.assert_array_equal(mu_maps.b0, c_maps.b0)


def test_compressed_full_rank_matches_uncompressed():
    """test_solver.py:249-262 (complex64 device state: 1e-5 instead of 1e-10)."""
    from paper_1810_01967_b200.dictionary import svd_compress
    from paper_1810_01967_b200.solver import SolverConfig, solve, solve_compressed
    fm = _ops()
    rng = np.random.default_rng(96)
    L = 12
    dct = manifold_dictionary(L)
    cdict = svd_compress(dct, L)
    A = fm.make_gaussian_operator(n=10, m=6, L=L, seed=97)
    X0, _, _ = on_model_image(rng, dct, 10)
    Y = A.apply(X0)
    Xu, _, gu, _ = solve(Y, A, dct, None, SolverConfig(mode="blip_exact"))
    Xc, _, gc, _ = solve_compressed(Y, A, cdict, None,
                                    SolverConfig(mode="blip_exact", compressed=L))
    np.testing.assert_allclose(Xc, Xu, atol=1e-5 * np.abs(Xu).max())
    np.testing.assert_allclose(gc, gu, atol=1e-5 * np.abs(gu).max())


def test_more_components_no_worse_fit():
    """test_solver.py:264-277."""
    from paper_1810_01967_b200.dictionary import svd_compress
    from paper_1810_01967_b200.solver import SolverConfig, solve_compressed
    fm = _ops()
    rng = np.random.default_rng(98)
    L = 40
    dct = manifold_dictionary(L, 6, 4, 5)
    A = fm.make_gaussian_operator(n=12, m=8, L=L, seed=99)
    X0, _, _ = on_model_image(rng, dct, 12)
    Y = A.apply(X0)
    fids = {}
    for s in (5, L):
        cdict = svd_compress(dct, s)
        _, _, _, trace = solve_compressed(Y, A, cdict, None,
                                          SolverConfig(mode="blip_exact", compressed=s))
        fids[s] = trace.fidelities()[-1]
    assert fids[L] <= fids[5] * (1 + 1e-6) + 1e-12


def test_weights_all_ones_match_disabled():
    """test_solver.py:333-347: the weighted residual path (cbb_residual with w)."""
    from paper_1810_01967_b200.solver import SolverConfig, solve
    fm = _ops()
    rng = np.random.default_rng(104)
    L = 12
    dct = manifold_dictionary(L)
    p = fm.make_epi_pattern((4, 4), 2, L)
    A_plain = fm.make_cartesian_operator(p)
    A_w = fm.make_cartesian_operator(p, weights=np.ones((p.m, L)))
    X0, _, _ = on_model_image(rng, dct, 16)
    Y = A_plain.apply(X0)
    X1, _, _, t1 = solve(Y, A_plain, dct, None, SolverConfig(mode="blip_exact"))
    X2, _, _, t2 = solve(Y, A_w, dct, None, SolverConfig(mode="blip_exact",
                                                         weights_enabled=True))
    np.testing.assert_allclose(X1, X2, atol=1e-12)
    assert t1.fidelities() == t2.fidelities()


def test_weights_change_the_objective():
    """Non-uniform weights enter the fidelity: sum w |AX - Y|^2 (solver.py:180-190)."""
    from paper_1810_01967_b200.solver import SolverConfig, solve
    fm = _ops()
    rng = np.random.default_rng(114)
    L = 12
    dct = manifold_dictionary(L)
    p = fm.make_epi_pattern((4, 4), 2, L)
    w = 0.5 + rng.random((p.m, L))
    A_w = fm.make_cartesian_operator(p, weights=w)
    X0, _, _ = on_model_image(rng, dct, 16)
    Y = A_w.apply(X0)
    Y = Y + 0.05 * np.linalg.norm(Y) / np.sqrt(Y.size) * rng.standard_normal(Y.shape)
    X, _, _, trace = solve(Y, A_w, dct, None, SolverConfig(mode="blip_exact",
                                                           weights_enabled=True, max_iters=5))
    R = A_w.apply(X) - Y
    assert abs(trace.fidelities()[-1] - np.sqrt(np.sum(w * np.abs(R) ** 2))) <= \
        1e-4 * trace.fidelities()[-1]


def test_fixed_step_no_shrinkage():
    """test_solver.py:349-360."""
    from paper_1810_01967_b200.solver import SolverConfig, solve
    fm = _ops()
    rng = np.random.default_rng(105)
    L = 12
    dct = manifold_dictionary(L)
    A = fm.make_gaussian_operator(n=16, m=12, L=L, seed=106)
    X0, _, _ = on_model_image(rng, dct, 16)
    _, _, _, trace = solve(A.apply(X0), A, dct, None,
                           SolverConfig(mode="blip_exact", fixed_step=0.5))
    assert all(r["shrinks"] == 0 for r in trace.records)
    assert all(r["mu"] == 0.5 for r in trace.records)


def test_carry_over_step_policy():
    """step_policy="carry_over" (solver.py:231-232): each iteration starts from the previous
    iteration's accepted step, so mu never increases along the trace."""
    from paper_1810_01967_b200.solver import SolverConfig, solve
    fm = _ops()
    rng = np.random.default_rng(111)
    L = 16
    dct = manifold_dictionary(L, 5, 3, 5)
    A = fm.make_gaussian_operator(n=24, m=8, L=L, seed=112)
    X0, _, _ = on_model_image(rng, dct, 24)
    Y = A.apply(X0)
    _, _, _, tr = solve(Y, A, dct, None, SolverConfig(mode="blip_exact", step_policy="carry_over",
                                                      max_iters=12))
    mus = [r["mu"] for r in tr.records]
    assert all(b <= a for a, b in zip(mus[1:], mus[2:]))
    assert_strictly_decreasing(tr)


def test_kappa_rejection_and_step_collapse_messages():
    """test_solver.py:192-197 (step-size collapse) and the config errors (solver.py:58-66)."""
    from paper_1810_01967_b200.forward_model import ForwardOperator
    from paper_1810_01967_b200.solver import SolverConfig, SolverError, solve
    fm = _ops()
    rng = np.random.default_rng(87)
    dct = manifold_dictionary(8)
    X0, _, _ = on_model_image(rng, dct, 16)
    big = ForwardOperator(kind="dense_gaussian", n=16, m=16, L=8,
                          matrix=1e6 * np.eye(16, dtype=complex))
    with pytest.raises(SolverError, match="step-size collapse"):
        solve(big.apply(X0), big, dct, None,
              SolverConfig(mode="blip_exact", mu_init=1.0, max_shrink_per_iter=3))
    with pytest.raises(ValueError, match="zeta"):
        SolverConfig(zeta=1.0)


def test_non_finite_voxels_follow_np_argmax():
    """Rows with +-inf components score NaN against some atoms and +-inf against others;
    np.argmax (projection.py:62) returns the first NaN, and gamma = max(NaN, 0) is NaN."""
    import paper_1810_01967_b200 as cb
    from oracle import projection as orc
    rng = np.random.default_rng(12)
    atoms = rng.standard_normal((700, 6)) + 1j * rng.standard_normal((700, 6))
    atoms /= np.linalg.norm(atoms, axis=1)[:, None]
    Z = rng.standard_normal((40, 6)) + 1j * rng.standard_normal((40, 6))
    Z[3, 0] = np.inf + 1j * np.inf           # NaN for atoms whose re / im signs differ
    Z[7, 2] = -np.inf                        # +-inf scores, no NaN
    Z[9, :] = np.nan
    with np.errstate(invalid="ignore", over="ignore"):
        ref = orc.project_cone_exact(Z, atoms)
    for algo in ("auto", "exhaustive", "ffma"):
        got = cb.project_cone_exact(Z, atoms, algo=algo)
        np.testing.assert_array_equal(got.indices, ref.indices, err_msg=algo)
        assert np.isnan(got.gammas[3]) and np.isnan(ref.gammas[3])
        assert np.isnan(got.gammas[9])
        fin = np.isfinite(ref.gammas)
        np.testing.assert_allclose(got.gammas[fin], ref.gammas[fin], rtol=1e-12)


def test_drop_in_reference_solve_loop(monkeypatch):
    """the reference's own solve_compressed with its module-global
    project_cone_exact replaced by the B200 projection (solver.py:22,175) reproduces the
    reference's cfg0 run (golden trace).  Needs the reference package (baseline/_ref)."""
    ref_path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_path, "coverblip")):
        pytest.skip("reference package not installed under baseline/_ref")
    sys.path.insert(0, ref_path)
    try:
        import coverblip.solver as rs
        from coverblip import dictionary as rd
        from coverblip import forward_model as rf
    except Exception as exc:  # pragma: no cover - environment dependent
        pytest.skip(f"reference package not importable: {exc!r}")
    finally:
        sys.path.remove(ref_path)
    import paper_1810_01967_b200 as cb
    from paper_1810_01967_b200 import workloads
    g = np.load(os.path.join(GOLD, "cfg0_reference.npz"))
    cfg = workloads.make_cfg0()
    parent = rd.Dictionary(atoms=cfg.dictionary.atoms, norms=cfg.dictionary.norms,
                           lookup_table=cfg.dictionary.lookup_table, tr_ms=cfg.dictionary.tr_ms,
                           L=cfg.dictionary.L)
    cd = rd.CompressedDictionary(basis=g["basis"], atoms_compressed=g["atoms_c"],
                                 renorm_factors=np.ones(g["atoms_c"].shape[0]), s=10,
                                 parent=parent)
    A = rf.make_cartesian_operator(rf.SamplingPattern(indices=cfg.pattern,
                                                      spatial_shape=cfg.spatial_shape))
    calls = []

    def b200_projection(Z, dictionary):
        calls.append(Z.shape)
        return cb.project_cone_exact(Z, dictionary)

    monkeypatch.setattr(rs, "project_cone_exact", b200_projection)
    X, maps, gam, trace = rs.solve_compressed(
        g["Y"], A, cd, None, rs.SolverConfig(mode="blip_exact", max_iters=20, zeta=2.0,
                                             compressed=10))
    assert calls, "the reference loop did not call the patched projection"
    fid = np.array([r["fidelity"] for r in trace.records])
    assert len(fid) == len(g["fidelity"])
    np.testing.assert_allclose(fid, g["fidelity"], rtol=1e-9)
    np.testing.assert_array_equal([r["shrinks"] for r in trace.records], g["shrinks"])
    np.testing.assert_allclose(gam, g["gammas"], rtol=1e-9, atol=1e-12)
