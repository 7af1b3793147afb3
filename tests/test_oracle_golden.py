"""Pin the CPU oracle to the REAL reference's outputs (tests/golden, made by make_golden.py).

CPU only (-m "not gpu").  The oracle must reproduce the reference bit-for-bit on the
projection / operator cases (same numpy arithmetic) and its IPG trace on the solver cases.
"""

import os

import numpy as np
import pytest

from oracle import operator as oop
from oracle import projection as orc
from oracle import solver as osv

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLD, name))


@pytest.mark.parametrize("case", ["tiny", "kat", "ties", "cfg1sub", "coherent"])
def test_projection_matches_reference(case):
    g = load("projection.npz")
    r = orc.project_cone_exact(g[f"{case}_Z"], g[f"{case}_atoms"])
    np.testing.assert_array_equal(r.indices, g[f"{case}_indices"])
    np.testing.assert_array_equal(r.gammas, g[f"{case}_gammas"])
    np.testing.assert_array_equal(r.projected, g[f"{case}_projected"])
    assert r.cost == int(g[f"{case}_cost"])


def test_projection_dimension_mismatch():
    with pytest.raises(ValueError, match="dimension mismatch"):
        orc.project_cone_exact(np.zeros((2, 7), complex), np.zeros((5, 6), complex))


def test_top2_consistent_with_argmax():
    g = load("projection.npz")
    Z, A = g["cfg1sub_Z"], g["cfg1sub_atoms"]
    i1, s1, s2 = orc.top2(Z, A)
    np.testing.assert_array_equal(i1, g["cfg1sub_indices"])
    assert np.all(s1 >= s2)


@pytest.mark.parametrize("case", ["epi8", "full8", "rand64", "epi_rect"])
def test_operator_matches_reference(case):
    g = load("operator.npz")
    A = oop.CartesianOperator(g[f"{case}_pattern"], tuple(g[f"{case}_shape"]))
    np.testing.assert_allclose(A.apply(g[f"{case}_X"]), g[f"{case}_AX"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(A.adjoint(g[f"{case}_Y"]), g[f"{case}_AHY"], rtol=0, atol=1e-12)


def test_coil_operator_matches_reference():
    """c = 3 coil maps: the oracle restatement against the reference's own outputs."""
    g = load("coils.npz")
    A = oop.CartesianOperator(g["op_pattern"], tuple(g["op_shape"]), coil_maps=g["op_coils"])
    np.testing.assert_allclose(A.apply(g["op_X"]), g["op_AX"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(A.adjoint(g["op_Y"]), g["op_AHY"], rtol=0, atol=1e-12)
    V, Xc = g["op_V"], g["op_Xc"]
    np.testing.assert_allclose(A.apply(Xc @ V.conj().T), g["op_AXc"], rtol=0, atol=1e-12)


def test_operator_adjoint_identity_3d():
    """3-D restatement (cfg4): <A X, Y> == <X, A^H Y>."""
    rng = np.random.default_rng(4)
    shape = (8, 6, 4)
    n = 8 * 6 * 4
    L, m = 3, 12
    pat = np.stack([rng.choice(n, size=m, replace=False) for _ in range(L)])
    A = oop.CartesianOperator(pat, shape)
    X = rng.standard_normal((n, L)) + 1j * rng.standard_normal((n, L))
    Y = rng.standard_normal((m, L)) + 1j * rng.standard_normal((m, L))
    lhs = np.vdot(A.apply(X), Y)
    rhs = np.vdot(X, A.adjoint(Y))
    assert abs(lhs - rhs) <= 1e-10 * abs(lhs)


def test_epi_pattern_matches_reference():
    g = load("operator.npz")
    np.testing.assert_array_equal(oop.make_epi_pattern((8, 8), 2, 5), g["epi8_pattern"])
    np.testing.assert_array_equal(oop.make_epi_pattern((16, 8), 4, 6), g["epi_rect_pattern"])
    with pytest.raises(ValueError, match="exceeds"):
        oop.make_epi_pattern((8, 8), 9, 3)


def _solve_from(g, iters):
    A = oop.CartesianOperator(g["pattern"], tuple(g["shape"]))
    return osv.solve_core(g["Y"], A, g["atoms_c"], basis=g["basis"], mode="blip_exact",
                          max_iters=iters, zeta=2.0)


def test_solver_small_matches_reference_trace():
    g = load("solver_small.npz")
    X, idx, gam, rec = _solve_from(g, 10)
    np.testing.assert_allclose([r["fidelity"] for r in rec], g["fidelity"], rtol=1e-12)
    np.testing.assert_array_equal([r["mu"] for r in rec], g["mu"])
    np.testing.assert_array_equal([r["shrinks"] for r in rec], g["shrinks"])
    np.testing.assert_allclose(gam, g["gammas"], rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose(X, g["X"], rtol=1e-10, atol=1e-12)
    np.testing.assert_array_equal(g["lookup"][idx, 0], g["t1"])


def test_cfg0_reference_trace():
    """BASELINE configs[0]: the oracle reproduces the reference's 20-iteration solve."""
    from paper_1810_01967_b200 import workloads
    g = load("cfg0_reference.npz")
    cfg = workloads.make_cfg0()
    np.testing.assert_array_equal(cfg.Y, g["Y"])
    np.testing.assert_array_equal(cfg.cdict.basis, g["basis"])
    A = oop.CartesianOperator(cfg.pattern, cfg.spatial_shape)
    X, idx, gam, rec = osv.solve_core(g["Y"], A, g["atoms_c"], basis=g["basis"],
                                      mode="blip_exact", max_iters=20, zeta=2.0)
    np.testing.assert_allclose([r["fidelity"] for r in rec], g["fidelity"], rtol=1e-12)
    np.testing.assert_array_equal([r["shrinks"] for r in rec], g["shrinks"])
    np.testing.assert_array_equal(idx, g["indices"])
    np.testing.assert_allclose(gam, g["gammas"], rtol=1e-10, atol=1e-14)


def test_step_shrinkage_known_constants():
    """test_solver.py:131-142 analogue: identity operator, mu0 = 4 -> mu = 1 after 2 shrinks."""
    rng = np.random.default_rng(87)
    from paper_1810_01967_b200.dictionary import ParameterGrid, generate_fingerprints
    grid = ParameterGrid(np.linspace(300.0, 2000.0, 4), np.linspace(40.0, 250.0, 3),
                         np.linspace(-60.0, 60.0, 4))
    dct = generate_fingerprints(grid, 10.0, 8)
    pat = oop.make_epi_pattern((4, 4), 4, 8)
    A = oop.CartesianOperator(pat, (4, 4), identity_transform=True)
    idx = rng.integers(dct.d, size=16)
    pd = 0.5 + rng.random(16)
    X0 = pd[:, None] * dct.atoms[idx]
    Y = A.apply(X0)
    X = np.zeros_like(X0)
    G = A.adjoint(A.apply(X) - Y)
    mu, proj, shrinks, fixed = osv.step_shrinkage(
        X, G, 4.0, lambda Z: orc.project_cone_exact(Z, dct.atoms), A.apply, 2.0, 60)
    assert not fixed and mu == 1.0 and shrinks == 2


def test_step_collapse_raises():
    rng = np.random.default_rng(3)
    atoms = rng.standard_normal((5, 4)) + 1j * rng.standard_normal((5, 4))
    atoms /= np.linalg.norm(atoms, axis=1)[:, None]
    X = np.zeros((3, 4), complex)
    G = -(rng.standard_normal((3, 4)) + 1j * rng.standard_normal((3, 4)))
    with pytest.raises(osv.SolverError, match="step-size collapse"):
        osv.step_shrinkage(X, G, 1.0, lambda Z: orc.project_cone_exact(Z, atoms),
                           lambda dX: 1e6 * dX, 2.0, 3)
