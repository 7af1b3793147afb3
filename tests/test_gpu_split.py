"""Split-operand tcgen05 screen (hi/lo fp16 operands, fp32 accumulators) on coherent
dictionaries: the fp16 screen, the split screen, the FFMA screen and the exhaustive fp64 scan
all return the fp64 argmax, so their indices are identical (not merely tie-tolerant) and their
gammas agree to the fp64 summation order of the rescoring kernels (1e-14); the automatic screen
choice follows the dictionary's coherence estimate."""

import numpy as np
import pytest

from oracle import projection as orc

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _coherent(L=160, s=10, n_t1=30, n_t2=30, n_b0=7):
    from paper_1810_01967_b200 import svd_compress
    from paper_1810_01967_b200.dictionary import Dictionary
    from paper_1810_01967_b200.workloads import bloch_irbssfp, sequence_schedule
    alpha, tr = sequence_schedule(L, seed=0)
    g = np.meshgrid(np.geomspace(100, 5000, n_t1), np.geomspace(50, 5000, n_t2),
                    np.linspace(-40, 40, n_b0), indexing="ij")
    p = np.stack([x.ravel() for x in g], axis=1)
    p = p[p[:, 1] < p[:, 0]]
    raw = bloch_irbssfp(p, alpha, tr)
    norms = np.linalg.norm(raw, axis=1)
    D = Dictionary(atoms=raw / norms[:, None], norms=norms, lookup_table=p,
                   tr_ms=float(np.mean(tr)), L=L)
    return svd_compress(D, s).atoms_compressed


@pytest.fixture(scope="module")
def coherent_atoms():
    return _coherent()


def _voxels(rng, atoms, n, noise):
    s = atoms.shape[1]
    j = rng.integers(len(atoms), size=n)
    Z = atoms[j] * rng.uniform(0.3, 1.0, size=(n, 1)) * np.exp(1j * rng.uniform(-0.3, 0.3, (n, 1)))
    Z += noise / np.sqrt(2 * s) * (rng.standard_normal((n, s)) + 1j * rng.standard_normal((n, s)))
    return Z


@pytest.fixture(scope="module")
def coherent_atoms20():
    return _coherent(s=20)


@pytest.mark.parametrize("s", [10, 20])
@pytest.mark.parametrize("noise", [0.0, 0.02, 0.3])
def test_all_screens_agree_on_coherent_dictionary(coherent_atoms, coherent_atoms20, noise, s):
    import paper_1810_01967_b200 as cb
    atoms = coherent_atoms if s == 10 else coherent_atoms20
    rng = np.random.default_rng(int(noise * 100) + 1)
    Z = _voxels(rng, atoms, 5000, noise)
    dd = cb.device_dictionary(atoms)
    out = {a: cb.project_cone_exact(Z, dd, algo=a)
           for a in ("tcgen05", "tcgen05_split", "ffma", "exhaustive")}
    ref = orc.project_cone_exact(Z, atoms)
    i1, s1, s2 = orc.top2(Z, atoms)
    bad = (out["exhaustive"].indices != ref.indices) & ~orc.near_tie_mask(s1, s2)
    assert not bad.any()
    for a in ("tcgen05", "tcgen05_split", "ffma"):
        np.testing.assert_array_equal(out[a].indices, out["exhaustive"].indices)
        np.testing.assert_allclose(out[a].gammas, out["exhaustive"].gammas, rtol=1e-14)
        np.testing.assert_allclose(out[a].projected, out["exhaustive"].projected, rtol=1e-14,
                                   atol=1e-16)


def test_split_near_ties(coherent_atoms):
    """Voxels on the bisector of two neighbouring atoms (exact-tie and 1-ulp-apart scores)."""
    import paper_1810_01967_b200 as cb
    atoms = coherent_atoms
    rng = np.random.default_rng(9)
    a = rng.integers(len(atoms) - 1, size=3000)
    Z = 0.5 * (atoms[a] + atoms[a + 1])
    Z[1000:2000] *= 1.0 + 1e-15 * rng.standard_normal((1000, 1))
    res = cb.project_cone_exact(Z, atoms, algo="tcgen05_split")
    ex = cb.project_cone_exact(Z, atoms, algo="exhaustive")
    np.testing.assert_array_equal(res.indices, ex.indices)
    np.testing.assert_allclose(res.gammas, ex.gammas, rtol=1e-14)


def test_auto_screen_follows_coherence(coherent_atoms):
    import paper_1810_01967_b200 as cb
    rng = np.random.default_rng(3)
    rand = rng.standard_normal((4000, 10)) + 1j * rng.standard_normal((4000, 10))
    rand /= np.linalg.norm(rand, axis=1)[:, None]
    d_rand = cb.device_dictionary(rand)
    d_coh = cb.device_dictionary(coherent_atoms)
    assert not d_rand.prefer_split
    assert d_coh.prefer_split
    assert d_coh.bounds()["coherence"] > 1.0 > d_rand.bounds()["coherence"]
    # s > 21: no split tiles, never preferred
    wide = rng.standard_normal((4000, 22)) + 1j * rng.standard_normal((4000, 22))
    assert not cb.device_dictionary(wide).prefer_split


def test_split_bounds_are_consistent(coherent_atoms):
    import paper_1810_01967_b200 as cb
    b = cb.device_dictionary(coherent_atoms).bounds()
    sd = b["scale_d"]
    assert 0.5 <= b["dmax"] * sd < 1.0
    # hi/lo reconstruction error ~ 2^-22 of the row, lo part ~ 2^-11 of it
    assert 0.0 <= b["delta_split"] <= 2.0 ** -20
    assert 0.0 < b["dlo_max"] <= 2.0 ** -10
    assert np.sqrt(2) * 0.5 <= b["split_row_max"] <= np.sqrt(2) * 1.01
