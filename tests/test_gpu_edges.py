"""GPU edge cases of the certified tcgen05 paths (fp16 screen and split hi/lo screen) against
the fp64 oracle.

* dictionary sizes around the 160- / 128-atom tiles and the 128-row storage tile (sentinel rows,
  partial tiles) and voxel counts around the 128-voxel tile;
* s at every K-step boundary of the sentinel layouts (2s + 1 = 16, 17, 32, 33, 63; split:
  6s + 1 = 13, 19, 31, 37, 43, 49, 61 | 67, 79, 85, 91, 97, 109, 115, 127);
* voxels spanning 60 orders of magnitude (power-of-two scaling of the fp16 operands);
* the IPG warm-start hint (random, out of range, negative) never changes the result.
"""

import ctypes

import numpy as np
import pytest

from oracle import projection as orc

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _atoms(rng, d, s):
    a = rng.standard_normal((d, s)) + 1j * rng.standard_normal((d, s))
    return a / np.linalg.norm(a, axis=1)[:, None]


def _check(Z, atoms, res):
    ref = orc.project_cone_exact(Z, atoms)
    i1, s1, s2 = orc.top2(Z, atoms)
    bad = (np.asarray(res.indices) != ref.indices) & ~orc.near_tie_mask(s1, s2)
    assert not bad.any(), f"{bad.sum()} index mismatches"
    same = np.asarray(res.indices) == ref.indices
    np.testing.assert_allclose(np.asarray(res.gammas)[same], ref.gammas[same], rtol=1e-12,
                               atol=1e-300)


ALGOS = ["tcgen05", "tcgen05_split"]


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("d", [321, 383, 384, 385, 479, 480, 481, 511, 512, 513, 639, 640, 641,
                               1280])
def test_dictionary_tile_boundaries(d, algo):
    import paper_1810_01967_b200 as cb
    rng = np.random.default_rng(d)
    atoms = _atoms(rng, d, 10)
    for n in (1, 127, 128, 129, 513):
        Z = rng.standard_normal((n, 10)) + 1j * rng.standard_normal((n, 10))
        Z[0] = 2.0 * atoms[-1]               # the last (sentinel-tile) atom must be findable
        res = cb.project_cone_exact(Z, atoms, algo=algo)
        _check(Z, atoms, res)
        assert res.indices[0] == d - 1


@pytest.mark.parametrize("s", [1, 7, 8, 15, 16, 31])
def test_k_step_boundaries(s):
    import paper_1810_01967_b200 as cb
    rng = np.random.default_rng(200 + s)
    atoms = _atoms(rng, 700, s)
    Z = rng.standard_normal((600, s)) + 1j * rng.standard_normal((600, s))
    _check(Z, atoms, cb.project_cone_exact(Z, atoms, algo="tcgen05"))
    _check(Z, atoms, cb.project_cone_exact(Z, atoms))        # auto


@pytest.mark.parametrize("s", [1, 2, 3, 5, 6, 7, 8, 10, 11, 13, 14, 15, 16, 18, 19, 21])
def test_split_k_step_boundaries(s):
    import paper_1810_01967_b200 as cb
    rng = np.random.default_rng(300 + s)
    atoms = _atoms(rng, 700, s)
    Z = rng.standard_normal((600, s)) + 1j * rng.standard_normal((600, s))
    _check(Z, atoms, cb.project_cone_exact(Z, atoms, algo="tcgen05_split"))


def test_split_rejects_wide_atoms():
    import paper_1810_01967_b200 as cb
    from paper_1810_01967_b200._lib import NativeError
    rng = np.random.default_rng(5)
    atoms = _atoms(rng, 700, 22)
    Z = rng.standard_normal((10, 22)) + 1j * rng.standard_normal((10, 22))
    with pytest.raises(NativeError):
        cb.project_cone_exact(Z, atoms, algo="tcgen05_split")


@pytest.mark.parametrize("algo", ALGOS)
def test_extreme_voxel_magnitudes(algo):
    import paper_1810_01967_b200 as cb
    rng = np.random.default_rng(77)
    atoms = _atoms(rng, 900, 10)
    Z = rng.standard_normal((400, 10)) + 1j * rng.standard_normal((400, 10))
    Z *= 10.0 ** rng.uniform(-30, 30, size=(400, 1))
    Z[5] = 1e-300 * atoms[3]                  # fp64 subnormal-range voxel
    Z[6] = 0.0                                # zero voxel -> index 0, gamma 0
    res = cb.project_cone_exact(Z, atoms, algo=algo)
    _check(Z, atoms, res)
    assert res.indices[5] == 3
    assert res.indices[6] == 0 and res.gammas[6] == 0.0


@pytest.mark.parametrize("algo", [1, 4])
def test_warm_start_hint_never_changes_results(algo):
    """cbb_project_step with random / out-of-range hints equals the unhinted projection."""
    import paper_1810_01967_b200 as cb
    from paper_1810_01967_b200 import _lib
    from paper_1810_01967_b200.device import workspace
    from paper_1810_01967_b200.workloads import cfg0_dictionary
    from paper_1810_01967_b200 import svd_compress
    lib = _lib.load()
    cd = svd_compress(cfg0_dictionary(L=120, n_t1=25, n_t2=25), 8)   # coherent MRF atoms
    dd = cb.device_dictionary(cd)
    rng = np.random.default_rng(8)
    n, s, d = 3000, 8, cd.atoms_compressed.shape[0]
    j = rng.integers(d, size=n)
    X = (0.5 + rng.random(n))[:, None] * cd.atoms_compressed[j]
    G = 0.05 * (rng.standard_normal((n, s)) + 1j * rng.standard_normal((n, s)))
    dev = torch.device("cuda")
    Xt = torch.from_numpy(X.astype(np.complex64)).to(dev)
    Gt = torch.from_numpy(G.astype(np.complex64)).to(dev)
    wsb = lib.cbb_project_workspace_bytes(n, s)
    ws = workspace(wsb, dev, "project")

    def step(hint):
        Z = torch.empty_like(Xt)
        idx = torch.empty(n, dtype=torch.int32, device=dev)
        gam = torch.empty(n, dtype=torch.float64, device=dev)
        Xn, dX = torch.empty_like(Xt), torch.empty_like(Xt)
        nd = torch.zeros(1, dtype=torch.float64, device=dev)
        h = None if hint is None else torch.from_numpy(hint.astype(np.int32)).to(dev)
        _lib.check(lib.cbb_project_step(Xt.data_ptr(), Gt.data_ptr(), 0.7, Z.data_ptr(), n,
                                        ctypes.byref(dd.view), None if h is None else h.data_ptr(),
                                        idx.data_ptr(), gam.data_ptr(), Xn.data_ptr(),
                                        dX.data_ptr(), nd.data_ptr(), ws.data_ptr(), wsb, algo,
                                        _lib.stream_ptr()), "step")
        return idx.cpu().numpy(), gam.cpu().numpy(), Xn.cpu().numpy(), Z.cpu().numpy()

    i0, g0, x0, z0 = step(None)
    ref = orc.project_cone_exact(z0.astype(np.complex128), cd.atoms_compressed)
    i1, s1, s2 = orc.top2(z0.astype(np.complex128), cd.atoms_compressed)
    bad = (i0 != ref.indices) & ~orc.near_tie_mask(s1, s2)
    assert not bad.any()
    for hint in (j, rng.integers(d, size=n), np.full(n, -1), np.full(n, d + 5), i0):
        ih, gh, xh, _ = step(hint)
        np.testing.assert_array_equal(ih, i0)
        np.testing.assert_array_equal(gh, g0)
        np.testing.assert_array_equal(xh, x0)
