"""Tile pruning of the split screen (IPG warm start on coherent dictionaries).

A coherent dictionary's split tiles are stored in a bisection order with per-tile / per-group
centroid + radius bounds; an IPG trial with a hint screens, per voxel tile (voxels sorted by the
position of their hint atom), only the atom tiles whose Cauchy-Schwarz bound reaches a voxel's
hint score.  The pruned projection must return exactly what the unpruned split screen and the
exhaustive fp64 scan return (reference semantics projection.py:58-62: fp64 argmax, first index
on ties), whatever the hint, including ties that straddle tiles."""

import ctypes

import numpy as np
import pytest

from oracle import projection as orc

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _coherent(L=160, s=10, n_t1=30, n_t2=30, n_b0=9):
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
def atoms10():
    return _coherent(s=10)


@pytest.fixture(scope="module")
def atoms20():
    return _coherent(s=20)


class _Stepper:
    """cbb_project_step on fixed (X, G, mu) with a chosen workspace size and algorithm."""

    def __init__(self, atoms, X, G, mu):
        import paper_1810_01967_b200 as cb
        from paper_1810_01967_b200 import _lib
        self.lib, self._lib = _lib.load(), _lib
        self.dd = cb.device_dictionary(atoms)
        self.dev = torch.device("cuda")
        self.n, self.s = X.shape
        self.X = torch.from_numpy(X.astype(np.complex64)).to(self.dev)
        self.G = torch.from_numpy(G.astype(np.complex64)).to(self.dev)
        self.mu = mu
        self.ws_plain = self.lib.cbb_project_workspace_bytes(self.n, self.s)
        self.ws_dict = self.lib.cbb_project_workspace_bytes_dict(self.n, ctypes.byref(self.dd.view))

    def __call__(self, hint, algo=4, pruned=True):
        n, dev = self.n, self.dev
        wsb = self.ws_dict if pruned else self.ws_plain
        ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
        Z = torch.empty_like(self.X)
        idx = torch.empty(n, dtype=torch.int32, device=dev)
        gam = torch.empty(n, dtype=torch.float64, device=dev)
        Xn, dX = torch.empty_like(self.X), torch.empty_like(self.X)
        nd = torch.zeros(1, dtype=torch.float64, device=dev)
        h = None if hint is None else torch.from_numpy(np.asarray(hint, np.int32)).to(dev)
        self._lib.check(self.lib.cbb_project_step(
            self.X.data_ptr(), self.G.data_ptr(), self.mu, Z.data_ptr(), n,
            ctypes.byref(self.dd.view), None if h is None else h.data_ptr(), idx.data_ptr(),
            gam.data_ptr(), Xn.data_ptr(), dX.data_ptr(), nd.data_ptr(), ws.data_ptr(), wsb,
            algo, self._lib.stream_ptr()), "cbb_project_step")
        listed, total = ctypes.c_int64(0), ctypes.c_int64(0)
        self._lib.check(self.lib.cbb_project_prune_stats(
            ws.data_ptr(), wsb, n, ctypes.byref(self.dd.view), ctypes.byref(listed),
            ctypes.byref(total), self._lib.stream_ptr()), "prune_stats")
        return dict(idx=idx.cpu().numpy(), gam=gam.cpu().numpy(), Xn=Xn.cpu().numpy(),
                    dX=dX.cpu().numpy(), nd=float(nd.item()), Z=Z.cpu().numpy(),
                    listed=listed.value, total=total.value)


def _state(rng, atoms, n, noise):
    d, s = atoms.shape
    j = rng.integers(d, size=n)
    X = (0.4 + 0.6 * rng.random(n))[:, None] * atoms[j]
    G = noise * (rng.standard_normal((n, s)) + 1j * rng.standard_normal((n, s))) / np.sqrt(2 * s)
    return X, G, j


def _assert_same(a, b):
    np.testing.assert_array_equal(a["idx"], b["idx"])
    np.testing.assert_array_equal(a["gam"], b["gam"])
    np.testing.assert_array_equal(a["Xn"], b["Xn"])
    np.testing.assert_array_equal(a["dX"], b["dX"])
    assert a["nd"] == b["nd"]


_atoms_cache = {}


def _atoms_for(s):
    if s not in _atoms_cache:
        _atoms_cache[s] = _coherent(s=s)
    return _atoms_cache[s]


@pytest.mark.parametrize("s,noise", [(10, 0.01), (10, 0.1), (10, 0.5), (20, 0.01), (20, 0.1),
                                     (20, 0.5), (8, 0.1), (21, 0.1)])
def test_pruned_step_equals_exhaustive(atoms10, atoms20, s, noise):
    """s = 8, 10, 20: the bound pass folded into the MMA (three spare K columns); s = 21: no
    spare columns, the epilogue evaluates the bound itself."""
    atoms = atoms10 if s == 10 else atoms20 if s == 20 else _atoms_for(s)
    rng = np.random.default_rng(int(noise * 1000) + s)
    n = 20000
    X, G, j = _state(rng, atoms, n, noise)
    st = _Stepper(atoms, X, G, 0.9)
    dd = st.dd
    assert dd.prefer_split and dd.view.tile_c, "coherent dictionary must be prune-capable"
    ref = st(None, algo=3, pruned=False)                        # exhaustive fp64 scan
    z = ref["Z"].astype(np.complex128)
    oref = orc.project_cone_exact(z, atoms)
    i1, s1, s2 = orc.top2(z, atoms)
    assert not ((ref["idx"] != oref.indices) & ~orc.near_tie_mask(s1, s2)).any()
    unpruned = st(j, algo=4, pruned=False)
    assert unpruned["listed"] == -1
    _assert_same(unpruned, ref)
    d = atoms.shape[0]
    neighbour = np.clip(j + rng.integers(-2, 3, size=n), 0, d - 1)
    for hint in (j, neighbour, ref["idx"], rng.integers(d, size=n), np.full(n, -1),
                 np.full(n, d + 3)):
        got = st(hint, algo=4, pruned=True)
        _assert_same(got, ref)
        assert 0 <= got["listed"] <= got["total"]
    # a good hint prunes most of the dictionary (the point of the exercise)
    good = st(ref["idx"], algo=4, pruned=True)
    if noise <= 0.01:
        assert good["listed"] < 0.5 * good["total"], (good["listed"], good["total"])
    elif noise <= 0.1:
        assert good["listed"] < 0.8 * good["total"], (good["listed"], good["total"])
    # no hint at all: nothing to prune with, the split screen runs unpruned
    assert st(None, algo=4, pruned=True)["listed"] == -1


def test_pruned_ties_straddling_tiles(atoms10):
    """Duplicated atoms (exact fp64 ties at indices j and j + d0, laid out by the bisection order
    possibly in different tiles) and voxels on the bisector of two neighbouring atoms: the lowest
    index wins, as np.argmax does (projection.py:62)."""
    rng = np.random.default_rng(5)
    base = atoms10[::2]
    d0 = base.shape[0]
    atoms = np.concatenate([base, base[::-1]])   # atom j == atom 2 d0 - 1 - j
    n = 12000
    a = rng.integers(d0 - 1, size=n)
    X = np.empty((n, atoms.shape[1]), np.complex128)
    X[: n // 2] = base[a[: n // 2]] * 0.8
    X[n // 2:] = 0.5 * (base[a[n // 2:]] + base[a[n // 2:] + 1])
    G = np.zeros_like(X)
    st = _Stepper(atoms, X, G, 0.0)
    assert st.dd.prefer_split and st.dd.view.tile_c
    ref = st(None, algo=3, pruned=False)
    assert (ref["idx"] < d0).all()              # lowest index of each duplicate pair
    for hint in (a, 2 * d0 - 1 - a, ref["idx"], 2 * d0 - 1 - ref["idx"]):
        got = st(hint, algo=4, pruned=True)
        _assert_same(got, ref)
        assert got["listed"] >= 0


def test_prune_order_is_a_permutation(atoms10):
    import paper_1810_01967_b200 as cb
    dd = cb.device_dictionary(atoms10)
    v = dd.view
    d = dd.d
    off_perm = int(v.tc2_atom) - dd.storage.data_ptr()
    off_pos = int(v.tc2_pos) - dd.storage.data_ptr()
    perm = dd.storage[off_perm:off_perm + 4 * d].view(torch.int32).cpu().numpy()
    pos = dd.storage[off_pos:off_pos + 4 * d].view(torch.int32).cpu().numpy()
    np.testing.assert_array_equal(np.sort(perm), np.arange(d))
    np.testing.assert_array_equal(perm[pos], np.arange(d))
    # tiles are compact: the median tile radius is far below the dictionary's spread
    rows = 128
    nt = v.n_tiles2
    off_r = int(v.tile_r) - dd.storage.data_ptr()
    rad = dd.storage[off_r:off_r + 4 * nt].view(torch.float32).cpu().numpy()
    a = atoms10[perm]
    for t in range(nt):
        blk = a[t * rows:(t + 1) * rows]
        c = blk.mean(0)
        assert np.linalg.norm(blk - c, axis=1).max() <= rad[t] * (1 + 1e-5) + 1e-6
    assert np.median(rad) < 0.5


@pytest.mark.parametrize("graphs", [True, False])
def test_representative_hint_leaves_the_trace_unchanged(graphs):
    """cbb_project_hint: from the second iteration on, the first trial's second warm-start atom
    is the best tile representative of X - mu G.  It is only a hint: with it (device-decided
    graphs or the host loop) the solve returns the same iterates, atoms, step sizes and
    fidelities as without, and in lockstep the atoms are the fp64 oracle's; the first-trial tile
    lists get shorter."""
    from paper_1810_01967_b200 import _lib, workloads
    from paper_1810_01967_b200.forward_model import SamplingPattern, make_cartesian_operator
    from paper_1810_01967_b200.solver import IpgState, SolverConfig, solve_compressed
    cfg = workloads.make_cfg4(shape=(32, 32, 8), L=80, s=10, undersample=8, n_t1=40, n_t2=40,
                              n_b0=6, device=torch.device("cuda"))
    cd = cfg.cdict
    A = make_cartesian_operator(SamplingPattern(cfg.pattern, cfg.spatial_shape))
    conf = SolverConfig(mode="blip_exact", max_iters=6, zeta=2.0, compressed=10)
    lib = _lib.load()
    old_min, old_cap = IpgState.rep_hint_min_voxels, IpgState.graph_capable
    runs = {}
    try:
        if not graphs:
            IpgState.graph_capable = lambda self, config: False
        for use in (False, True):
            IpgState.rep_hint_min_voxels = 0 if use else 1 << 62
            from paper_1810_01967_b200 import solver as _solver
            _solver._state_cache.clear()              # a fresh state (the flag is cached on it)
            snaps, listed = [], []

            def on_iter(k, st, mu, shrinks, fixed):
                assert st.rep_hint_ready() == use
                snaps.append((k, mu, shrinks, st.idx_n.cpu().numpy().copy(),
                              st.Z.cpu().numpy().copy()))
                a, b = ctypes.c_int64(0), ctypes.c_int64(0)
                ws = st.project_workspace()
                lib.cbb_project_prune_stats(ws.data_ptr(), st.pws_bytes, st.n,
                                            ctypes.byref(st.dd.view), ctypes.byref(a),
                                            ctypes.byref(b), _lib.stream_ptr())
                listed.append((shrinks, a.value, b.value))

            X, maps, gam, trace = solve_compressed(cfg.Y, A, cd, None, conf, on_iter=on_iter)
            runs[use] = (X, gam, trace, snaps, listed)
    finally:
        IpgState.rep_hint_min_voxels, IpgState.graph_capable = old_min, old_cap
    (X0, g0, t0, s0, l0), (X1, g1, t1, s1, l1) = runs[False], runs[True]
    assert t0.iterations == t1.iterations >= 3
    assert [r["shrinks"] for r in t0.records] == [r["shrinks"] for r in t1.records]
    assert t0.fidelities() == t1.fidelities()
    np.testing.assert_array_equal(X0, X1)
    np.testing.assert_array_equal(g0, g1)
    for (k, mu, sh, idx, Z), (k1, mu1, sh1, idx1, Z1) in zip(s0, s1):
        assert (k, mu, sh) == (k1, mu1, sh1)
        np.testing.assert_array_equal(idx, idx1)
        np.testing.assert_array_equal(Z, Z1)
    # lockstep against the oracle on the last accepted trial
    k, mu, sh, idx, Z = s1[-1]
    Zd = Z.astype(np.complex128)
    ref = orc.project_cone_exact(Zd, cd.atoms_compressed)
    i1, a1, a2 = orc.top2(Zd, cd.atoms_compressed)
    bad = (idx != ref.indices) & ~orc.near_tie_mask(a1, a2)
    assert not bad.any()
    # pruning was active, and iterations accepted at their first trial list no more tiles with
    # the representative hint than without
    assert all(b > 0 and a >= 0 for _, a, b in l1)
    first0 = [a for (sh, a, b) in l0[1:] if sh == 0]
    first1 = [a for (sh, a, b) in l1[1:] if sh == 0]
    if first0:
        assert sum(first1) <= sum(first0)
