"""GPU pieces of the sharded paths (one GPU): shard kernels + exact combine.

Two atom shards are processed on the same device and combined with the same device
kernels the multi-rank path uses (``cbb_project_best`` -> max -> ``cbb_argmax_select``
-> min -> ``cbb_scaled_rows``); the result must equal the unsharded projection.  The
collective wrapper itself is exercised with a world-size-1 NCCL group.
"""

import ctypes
import socket

import numpy as np
import pytest

from oracle import projection as orc

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def test_two_shard_emulation_matches_full_projection():
    import paper_1810_01967_b200 as cb
    from paper_1810_01967_b200 import _lib
    from paper_1810_01967_b200.device import workspace
    from paper_1810_01967_b200.distributed import cuda_select, shard_range
    rng = np.random.default_rng(5)
    d, s, n = 3000, 10, 4000
    atoms = rng.standard_normal((d, s)) + 1j * rng.standard_normal((d, s))
    atoms /= np.linalg.norm(atoms, axis=1)[:, None]
    atoms[2500] = atoms[40]
    Z = rng.standard_normal((n, s)) + 1j * rng.standard_normal((n, s))
    Z[7] = 3 * atoms[2500]
    Z[9] = 0
    zt = torch.from_numpy(Z).cuda()
    lib = _lib.load()
    scores, idxs, views = [], [], []
    for r in range(2):
        lo, hi = shard_range(d, 2, r)
        dd = cb.device_dictionary(atoms[lo:hi].copy())
        idx = torch.empty(n, dtype=torch.int64, device="cuda")
        sc = torch.empty(n, dtype=torch.float64, device="cuda")
        wsb = lib.cbb_project_workspace_bytes(n, s)
        ws = workspace(wsb, torch.device("cuda", 0), "project")
        _lib.check(lib.cbb_project_best(zt.data_ptr(), 1, n, ctypes.byref(dd.view), lo,
                                        idx.data_ptr(), sc.data_ptr(), ws.data_ptr(), wsb, 0,
                                        _lib.stream_ptr()), "best")
        scores.append(sc)
        idxs.append(idx)
        views.append((dd, lo))
    gmax = torch.maximum(scores[0], scores[1])
    cand = torch.minimum(cuda_select(scores[0], idxs[0], gmax), cuda_select(scores[1], idxs[1], gmax))
    gamma = torch.clamp(gmax, min=0)
    proj = torch.zeros((n, s), dtype=torch.complex128, device="cuda")
    for dd, lo in views:
        part = torch.empty_like(proj)
        _lib.check(lib.cbb_scaled_rows(ctypes.byref(dd.view), lo, cand.data_ptr(),
                                       gamma.data_ptr(), n, part.data_ptr(), 1,
                                       _lib.stream_ptr()), "rows")
        proj += part
    ref = orc.project_cone_exact(Z, atoms)
    np.testing.assert_array_equal(cand.cpu().numpy(), ref.indices)
    assert int(cand[7]) == 40 and int(cand[9]) == 0
    np.testing.assert_allclose(gamma.cpu().numpy(), ref.gammas, rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(proj.cpu().numpy(), ref.projected, rtol=1e-12, atol=1e-14)


def test_project_atom_sharded_world1_nccl():
    import torch.distributed as dist
    from paper_1810_01967_b200.distributed import project_atom_sharded
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        rng = np.random.default_rng(6)
        atoms = rng.standard_normal((1000, 10)) + 1j * rng.standard_normal((1000, 10))
        atoms /= np.linalg.norm(atoms, axis=1)[:, None]
        Z = rng.standard_normal((500, 10)) + 1j * rng.standard_normal((500, 10))
        idx, gam, proj = project_atom_sharded(torch.from_numpy(Z).cuda(), atoms, 0,
                                              proj_c128=True)
        ref = orc.project_cone_exact(Z, atoms)
        np.testing.assert_array_equal(idx.cpu().numpy(), ref.indices)
        np.testing.assert_allclose(proj.cpu().numpy(), ref.projected, rtol=1e-12, atol=1e-14)
    finally:
        dist.destroy_process_group()


def test_sharded_solve_world1_nccl_matches_single_gpu_solve():
    """The CUDA ShardedIpgState (NCCL collectives, frame-sharded s-channel operator, voxel
    shards) against the one-GPU solve_compressed on a reduced cfg0 problem."""
    import torch.distributed as dist
    from paper_1810_01967_b200 import workloads
    from paper_1810_01967_b200.forward_model import SamplingPattern, make_cartesian_operator
    from paper_1810_01967_b200.sharded import solve_compressed_sharded
    from paper_1810_01967_b200.solver import SolverConfig, solve_compressed
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        cfg = workloads.make_cfg0(h=24, w=24, L=40, s=6, lines=6, n_t1=12, n_t2=12)
        A = make_cartesian_operator(SamplingPattern(cfg.pattern, cfg.spatial_shape))
        conf = SolverConfig(mode="blip_exact", max_iters=6, zeta=2.0, compressed=6)
        X1, maps1, gam1, tr1 = solve_compressed(cfg.Y, A, cfg.cdict, None, conf)
        X2, maps2, gam2, tr2 = solve_compressed_sharded(cfg.Y, A, cfg.cdict, conf)
        assert [r["shrinks"] for r in tr1.records] == [r["shrinks"] for r in tr2.records]
        np.testing.assert_allclose([r["mu"] for r in tr2.records],
                                   [r["mu"] for r in tr1.records], rtol=1e-6)
        np.testing.assert_allclose(tr2.fidelities(), tr1.fidelities(), rtol=1e-5)
        np.testing.assert_array_equal(maps2.t1, maps1.t1)
        assert np.linalg.norm(X2 - X1) <= 1e-5 * np.linalg.norm(X1)
    finally:
        dist.destroy_process_group()
