"""Multi-process (gloo, world size 2, CPU) tests of the sharding host logic.

The per-shard local argmax comes from the oracle here (no GPU); the product's collective
protocol (``combine_atom_shards``) must reproduce the global first-index argmax of the
full dictionary exactly, including ties that straddle shards and all-zero voxels.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import projection as orc


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _cpu_select(score, gidx, gmax):
    return torch.where(score == gmax, gidx, torch.full_like(gidx, np.iinfo(np.int64).max))


def _worker(rank, world, port, Z, atoms, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1810_01967_b200.distributed import combine_atom_shards, shard_range
        lo, hi = shard_range(atoms.shape[0], world, rank)
        shard = atoms[lo:hi]
        corr = (Z @ shard.conj().T).real
        li = np.argmax(corr, axis=1)
        score = torch.from_numpy(corr[np.arange(len(Z)), li].copy())
        gidx = torch.from_numpy((li + lo).astype(np.int64))
        idx, gmax = combine_atom_shards(score, gidx, select=_cpu_select)
        q.put((rank, idx.numpy(), gmax.numpy()))
    finally:
        dist.destroy_process_group()


def test_shard_range_partitions():
    from paper_1810_01967_b200.distributed import shard_range
    for total in (0, 1, 7, 100, 131072):
        for world in (1, 2, 3, 8):
            parts = [shard_range(total, world, r) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [h - l for l, h in parts]
            assert max(sizes) - min(sizes) <= 1


def test_atom_sharded_combine_gloo_world2():
    rng = np.random.default_rng(21)
    d, s, n = 301, 6, 64
    atoms = rng.standard_normal((d, s)) + 1j * rng.standard_normal((d, s))
    atoms /= np.linalg.norm(atoms, axis=1)[:, None]
    atoms[200] = atoms[17]            # duplicate straddling the two shards -> lowest index 17
    Z = rng.standard_normal((n, s)) + 1j * rng.standard_normal((n, s))
    Z[3] = 2.0 * atoms[200]
    Z[5] = 0.0                        # all-zero voxel -> index 0
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, Z, atoms, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = orc.project_cone_exact(Z, atoms)
    for rank, idx, gmax in out:
        np.testing.assert_array_equal(idx, ref.indices)
        assert idx[3] == 17 and idx[5] == 0
        np.testing.assert_allclose(np.maximum(gmax, 0), ref.gammas, rtol=1e-12, atol=1e-15)
