"""Multi-process (gloo, world size 2, CPU) test of the sharded compressed IPG.

The product's shared IPG loop (``solver._ipg_loop``) and its shard bookkeeping / collectives
(``sharded.ShardComm``: voxel-shard all-gather, partial-gradient reduce-scatter, scalar
all-reduces) drive a per-rank state whose local arithmetic is the fp64 oracle (the CUDA kernels
cannot run here).  The voxel count does not divide by the world size, so the padded last shard is
exercised too.  The run must reproduce the single-process oracle solve: identical step sizes and
shrink counts, fidelities and image to fp64 rounding.
"""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import operator as oop
from oracle import projection as orc
from oracle import solver as osv


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem():
    from paper_1810_01967_b200 import workloads
    cfg = workloads.make_cfg0(h=15, w=15, L=24, s=4, lines=4, n_t1=8, n_t2=8)
    return (cfg.Y, cfg.pattern, cfg.spatial_shape, cfg.cdict.atoms_compressed,
            np.ascontiguousarray(cfg.cdict.basis))


class OracleShardState:
    """The ShardedIpgState interface with fp64 oracle arithmetic on CPU tensors."""

    def __init__(self, Y, pattern, shape, atoms, V, comm):
        self.comm = comm
        t0, t1 = comm.t0, comm.t1
        self.Aop = oop.CartesianOperator(pattern[t0:t1], shape)
        self.V, self.Vr = V, V[t0:t1]
        self.Y = np.asarray(Y)[:, t0:t1]
        self.atoms = atoms
        self.n = comm.n
        nl, s = comm.n_loc, V.shape[1]
        c128 = dict(dtype=torch.complex128)
        self.X, self.Xn, self.G, self.dX = (torch.zeros((nl, s), **c128) for _ in range(4))
        self.Xfull = torch.zeros((comm.n_pad, s), **c128)
        self.Gfull = torch.zeros((comm.n_pad, s), **c128)
        self.idx = torch.zeros(nl, dtype=torch.int64)
        self.idx_n = torch.zeros(nl, dtype=torch.int64)
        self.gam = torch.zeros(nl, dtype=torch.float64)
        self.gam_n = torch.zeros(nl, dtype=torch.float64)
        self.AX = torch.zeros(self.Y.shape, **c128)
        self.R = None
        self.scal = torch.zeros(8, dtype=torch.float64)

    def read(self, *slots):
        vals = self.comm.allreduce_(self.scal[list(slots)].clone())
        return [float(v) for v in vals]

    def _full(self, Xs):
        return self.comm.gather(Xs, self.Xfull)[:self.n].numpy()

    def residual(self, slot):
        self.R = self.AX.numpy() - self.Y
        self.scal[slot] = float(np.vdot(self.R, self.R).real)

    def apply(self, Xs, out):
        out.copy_(torch.from_numpy(self.Aop.apply(self._full(Xs) @ self.Vr.conj().T)))
        return out

    def apply_norm2(self, Xs, slot):
        y = self.Aop.apply(self._full(Xs) @ self.Vr.conj().T)
        self.scal[slot] = float(np.vdot(y, y).real)

    def gradient(self):
        self.Gfull[:self.n] = torch.from_numpy(self.Aop.adjoint(self.R) @ self.Vr)
        self.comm.scatter_sum(self.Gfull, self.G)

    def project_step(self, mu, slot):
        r = orc.project_cone_exact((self.X - mu * self.G).numpy(), self.atoms)
        self.Xn = torch.from_numpy(np.ascontiguousarray(r.projected))
        self.idx_n = torch.from_numpy(r.indices)
        self.gam_n = torch.from_numpy(r.gammas)
        self.dX = self.Xn - self.X
        self.scal[slot] = float((self.dX.abs() ** 2).sum())

    def scaled_obj(self, alpha, slot):
        r = alpha * self.AX.numpy() - self.Y
        self.scal[slot] = float(np.vdot(r, r).real)

    def norm2(self, t, slot):
        self.scal[slot] = float((t.abs() ** 2).sum())

    def scale(self, t, alpha):
        t.mul_(alpha)

    def decompress(self, Xs):
        return torch.from_numpy(self._full(Xs) @ self.V.conj().T)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1810_01967_b200.sharded import ShardComm
        from paper_1810_01967_b200.solver import SolverConfig, _ipg_loop
        Y, pattern, shape, atoms, V = _problem()
        n, L = int(np.prod(shape)), pattern.shape[0]
        comm = ShardComm(n, L)
        st = OracleShardState(Y, pattern, shape, atoms, V, comm)
        conf = SolverConfig(mode="blip_exact", max_iters=8, zeta=2.0, compressed=V.shape[1])
        trace, _ = _ipg_loop(st, conf, n / pattern.shape[1], float(np.linalg.norm(Y)), None, None,
                             n, atoms.shape[0])
        img = st.decompress(st.X).numpy()
        q.put((rank, comm.n_loc, comm.t0, comm.t1, [r["mu"] for r in trace.records],
               [r["shrinks"] for r in trace.records], trace.fidelities(), img))
    finally:
        dist.destroy_process_group()


def test_sharded_ipg_gloo_world2_matches_single_process_oracle():
    Y, pattern, shape, atoms, V = _problem()
    A = oop.CartesianOperator(pattern, shape)
    img_ref, _, _, recs = osv.solve_core(Y, A, atoms, basis=V, mode="blip_exact", max_iters=8,
                                         zeta=2.0)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = int(np.prod(shape))
    assert n % 2 == 1                      # the padded last voxel shard is exercised
    for rank, n_loc, t0, t1, mu, shrinks, fid, img in out:
        assert n_loc == (n + 1) // 2 and t1 - t0 == pattern.shape[0] // 2
        np.testing.assert_allclose(mu, [r["mu"] for r in recs], rtol=1e-12)
        assert shrinks == [r["shrinks"] for r in recs]
        np.testing.assert_allclose(fid, [r["fidelity"] for r in recs], rtol=1e-10)
        np.testing.assert_allclose(img, img_ref, rtol=1e-9, atol=1e-12)
