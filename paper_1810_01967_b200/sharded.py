"""Multi-GPU compressed IPG: voxel-sharded projection, frame-sharded operator.

One process per GPU.  Every rank holds

* a **voxel shard** of the IPG state: rows [v0, v0 + n_loc) of X~, G~, Z, dX (n_loc = ceil(n/W);
  the last shard is zero-padded -- zero voxels project to index 0, gamma 0 and stay zero), the
  projection of those voxels (no collective: the dictionary is replicated);
* a **frame shard** of the measurements: frames [t0, t1) of Y, A X and the residual R, with its
  own s-channel operator A_r (the rank's rows of the sampling pattern and of the basis V).

The layouts meet at two exchanges per operator application (s-channel operator, §4.3 of DESIGN):

* forward: all-gather the voxel shards of X~ (n x s complex64) -> every rank FFTs the s channel
  images of the full volume and gathers its own frames;
* adjoint: every rank builds the partial gradient of its frames over the full volume,
  G~_r = compress(A_r^H R_r) (n x s), and a reduce-scatter sums the partials into the voxel shards.

Every scalar of the step rule (||dX||^2 over voxel shards, ||A dX||^2 / fidelity / kappa terms over
frame shards) is a partial sum all-reduced before the host reads it, so all ranks take the same
accept / shrink decisions.  This replaces the all-to-all of the uncompressed layout exchange:
with s << L the n x s coordinates are L/s times smaller than the n x L frame stack.
"""

from __future__ import annotations

import ctypes
import time

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .dictionary import device_dictionary
from .distributed import shard_range
from .forward_model import ForwardOperator, SamplingPattern, as_device_operator
from .solver import IpgState, SolverError, _image_to_host, _ipg_loop, _maps_from

__all__ = ["ShardComm", "ShardedIpgState", "solve_compressed_sharded"]


class ShardComm:
    """Shard bookkeeping and the three collectives of the sharded IPG."""

    def __init__(self, n: int, L: int, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if L < self.world:
            raise SolverError(f"{L} frames cannot be split over {self.world} ranks")
        self.n = int(n)
        self.n_loc = -(-self.n // self.world)
        self.n_pad = self.n_loc * self.world
        self.v0 = self.rank * self.n_loc
        self.t0, self.t1 = shard_range(L, self.world, self.rank)
        self.nccl = dist.get_backend(group) == "nccl"

    @staticmethod
    def _real(t):
        return torch.view_as_real(t) if t.is_complex() else t

    def gather(self, shard: torch.Tensor, full: torch.Tensor) -> torch.Tensor:
        """Voxel shards (n_loc, ...) of every rank -> full (n_pad, ...) on every rank."""
        if self.nccl:
            dist.all_gather_into_tensor(self._real(full), self._real(shard), group=self.group)
        else:
            parts = [torch.empty_like(self._real(shard)) for _ in range(self.world)]
            dist.all_gather(parts, self._real(shard).contiguous(), group=self.group)
            self._real(full).copy_(torch.cat(parts, 0))
        return full

    def scatter_sum(self, full: torch.Tensor, shard: torch.Tensor) -> torch.Tensor:
        """Per-rank partials (n_pad, ...) -> their sum's voxel shard (n_loc, ...)."""
        if self.nccl:
            dist.reduce_scatter_tensor(self._real(shard), self._real(full),
                                       op=dist.ReduceOp.SUM, group=self.group)
        else:  # gloo has no reduce-scatter: all-reduce, keep the own rows
            dist.all_reduce(self._real(full), op=dist.ReduceOp.SUM, group=self.group)
            shard.copy_(full[self.v0:self.v0 + self.n_loc])
        return shard

    def allreduce_(self, t: torch.Tensor) -> torch.Tensor:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t


class ShardedIpgState(IpgState):
    """``IpgState`` with the voxel / frame shards of ``ShardComm`` (CUDA kernels per rank)."""

    def __init__(self, Y, A: ForwardOperator, dictionary, basis, weights, device, comm: ShardComm):
        if A.kind != "cartesian_dft" or basis is None:
            raise SolverError("the sharded solver needs a compressed Cartesian problem")
        lib = _lib.load()
        self.lib = lib
        self.comm = comm
        self.dev = device
        self.dd = device_dictionary(dictionary, device)
        self.n_glob, self.m, self.L = A.n, A.m, A.L
        self.cm = A.c * A.m
        self.dim = self.dd.s
        t0, t1 = comm.t0, comm.t1
        pat = np.asarray(A.pattern.indices)[t0:t1]
        self.A = ForwardOperator("cartesian_dft", A.n, A.m, t1 - t0, c=A.c,
                                 pattern=SamplingPattern(pat, A.pattern.spatial_shape),
                                 coil_maps=A.coil_maps,
                                 identity_transform=A.identity_transform, device=device)
        Vfull = np.ascontiguousarray(basis, dtype=np.complex64)
        self.V_full = torch.from_numpy(Vfull).to(device)
        self.V = self.V_full[t0:t1].contiguous()
        Yfm = np.ascontiguousarray(np.asarray(Y)[:, t0:t1].T, dtype=np.complex64)
        self.Y = torch.from_numpy(Yfm).to(device)                      # (L_r, c*m)
        self.w = None
        if weights is not None:
            wf = np.broadcast_to(weights, np.asarray(Y).shape)[:, t0:t1].T
            self.w = torch.from_numpy(np.ascontiguousarray(wf, dtype=np.float32)).to(device)
        c64 = dict(dtype=torch.complex64, device=device)
        nl, dim = comm.n_loc, self.dim
        self.n = nl                                                     # projected voxels
        self.X = torch.zeros((nl, dim), **c64)
        self.Xn = torch.empty((nl, dim), **c64)
        self.G = torch.empty((nl, dim), **c64)
        self.Z = torch.empty((nl, dim), **c64)
        self.dX = torch.empty((nl, dim), **c64)
        self.Xfull = torch.zeros((comm.n_pad, dim), **c64)
        self.Gfull = torch.zeros((comm.n_pad, dim), **c64)             # rows >= n stay zero
        L_r = t1 - t0
        self.AX = torch.zeros((L_r, self.cm), **c64)
        self.R = torch.empty((L_r, self.cm), **c64)
        self.idx = torch.zeros(nl, dtype=torch.int32, device=device)
        self.idx_n = torch.zeros(nl, dtype=torch.int32, device=device)
        self.gam = torch.zeros(nl, dtype=torch.float64, device=device)
        self.gam_n = torch.empty(nl, dtype=torch.float64, device=device)
        self.scal = torch.zeros(8, dtype=torch.float64, device=device)
        self.host = torch.zeros(8, dtype=torch.float64, pin_memory=True)
        self.pws_bytes = lib.cbb_project_workspace_bytes_dict(nl, ctypes.byref(self.dd.view))
        self.rws_bytes = lib.cbb_reduce_workspace_bytes()
        self.algo = 0

    def read(self, *slots):
        """All-reduce the requested partial scalars, then read them on the host."""
        idx = torch.as_tensor(list(slots), device=self.dev)
        vals = self.comm.allreduce_(self.scal.index_select(0, idx))
        self.scal.index_copy_(0, idx, vals)
        return super().read(*slots)

    def _full(self, Xs):
        return self.comm.gather(Xs, self.Xfull)[:self.n_glob]

    def apply(self, Xs, out):
        self.A.fm_apply_compressed(self._full(Xs), self.V, out=out)
        return out

    def apply_norm2(self, Xs, slot):
        self.A.fm_apply_norm2_compressed(self._full(Xs), self.V, self.scal[slot:slot + 1])

    def gradient(self):
        self.A.fm_adjoint_compressed(self.R, self.V, out=self.Gfull[:self.n_glob])
        self.comm.scatter_sum(self.Gfull, self.G)

    def decompress(self, Xs):
        return self._full(Xs) @ self.V_full.conj().transpose(0, 1)

    def gather_outputs(self):
        """Full-image (idx int64, gamma, X~) on every rank."""
        nl, n = self.comm.n_loc, self.n_glob
        idx = torch.empty(self.comm.n_pad, dtype=torch.int32, device=self.dev)
        gam = torch.empty(self.comm.n_pad, dtype=torch.float64, device=self.dev)
        self.comm.gather(self.idx[:nl], idx)
        self.comm.gather(self.gam[:nl], gam)
        X = self.comm.gather(self.X, torch.empty_like(self.Xfull))
        return idx[:n], gam[:n], X[:n]


def solve_compressed_sharded(Y, A, cdict, config, gt=None, group=None, on_iter=None):
    """``solve_compressed`` (solver.py:269-275) with the IPG state sharded over the ranks of
    `group` (one process per GPU, ``torch.distributed`` initialised).  Every rank passes the same
    inputs and returns the same (image, maps, gammas, trace)."""
    if config.compressed != cdict.s:
        raise SolverError("config.compressed does not match dictionary rank")
    if config.mode == "coverblip":
        raise SolverError("the sharded solver runs the exact projection (mode blip_exact)")
    Ad = as_device_operator(A)
    dev = Ad.device
    weights = None
    if config.weights_enabled:
        if getattr(A, "weights", None) is None:
            raise SolverError("weights enabled but operator carries none")
        weights = np.asarray(A.weights, dtype=float)
    Ynp = np.asarray(Y, dtype=complex)
    with torch.cuda.device(dev):
        comm = ShardComm(Ad.n, Ad.L, group)
        st = ShardedIpgState(Ynp, Ad, cdict, cdict.basis, weights, dev, comm)
        n, d = Ad.n, st.dd.d
        if config.fixed_step is not None:
            mu_base = config.fixed_step
        elif config.mu_init is not None:
            mu_base = config.mu_init
        else:
            mu_base = n / Ad.m
        y_norm = float(np.linalg.norm(Ynp))
        gt_t, gt_norm = None, None
        if gt is not None:
            gt_data = gt.data if hasattr(gt, "data") and not isinstance(gt, np.ndarray) else gt
            gt_t = torch.from_numpy(np.ascontiguousarray(gt_data, dtype=np.complex64)).to(dev)
            gt_norm = float(np.linalg.norm(gt_data))
        trace, have_proj = _ipg_loop(st, config, mu_base, y_norm, gt_t, gt_norm, n, d, on_iter)
        torch.cuda.current_stream(dev).synchronize()
        trace.total_time = time.perf_counter() - trace.start
        idx, gam, Xs = st.gather_outputs()
        idx = idx.cpu().numpy().astype(np.int64) if have_proj else np.zeros(n, np.int64)
        gam = gam.cpu().numpy() if have_proj else np.zeros(n)
        maps = _maps_from(cdict, idx, gam)
        out = _image_to_host(Xs, st.V_full)
        return out, maps, gam, trace
