"""Multi-GPU partitioning of the exact projection, one process per GPU.

* Voxel sharding (cfg1): voxels are independent units; every rank projects its own
  contiguous voxel range against the replicated dictionary.  No data-path collective
  (``shard_range`` + ``project_cone_exact``; ``bench.py`` reports weak scaling).
* Atom sharding (cfg3, D = 2^20 too large to replicate cheaply with its fp16 / fp32 / fp64
  copies): every rank screens its dictionary shard (``cbb_project_best``: shard-local exact
  fp64 argmax as a GLOBAL index + its raw score), then the first-index global argmax of
  ``projection.py:62`` is recovered EXACTLY with two collectives over NCCL:
      all-reduce MAX of the fp64 scores  ->  cand = (score == max) ? idx : INT64_MAX
      (``cbb_argmax_select``)  ->  all-reduce MIN of cand.
  No precision is lost (no packing of a rounded score with the index).  Every rank then
  writes all projected rows gamma * d_j* itself from a replicated copy of the dictionary
  (``cbb_scaled_rows`` over the full view: 2^20 x 10 complex atoms are 168 MB of fp64 rows),
  so the n x s rows never cross NVLink; without the replicated copy the owner shard writes its
  rows and a SUM all-reduce assembles them.

The collectives go through ``torch.distributed`` (NCCL on the box, gloo in the CPU tests).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .device import workspace

__all__ = ["shard_range", "combine_atom_shards", "project_atom_sharded", "cuda_select"]

INT64_MAX = np.iinfo(np.int64).max


def shard_range(total: int, world: int, rank: int):
    """Contiguous, balanced [lo, hi) range of `total` units for `rank` of `world`."""
    base, rem = divmod(int(total), int(world))
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def cuda_select(score: torch.Tensor, gidx: torch.Tensor, gmax: torch.Tensor) -> torch.Tensor:
    """cand = (score == gmax) ? gidx : INT64_MAX on the GPU (``cbb_argmax_select``)."""
    cand = torch.empty_like(gidx)
    _lib.check(_lib.load().cbb_argmax_select(score.data_ptr(), gidx.data_ptr(), gmax.data_ptr(),
                                             score.numel(), cand.data_ptr(), _lib.stream_ptr()),
               "cbb_argmax_select")
    return cand


def combine_atom_shards(score: torch.Tensor, gidx: torch.Tensor, group=None,
                        select=cuda_select):
    """Exact global (max score, lowest index) over ranks.  Returns (global idx, global score).

    ``select`` is the elementwise candidate step (the CUDA kernel on the product path; the CPU
    gloo tests inject an equivalent so the collective protocol can be exercised without GPUs).
    """
    gmax = score.clone()
    dist.all_reduce(gmax, op=dist.ReduceOp.MAX, group=group)
    cand = select(score, gidx, gmax)
    dist.all_reduce(cand, op=dist.ReduceOp.MIN, group=group)
    return cand, gmax


def project_atom_sharded(Z: torch.Tensor, atoms_shard, atom_offset: int, group=None,
                         proj_c128=False, atoms_full=None):
    """Atom-sharded exact projection of the (replicated) voxels Z on this rank's shard.

    ``atoms_full`` (optional, the whole dictionary or its ``DeviceDictionary``): the projected
    rows are written locally from it instead of being summed over the ranks.
    Returns (indices int64, gammas float64, projected) identical on every rank.
    """
    from .dictionary import device_dictionary
    dd = device_dictionary(atoms_shard, Z.device)
    lib = _lib.load()
    n = int(Z.shape[0])
    idx = torch.empty(n, dtype=torch.int64, device=Z.device)
    score = torch.empty(n, dtype=torch.float64, device=Z.device)
    wsb = lib.cbb_project_workspace_bytes(n, dd.s)
    ws = workspace(wsb, Z.device, "project")
    _lib.check(lib.cbb_project_best(Z.data_ptr(), int(Z.dtype == torch.complex128), n,
                                    ctypes.byref(dd.view), int(atom_offset), idx.data_ptr(),
                                    score.data_ptr(), ws.data_ptr(), wsb, 0, _lib.stream_ptr()),
               "cbb_project_best")
    gidx, gscore = combine_atom_shards(score, idx, group)
    gamma = torch.clamp(gscore, min=0.0)
    proj = torch.empty((n, dd.s), dtype=torch.complex128 if proj_c128 else torch.complex64,
                       device=Z.device)
    if atoms_full is not None:       # every rank owns every atom: local rows, no collective
        full = device_dictionary(atoms_full, Z.device)
        _lib.check(lib.cbb_scaled_rows(ctypes.byref(full.view), 0, gidx.data_ptr(),
                                       gamma.data_ptr(), n, proj.data_ptr(), int(proj_c128),
                                       _lib.stream_ptr()), "cbb_scaled_rows")
        return gidx, gamma, proj
    _lib.check(lib.cbb_scaled_rows(ctypes.byref(dd.view), int(atom_offset), gidx.data_ptr(),
                                   gamma.data_ptr(), n, proj.data_ptr(), int(proj_c128),
                                   _lib.stream_ptr()), "cbb_scaled_rows")
    dist.all_reduce(proj, op=dist.ReduceOp.SUM, group=group)
    return gidx, gamma, proj
