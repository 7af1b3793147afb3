"""Exact cone projection -- drop-in for ``coverblip.projection.project_cone_exact``.

Reference semantics (``coverblip/projection.py:45-67``): for every voxel row
``Z_v`` pick ``j* = argmax_j Re<Z_v, D_j>`` (first index on ties, ``:62``), set
``gamma_v = max(Re<Z_v, D_j*>, 0)`` (``_gammas_for``, ``:38-42``) and
``projected_v = gamma_v * D_j*`` (``:64``); ``cost = n * d`` (``:67``); a shape
mismatch raises ``ValueError("dimension mismatch: ...")`` (``:53-56``).

B200 path: ``cbb_project_cone_exact`` (tcgen05 fp16 screening with a certified
window + fp64 rescoring, see ``csrc/cbb_project.cuh``).  numpy inputs return
numpy outputs with the reference dtypes (int64 / float64 / complex128); torch
CUDA inputs stay on the device.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .device import require_cuda, workspace
from .dictionary import DeviceDictionary, atoms_of, device_dictionary

__all__ = ["ConeProjection", "project_cone_exact", "project_device"]


@dataclass
class ConeProjection:
    """Mirror of ``projection.py:18-23``."""
    indices: object      # n chosen atom ids (int64)
    gammas: object       # n nonnegative scales (float64)
    projected: object    # n x dim complex, row v = gammas[v] * atoms[j_v]
    cost: int            # distance evaluations (n * d for the exact path)


def _as_array(Z):
    """``projection.py:32-35``: ``.data`` else the array itself."""
    if hasattr(Z, "data") and not isinstance(Z, (np.ndarray, torch.Tensor)):
        Z = Z.data
    if isinstance(Z, torch.Tensor):
        return Z
    return np.asarray(Z)


def _atoms_shape(dictionary):
    a = atoms_of(dictionary)
    if isinstance(a, DeviceDictionary):
        return a.shape
    return tuple(a.shape)


def project_device(Z: torch.Tensor, dd: DeviceDictionary, *, algo: str = "auto",
                   idx_int64: bool = True, proj_c128: bool = None, out=None):
    """Device-resident projection.  ``Z`` is a CUDA complex64/complex128 (n, s) tensor.

    Returns ``(indices, gammas, projected)`` device tensors.
    """
    lib = _lib.load()
    n, s = int(Z.shape[0]), int(Z.shape[1])
    z128 = Z.dtype == torch.complex128
    if proj_c128 is None:
        proj_c128 = z128
    dev = Z.device
    if out is None:
        idx = torch.empty(n, dtype=torch.int64 if idx_int64 else torch.int32, device=dev)
        gam = torch.empty(n, dtype=torch.float64, device=dev)
        proj = torch.empty((n, s), dtype=torch.complex128 if proj_c128 else torch.complex64,
                           device=dev)
    else:
        idx, gam, proj = out
    wsb = lib.cbb_project_workspace_bytes(n, s)
    ws = workspace(wsb, dev, "project")
    _last_ws[dev.index] = (ws, n, s, torch.cuda.current_stream(dev))
    rc = lib.cbb_project_cone_exact(Z.data_ptr() if n else None, int(z128), n,
                                    ctypes.byref(dd.view), idx.data_ptr(),
                                    int(idx.dtype == torch.int64), gam.data_ptr(),
                                    proj.data_ptr(), int(proj.dtype == torch.complex128),
                                    ws.data_ptr(), wsb, _lib.ALGOS[algo], _lib.stream_ptr())
    _lib.check(rc, "cbb_project_cone_exact")
    return idx, gam, proj


def project_cone_exact(Z, dictionary, *, algo: str = "auto") -> ConeProjection:
    """Drop-in for ``coverblip.projection.project_cone_exact`` (projection.py:45-67)."""
    Z = _as_array(Z)
    ashape = _atoms_shape(dictionary)
    if Z.ndim != 2 or Z.shape[1] != ashape[1]:
        raise ValueError(
            f"dimension mismatch: image is {tuple(Z.shape)}, atoms are {ashape}")
    n, d = int(Z.shape[0]), int(ashape[0])
    if isinstance(Z, torch.Tensor):
        dev = require_cuda(Z.device if Z.is_cuda else None)
        dd = device_dictionary(dictionary, dev)
        zt = Z.to(dev)
        if zt.dtype not in (torch.complex64, torch.complex128):
            zt = zt.to(torch.complex128)
        with torch.cuda.device(dev):
            idx, gam, proj = project_device(zt.contiguous(), dd, algo=algo)
        return ConeProjection(indices=idx, gammas=gam, projected=proj, cost=n * d)
    dev = require_cuda()
    dd = device_dictionary(dictionary, dev)
    if not np.iscomplexobj(Z) or Z.dtype not in (np.complex64, np.complex128):
        Z = Z.astype(np.complex128)
    Z = np.ascontiguousarray(Z)
    zh = torch.from_numpy(Z)
    with torch.cuda.device(dev):
        if zh.is_pinned() and n >= _PIPELINE_MIN:
            idx, gam, proj = _project_pipelined(zh, dd, algo, dev)
        else:
            zt = zh.to(dev, non_blocking=True)
            didx, dgam, dproj = project_device(zt, dd, algo=algo, proj_c128=True)
            idx = torch.empty(n, dtype=torch.int64, pin_memory=True)
            gam = torch.empty(n, dtype=torch.float64, pin_memory=True)
            proj = torch.empty((n, Z.shape[1]), dtype=torch.complex128, pin_memory=True)
            idx.copy_(didx, non_blocking=True)
            gam.copy_(dgam, non_blocking=True)
            proj.copy_(dproj, non_blocking=True)
            torch.cuda.current_stream(dev).synchronize()
    return ConeProjection(indices=idx.numpy(), gammas=gam.numpy(), projected=proj.numpy(),
                          cost=n * d)


_PIPELINE_MIN = 1 << 16
_streams: dict = {}


def _pipe_streams(dev):
    key = dev.index
    if key not in _streams:
        _streams[key] = tuple(torch.cuda.Stream(device=dev) for _ in range(3))
    return _streams[key]


def _pipeline_bounds(n: int, dev):
    """Chunk boundaries of the pipelined call, in units of one voxel tile per SM (so every chunk
    fills the persistent screen's grid evenly): 1, 2, 4 units first and 4, 2, 1 last, so the
    first upload and the last download that nothing overlaps stay short; 8 units in between."""
    unit = 128 * torch.cuda.get_device_properties(dev).multi_processor_count
    total = -(-n // unit)
    if total <= 16:
        sizes = [1] * total if total <= 4 else [max(1, total // 4)] * 4
    else:
        mid = total - 14
        sizes = [1, 2, 4] + [8] * (mid // 8) + ([mid % 8] if mid % 8 else []) + [4, 2, 1]
    bounds, lo = [], 0
    for k in sizes:
        if lo >= n:
            break
        hi = min(n, lo + k * unit)
        bounds.append((lo, hi))
        lo = hi
    if lo < n:
        bounds.append((lo, n))
    return bounds


def _project_pipelined(zh: torch.Tensor, dd: DeviceDictionary, algo: str, dev):
    """Pinned host input: H2D of chunk i+1 and D2H of chunk i-1 overlap the projection of
    chunk i (copy engines in both directions run concurrently with the SMs)."""
    n, s = int(zh.shape[0]), int(zh.shape[1])
    s_in, s_cmp, s_out = _pipe_streams(dev)
    cur = torch.cuda.current_stream(dev)
    for st in (s_in, s_cmp, s_out):
        st.wait_stream(cur)
    zt = torch.empty((n, s), dtype=zh.dtype, device=dev)
    didx = torch.empty(n, dtype=torch.int64, device=dev)
    dgam = torch.empty(n, dtype=torch.float64, device=dev)
    dproj = torch.empty((n, s), dtype=torch.complex128, device=dev)
    hidx = torch.empty(n, dtype=torch.int64, pin_memory=True)
    hgam = torch.empty(n, dtype=torch.float64, pin_memory=True)
    hproj = torch.empty((n, s), dtype=torch.complex128, pin_memory=True)
    for lo, hi in _pipeline_bounds(n, dev):
        e_in = torch.cuda.Event()
        with torch.cuda.stream(s_in):
            zt[lo:hi].copy_(zh[lo:hi], non_blocking=True)
            e_in.record(s_in)
        s_cmp.wait_event(e_in)
        e_cmp = torch.cuda.Event()
        with torch.cuda.stream(s_cmp):
            project_device(zt[lo:hi], dd, algo=algo, proj_c128=True,
                           out=(didx[lo:hi], dgam[lo:hi], dproj[lo:hi]))
            e_cmp.record(s_cmp)
        s_out.wait_event(e_cmp)
        with torch.cuda.stream(s_out):
            hidx[lo:hi].copy_(didx[lo:hi], non_blocking=True)
            hgam[lo:hi].copy_(dgam[lo:hi], non_blocking=True)
            hproj[lo:hi].copy_(dproj[lo:hi], non_blocking=True)
    s_out.synchronize()
    for t in (zt, didx, dgam, dproj):
        t.record_stream(s_in)
        t.record_stream(s_cmp)
        t.record_stream(s_out)
    return hidx, hgam, hproj


_last_ws: dict = {}   # device index -> (workspace, n, s, stream) of the last project_device call


def _last_workspace(n, s):
    dev = require_cuda()
    rec = _last_ws.get(dev.index)
    if rec is None:
        raise ValueError("no projection has run on this device")
    ws, n0, s0, stream = rec
    if (n is not None and n != n0) or (s is not None and s != s0):
        raise ValueError(f"the last projection on this device was {n0} x s={s0}, not {n} x s={s}")
    return ws, n0, s0, stream


def overflow_counts(n: int = None, s: int = None):
    """(voxels rescanned exhaustively in fp64, voxels with many tcgen05 candidate chunks that
    were rescored warp-cooperatively) of the last ``project_device`` call on the current device
    -- for the pipelined numpy path, its last chunk (diagnostic; read on that call's stream)."""
    lib = _lib.load()
    ws, n0, s0, stream = _last_workspace(n, s)
    out = (ctypes.c_int32 * 2)()
    _lib.check(lib.cbb_project_overflow_counts(ws.data_ptr(), n0, s0, out, stream.cuda_stream),
               "overflow_counts")
    return int(out[0]), int(out[1])


def overflow_count(n: int = None, s: int = None) -> int:
    """Voxels the last ``project_device`` call rescanned exhaustively in fp64 (diagnostic)."""
    return overflow_counts(n, s)[0]
