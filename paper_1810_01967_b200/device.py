"""Device plumbing: CUDA checks, grow-only workspaces, pinned host staging.

PyTorch provides device memory, streams and the pinned host allocator; the
arithmetic of the hot path lives in ``libcoverblip_b200.so``.
"""

from __future__ import annotations

import threading

import numpy as np
import torch

_ws_lock = threading.Lock()
_workspaces: dict = {}


def require_cuda(device=None) -> torch.device:
    """Fail loudly without a GPU: the B200 path has no CPU fallback."""
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_1810_01967_b200 needs a CUDA (sm_100a) device; no CPU fallback exists")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device)
    if dev.type != "cuda":
        raise RuntimeError(f"device {dev} is not a CUDA device")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


def workspace(nbytes: int, device: torch.device, tag: str = "default") -> torch.Tensor:
    """Grow-only per-(device, tag, stream) scratch buffer."""
    idx = device.index if device.index is not None else torch._C._cuda_getDevice()
    key = (idx, tag, torch._C._cuda_getCurrentRawStream(idx))
    with _ws_lock:
        buf = _workspaces.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)
            _workspaces[key] = buf
        return buf


def pinned_empty(shape, dtype) -> np.ndarray:
    """numpy array backed by pinned (page-locked) host memory (for fast H2D/D2H)."""
    tdt = {np.dtype(np.complex128): torch.complex128, np.dtype(np.complex64): torch.complex64,
           np.dtype(np.float64): torch.float64, np.dtype(np.float32): torch.float32,
           np.dtype(np.int64): torch.int64, np.dtype(np.int32): torch.int32}[np.dtype(dtype)]
    return torch.empty(tuple(shape), dtype=tdt, pin_memory=True).numpy()


def to_device(arr: np.ndarray, device: torch.device, dtype=None) -> torch.Tensor:
    """Host numpy -> device tensor (non-blocking when the host buffer is pinned)."""
    a = np.ascontiguousarray(arr if dtype is None else arr.astype(dtype, copy=False))
    t = torch.from_numpy(a)
    return t.to(device, non_blocking=True)
