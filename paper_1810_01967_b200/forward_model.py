"""Acquisition operator A = P_Omega F (per-frame unitary DFT) on the GPU.

Drop-in for the reference ``coverblip.forward_model`` pieces on the hot path:
``MrfImage`` (``forward_model.py:38-50``), ``SamplingPattern`` (``:53-79``),
``ForwardOperator`` with ``apply`` / ``adjoint`` (``:82-167``),
``make_epi_pattern`` (``:170-187``) and ``make_cartesian_operator`` (``:190-198``).
The dense Gaussian operator (``:201-208``, test-only in the reference) is kept
for API completeness and runs as a cuBLAS matrix product.

Cartesian apply/adjoint run in ``libcoverblip_b200.so``: cuFFT batched C2C over
the L frames (frame-major device layout) with hand-written gather / zero-fill
scatter / transpose kernels; the unitary 1/sqrt(n) is folded into them.  The
public methods take and return numpy arrays in the reference layouts and dtypes
(voxel-major (n, L) images, (m, L) measurements, complex128); the solver uses the
``fm_*`` device methods, which keep complex64 frame-major (L, m) measurements.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .device import require_cuda, workspace

__all__ = ["MrfImage", "SamplingPattern", "ForwardOperator", "make_epi_pattern",
           "make_cartesian_operator", "make_gaussian_operator", "as_device_operator"]


@dataclass
class MrfImage:
    """Spatio-temporal image: row v is voxel v, column t is frame t (forward_model.py:38-50)."""
    data: np.ndarray
    spatial_shape: tuple

    def __post_init__(self):
        if self.data.shape[0] != int(np.prod(self.spatial_shape)):
            raise ValueError("spatial shape does not match number of voxels")
        if not np.all(np.isfinite(self.data)):
            raise ValueError("image contains non-finite entries")


class SamplingPattern:
    """Per-frame sampled flat voxel indices, (L, m) (forward_model.py:53-79)."""

    def __init__(self, indices, spatial_shape, lines_per_frame=None):
        self.indices = np.asarray(indices, dtype=np.int64)
        self.spatial_shape = tuple(int(x) for x in spatial_shape)
        self.lines_per_frame = lines_per_frame
        n = int(np.prod(self.spatial_shape))
        if self.indices.ndim != 2:
            raise ValueError("indices must be an L x m array")
        if self.indices.min() < 0 or self.indices.max() >= n:
            raise ValueError("sample index out of range")
        srt = np.sort(self.indices, axis=1)
        dup = np.any(srt[:, 1:] == srt[:, :-1], axis=1)
        if dup.any():
            raise ValueError(f"duplicate sample index in frame {int(np.argmax(dup))}")

    @property
    def L(self) -> int:
        return self.indices.shape[0]

    @property
    def m(self) -> int:
        return self.indices.shape[1]


def make_epi_pattern(spatial_shape, lines_per_frame: int, L: int) -> SamplingPattern:
    """forward_model.py:170-187: frame t samples rows (t % (h//k) + (h//k) j) % h, j < k."""
    h, w = spatial_shape
    k = lines_per_frame
    if k > h:
        raise ValueError("lines_per_frame exceeds grid height")
    if k < 1 or L < 1:
        raise ValueError("lines_per_frame and L must be positive")
    spacing = h // k
    t = np.arange(L)[:, None]
    rows = (t % spacing + spacing * np.arange(k)[None, :]) % h          # (L, k)
    idx = (rows[:, :, None] * w + np.arange(w)[None, None, :]).reshape(L, k * w)
    return SamplingPattern(indices=idx, spatial_shape=(h, w), lines_per_frame=k)


def _dims_of(shape):
    shape = tuple(int(x) for x in shape)
    if len(shape) not in (2, 3):
        raise ValueError("spatial shape must be 2-D or 3-D")
    return shape


class ForwardOperator:
    """A = P_Omega F S (cartesian_dft) or a dense Gaussian matrix (forward_model.py:82-113)."""

    def __init__(self, kind, n, m, L, c=1, pattern=None, coil_maps=None, weights=None,
                 matrix=None, identity_transform=False, spatial_shape=None, device=None):
        if kind not in ("cartesian_dft", "dense_gaussian"):
            raise ValueError(f"unknown operator kind {kind!r}")
        self.kind, self.n, self.m, self.L, self.c = kind, int(n), int(m), int(L), int(c)
        self.pattern = pattern
        self.weights = weights
        self.matrix = matrix
        self.identity_transform = bool(identity_transform)
        self.coil_maps = coil_maps
        self.device = require_cuda(device)
        self._op = None
        if weights is not None and np.any(np.asarray(weights) < 0):
            raise ValueError("weights must be nonnegative")
        if kind == "cartesian_dft":
            if pattern is None:
                raise ValueError("cartesian operator needs a pattern")
            self.spatial_shape = _dims_of(pattern.spatial_shape)
            if coil_maps is None:
                coil_maps = np.ones((self.c, self.n), dtype=complex)   # forward_model.py:104-105
            elif tuple(np.shape(coil_maps)) != (self.c, self.n):
                raise ValueError("coil map shape mismatch")
            self.coil_maps = coil_maps
            lib = _lib.load()
            pat = np.asarray(pattern.indices)
            if pat.shape != (self.L, self.m):
                raise ValueError("pattern shape does not match (L, m)")
            self._pattern_dev = torch.from_numpy(pat.astype(np.int32)).to(self.device)
            dims = (ctypes.c_int32 * 3)(*(list(self.spatial_shape) + [1])[:3])
            handle = ctypes.c_void_p()
            _lib.check(lib.cbb_op_create(len(self.spatial_shape), dims, self.L, self.m,
                                         self._pattern_dev.data_ptr(),
                                         1 if self.identity_transform else 0,
                                         ctypes.byref(handle)), "cbb_op_create")
            self._op = handle
            # unit maps stay implicit (no multiply); otherwise a device copy the op points to
            self._coils_dev = None
            if self.c > 1 or not np.allclose(np.asarray(coil_maps), 1.0):
                self._coils_dev = torch.from_numpy(
                    np.ascontiguousarray(coil_maps, dtype=np.complex64)).to(self.device)
            _lib.check(lib.cbb_op_set_coils(
                handle, self.c, None if self._coils_dev is None else self._coils_dev.data_ptr()),
                "cbb_op_set_coils")
            self._ws_bytes = int(lib.cbb_op_workspace_bytes(handle))
            self._wsbuf = {}    # per-operator workspaces (freed with the operator)
        else:
            if matrix is None:
                raise ValueError("gaussian operator needs a matrix")
            self.spatial_shape = spatial_shape
            self._mat = torch.from_numpy(np.asarray(matrix, dtype=np.complex64)).to(self.device)

    def __del__(self):
        op = getattr(self, "_op", None)
        if op is not None:
            try:
                _lib.load().cbb_op_destroy(op)
            except Exception:
                pass
            self._op = None

    # ------------------------------------------------------------------ reference API
    def _check_image(self, X):
        if isinstance(X, MrfImage):
            X = X.data
        if isinstance(X, torch.Tensor):
            if tuple(X.shape) != (self.n, self.L):
                raise ValueError(f"dimension mismatch: expected {(self.n, self.L)} image, "
                                 f"got {tuple(X.shape)}")
            return X
        X = np.asarray(X)
        if X.shape != (self.n, self.L):
            raise ValueError(
                f"dimension mismatch: expected {(self.n, self.L)} image, got {X.shape}")
        return X

    def apply(self, X):
        """Forward map to measurements (c*m, L) (forward_model.py:123-142)."""
        X = self._check_image(X)
        host = not isinstance(X, torch.Tensor)
        Xd = self._to_dev(X)
        Yfm = self.fm_apply(Xd)                       # (L, c*m) frame-major complex64
        Y = Yfm.transpose(0, 1)
        return Y.contiguous().cpu().numpy().astype(np.complex128) if host else Y

    def adjoint(self, Y):
        """Exact adjoint, returns an (n, L) image (forward_model.py:144-167)."""
        shape = tuple(Y.shape)
        if shape != (self.c * self.m, self.L):
            raise ValueError(f"dimension mismatch: expected {(self.c * self.m, self.L)} "
                             f"measurements, got {shape}")
        host = not isinstance(Y, torch.Tensor)
        Yd = self._to_dev(Y).transpose(0, 1).contiguous()
        X = self.fm_adjoint(Yd)
        return X.cpu().numpy().astype(np.complex128) if host else X

    # ------------------------------------------------------------------ device API
    def _to_dev(self, a):
        if isinstance(a, torch.Tensor):
            t = a.to(self.device)
            return t.to(torch.complex64).contiguous()
        return torch.from_numpy(np.ascontiguousarray(np.asarray(a), dtype=np.complex64)).to(
            self.device)

    def _ws(self, s=None):
        """This operator's workspace: the frame-stack layout of the uncompressed calls, or the
        s-channel layout (2 c s n complex64 + partials) of the compressed calls with rank s."""
        key = "full" if s is None else int(s)
        nbytes = (self._ws_bytes if s is None else
                  int(_lib.load().cbb_op_workspace_bytes_compressed(self._op, int(s))))
        buf = self._wsbuf.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            self._wsbuf[key] = buf
        return buf

    @property
    def cm(self) -> int:
        """Measurement columns per frame (c coils x m samples)."""
        return self.c * self.m

    def fm_apply(self, X: torch.Tensor) -> torch.Tensor:
        """(n, L) complex64 -> (L, c*m) complex64 frame-major."""
        X = X.contiguous()
        if self.kind == "dense_gaussian":
            return self._dense_apply(X)
        Y = torch.empty((self.L, self.cm), dtype=torch.complex64, device=self.device)
        _lib.check(_lib.load().cbb_op_apply(self._op, X.data_ptr(), Y.data_ptr(),
                                            self._ws().data_ptr(), _lib.stream_ptr()),
                   "cbb_op_apply")
        return Y

    def fm_adjoint(self, Yfm: torch.Tensor) -> torch.Tensor:
        """(L, c*m) complex64 frame-major -> (n, L) complex64."""
        Yfm = Yfm.contiguous()
        if self.kind == "dense_gaussian":
            return self._dense_adjoint(Yfm)
        X = torch.empty((self.n, self.L), dtype=torch.complex64, device=self.device)
        _lib.check(_lib.load().cbb_op_adjoint(self._op, Yfm.data_ptr(), X.data_ptr(),
                                              self._ws().data_ptr(), _lib.stream_ptr()),
                   "cbb_op_adjoint")
        return X

    def fm_apply_compressed(self, Xc, V, out=None):
        """A(Xc V^H): (n, s) c64 coordinates -> (L, c*m) frame-major (s-channel operator:
        c*s FFTs of the subspace channel images, no (L, n) frame stack)."""
        Xc, V = Xc.contiguous(), V.contiguous()
        s = int(Xc.shape[1])
        if self.kind == "dense_gaussian" or s > 32:   # decompress, then the frame path
            Y = self.fm_apply(Xc @ V.conj().transpose(0, 1))
            if out is None:
                return Y
            out.copy_(Y)
            return out
        Y = out if out is not None else torch.empty((self.L, self.cm), dtype=torch.complex64,
                                                    device=self.device)
        _lib.check(_lib.load().cbb_op_apply_compressed(self._op, Xc.data_ptr(), V.data_ptr(), s,
                                                       Y.data_ptr(), self._ws(s).data_ptr(),
                                                       _lib.stream_ptr()),
                   "cbb_op_apply_compressed")
        return Y

    def fm_apply_norm2_compressed(self, Xc, V, out):
        """||A(Xc V^H)||^2 into the fp64 device scalar `out` (apply_diff, solver.py:135)."""
        Xc, V = Xc.contiguous(), V.contiguous()
        s = int(Xc.shape[1])
        if self.kind == "dense_gaussian" or s > 32:
            Y = self.fm_apply_compressed(Xc, V)
            return _norm2(Y, out)
        _lib.check(_lib.load().cbb_op_apply_norm2_compressed(self._op, Xc.data_ptr(),
                                                             V.data_ptr(), s, out.data_ptr(),
                                                             self._ws(s).data_ptr(),
                                                             _lib.stream_ptr()),
                   "cbb_op_apply_norm2_compressed")
        return out

    def fm_adjoint_compressed(self, R, V, out=None):
        """(A^H R) V: (L, c*m) frame-major residual -> (n, s) coordinates (s-channel adjoint:
        deterministic per-channel k-space build, c*s inverse FFTs, coil combine)."""
        R, V = R.contiguous(), V.contiguous()
        s = int(V.shape[1])
        if self.kind == "dense_gaussian" or s > 32:   # frame path, then compress
            G = self.fm_adjoint(R) @ V
            if out is None:
                return G
            out.copy_(G)
            return out
        G = out if out is not None else torch.empty((self.n, s), dtype=torch.complex64,
                                                    device=self.device)
        _lib.check(_lib.load().cbb_op_adjoint_compressed(self._op, R.data_ptr(), V.data_ptr(), s,
                                                         G.data_ptr(), self._ws(s).data_ptr(),
                                                         _lib.stream_ptr()),
                   "cbb_op_adjoint_compressed")
        return G

    # dense Gaussian (test-only operator kind in the reference) -- cuBLAS products
    def _dense_apply(self, X):
        if self._mat.dim() == 2:
            return (self._mat @ X).transpose(0, 1).contiguous()
        return torch.einsum("tmn,nt->tm", self._mat, X).contiguous()

    def _dense_adjoint(self, Yfm):
        if self._mat.dim() == 2:
            return self._mat.conj().transpose(0, 1) @ Yfm.transpose(0, 1)
        return torch.einsum("tmn,tm->nt", self._mat.conj(), Yfm).contiguous()


def _norm2(a: torch.Tensor, out: torch.Tensor):
    lib = _lib.load()
    ws = workspace(lib.cbb_reduce_workspace_bytes(), a.device, "reduce")
    _lib.check(lib.cbb_norm2_c64(a.data_ptr(), a.numel(), out.data_ptr(), ws.data_ptr(),
                                 _lib.stream_ptr()), "cbb_norm2_c64")
    return out


def make_cartesian_operator(pattern: SamplingPattern, coil_maps=None, weights=None,
                            identity_transform=False, device=None) -> ForwardOperator:
    """forward_model.py:190-198."""
    shape = pattern.spatial_shape
    c = 1 if coil_maps is None else coil_maps.shape[0]
    return ForwardOperator(kind="cartesian_dft", n=int(np.prod(shape)), m=pattern.m,
                           L=pattern.L, c=c, pattern=pattern, coil_maps=coil_maps,
                           weights=weights, identity_transform=identity_transform,
                           device=device)


def make_gaussian_operator(n: int, m: int, L: int, seed: int, per_frame: bool = False,
                           device=None) -> ForwardOperator:
    """forward_model.py:201-208 (same seeded matrix as the reference)."""
    rng = np.random.default_rng(seed)
    shape = (L, m, n) if per_frame else (m, n)
    mat = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    mat /= np.sqrt(2.0) * np.sqrt(m)
    return ForwardOperator(kind="dense_gaussian", n=n, m=m, L=L, matrix=mat, device=device)


def as_device_operator(A, device=None) -> ForwardOperator:
    """Wrap a reference ``ForwardOperator`` (duck-typed: kind, n, m, L, pattern, ...)."""
    if isinstance(A, ForwardOperator):
        return A
    kind = getattr(A, "kind", None)
    if kind == "cartesian_dft":
        pat = A.pattern
        sp = SamplingPattern(np.asarray(pat.indices), pat.spatial_shape,
                             getattr(pat, "lines_per_frame", None))
        return ForwardOperator(kind="cartesian_dft", n=A.n, m=A.m, L=A.L, c=getattr(A, "c", 1),
                               pattern=sp, coil_maps=getattr(A, "coil_maps", None),
                               weights=getattr(A, "weights", None),
                               identity_transform=getattr(A, "identity_transform", False),
                               device=device)
    if kind == "dense_gaussian":
        return ForwardOperator(kind="dense_gaussian", n=A.n, m=A.m, L=A.L, matrix=A.matrix,
                               weights=getattr(A, "weights", None), device=device)
    raise ValueError(f"unsupported operator {A!r}")
