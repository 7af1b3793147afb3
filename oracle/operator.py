"""Cartesian acquisition operator, restated from the reference (TEST INFRASTRUCTURE).

Reference: ``coverblip/forward_model.py``.
* ``CartesianOperator.apply``   follows ``forward_model.py:123-142``: per coil,
  multiply by the coil map, unitary DFT over the spatial axes of the
  voxel-major ``(n, L)`` image reshaped to ``(*spatial, L)`` (``norm="ortho"``,
  ``:138``), then ``take_along_axis`` with ``pattern.T`` (``:133,140``).
* ``CartesianOperator.adjoint`` follows ``forward_model.py:144-167``: zero
  fill with ``put_along_axis``, inverse unitary DFT, conjugate-coil sum.
* ``make_epi_pattern``          follows ``forward_model.py:170-187``.
* 3-D spatial shapes (SURVEY 8c restatement 2, needed by cfg4; the reference
  is 2-D only) use ``np.fft.fftn`` over all spatial axes with the same
  gather/scatter semantics.
"""

from __future__ import annotations

import numpy as np


def make_epi_pattern(spatial_shape, lines_per_frame, L):
    """``forward_model.py:170-187``: frame t samples rows
    ``(t % (h//k) + (h//k)*j) % h`` (j < k), all columns; returns (L, m)."""
    h, w = spatial_shape
    k = lines_per_frame
    if k > h:
        raise ValueError("lines_per_frame exceeds grid height")
    if k < 1 or L < 1:
        raise ValueError("lines_per_frame and L must be positive")
    spacing = h // k
    cols = np.arange(w)
    frames = []
    for t in range(L):
        rows = (t % spacing + spacing * np.arange(k)) % h
        frames.append((rows[:, None] * w + cols[None, :]).ravel())
    return np.array(frames, dtype=np.int64)


class CartesianOperator:
    """A = P_Omega F S with exact adjoint (``forward_model.py:82-167``)."""

    def __init__(self, pattern, spatial_shape, coil_maps=None,
                 identity_transform=False):
        self.pattern = np.asarray(pattern, dtype=np.int64)   # (L, m)
        self.spatial_shape = tuple(int(x) for x in spatial_shape)
        self.n = int(np.prod(self.spatial_shape))
        self.L, self.m = self.pattern.shape
        self.c = 1 if coil_maps is None else coil_maps.shape[0]
        self.coil_maps = (np.ones((1, self.n), dtype=complex)
                          if coil_maps is None else np.asarray(coil_maps))
        self.identity_transform = identity_transform
        self.weights = None
        self._axes = tuple(range(len(self.spatial_shape)))

    def apply(self, X):
        X = np.asarray(X)
        if X.shape != (self.n, self.L):
            raise ValueError(
                f"dimension mismatch: expected {(self.n, self.L)} image, "
                f"got {X.shape}")
        X = X.astype(complex, copy=False)
        idx = self.pattern.T
        out = np.empty((self.c * self.m, self.L), dtype=complex)
        for ci in range(self.c):
            sx = X * self.coil_maps[ci][:, None]
            if not self.identity_transform:
                sx = np.fft.fftn(sx.reshape(*self.spatial_shape, self.L),
                                 axes=self._axes,
                                 norm="ortho").reshape(self.n, self.L)
            out[ci * self.m:(ci + 1) * self.m] = np.take_along_axis(
                sx, idx, axis=0)
        return out

    def adjoint(self, Y):
        Y = np.asarray(Y)
        if Y.shape != (self.c * self.m, self.L):
            raise ValueError(
                f"dimension mismatch: expected {(self.c * self.m, self.L)} "
                f"measurements, got {Y.shape}")
        Y = Y.astype(complex, copy=False)
        idx = self.pattern.T
        X = np.zeros((self.n, self.L), dtype=complex)
        for ci in range(self.c):
            K = np.zeros((self.n, self.L), dtype=complex)
            np.put_along_axis(K, idx, Y[ci * self.m:(ci + 1) * self.m],
                              axis=0)
            if not self.identity_transform:
                K = np.fft.ifftn(K.reshape(*self.spatial_shape, self.L),
                                 axes=self._axes,
                                 norm="ortho").reshape(self.n, self.L)
            X += K * self.coil_maps[ci].conj()[:, None]
        return X


def simulate_measurements(X0, A, snr_db, seed):
    """``harness.py:145-153``: Y = A X0 + xi, ||xi|| = ||A X0|| 10^(-snr/20)."""
    Y = A.apply(X0)
    if np.isinf(snr_db):
        return Y
    rng = np.random.default_rng(seed)
    xi = rng.standard_normal(Y.shape) + 1j * rng.standard_normal(Y.shape)
    xi *= np.linalg.norm(Y) / np.linalg.norm(xi) * 10 ** (-snr_db / 20.0)
    return Y + xi
