"""Exact cone projection, restated from the reference (TEST INFRASTRUCTURE).

Reference: ``coverblip/projection.py``.
* ``project_cone_exact``  follows ``projection.py:45-67``: row-blocked Gram
  product ``Re(Z @ atoms^H)`` with blocks of ``max(1, 5e7 // d)`` rows
  (``:58``), first-index ``argmax`` (``:62``), gammas via the shared einsum
  (``_gammas_for``, ``:38-42``), write-back ``gamma * atom`` (``:64``) and
  ``cost = n * d`` (``:67``).
* ``top2``                is SURVEY 8c restatement (1): the same fp64 blocked
  product, recording the best and second-best real scores so parity tests can
  classify documented near-ties ``(s1 - s2) / |s1| < 1e-5``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

NEAR_TIE_REL = 1e-5


@dataclass
class ConeProjection:
    """Mirror of ``projection.py:18-23``."""
    indices: np.ndarray
    gammas: np.ndarray
    projected: np.ndarray
    cost: int


def atoms_of(dictionary) -> np.ndarray:
    """``projection.py:26-29``: ``.atoms`` else ``.atoms_compressed``."""
    if isinstance(dictionary, np.ndarray):
        return dictionary
    if hasattr(dictionary, "atoms"):
        return dictionary.atoms
    return dictionary.atoms_compressed


def as_array(Z) -> np.ndarray:
    """``projection.py:32-35``."""
    if hasattr(Z, "data") and not isinstance(Z, np.ndarray):
        Z = Z.data
    return np.asarray(Z)


def gammas_for(Z, atoms, indices):
    """``projection.py:38-42``."""
    raw = np.einsum("ij,ij->i", Z, atoms[indices].conj()).real
    return np.maximum(raw, 0.0)


def project_cone_exact(Z, dictionary) -> ConeProjection:
    """``projection.py:45-67`` restated (complex128 arithmetic)."""
    Z = as_array(Z)
    atoms = atoms_of(dictionary)
    if Z.ndim != 2 or Z.shape[1] != atoms.shape[1]:
        raise ValueError(
            f"dimension mismatch: image is {Z.shape}, atoms are {atoms.shape}")
    block = max(1, 5 * 10 ** 7 // max(atoms.shape[0], 1))
    indices = np.empty(Z.shape[0], dtype=np.int64)
    at_h = atoms.conj().T
    for lo in range(0, Z.shape[0], block):
        corr = (Z[lo:lo + block] @ at_h).real
        indices[lo:lo + block] = np.argmax(corr, axis=1)
    gammas = gammas_for(Z, atoms, indices)
    projected = gammas[:, None] * atoms[indices]
    return ConeProjection(indices=indices, gammas=gammas, projected=projected,
                          cost=Z.shape[0] * atoms.shape[0])


def top2(Z, atoms, block_rows: int | None = None):
    """Best / second-best ``Re<Z_v, D_j>`` per row (fp64), first-index argmax.

    Returns ``(idx1, s1, s2)``.  Same arithmetic as ``projection.py:61``.
    """
    Z = np.asarray(Z)
    d = atoms.shape[0]
    block = block_rows or max(1, 5 * 10 ** 7 // max(d, 1))
    n = Z.shape[0]
    idx1 = np.empty(n, dtype=np.int64)
    s1 = np.empty(n)
    s2 = np.full(n, -np.inf)
    at_h = atoms.conj().T
    for lo in range(0, n, block):
        corr = (Z[lo:lo + block] @ at_h).real
        i1 = np.argmax(corr, axis=1)
        r = np.arange(corr.shape[0])
        idx1[lo:lo + block] = i1
        s1[lo:lo + block] = corr[r, i1]
        if d > 1:
            corr[r, i1] = -np.inf
            s2[lo:lo + block] = corr.max(axis=1)
    return idx1, s1, s2


def near_tie_mask(s1, s2, rel=NEAR_TIE_REL):
    """Documented near-ties: top-2 gap below ``rel`` relative to ``|s1|``."""
    gap = s1 - s2
    return gap <= rel * np.abs(s1)
