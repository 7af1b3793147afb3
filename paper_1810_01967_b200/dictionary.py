"""Dictionary data model (host) and its device-resident prepared form.

Host side mirrors the reference types consumed by the hot path
(``coverblip/dictionary.py``): ``ParameterGrid`` (``:40-70``), ``Dictionary``
(``:73-96``), ``CompressedDictionary`` (``:99-128``; ``compress`` ``:116-118``,
``decompress`` ``:120-122``), ``svd_compress`` (``:163-189``) and the surrogate
``generate_fingerprints`` (``:131-160``).  Generation and the SVD are one-time
host setup: they run in numpy exactly like the reference so the
GPU path consumes the same basis.

``DeviceDictionary`` is the B200 form: fp64 atoms for exact rescoring, fp32
planar atoms for FFMA screening, power-of-two scaled fp16 UMMA tiles for tcgen05
screening and the certified rounding bounds (``cbb_dict_prepare``).  Any
object exposing ``.atoms`` or ``.atoms_compressed`` (the reference's duck
typing, ``projection.py:26-29``) can be prepared.
"""

from __future__ import annotations

import ctypes
from collections import OrderedDict
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .device import require_cuda

__all__ = ["ParameterGrid", "Dictionary", "CompressedDictionary", "DeviceDictionary",
           "generate_fingerprints", "fingerprint_trajectories", "svd_compress", "atoms_of",
           "device_dictionary"]


def _parse_axis(values) -> np.ndarray:
    if len(values) and isinstance(values[0], (list, tuple)):
        values = np.concatenate([np.arange(a, b + 0.5 * abs(c), c) for a, b, c in values])
    return np.asarray(values, dtype=float)


@dataclass
class ParameterGrid:
    """T1/T2 (ms) and B0 (Hz) quantisation grids (reference dictionary.py:40-70)."""
    t1_values: np.ndarray
    t2_values: np.ndarray
    b0_values: np.ndarray

    def __post_init__(self):
        self.t1_values = _parse_axis(self.t1_values)
        self.t2_values = _parse_axis(self.t2_values)
        self.b0_values = _parse_axis(self.b0_values)
        for name, ax in (("t1", self.t1_values), ("t2", self.t2_values), ("b0", self.b0_values)):
            if ax.size == 0:
                raise ValueError(f"empty {name} axis")
            if np.any(np.diff(ax) <= 0):
                raise ValueError(f"{name} axis must be strictly increasing")
        if np.any(self.t1_values <= 0) or np.any(self.t2_values <= 0):
            raise ValueError("relaxation times must be positive")

    def combinations(self) -> np.ndarray:
        t1, t2, b0 = np.meshgrid(self.t1_values, self.t2_values, self.b0_values, indexing="ij")
        triples = np.stack([t1.ravel(), t2.ravel(), b0.ravel()], axis=1)
        return triples[triples[:, 1] <= triples[:, 0]]


@dataclass
class Dictionary:
    """Unit atoms (d, L) complex + lookup table (d, 3) (reference dictionary.py:73-96)."""
    atoms: np.ndarray
    norms: np.ndarray
    lookup_table: np.ndarray
    tr_ms: float
    L: int

    @property
    def d(self) -> int:
        return self.atoms.shape[0]

    def lookup(self, j: int):
        if not 0 <= j < self.d:
            raise IndexError(f"atom index {j} out of range [0, {self.d})")
        t1, t2, b0 = self.lookup_table[j]
        return float(t1), float(t2), float(b0)


@dataclass
class CompressedDictionary:
    """Atoms on the top-s SVD subspace (reference dictionary.py:99-128)."""
    basis: np.ndarray
    atoms_compressed: np.ndarray
    renorm_factors: np.ndarray
    s: int
    parent: Dictionary = field(repr=False)

    @property
    def d(self) -> int:
        return self.atoms_compressed.shape[0]

    def lookup(self, j: int):
        return self.parent.lookup(j)

    def compress(self, rows: np.ndarray) -> np.ndarray:
        return rows @ self.basis

    def decompress(self, rows_c: np.ndarray) -> np.ndarray:
        return rows_c @ self.basis.conj().T


def fingerprint_trajectories(params, tr_ms, L):
    """Reference surrogate (dictionary.py:131-141):
    (1 - 2 e^{-t TR/T1}) e^{-t TR/T2} e^{i 2 pi B0 t TR / 1000}, t = 1..L."""
    params = np.atleast_2d(np.asarray(params, dtype=float))
    t = np.arange(1, L + 1, dtype=float)
    t1, t2, b0 = params[:, 0:1], params[:, 1:2], params[:, 2:3]
    envelope = (1.0 - 2.0 * np.exp(-t * tr_ms / t1)) * np.exp(-t * tr_ms / t2)
    return envelope * np.exp(2j * np.pi * b0 * t * tr_ms / 1000.0)


def generate_fingerprints(grid: ParameterGrid, tr_ms: float, L: int) -> Dictionary:
    """Reference dictionary.py:144-160 (surrogate atoms, unit-normalised)."""
    if tr_ms <= 0:
        raise ValueError("TR must be positive")
    if L < 2:
        raise ValueError("sequence length must be at least 2")
    triples = grid.combinations()
    if len(triples) == 0:
        raise ValueError("degenerate grid: no combinations with T2 <= T1")
    raw = fingerprint_trajectories(triples, tr_ms, L)
    norms = np.linalg.norm(raw, axis=1)
    if np.any(norms == 0):
        raise ValueError("degenerate grid: zero-norm fingerprint")
    return Dictionary(atoms=raw / norms[:, None], norms=norms, lookup_table=triples,
                      tr_ms=float(tr_ms), L=int(L))


def svd_compress(dictionary, s: int) -> CompressedDictionary:
    """Top-s right singular subspace (reference dictionary.py:163-189): dense SVD when
    d*L <= 1e7, else the L x L second-moment matrix + eigh; atoms renormalised."""
    L = dictionary.atoms.shape[1]
    if not 1 <= s <= L:
        raise ValueError(f"s must be in [1, {L}], got {s}")
    M = dictionary.atoms
    if M.size <= 10 ** 7:
        _, _, vh = np.linalg.svd(M, full_matrices=False)
        basis = vh.conj().T[:, :s]
    else:
        gram = np.zeros((L, L), dtype=complex)
        step = max(1, 10 ** 7 // L)
        for lo in range(0, M.shape[0], step):
            block = M[lo:lo + step]
            gram += block.T @ block.conj()
        _, vecs = np.linalg.eigh(gram)
        basis = vecs[:, ::-1][:, :s].conj()
    raw = M @ basis
    factors = np.linalg.norm(raw, axis=1)
    return CompressedDictionary(basis=basis, atoms_compressed=raw / factors[:, None],
                                renorm_factors=factors, s=int(s), parent=dictionary)


def atoms_of(dictionary):
    """``projection.py:26-29``: ``.atoms`` else ``.atoms_compressed`` (arrays pass through)."""
    if isinstance(dictionary, (np.ndarray, torch.Tensor)):
        return dictionary
    if isinstance(dictionary, DeviceDictionary):
        return dictionary
    if hasattr(dictionary, "atoms"):
        return dictionary.atoms
    return dictionary.atoms_compressed


def lookup_table_of(dictionary):
    """``solver.py:147-152``: ``.parent.lookup_table`` else ``.lookup_table``."""
    if hasattr(dictionary, "parent"):
        return dictionary.parent.lookup_table
    return getattr(dictionary, "lookup_table", None)


class DeviceDictionary:
    """Prepared, device-resident dictionary (one ``cbb_dict_prepare`` launch)."""

    def __init__(self, atoms, device=None, lookup_table=None):
        dev = require_cuda(device)
        lib = _lib.load()
        if isinstance(atoms, torch.Tensor):
            src = atoms.to(dev)
            if src.dtype not in (torch.complex64, torch.complex128):
                src = src.to(torch.complex128)
            src = src.contiguous()
            shape = tuple(src.shape)
        else:
            a = np.asarray(atoms)
            if not np.iscomplexobj(a):
                a = a.astype(np.complex128)
            elif a.dtype not in (np.complex64, np.complex128):
                a = a.astype(np.complex128)
            shape = a.shape
            src = torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        if len(shape) != 2 or shape[0] < 1 or shape[1] < 1:
            raise ValueError(f"atoms must be a non-empty (d, dim) matrix, got {shape}")
        self.d, self.s = int(shape[0]), int(shape[1])
        self.device = dev
        self.lookup_table = lookup_table
        nbytes = lib.cbb_dict_storage_bytes(self.d, self.s)
        self.storage = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        self.view = _lib.DictView()
        with torch.cuda.device(dev):
            rc = lib.cbb_dict_prepare(src.data_ptr(), int(src.dtype == torch.complex128), self.d,
                                      self.s, self.storage.data_ptr(), ctypes.byref(self.view),
                                      _lib.stream_ptr())
        _lib.check(rc, "cbb_dict_prepare")
        self._src = src  # keep alive until the prepare kernel has run

    @property
    def shape(self):
        return (self.d, self.s)

    def atoms64(self) -> torch.Tensor:
        """fp64 complex atoms (d, s) as a device tensor view."""
        n = self.d * self.s * 16
        raw = self.storage[:n]
        return raw.view(torch.complex128).view(self.d, self.s)

    BOUND_SLOTS = ("delta_h", "dmax", "dh_max", "delta32", "d32max", "scale_d", "delta_split",
                   "dlo_max", "split_row_max", "coherence")

    @property
    def prefer_split(self) -> bool:
        """Auto mode screens with the split (hi/lo fp16, fp32-accumulated) tiles: the sampled
        atoms have near-duplicates inside the fp16 screen's window (``coherence`` bound)."""
        return bool(self.view.prefer_split)

    def representatives(self):
        """For a prune-capable (coherent, bisection-ordered) dictionary: the atom nearest to
        each split tile's centroid, as (atom indices int32 on the device, their prepared
        ``DeviceDictionary``); None otherwise.  A projection onto these few atoms gives every
        voxel a good warm-start atom when it has none (the IPG's first iteration, X = 0)."""
        if not self.view.tile_c:
            return None
        rep = self.__dict__.get("_reps")
        if rep is None:
            d, s = self.d, self.s
            nt = int(self.view.n_tiles2)
            rows = 128 if s <= 10 else 64                              # split_rows(split_kp(s))
            base = self.storage.data_ptr()
            perm = self.storage[int(self.view.tc2_atom) - base:][:4 * d].view(torch.int32)
            perm = perm.to(torch.int64)
            a = self.atoms64()[perm]                                   # bisection order
            idx = torch.arange(nt * rows, device=self.device).clamp_max(d - 1)
            tiles = a[idx].view(nt, rows, s)
            valid = (torch.arange(nt * rows, device=self.device) < d).view(nt, rows)
            cnt = valid.sum(1, keepdim=True)
            cen = (tiles * valid[..., None]).sum(1) / cnt
            dist = torch.linalg.vector_norm(tiles - cen[:, None, :], dim=2)
            dist = torch.where(valid, dist, torch.full_like(dist, float("inf")))
            best = dist.argmin(1)                                      # row inside the tile
            pos = torch.arange(nt, device=self.device) * rows + best
            atoms_idx = perm[pos].to(torch.int32)
            rep = self._reps = (atoms_idx, DeviceDictionary(self.atoms64()[atoms_idx.long()],
                                                             self.device))
        return rep

    def bounds(self) -> dict:
        """Certified rounding bounds of the prepared copies (``cbb_project.cuh`` kB* slots)."""
        off = int(self.view.bounds) - self.storage.data_ptr()
        vals = self.storage[off:off + 4 * len(self.BOUND_SLOTS)].view(torch.float32).cpu().tolist()
        return dict(zip(self.BOUND_SLOTS, vals))


_cache_lock = __import__("threading").Lock()
_cache: OrderedDict = OrderedDict()
_CACHE_MAX = 6


def device_dictionary(dictionary, device=None) -> DeviceDictionary:
    """Prepared device copy of ``dictionary`` (cached per atom array; dictionaries are
    immutable, reference SPEC "shared and immutable")."""
    if isinstance(dictionary, DeviceDictionary):
        return dictionary
    atoms = atoms_of(dictionary)
    if isinstance(atoms, DeviceDictionary):
        return atoms
    dev = require_cuda(device)
    if isinstance(atoms, torch.Tensor):
        key = ("t", atoms.data_ptr(), tuple(atoms.shape), str(atoms.dtype), dev.index)
    else:
        arr = np.asarray(atoms)
        key = ("n", id(atoms), arr.__array_interface__["data"][0], arr.shape, str(arr.dtype),
               dev.index)
    with _cache_lock:
        hit = _cache.get(key)
        if hit is not None:
            _cache.move_to_end(key)
            return hit[0]
    dd = DeviceDictionary(atoms, dev, lookup_table=lookup_table_of(dictionary)
                          if not isinstance(dictionary, (np.ndarray, torch.Tensor)) else None)
    with _cache_lock:
        _cache[key] = (dd, atoms)  # holding `atoms` pins its id while cached
        while len(_cache) > _CACHE_MAX:
            _cache.popitem(last=False)
    return dd
