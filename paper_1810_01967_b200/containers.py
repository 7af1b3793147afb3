"""Dictionary / measurement / pattern containers, read straight to the device.

Byte-compatible with the reference's wire formats:

* ``CBDICT01`` (``dictionary.py:192-224``): magic, ``<qqd`` (d, L, tr_ms), d x L ``<c16`` atoms,
  d ``<f8`` norms, d x 3 ``<f8`` lookup table (T1, T2, B0).
* ``CBMEAS01`` (``forward_model.py:310-329``): magic, ``<qq`` (rows, cols), rows x cols ``<c16``.
* EPI pattern JSON (``forward_model.py:290-307``): ``{h, w, L, lines_per_frame, offset_rule}``.

``save_*`` / ``load_*`` mirror the reference functions (same names, same ``ValueError`` messages).
``load_dictionary_device`` / ``load_measurements_device`` stream the payload from the file through
two pinned staging buffers into device tensors (copies overlap the file reads), so a multi-GB
dictionary never needs a full host copy; the device tensors come out in the layouts the B200 path
consumes (atoms (d, L) complex128 for ``DeviceDictionary``; measurements frame-major (L, rows)
complex64 for the solver).
"""

from __future__ import annotations

import json
import os
import struct

import numpy as np
import torch

from .device import require_cuda
from .dictionary import Dictionary
from .forward_model import SamplingPattern, make_epi_pattern

__all__ = ["save_dictionary", "load_dictionary", "load_dictionary_device", "save_measurements",
           "load_measurements", "load_measurements_device", "save_pattern", "load_pattern",
           "DICT_MAGIC", "MEAS_MAGIC"]

DICT_MAGIC = b"CBDICT01"
MEAS_MAGIC = b"CBMEAS01"
_DICT_HDR = "<qqd"
_MEAS_HDR = "<qq"
_STAGE_BYTES = 64 << 20


# ------------------------------------------------------------------ host (reference API)
def save_dictionary(dictionary, path) -> None:
    """``dictionary.py:192-201``."""
    with open(path, "wb") as fh:
        fh.write(DICT_MAGIC)
        fh.write(struct.pack(_DICT_HDR, dictionary.d, dictionary.L, dictionary.tr_ms))
        fh.write(np.ascontiguousarray(dictionary.atoms, dtype="<c16").tobytes())
        fh.write(np.ascontiguousarray(dictionary.norms, dtype="<f8").tobytes())
        fh.write(np.ascontiguousarray(dictionary.lookup_table, dtype="<f8").tobytes())


def _dict_header(fh):
    if fh.read(len(DICT_MAGIC)) != DICT_MAGIC:
        raise ValueError("not a dictionary file")
    header = fh.read(struct.calcsize(_DICT_HDR))
    if len(header) != struct.calcsize(_DICT_HDR):
        raise ValueError("truncated dictionary file")
    d, L, tr_ms = struct.unpack(_DICT_HDR, header)
    return int(d), int(L), float(tr_ms)


def load_dictionary(path) -> Dictionary:
    """``dictionary.py:204-224``."""
    with open(path, "rb") as fh:
        d, L, tr_ms = _dict_header(fh)
        blob = fh.read()
    need = d * L * 16 + d * 8 + d * 24
    if len(blob) < need:
        raise ValueError("truncated dictionary file")
    atoms = np.frombuffer(blob[:d * L * 16], dtype="<c16").reshape(d, L)
    off = d * L * 16
    norms = np.frombuffer(blob[off:off + d * 8], dtype="<f8")
    off += d * 8
    lookup = np.frombuffer(blob[off:off + d * 24], dtype="<f8").reshape(d, 3)
    return Dictionary(atoms=np.array(atoms), norms=np.array(norms), lookup_table=np.array(lookup),
                      tr_ms=float(tr_ms), L=int(L))


def save_measurements(Y, path) -> None:
    """``forward_model.py:310-315``."""
    Y = np.asarray(Y)
    with open(path, "wb") as fh:
        fh.write(MEAS_MAGIC)
        fh.write(struct.pack(_MEAS_HDR, *Y.shape))
        fh.write(np.ascontiguousarray(Y, dtype="<c16").tobytes())


def _meas_header(fh):
    if fh.read(len(MEAS_MAGIC)) != MEAS_MAGIC:
        raise ValueError("not a measurement file")
    header = fh.read(16)
    if len(header) != 16:
        raise ValueError("truncated measurement file")
    rows, cols = struct.unpack(_MEAS_HDR, header)
    return int(rows), int(cols)


def load_measurements(path) -> np.ndarray:
    """``forward_model.py:318-329``."""
    with open(path, "rb") as fh:
        rows, cols = _meas_header(fh)
        blob = fh.read()
    if len(blob) < rows * cols * 16:
        raise ValueError("truncated measurement file")
    return np.frombuffer(blob[:rows * cols * 16], dtype="<c16").reshape(rows, cols).copy()


def save_pattern(pattern: SamplingPattern, path) -> None:
    """``forward_model.py:290-298`` (EPI-style patterns only)."""
    if getattr(pattern, "lines_per_frame", None) is None:
        raise ValueError("only EPI-style patterns can be saved as JSON")
    h, w = pattern.spatial_shape
    with open(path, "w") as fh:
        json.dump({"h": h, "w": w, "L": pattern.L, "lines_per_frame": pattern.lines_per_frame,
                   "offset_rule": "cyclic"}, fh)


def load_pattern(path) -> SamplingPattern:
    """``forward_model.py:301-307``."""
    with open(path) as fh:
        spec = json.load(fh)
    if spec.get("offset_rule") != "cyclic":
        raise ValueError("unknown offset rule in pattern file")
    return make_epi_pattern((spec["h"], spec["w"]), spec["lines_per_frame"], spec["L"])


# ------------------------------------------------------------------ straight to the device
def _stream_to_device(fh, nbytes: int, dst: torch.Tensor) -> None:
    """Read `nbytes` from the file position into the byte view of `dst` (device) through two
    pinned staging buffers: the H2D copy of one chunk overlaps the read of the next."""
    out = dst.view(torch.uint8).reshape(-1)
    if out.numel() != nbytes:
        raise ValueError("staging size mismatch")
    chunk = min(_STAGE_BYTES, max(nbytes, 1))
    bufs = [torch.empty(chunk, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    events = [None, None]
    stream = torch.cuda.Stream(device=dst.device)
    done = 0
    k = 0
    while done < nbytes:
        n = min(chunk, nbytes - done)
        b = k & 1
        if events[b] is not None:
            events[b].synchronize()          # the previous copy out of this buffer finished
        got = fh.readinto(memoryview(bufs[b].numpy())[:n])
        if got != n:
            raise ValueError("truncated file")
        with torch.cuda.stream(stream):
            out[done:done + n].copy_(bufs[b][:n], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
        events[b] = ev
        done += n
        k += 1
    stream.synchronize()
    torch.cuda.current_stream(dst.device).wait_stream(stream)


def load_dictionary_device(path, device=None):
    """CBDICT01 -> (atoms (d, L) complex128 device tensor, Dictionary metadata with atoms=None
    replaced by a zero-width host placeholder).  The norms and lookup table stay on the host
    (they are d-length metadata)."""
    dev = require_cuda(device)
    size = os.path.getsize(path)
    with open(path, "rb") as fh:
        d, L, tr_ms = _dict_header(fh)
        hdr = len(DICT_MAGIC) + struct.calcsize(_DICT_HDR)
        if size - hdr < d * L * 16 + d * 32:
            raise ValueError("truncated dictionary file")
        atoms = torch.empty((d, L), dtype=torch.complex128, device=dev)
        _stream_to_device(fh, d * L * 16, atoms)
        norms = np.frombuffer(fh.read(d * 8), dtype="<f8").copy()
        lookup = np.frombuffer(fh.read(d * 24), dtype="<f8").reshape(d, 3).copy()
    meta = Dictionary(atoms=np.zeros((d, 0), dtype=complex), norms=norms, lookup_table=lookup,
                      tr_ms=tr_ms, L=L)
    return atoms, meta


def load_measurements_device(path, device=None, frame_major: bool = True) -> torch.Tensor:
    """CBMEAS01 (rows = c*m, cols = L) -> device complex64; frame-major (L, c*m) by default (the
    solver's layout), else the reference's (c*m, L)."""
    dev = require_cuda(device)
    size = os.path.getsize(path)
    with open(path, "rb") as fh:
        rows, cols = _meas_header(fh)
        if size - len(MEAS_MAGIC) - 16 < rows * cols * 16:
            raise ValueError("truncated measurement file")
        raw = torch.empty((rows, cols), dtype=torch.complex128, device=dev)
        _stream_to_device(fh, rows * cols * 16, raw)
    out = raw.to(torch.complex64)
    return out.transpose(0, 1).contiguous() if frame_major else out
