"""ctypes binding of ``libcoverblip_b200.so`` (C ABI in ``include/coverblip_b200.h``).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_1810_01967_b200/csrc``).  There is NO fallback: if the library
is missing or a CUDA device is absent, every hot-path call raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CBB_LIB_PATH") or os.path.join(_HERE, "libcoverblip_b200.so")

c_int = ctypes.c_int
c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_size = ctypes.c_size_t
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p

ERR_ARGUMENT, ERR_CUDA, ERR_UNSUPPORTED, ERR_CUFFT = 1, 2, 3, 4

ALGOS = {"auto": 0, "tcgen05": 1, "ffma": 2, "exhaustive": 3, "tcgen05_split": 4}


class DictView(ctypes.Structure):
    _fields_ = [("d", c_i64), ("s", c_i32), ("s_pad", c_i32), ("kpad", c_i32),
                ("n_btiles", c_i32), ("atoms64", c_vp), ("atoms32", c_vp),
                ("atoms_tc", c_vp), ("bounds", c_vp), ("atoms_tc2", c_vp),
                ("prefer_split", c_i32), ("reserved", c_i32), ("n_tiles2", c_i32),
                ("reserved2", c_i32), ("tc2_atom", c_vp), ("tc2_pos", c_vp), ("tile_c", c_vp),
                ("tile_r", c_vp), ("ctr_tc2", c_vp), ("tile_rs", c_vp)]


# name -> (restype, argtypes); every symbol declared in include/coverblip_b200.h
SIGNATURES = {
    "cbb_abi_version": (c_int, []),
    "cbb_last_error": (ctypes.c_char_p, []),
    "cbb_device_sm_count": (c_int, [ctypes.POINTER(c_int)]),
    "cbb_stats_kernel_launches": (ctypes.c_ulonglong, []),
    "cbb_timing_enable": (c_int, [c_i32]),
    "cbb_timing_last_ms": (c_int, [ctypes.POINTER(ctypes.c_float)]),
    "cbb_dict_storage_bytes": (c_size, [c_i64, c_i32]),
    "cbb_dict_prepare": (c_int, [c_vp, c_i32, c_i64, c_i32, c_vp, ctypes.POINTER(DictView), c_vp]),
    "cbb_project_workspace_bytes": (c_size, [c_i64, c_i32]),
    "cbb_project_workspace_bytes_dict": (c_size, [c_i64, ctypes.POINTER(DictView)]),
    "cbb_project_cone_exact": (c_int, [c_vp, c_i32, c_i64, ctypes.POINTER(DictView), c_vp, c_i32,
                                       c_vp, c_vp, c_i32, c_vp, c_size, c_i32, c_vp]),
    "cbb_project_step": (c_int, [c_vp, c_vp, c_dbl, c_vp, c_i64, ctypes.POINTER(DictView), c_vp,
                                 c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_size, c_i32, c_vp]),
    "cbb_project_step_ex": (c_int, [c_vp, c_vp, c_dbl, c_vp, c_vp, c_i64,
                                    ctypes.POINTER(DictView), c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                    c_vp, c_vp, c_size, c_i32, c_vp]),
    "cbb_trial_state_bytes": (c_size, []),
    "cbb_trial_init": (c_int, [c_vp, c_vp]),
    "cbb_trial_carry": (c_int, [c_vp, c_vp]),
    "cbb_graph_capture_begin": (c_int, [c_vp, ctypes.POINTER(c_vp)]),
    "cbb_graph_while_begin": (c_int, [c_vp, c_vp]),
    "cbb_trial_decide": (c_int, [c_vp, c_vp, c_vp, c_vp, c_dbl, c_i32]),
    "cbb_graph_while_end": (c_int, [c_vp]),
    "cbb_graph_capture_end": (c_int, [c_vp]),
    "cbb_graph_launch": (c_int, [c_vp, c_vp]),
    "cbb_graph_destroy": (c_int, [c_vp]),
    "cbb_project_best": (c_int, [c_vp, c_i32, c_i64, ctypes.POINTER(DictView), c_i64, c_vp, c_vp,
                                 c_vp, c_size, c_i32, c_vp]),
    "cbb_scaled_rows": (c_int, [ctypes.POINTER(DictView), c_i64, c_vp, c_vp, c_i64, c_vp, c_i32,
                                c_vp]),
    "cbb_project_overflow_counts": (c_int, [c_vp, c_i64, c_i32, c_vp, c_vp]),
    "cbb_project_overflow_count": (c_int, [c_vp, c_i64, c_i32, ctypes.POINTER(c_int), c_vp]),
    "cbb_project_hint": (c_int, [c_vp, c_vp, c_dbl, c_vp, c_vp, c_i64, ctypes.POINTER(DictView), c_vp, c_vp,
                         c_vp, c_size, c_vp]),
    "cbb_project_prune_detail": (c_int, [c_vp, c_size, c_i64, ctypes.POINTER(DictView), c_vp, c_vp, c_vp]),
    "cbb_project_prune_stats": (c_int, [c_vp, c_size, c_i64, ctypes.POINTER(DictView),
                                        ctypes.POINTER(c_i64), ctypes.POINTER(c_i64), c_vp]),
    "cbb_project_prologue": (c_int, [c_vp, c_i32, c_i64, ctypes.POINTER(DictView), c_vp, c_size,
                                     c_vp]),
    "cbb_debug_tc_scores": (c_int, [c_vp, ctypes.POINTER(DictView), c_i32, c_i32, c_vp, c_vp]),
    "cbb_op_create": (c_int, [c_i32, ctypes.POINTER(c_i32), c_i32, c_i32, c_vp, c_i32,
                              ctypes.POINTER(c_vp)]),
    "cbb_op_destroy": (c_int, [c_vp]),
    "cbb_op_set_coils": (c_int, [c_vp, c_i32, c_vp]),
    "cbb_op_workspace_bytes": (c_size, [c_vp]),
    "cbb_op_workspace_bytes_compressed": (c_size, [c_vp, c_i32]),
    "cbb_op_apply": (c_int, [c_vp, c_vp, c_vp, c_vp, c_vp]),
    "cbb_op_adjoint": (c_int, [c_vp, c_vp, c_vp, c_vp, c_vp]),
    "cbb_op_apply_compressed": (c_int, [c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, c_vp]),
    "cbb_op_apply_norm2_compressed": (c_int, [c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, c_vp]),
    "cbb_op_adjoint_compressed": (c_int, [c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, c_vp]),
    "cbb_residual": (c_int, [c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "cbb_scaled_residual_norm2": (c_int, [c_vp, c_dbl, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "cbb_norm2_c64": (c_int, [c_vp, c_i64, c_vp, c_vp, c_vp]),
    "cbb_scale_c64": (c_int, [c_vp, c_dbl, c_i64, c_vp]),
    "cbb_reduce_workspace_bytes": (c_size, []),
    "cbb_argmax_select": (c_int, [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp]),
}

_lock = threading.Lock()
_lib = None


class NativeError(RuntimeError):
    pass


def load():
    """Load the library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                    "(there is no CPU fallback for the B200 hot path)")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def exported_symbols():
    return sorted(SIGNATURES)


def check(rc: int, what: str):
    """Map a C status to the reference's exception types."""
    if rc == 0:
        return
    msg = load().cbb_last_error().decode(errors="replace")
    if rc == ERR_ARGUMENT:
        raise ValueError(f"{what}: invalid argument {msg}".strip())
    raise NativeError(f"{what} failed with status {rc}: {msg}")


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None -> NULL)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_ptr(stream=None) -> int:
    """cudaStream_t of `stream`, or of the current device's current stream.  The raw-stream
    query skips torch.cuda.current_stream()'s Python wrapper (~10 us per call, a third of the
    host time of a latency-bound cfg0 IPG solve)."""
    import torch
    if stream is not None:
        return stream.cuda_stream
    return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())
