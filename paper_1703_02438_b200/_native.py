"""ctypes binding of libnmkgpu.so (the C ABI declared in include/nmk_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` / ``make``.  There
is no fallback: if the library or a CUDA device is missing, every product
entry point raises :class:`NativeUnavailable`.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libnmkgpu.so")

NMK_OK = 0
NMK_ERR_ARG = -1
NMK_ERR_CUDA = -2
NMK_ERR_EMPTY_HIST = -6
NMK_ERR_NEEDS_SPARSE = -7
NMK_SPAN_SPARSE = 0xFFFFFFFFFFFFFFFF
NMK_DEV_MAX_SEG = 4

NMK_F32 = 0
NMK_F64 = 1

u64 = ctypes.c_uint64
i32 = ctypes.c_int
u32 = ctypes.c_uint32
dbl = ctypes.c_double
vp = ctypes.c_void_p
sz = ctypes.c_size_t
u64p = ctypes.POINTER(ctypes.c_uint64)


class NmkStats(ctypes.Structure):
    _fields_ = [("gmin", ctypes.c_double), ("gmax", ctypes.c_double),
                ("nvalid", ctypes.c_uint64), ("reserved", ctypes.c_uint64)]


class NmkModel(ctypes.Structure):
    _fields_ = [("bits", ctypes.c_int32), ("k", ctypes.c_int32), ("status", ctypes.c_int32),
                ("m_selectable", ctypes.c_int32), ("tol_bin", ctypes.c_double),
                ("coverage", ctypes.c_uint64 * 17)]


class NmkDecodeErr(ctypes.Structure):
    _fields_ = [("bad_index", ctypes.c_uint32), ("max_bad_index", ctypes.c_uint32),
                ("exhausted", ctypes.c_uint32), ("reserved", ctypes.c_uint32)]


class NmkSegmentInfo(ctypes.Structure):
    _fields_ = [("inc_before", ctypes.c_uint64), ("n_sentinel", ctypes.c_uint64)]


# name -> (restype, argtypes); mirrors include/nmk_b200.h one to one
SIGNATURES = {
    "nmk_last_error": (ctypes.c_char_p, []),
    "nmk_version": (i32, []),
    "nmk_ratio": (i32, [vp, vp, u64, i32, vp, vp, vp]),
    "nmk_minmax_ws_bytes": (sz, [u64]),
    "nmk_minmax": (i32, [vp, vp, u64, i32, vp, vp, vp, sz, vp]),
    "nmk_hist_dense": (i32, [vp, vp, u64, i32, vp, dbl, u64, vp, vp]),
    "nmk_hist_sparse_ws_bytes": (sz, [u64]),
    "nmk_hist_sparse": (i32, [vp, vp, u64, i32, vp, dbl, vp, vp, vp, vp, sz, vp]),
    "nmk_hist_merge_ws_bytes": (sz, [u64]),
    "nmk_hist_merge": (i32, [vp, vp, u64, vp, vp, sz, vp]),
    "nmk_hist_values_ws_bytes": (sz, [u64]),
    "nmk_hist_values": (i32, [vp, vp, u64, dbl, dbl, vp, vp, vp, vp, sz, vp]),
    "nmk_hist_merge_values": (i32, [vp, vp, u64, vp, vp, sz, vp]),
    "nmk_coverage": (i32, [vp, vp, u64, vp, vp, dbl, i32, i32, vp, vp, vp]),
    "nmk_nearest_center": (i32, [vp, u64, vp, i32, vp, vp, vp]),
    "nmk_compressible_mask": (i32, [vp, vp, u64, vp, i32, dbl, vp, vp, vp]),
    "nmk_select": (i32, [vp, vp, u64, vp, vp, dbl, dbl, i32, u64, i32, vp, vp, vp, u64, vp, vp]),
    "nmk_encode_ws_bytes": (sz, [u64, u64, u64, i32]),
    "nmk_encode": (i32, [vp, vp, u64, u64, u64, i32, vp, vp, i32, i32, dbl, dbl, u64, vp, u64, vp,
                         vp, vp, vp, vp, sz, vp]),
    "nmk_decode_ws_bytes": (sz, [u64p, u64p, i32, u64, u64]),
    "nmk_decode": (i32, [vp, u64, u64, i32, u64, u64, vp, vp, i32, vp, u64, vp, vp, i32,
                         u64p, u64p, u64p, i32, vp, vp, vp, sz, vp]),
    "nmk_hist_prep": (i32, [vp, dbl, u64, vp, vp]),
    "nmk_hist_dense_dev": (i32, [vp, vp, vp, u64, i32, vp, dbl, vp, vp]),
    "nmk_hist_dense_dev2": (i32, [vp, vp, vp, u64, i32, vp, dbl, vp, u64, i32, vp]),
    "nmk_encode_dev": (i32, [vp, vp, u64, u64, u64, i32, vp, vp, vp, i32, i32, dbl, u64, vp, u64, vp,
                             vp, vp, vp, vp, sz, vp]),
    "nmk_encode_keyed_dev": (i32, [vp, vp, dbl, vp, vp, u64, u64, u64, i32, vp, vp, vp, i32, i32, dbl, u64, vp,
                                   u64, vp, vp, vp, vp, vp, sz, vp]),
    "nmk_decode_dev": (i32, [vp, u64, u64, i32, u64, u64, vp, vp, vp, vp, vp, vp, vp, i32,
                             u64p, u64p, u64p, i32, vp, vp, vp, sz, vp]),
    "nmk_minmax_prep": (i32, [vp, vp, u64, i32, vp, vp, dbl, u64, vp, vp, sz, vp]),
    "nmk_encode_keyed_dev2": (i32, [vp, vp, dbl, vp, vp, u64, u64, u64, i32, vp, vp, vp, i32, i32, dbl, u64, vp,
                                    u64, vp, vp, vp, vp, i32, vp, sz, vp]),
    "nmk_encode_ws_mode_offset": (sz, [u64, u64, u64, i32]),
    "nmk_decode_dev2": (i32, [vp, u64, u64, i32, u64, u64, vp, vp, vp, vp, vp, vp, vp, i32,
                              u64p, u64p, u64p, i32, vp, vp, i32, vp, sz, vp]),
    "nmk_decode_ring_for": (i32, [u64, u64]),
    "nmk_deflate_ws_bytes": (sz, [u64, u64, u32]),
    "nmk_deflate_bound": (u64, [u64, u64, u32]),
    "nmk_deflate": (i32, [vp, u64, u64, u64, u64, u32, vp, vp, vp, sz, vp]),
    "nmk_inflate": (i32, [vp, vp, u64, vp, u64, vp, vp, vp, vp]),
    "nmk_sort64_ws_bytes": (sz, [u64, i32]),
    "nmk_sort64": (i32, [vp, vp, vp, vp, u64, vp, sz, vp]),
    "nmk_pack": (i32, [vp, u64, i32, vp, vp]),
    "nmk_unpack": (i32, [vp, u64, i32, vp, vp]),
}


class NativeUnavailable(RuntimeError):
    """The CUDA library or device is missing — there is no CPU fallback."""


class NativeError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


_lib = None
_lock = threading.Lock()


def load(path: str | None = None) -> ctypes.CDLL:
    """Load libnmkgpu.so and bind every exported symbol (no device needed)."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise NativeUnavailable(
                f"{p} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` or `make`")
        lib = ctypes.CDLL(p)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def lib() -> ctypes.CDLL:
    return _lib if _lib is not None else load()


def check(code: int) -> None:
    if code != NMK_OK:
        msg = lib().nmk_last_error().decode(errors="replace")
        raise NativeError(code, msg or f"libnmkgpu error {code}")


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the B200 path has no CPU fallback")
    lib()
    return torch


def dtype_code(np_dtype) -> int:
    import numpy as np
    dt = np.dtype(np_dtype)
    if dt.kind != "f" or dt.itemsize not in (4, 8):
        raise ValueError(f"unsupported snapshot dtype {dt}")
    return NMK_F32 if dt.itemsize == 4 else NMK_F64
