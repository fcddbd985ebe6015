"""ctypes binding of libdctadj.so (the C-ABI declared in include/dctadj.h).

This is the binding a maintainer of the reference would add: plain pointers,
sizes and a stream handle in, an int status out, mapped to the reference's
exception classes.  There is no fallback: if the library or a CUDA device is
missing, every call raises CudaError.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

from . import errors

LIB_PATH = Path(os.environ.get("DCTADJ_LIB", Path(__file__).resolve().parent / "libdctadj.so"))

F32, F64 = 0, 1
BASE_DCT2, BASE_DST3, BASE_DCT3 = 0, 1, 2
ADJ_NONE, ADJ_BAND, ADJ_SUBBLOCK, ADJ_DENSE = 0, 1, 2, 3
SIDE_PRE, SIDE_POST = 0, 1

_ERRORS = {
    1: errors.InvalidDimensionError,
    2: errors.ShapeError,
    3: errors.PatternError,
    4: errors.ConfigurationError,
    5: errors.KindMismatchError,
    6: errors.CudaError,
    7: errors.UnsupportedError,
    8: ValueError,
}


class Axis(ctypes.Structure):
    """struct dctadj_axis"""

    _fields_ = [
        ("n", ctypes.c_int32),
        ("base", ctypes.c_int32),
        ("adj", ctypes.c_int32),
        ("side", ctypes.c_int32),
        ("taps", ctypes.c_int32),
        ("order", ctypes.c_int32),
        ("mat", ctypes.POINTER(ctypes.c_double)),
        ("givens", ctypes.POINTER(ctypes.c_double)),
        ("ngivens", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_DP = ctypes.POINTER(ctypes.c_double)
_AP = ctypes.POINTER(Axis)

SIGNATURES = {
    "dctadj_dct2": [_P, _P, _I64, _I32, _I32, _P],
    "dctadj_idct2": [_P, _P, _I64, _I32, _I32, _P],
    "dctadj_dst3": [_P, _P, _I64, _I32, _I32, _P],
    "dctadj_idst3": [_P, _P, _I64, _I32, _I32, _P],
    "dctadj_band": [_DP, _I32, _P, _P, _I64, _I32, _I32, _P],
    "dctadj_subblock": [_DP, _I32, _P, _P, _I64, _I32, _I32, _P],
    "dctadj_dense": [_DP, _I32, _P, _P, _I64, _I32, _I32, _P],
    "dctadj_forward_1d": [_AP, _P, _P, _I64, _I32, _P],
    "dctadj_inverse_1d": [_AP, _P, _P, _I64, _I32, _P],
    "dctadj_forward_2d": [_AP, _AP, _P, _P, _I64, _I32, _P],
    "dctadj_inverse_2d": [_AP, _AP, _P, _P, _I64, _I32, _P],
    "dctadj_roundtrip_2d": [_AP, _AP, _P, _P, _P, _I64, _I32, _P],
    "dctadj_roundtrip_fused": [_AP, _AP, _I32],
    "dctadj_forward_2d_host": [_AP, _AP, _P, _P, _I64, _I32, _I32],
    "dctadj_inverse_2d_host": [_AP, _AP, _P, _P, _I64, _I32, _I32],
    "dctadj_roundtrip_2d_host": [_AP, _AP, _P, _P, _P, _I64, _I32, _I32],
    "dctadj_forward_frames": [_AP, _AP, _P, _P, _I32, _I32, _I32, _I32, _P],
    "dctadj_inverse_frames": [_AP, _AP, _P, _P, _I32, _I32, _I32, _I32, _P],
    "dctadj_forward_frames_exact": [_AP, _AP, _AP, _AP, _P, _P, _P, _P, _I32, _I32, _I32, _I32, _P],
    "dctadj_copy_tiles": [_P, _P, _I64, _I32, _I32, _I32, _P],
    "dctadj_encoder_eval": [_AP, _AP, _P, ctypes.POINTER(_P), _I64, _I32, _P],
    "dctadj_mixed_create": [_P, _P, _P, _I64, _P, _I32, _I64, ctypes.POINTER(_P)],
    "dctadj_mixed_forward": [_P, _AP, _P, _P, _I32, _P],
    "dctadj_mixed_inverse": [_P, _AP, _P, _P, _I32, _P],
    "dctadj_mixed_roundtrip": [_P, _AP, _P, _P, _P, _I32, _P],
    "dctadj_mixed_roundtrip_fused": [_P, _AP, _I32],
    "dctadj_design_cd": [_I32, _P, _P, _P, _I32, _I32, _P, _P, _I32, _P, _I32, ctypes.c_double,
                         _P, _P, _P, _P, _I32],
    "dctadj_mixed_destroy": [_P],
    "dctadj_status_string": [_I32],
    "dctadj_last_error": [],
    "dctadj_version": [],
    "dctadj_kernel_count": [],
    "dctadj_dense_cache_state": [ctypes.POINTER(_I32), ctypes.POINTER(_I32)],
    "dctadj_tuning_build": [],
    "dctadj_pdl_probe": [_P, _P, ctypes.c_uint64, _P, ctypes.c_uint64, _I32],
}

_lib = None


def load() -> ctypes.CDLL:
    """Load (once) and type the library.  Raises CudaError if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise errors.CudaError(
            f"{LIB_PATH} is not built; run __graft_entry__.build() (nvcc, sm_100a)")
    lib = ctypes.CDLL(str(LIB_PATH))
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_char_p if name in ("dctadj_status_string",
                                                 "dctadj_last_error") else ctypes.c_int32
    _lib = lib
    return lib


def check(status: int) -> None:
    if status == 0:
        return
    lib = load()
    msg = lib.dctadj_last_error().decode(errors="replace")
    name = lib.dctadj_status_string(status).decode()
    raise _ERRORS.get(status, errors.DctAdjustError)(msg or name)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))


def dptr(a) -> ctypes.POINTER(ctypes.c_double):
    """Pointer to a C-contiguous float64 numpy array (caller keeps it alive)."""
    return a.ctypes.data_as(_DP)
