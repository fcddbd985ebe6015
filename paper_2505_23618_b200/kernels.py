"""The kernel plugin API, backed by sm_100a kernels.

Mirrors the reference's backend module contract (reference
pkg/src/dctadjust/kernels/__init__.py:33-73): `BACKEND_NAME`, the seven batch
functions dct2 / idct2 / dst3 / idst3 / band / subblock / dense over (nvec, N)
batches returning NEW arrays, `available_backends()` and `use_backend()`.
There is exactly one backend ("cuda"); no CPU fallback, no multi-backend
dispatch -- asking for any other backend is a ValueError, as in the reference.
Each call is one C-ABI call (include/dctadj.h) on torch's current stream.
"""
from __future__ import annotations

import contextlib
import sys

import numpy as np

from . import _device, _lib
from .errors import ShapeError

BACKEND_NAME = "cuda"
BACKEND = BACKEND_NAME


def _batch(x):
    t, as_np = _device.to_device(x)
    if t.dim() != 2:
        raise ShapeError(f"expected a (nvec, N) batch, got ndim={t.dim()}")
    return t, as_np


def _prim(fn: str, x):
    t, as_np = _batch(x)
    y = _device.empty_like(t)
    _lib.call(fn, t.data_ptr(), y.data_ptr(), t.shape[0], t.shape[1], _device.dtype_code(t),
              _device.stream_handle())
    return _device.from_device(y, as_np)


def dct2(x):
    """Orthonormal DCT-2 of each row (reference _fastcore.pyx:188-198)."""
    return _prim("dctadj_dct2", x)


def idct2(y):
    """Inverse DCT-2 (= DCT-3) of each row (_fastcore.pyx:201-211)."""
    return _prim("dctadj_idct2", y)


def dst3(x):
    """DST-3 via reversal + inverse DCT-2 + sign flips (_fastcore.pyx:214-230)."""
    return _prim("dctadj_dst3", x)


def idst3(y):
    """Inverse DST-3 (_fastcore.pyx:233-250)."""
    return _prim("dctadj_idst3", y)


def _host_matrix(m, what: str):
    a = np.ascontiguousarray(np.asarray(m, dtype=np.float64))
    if a.ndim != 2:
        raise ShapeError(f"{what} must be 2-D, got ndim={a.ndim}")
    return a


def band(a, taps: int, x):
    """y[i, r] = sum_{|r-j| < taps} a[r, j] x[i, j] (_fastcore.pyx:253-273)."""
    am = _host_matrix(a, "band matrix")
    t, as_np = _batch(x)
    n = t.shape[1]
    if am.shape != (n, n):
        raise ShapeError(f"band matrix {am.shape} vs batch width {n}")
    y = _device.empty_like(t)
    _lib.call("dctadj_band", _lib.dptr(am), int(taps), t.data_ptr(), y.data_ptr(), t.shape[0],
              n, _device.dtype_code(t), _device.stream_handle())
    return _device.from_device(y, as_np)


def subblock(blk, x):
    """Copy of x with the leading B entries replaced by blk @ x[:B]; the tail
    is passed through bit-identically (_fastcore.pyx:276-290)."""
    bm = _host_matrix(blk, "sub-block")
    t, as_np = _batch(x)
    b = bm.shape[0]
    if bm.shape != (b, b) or b > t.shape[1]:
        raise ShapeError(f"sub-block {bm.shape} vs batch width {t.shape[1]}")
    y = _device.empty_like(t)
    _lib.call("dctadj_subblock", _lib.dptr(bm), b, t.data_ptr(), y.data_ptr(), t.shape[0],
              t.shape[1], _device.dtype_code(t), _device.stream_handle())
    return _device.from_device(y, as_np)


def dense(m, x):
    """y = x @ m.T, m of shape (R, N) (_fastcore.pyx:293-307)."""
    mm = _host_matrix(m, "dense matrix")
    t, as_np = _batch(x)
    if mm.shape[1] != t.shape[1]:
        raise ShapeError(f"dense matrix {mm.shape} vs batch width {t.shape[1]}")
    y = _device.empty_like(t, (t.shape[0], mm.shape[0]))
    _lib.call("dctadj_dense", _lib.dptr(mm), mm.shape[0], t.data_ptr(), y.data_ptr(),
              t.shape[0], t.shape[1], _device.dtype_code(t), _device.stream_handle())
    return _device.from_device(y, as_np)


def available_backends() -> dict[str, object]:
    return {BACKEND_NAME: sys.modules[__name__]}


@contextlib.contextmanager
def use_backend(name: str):
    """Kept for API compatibility with the reference; only "cuda" exists."""
    mod = available_backends().get(name)
    if mod is None:
        raise ValueError(f"backend {name!r} is not available")
    yield mod
