"""Python face of the CPU parity oracle.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
--impl reference) may import this module -- as the checker, never as the thing
measured or shipped.  Two oracles live here:

* `liboracle.so` -- the C restatement of the reference path
  (dctadj_oracle.c; each function cites the reference file:line it follows).
  Pinned against golden vectors produced by the reference itself
  (tests/golden/gen_golden.py) in tests/test_oracle.py.
* `_ref/_fastcore*.so` -- the reference's own compiled core, built from
  /root/reference/pkg/src/dctadjust/kernels/_fastcore.pyx by `make ref`
  (only in the build container; the .so then travels with the repo).  The
  policy layer around it (forward_adjusted = band -> dst3 etc.) is restated in
  `RefPipeline` below from reference pipeline.py:158-191 since the reference's
  Python sources do not travel.
"""
from __future__ import annotations

import ctypes
import importlib.util
import os
import subprocess
import sysconfig
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / f"_fastcore{sysconfig.get_config_var('EXT_SUFFIX')}"

BASE_DCT2, BASE_DST3, BASE_DCT3 = 0, 1, 2
ADJ_NONE, ADJ_BAND, ADJ_SUBBLOCK, ADJ_DENSE = 0, 1, 2, 3
SIDE_PRE, SIDE_POST = 0, 1


class _Axis(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("base", ctypes.c_int32), ("adj", ctypes.c_int32),
                ("side", ctypes.c_int32), ("taps", ctypes.c_int32), ("order", ctypes.c_int32),
                ("mat", ctypes.POINTER(ctypes.c_double))]


@dataclass(frozen=True)
class OAxis:
    """One axis of an adjusted transform, in plain data."""
    n: int
    base: int = BASE_DCT2
    adj: int = ADJ_NONE
    side: int = SIDE_POST
    taps: int = 0
    order: int = 0
    mat: np.ndarray | None = None

    def c(self):
        m = None if self.mat is None else np.ascontiguousarray(self.mat, dtype=np.float64)
        ax = _Axis(self.n, self.base, self.adj, self.side, self.taps, self.order,
                   m.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if m is not None else None)
        return ax, m


_lib = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        _lib = ctypes.CDLL(str(LIB))
        dp = ctypes.POINTER(ctypes.c_double)
        for name in ("or_dct2", "or_idct2", "or_dst3", "or_idst3"):
            getattr(_lib, name).argtypes = [dp, dp, ctypes.c_int64, ctypes.c_int]
        for name in ("or_band", "or_subblock", "or_dense"):
            getattr(_lib, name).argtypes = [dp, ctypes.c_int, dp, dp, ctypes.c_int64, ctypes.c_int]
        ap = ctypes.POINTER(_Axis)
        _lib.or_adjusted_1d.argtypes = [ap, ctypes.c_int, dp, dp, ctypes.c_int64]
        _lib.or_adjusted_2d.argtypes = [ap, ap, ctypes.c_int, dp, dp, ctypes.c_int64, ctypes.c_int]
        fp = ctypes.POINTER(ctypes.c_float)
        _lib.or_adjusted_2d_f32.argtypes = [ap, ap, ctypes.c_int, fp, fp, ctypes.c_int64,
                                            ctypes.c_int]
    return _lib


def _d(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _f64(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


def _unary(name, x):
    x = _f64(x)
    y = np.empty_like(x)
    rc = getattr(lib(), name)(_d(x), _d(y), x.shape[0], x.shape[1])
    if rc:
        raise ValueError(f"{name}: bad size {x.shape}")
    return y


def dct2(x): return _unary("or_dct2", x)
def idct2(x): return _unary("or_idct2", x)
def dst3(x): return _unary("or_dst3", x)
def idst3(x): return _unary("or_idst3", x)


def band(a, taps, x):
    a, x = _f64(a), _f64(x)
    y = np.empty_like(x)
    lib().or_band(_d(a), int(taps), _d(x), _d(y), x.shape[0], x.shape[1])
    return y


def subblock(blk, x):
    blk, x = _f64(blk), _f64(x)
    y = np.empty_like(x)
    lib().or_subblock(_d(blk), blk.shape[0], _d(x), _d(y), x.shape[0], x.shape[1])
    return y


def dense(m, x):
    m, x = _f64(m), _f64(x)
    y = np.empty((x.shape[0], m.shape[0]))
    lib().or_dense(_d(m), m.shape[0], _d(x), _d(y), x.shape[0], x.shape[1])
    return y


def adjusted_1d(ax: OAxis, x, inverse=False):
    x = _f64(x)
    y = np.empty_like(x)
    c, _keep = ax.c()
    lib().or_adjusted_1d(ctypes.byref(c), int(inverse), _d(x), _d(y), x.shape[0])
    return y


def adjusted_2d(ah: OAxis, av: OAxis, x, inverse=False, threads=1):
    """(nblk, H, W) blocks; float32 in -> float32 out (computed in float64)."""
    ch, _kh = ah.c()
    cv, _kv = av.c()
    if np.asarray(x).dtype == np.float32:
        x = np.ascontiguousarray(x)
        y = np.empty_like(x)
        fp = ctypes.POINTER(ctypes.c_float)
        lib().or_adjusted_2d_f32(ctypes.byref(ch), ctypes.byref(cv), int(inverse),
                                 x.ctypes.data_as(fp), y.ctypes.data_as(fp), x.shape[0], threads)
        return y
    x = _f64(x)
    y = np.empty_like(x)
    lib().or_adjusted_2d(ctypes.byref(ch), ctypes.byref(cv), int(inverse), _d(x), _d(y),
                         x.shape[0], threads)
    return y


def threads_available() -> int:
    return len(os.sched_getaffinity(0))


# ------------------------------------------------------------------ reference core
def ref_fastcore():
    """The reference's compiled core (oracle/_ref), or None if not built."""
    if not REF_SO.exists():
        return None
    spec = importlib.util.spec_from_file_location("_fastcore", REF_SO)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


class RefPipeline:
    """Reference policy layer over its compiled core: _apply_adjustment,
    _base_forward/_inverse and forward/inverse_adjusted restated from reference
    pipeline.py:158-191, and the 2-D composition of SURVEY.md 3.3 (rows then
    columns through numpy transposes, as _dct2_2d, pipeline.py:236-239)."""

    def __init__(self, core=None):
        self.k = core or ref_fastcore()
        if self.k is None:
            raise FileNotFoundError(f"{REF_SO} not built (make -C oracle ref)")

    def _adj(self, ax: OAxis, x, transpose):
        m = ax.mat.T if transpose else ax.mat
        if ax.adj == ADJ_BAND:
            return self.k.band(np.ascontiguousarray(m), ax.taps, x)
        if ax.adj == ADJ_SUBBLOCK:
            b = ax.order
            return self.k.subblock(np.ascontiguousarray(m[:b, :b]), x)
        if ax.adj == ADJ_DENSE:
            return self.k.dense(np.ascontiguousarray(m), x)
        return x

    def _base(self, ax: OAxis, x, inverse):
        if ax.base == BASE_DCT2:
            return self.k.idct2(x) if inverse else self.k.dct2(x)
        if ax.base == BASE_DST3:
            return self.k.idst3(x) if inverse else self.k.dst3(x)
        return self.k.dct2(x) if inverse else self.k.idct2(x)

    def forward(self, ax: OAxis, x):
        x = np.asarray(x, dtype=float)
        if ax.side == SIDE_PRE:
            return self._base(ax, self._adj(ax, x, False), False)
        return self._adj(ax, self._base(ax, x, False), False)

    def inverse(self, ax: OAxis, y):
        y = np.asarray(y, dtype=float)
        if ax.side == SIDE_PRE:
            return self._adj(ax, self._base(ax, y, True), True)
        return self._base(ax, self._adj(ax, y, True), True)

    def forward_2d(self, ah: OAxis, av: OAxis, x):
        b, h, w = x.shape
        rows = self.forward(ah, np.asarray(x, dtype=float).reshape(b * h, w)).reshape(b, h, w)
        cols = np.ascontiguousarray(rows.transpose(0, 2, 1)).reshape(b * w, h)
        return np.ascontiguousarray(self.forward(av, cols).reshape(b, w, h).transpose(0, 2, 1))

    def inverse_2d(self, ah: OAxis, av: OAxis, y):
        b, h, w = y.shape
        cols = np.ascontiguousarray(np.asarray(y, dtype=float).transpose(0, 2, 1)).reshape(b * w, h)
        t = np.ascontiguousarray(self.inverse(av, cols).reshape(b, w, h).transpose(0, 2, 1))
        return self.inverse(ah, t.reshape(b * h, w)).reshape(b, h, w)


# ------------------------------------------------------------------ full-batch checkers
class _CheckResult(ctypes.Structure):
    _fields_ = [("max_err", ctypes.c_double), ("worst", ctypes.c_int64), ("over", ctypes.c_int64)]


def _check_lib():
    lb = lib()
    if not getattr(lb, "_check_typed", False):
        ap, vp = ctypes.POINTER(_Axis), ctypes.c_void_p
        i32p, i64p = ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int64)
        rp = ctypes.POINTER(_CheckResult)
        lb.or_check_2d.argtypes = [ap, ap, ctypes.c_int, ctypes.c_int, vp, vp, ctypes.c_int64,
                                   ctypes.c_int, ctypes.c_double, rp]
        lb.or_check_mixed.argtypes = [ap, ctypes.c_int, i32p, i32p, i64p, ctypes.c_int64,
                                      ctypes.c_int, ctypes.c_int, vp, vp, ctypes.c_int,
                                      ctypes.c_double, rp]
        lb.or_check_frames.argtypes = [ap, ap, ctypes.c_int, vp, vp, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int, ctypes.c_int, ctypes.c_double, rp]
        lb._check_typed = True
    return lb


def _dtype_code(a: np.ndarray) -> int:
    if a.dtype == np.float32:
        return 0
    if a.dtype == np.float64:
        return 1
    raise TypeError(f"checker needs float32 / float64 arrays, got {a.dtype}")


def _result(r: _CheckResult, nblk: int) -> dict:
    return {"max_err": float(r.max_err), "worst_block": int(r.worst), "over_tol": int(r.over),
            "blocks": int(nblk)}


def check_2d(ah: OAxis, av: OAxis, x, y, inverse=False, threads=None, tol=0.0) -> dict:
    """Every block of y against the oracle applied to x ((nblk, H, W), same dtype):
    {max_err, worst_block, over_tol, blocks} (per-block normwise relative error)."""
    x, y = np.ascontiguousarray(x), np.ascontiguousarray(y)
    if x.shape != y.shape or x.dtype != y.dtype or x.ndim != 3:
        raise ValueError(f"check_2d: x {x.shape} {x.dtype} vs y {y.shape} {y.dtype}")
    ch, _kh = ah.c()
    cv, _kv = av.c()
    r = _CheckResult()
    rc = _check_lib().or_check_2d(ctypes.byref(ch), ctypes.byref(cv), int(inverse), _dtype_code(x),
                                  x.ctypes.data, y.ctypes.data, x.shape[0],
                                  threads or threads_available(), float(tol), ctypes.byref(r))
    if rc:
        raise ValueError("or_check_2d: bad geometry")
    return _result(r, x.shape[0])


def check_mixed(table, h_index, v_index, offsets, x, y, inverse=False, threads=None,
                tol=0.0) -> dict:
    """Packed mixed-shape batch (config 3): block i at offsets[i], rows through
    table[h_index[i]], columns through table[v_index[i]]."""
    x, y = np.ascontiguousarray(x), np.ascontiguousarray(y)
    if x.shape != y.shape or x.dtype != y.dtype:
        raise ValueError("check_mixed: x / y mismatch")
    axes = (_Axis * len(table))()
    keep = []
    for k, ax in enumerate(table):
        c, m = ax.c()
        axes[k] = c
        keep.append(m)
    hi = np.ascontiguousarray(h_index, dtype=np.int32)
    vi = np.ascontiguousarray(v_index, dtype=np.int32)
    of = np.ascontiguousarray(offsets, dtype=np.int64)
    r = _CheckResult()
    rc = _check_lib().or_check_mixed(
        axes, len(table), hi.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
        vi.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
        of.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), len(of), int(inverse), _dtype_code(x),
        x.ctypes.data, y.ctypes.data, threads or threads_available(), float(tol), ctypes.byref(r))
    if rc:
        raise ValueError("or_check_mixed: bad table index or size")
    return _result(r, len(of))


def check_frames(ah: OAxis, av: OAxis, frames, coefs, inverse=False, threads=None,
                 tol=0.0) -> dict:
    """fp32 frame stack (F, height, width) vs block-major coefficients (config 5;
    bottom zero padding).  Forward: coefs vs oracle(frames);
    inverse: frames vs oracle^-1(coefs), rows inside the frame only."""
    frames = np.ascontiguousarray(frames, dtype=np.float32)
    coefs = np.ascontiguousarray(coefs, dtype=np.float32)
    f, height, width = frames.shape
    ch, _kh = ah.c()
    cv, _kv = av.c()
    ty, tx = -(-height // av.n), width // ah.n
    if coefs.size != f * ty * tx * ah.n * av.n:
        raise ValueError(f"check_frames: {coefs.shape} coefficients for {frames.shape} frames")
    r = _CheckResult()
    rc = _check_lib().or_check_frames(ctypes.byref(ch), ctypes.byref(cv), int(inverse),
                                      frames.ctypes.data, coefs.ctypes.data, f, height, width,
                                      threads or threads_available(), float(tol), ctypes.byref(r))
    if rc:
        raise ValueError("or_check_frames: bad geometry")
    return _result(r, f * ty * tx)
