"""Adjusted-transform pipelines: the reference's drop-in entry points plus the
fused 2-D / frame entries of the B200 build.

Reference names and semantics kept (reference pkg/src/dctadjust/pipeline.py):
  FAST_SIZES, BasePath                                   :32-37
  fast_dct2 / fast_idct2 / fast_dst3_via_dct2 / fast_idst3 :64-87
  apply_band / apply_subblock                            :90-108
  AdjustedTransform / make_adjusted_transform            :127-155
  forward_adjusted / inverse_adjusted                    :176-191
  dense_matrix                                           :194-199
Each call is ONE fused kernel (adjustment + butterfly, no intermediate HBM
round trip) behind the C-ABI.  New entries:
  forward_adjusted_2d / inverse_adjusted_2d   (nblk, H, W) blocks, rows then
                                              columns (the order of _dct2_2d,
                                              pipeline.py:236-239), one kernel
  forward_frames / inverse_frames             whole frames tiled into blocks
  forward_adjusted_2d_host / ..._host         host buffers, pipelined copies
  roundtrip_adjusted_2d(_host)                forward + inverse in one kernel (device / host buffers)
  MixedBatch / mixed_forward / mixed_inverse  packed mixed-shape batches (config 3)
  mixed_roundtrip                             both, one fused kernel per class
Extension: base DCT-3 is accepted (the DCT-8 pre-adjustment, SURVEY.md App. A
D3, built with design.flip_pre_adjustment); the reference raises
ConfigurationError for it.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import _device, _lib, kernels
from .design import AdjustmentMatrix, PatternKind, Side
from .errors import ConfigurationError, InvalidDimensionError, PatternError, ShapeError
from .transforms import TransformKind, build_transform

FAST_SIZES = (4, 8, 16, 32, 64)


class BasePath(Enum):
    FAST_DCT2 = "fast_dct2"
    FAST_DST3_VIA_DCT2 = "fast_dst3_via_dct2"
    FAST_DCT3 = "fast_dct3"  # extension: DCT-8 pre flip (App. A D3)


_BASE_CODE = {BasePath.FAST_DCT2: _lib.BASE_DCT2, BasePath.FAST_DST3_VIA_DCT2: _lib.BASE_DST3,
              BasePath.FAST_DCT3: _lib.BASE_DCT3}
_ADJ_CODE = {PatternKind.BAND: _lib.ADJ_BAND, PatternKind.SUBBLOCK: _lib.ADJ_SUBBLOCK,
             PatternKind.DENSE: _lib.ADJ_DENSE}


def _check_fast_size(n: int) -> None:
    if n not in FAST_SIZES:
        raise InvalidDimensionError(f"fast transforms support sizes {FAST_SIZES}, got {n}")


def _width(x) -> int:
    shape = tuple(x.shape) if hasattr(x, "shape") else np.shape(x)
    return shape[-1] if shape else 0


def _as_batch(x, n: int):
    """(contiguous device batch (nvec, n), was_vector, returns_numpy)."""
    t, as_np = _device.to_device(x)
    if t.dim() == 1:
        if t.shape[0] != n:
            raise ShapeError(f"vector length {t.shape[0]}, expected {n}")
        return t.reshape(1, n), True, as_np
    if t.dim() == 2:
        if t.shape[1] != n:
            raise ShapeError(f"batch width {t.shape[1]}, expected {n}")
        return t, False, as_np
    raise ShapeError(f"expected a vector or batch of vectors, got ndim={t.dim()}")


def _debatch(t, was_vector: bool, as_np: bool):
    out = _device.from_device(t, as_np)
    return out[0] if was_vector else out


def _fast(fn, x):
    n = _width(x)
    _check_fast_size(n)
    t, single, as_np = _as_batch(x, n)
    y = _device.empty_like(t)
    _lib.call(fn, t.data_ptr(), y.data_ptr(), t.shape[0], n, _device.dtype_code(t),
              _device.stream_handle())
    return _debatch(y, single, as_np)


def fast_dct2(x):
    """Orthonormal DCT-2 through the fast butterfly."""
    return _fast("dctadj_dct2", x)


def fast_idct2(y):
    return _fast("dctadj_idct2", y)


def fast_dst3_via_dct2(x):
    """DST-3 at DCT-2 cost: reversal + inverse fast DCT-2 + sign flips."""
    return _fast("dctadj_dst3", x)


def fast_idst3(y):
    return _fast("dctadj_idst3", y)


def apply_band(adj: AdjustmentMatrix, x):
    """y = A x for a band adjustment (only the K-tap window of each row)."""
    if adj.pattern.kind is not PatternKind.BAND:
        raise PatternError(f"apply_band needs a band adjustment, got {adj.pattern.label()}")
    t, single, as_np = _as_batch(x, adj.pattern.size)
    return _debatch(kernels.band(adj.realized, adj.pattern.taps, t), single, as_np)


def apply_subblock(adj: AdjustmentMatrix, y):
    """Leading B coefficients times the block; the rest bit-identical."""
    if adj.pattern.kind is not PatternKind.SUBBLOCK:
        raise PatternError(
            f"apply_subblock needs a sub-block adjustment, got {adj.pattern.label()}")
    t, single, as_np = _as_batch(y, adj.pattern.size)
    b = adj.pattern.order
    return _debatch(kernels.subblock(adj.realized[:b, :b], t), single, as_np)


@dataclass(frozen=True)
class AdjustedTransform:
    """A runnable approximation of DST-7 or DCT-8: adjustment + fast base."""

    target: TransformKind
    size: int
    adjustment: AdjustmentMatrix
    base_path: BasePath

    def axis(self):
        """The C-ABI descriptor (and the host buffers it points into)."""
        adj = self.adjustment
        mat = np.ascontiguousarray(adj.realized, dtype=np.float64)
        ax = _lib.Axis(self.size, _BASE_CODE[self.base_path], _ADJ_CODE[adj.pattern.kind],
                       _lib.SIDE_PRE if adj.side is Side.PRE else _lib.SIDE_POST,
                       adj.pattern.taps or 0, adj.pattern.order or 0, _lib.dptr(mat))
        angles = brickwall_angles(adj)
        if angles is not None:
            ax.givens = _lib.dptr(angles)
            ax.ngivens = len(angles)
        return ax, (mat, angles)


def brickwall_angles(adj: AdjustmentMatrix):
    """The schedule angles of a band adjustment whose Givens schedule is the
    reference's brick-wall structure (taps-1 layers, layer l pairing (i, i+1)
    for i = l%2, l%2+2, ...; design.py:225-243), in layer order -- else None."""
    if adj.pattern.kind is not PatternKind.BAND:
        return None
    n, k = adj.pattern.size, adj.pattern.taps
    layers = adj.schedule.layers
    if len(layers) != k - 1:
        return None
    for level, layer in enumerate(layers):
        want = [(i, i + 1) for i in range(level % 2, n - 1, 2)]
        if [(r.i, r.j) for r in layer] != want:
            return None
    return np.ascontiguousarray([r.theta for layer in layers for r in layer], dtype=np.float64)


def make_adjusted_transform(adj: AdjustmentMatrix) -> AdjustedTransform:
    """Bind an adjustment to its fast base (DST-3 for pre, DCT-2 for post)."""
    _check_fast_size(adj.pattern.size)
    if adj.base is TransformKind.DCT2:
        path = BasePath.FAST_DCT2
    elif adj.base is TransformKind.DST3:
        path = BasePath.FAST_DST3_VIA_DCT2
    elif adj.base is TransformKind.DCT3:
        path = BasePath.FAST_DCT3
    else:
        raise ConfigurationError(
            f"no fast path for base transform {adj.base}; use dct2, dst3 or dct3")
    return AdjustedTransform(adj.target, adj.pattern.size, adj, path)


def _run_1d(fn: str, t: AdjustedTransform, x):
    arr, single, as_np = _as_batch(x, t.size)
    y = _device.empty_like(arr)
    ax, _keep = t.axis()
    _lib.call(fn, ctypes.byref(ax), arr.data_ptr(), y.data_ptr(), arr.shape[0],
              _device.dtype_code(arr), _device.stream_handle())
    return _debatch(y, single, as_np)


def forward_adjusted(t: AdjustedTransform, x):
    """PRE: y = B(A x);  POST: y = C(B x) -- one fused kernel."""
    return _run_1d("dctadj_forward_1d", t, x)


def inverse_adjusted(t: AdjustedTransform, y):
    """PRE: x = A^T(B^-1 y);  POST: x = B^-1(C^T y) -- one fused kernel."""
    return _run_1d("dctadj_inverse_1d", t, y)


def dense_matrix(t: AdjustedTransform) -> np.ndarray:
    """The exact H this pipeline realizes (oracle / comparison path)."""
    base = build_transform(t.adjustment.base, t.size).entries
    a = t.adjustment.realized
    return base @ a if t.adjustment.side is Side.PRE else a @ base


# ---------------------------------------------------------------- 2-D blocks
def _as_blocks(x, h: int, w: int):
    t, as_np = _device.to_device(x)
    if t.dim() == 2:
        if tuple(t.shape) != (h, w):
            raise ShapeError(f"block {tuple(t.shape)}, expected ({h}, {w})")
        return t.reshape(1, h, w), True, as_np
    if t.dim() == 3:
        if tuple(t.shape[1:]) != (h, w):
            raise ShapeError(f"blocks {tuple(t.shape[1:])}, expected ({h}, {w})")
        return t, False, as_np
    raise ShapeError(f"expected (H, W) or (nblk, H, W) blocks, got ndim={t.dim()}")


def _run_2d(fn: str, th: AdjustedTransform, tv: AdjustedTransform, x):
    blk, single, as_np = _as_blocks(x, tv.size, th.size)
    y = _device.empty_like(blk)
    (axh, _kh), (axv, _kv) = th.axis(), tv.axis()
    _lib.call(fn, ctypes.byref(axh), ctypes.byref(axv), blk.data_ptr(), y.data_ptr(),
              blk.shape[0], _device.dtype_code(blk), _device.stream_handle())
    return _debatch(y, single, as_np)


def forward_adjusted_2d(th: AdjustedTransform, tv: AdjustedTransform, x):
    """Y = T_v X T_h^T per (H, W) block: rows with th (length W), then columns
    with tv (length H), fused in one kernel."""
    return _run_2d("dctadj_forward_2d", th, tv, x)


def inverse_adjusted_2d(th: AdjustedTransform, tv: AdjustedTransform, y):
    """X = T_v^T Y T_h: columns, then rows (the mirror of the forward)."""
    return _run_2d("dctadj_inverse_2d", th, tv, y)


def roundtrip_adjusted_2d(th: AdjustedTransform, tv: AdjustedTransform, x):
    """(forward_adjusted_2d(x), inverse_adjusted_2d(of that)) in one kernel: x is
    read once, the coefficients and the reconstruction are written once.  Bit-
    identical to the two calls.  Returns (y, xr)."""
    blk, single, as_np = _as_blocks(x, tv.size, th.size)
    y = _device.empty_like(blk)
    xr = _device.empty_like(blk)
    (axh, _kh), (axv, _kv) = th.axis(), tv.axis()
    _lib.call("dctadj_roundtrip_2d", ctypes.byref(axh), ctypes.byref(axv), blk.data_ptr(),
              y.data_ptr(), xr.data_ptr(), blk.shape[0], _device.dtype_code(blk),
              _device.stream_handle())
    return _debatch(y, single, as_np), _debatch(xr, single, as_np)


def _host_out(arr: np.ndarray, out):
    """A fresh output like `arr`, or the caller's array checked to be a writable
    C-contiguous ndarray of the same shape and dtype (the library writes it raw)."""
    if out is None:
        return np.empty_like(arr)
    if not isinstance(out, np.ndarray) or out.shape != arr.shape or out.dtype != arr.dtype \
            or not out.flags.c_contiguous or not out.flags.writeable:
        raise ShapeError(f"out must be a writable C-contiguous {arr.dtype} array of shape {arr.shape}")
    return out


def _run_2d_host(fn: str, th: AdjustedTransform, tv: AdjustedTransform, x, out=None):
    arr = np.asarray(x)
    if arr.dtype not in (np.float32, np.float64):
        arr = arr.astype(np.float64)
    arr = np.ascontiguousarray(arr)
    if arr.ndim != 3 or arr.shape[1:] != (tv.size, th.size):
        raise ShapeError(f"expected (nblk, {tv.size}, {th.size}) blocks, got {arr.shape}")
    y = _host_out(arr, out)
    (axh, _kh), (axv, _kv) = th.axis(), tv.axis()
    _device.require_cuda()
    _lib.call(fn, ctypes.byref(axh), ctypes.byref(axv), arr.ctypes.data, y.ctypes.data,
              arr.shape[0], _lib.F32 if arr.dtype == np.float32 else _lib.F64,
              _device.torch.cuda.current_device())
    return y


def forward_adjusted_2d_host(th, tv, x, out=None):
    """forward_adjusted_2d on host arrays (pinned for full speed); the copies
    and kernels are pipelined inside the library."""
    return _run_2d_host("dctadj_forward_2d_host", th, tv, x, out)


def inverse_adjusted_2d_host(th, tv, y, out=None):
    return _run_2d_host("dctadj_inverse_2d_host", th, tv, y, out)


def roundtrip_adjusted_2d_host(th, tv, x, out=None, out_inv=None):
    """(forward_adjusted_2d(x), inverse_adjusted_2d(of that)) on host arrays in one
    pipelined pass: the coefficients stay on the device for the inverse and
    cross PCIe once.  Returns (y, xr)."""
    arr = np.asarray(x)
    if arr.dtype not in (np.float32, np.float64):
        arr = arr.astype(np.float64)
    arr = np.ascontiguousarray(arr)
    if arr.ndim != 3 or arr.shape[1:] != (tv.size, th.size):
        raise ShapeError(f"expected (nblk, {tv.size}, {th.size}) blocks, got {arr.shape}")
    y = _host_out(arr, out)
    xr = _host_out(arr, out_inv)
    (axh, _kh), (axv, _kv) = th.axis(), tv.axis()
    _device.require_cuda()
    _lib.call("dctadj_roundtrip_2d_host", ctypes.byref(axh), ctypes.byref(axv), arr.ctypes.data,
              y.ctypes.data, xr.ctypes.data, arr.shape[0],
              _lib.F32 if arr.dtype == np.float32 else _lib.F64,
              _device.torch.cuda.current_device())
    return y, xr


# ---------------------------------------------------------------- frames
def frame_block_count(nframes: int, height: int, width: int, h: int, w: int) -> int:
    return nframes * (-(-height // h)) * (width // w)


def forward_frames(th: AdjustedTransform, tv: AdjustedTransform, frames):
    """(F, height, width) frames -> block-major coefficients (nblk, H, W), blocks
    in raster order per frame; rows past `height` are zero padding."""
    t, as_np = _device.to_device(frames)
    if t.dim() != 3:
        raise ShapeError(f"expected (F, height, width) frames, got ndim={t.dim()}")
    f, hh, ww = t.shape
    nblk = frame_block_count(f, hh, ww, tv.size, th.size)
    y = _device.empty_like(t, (nblk, tv.size, th.size))
    (axh, _kh), (axv, _kv) = th.axis(), tv.axis()
    _lib.call("dctadj_forward_frames", ctypes.byref(axh), ctypes.byref(axv), t.data_ptr(),
              y.data_ptr(), f, hh, ww, _device.dtype_code(t), _device.stream_handle())
    return _device.from_device(y, as_np)


def forward_frames_exact(th: AdjustedTransform, tv: AdjustedTransform, eh: AdjustedTransform,
                         ev: AdjustedTransform, frames, with_error: bool = True):
    """Config 5's comparison step: adjusted (th, tv) and exact (eh, ev) forward
    transforms of the same frames plus the per-frame approximation error.

    Returns (y_adj, y_exact, err) with err of shape (F, 4): sum (Ya - Ye)^2 and
    sum Ye^2 over all tiles, then over the tile rows entirely inside the frame.
    fp32 32x32 sub8-post / band6-pre with dense exact axes runs as one tensor-
    core kernel reading the frames once (C-ABI dctadj_forward_frames_exact);
    with_error=False skips the sums (err is None) and runs the two transforms as
    separate launches, which is faster when the error is not wanted."""
    import torch
    t, as_np = _device.to_device(frames)
    if t.dim() != 3:
        raise ShapeError(f"expected (F, height, width) frames, got ndim={t.dim()}")
    f, hh, ww = t.shape
    nblk = frame_block_count(f, hh, ww, tv.size, th.size)
    y = _device.empty_like(t, (nblk, tv.size, th.size))
    ye = _device.empty_like(t, (nblk, tv.size, th.size))
    err = torch.empty((f, 4), dtype=torch.float64, device=t.device) if with_error else None
    axes = [a.axis() for a in (th, tv, eh, ev)]
    _lib.call("dctadj_forward_frames_exact", *[ctypes.byref(a) for a, _k in axes], t.data_ptr(),
              y.data_ptr(), ye.data_ptr(), err.data_ptr() if with_error else None, f, hh, ww,
              _device.dtype_code(t), _device.stream_handle())
    return (_device.from_device(y, as_np), _device.from_device(ye, as_np),
            _device.from_device(err, as_np) if with_error else None)


def inverse_frames(th: AdjustedTransform, tv: AdjustedTransform, coefs, height: int,
                   width: int):
    """Block-major coefficients -> (F, height, width) frames (padding clipped)."""
    t, as_np = _device.to_device(coefs)
    if t.dim() != 3 or tuple(t.shape[1:]) != (tv.size, th.size):
        raise ShapeError(f"expected (nblk, {tv.size}, {th.size}) coefficients")
    per = frame_block_count(1, height, width, tv.size, th.size)
    if per == 0 or t.shape[0] % per:
        raise ShapeError(f"{t.shape[0]} blocks do not tile frames of {height} x {width}")
    f = t.shape[0] // per
    y = _device.empty_like(t, (f, height, width))
    (axh, _kh), (axv, _kv) = th.axis(), tv.axis()
    _lib.call("dctadj_inverse_frames", ctypes.byref(axh), ctypes.byref(axv), t.data_ptr(),
              y.data_ptr(), f, height, width, _device.dtype_code(t), _device.stream_handle())
    return _device.from_device(y, as_np)


# ---------------------------------------------------------------- mixed batches
class MixedBatch:
    """Blocks of different shapes packed back to back in one buffer (config 3).

    Block i occupies heights[i] x widths[i] samples starting at element
    `offsets[i]`; its rows use table entry h_index[i] and its columns entry
    v_index[i] of the AdjustedTransform table passed to mixed_forward /
    mixed_inverse (sizes fixed here).  The blocks are bucketed by (h, v) class
    once, in the C-ABI plan (dctadj_mixed_create); every call is then one
    gather kernel per class.
    """

    def __init__(self, offsets, h_index, v_index, sizes, total_elements: int):
        _device.require_cuda()
        self.offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        self.h_index = np.ascontiguousarray(h_index, dtype=np.int32)
        self.v_index = np.ascontiguousarray(v_index, dtype=np.int32)
        self.sizes = np.ascontiguousarray(sizes, dtype=np.int32)
        self.total_elements = int(total_elements)
        n = self.offsets.shape[0]
        if not (self.h_index.shape[0] == self.v_index.shape[0] == n):
            raise ShapeError("offsets, h_index and v_index must have one entry per block")
        self._plan = ctypes.c_void_p()
        _lib.call("dctadj_mixed_create", self.offsets.ctypes.data, self.h_index.ctypes.data,
                  self.v_index.ctypes.data, n, self.sizes.ctypes.data, len(self.sizes),
                  self.total_elements, ctypes.byref(self._plan))

    @staticmethod
    def packed(h_index, v_index, sizes) -> "MixedBatch":
        """Pack blocks contiguously in the given order."""
        sizes = np.asarray(sizes, dtype=np.int64)
        areas = sizes[np.asarray(h_index)] * sizes[np.asarray(v_index)]
        offsets = np.concatenate([[0], np.cumsum(areas)[:-1]]) if len(areas) else np.zeros(0, np.int64)
        return MixedBatch(offsets, h_index, v_index, sizes, int(areas.sum()))

    @property
    def nblk(self) -> int:
        return int(self.offsets.shape[0])

    def block_slices(self):
        """(offset, H, W) per block (host-side view helper)."""
        for o, hi, vi in zip(self.offsets, self.h_index, self.v_index):
            yield int(o), int(self.sizes[vi]), int(self.sizes[hi])

    def __del__(self):
        plan = getattr(self, "_plan", None)
        if plan is not None and plan.value and _lib._lib is not None:
            _lib._lib.dctadj_mixed_destroy(plan)
            self._plan = None


def _mixed_args(batch: MixedBatch, table, x):
    t, as_np = _device.to_device(x)
    if t.dim() != 1 or t.shape[0] != batch.total_elements:
        raise ShapeError(f"expected a packed buffer of {batch.total_elements} samples")
    if len(table) != len(batch.sizes):
        raise ShapeError(f"table has {len(table)} entries, plan expects {len(batch.sizes)}")
    axes = (_lib.Axis * len(table))()
    keep = []
    for k, tr in enumerate(table):
        ax, m = tr.axis()
        axes[k] = ax
        keep.append(m)
    return t, as_np, axes, keep


def _mixed(fn: str, batch: MixedBatch, table, x):
    t, as_np, axes, _keep = _mixed_args(batch, table, x)
    y = _device.empty_like(t)
    _lib.call(fn, batch._plan, axes, t.data_ptr(), y.data_ptr(), _device.dtype_code(t),
              _device.stream_handle())
    return _device.from_device(y, as_np)


def mixed_forward(batch: MixedBatch, table, x):
    """Forward adjusted 2-D transform of every block of a packed mixed batch."""
    return _mixed("dctadj_mixed_forward", batch, table, x)


def mixed_inverse(batch: MixedBatch, table, y):
    return _mixed("dctadj_mixed_inverse", batch, table, y)


def mixed_roundtrip(batch: MixedBatch, table, x):
    """(mixed_forward(x), mixed_inverse(of that)) with one fused kernel per class:
    x read once, coefficients and reconstruction written once.  Bit-identical to
    the two calls.  Returns (y, xr)."""
    t, as_np, axes, _keep = _mixed_args(batch, table, x)
    y = _device.empty_like(t)
    xr = _device.empty_like(t)
    _lib.call("dctadj_mixed_roundtrip", batch._plan, axes, t.data_ptr(), y.data_ptr(),
              xr.data_ptr(), _device.dtype_code(t), _device.stream_handle())
    return _device.from_device(y, as_np), _device.from_device(xr, as_np)


# ---------------------------------------------------------------- encoder evaluation
ENCODER_KEYS = (("dct2", "dct2"), ("dst7", "dst7"), ("dct8", "dst7"), ("dst7", "dct8"),
                ("dct8", "dct8"))


@dataclass(frozen=True)
class EncoderContext:
    """Sub-block DST-7 post-adjustments for both axes of a block; the DCT-8
    counterparts follow from the chessboard relation (reference
    pipeline.py:202-233)."""

    horizontal: AdjustmentMatrix | None = None
    vertical: AdjustmentMatrix | None = None

    def require(self, width: int, height: int) -> tuple[AdjustmentMatrix, AdjustmentMatrix]:
        if self.horizontal is None or self.vertical is None:
            raise ConfigurationError(
                "simultaneous evaluation needs sub-block adjustments for both dimensions")
        for adj, size, name in ((self.horizontal, width, "horizontal"),
                                (self.vertical, height, "vertical")):
            if adj.pattern.kind is not PatternKind.SUBBLOCK:
                raise ConfigurationError(f"{name} adjustment must be a sub-block design")
            if adj.pattern.size != size:
                raise ConfigurationError(
                    f"{name} adjustment is for size {adj.pattern.size}, block needs {size}")
            if adj.side is not Side.POST or adj.base is not TransformKind.DCT2 \
                    or adj.target is not TransformKind.DST7:
                raise ConfigurationError(f"{name} adjustment must be post-side dct2 -> dst7")
        return self.horizontal, self.vertical


def simultaneous_encoder_eval(block, ctx: EncoderContext) -> dict:
    """The five encoder transform candidates of each residual block, keyed
    (horizontal, vertical): ("dct2","dct2") and the four DST-7/DCT-8 pairs.
    One fused kernel: one read, one shared 2-D DCT-2, five planes written;
    coefficients outside the first 8 rows and columns are bit-identical across
    the five outputs (reference pipeline.py:256-293)."""
    t, as_np = _device.to_device(block)
    single = t.dim() == 2
    if t.dim() not in (2, 3):
        raise ShapeError(f"expected a 2-D block or a batch of blocks, got ndim={t.dim()}")
    blk = t.reshape(1, *t.shape) if single else t
    height, width = int(blk.shape[1]), int(blk.shape[2])
    _check_fast_size(width)
    _check_fast_size(height)
    h_adj, v_adj = ctx.require(width, height)
    th, tv = make_adjusted_transform(h_adj), make_adjusted_transform(v_adj)
    outs = [_device.empty_like(blk) for _ in ENCODER_KEYS]
    ptrs = (ctypes.c_void_p * 5)(*[o.data_ptr() for o in outs])
    (axh, _kh), (axv, _kv) = th.axis(), tv.axis()
    _lib.call("dctadj_encoder_eval", ctypes.byref(axh), ctypes.byref(axv), blk.data_ptr(),
              ptrs, blk.shape[0], _device.dtype_code(blk), _device.stream_handle())
    res = {}
    for key, o in zip(ENCODER_KEYS, outs):
        o = _device.from_device(o, as_np)
        res[key] = o[0] if single else o
    return res


def naive_encoder_eval(block, ctx: EncoderContext) -> dict:
    """The same five outputs as independent dense separable transforms (the
    comparison path, reference pipeline.py:296-323): five fused 2-D kernels
    with the exact H = C B of each axis as a dense matrix."""
    from .design import dct8_adjustment_from_dst7, pattern_schedule_template, SparsityPattern
    t, as_np = _device.to_device(block)
    single = t.dim() == 2
    blk = t.reshape(1, *t.shape) if single else t
    height, width = int(blk.shape[1]), int(blk.shape[2])
    h_adj, v_adj = ctx.require(width, height)

    def dense(adj):
        h = dense_matrix(make_adjusted_transform(adj))
        n = h.shape[0]
        rec = AdjustmentMatrix(SparsityPattern.dense(n), Side.POST, TransformKind.DCT2,
                               adj.target, pattern_schedule_template(SparsityPattern.dense(n)),
                               h @ build_transform(TransformKind.DCT2, n).entries.T)
        return make_adjusted_transform(rec)

    def ident(n):
        from .design import identity_adjustment
        return make_adjusted_transform(identity_adjustment(
            SparsityPattern.subblock(1, n), Side.POST, TransformKind.DCT2, TransformKind.DCT2))

    hs = {"dct2": ident(width), "dst7": dense(h_adj), "dct8": dense(dct8_adjustment_from_dst7(h_adj))}
    vs = {"dct2": ident(height), "dst7": dense(v_adj), "dct8": dense(dct8_adjustment_from_dst7(v_adj))}
    res = {}
    for key in ENCODER_KEYS:
        o = _device.from_device(forward_adjusted_2d(hs[key[0]], vs[key[1]], blk), as_np)
        res[key] = o[0] if single else o
    return res
