"""CPU: host-side logic -- records, file formats, shipped designs, the C-ABI
library's exported surface, error mapping, partitioning.  No device calls."""
import ctypes
import hashlib
import io
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2505_23618_b200 import _lib, errors, matio, shard
from paper_2505_23618_b200.design import (GivensSchedule, PlaneRotation, Side, SparsityPattern,
                                          dct8_adjustment_from_dst7, flip_pre_adjustment,
                                          givens_to_matrix, identity_adjustment,
                                          pattern_schedule_template, random_adjustment)
from paper_2505_23618_b200.transforms import (TransformKind, build_transform, flip_to_dct8,
                                              orthonormality_error)

ROOT = Path(__file__).resolve().parents[1]


# ---------------------------------------------------------------- transforms
@pytest.mark.parametrize("kind", list(TransformKind))
@pytest.mark.parametrize("n", [4, 8, 16, 32, 64])
def test_transforms_orthonormal(kind, n):
    assert orthonormality_error(build_transform(kind, n).entries) < 1e-12


def test_transform_identities():
    n = 16
    d7 = build_transform(TransformKind.DST7, n)
    assert np.array_equal(flip_to_dct8(d7).entries, build_transform(TransformKind.DCT8, n).entries)
    # DST-7 rows diagonalise min(i,j)+1 (reference test_transforms.py:49-64)
    k = np.minimum.outer(np.arange(n), np.arange(n)) + 1.0
    m = d7.entries @ k @ d7.entries.T
    assert np.abs(m - np.diag(np.diag(m))).max() < 1e-9
    c2 = build_transform(TransformKind.DCT2, 2).entries
    assert np.allclose(c2, np.array([[1, 1], [1, -1]]) / np.sqrt(2))


# ---------------------------------------------------------------- design records
def test_band_template_is_banded():
    for taps in (2, 4, 6):
        adj = random_adjustment(SparsityPattern.band(taps, 32), Side.PRE, TransformKind.DST3, 1)
        i, j = np.indices((32, 32))
        assert np.all(adj.realized[np.abs(i - j) >= taps] == 0.0)
        assert orthonormality_error(adj.realized) < 1e-13


def test_subblock_template_identity_outside():
    adj = random_adjustment(SparsityPattern.subblock(8, 32), Side.POST, TransformKind.DCT2, 2)
    assert np.array_equal(adj.realized[8:, 8:], np.eye(24))
    assert np.all(adj.realized[:8, 8:] == 0) and np.all(adj.realized[8:, :8] == 0)
    assert pattern_schedule_template(SparsityPattern.subblock(8, 32)).n_rotations == 28


def test_schedule_validation():
    with pytest.raises(errors.InvalidScheduleError):
        GivensSchedule(4, ((PlaneRotation(0, 1, 0.1), PlaneRotation(1, 2, 0.1)),))
    with pytest.raises(errors.InvalidScheduleError):
        GivensSchedule(4, ((PlaneRotation(2, 1, 0.1),),))
    with pytest.raises(errors.PatternError):
        SparsityPattern.band(0, 8)
    with pytest.raises(errors.PatternError):
        SparsityPattern.from_label("wedge:3", 8)


def test_dct8_post_chessboard_and_involution():
    a = matio.load_designed("sub8_post_dct2_dst7_n32")
    b = dct8_adjustment_from_dst7(a)
    s = (-1.0) ** np.arange(32)
    assert np.array_equal(b.realized, np.outer(s, s) * a.realized)
    assert np.allclose(givens_to_matrix(b.schedule), b.realized, atol=1e-12)
    assert np.array_equal(dct8_adjustment_from_dst7(b).realized, a.realized)
    with pytest.raises(errors.KindMismatchError):
        dct8_adjustment_from_dst7(matio.load_designed("band6_pre_dst3_dst7_n32"))


def test_flip_pre_adjustment_realizes_dct8_flip():
    a = matio.load_designed("band6_pre_dst3_dst7_n32")
    f = flip_pre_adjustment(a)
    assert f.base is TransformKind.DCT3 and f.target is TransformKind.DCT8
    assert np.allclose(givens_to_matrix(f.schedule), f.realized, atol=1e-12)
    # H8 = DCT3 (R A R) == S (DST3 A) R
    h7 = build_transform(TransformKind.DST3, 32).entries @ a.realized
    s = (-1.0) ** np.arange(32)
    h8 = build_transform(TransformKind.DCT3, 32).entries @ f.realized
    assert np.abs(h8 - (s[:, None] * h7)[:, ::-1]).max() < 1e-13


# ---------------------------------------------------------------- matio + fixtures
def test_adjustment_roundtrip_and_corruption():
    a = random_adjustment(SparsityPattern.band(4, 16), Side.PRE, TransformKind.DST3, 3)
    buf = io.StringIO()
    matio.write_adjustment(buf, a)
    b = matio.read_adjustment(io.StringIO(buf.getvalue()))
    assert np.array_equal(a.realized, b.realized)
    assert b.pattern == a.pattern and b.side is a.side
    lines = buf.getvalue().splitlines()
    lines[-1] = " ".join(["0.5"] * 16)  # corrupt the realized matrix
    with pytest.raises(errors.MatrixFormatError):
        matio.read_adjustment(io.StringIO("\n".join(lines) + "\n"))
    with pytest.raises(errors.MatrixFormatError):
        matio.read_adjustment(io.StringIO(""))


def test_shipped_designs_hashes_and_quality():
    d = ROOT / "paper_2505_23618_b200" / "adjustments"
    for line in (d / "SHA256SUMS").read_text().split("\n"):
        if line.strip():
            h, name = line.split()
            assert hashlib.sha256((d / name).read_bytes()).hexdigest() == h, name
    for n in (16, 32, 64):
        a = matio.load_designed(f"band6_pre_dst3_dst7_n{n}")
        assert a.pattern.taps == 6 and a.side is Side.PRE and a.base is TransformKind.DST3
        i, j = np.indices((n, n))
        assert np.all(a.realized[np.abs(i - j) >= 6] == 0.0)
    # the designed band beats the identity (weighted error, reference design.py:253-270)
    a = matio.load_designed("band6_pre_dst3_dst7_n32")
    alpha = np.log(100.0) / 32
    w = np.exp(-alpha * np.arange(32))[:, None]
    b, t = build_transform(TransformKind.DST3, 32).entries, build_transform(TransformKind.DST7, 32).entries
    e_adj = float((w * (b @ a.realized - t) ** 2).sum())
    e_id = float((w * (b - t) ** 2).sum())
    assert e_adj / e_id < 0.06   # 0.0523 measured in SURVEY.md App. A D1


# ---------------------------------------------------------------- C-ABI surface
def _header_symbols():
    text = (ROOT / "include" / "dctadj.h").read_text()
    return sorted(set(re.findall(r"\b(dctadj_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert set(_header_symbols()) == set(_lib.SIGNATURES)


def test_library_exports_every_symbol():
    if not _lib.LIB_PATH.exists():
        pytest.skip("libdctadj.so not built")
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    for name in _header_symbols():
        assert hasattr(lib, name), name
    lib = _lib.load()
    assert lib.dctadj_version() == 1
    assert lib.dctadj_kernel_count() > 100
    assert lib.dctadj_status_string(3) == b"PatternError"


def test_validation_errors_without_device():
    """Argument validation happens before any device work, so the error
    mapping is testable on CPU."""
    if not _lib.LIB_PATH.exists():
        pytest.skip("libdctadj.so not built")
    lib = _lib.load()
    ax = _lib.Axis(12, 0, 0, 1, 0, 0, None)
    with pytest.raises(errors.InvalidDimensionError):
        _lib.check(lib.dctadj_forward_1d(ctypes.byref(ax), None, None, 4, 0, None))
    ax = _lib.Axis(32, 7, 0, 1, 0, 0, None)
    with pytest.raises(errors.ConfigurationError):
        _lib.check(lib.dctadj_forward_1d(ctypes.byref(ax), None, None, 4, 0, None))
    m = np.eye(32)
    ax = _lib.Axis(32, 1, 1, 0, 40, 0, _lib.dptr(m))
    with pytest.raises(errors.PatternError):
        _lib.check(lib.dctadj_forward_1d(ctypes.byref(ax), None, None, 4, 0, None))
    with pytest.raises(ValueError):
        _lib.check(lib.dctadj_dct2(None, None, 4, 128, 0, None))
    with pytest.raises(ValueError):
        _lib.check(lib.dctadj_dct2(None, None, 4, 32, 9, None))
    ax = _lib.Axis(32, 0, 0, 1, 0, 0, None)
    with pytest.raises(errors.ShapeError):
        _lib.check(lib.dctadj_forward_frames(ctypes.byref(ax), ctypes.byref(ax), None, None,
                                             1, 64, 40, 0, None))
    # empty batches are a no-op success
    _lib.check(lib.dctadj_forward_1d(ctypes.byref(ax), None, None, 0, 0, None))
    _lib.check(lib.dctadj_roundtrip_2d_host(ctypes.byref(ax), ctypes.byref(ax), None, None, None,
                                            0, 0, 0))
    with pytest.raises(ValueError):
        _lib.check(lib.dctadj_roundtrip_2d_host(ctypes.byref(ax), ctypes.byref(ax), None, None,
                                                None, 4, 0, 0))


def test_host_entry_rejects_bad_out_arrays():
    """The host entries write caller arrays raw: shape, dtype, contiguity and
    writability are checked before any device work."""
    from paper_2505_23618_b200 import pipeline
    from paper_2505_23618_b200.design import dct8_adjustment_from_dst7
    t = pipeline.make_adjusted_transform(
        dct8_adjustment_from_dst7(matio.load_designed("sub8_post_dct2_dst7_n32")))
    x = np.zeros((4, 32, 32), np.float32)
    ro = np.zeros_like(x)
    ro.flags.writeable = False
    for bad in (np.zeros((3, 32, 32), np.float32), np.zeros_like(x, dtype=np.float64),
                np.zeros((4, 32, 64), np.float32)[:, :, ::2], ro):
        with pytest.raises(errors.ShapeError):
            pipeline.forward_adjusted_2d_host(t, t, x, out=bad)
        with pytest.raises(errors.ShapeError):
            pipeline.roundtrip_adjusted_2d_host(t, t, x, out_inv=bad)


# ---------------------------------------------------------------- partitioning
def test_block_range_covers_exactly():
    for world in (1, 2, 3, 4, 8):
        ranges = [shard.block_range(r, world, 65536 + 3) for r in range(world)]
        assert ranges[0][0] == 0 and ranges[-1][1] == 65539
        assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
        sizes = [b - a for a, b in ranges]
        assert max(sizes) - min(sizes) <= 1


def test_weighted_ranges_balance():
    rng = np.random.default_rng(0)
    w = rng.choice([256, 512, 1024], size=10000)
    for world in (2, 4, 8):
        rs = shard.weighted_ranges(w, world)
        assert rs[0][0] == 0 and rs[-1][1] == w.size
        loads = [w[a:b].sum() for a, b in rs]
        assert max(loads) - min(loads) <= 2 * w.max()


def _lifting_apply(angles, n, k, x, inverse=False):
    """Python restatement of the kernel's Givens lifting stage (butterfly.cuh
    ST_GIVENS) with the C-ABI packing rule (abi.cu pack_givens)."""
    rots = [(n - (l % 2)) // 2 for l in range(k - 1)]
    start = np.concatenate([[0], np.cumsum(rots)])
    x = np.array(x, dtype=float)
    for a in range(k - 1):
        l = k - 2 - a if inverse else a
        for r in range(rots[l]):
            th = angles[start[l] + r] * (-1 if inverse else 1)
            t, s = np.tan(th / 2), np.sin(th)
            i = (a % 2) + 2 * r
            aa = x[i] - t * x[i + 1]
            b = x[i + 1] + s * aa
            x[i], x[i + 1] = aa - t * b, b
    return x


@pytest.mark.parametrize("name", ["band6_pre_dst3_dst7_n16", "band6_pre_dst3_dst7_n32",
                                  "band4_pre_dst3_dst7_n64"])
def test_brickwall_lifting_reproduces_realized(name):
    from paper_2505_23618_b200.pipeline import brickwall_angles
    for adj in (matio.load_designed(name), flip_pre_adjustment(matio.load_designed(name))):
        n, k = adj.pattern.size, adj.pattern.taps
        ang = brickwall_angles(adj)
        assert ang is not None and len(ang) == sum((n - (l % 2)) // 2 for l in range(k - 1))
        eye = np.eye(n)
        fwd = np.stack([_lifting_apply(ang, n, k, eye[:, j]) for j in range(n)], axis=1)
        inv = np.stack([_lifting_apply(ang, n, k, eye[:, j], True) for j in range(n)], axis=1)
        assert np.abs(fwd - adj.realized).max() < 1e-13
        assert np.abs(inv - adj.realized.T).max() < 1e-13


def test_brickwall_detection_rejects_other_schedules():
    from dataclasses import replace
    from paper_2505_23618_b200.pipeline import brickwall_angles
    assert brickwall_angles(matio.load_designed("sub8_post_dct2_dst7_n32")) is None
    a = matio.load_designed("band6_pre_dst3_dst7_n32")
    odd = GivensSchedule(32, a.schedule.layers[:-1])  # one layer short
    assert brickwall_angles(replace(a, schedule=odd, pattern=SparsityPattern.band(6, 32))) is None


def test_library_resolves_all_symbols_eagerly():
    """RTLD_NOW: a stale or partial build (missing instantiation objects) fails here."""
    import os
    if not _lib.LIB_PATH.exists():
        pytest.skip("libdctadj.so not built")
    ctypes.CDLL(str(_lib.LIB_PATH), mode=os.RTLD_NOW)


def test_roundtrip_fused_query():
    """dctadj_roundtrip_fused says which round trips run as the one fused kernel
    (host-side planning only, no device work)."""
    if not _lib.LIB_PATH.exists():
        pytest.skip("libdctadj.so not built")
    from paper_2505_23618_b200 import pipeline
    from paper_2505_23618_b200.design import dct8_adjustment_from_dst7
    lib = _lib.load()

    def fused(name, dtype, c8=False):
        adj = matio.load_designed(name)
        t = pipeline.make_adjusted_transform(dct8_adjustment_from_dst7(adj) if c8 else adj)
        ax, _keep = t.axis()
        return lib.dctadj_roundtrip_fused(ctypes.byref(ax), ctypes.byref(ax), dtype)

    assert fused("sub8_post_dct2_dst7_n32", _lib.F32, c8=True) == 1   # config 2
    assert fused("band6_pre_dst3_dst7_n32", _lib.F32) == 1
    assert fused("sub8_post_dct2_dst7_n32", _lib.F64) == 0           # fp64: two kernels
    assert fused("sub8_post_dct2_dst7_n64", _lib.F32) == 0           # 64x64: two kernels
    assert fused("sub8_post_dct2_dst7_n32", 7) == 0                  # invalid dtype
