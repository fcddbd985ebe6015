"""GPU parity: every entry point of the C-ABI (through the Python mirror) against
the CPU oracle and the reference's golden vectors.

Tolerances (BASELINE.json north_star): per-block normwise
relative error <= 1e-9 for fp64, <= 1e-5 for fp32.  Bit-exact checks: the
sub-block tail equals the build's own base output, the identity adjustment
equals the base, and rint(inverse(forward(x))) == x for integer residuals.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from conftest import rel_err  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2505_23618_b200 import kernels, matio, pipeline  # noqa: E402
from paper_2505_23618_b200.design import (SparsityPattern, Side, dct8_adjustment_from_dst7,  # noqa: E402
                                          flip_pre_adjustment, identity_adjustment,
                                          random_adjustment)
from paper_2505_23618_b200.errors import (InvalidDimensionError, PatternError,  # noqa: E402
                                          ShapeError, ConfigurationError)
from paper_2505_23618_b200.transforms import TransformKind, build_transform  # noqa: E402

pytestmark = pytest.mark.gpu

F64_TOL = 1e-9
F32_TOL = 1e-5


def oaxis(adj):
    base = {"dct2": O.BASE_DCT2, "dst3": O.BASE_DST3, "dct3": O.BASE_DCT3}[adj.base.value]
    kind = {"band": O.ADJ_BAND, "subblock": O.ADJ_SUBBLOCK, "dense": O.ADJ_DENSE}[adj.pattern.kind.value]
    return O.OAxis(adj.pattern.size, base, kind, O.SIDE_PRE if adj.side is Side.PRE else O.SIDE_POST,
                   adj.pattern.taps or 0, adj.pattern.order or 0, np.array(adj.realized))


def dev(x, dtype=torch.float32):
    return torch.as_tensor(np.ascontiguousarray(x)).to("cuda", dtype)


# ---------------------------------------------------------------- primitives
@pytest.mark.parametrize("n", [4, 8, 16, 32, 64])
@pytest.mark.parametrize("fn", ["dct2", "idct2", "dst3", "idst3"])
def test_primitives_fp64_numpy(golden, n, fn):
    x = golden[f"prim/x/{n}"]
    got = getattr(kernels, fn)(x)
    assert isinstance(got, np.ndarray) and got.dtype == np.float64
    assert rel_err(got, golden[f"prim/{fn}/{n}"]) < F64_TOL


@pytest.mark.parametrize("n", [4, 8, 16, 32, 64])
@pytest.mark.parametrize("fn", ["dct2", "idct2", "dst3", "idst3"])
def test_primitives_fp32_tensor(golden, n, fn):
    x = golden[f"prim/x/{n}"]
    got = getattr(kernels, fn)(dev(x))
    assert got.dtype == torch.float32 and got.is_cuda
    assert rel_err(got.cpu().numpy(), golden[f"prim/{fn}/{n}"]) < F32_TOL


@pytest.mark.parametrize("n", [4, 8, 16, 32, 64])
def test_band_subblock_dense(golden, n):
    x = golden[f"prim/x/{n}"]
    for taps in (3, 4, 6):
        key = f"prim/band/{n}/{taps}"
        if key in golden:
            a = golden[f"prim/band_a/{n}/{taps}"]
            assert rel_err(kernels.band(a, taps, x), golden[key]) < F64_TOL
            assert rel_err(kernels.band(a, taps, dev(x)).cpu().numpy(), golden[key]) < F32_TOL
    for b in (5, 8):
        key = f"prim/sub/{n}/{b}"
        if key in golden:
            blk = golden[f"prim/sub_blk/{n}/{b}"]
            got = kernels.subblock(blk, x)
            assert rel_err(got, golden[key]) < F64_TOL
            assert np.array_equal(got[:, b:], x[:, b:])  # tail bit-identical
            got32 = kernels.subblock(blk, dev(x)).cpu().numpy()
            assert np.array_equal(got32[:, b:], x[:, b:].astype(np.float32))
    assert rel_err(kernels.dense(golden[f"prim/dense_m/{n}"], x), golden[f"prim/dense/{n}"]) < F64_TOL


def test_dense_rect(golden):
    got = kernels.dense(golden["prim/dense_rect_m"], golden["prim/dense_rect_x"])
    assert got.shape == (37, 16)
    assert rel_err(got, golden["prim/dense_rect"]) < F64_TOL


# ---------------------------------------------------------------- 1-D adjusted
ONE_D = ["band6_pre_dst3_dst7_n16", "band6_pre_dst3_dst7_n32", "band6_pre_dst3_dst7_n64",
         "band4_pre_dst3_dst7_n32", "sub8_post_dct2_dst7_n16", "sub8_post_dct2_dst7_n32",
         "sub8_post_dct2_dst7_n64", "sub8_post_dct2_dct8_n32"]


def _design(name):
    if name == "sub8_post_dct2_dct8_n32":
        return dct8_adjustment_from_dst7(matio.load_designed("sub8_post_dct2_dst7_n32"))
    return matio.load_designed(name)


@pytest.mark.parametrize("name", ONE_D)
def test_adjusted_1d(golden, name):
    adj = _design(name)
    t = pipeline.make_adjusted_transform(adj)
    x = golden[f"adj1d/{name}/x"]
    assert rel_err(pipeline.forward_adjusted(t, x), golden[f"adj1d/{name}/fwd"]) < F64_TOL
    assert rel_err(pipeline.inverse_adjusted(t, x), golden[f"adj1d/{name}/inv"]) < F64_TOL
    y32 = pipeline.forward_adjusted(t, dev(x)).cpu().numpy()
    assert rel_err(y32, golden[f"adj1d/{name}/fwd"]) < F32_TOL
    if "pre" in name:
        tf = pipeline.make_adjusted_transform(flip_pre_adjustment(adj))
        assert rel_err(pipeline.forward_adjusted(tf, x), golden[f"adj1d/{name}/fwd_flip"]) < F64_TOL
        assert rel_err(pipeline.inverse_adjusted(tf, x), golden[f"adj1d/{name}/inv_flip"]) < F64_TOL


def test_vector_input_and_roundtrip():
    t = pipeline.make_adjusted_transform(matio.load_designed("sub8_post_dct2_dst7_n32"))
    x = np.random.default_rng(1).standard_normal(32)
    y = pipeline.forward_adjusted(t, x)
    assert y.shape == (32,)
    assert np.abs(y - pipeline.dense_matrix(t) @ x).max() < 1e-9
    assert np.abs(pipeline.inverse_adjusted(t, y) - x).max() < 1e-9


@pytest.mark.parametrize("size", [16, 32, 64])
@pytest.mark.parametrize("kind", ["band", "subblock"])
def test_random_adjustments_match_dense(size, kind):
    # reference test_pipeline.py:161-176 with random-angle schedules
    if kind == "band":
        adj = random_adjustment(SparsityPattern.band(6, size), Side.PRE, TransformKind.DST3, 3)
    else:
        adj = random_adjustment(SparsityPattern.subblock(8, size), Side.POST, TransformKind.DCT2, 3)
    t = pipeline.make_adjusted_transform(adj)
    x = np.random.default_rng(size).standard_normal((50, size))
    y = pipeline.forward_adjusted(t, x)
    assert np.abs(y - x @ pipeline.dense_matrix(t).T).max() < 1e-9
    assert np.abs(pipeline.inverse_adjusted(t, y) - x).max() < 1e-9


@pytest.mark.parametrize("taps,order", [(3, None), (5, None), (None, 4), (None, 16)])
def test_generic_patterns_dense_composite(taps, order):
    """Widths without a specialised kernel run as a fused dense composite."""
    n = 32
    if taps:
        adj = random_adjustment(SparsityPattern.band(taps, n), Side.PRE, TransformKind.DST3, 7)
    else:
        adj = random_adjustment(SparsityPattern.subblock(order, n), Side.POST, TransformKind.DCT2, 7)
    t = pipeline.make_adjusted_transform(adj)
    x = np.random.default_rng(2).standard_normal((40, n))
    assert np.abs(pipeline.forward_adjusted(t, x) - x @ pipeline.dense_matrix(t).T).max() < 1e-9


def test_identity_adjustment_equals_base_bitwise():
    adj = identity_adjustment(SparsityPattern.band(6, 32), Side.PRE, TransformKind.DST3,
                              TransformKind.DST7)
    t = pipeline.make_adjusted_transform(adj)
    x = np.random.default_rng(3).standard_normal((70, 32))
    assert np.array_equal(pipeline.forward_adjusted(t, x), pipeline.fast_dst3_via_dct2(x))
    xd = dev(x)
    assert torch.equal(pipeline.forward_adjusted(t, xd), pipeline.fast_dst3_via_dct2(xd))


def test_subblock_tail_equals_own_dct2_bitwise():
    adj = random_adjustment(SparsityPattern.subblock(8, 32), Side.POST, TransformKind.DCT2, 4)
    t = pipeline.make_adjusted_transform(adj)
    x = dev(np.random.default_rng(4).standard_normal((100, 32)))
    y = pipeline.forward_adjusted(t, x)
    assert torch.equal(y[:, 8:], pipeline.fast_dct2(x)[:, 8:])


def test_zero_and_constant():
    z = np.zeros((5, 16))
    assert np.array_equal(pipeline.fast_dct2(z), z)
    y = pipeline.fast_dct2(np.full((1, 16), 1.7))
    assert abs(y[0, 0] - 1.7 * 4.0) < 1e-10 and np.abs(y[0, 1:]).max() < 1e-10


def test_linearity():
    t = pipeline.make_adjusted_transform(matio.load_designed("sub8_post_dct2_dst7_n32"))
    rng = np.random.default_rng(9)
    x1, x2 = rng.standard_normal(32), rng.standard_normal(32)
    lhs = pipeline.forward_adjusted(t, 2.5 * x1 - 0.7 * x2)
    rhs = 2.5 * pipeline.forward_adjusted(t, x1) - 0.7 * pipeline.forward_adjusted(t, x2)
    assert np.abs(lhs - rhs).max() < 1e-9


# ---------------------------------------------------------------- errors / edges
def test_errors_match_reference_classes():
    with pytest.raises(InvalidDimensionError):
        pipeline.fast_dct2(np.zeros((2, 12)))
    with pytest.raises(InvalidDimensionError):
        pipeline.fast_dct2(np.zeros((2, 128)))
    t = pipeline.make_adjusted_transform(matio.load_designed("sub8_post_dct2_dst7_n32"))
    with pytest.raises(ShapeError):
        pipeline.forward_adjusted(t, np.zeros(16))
    with pytest.raises(ShapeError):
        pipeline.forward_adjusted(t, np.zeros((2, 2, 32)))
    band = matio.load_designed("band6_pre_dst3_dst7_n32")
    with pytest.raises(PatternError):
        pipeline.apply_subblock(band, np.zeros(32))
    with pytest.raises(PatternError):
        pipeline.apply_band(matio.load_designed("sub8_post_dct2_dst7_n32"), np.zeros(32))
    bad = identity_adjustment(SparsityPattern.band(4, 16), Side.PRE, TransformKind.DST2,
                              TransformKind.DST7)
    with pytest.raises(ConfigurationError):
        pipeline.make_adjusted_transform(bad)


@pytest.mark.parametrize("nvec", [0, 1, 31, 33, 1000])
def test_ragged_and_empty_batches(nvec):
    x = np.random.default_rng(nvec).standard_normal((nvec, 32))
    y = kernels.dst3(x)
    assert y.shape == (nvec, 32)
    if nvec:
        assert np.abs(y - O.dst3(x)).max() < 1e-12


def test_readonly_input_accepted():
    x = np.random.default_rng(0).standard_normal((4, 16))
    x.setflags(write=False)
    kernels.dct2(x)


# ---------------------------------------------------------------- 2-D configs
def test_c1_forward_fp64(golden):
    t = pipeline.make_adjusted_transform(matio.load_designed("band6_pre_dst3_dst7_n32"))
    y = pipeline.forward_adjusted_2d(t, t, dev(golden["c1/x"], torch.float64))
    assert rel_err(y.cpu().numpy(), golden["c1/y"]) < F64_TOL


def test_c2_roundtrip_fp32_integer(golden):
    t = pipeline.make_adjusted_transform(
        dct8_adjustment_from_dst7(matio.load_designed("sub8_post_dct2_dst7_n32")))
    x = dev(golden["c2/x"])
    y = pipeline.forward_adjusted_2d(t, t, x)
    assert rel_err(y.cpu().numpy(), golden["c2/y"]) < F32_TOL
    xr = pipeline.inverse_adjusted_2d(t, t, y)
    assert rel_err(xr.cpu().numpy(), golden["c2/x"]) < F32_TOL
    assert torch.equal(torch.round(xr), x)  # bit-exact integer recovery (D7 iii)


# ---------------------------------------------------------------- fused round trip
def _rt_transforms(n=32):
    s7 = matio.load_designed(f"sub8_post_dct2_dst7_n{n}")
    b6 = matio.load_designed(f"band6_pre_dst3_dst7_n{n}")
    return {"dct8_post": dct8_adjustment_from_dst7(s7), "dst7_post": s7, "dst7_pre": b6,
            "dct8_pre": flip_pre_adjustment(b6)}


@pytest.mark.parametrize("tag", ["dct8_post", "dst7_post", "dst7_pre", "dct8_pre"])
@pytest.mark.parametrize("n,nblk", [(32, 1), (32, 3), (32, 1000), (32, 4099), (64, 1), (64, 777)])
def test_roundtrip_fused_equals_two_calls(tag, n, nblk):
    """One-kernel round trip == forward_adjusted_2d then inverse_adjusted_2d, bit
    for bit (partial super-tiles included), and y matches the oracle."""
    adj = _rt_transforms(n)[tag]
    t = pipeline.make_adjusted_transform(adj)
    g = torch.Generator(device="cuda").manual_seed(nblk)
    x = torch.randn(nblk, n, n, device="cuda", generator=g) * 24
    y, xr = pipeline.roundtrip_adjusted_2d(t, t, x)
    y2 = pipeline.forward_adjusted_2d(t, t, x)
    xr2 = pipeline.inverse_adjusted_2d(t, t, y2)
    assert torch.equal(y, y2) and torch.equal(xr, xr2)
    assert rel_err(xr.cpu().numpy(), x.cpu().numpy()) < F32_TOL
    ax = oaxis(adj)
    k = min(nblk, 64)
    ref = O.adjusted_2d(ax, ax, x[:k].cpu().numpy().astype(np.float64))
    assert rel_err(y[:k].cpu().numpy(), ref) < F32_TOL


def test_roundtrip_c2_integer_exact_and_fp64(golden):
    t = pipeline.make_adjusted_transform(_rt_transforms()["dct8_post"])
    x = dev(golden["c2/x"])
    y, xr = pipeline.roundtrip_adjusted_2d(t, t, x)
    assert rel_err(y.cpu().numpy(), golden["c2/y"]) < F32_TOL
    assert torch.equal(torch.round(xr), x)  # D7 (iii)
    # fp64 (no fused instantiation: the two-kernel path, same contract)
    x64 = x.double()
    y64, xr64 = pipeline.roundtrip_adjusted_2d(t, t, x64)
    assert rel_err(y64.cpu().numpy(), golden["c2/y"]) < F32_TOL
    assert torch.equal(y64, pipeline.forward_adjusted_2d(t, t, x64))
    assert rel_err(xr64.cpu().numpy(), x64.cpu().numpy()) < F64_TOL


def test_roundtrip_empty_and_bad_shapes():
    t = pipeline.make_adjusted_transform(_rt_transforms()["dct8_post"])
    y, xr = pipeline.roundtrip_adjusted_2d(t, t, torch.empty(0, 32, 32, device="cuda"))
    assert y.shape == (0, 32, 32) and xr.shape == (0, 32, 32)
    yh, xh = pipeline.roundtrip_adjusted_2d_host(t, t, np.zeros((0, 32, 32), np.float32))
    assert yh.shape == (0, 32, 32) and xh.shape == (0, 32, 32)
    with pytest.raises(ShapeError):
        pipeline.roundtrip_adjusted_2d(t, t, torch.zeros(4, 32, 16, device="cuda"))
    with pytest.raises(ShapeError):
        pipeline.roundtrip_adjusted_2d_host(t, t, np.zeros((4, 16, 32), np.float32))
    batch = pipeline.MixedBatch.packed(np.zeros(0, np.int64), np.zeros(0, np.int64), [16, 16, 32, 32])
    y, xr = pipeline.mixed_roundtrip(batch, _c3_table("post"), torch.empty(0, device="cuda"))
    assert y.numel() == 0 and xr.numel() == 0


def test_roundtrip_in_place_and_alias_rule():
    """xr may alias x (C-ABI); y aliasing xr is rejected before any work."""
    import ctypes
    from paper_2505_23618_b200 import _lib
    t = pipeline.make_adjusted_transform(_rt_transforms()["dct8_post"])
    x = torch.randn(257, 32, 32, device="cuda") * 24
    y_ref, xr_ref = pipeline.roundtrip_adjusted_2d(t, t, x)
    buf = x.clone()
    y = torch.empty_like(x)
    (ax, _k) = t.axis()
    lib = _lib.load()
    st = torch.cuda.current_stream().cuda_stream
    _lib.check(lib.dctadj_roundtrip_2d(ctypes.byref(ax), ctypes.byref(ax), buf.data_ptr(),
                                       y.data_ptr(), buf.data_ptr(), 257, _lib.F32, st))
    assert torch.equal(y, y_ref) and torch.equal(buf, xr_ref)
    with pytest.raises(ValueError):
        _lib.check(lib.dctadj_roundtrip_2d(ctypes.byref(ax), ctypes.byref(ax), x.data_ptr(),
                                           y.data_ptr(), y.data_ptr(), 257, _lib.F32, st))


def test_c2_host_entry(golden):
    t = pipeline.make_adjusted_transform(
        dct8_adjustment_from_dst7(matio.load_designed("sub8_post_dct2_dst7_n32")))
    x = np.ascontiguousarray(golden["c2/x"])
    y = pipeline.forward_adjusted_2d_host(t, t, x)
    assert y.dtype == np.float32
    assert rel_err(y, golden["c2/y"]) < F32_TOL
    xr = pipeline.inverse_adjusted_2d_host(t, t, y)
    assert np.array_equal(np.rint(xr), x)
    # round trip in one pipelined pass: identical to the two calls, bit for bit,
    # also across several pipeline chunks (1 MB chunks -> 16+ chunks here)
    y2, xr2 = pipeline.roundtrip_adjusted_2d_host(t, t, x)
    assert np.array_equal(y2, y) and np.array_equal(xr2, xr)
    big = np.ascontiguousarray(np.tile(x, (max(1, 4096 // x.shape[0]), 1, 1)))
    yb, xb = pipeline.roundtrip_adjusted_2d_host(t, t, big)
    assert np.array_equal(yb, pipeline.forward_adjusted_2d_host(t, t, big))
    assert np.array_equal(np.rint(xb), big)
    for fp64 in (False, True):
        xin = big.astype(np.float64) if fp64 else big
        yb, xb = pipeline.roundtrip_adjusted_2d_host(t, t, xin)
        assert rel_err(xb, xin) < (F64_TOL if fp64 else F32_TOL)


@pytest.mark.parametrize("tag", ["dst7_pre", "dct8_pre", "dst7_post", "dct8_post"])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_c4_n64_variants(golden, tag, dtype):
    b6 = matio.load_designed("band6_pre_dst3_dst7_n64")
    s7 = matio.load_designed("sub8_post_dct2_dst7_n64")
    adj = {"dst7_pre": b6, "dct8_pre": flip_pre_adjustment(b6), "dst7_post": s7,
           "dct8_post": dct8_adjustment_from_dst7(s7)}[tag]
    t = pipeline.make_adjusted_transform(adj)
    tol = F32_TOL if dtype == torch.float32 else F64_TOL
    x = dev(golden["c4/x"], dtype)
    assert rel_err(pipeline.forward_adjusted_2d(t, t, x).cpu().numpy(), golden[f"c4/{tag}/y"]) < tol
    assert rel_err(pipeline.inverse_adjusted_2d(t, t, x).cpu().numpy(), golden[f"c4/{tag}/xr"]) < tol


@pytest.mark.parametrize("shape", [(16, 16), (16, 32), (32, 16), (32, 32)])
@pytest.mark.parametrize("side", ["pre", "post"])
def test_c3_shapes_and_pairs(golden, shape, side):
    h, w = shape
    pre = {n: matio.load_designed(f"band6_pre_dst3_dst7_n{n}") for n in (16, 32)}
    post = {n: matio.load_designed(f"sub8_post_dct2_dst7_n{n}") for n in (16, 32)}

    def adj(n, kind):
        if side == "pre":
            return pre[n] if kind == "dst7" else flip_pre_adjustment(pre[n])
        return post[n] if kind == "dst7" else dct8_adjustment_from_dst7(post[n])

    x = dev(golden[f"c3/{h}x{w}/x"])
    for kh in ("dst7", "dct8"):
        for kv in ("dst7", "dct8"):
            th = pipeline.make_adjusted_transform(adj(w, kh))
            tv = pipeline.make_adjusted_transform(adj(h, kv))
            k = f"c3/{h}x{w}/{side}/{kh}_{kv}"
            assert rel_err(pipeline.forward_adjusted_2d(th, tv, x).cpu().numpy(), golden[k + "/y"]) < F32_TOL
            assert rel_err(pipeline.inverse_adjusted_2d(th, tv, x).cpu().numpy(), golden[k + "/xr"]) < F32_TOL


def test_c5_frames(golden):
    t = pipeline.make_adjusted_transform(matio.load_designed("sub8_post_dct2_dst7_n32"))
    frames = dev(golden["c5/frames"])
    y = pipeline.forward_frames(t, t, frames)
    assert tuple(y.shape) == (12, 32, 32)
    assert rel_err(y.cpu().numpy(), golden["c5/y"]) < F32_TOL
    back = pipeline.inverse_frames(t, t, y, 48, 96)
    assert rel_err(back.cpu().numpy(), golden["c5/frames"]) < F32_TOL
    # exact dense DST-7 comparison path on the same tiles
    d7 = build_transform(TransformKind.DST7, 32).entries
    from paper_2505_23618_b200.design import AdjustmentMatrix, pattern_schedule_template
    dense = AdjustmentMatrix(SparsityPattern.dense(32), Side.POST, TransformKind.DCT2,
                             TransformKind.DST7, pattern_schedule_template(SparsityPattern.dense(32)),
                             d7 @ build_transform(TransformKind.DCT2, 32).entries.T)
    td = pipeline.make_adjusted_transform(dense)
    ye = pipeline.forward_frames(td, td, frames)
    assert rel_err(ye.cpu().numpy(), golden["c5/y_exact"]) < F32_TOL


def test_2d_identity_tail_bitwise():
    """Coefficients outside the first 8 rows/cols of a sub8-post 2-D transform
    equal the plain 2-D DCT-2 bit for bit (reference test_pipeline.py:235-241)."""
    adj = random_adjustment(SparsityPattern.subblock(8, 32), Side.POST, TransformKind.DCT2, 5)
    t = pipeline.make_adjusted_transform(adj)
    plain = pipeline.make_adjusted_transform(identity_adjustment(
        SparsityPattern.subblock(8, 32), Side.POST, TransformKind.DCT2, TransformKind.DCT2))
    x = dev(np.random.default_rng(6).standard_normal((64, 32, 32)))
    y = pipeline.forward_adjusted_2d(t, t, x)
    y0 = pipeline.forward_adjusted_2d(plain, plain, x)
    assert torch.equal(y[:, 8:, 8:], y0[:, 8:, 8:])


def test_large_batch_properties():
    """Full-size style check without the oracle: round trip + linearity on
    65,536 blocks (config 2's size)."""
    t = pipeline.make_adjusted_transform(
        dct8_adjustment_from_dst7(matio.load_designed("sub8_post_dct2_dst7_n32")))
    g = torch.Generator(device="cuda").manual_seed(2)
    x = torch.round(torch.randn(65536, 32, 32, device="cuda", generator=g) * 24).clamp_(-512, 511)
    y = pipeline.forward_adjusted_2d(t, t, x)
    xr = pipeline.inverse_adjusted_2d(t, t, y)
    assert torch.equal(torch.round(xr), x)
    # energy preservation (orthogonal transform)
    e_in, e_out = (x.double() ** 2).sum().item(), (y.double() ** 2).sum().item()
    assert abs(e_out / e_in - 1) < 1e-6
    # spot-check 512 random blocks against the oracle
    idx = torch.randint(0, 65536, (512,), device="cuda", generator=g)
    xs = x[idx].cpu().numpy().astype(np.float64)
    ax = oaxis(t.adjustment)
    assert rel_err(y[idx].cpu().numpy(), O.adjusted_2d(ax, ax, xs)) < F32_TOL


# ---------------------------------------------------------------- mixed batches (C3)
def _c3_table(side):
    from paper_2505_23618_b200.design import dct8_adjustment_from_dst7 as d8
    tab = []
    for n in (16, 32):
        if side == "pre":
            a = matio.load_designed(f"band6_pre_dst3_dst7_n{n}")
            tab += [a, flip_pre_adjustment(a)]
        else:
            a = matio.load_designed(f"sub8_post_dct2_dst7_n{n}")
            tab += [a, d8(a)]
    return [pipeline.make_adjusted_transform(a) for a in tab]  # [16/dst7, 16/dct8, 32/dst7, 32/dct8]


@pytest.mark.parametrize("side", ["pre", "post"])
@pytest.mark.parametrize("nblk", [1, 7, 301])
def test_mixed_batch_matches_oracle(side, nblk):
    rng = np.random.default_rng(nblk)
    h_index = rng.integers(0, 4, nblk)
    v_index = rng.integers(0, 4, nblk)
    batch = pipeline.MixedBatch.packed(h_index, v_index, [16, 16, 32, 32])
    table = _c3_table(side)
    x = rng.standard_normal(batch.total_elements).astype(np.float32) * 20
    y = pipeline.mixed_forward(batch, table, dev(x)).cpu().numpy()
    xr = pipeline.mixed_inverse(batch, table, dev(y)).cpu().numpy()
    for (o, h, w), hi, vi in zip(batch.block_slices(), h_index, v_index):
        blk = x[o:o + h * w].reshape(1, h, w).astype(np.float64)
        ref = O.adjusted_2d(oaxis(table[hi].adjustment), oaxis(table[vi].adjustment), blk)
        assert rel_err(y[o:o + h * w].reshape(1, h, w), ref) < F32_TOL
        assert rel_err(xr[o:o + h * w].reshape(1, h, w), blk) < F32_TOL


@pytest.mark.parametrize("side", ["pre", "post"])
@pytest.mark.parametrize("nblk", [1, 7, 301, 5000])
def test_mixed_roundtrip_equals_two_calls(side, nblk):
    """Fused per-class round trip == mixed_forward then mixed_inverse, bit for bit
    (partial super-tiles of every class), also with shuffled block offsets."""
    from paper_2505_23618_b200 import _lib
    rng = np.random.default_rng(100 + nblk)
    h_index = rng.integers(0, 4, nblk)
    v_index = rng.integers(0, 4, nblk)
    sizes = np.array([16, 16, 32, 32])
    areas = sizes[h_index] * sizes[v_index]
    order = rng.permutation(nblk)
    offs = np.zeros(nblk, np.int64)
    offs[order] = np.concatenate([[0], np.cumsum(areas[order])[:-1]])
    batch = pipeline.MixedBatch(offs, h_index, v_index, sizes, int(areas.sum()))
    table = _c3_table(side)
    axes = (_lib.Axis * 4)()
    keep = []
    for k, tr in enumerate(table):
        axes[k], m = tr.axis()
        keep.append(m)
    assert _lib.load().dctadj_mixed_roundtrip_fused(batch._plan, axes, _lib.F32) == 1
    x = dev(rng.standard_normal(batch.total_elements).astype(np.float32) * 20)
    y, xr = pipeline.mixed_roundtrip(batch, table, x)
    y2 = pipeline.mixed_forward(batch, table, x)
    assert torch.equal(y, y2)
    assert torch.equal(xr, pipeline.mixed_inverse(batch, table, y2))


def test_mixed_batch_shuffled_offsets_and_errors():
    rng = np.random.default_rng(3)
    nblk = 64
    h_index = rng.integers(0, 4, nblk)
    v_index = rng.integers(0, 4, nblk)
    sizes = np.array([16, 16, 32, 32])
    areas = sizes[h_index] * sizes[v_index]
    order = rng.permutation(nblk)                      # blocks stored out of order
    offs = np.zeros(nblk, np.int64)
    offs[order] = np.concatenate([[0], np.cumsum(areas[order])[:-1]])
    batch = pipeline.MixedBatch(offs, h_index, v_index, sizes, int(areas.sum()))
    table = _c3_table("post")
    x = rng.standard_normal(batch.total_elements).astype(np.float32)
    y = pipeline.mixed_forward(batch, table, dev(x)).cpu().numpy()
    for (o, h, w), hi, vi in zip(batch.block_slices(), h_index, v_index):
        ref = O.adjusted_2d(oaxis(table[hi].adjustment), oaxis(table[vi].adjustment),
                            x[o:o + h * w].reshape(1, h, w).astype(np.float64))
        assert rel_err(y[o:o + h * w].reshape(1, h, w), ref) < F32_TOL
    with pytest.raises(ShapeError):
        pipeline.MixedBatch([8], [2], [2], sizes, 4096)        # offset not a multiple of W
    with pytest.raises(ShapeError):
        pipeline.MixedBatch([0], [2], [2], sizes, 512)         # block overruns the buffer
    with pytest.raises(ShapeError):
        pipeline.mixed_forward(batch, table[:2], dev(x))


# ---------------------------------------------------------------- encoder evaluation (Table 1 "Multiple")
@pytest.mark.parametrize("tag,hn,vn", [("32x32", 32, 32), ("32x64", 64, 32), ("16x16", 16, 16)])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_encoder_eval_matches_reference(golden, tag, hn, vn, dtype):
    ctx = pipeline.EncoderContext(horizontal=matio.load_designed(f"sub8_post_dct2_dst7_n{hn}"),
                                  vertical=matio.load_designed(f"sub8_post_dct2_dst7_n{vn}"))
    x = dev(golden[f"enc5/{tag}/x"], dtype)
    res = pipeline.simultaneous_encoder_eval(x, ctx)
    tol = F32_TOL if dtype == torch.float32 else F64_TOL
    assert set(res) == set(pipeline.ENCODER_KEYS)
    for k, v in res.items():
        assert rel_err(v.cpu().numpy(), golden[f"enc5/{tag}/{k[0]}_{k[1]}"]) < tol, k
    ref = res[("dct2", "dct2")]
    for k, v in res.items():  # untouched coefficients bit-identical (test_pipeline.py:235-241)
        assert torch.equal(v[:, 8:, 8:], ref[:, 8:, 8:]), k
    naive = pipeline.naive_encoder_eval(x, ctx)
    for k in res:
        assert rel_err(res[k].cpu().numpy(), naive[k].cpu().numpy().astype(np.float64)) < tol, k


def test_encoder_eval_errors_and_numpy_block():
    ctx = pipeline.EncoderContext()
    with pytest.raises(ConfigurationError):
        pipeline.simultaneous_encoder_eval(np.zeros((32, 32)), ctx)
    band = matio.load_designed("band6_pre_dst3_dst7_n32")
    with pytest.raises(ConfigurationError):
        pipeline.simultaneous_encoder_eval(np.zeros((32, 32)),
                                           pipeline.EncoderContext(band, band))
    s32 = matio.load_designed("sub8_post_dct2_dst7_n32")
    with pytest.raises(ConfigurationError):
        pipeline.simultaneous_encoder_eval(np.zeros((64, 64)), pipeline.EncoderContext(s32, s32))
    out = pipeline.simultaneous_encoder_eval(np.zeros((32, 32)), pipeline.EncoderContext(s32, s32))
    assert len(out) == 5 and all(np.array_equal(v, np.zeros((32, 32))) for v in out.values())


# ------------------------------------------- dense 32x32 fp32 on the tensor cores
# (csrc/dense_tc.cuh: 3xTF32 tcgen05 kernel, TMEM operands, dynamic tile counter)
def _dense_pair(seed_h, seed_v):
    mk = lambda s: pipeline.make_adjusted_transform(  # noqa: E731
        random_adjustment(SparsityPattern.dense(32), Side.POST, TransformKind.DCT2, s))
    return mk(seed_h), mk(seed_v)


@pytest.mark.parametrize("nblk", [1, 3, 4, 5, 37, 600, 4099])
def test_dense_tc_2d_ragged(nblk):
    """Row and column matrices differ (catches a transposed pass); block counts
    that are not multiples of the 4-block super-tile; oracle parity both ways."""
    th, tv = _dense_pair(11, 12)
    x = np.random.default_rng(nblk).standard_normal((nblk, 32, 32))
    ah, av = oaxis(th.adjustment), oaxis(tv.adjustment)
    y = pipeline.forward_adjusted_2d(th, tv, dev(x)).cpu().numpy()
    assert rel_err(y, O.adjusted_2d(ah, av, x)) < F32_TOL
    xr = pipeline.inverse_adjusted_2d(th, tv, dev(y)).cpu().numpy()
    assert rel_err(xr, O.adjusted_2d(ah, av, y.astype(np.float64), inverse=True)) < F32_TOL


def test_dense_tc_repeat_and_streams():
    """The dynamic tile counter re-arms itself: repeated launches on one stream and
    launches on a second stream give identical results."""
    th, tv = _dense_pair(13, 14)
    x = torch.randn(20000, 32, 32, device="cuda")
    y0 = pipeline.forward_adjusted_2d(th, tv, x)
    for _ in range(3):
        assert torch.equal(pipeline.forward_adjusted_2d(th, tv, x), y0)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        y1 = pipeline.forward_adjusted_2d(th, tv, x)
    s.synchronize()
    assert torch.equal(y1, y0)


@pytest.mark.parametrize("shape", [(2, 70, 256), (1, 32, 128), (3, 33, 384)])
def test_dense_tc_frames_4wide(shape):
    """Frames whose width holds a multiple of 4 blocks take the one-box-per-
    super-tile TMA path (FRAME4): forward against numpy on zero-padded tiles,
    inverse back to the (clipped) frames."""
    th, tv = _dense_pair(15, 16)
    f, h, w = shape
    fr = np.random.default_rng(h).standard_normal(shape)
    ty, tx = -(-h // 32), w // 32
    pad = np.zeros((f, ty * 32, w))
    pad[:, :h] = fr
    blocks = pad.reshape(f, ty, 32, tx, 32).transpose(0, 1, 3, 2, 4).reshape(-1, 32, 32)
    mh, mv = pipeline.dense_matrix(th), pipeline.dense_matrix(tv)
    want = mv @ blocks @ mh.T
    y = pipeline.forward_frames(th, tv, dev(fr))
    assert rel_err(y.cpu().numpy(), want) < F32_TOL
    back = pipeline.inverse_frames(th, tv, y, h, w).cpu().numpy()
    assert rel_err(back.reshape(f, h, w), fr) < F32_TOL


def _frame_tiles(fr, ty, tx):
    f, h, w = fr.shape
    pad = np.zeros((f, ty * 32, tx * 32))
    pad[:, :h, :w] = fr
    return pad.reshape(f, ty, 32, tx, 32).transpose(0, 1, 3, 2, 4).reshape(-1, 32, 32)


@pytest.mark.parametrize("shape", [(2, 70, 128), (1, 64, 64), (3, 40, 192), (2, 33, 96)])
@pytest.mark.parametrize("name", ["sub8_post_dct2_dst7_n32", "band6_pre_dst3_dst7_n32"])
def test_frames_interleaved_and_fallback(shape, name):
    """Frame widths holding whole super-tiles take the interleaved one-box path
    (FRAME_IL / LINEAR_IL); odd block counts per row (96 = 3 blocks) fall back to
    per-block boxes.  Oracle parity forward, exact round trip back."""
    adj = matio.load_designed(name)
    t = pipeline.make_adjusted_transform(adj)
    f, h, w = shape
    fr = np.round(np.random.default_rng(w + h).standard_normal(shape) * 40)
    y = pipeline.forward_frames(t, t, dev(fr))
    ax = oaxis(adj)
    want = O.adjusted_2d(ax, ax, _frame_tiles(fr, -(-h // 32), w // 32))
    assert rel_err(y.cpu().numpy(), want) < F32_TOL
    back = pipeline.inverse_frames(t, t, y, h, w)
    assert torch.equal(torch.round(back), dev(fr))


def _exact_dst7_transform():
    from paper_2505_23618_b200.design import AdjustmentMatrix, pattern_schedule_template
    d7 = build_transform(TransformKind.DST7, 32).entries
    dense = AdjustmentMatrix(SparsityPattern.dense(32), Side.POST, TransformKind.DCT2,
                             TransformKind.DST7, pattern_schedule_template(SparsityPattern.dense(32)),
                             d7 @ build_transform(TransformKind.DCT2, 32).entries.T)
    return pipeline.make_adjusted_transform(dense)


@pytest.mark.parametrize("shape", [(2, 70, 256), (1, 64, 128), (3, 40, 384), (2, 33, 96)])
@pytest.mark.parametrize("name", ["sub8_post_dct2_dst7_n32", "band6_pre_dst3_dst7_n32"])
def test_frames_exact_fused(shape, name):
    """Config 5's comparison step in one call (fused tensor-core kernel when the
    width holds 4-block super-tiles, the two-launch path otherwise): both outputs
    against the oracle / numpy, the per-frame error sums against numpy on them."""
    adj = matio.load_designed(name)
    t = pipeline.make_adjusted_transform(adj)
    te = _exact_dst7_transform()
    f, h, w = shape
    fr = np.random.default_rng(h * w).standard_normal(shape) * 30
    ya, ye, err = pipeline.forward_frames_exact(t, t, te, te, dev(fr))
    ty, tx = -(-h // 32), w // 32
    blocks = _frame_tiles(fr, ty, tx)
    ax = oaxis(adj)
    assert rel_err(ya.cpu().numpy(), O.adjusted_2d(ax, ax, blocks)) < F32_TOL
    me = pipeline.dense_matrix(te)
    assert rel_err(ye.cpu().numpy(), me @ blocks @ me.T) < F32_TOL
    a = ya.double().cpu().numpy().reshape(f, ty, tx, 32, 32)
    e = ye.double().cpu().numpy().reshape(f, ty, tx, 32, 32)
    full = h // 32
    want = np.stack([((a - e) ** 2).sum(axis=(1, 2, 3, 4)), (e ** 2).sum(axis=(1, 2, 3, 4)),
                     ((a - e)[:, :full] ** 2).sum(axis=(1, 2, 3, 4)),
                     (e[:, :full] ** 2).sum(axis=(1, 2, 3, 4))], axis=1)
    got = err.cpu().numpy()
    assert got.shape == (f, 4)
    assert np.allclose(got, want, rtol=1e-5, atol=1e-9 * want[:, 1:2].max())


def test_frames_exact_without_error_matches():
    """err = NULL takes the two-launch path; its outputs agree with the fused one."""
    t = pipeline.make_adjusted_transform(matio.load_designed("sub8_post_dct2_dst7_n32"))
    te = _exact_dst7_transform()
    fr = dev(np.random.default_rng(9).standard_normal((2, 64, 256)) * 30)
    ya, ye, err = pipeline.forward_frames_exact(t, t, te, te, fr)
    yb, yeb, none = pipeline.forward_frames_exact(t, t, te, te, fr, with_error=False)
    assert none is None
    assert rel_err(ya.cpu().numpy(), yb.double().cpu().numpy()) < F32_TOL
    assert rel_err(ye.cpu().numpy(), yeb.double().cpu().numpy()) < F32_TOL


def test_misaligned_views_and_pointers():
    """A tensor view at a non-16-byte offset is copied by the Python layer (like
    the reference's ascontiguousarray); a raw misaligned pointer through the
    C-ABI is a ValueError, not a TMA fault."""
    import ctypes
    from paper_2505_23618_b200 import _lib
    t = pipeline.make_adjusted_transform(matio.load_designed("sub8_post_dct2_dst7_n32"))
    base = torch.randn(5 * 32 + 1, 32, device="cuda")
    view = base.view(-1)[1:1 + 4 * 32 * 32].view(4, 32, 32)  # 4-byte offset
    assert view.data_ptr() % 16
    got = pipeline.forward_adjusted_2d(t, t, view)
    want = pipeline.forward_adjusted_2d(t, t, view.clone())
    assert torch.equal(got, want)
    ax, _keep = t.axis()
    out = torch.empty(4, 32, 32, device="cuda")
    with pytest.raises(ValueError):
        _lib.call("dctadj_forward_2d", ctypes.byref(ax), ctypes.byref(ax), view.data_ptr(),
                  out.data_ptr(), 4, _lib.F32, torch.cuda.current_stream().cuda_stream)


def _dense_pair_n(n, seed_h, seed_v):
    mk = lambda s: pipeline.make_adjusted_transform(  # noqa: E731
        random_adjustment(SparsityPattern.dense(n), Side.POST, TransformKind.DCT2, s))
    return mk(seed_h), mk(seed_v)


@pytest.mark.parametrize("nblk", [1, 2, 3, 37, 1001])
def test_dense_tc64_2d_ragged(nblk):
    """64x64 fp32 dense on the tensor cores (dense_tc64.cuh): distinct row / column
    matrices, odd block counts (half-empty 2-block super-tiles), oracle parity."""
    th, tv = _dense_pair_n(64, 21, 22)
    x = np.random.default_rng(nblk).standard_normal((nblk, 64, 64))
    ah, av = oaxis(th.adjustment), oaxis(tv.adjustment)
    y = pipeline.forward_adjusted_2d(th, tv, dev(x)).cpu().numpy()
    assert rel_err(y, O.adjusted_2d(ah, av, x)) < F32_TOL
    xr = pipeline.inverse_adjusted_2d(th, tv, dev(y)).cpu().numpy()
    assert rel_err(xr, O.adjusted_2d(ah, av, y.astype(np.float64), inverse=True)) < F32_TOL


def test_dense_tc64_repeat_and_streams():
    th, tv = _dense_pair_n(64, 23, 24)
    x = torch.randn(5000, 64, 64, device="cuda")
    y0 = pipeline.forward_adjusted_2d(th, tv, x)
    for _ in range(3):
        assert torch.equal(pipeline.forward_adjusted_2d(th, tv, x), y0)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        y1 = pipeline.forward_adjusted_2d(th, tv, x)
    s.synchronize()
    assert torch.equal(y1, y0)


@pytest.mark.parametrize("n", [16, 32, 64])
@pytest.mark.parametrize("big", [False, True])
def test_givens_scaled_rotations_and_large_angle_fallback(n, big):
    """Band pre-adjustments run their Givens schedule as scaled rotations (2 FMAs
    each, csrc/butterfly.cuh ST_GIVENS2) when every |cos theta| >= 0.2; a schedule
    with a steeper rotation falls back to the band product / dense composite.  Both
    must match the oracle (the realized matrix) in fp64 and fp32, 1-D and 2-D,
    forward and inverse."""
    import dataclasses

    from paper_2505_23618_b200.design import givens_to_matrix

    adj = matio.load_designed(f"band6_pre_dst3_dst7_n{n}")
    if big:  # one rotation at 84 degrees (cos 0.10): below the scaled form's bound
        th = adj.schedule.angles().copy()
        th[len(th) // 3] = np.radians(84.0)
        sch = adj.schedule.with_angles(th)
        adj = dataclasses.replace(adj, schedule=sch, realized=givens_to_matrix(sch))
    t = pipeline.make_adjusted_transform(adj)
    ax = oaxis(adj)
    rng = np.random.default_rng(n + 7 * big)
    x = rng.standard_normal((40, n, n)) * 24
    v = rng.standard_normal((100, n)) * 24
    for dtype, tol in ((torch.float64, F64_TOL), (torch.float32, F32_TOL)):
        xd = dev(x, dtype)
        y = pipeline.forward_adjusted_2d(t, t, xd)
        assert rel_err(y.cpu().numpy(), O.adjusted_2d(ax, ax, x)) < tol
        xr = pipeline.inverse_adjusted_2d(t, t, y)
        assert rel_err(xr.cpu().numpy(), x) < 10 * tol
        y1 = pipeline.forward_adjusted(t, dev(v, dtype))
        assert rel_err(y1.cpu().numpy(), O.adjusted_1d(ax, v)) < tol
        x1 = pipeline.inverse_adjusted(t, y1)
        assert rel_err(x1.cpu().numpy(), O.adjusted_1d(ax, y1.cpu().numpy().astype(np.float64),
                                                      inverse=True)) < tol
