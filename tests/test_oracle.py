"""CPU: the C oracle (oracle/dctadj_oracle.c) is pinned against golden vectors
the reference itself produced (tests/golden/gen_golden.py) and, when
oracle/_ref was built, against the reference's compiled core directly."""
import numpy as np
import pytest

from oracle import oracle as O

from conftest import rel_err

from paper_2505_23618_b200 import matio
from paper_2505_23618_b200.design import dct8_adjustment_from_dst7, flip_pre_adjustment


def oaxis(adj, base_code=None):
    """OAxis from an AdjustmentMatrix record (host records only, no device)."""
    base = {"dct2": O.BASE_DCT2, "dst3": O.BASE_DST3, "dct3": O.BASE_DCT3}[adj.base.value]
    kind = {"band": O.ADJ_BAND, "subblock": O.ADJ_SUBBLOCK, "dense": O.ADJ_DENSE}[adj.pattern.kind.value]
    return O.OAxis(adj.pattern.size, base if base_code is None else base_code, kind,
                   O.SIDE_PRE if adj.side.value == "pre" else O.SIDE_POST,
                   adj.pattern.taps or 0, adj.pattern.order or 0, np.array(adj.realized))


@pytest.mark.parametrize("n", [4, 8, 16, 32, 64])
@pytest.mark.parametrize("fn", ["dct2", "idct2", "dst3", "idst3"])
def test_transforms_match_reference(golden, n, fn):
    x = golden[f"prim/x/{n}"]
    got = getattr(O, fn)(x)
    # same factorization, same order, no FMA on x86-64 baseline: bit-identical
    assert np.array_equal(got, golden[f"prim/{fn}/{n}"])


@pytest.mark.parametrize("n", [4, 8, 16, 32, 64])
def test_band_sub_dense_match_reference(golden, n):
    x = golden[f"prim/x/{n}"]
    for taps in (3, 4, 6):
        key = f"prim/band/{n}/{taps}"
        if key in golden:
            assert np.array_equal(O.band(golden[f"prim/band_a/{n}/{taps}"], taps, x), golden[key])
    for b in (5, 8):
        key = f"prim/sub/{n}/{b}"
        if key in golden:
            got = O.subblock(golden[f"prim/sub_blk/{n}/{b}"], x)
            assert np.array_equal(got, golden[key])
            assert np.array_equal(got[:, b:], x[:, b:])
    assert np.abs(O.dense(golden[f"prim/dense_m/{n}"], x) - golden[f"prim/dense/{n}"]).max() < 1e-12


def test_dense_rect(golden):
    got = O.dense(golden["prim/dense_rect_m"], golden["prim/dense_rect_x"])
    assert np.abs(got - golden["prim/dense_rect"]).max() < 1e-12


ONE_D = ["band6_pre_dst3_dst7_n16", "band6_pre_dst3_dst7_n32", "band6_pre_dst3_dst7_n64",
         "band4_pre_dst3_dst7_n32", "sub8_post_dct2_dst7_n16", "sub8_post_dct2_dst7_n32",
         "sub8_post_dct2_dst7_n64", "sub8_post_dct2_dct8_n32"]


@pytest.mark.parametrize("name", ONE_D)
def test_adjusted_1d_match_reference(golden, name):
    adj = matio.load_designed(name)
    ax = oaxis(adj)
    x = golden[f"adj1d/{name}/x"]
    assert np.array_equal(O.adjusted_1d(ax, x), golden[f"adj1d/{name}/fwd"])
    assert np.array_equal(O.adjusted_1d(ax, x, inverse=True), golden[f"adj1d/{name}/inv"])
    if "pre" in name:
        # D3: DCT-3 base with the reversed band == reference flip form, to rounding
        fx = oaxis(flip_pre_adjustment(adj))
        assert rel_err(O.adjusted_1d(fx, x), golden[f"adj1d/{name}/fwd_flip"]) < 1e-13
        assert rel_err(O.adjusted_1d(fx, x, inverse=True), golden[f"adj1d/{name}/inv_flip"]) < 1e-13


def test_c1_c2_2d(golden):
    a6 = oaxis(matio.load_designed("band6_pre_dst3_dst7_n32"))
    assert np.array_equal(O.adjusted_2d(a6, a6, golden["c1/x"]), golden["c1/y"])
    s8 = oaxis(dct8_adjustment_from_dst7(matio.load_designed("sub8_post_dct2_dst7_n32")))
    x = golden["c2/x"].astype(np.float64)
    assert np.array_equal(O.adjusted_2d(s8, s8, x), golden["c2/y"])
    assert np.array_equal(O.adjusted_2d(s8, s8, golden["c2/y"], inverse=True), golden["c2/xr"])
    # integer round trip (App. A D7 iii)
    assert np.array_equal(np.rint(golden["c2/xr"]), x)


def test_c4_variants(golden):
    b6 = matio.load_designed("band6_pre_dst3_dst7_n64")
    s7 = matio.load_designed("sub8_post_dct2_dst7_n64")
    axes = {"dst7_pre": oaxis(b6), "dct8_pre": oaxis(flip_pre_adjustment(b6)),
            "dst7_post": oaxis(s7), "dct8_post": oaxis(dct8_adjustment_from_dst7(s7))}
    x = golden["c4/x"]
    for tag, ax in axes.items():
        assert rel_err(O.adjusted_2d(ax, ax, x), golden[f"c4/{tag}/y"]) < 1e-13, tag
        assert rel_err(O.adjusted_2d(ax, ax, x, inverse=True), golden[f"c4/{tag}/xr"]) < 1e-13, tag


def test_c3_mixed_shapes(golden):
    pre = {n: matio.load_designed(f"band6_pre_dst3_dst7_n{n}") for n in (16, 32)}
    post = {n: matio.load_designed(f"sub8_post_dct2_dst7_n{n}") for n in (16, 32)}
    for h, w in ((16, 16), (16, 32), (32, 16), (32, 32)):
        x = golden[f"c3/{h}x{w}/x"].astype(np.float64)
        for kh in ("dst7", "dct8"):
            for kv in ("dst7", "dct8"):
                ah = oaxis(pre[w] if kh == "dst7" else flip_pre_adjustment(pre[w]))
                av = oaxis(pre[h] if kv == "dst7" else flip_pre_adjustment(pre[h]))
                k = f"c3/{h}x{w}/pre/{kh}_{kv}"
                assert rel_err(O.adjusted_2d(ah, av, x), golden[k + "/y"]) < 1e-13
                assert rel_err(O.adjusted_2d(ah, av, x, inverse=True), golden[k + "/xr"]) < 1e-13
                ph = post[w] if kh == "dst7" else dct8_adjustment_from_dst7(post[w])
                pv = post[h] if kv == "dst7" else dct8_adjustment_from_dst7(post[h])
                k = f"c3/{h}x{w}/post/{kh}_{kv}"
                assert np.array_equal(O.adjusted_2d(oaxis(ph), oaxis(pv), x), golden[k + "/y"])


def test_f32_wrapper_and_threads(golden):
    s8 = oaxis(dct8_adjustment_from_dst7(matio.load_designed("sub8_post_dct2_dst7_n32")))
    y32 = O.adjusted_2d(s8, s8, golden["c2/x"], threads=2)
    assert y32.dtype == np.float32
    assert np.array_equal(y32, golden["c2/y"].astype(np.float32))


def test_against_reference_core_if_built():
    core = O.ref_fastcore()
    if core is None:
        pytest.skip("oracle/_ref not built (make -C oracle ref)")
    rng = np.random.default_rng(5)
    for n in (4, 8, 16, 32, 64):
        x = rng.standard_normal((33, n))
        for fn in ("dct2", "idct2", "dst3", "idst3"):
            assert np.array_equal(getattr(O, fn)(x), getattr(core, fn)(x))
    ref = O.RefPipeline(core)
    adj = oaxis(matio.load_designed("band6_pre_dst3_dst7_n32"))
    xb = rng.standard_normal((3, 32, 32))
    assert np.array_equal(O.adjusted_2d(adj, adj, xb), ref.forward_2d(adj, adj, xb))
    assert np.array_equal(O.adjusted_2d(adj, adj, xb, inverse=True), ref.inverse_2d(adj, adj, xb))


# ------------------------------------------------------------------ full-batch checkers
def test_check_2d_against_golden(golden):
    """The checkers the full-size GPU gates use: zero error on the reference's own
    outputs, and a perturbed / NaN block is found and counted."""
    a6 = oaxis(matio.load_designed("band6_pre_dst3_dst7_n32"))
    r = O.check_2d(a6, a6, golden["c1/x"], golden["c1/y"], tol=1e-9)
    assert r["max_err"] == 0.0 and r["over_tol"] == 0 and r["blocks"] == 6
    s8 = oaxis(dct8_adjustment_from_dst7(matio.load_designed("sub8_post_dct2_dst7_n32")))
    x32 = golden["c2/x"]
    y32 = golden["c2/y"].astype(np.float32)
    r = O.check_2d(s8, s8, x32, y32, tol=1e-5)
    assert r["max_err"] < 1e-7 and r["over_tol"] == 0  # fp32 rounding of the golden output only
    r = O.check_2d(s8, s8, y32, golden["c2/xr"].astype(np.float32), inverse=True, tol=1e-5)
    assert r["max_err"] < 1e-6
    bad = y32.copy()
    bad[4, 7, 7] += 0.01 * np.abs(bad[4]).max()
    bad[1, 0, 3] = np.nan
    r = O.check_2d(s8, s8, x32, bad, tol=1e-5, threads=3)
    assert r["over_tol"] == 2 and r["worst_block"] == 1 and r["max_err"] == np.inf


def test_check_mixed_and_frames_against_golden(golden):
    pre = {n: matio.load_designed(f"band6_pre_dst3_dst7_n{n}") for n in (16, 32)}
    table = [oaxis(pre[16]), oaxis(flip_pre_adjustment(pre[16])), oaxis(pre[32]),
             oaxis(flip_pre_adjustment(pre[32]))]
    xs, ys, hi, vi, offs = [], [], [], [], []
    off = 0
    for h, w in ((16, 16), (16, 32), (32, 16), (32, 32)):
        x = golden[f"c3/{h}x{w}/x"].astype(np.float64)
        for kh, kv in (("dst7", "dct8"), ("dct8", "dst7")):
            y = golden[f"c3/{h}x{w}/pre/{kh}_{kv}/y"]
            for b in range(x.shape[0]):
                xs.append(x[b].ravel())
                ys.append(y[b].ravel())
                hi.append((0 if w == 16 else 2) + (kh == "dct8"))
                vi.append((0 if h == 16 else 2) + (kv == "dct8"))
                offs.append(off)
                off += h * w
    xp, yp = np.concatenate(xs), np.concatenate(ys)
    r = O.check_mixed(table, hi, vi, offs, xp, yp, tol=1e-9)
    assert r["max_err"] < 1e-13 and r["over_tol"] == 0 and r["blocks"] == len(offs)
    yp[offs[5] + 3] += 1.0
    assert O.check_mixed(table, hi, vi, offs, xp, yp, tol=1e-9)["worst_block"] == 5
    # frames (config 5): padded 48 -> 64 rows, block-major coefficients
    s7 = oaxis(matio.load_designed("sub8_post_dct2_dst7_n32"))
    fr = golden["c5/frames"]
    r = O.check_frames(s7, s7, fr, golden["c5/y"].astype(np.float32), tol=1e-5)
    assert r["max_err"] < 1e-6 and r["blocks"] == golden["c5/y"].shape[0]
    inv = O.check_frames(s7, s7, fr, golden["c5/y"].astype(np.float32), inverse=True, tol=1e-5)
    assert inv["max_err"] < 1e-5
