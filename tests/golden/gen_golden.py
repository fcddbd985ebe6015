"""Generate golden input/output vectors by running the REFERENCE itself.

Fixture infrastructure (build container only; /root/reference does not exist
on the GPU box).  Imports the reference package `dctadjust` from a writable,
built copy of /root/reference/pkg (see gen_adjustments.py for the recipe),
runs its own kernels / pipeline entry points on seeded inputs, and writes
tests/golden/golden.npz.  The composition used for 2-D cases is the one the
reference's only 2-D code uses (rows, then columns: pipeline.py:236-239); the
inverse is its mirror (columns, then rows).  DCT-8 pre-adjustment cases use
the Eq. (3) flip of the DST-7 pipeline, forward_adjusted(t7, x[..., ::-1]) * S
(SURVEY.md App. A D3).

    REFPKG=/tmp/refbuild/src python tests/golden/gen_golden.py
"""
from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REFPKG = os.environ.get("REFPKG", "/tmp/refbuild/src")
sys.path.insert(0, REFPKG)

from dctadjust import kernels, matio  # noqa: E402
from dctadjust.design import (SparsityPattern, Side, dct8_adjustment_from_dst7,  # noqa: E402
                              givens_to_matrix, pattern_schedule_template, AdjustmentMatrix)
from dctadjust.pipeline import (forward_adjusted, inverse_adjusted,  # noqa: E402
                                make_adjusted_transform)
from dctadjust.transforms import TransformKind, alternating_signs, build_transform  # noqa: E402

assert kernels.BACKEND == "compiled", "build the reference's compiled core first"

HERE = Path(__file__).resolve().parent
ADJ = HERE.parents[1] / "paper_2505_23618_b200" / "adjustments"
out: dict[str, np.ndarray] = {}


def ar1_blocks(rng, nblk, h, w, rho, sigma):
    def chol(n):
        i = np.arange(n)
        return np.linalg.cholesky(rho ** np.abs(i[:, None] - i[None, :]).astype(float))
    lv, lh = chol(h), chol(w)
    z = rng.standard_normal((nblk, h, w))
    return sigma * lv @ z @ lh.T


def design(name):
    return matio.read_adjustment(ADJ / f"{name}.adj")


def fwd1(t, x, flip=False):
    """1-D forward through the reference; flip = DCT-8 pre via Eq. (3)."""
    if flip:
        s = alternating_signs(t.size)
        return forward_adjusted(t, np.ascontiguousarray(x[:, ::-1])) * s
    return forward_adjusted(t, x)


def inv1(t, y, flip=False):
    if flip:
        s = alternating_signs(t.size)
        return np.ascontiguousarray(inverse_adjusted(t, y * s)[:, ::-1])
    return inverse_adjusted(t, y)


def fwd2(th, tv, x, fh=False, fv=False):
    b, h, w = x.shape
    rows = fwd1(th, x.reshape(b * h, w), fh).reshape(b, h, w)
    cols = np.ascontiguousarray(rows.transpose(0, 2, 1)).reshape(b * w, h)
    return np.ascontiguousarray(fwd1(tv, cols, fv).reshape(b, w, h).transpose(0, 2, 1))


def inv2(th, tv, y, fh=False, fv=False):
    b, h, w = y.shape
    cols = np.ascontiguousarray(y.transpose(0, 2, 1)).reshape(b * w, h)
    t = np.ascontiguousarray(inv1(tv, cols, fv).reshape(b, w, h).transpose(0, 2, 1))
    return inv1(th, t.reshape(b * h, w), fh).reshape(b, h, w)


rng = np.random.default_rng(20250529)

# ---- the seven primitives (reference kernels/_fastcore.pyx:188-307) ----------
for n in (4, 8, 16, 32, 64):
    x = rng.standard_normal((37, n))  # 37: not a multiple of the 32-vector tile
    out[f"prim/x/{n}"] = x
    for fn in ("dct2", "idct2", "dst3", "idst3"):
        out[f"prim/{fn}/{n}"] = getattr(kernels, fn)(x)
    for taps in (4, 6, 3):
        if taps > n:
            continue
        a = rng.standard_normal((n, n))  # entries outside the band are IGNORED by band()
        out[f"prim/band_a/{n}/{taps}"] = a
        out[f"prim/band/{n}/{taps}"] = kernels.band(a, taps, x)
    for b in (8, 5):
        if b > n:
            continue
        blk = rng.standard_normal((b, b))
        out[f"prim/sub_blk/{n}/{b}"] = blk
        out[f"prim/sub/{n}/{b}"] = kernels.subblock(blk, x)
    m = rng.standard_normal((n, n))
    out[f"prim/dense_m/{n}"] = m
    out[f"prim/dense/{n}"] = kernels.dense(m, x)
m = rng.standard_normal((16, 32))
out["prim/dense_rect_m"] = m
out["prim/dense_rect_x"] = out["prim/x/32"]
out["prim/dense_rect"] = kernels.dense(m, out["prim/x/32"])

# ---- 1-D adjusted transforms with the designed adjustments ------------------
ONE_D = ["band6_pre_dst3_dst7_n16", "band6_pre_dst3_dst7_n32", "band6_pre_dst3_dst7_n64",
         "band4_pre_dst3_dst7_n32", "sub8_post_dct2_dst7_n16", "sub8_post_dct2_dst7_n32",
         "sub8_post_dct2_dst7_n64", "sub8_post_dct2_dct8_n32"]
for name in ONE_D:
    t = make_adjusted_transform(design(name))
    x = rng.standard_normal((45, t.size)) * 20.0
    out[f"adj1d/{name}/x"] = x
    out[f"adj1d/{name}/fwd"] = forward_adjusted(t, x)
    out[f"adj1d/{name}/inv"] = inverse_adjusted(t, x)
    if "pre" in name:  # the D3 DCT-8 flip of the same design
        out[f"adj1d/{name}/fwd_flip"] = fwd1(t, x, True)
        out[f"adj1d/{name}/inv_flip"] = inv1(t, x, True)

# ---- 2-D config-shaped cases (small batches) --------------------------------
# C1: forward band6-pre DST-7, N=32, fp64 AR(1) rho=0.9 sigma=32
t = make_adjusted_transform(design("band6_pre_dst3_dst7_n32"))
x = ar1_blocks(rng, 6, 32, 32, 0.9, 32.0)
out["c1/x"] = x
out["c1/y"] = fwd2(t, t, x)

# C2: DCT-8 post round trip, N=32, integer residuals in [-512, 511] (stored fp32)
t8 = make_adjusted_transform(dct8_adjustment_from_dst7(design("sub8_post_dct2_dst7_n32")))
x = np.clip(np.rint(ar1_blocks(rng, 6, 32, 32, 0.85, 24.0)), -512, 511).astype(np.float32)
out["c2/x"] = x
out["c2/y"] = fwd2(t8, t8, x.astype(np.float64))
out["c2/xr"] = inv2(t8, t8, out["c2/y"])

# C4: N=64, {DST-7, DCT-8} x {band6 pre, sub8 post}, forward + inverse
t6 = make_adjusted_transform(design("band6_pre_dst3_dst7_n64"))
s7 = make_adjusted_transform(design("sub8_post_dct2_dst7_n64"))
s8 = make_adjusted_transform(dct8_adjustment_from_dst7(design("sub8_post_dct2_dst7_n64")))
x = ar1_blocks(rng, 3, 64, 64, 0.95, 40.0)
out["c4/x"] = x
for tag, (tt, flip) in {"dst7_pre": (t6, False), "dct8_pre": (t6, True),
                        "dst7_post": (s7, False), "dct8_post": (s8, False)}.items():
    out[f"c4/{tag}/y"] = fwd2(tt, tt, x, flip, flip)
    out[f"c4/{tag}/xr"] = inv2(tt, tt, x, flip, flip)  # inverse applied to x itself

# C3: mixed shapes (H x W in {16,32}^2), per-axis DST-7/DCT-8, pre and post
pre = {16: make_adjusted_transform(design("band6_pre_dst3_dst7_n16")),
       32: make_adjusted_transform(design("band6_pre_dst3_dst7_n32"))}
post7 = {n: make_adjusted_transform(design(f"sub8_post_dct2_dst7_n{n}")) for n in (16, 32)}
post8 = {n: make_adjusted_transform(dct8_adjustment_from_dst7(design(f"sub8_post_dct2_dst7_n{n}")))
         for n in (16, 32)}
for h, w in ((16, 16), (16, 32), (32, 16), (32, 32)):
    z = rng.laplace(0.0, 1.0 / np.sqrt(2.0), size=(4, h, w))
    lv = np.linalg.cholesky(0.9 ** np.abs(np.subtract.outer(np.arange(h), np.arange(h))).astype(float))
    lh = np.linalg.cholesky(0.9 ** np.abs(np.subtract.outer(np.arange(w), np.arange(w))).astype(float))
    x = (16.0 * np.sqrt(2.0) * lv @ z @ lh.T).astype(np.float32)
    out[f"c3/{h}x{w}/x"] = x
    for kh in ("dst7", "dct8"):
        for kv in ("dst7", "dct8"):
            xs = x.astype(np.float64)
            out[f"c3/{h}x{w}/pre/{kh}_{kv}/y"] = fwd2(pre[w], pre[h], xs, kh == "dct8", kv == "dct8")
            out[f"c3/{h}x{w}/pre/{kh}_{kv}/xr"] = inv2(pre[w], pre[h], xs, kh == "dct8", kv == "dct8")
            th = post7[w] if kh == "dst7" else post8[w]
            tv = post7[h] if kv == "dst7" else post8[h]
            out[f"c3/{h}x{w}/post/{kh}_{kv}/y"] = fwd2(th, tv, xs)
            out[f"c3/{h}x{w}/post/{kh}_{kv}/xr"] = inv2(th, tv, xs)

# C5: a small frame stack (height not a multiple of 32 -> zero pad), post sub8
# DST-7 forward + exact dense DST-7 forward, block-major raster order
frames = rng.standard_normal((2, 48, 96)).astype(np.float32) * 30.0
pad = np.zeros((2, 64, 96), dtype=np.float64)
pad[:, :48] = frames
blocks = pad.reshape(2, 2, 32, 3, 32).transpose(0, 1, 3, 2, 4).reshape(-1, 32, 32)
out["c5/frames"] = frames
out["c5/y"] = fwd2(post7[32], post7[32], np.ascontiguousarray(blocks))
t7 = build_transform(TransformKind.DST7, 32).entries
out["c5/y_exact"] = np.einsum("ij,bjk,lk->bil", t7, blocks, t7)

# simultaneous five-output encoder evaluation (pipeline.py:256-323)
from dctadjust.pipeline import EncoderContext, simultaneous_encoder_eval  # noqa: E402
KEYS = (("dct2", "dct2"), ("dst7", "dst7"), ("dct8", "dst7"), ("dst7", "dct8"), ("dct8", "dct8"))
for tag, (hn, vn) in {"32x32": (32, 32), "32x64": (64, 32), "16x16": (16, 16)}.items():
    ctx = EncoderContext(horizontal=design(f"sub8_post_dct2_dst7_n{hn}"),
                         vertical=design(f"sub8_post_dct2_dst7_n{vn}"))
    blocks = rng.standard_normal((3, vn, hn)) * 16.0
    out[f"enc5/{tag}/x"] = blocks
    res = [simultaneous_encoder_eval(b, ctx) for b in blocks]
    for k in KEYS:
        out[f"enc5/{tag}/{k[0]}_{k[1]}"] = np.stack([r[k] for r in res])

np.savez_compressed(HERE / "golden.npz", **out)
print(f"wrote {len(out)} arrays, {(HERE / 'golden.npz').stat().st_size / 1e6:.2f} MB")
