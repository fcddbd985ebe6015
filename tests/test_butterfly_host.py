"""CPU unit tests of the DEVICE butterflies (csrc/butterfly.cuh) and of the host
packing that goes with them (csrc/givens_pack.h), compiled for the host through
tests/butterfly_host.cpp: the scaled rotations of the inverse direction, the
deferred-scale forward DCT-2 (dct2d) and the rule that lets a trailing Givens
stage absorb its scales -- against the C oracle (reference _fastcore.pyx:50-307,
pipeline.py:158-199).  No GPU needed; the same templates are what nvcc compiles
into the kernels."""
import ctypes
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O
from paper_2505_23618_b200 import matio
from paper_2505_23618_b200.design import flip_pre_adjustment
from paper_2505_23618_b200.pipeline import brickwall_angles

HERE = Path(__file__).resolve().parent
ST_NONE, ST_DCT2, ST_IDCT2, ST_DST3, ST_IDST3, ST_GIVENS2 = 0, 1, 2, 3, 4, 9
P = ctypes.POINTER(ctypes.c_double)


@pytest.fixture(scope="module")
def bf(tmp_path_factory):
    so = tmp_path_factory.mktemp("bf") / "bf_host.so"
    subprocess.run(["g++", "-std=c++17", "-O1", "-shared", "-fPIC", "-o", str(so),
                    str(HERE / "butterfly_host.cpp")], check=True)
    lib = ctypes.CDLL(str(so))
    lib.bf_apply.argtypes = [ctypes.c_int] * 5 + [P, P, P]
    lib.bf_pack_givens2.argtypes = [ctypes.c_int, ctypes.c_int, P, ctypes.c_int, ctypes.c_double,
                                    ctypes.c_int, P, ctypes.c_int]
    lib.bf_deferred_scale.restype = ctypes.c_double
    lib.bf_deferred_scale.argtypes = [ctypes.c_int] * 3
    lib.bf_dct2d.argtypes = [ctypes.c_int, ctypes.c_int, P, P, P]
    lib.bf_idct2.argtypes = [ctypes.c_int, ctypes.c_int, P, P]
    lib.bf_fold_sub.argtypes = [ctypes.c_int, ctypes.c_int, P]
    lib.bf_fold_sub.restype = None
    return lib


def _p(a):
    return a.ctypes.data_as(P)


def apply(lib, n, s1, s2, k, vtype, coef, x):
    coef = np.ascontiguousarray(coef if coef is not None else np.zeros(1), dtype=np.float64)
    out = np.empty((len(x), n))
    for i, row in enumerate(np.ascontiguousarray(x, dtype=np.float64)):
        assert lib.bf_apply(n, s1, s2, k, vtype, _p(coef), _p(row), _p(out[i])) == 0
    return out


def rel(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


TOL = {0: 2e-6, 1: 1e-13, 2: 2e-6}  # float, double, packed f2


@pytest.mark.parametrize("n", [4, 8, 16, 32, 64])
@pytest.mark.parametrize("vtype", [0, 1, 2])
def test_base_stages_match_oracle(bf, n, vtype):
    """dct2 / idct2 / dst3 / idst3 (unnormalized: gain sqrt(n)) against the oracle."""
    x = np.random.default_rng(n).standard_normal((5, n)) * 30
    g = np.sqrt(n)
    for st, ref in ((ST_DCT2, O.dct2), (ST_IDCT2, O.idct2), (ST_DST3, O.dst3), (ST_IDST3, O.idst3)):
        assert rel(apply(bf, n, st, ST_NONE, 0, vtype, None, x) / g, ref(x)) < TOL[vtype]


@pytest.mark.parametrize("n", [2, 4, 8, 16, 32, 64])
def test_deferred_dct2_scales(bf, n):
    """dct2d: held[k] * scale[k] is the unnormalized DCT-2 (of the sign-alternated
    input for the idst3 form); every scale is a finite non-zero constant."""
    x = np.random.default_rng(n).standard_normal(n) * 30
    for alt in (0, 1):
        held, scale = np.empty(n), np.empty(n)
        assert bf.bf_dct2d(n, alt, _p(x), _p(held), _p(scale)) == 0
        assert np.isfinite(scale).all() and (np.abs(scale) > 0.05).all() and (np.abs(scale) < 3).all()
        xin = x * np.where(np.arange(n) % 2, -1.0, 1.0) if alt else x
        want = O.dct2(xin[None])[0] * np.sqrt(n) if n >= 4 else None
        if n == 2:
            want = np.array([xin[0] + xin[1], xin[0] - xin[1]])
        assert rel(held * scale, want) < 1e-13


@pytest.mark.parametrize("n", [4, 8, 16, 32, 64])
def test_both_inverse_forms(bf, n):
    """idct2s (scaled rotations) and idct2p (plain) are the same transform, whatever
    form the (type, size) policy gives the kernels."""
    y = np.random.default_rng(n).standard_normal(n) * 30
    want = O.idct2(y[None])[0] * np.sqrt(n)
    for scaled in (0, 1):
        x = np.empty(n)
        assert bf.bf_idct2(n, scaled, _p(y), _p(x)) == 0
        assert rel(x, want) < 1e-13


def test_policy_is_type_and_size_only(bf):
    """fp32 up to 32 points runs the scaled / deferred forms; fp64 and 64 points the plain
    ones (measured, profiles/r02_tuning.md)."""
    for n in (4, 8, 16, 32, 64):
        assert bf.bf_deferred_policy(0, n) == bf.bf_idct_scaled_policy(0, n) == int(n <= 32)
        assert bf.bf_deferred_policy(1, n) == bf.bf_idct_scaled_policy(1, n) == 0


def _before(lib, vtype, n, base):
    """base_before of abi.cu's plan_axis: the deferred base only where the kernel runs it."""
    return base if lib.bf_deferred_policy(int(vtype == 1), n) else ST_NONE


def _pack(lib, n, k, ang, inverse, gain, base_before):
    out = np.empty(2 * len(ang) + n)
    cnt = lib.bf_pack_givens2(n, k, _p(np.ascontiguousarray(ang)), int(inverse), gain, base_before,
                              _p(out), len(out))
    assert cnt == len(out)
    return out


def _oaxis(adj):
    base = {"dct2": O.BASE_DCT2, "dst3": O.BASE_DST3, "dct3": O.BASE_DCT3}[adj.base.value]
    return O.OAxis(adj.pattern.size, base, O.ADJ_BAND, O.SIDE_PRE, adj.pattern.taps, 0,
                   np.array(adj.realized))


@pytest.mark.parametrize("name", ["band6_pre_dst3_dst7_n16", "band6_pre_dst3_dst7_n32",
                                  "band6_pre_dst3_dst7_n64", "band4_pre_dst3_dst7_n32"])
@pytest.mark.parametrize("vtype", [0, 1, 2])
def test_pre_adjusted_axis_with_deferred_base(bf, name, vtype):
    """Forward (Givens -> DST-3) and inverse (deferred IDST-3 -> Givens^T whose input
    scales absorb the deferral, gain folded) of the shipped band pre-adjustments
    against the oracle's forward_adjusted / inverse_adjusted."""
    adj = matio.load_designed(name)
    n, k = adj.pattern.size, adj.pattern.taps
    ang = brickwall_angles(adj)
    ax = _oaxis(adj)
    x = np.random.default_rng(1).standard_normal((4, n)) * 30
    fwd = apply(bf, n, ST_GIVENS2, ST_DST3, k, vtype, _pack(bf, n, k, ang, False, 1.0, ST_NONE), x)
    want = O.adjusted_1d(ax, x)
    assert rel(fwd / np.sqrt(n), want) < TOL[vtype]
    coef = _pack(bf, n, k, ang, True, 1.0 / np.sqrt(n), _before(bf, vtype, n, ST_IDST3))
    inv = apply(bf, n, ST_IDST3, ST_GIVENS2, k, vtype, coef, want)
    assert rel(inv, O.adjusted_1d(ax, want, inverse=True)) < TOL[vtype]
    assert rel(inv, x) < 5 * TOL[vtype]


@pytest.mark.parametrize("vtype", [0, 1, 2])
def test_flipped_dct8_pre_axis_with_deferred_base(bf, vtype):
    """The DCT-8 flip (base DCT-3): forward Givens -> idct2, inverse deferred dct2 -> Givens^T."""
    adj = flip_pre_adjustment(matio.load_designed("band6_pre_dst3_dst7_n32"))
    n, k = 32, 6
    ang = brickwall_angles(adj)
    assert ang is not None
    ax = _oaxis(adj)
    x = np.random.default_rng(2).standard_normal((4, n)) * 30
    want = O.adjusted_1d(ax, x)
    # run_n in the harness instantiates (GIVENS2, IDCT2) / (DCT2, GIVENS2) for k = 6
    fwd = apply(bf, n, ST_GIVENS2, ST_IDCT2, k, vtype, _pack(bf, n, k, ang, False, 1.0, ST_NONE), x)
    assert rel(fwd / np.sqrt(n), want) < TOL[vtype]
    coef = _pack(bf, n, k, ang, True, 1.0 / np.sqrt(n), _before(bf, vtype, n, ST_DCT2))
    inv = apply(bf, n, ST_DCT2, ST_GIVENS2, k, vtype, coef, want)
    assert rel(inv, x) < 5 * TOL[vtype]


@pytest.mark.parametrize("n", [8, 16, 32, 64])
@pytest.mark.parametrize("vtype", [0, 1, 2])
def test_post_adjusted_axis_with_deferred_base(bf, n, vtype):
    """Forward post (deferred DCT-2 -> 8x8 block with the held inputs' scales folded into its
    columns, tail finalized) and inverse post (block^T -> scaled inverse DCT-2) against the
    oracle; the untouched tail equals the kernel's own plain DCT-2 output bit for bit, and an
    identity block reproduces the plain DCT-2 everywhere (the kernels' invariants)."""
    ST_SUB = 6
    name = f"sub8_post_dct2_dst7_n{max(n, 16)}"
    blk = np.ascontiguousarray(np.array(matio.load_designed(name).realized)[:8, :8])
    x = np.random.default_rng(3).standard_normal((4, n)) * 30
    plain = apply(bf, n, ST_DCT2, ST_NONE, 0, vtype, None, x)

    def fwd(block):
        c = np.ascontiguousarray(block, dtype=np.float64).copy()
        if bf.bf_deferred_policy(int(vtype == 1), n):
            bf.bf_fold_sub(n, 8, _p(c))
        return apply(bf, n, ST_DCT2, ST_SUB, 8, vtype, c.ravel(), x)

    y = fwd(blk)
    want = O.dct2(x)
    want[:, :8] = want[:, :8] @ blk.T
    assert rel(y / np.sqrt(n), want) < TOL[vtype]
    assert np.array_equal(y[:, 8:], plain[:, 8:])
    assert np.array_equal(fwd(np.eye(8)), plain)
    inv = apply(bf, n, ST_SUB, ST_IDCT2, 8, vtype, np.ascontiguousarray(blk.T).ravel(), want)
    assert rel(inv / np.sqrt(n), x) < 5 * TOL[vtype]


def _gain(n):
    """tile_kernel.cuh inv_sqrt_pow2(n): 1 / sqrt(n) as the kernels apply it."""
    e = int(np.log2(n))
    return 0.5 ** (e // 2) * (0.7071067811865476 if e % 2 else 1.0)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [8, 16, 32, 64])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_device_primitives_match_host_shim(bf, n, dtype):
    """The B200 kernels and the host shim compile the SAME butterfly templates; the only
    difference is nvcc contracting a multiply into a following add (-fmad) where g++ keeps two
    roundings, so the four base primitives on the GPU equal the host-compiled templates to a
    rounding or two -- far inside the parity bar -- which is what makes the CPU tests above
    tests of the device arithmetic.  (The forward DCT-2 has no such pair: bit-identical.)"""
    import torch
    from paper_2505_23618_b200 import kernels
    x = (np.random.default_rng(n).standard_normal((37, n)) * 30).astype(dtype)
    vtype = 0 if dtype == np.float32 else 1
    tol = 3e-7 if dtype == np.float32 else 1e-15
    xd = torch.from_numpy(x).cuda()
    for name, st in (("dct2", ST_DCT2), ("idct2", ST_IDCT2), ("dst3", ST_DST3), ("idst3", ST_IDST3)):
        got = getattr(kernels, name)(xd).cpu().numpy()
        held = apply(bf, n, st, ST_NONE, 0, vtype, None, x.astype(np.float64)).astype(dtype)
        want = held * dtype(_gain(n))
        assert got.dtype == dtype
        assert rel(got.astype(np.float64), want.astype(np.float64)) < tol, (name, n, dtype)
