"""Full BASELINE.json sizes, checked through size-independent properties (the
oracle is too slow at these sizes): exact-orthogonality round trips, energy
preservation, linearity, and a seeded sample of blocks against the oracle.
The workloads are bench.py's own (same inputs as the measured runs)."""
import sys
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

pytestmark = pytest.mark.gpu
TOL = 1e-5


def _energy(t):
    return float((t.double() ** 2).sum())


@pytest.mark.parametrize("cfg", ["c4_dst7_pre", "c4_dct8_pre", "c4_dst7_post", "c4_dct8_post"])
def test_c4_full_size_round_trip(cfg):
    import bench
    w = bench.Uniform(cfg, 0)  # 262,144 x 64x64 fp32 (4.3 GB)
    for _, fn in w.launches:
        fn()
    torch.cuda.synchronize()
    err = (w.xr - w.x).abs().max().item() / w.x.abs().max().item()
    assert err < TOL
    assert abs(_energy(w.y) / _energy(w.x) - 1) < TOL
    assert w.gate() < TOL  # 256 evenly spaced blocks against the oracle
    # linearity: T(2x) == 2 T(x) exactly in binary floating point
    from paper_2505_23618_b200 import pipeline
    x2 = w.x[:4096] * 2
    assert torch.equal(pipeline.forward_adjusted_2d(w.t, w.t, x2), 2 * w.y[:4096])


@pytest.mark.parametrize("side", ["pre", "post"])
def test_c3_full_size_round_trip(side):
    import bench
    w = bench.Mixed(side, 0)  # 1,048,576 mixed-shape blocks
    for _, fn in w.launches:
        fn()
    torch.cuda.synchronize()
    err = (w.xr - w.x).abs().max().item() / w.x.abs().max().item()
    assert err < TOL
    assert abs(_energy(w.y) / _energy(w.x) - 1) < TOL
    assert w.gate() < TOL


def test_c5_full_size_frames():
    import bench
    w = bench.Frames(0, 1)  # 64 frames 3840x2160
    for _, fn in w.launches:
        fn()
    torch.cuda.synchronize()
    err = (w.back - w.frames).abs().max().item() / w.frames.abs().max().item()
    assert err < TOL
    assert w.gate() < TOL
    # the fused launch's error sums agree with a reduction over its own outputs
    e = np.array(w.approximation_error())
    assert 0.05 < e[0] / e[1] < 0.09  # ~7 % of the energy (config 5)
    # energy: padded tile rows are zero, so the adjusted coefficients carry the frames' energy
    assert abs(_energy(w.y) / _energy(w.frames) - 1) < TOL


def test_c2_full_size_fused_round_trip():
    """The bench step itself (65,536 x 32x32 fp32 integer residuals, one fused
    round-trip kernel): x' recovers x exactly after rounding (D7 iii), and the
    coefficients / reconstruction equal the two-kernel schedule bit for bit."""
    import bench
    w = bench.Uniform("c2", 0, fused_roundtrip=True)
    assert [n for n, _ in w.launches] == ["roundtrip_2d"]
    for _, fn in w.launches:
        fn()
    torch.cuda.synchronize()
    y, xr = w.y.clone(), w.xr.clone()
    assert torch.equal(torch.round(xr), w.x)
    assert abs(_energy(y) / _energy(w.x) - 1) < TOL
    for _, fn in w.two_kernel:
        fn()
    torch.cuda.synchronize()
    assert torch.equal(y, w.y) and torch.equal(xr, w.xr)
    assert w.gate() < TOL


@pytest.mark.parametrize("side", ["pre", "post"])
def test_c3_full_size_fused_round_trip(side):
    import bench
    w = bench.Mixed(side, 0, fused_roundtrip=True)  # 1,048,576 blocks, one kernel per class
    assert [n for n, _ in w.launches] == ["mixed_roundtrip"]
    for _, fn in w.launches:
        fn()
    torch.cuda.synchronize()
    y, xr = w.y.clone(), w.xr.clone()
    err = (xr - w.x).abs().max().item() / w.x.abs().max().item()
    assert err < TOL
    for _, fn in w.two_kernel:
        fn()
    torch.cuda.synchronize()
    assert torch.equal(y, w.y) and torch.equal(xr, w.xr)
