"""The Table-1 ratio harness port (paper_2505_23618_b200/benchmark.py), mirroring
the reference's own harness tests (reference tests/test_benchmark.py:1-40):
report structure, dense self-ratio exactly 1.0, "multiple" faster than five
dense transforms, the 30-sample floor, the rendered table -- plus the refusal
to time a pipeline that fails its oracle (reference benchmark.py:181-190)."""
import pytest

from paper_2505_23618_b200.benchmark import BenchReport, report_table
from paper_2505_23618_b200.errors import ConfigurationError

FAST = dict(sizes=(32,), samples=30, warmup=1, vectors=1 << 14, blocks=1 << 10)


def test_sample_floor_enforced():
    with pytest.raises(ConfigurationError):
        BenchReport("dense", 32, "forward", 1.0, 1.0, samples=5, dispersion=0.0)


def test_report_table_renders_paper_layout():
    reps = [BenchReport("dense", 32, d, 1e9, 1.0, 30, 0.0) for d in ("forward", "inverse")]
    reps += [BenchReport("band6", 32, "forward", 2e9, 2.0, 30, 0.01),
             BenchReport("band6", 64, "inverse", 3e9, 3.0, 30, 0.01, "2d")]
    table = report_table(reps)
    assert "band6" in table and "forward/32" in table and "inverse/64" in table
    assert "| band6 | 2.00 | - | - | 3.00 |" in table
    assert "inverse/64" not in report_table(reps, layout="1d")


@pytest.mark.gpu
def test_reports_structure():
    from paper_2505_23618_b200.benchmark import run_benchmark
    reports = run_benchmark(pipelines=("band6", "subblock8"), **FAST)
    keys = {(r.pipeline, r.size, r.direction, r.layout) for r in reports}
    for layout in ("1d", "2d"):
        assert ("dense", 32, "forward", layout) in keys
        assert ("dense", 32, "inverse", layout) in keys
        assert ("band6", 32, "forward", layout) in keys
        assert ("subblock8", 32, "inverse", layout) in keys
    assert ("dense_tc", 32, "forward", "2d") in keys
    for r in reports:
        assert r.samples >= 30
        assert r.coefficients_per_second > 0
        assert r.dispersion == r.dispersion  # finite, not NaN


@pytest.mark.gpu
def test_dense_self_ratio_is_one():
    from paper_2505_23618_b200.benchmark import run_benchmark
    reports = run_benchmark(pipelines=(), **FAST)
    dense = [r for r in reports if r.pipeline == "dense"]
    assert len(dense) == 4  # forward / inverse x 1-D / 2-D
    assert all(r.ratio_vs_dense == 1.0 for r in dense)


@pytest.mark.gpu
def test_multiple_pipeline_reports():
    from paper_2505_23618_b200.benchmark import run_benchmark
    reports = run_benchmark(pipelines=("multiple",), **FAST)
    multi = [r for r in reports if r.pipeline == "multiple"]
    assert len(multi) == 1
    assert multi[0].ratio_vs_dense > 1.0


@pytest.mark.gpu
def test_refuses_to_time_a_pipeline_that_fails_its_oracle(monkeypatch):
    from paper_2505_23618_b200 import benchmark, pipeline
    real = pipeline.forward_adjusted
    monkeypatch.setattr(pipeline, "forward_adjusted", lambda t, x: real(t, x) * 1.001)
    with pytest.raises(AssertionError, match="failed its oracle"):
        benchmark.run_benchmark(pipelines=("subblock8",), **FAST)
