"""The paper's Table 1 on the GPU: throughput ratios of the adjusted pipelines
against the full-matrix (dense) transform.

Methodology of the reference harness (reference benchmark.py:1-13, 130-260),
kept: every pipeline is checked against its dense oracle before it is timed,
inputs are shared across pipelines, each configuration is timed over >= 30
samples (median throughput, dispersion = IQR / median), and the ratio is the
pipeline's median throughput over the dense baseline's for the same size and
direction; "multiple" is the simultaneous five-output encoder evaluation
against five independent dense separable transforms.  Differences: samples are
CUDA-event timings of one batched launch on device-resident data, and besides
the reference's 1-D batches the 2-D block transforms are measured too.
"""
from __future__ import annotations

import contextlib
import os
from dataclasses import dataclass

import numpy as np

from . import kernels, pipeline
from .design import (AdjustmentMatrix, Side, SparsityPattern, givens_to_matrix,
                     pattern_schedule_template)
from .errors import ConfigurationError
from .transforms import TransformKind, build_transform

DEFAULT_PIPELINES = ("band4", "band6", "subblock8", "multiple")


@dataclass(frozen=True)
class BenchReport:
    pipeline: str
    size: int
    direction: str
    coefficients_per_second: float
    ratio_vs_dense: float
    samples: int
    dispersion: float
    layout: str = "1d"

    def __post_init__(self):
        if self.samples < 30:
            raise ConfigurationError("need at least 30 samples per measurement")


def _random_pattern_adjustment(pattern, side, base, seed) -> AdjustmentMatrix:
    """Valid random-angle adjustment (reference benchmark.py:58-73): speed does
    not depend on the designed values."""
    template = pattern_schedule_template(pattern)
    rng = np.random.default_rng([seed, pattern.size, template.n_rotations])
    sched = template.with_angles(rng.uniform(-0.3, 0.3, template.n_rotations))
    return AdjustmentMatrix(pattern=pattern, side=side, base=base, target=TransformKind.DST7,
                            schedule=sched, realized=givens_to_matrix(sched))


def _dense_transform(h: np.ndarray):
    """An AdjustedTransform whose whole axis is the dense matrix h (post side on
    a DCT-2 base, C = h DCT2^T): the full-matrix baseline as one fused kernel."""
    n = h.shape[0]
    c = h @ build_transform(TransformKind.DCT2, n).entries.T
    rec = AdjustmentMatrix(SparsityPattern.dense(n), Side.POST, TransformKind.DCT2,
                           TransformKind.DST7, pattern_schedule_template(SparsityPattern.dense(n)), c)
    return pipeline.make_adjusted_transform(rec)


@contextlib.contextmanager
def dense_on_cuda_cores():
    """Route dense 2-D transforms to the CUDA-core FMA kernel (DCTADJ_DENSE_TC=0,
    read by the library per call) -- the reference's full-matrix product."""
    old = os.environ.get("DCTADJ_DENSE_TC")
    os.environ["DCTADJ_DENSE_TC"] = "0"
    try:
        yield
    finally:
        if old is None:
            del os.environ["DCTADJ_DENSE_TC"]
        else:
            os.environ["DCTADJ_DENSE_TC"] = old


def _measure(fn, samples: int, warmup: int):
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    times = np.empty(samples)
    for i in range(samples):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # keep the device busy (~1 ms) while the host enqueues the call, so the
        # events bracket the kernels rather than the Python / ctypes overhead
        torch.cuda._sleep(2_000_000)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        times[i] = e0.elapsed_time(e1) / 1e3
    return times


def _stats(times, coeffs):
    thr = coeffs / times
    med = float(np.median(thr))
    q25, q75 = np.percentile(thr, [25, 75])
    return med, float((q75 - q25) / med)


def run_benchmark(pipelines=DEFAULT_PIPELINES, sizes=(32, 64), samples: int = 31,
                  warmup: int = 3, seed: int = 0, vectors: int = 1 << 22, blocks: int = 1 << 16,
                  dtype: str = "float32") -> list[BenchReport]:
    import torch
    tdt = getattr(torch, dtype)
    reports: list[BenchReport] = []
    g = torch.Generator(device="cuda").manual_seed(seed)
    for size in sizes:
        adj = {
            "band4": _random_pattern_adjustment(SparsityPattern.band(4, size), Side.PRE,
                                                TransformKind.DST3, seed),
            "band6": _random_pattern_adjustment(SparsityPattern.band(6, size), Side.PRE,
                                                TransformKind.DST3, seed),
            "subblock8": _random_pattern_adjustment(SparsityPattern.subblock(8, size), Side.POST,
                                                    TransformKind.DCT2, seed),
        }
        h_ref = pipeline.dense_matrix(pipeline.make_adjusted_transform(adj["subblock8"]))
        td = _dense_transform(h_ref)
        x1 = torch.randn(vectors, size, device="cuda", generator=g, dtype=tdt)
        nb = max(1, blocks * 1024 // (size * size))
        x2 = torch.randn(nb, size, size, device="cuda", generator=g, dtype=tdt)
        tol = 1e-5 if dtype == "float32" else 1e-9

        for layout, x, coeffs in (("1d", x1, x1.numel()), ("2d", x2, x2.numel())):
            if layout == "1d":
                dfwd = lambda: kernels.dense(h_ref, x)        # noqa: E731
                dinv = lambda: kernels.dense(h_ref.T, x)      # noqa: E731
            else:
                dfwd = lambda: pipeline.forward_adjusted_2d(td, td, x)   # noqa: E731
                dinv = lambda: pipeline.inverse_adjusted_2d(td, td, x)   # noqa: E731
            dense_med = {}
            for direction, fn in (("forward", dfwd), ("inverse", dinv)):
                # the paper's full-matrix baseline: the FMA matrix product (CUDA cores)
                with dense_on_cuda_cores():
                    med, disp = _stats(_measure(fn, samples, warmup), coeffs)
                dense_med[direction] = med
                reports.append(BenchReport("dense", size, direction, med, 1.0, samples, disp, layout))
                if layout == "2d" and dtype == "float32":
                    # the same product on the tensor cores (3xTF32 tcgen05, dense_tc.cuh)
                    med, disp = _stats(_measure(fn, samples, warmup), coeffs)
                    reports.append(BenchReport("dense_tc", size, direction, med,
                                               med / dense_med[direction], samples, disp, layout))
            for name in pipelines:
                if name == "multiple":
                    continue
                t = pipeline.make_adjusted_transform(adj[name])
                h = pipeline.dense_matrix(t)
                if layout == "1d":
                    fwd = lambda t=t: pipeline.forward_adjusted(t, x)   # noqa: E731
                    inv = lambda t=t: pipeline.inverse_adjusted(t, x)   # noqa: E731
                    probe = x[:64].double().cpu().numpy()
                    oracles = {"forward": probe @ h.T, "inverse": probe @ h}
                    got = {"forward": fwd()[:64], "inverse": inv()[:64]}
                else:
                    fwd = lambda t=t: pipeline.forward_adjusted_2d(t, t, x)  # noqa: E731
                    inv = lambda t=t: pipeline.inverse_adjusted_2d(t, t, x)  # noqa: E731
                    probe = x[:16].double().cpu().numpy()
                    oracles = {"forward": h @ probe @ h.T, "inverse": h.T @ probe @ h}
                    got = {"forward": fwd()[:16], "inverse": inv()[:16]}
                for direction, fn in (("forward", fwd), ("inverse", inv)):
                    o = oracles[direction]
                    err = np.abs(got[direction].double().cpu().numpy() - o).max() / np.abs(o).max()
                    if err >= tol:
                        raise AssertionError(f"{name} {layout} {direction} failed its oracle "
                                             f"check ({err:.2e}); not timing it")
                    med, disp = _stats(_measure(fn, samples, warmup), coeffs)
                    reports.append(BenchReport(name, size, direction, med,
                                               med / dense_med[direction], samples, disp, layout))
        if "multiple" in pipelines:
            reports.extend(_bench_multiple(adj["subblock8"], x2, samples, warmup, tol))
    return reports


def _bench_multiple(sub_adj, blocks, samples, warmup, tol) -> BenchReport:
    """Shared five-output encoder evaluation vs five independent dense
    separable 2-D transforms (reference benchmark.py:206-238)."""
    import torch
    ctx = pipeline.EncoderContext(horizontal=sub_adj, vertical=sub_adj)
    shared = pipeline.simultaneous_encoder_eval(blocks[:8], ctx)
    naive = pipeline.naive_encoder_eval(blocks[:8], ctx)
    for key in naive:
        a, b = shared[key].double(), naive[key].double()
        if float((a - b).abs().max() / b.abs().max()) >= tol:
            raise AssertionError("shared encoder path failed its oracle check")
    coeffs = 5 * blocks.numel()
    t_s = _measure(lambda: pipeline.simultaneous_encoder_eval(blocks, ctx), samples, warmup)
    with dense_on_cuda_cores():
        t_n = _measure(lambda: pipeline.naive_encoder_eval(blocks, ctx), samples, warmup)
    med_s, disp = _stats(t_s, coeffs)
    med_n, _ = _stats(t_n, coeffs)
    out = [BenchReport("multiple", sub_adj.pattern.size, "forward", med_s, med_s / med_n,
                       samples, disp, "2d")]
    if sub_adj.pattern.size == 32 and blocks.dtype == torch.float32:
        # the naive side's five dense transforms on the tensor cores instead
        med_t, _ = _stats(_measure(lambda: pipeline.naive_encoder_eval(blocks, ctx), samples,
                                   warmup), coeffs)
        out.append(BenchReport("multiple_vs_tc", sub_adj.pattern.size, "forward", med_s,
                               med_s / med_t, samples, disp, "2d"))
    return out


def report_table(reports: list[BenchReport], layout: str | None = None) -> str:
    """Ratio table in the paper's layout: pipeline x (direction, size)."""
    reps = [r for r in reports if layout is None or r.layout == layout]
    sizes = sorted({r.size for r in reps})
    names = []
    for r in reps:
        if r.pipeline not in names:
            names.append(r.pipeline)
    head = ["pipeline"] + [f"{d}/{s}" for d in ("forward", "inverse") for s in sizes]
    lines = ["| " + " | ".join(head) + " |", "|" + "---|" * len(head)]
    for name in names:
        row = [name]
        for d in ("forward", "inverse"):
            for s in sizes:
                hit = [r for r in reps if r.pipeline == name and r.direction == d and r.size == s]
                row.append(f"{hit[0].ratio_vs_dense:.2f}" if hit else "-")
        lines.append("| " + " | ".join(row) + " |")
    return "\n".join(lines)
