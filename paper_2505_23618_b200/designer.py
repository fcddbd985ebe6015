"""The adjustment designer on the GPU.

`optimize_adjustment` keeps the reference's signature and semantics
(reference design.py:560-613): a zero-angle start plus `config.restarts`
seeded random restarts of the cyclic coordinate descent over the angles of the
pattern's rotation skeleton, merged by lowest objective (then lowest restart
index), with the identity adjustment as a candidate.  The descent itself
(reference design.py:377-543) runs in `dctadj_design_cd` (csrc/designer.cu),
all restarts at once, one CTA each; this module only prepares the inputs and
rebuilds the record in numpy exactly as the reference does.  There is no CPU
fallback: without the CUDA library every call raises.

Also mirrored (host arithmetic the designer and its callers use):
  DesignConfig                         reference design.py:273-295
  default_alpha / frequency_weights    reference design.py:253-259
  weighted_error                       reference design.py:262-270
  restart_angles                       reference design.py:546-550
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _device, _lib
from .design import (AdjustmentMatrix, GivensSchedule, Side, SparsityPattern,
                     givens_to_matrix, pattern_schedule_template)
from .errors import ShapeError
from .transforms import TransformMatrix


@dataclass(frozen=True)
class DesignConfig:
    """Optimizer knobs.  alpha=None means ln(100)/N resolved at run time."""

    alpha: float | None = None
    max_iterations: int = 2000
    tolerance: float = 1e-10
    restarts: int = 4
    rng_seed: int = 0
    sparsity_epsilon: float = 0.05

    def __post_init__(self):
        if self.alpha is not None and self.alpha <= 0:
            raise ValueError(f"alpha must be positive, got {self.alpha}")
        if self.tolerance <= 0:
            raise ValueError(f"tolerance must be positive, got {self.tolerance}")
        if self.max_iterations < 1:
            raise ValueError("max_iterations must be >= 1")
        if self.restarts < 0:
            raise ValueError("restarts must be >= 0")

    def resolve_alpha(self, size: int) -> float:
        return self.alpha if self.alpha is not None else default_alpha(size)


def default_alpha(size: int) -> float:
    """The frequency-weight decay rate ln(10^2)/N."""
    return math.log(100.0) / size


def frequency_weights(size: int, alpha: float) -> np.ndarray:
    return np.exp(-alpha * np.arange(size))


def weighted_error(h: np.ndarray, d: np.ndarray, alpha: float) -> float:
    """sum_ij exp(-alpha*i) * (H[i,j] - D[i,j])^2 with i the frequency row index."""
    h = np.asarray(h, dtype=float)
    d = np.asarray(d, dtype=float)
    if h.shape != d.shape or h.ndim != 2:
        raise ShapeError(f"mismatched shapes {h.shape} vs {d.shape}")
    diff = h - d
    return float(np.einsum("i,ij,ij->", frequency_weights(h.shape[0], alpha), diff, diff))


def restart_angles(m: int, seed: int, restart: int) -> np.ndarray:
    """Start angles of restart `restart`: zeros, then uniform(-0.3, 0.3) draws."""
    if restart == 0:
        return np.zeros(m)
    rng = np.random.default_rng([seed & 0xFFFFFFFFFFFFFFFF, restart])
    return rng.uniform(-0.3, 0.3, size=m)


@dataclass(frozen=True)
class DescentRun:
    """One restart's coordinate-descent result (the reference's run() tuple)."""

    theta: np.ndarray
    trace: tuple[float, ...]
    converged: bool


def coordinate_descent(base: np.ndarray, desired: np.ndarray, template: GivensSchedule,
                       side: Side, alpha: float, starts: np.ndarray, max_sweeps: int,
                       tol: float) -> list[DescentRun]:
    """Run the cyclic coordinate descent from every row of `starts` (restarts x
    m angles) on the GPU; one DescentRun per start."""
    n = base.shape[0]
    rots = template.rotations()
    m = len(rots)
    starts = np.ascontiguousarray(np.atleast_2d(starts), dtype=np.float64)
    if m and starts.shape[1] != m:
        raise ShapeError(f"expected {m} start angles per restart, got {starts.shape[1]}")
    nr = starts.shape[0]
    b = np.ascontiguousarray(base, dtype=np.float64)
    d = np.ascontiguousarray(desired, dtype=np.float64)
    w = np.ascontiguousarray(frequency_weights(n, alpha))
    rp = np.ascontiguousarray([r.i for r in rots], dtype=np.int32)
    rq = np.ascontiguousarray([r.j for r in rots], dtype=np.int32)
    theta = np.zeros((nr, max(m, 1)))
    trace = np.zeros((nr, max_sweeps + 1))
    sweeps = np.zeros(nr, np.int32)
    conv = np.zeros(nr, np.int32)
    _device.require_cuda()
    ptr = lambda a: a.ctypes.data if a.size else None  # noqa: E731
    _lib.call("dctadj_design_cd", n, b.ctypes.data, d.ctypes.data, w.ctypes.data,
              0 if side is Side.PRE else 1, m, ptr(rp), ptr(rq), nr, ptr(starts), max_sweeps,
              float(tol), theta.ctypes.data, trace.ctypes.data, sweeps.ctypes.data,
              conv.ctypes.data, _device.torch.cuda.current_device())
    return [DescentRun(theta[r, :m].copy(), tuple(float(v) for v in trace[r, :sweeps[r] + 1]),
                       bool(conv[r])) for r in range(nr)]


def _realize(template: GivensSchedule, theta: np.ndarray) -> np.ndarray:
    return givens_to_matrix(template.with_angles(theta))


def optimize_adjustment(b: TransformMatrix, d: TransformMatrix, pattern: SparsityPattern,
                        side: Side, config: DesignConfig = DesignConfig()) -> AdjustmentMatrix:
    """Minimize the weighted error of H = B*A (pre) or A*B (post) over the
    orthogonal matrices conforming to `pattern` (reference design.py:560-613);
    every restart of the coordinate descent runs concurrently on the GPU."""
    if b.size != d.size:
        raise ShapeError(f"base size {b.size} != desired size {d.size}")
    if pattern.size != b.size:
        raise ShapeError(f"pattern size {pattern.size} != transform size {b.size}")
    alpha = config.resolve_alpha(b.size)
    template = pattern_schedule_template(pattern)
    identity_obj = weighted_error(b.entries, d.entries, alpha)
    m = template.n_rotations
    starts = np.stack([restart_angles(m, config.rng_seed, r) for r in range(config.restarts + 1)])
    runs = coordinate_descent(b.entries, d.entries, template, side, alpha, starts,
                              config.max_iterations, config.tolerance)

    def compose(a):
        return b.entries @ a if side is Side.PRE else a @ b.entries

    best = None  # (objective, restart, theta, trace, converged)
    for r, run in enumerate(runs):
        obj = weighted_error(compose(_realize(template, run.theta)), d.entries, alpha)
        if best is None or obj < best[0]:
            best = (obj, r, run.theta, run.trace, run.converged)
    obj, restart, theta, trace, conv = best
    if identity_obj <= obj:
        schedule, realized = template, np.eye(b.size)
        obj, trace, conv, restart = identity_obj, (identity_obj,), True, -1
    else:
        schedule = template.with_angles(theta)
        realized = givens_to_matrix(schedule)
    return AdjustmentMatrix(pattern=pattern, side=side, base=b.kind, target=d.kind,
                            schedule=schedule, realized=realized, objective=float(obj),
                            identity_objective=float(identity_obj), converged=conv,
                            objective_trace=tuple(trace), restart_index=restart)
