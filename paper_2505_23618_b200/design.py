"""Adjustment parameter records (host side).

The adjustment *designer* (the reference's coordinate-descent optimizer,
design.py:333-613) is offline: designed adjustments arrive as files in the
reference's text format (matio.py) -- see adjustments/ -- and designer.py runs
the optimizer itself on the GPU.  This
module keeps the records and structural helpers the data path needs, with the
reference's semantics:

  SparsityPattern / PatternKind / Side        reference design.py:43-109
  PlaneRotation / GivensSchedule              reference design.py:131-191
  givens_to_matrix                            reference design.py:194-204
  pattern_schedule_template                   reference design.py:225-250
  AdjustmentMatrix                            reference design.py:298-315
  dct8_adjustment_from_dst7 (C8 = S C7 S)     reference design.py:677-715
  identity_adjustment                         reference design.py:718-733
plus flip_pre_adjustment, the DCT-8 pre-adjustment of SURVEY.md App. A D3
(H8 = S H7 R = DCT3 (R A R)), which the reference has no record for.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from enum import Enum
from typing import NamedTuple, Sequence

import numpy as np

from .errors import InvalidScheduleError, KindMismatchError, PatternError, ShapeError
from .transforms import TransformKind, alternating_signs


class PatternKind(Enum):
    BAND = "band"
    SUBBLOCK = "subblock"
    DENSE = "dense"


class Side(Enum):
    PRE = "pre"
    POST = "post"

    def __str__(self) -> str:
        return self.value


@dataclass(frozen=True)
class SparsityPattern:
    """band(K): non-zeros only where |i-j| < K; subblock(B): identity outside
    the leading B x B block; dense: unrestricted."""

    kind: PatternKind
    size: int
    taps: int | None = None
    order: int | None = None

    def __post_init__(self):
        if self.size < 1:
            raise PatternError(f"pattern size must be >= 1, got {self.size}")
        if self.kind is PatternKind.BAND and not (self.taps and 1 <= self.taps <= self.size):
            raise PatternError(f"band taps must be in 1..{self.size}, got {self.taps}")
        if self.kind is PatternKind.SUBBLOCK and not (self.order and 1 <= self.order <= self.size):
            raise PatternError(f"sub-block order must be in 1..{self.size}, got {self.order}")

    @staticmethod
    def band(taps: int, size: int) -> "SparsityPattern":
        return SparsityPattern(PatternKind.BAND, size, taps=taps)

    @staticmethod
    def subblock(order: int, size: int) -> "SparsityPattern":
        return SparsityPattern(PatternKind.SUBBLOCK, size, order=order)

    @staticmethod
    def dense(size: int) -> "SparsityPattern":
        return SparsityPattern(PatternKind.DENSE, size)

    def label(self) -> str:
        return {PatternKind.BAND: f"band:{self.taps}",
                PatternKind.SUBBLOCK: f"subblock:{self.order}",
                PatternKind.DENSE: "dense"}[self.kind]

    @staticmethod
    def from_label(label: str, size: int) -> "SparsityPattern":
        if label == "dense":
            return SparsityPattern.dense(size)
        name, sep, arg = label.partition(":")
        if sep and arg.isdigit():
            if name == "band":
                return SparsityPattern.band(int(arg), size)
            if name == "subblock":
                return SparsityPattern.subblock(int(arg), size)
        raise PatternError(f"unknown pattern label {label!r}")


class PlaneRotation(NamedTuple):
    i: int
    j: int
    theta: float


@dataclass(frozen=True)
class GivensSchedule:
    """Layers of index-disjoint plane rotations applied in order.  (i, j, t)
    maps x_i <- cos t x_i - sin t x_j, x_j <- sin t x_i + cos t x_j."""

    size: int
    layers: tuple[tuple[PlaneRotation, ...], ...]

    def __post_init__(self):
        for layer in self.layers:
            used: set[int] = set()
            for r in layer:
                if not 0 <= r.i < r.j < self.size:
                    raise InvalidScheduleError(
                        f"rotation indices ({r.i},{r.j}) out of range for size {self.size}")
                if r.i in used or r.j in used:
                    raise InvalidScheduleError(f"index reused within a layer at ({r.i},{r.j})")
                used.update((r.i, r.j))

    @property
    def n_rotations(self) -> int:
        return sum(map(len, self.layers))

    def rotations(self) -> list[PlaneRotation]:
        return [r for layer in self.layers for r in layer]

    def angles(self) -> np.ndarray:
        return np.array([r.theta for r in self.rotations()], dtype=float)

    def with_angles(self, thetas: Sequence[float]) -> "GivensSchedule":
        thetas = [float(t) for t in thetas]
        if len(thetas) != self.n_rotations:
            raise InvalidScheduleError(f"expected {self.n_rotations} angles, got {len(thetas)}")
        it = iter(thetas)
        return GivensSchedule(self.size, tuple(
            tuple(PlaneRotation(r.i, r.j, next(it)) for r in layer) for layer in self.layers))


def givens_to_matrix(schedule: GivensSchedule) -> np.ndarray:
    """The orthogonal matrix of the schedule (row updates, layers in order)."""
    m = np.eye(schedule.size)
    for layer in schedule.layers:
        for i, j, theta in layer:
            c, s = math.cos(theta), math.sin(theta)
            mi, mj = m[i].copy(), m[j].copy()
            m[i] = c * mi - s * mj
            m[j] = s * mi + c * mj
    return m


def _circle_pairings(idx: list[int]) -> list[list[tuple[int, int]]]:
    """Round-robin (circle method) all-pairs schedule in disjoint layers."""
    ring: list[int | None] = list(idx) + ([None] if len(idx) % 2 else [])
    m = len(ring)
    out = []
    for _ in range(m - 1):
        layer = sorted((min(a, b), max(a, b)) for a, b in
                       ((ring[k], ring[m - 1 - k]) for k in range(m // 2))
                       if a is not None and b is not None)
        out.append(layer)
        ring = [ring[0], ring[-1], *ring[1:-1]]
    return out


def pattern_schedule_template(pattern: SparsityPattern) -> GivensSchedule:
    """Zero-angle skeleton: band(K) = K-1 brick-wall layers of adjacent pairs
    (bandwidth <= K-1 by construction); subblock(B) / dense = all pairs below
    B (resp. N) in round-robin layers."""
    n = pattern.size
    if pattern.kind is PatternKind.BAND:
        layers = []
        for level in range(pattern.taps - 1):
            layer = tuple(PlaneRotation(i, i + 1, 0.0) for i in range(level % 2, n - 1, 2))
            if layer:
                layers.append(layer)
        return GivensSchedule(n, tuple(layers))
    span = pattern.order if pattern.kind is PatternKind.SUBBLOCK else n
    return GivensSchedule(n, tuple(
        tuple(PlaneRotation(a, b, 0.0) for a, b in layer)
        for layer in _circle_pairings(list(range(span))) if layer))


@dataclass(frozen=True)
class AdjustmentMatrix:
    """A sparse orthogonal adjustment: H = B A (pre) or C B (post)."""

    pattern: SparsityPattern
    side: Side
    base: TransformKind
    target: TransformKind
    schedule: GivensSchedule
    realized: np.ndarray
    objective: float | None = None
    identity_objective: float | None = None
    converged: bool = True
    objective_trace: tuple[float, ...] = field(default=(), repr=False)
    restart_index: int = 0

    def __post_init__(self):
        if self.realized.shape != (self.pattern.size, self.pattern.size):
            raise ShapeError(f"realized {self.realized.shape} vs pattern size {self.pattern.size}")
        self.realized.setflags(write=False)


def dct8_adjustment_from_dst7(c_s7: AdjustmentMatrix) -> AdjustmentMatrix:
    """Post-side DCT-8 adjustment from the DST-7 one: C8 = S C7 S (chessboard
    signs); rotation (i, j) flips its angle iff i + j is odd."""
    if c_s7.side is not Side.POST or c_s7.base is not TransformKind.DCT2:
        raise KindMismatchError(
            f"sign-flip derivation needs side=post, base=dct2; got side={c_s7.side}, "
            f"base={c_s7.base}")
    swap = {TransformKind.DST7: TransformKind.DCT8, TransformKind.DCT8: TransformKind.DST7}
    if c_s7.target not in swap:
        raise KindMismatchError(f"target must be dst7 or dct8, got {c_s7.target}")
    s = alternating_signs(c_s7.pattern.size)
    thetas = [r.theta if (r.i + r.j) % 2 == 0 else -r.theta for r in c_s7.schedule.rotations()]
    return AdjustmentMatrix(
        pattern=c_s7.pattern, side=c_s7.side, base=c_s7.base, target=swap[c_s7.target],
        schedule=c_s7.schedule.with_angles(thetas),
        realized=np.outer(s, s) * c_s7.realized,
        objective=c_s7.objective, identity_objective=c_s7.identity_objective,
        converged=c_s7.converged, objective_trace=c_s7.objective_trace,
        restart_index=c_s7.restart_index)


def flip_pre_adjustment(a7: AdjustmentMatrix) -> AdjustmentMatrix:
    """DCT-8 pre-adjustment from a DST-7 one.

    H8 = S H7 R with H7 = DST3 A (reference PAPER.md Eq. (3), transforms.py:132-138);
    since S DST3 = DCT2^T R, H8 = DCT3 (R A R): a DCT-3 base with the reversed band.
    R A R keeps the band pattern; its rotations are the reversed pairs
    (N-2-i, N-1-i) with negated angles, layer order unchanged.
    """
    if a7.side is not Side.PRE or a7.base is not TransformKind.DST3:
        raise KindMismatchError(
            f"flip needs side=pre, base=dst3; got side={a7.side}, base={a7.base}")
    n = a7.pattern.size
    layers = tuple(tuple(sorted((PlaneRotation(n - 1 - r.j, n - 1 - r.i, -r.theta)
                                 for r in layer), key=lambda r: r.i))
                   for layer in a7.schedule.layers)
    target = {TransformKind.DST7: TransformKind.DCT8,
              TransformKind.DCT8: TransformKind.DST7}.get(a7.target, a7.target)
    return AdjustmentMatrix(
        pattern=a7.pattern, side=Side.PRE, base=TransformKind.DCT3, target=target,
        schedule=GivensSchedule(n, layers),
        realized=np.ascontiguousarray(a7.realized[::-1, ::-1]),
        objective=a7.objective, identity_objective=a7.identity_objective,
        converged=a7.converged, restart_index=a7.restart_index)


def identity_adjustment(pattern: SparsityPattern, side: Side, base: TransformKind,
                        target: TransformKind) -> AdjustmentMatrix:
    return AdjustmentMatrix(pattern=pattern, side=side, base=base, target=target,
                            schedule=pattern_schedule_template(pattern),
                            realized=np.eye(pattern.size))


def random_adjustment(pattern: SparsityPattern, side: Side, base: TransformKind,
                      seed: int, spread: float = 0.35) -> AdjustmentMatrix:
    """Pattern-conformant orthogonal adjustment with uniform random angles in
    [-spread, spread] (the reference's test/benchmark helper, test_pipeline.py:42-49,
    benchmark.py:58-73: speed and parity do not depend on designed values)."""
    template = pattern_schedule_template(pattern)
    rng = np.random.default_rng(seed)
    sched = template.with_angles(rng.uniform(-spread, spread, template.n_rotations))
    return AdjustmentMatrix(pattern=pattern, side=side, base=base, target=TransformKind.DST7,
                            schedule=sched, realized=givens_to_matrix(sched))
