"""Multi-GPU partitioning: blocks are independent (reference SPEC.md:313-314),
so ranks split the work by range and never exchange data on the hot path.
torch.distributed (NCCL on B200, gloo in the CPU tests) only carries scalars
after the timed region: elapsed times (max), coefficient counts and error
energies (sum), the worst relative error (max).

  block_range(rank, world, nblk)      contiguous, sizes differ by at most 1 (C1, C2, C4)
  weighted_ranges(weights, world)     equal-work split by prefix sum (C3: coefficient counts)
  frame_range(rank, world, nframes)   frames per rank (C5)
  reduce_stats(stats)                 the post-timing scalar reduction
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def block_range(rank: int, world: int, nblk: int) -> tuple[int, int]:
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    return rank * nblk // world, (rank + 1) * nblk // world


def frame_range(rank: int, world: int, nframes: int) -> tuple[int, int]:
    return block_range(rank, world, nframes)


def weighted_ranges(weights, world: int) -> list[tuple[int, int]]:
    """Split items into `world` contiguous ranges of ~equal total weight
    (split points where the prefix sum crosses k/world of the total)."""
    w = np.asarray(weights, dtype=np.int64)
    if w.size == 0:
        return [(0, 0)] * world
    csum = np.cumsum(w)
    total = int(csum[-1])
    cuts = [0]
    for k in range(1, world):
        cuts.append(int(np.searchsorted(csum, k * total / world, side="left")) + 1)
    cuts.append(w.size)
    cuts = np.maximum.accumulate(np.minimum(cuts, w.size))
    return [(int(cuts[k]), int(cuts[k + 1])) for k in range(world)]


@dataclass
class Stats:
    elapsed_ms: float = 0.0       # max over ranks (device-timed region)
    coefficients: int = 0         # sum
    err_energy: float = 0.0       # sum  ||Y_adj - Y_exact||^2
    ref_energy: float = 0.0       # sum  ||Y_exact||^2
    max_rel_err: float = 0.0      # max
    e2e_ms: float = 0.0           # max (host-buffer step)
    err_energy_full: float = 0.0  # sum, unpadded tile rows only (config 5)
    ref_energy_full: float = 0.0  # sum, unpadded tile rows only


def reduce_stats(stats: Stats, device=None) -> Stats:
    """All-reduce the per-rank scalars (no-op without an initialised group):
    MAX of the times and the error, SUM of the counts and energies."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return stats
    mx = torch.tensor([stats.elapsed_ms, stats.max_rel_err, stats.e2e_ms], dtype=torch.float64,
                      device=device)
    sm = torch.tensor([float(stats.coefficients), stats.err_energy, stats.ref_energy,
                       stats.err_energy_full, stats.ref_energy_full], dtype=torch.float64,
                      device=device)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    return Stats(elapsed_ms=float(mx[0]), coefficients=int(round(float(sm[0]))),
                 err_energy=float(sm[1]), ref_energy=float(sm[2]), max_rel_err=float(mx[1]),
                 e2e_ms=float(mx[2]), err_energy_full=float(sm[3]), ref_energy_full=float(sm[4]))
