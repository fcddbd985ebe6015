"""CPU, world_size 2 over gloo: the multi-GPU host path (block-range sharding,
per-rank work, post-timing scalar reduction) with the CPU oracle standing in
for the device kernels.  The data path has no collective; only scalars move."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_23618_b200 import shard


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_2505_23618_b200 import matio
    adj = matio.load_designed("sub8_post_dct2_dst7_n32")
    ax = O.OAxis(32, O.BASE_DCT2, O.ADJ_SUBBLOCK, O.SIDE_POST, 0, 8, np.array(adj.realized))
    nblk = 101
    x = np.random.default_rng(11).standard_normal((nblk, 32, 32))  # same global array on every rank
    b0, b1 = shard.block_range(rank, world, nblk)
    y = O.adjusted_2d(ax, ax, x[b0:b1])
    xr = O.adjusted_2d(ax, ax, y, inverse=True)
    st = shard.Stats(elapsed_ms=float(rank + 1), coefficients=(b1 - b0) * 1024,
                     err_energy=float(((xr - x[b0:b1]) ** 2).sum()),
                     ref_energy=float((x[b0:b1] ** 2).sum()),
                     max_rel_err=float(np.abs(xr - x[b0:b1]).max()))
    tot = shard.reduce_stats(st)
    full = O.adjusted_2d(ax, ax, x)
    q.put((rank, b0, b1, np.array_equal(y, full[b0:b1]), tot.coefficients, tot.elapsed_ms,
           tot.max_rel_err, tot.ref_energy))
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_two_rank_sharded_roundtrip():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=100) for _ in range(world))
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    assert res[0][1] == 0 and res[0][2] == res[1][1] and res[1][2] == 101
    assert all(r[3] for r in res)              # shard results == unsharded results
    assert all(r[4] == 101 * 1024 for r in res)  # SUM of coefficients
    assert all(r[5] == 2.0 for r in res)       # MAX of elapsed
    assert all(r[6] < 1e-12 for r in res)
    assert res[0][7] == res[1][7]


def _dry_run(gpus: int, scaling: str = "strong") -> dict:
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", str(gpus), "--dry-run",
                        "--scaling", scaling], capture_output=True, text=True, timeout=240,
                       env=env, cwd=root)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    return json.loads(lines[0])


@pytest.mark.timeout(300)
@pytest.mark.parametrize("gpus", [2, 3])
def test_bench_spawns_ranks_that_cover_each_config_once(gpus):
    """`bench.py --gpus N` self-launches N ranks (torchrun; gloo in --dry-run):
    their shards tile every BASELINE config exactly once (C1/C2/C4 block ranges,
    C3 equal-coefficient ranges, C5 frames), and the post-timing reduction sums
    the per-rank coefficient counts and takes the max of the times."""
    out = _dry_run(gpus)
    assert out["world"] == gpus
    full = _dry_run(1)
    for cfg, per_rank in out["per_rank"].items():
        assert len(per_rank) == gpus
        assert per_rank[0][0] == 0 and per_rank[-1][1] == out["totals"][cfg]
        for a, b in zip(per_rank, per_rank[1:]):
            assert a[1] == b[0] and a[0] <= a[1]  # contiguous, no gap, no overlap
        assert out["coefficients"][cfg] == full["coefficients"][cfg]  # same total work
    c3 = [b - a for a, b in out["per_rank"]["c3_pre"]]
    assert max(c3) - min(c3) < 0.01 * sum(c3)  # equal coefficient counts, not block counts
    assert out["reduced"]["c2_coefficients_sum"] == 65536 * 1024
    assert out["reduced"]["elapsed_ms_max"] == float(gpus)
    assert full["coefficients"]["c4_dst7_pre"] == 262144 * 4096
    assert full["coefficients"]["c5"] == 64 * 68 * 120 * 1024


@pytest.mark.timeout(300)
def test_bench_weak_scaling_gives_every_rank_the_config():
    out = _dry_run(2, "weak")
    for cfg, per_rank in out["per_rank"].items():
        assert per_rank == [[0, out["totals"][cfg]]] * 2
