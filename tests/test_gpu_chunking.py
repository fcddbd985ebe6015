"""Batches larger than one launch's 32-bit TMA row range run as several launches.
DCTADJ_MAX_ROWS (read once per process) lowers the limit so a small batch
exercises the split; results must equal the single-launch ones bit for bit."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

SCRIPT = r"""
import sys, torch
sys.path.insert(0, %r)
from paper_2505_23618_b200 import matio, pipeline, benchmark
from paper_2505_23618_b200.transforms import TransformKind, build_transform
t = pipeline.make_adjusted_transform(matio.load_designed("sub8_post_dct2_dst7_n32"))
g = torch.Generator(device="cuda").manual_seed(5)
x = torch.randn(1000, 32, 32, device="cuda", generator=g)
v = torch.randn(3001, 32, device="cuda", generator=g)
td = benchmark._dense_transform(build_transform(TransformKind.DST7, 32).entries)
torch.save({"y2": pipeline.forward_adjusted_2d(t, t, x).cpu(),
            "y1": pipeline.forward_adjusted(t, v).cpu(),
            "yd": pipeline.forward_adjusted_2d(td, td, x).cpu(),
            "rt": torch.stack(pipeline.roundtrip_adjusted_2d(t, t, x)).cpu()}, sys.argv[1])
"""


def _run(tmp_path, name, env):
    out = tmp_path / f"{name}.pt"
    subprocess.run([sys.executable, "-c", SCRIPT % str(ROOT), str(out)], check=True,
                   env={**os.environ, **env}, timeout=300)
    import torch
    return torch.load(out)


def test_linear_batches_split_across_launches(tmp_path):
    import torch
    one = _run(tmp_path, "one", {})
    split = _run(tmp_path, "split", {"DCTADJ_MAX_ROWS": "1000"})  # 31 blocks / 1000 vectors
    for k in one:
        assert torch.equal(one[k], split[k]), k
