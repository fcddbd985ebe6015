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


RT_SCRIPT = r"""
import sys, torch
sys.path.insert(0, %r)
from paper_2505_23618_b200 import matio, pipeline
from paper_2505_23618_b200.design import dct8_adjustment_from_dst7, flip_pre_adjustment
g = torch.Generator(device="cuda").manual_seed(9)
x = torch.randn(300, 64, 64, device="cuda", generator=g) * 40
s7 = matio.load_designed("sub8_post_dct2_dst7_n64")
b6 = matio.load_designed("band6_pre_dst3_dst7_n64")
out = {}
for name, adj in (("post", dct8_adjustment_from_dst7(s7)), ("pre7", b6), ("pre8", flip_pre_adjustment(b6))):
    t = pipeline.make_adjusted_transform(adj)
    out[name] = torch.stack(pipeline.roundtrip_adjusted_2d(t, t, x)).cpu()
torch.save(out, sys.argv[1])
"""


@pytest.mark.parametrize("variant", ["1", "2"])
def test_roundtrip_tuning_variants_64(tmp_path, variant):
    """The 64x64 fused round-trip kernels are tuning variants (DCTADJ_RT_VARIANT,
    read once per process): bit-identical to the default two-kernel path.  They
    exist only in a DCTADJ_TUNING=1 build of the library."""
    import torch
    from paper_2505_23618_b200 import _lib
    if not _lib.load().dctadj_tuning_build():
        pytest.skip("library built without DCTADJ_TUNING=1: no tuning variants to compare")

    def run(name, env):
        out = tmp_path / f"{name}.pt"
        subprocess.run([sys.executable, "-c", RT_SCRIPT % str(ROOT), str(out)], check=True,
                       env={**os.environ, **env}, timeout=300)
        return torch.load(out)

    two = run("two", {"DCTADJ_RT_UNFUSED": "1"})
    fused = run(f"v{variant}", {"DCTADJ_RT_VARIANT": variant})
    for k in two:
        assert torch.equal(two[k], fused[k]), k
