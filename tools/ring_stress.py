"""Stress the shared-ring kernel (ring_kernel, tile_kernel.cuh) on config-4-sized
batches: REPEATS back-to-back forward and inverse launches over 262,144 64x64
fp32 blocks per op, every output compared bit for bit with the first launch of
the same variant and against the default build's (variant 0) result.

Usage (one variant per process, so a hang is bounded by `timeout`):
    DCTADJ_LIB=<lib> DCTADJ_VARIANT=<k> python tools/ring_stress.py <op> [repeats]
op: sub8 | band6.  Prints one line per direction: launches, mismatching launches,
max relative error against the variant-0 result computed in the same process
(DCTADJ_VARIANT is read once per process, so variant 0 comes from the oracle-gated
tile path of a second process -- here: the forward / inverse pair's own round
trip error is checked instead)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2505_23618_b200 import matio, pipeline  # noqa: E402

op = sys.argv[1] if len(sys.argv) > 1 else "sub8"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
name = {"sub8": "sub8_post_dct2_dst7_n64", "band6": "band6_pre_dst3_dst7_n64"}[op]
t = pipeline.make_adjusted_transform(matio.load_designed(name))
g = torch.Generator(device="cuda").manual_seed(7)
x = torch.randn(262144, 64, 64, device="cuda", generator=g) * 40
y0 = pipeline.forward_adjusted_2d(t, t, x)
x0 = pipeline.inverse_adjusted_2d(t, t, y0)
torch.cuda.synchronize()
rt = ((x0 - x).abs().amax() / x.abs().amax()).item()
bad_f = bad_i = 0
for _ in range(reps):
    y = pipeline.forward_adjusted_2d(t, t, x)
    xr = pipeline.inverse_adjusted_2d(t, t, y0)
    torch.cuda.synchronize()
    bad_f += int(not torch.equal(y, y0))
    bad_i += int(not torch.equal(xr, x0))
print(f"{op}: {reps} repeats, forward mismatches {bad_f}, inverse mismatches {bad_i}, "
      f"round-trip rel err {rt:.2e}, y0 sum {y0.double().sum().item():.6e}, x0 sum {x0.double().sum().item():.6e}",
      flush=True)
