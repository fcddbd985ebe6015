"""Config-1 forward (4,096 x 32x32 fp64, DST-7 band6-pre), back-to-back launches."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402

w = bench.Uniform("c1", 0)
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 3
fn = w.launches[0][1]
fn()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(iters):
    fn()
e1.record()
torch.cuda.synchronize()
print(f"c1 fwd {e0.elapsed_time(e1) / iters * 1e3:.2f} us per launch")
