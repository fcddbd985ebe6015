"""Config-4 band6-pre DST-7 forward / inverse (262,144 x 64x64 fp32), a few launches."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2505_23618_b200 import matio, pipeline  # noqa: E402

t = pipeline.make_adjusted_transform(matio.load_designed("band6_pre_dst3_dst7_n64"))
x = torch.randn(262144, 64, 64, device="cuda")
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 3
inv = len(sys.argv) > 2 and sys.argv[2] == "inv"
fn = pipeline.inverse_adjusted_2d if inv else pipeline.forward_adjusted_2d
y = fn(t, t, x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(iters):
    y = fn(t, t, x)
e1.record()
torch.cuda.synchronize()
print(f"c4 pre {'inv' if inv else 'fwd'} {e0.elapsed_time(e1) / iters * 1e3:.1f} us per launch")
