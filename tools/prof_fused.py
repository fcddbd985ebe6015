"""Config-5 comparison step (adjusted + exact forward + error sums, the fused
tensor-core kernel) over 64 frames 2160 x 3840; a few launches (ncu / timing)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2505_23618_b200 import benchmark, matio, pipeline  # noqa: E402
from paper_2505_23618_b200.transforms import TransformKind, build_transform  # noqa: E402

td = benchmark._dense_transform(build_transform(TransformKind.DST7, 32).entries)
ta = pipeline.make_adjusted_transform(matio.load_designed("sub8_post_dct2_dst7_n32"))
x = torch.randn(64, 2160, 3840, device="cuda")
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 3
pipeline.forward_frames_exact(ta, ta, td, td, x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(iters):
    pipeline.forward_frames_exact(ta, ta, td, td, x)
e1.record()
torch.cuda.synchronize()
print(f"fused frames_exact {e0.elapsed_time(e1) / iters * 1e3:.1f} us per call")
