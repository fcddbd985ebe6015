"""Dense 32x32 (or 64x64: argv[2]) fp32 2-D transform (tensor-core path unless
DCTADJ_DENSE_TC=0), 64 M coefficients, a few back-to-back launches (ncu / timing)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2505_23618_b200 import benchmark, pipeline  # noqa: E402
from paper_2505_23618_b200.transforms import TransformKind, build_transform  # noqa: E402

n = int(sys.argv[2]) if len(sys.argv) > 2 else 32  # block size: 32 or 64
td = benchmark._dense_transform(build_transform(TransformKind.DST7, n).entries)
x = torch.randn(65536 * 1024 // (n * n), n, n, device="cuda")
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for _ in range(3):
    y = pipeline.forward_adjusted_2d(td, td, x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(iters):
    y = pipeline.forward_adjusted_2d(td, td, x)
e1.record()
torch.cuda.synchronize()
print(f"dense {n}x{n} fwd {e0.elapsed_time(e1) / iters * 1e3:.1f} us per launch (HBM floor {x.numel() * 8 / 6553.6e3:.1f} us)")
import time  # noqa: E402
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(iters):
    y = pipeline.forward_adjusted_2d(td, td, x)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"host enqueue {(t1 - t0) / iters * 1e6:.1f} us per call")
