"""e2e experiment: PCIe copy rates and the pipelined host-buffer entry."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2505_23618_b200 import pipeline, workloads  # noqa: E402

t = bench._post(32, "dct8")
x = workloads.c2_inputs("cuda", 65536)
xh = x.cpu().pin_memory()
yh = torch.empty_like(xh).pin_memory()
d = torch.empty_like(x)
nb = x.numel() * 4


def tm(fn, n=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n


print(f"H2D  {nb / tm(lambda: d.copy_(xh, non_blocking=True)) / 1e9:.1f} GB/s")
print(f"D2H  {nb / tm(lambda: yh.copy_(d, non_blocking=True)) / 1e9:.1f} GB/s")
s2 = torch.cuda.Stream()


def both():
    d.copy_(xh, non_blocking=True)
    with torch.cuda.stream(s2):
        yh.copy_(x, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)


print(f"H2D||D2H  {2 * nb / tm(both) / 1e9:.1f} GB/s total")
xn, yn = xh.numpy(), yh.numpy()
dt = tm(lambda: pipeline.forward_adjusted_2d_host(t, t, xn, out=yn))
print(f"forward_2d_host: {dt * 1e3:.2f} ms  -> {65536 * 1024 / dt / 1e9:.2f} Gcoef/s, {2 * nb / dt / 1e9:.1f} GB/s moved")
ok = np.allclose(yn, pipeline.forward_adjusted_2d(t, t, x).cpu().numpy())
print("correct", ok)
