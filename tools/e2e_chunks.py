"""e2e (host buffers) throughput of the config-2 step for the current
DCTADJ_HOST_CHUNK_MB (one value per process: the library reads it once)."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402

w = bench.Uniform("c2", 0)
w.e2e()
torch.cuda.synchronize()
n = 5
t = time.perf_counter()
for _ in range(n):
    w.e2e()
dt = (time.perf_counter() - t) / n
print(f"chunk {os.environ.get('DCTADJ_HOST_CHUNK_MB', 'default')} MB: e2e {w.coef_per_step / dt / 1e9:.2f} G coef/s, "
      f"{(w.e2e_bytes[0] + w.e2e_bytes[1]) / dt / 1e9:.1f} GB/s duplex")
