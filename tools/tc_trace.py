"""Per-tile event clocks of the tensor-core dense kernel (CTA 0), via DCTADJ_TC_TRACE.
Events: 0 loop top, 1 X landed, 2 A1 stored (a1_ready), 3 D1 ready, 4 A2 stored,
5 D2 ready, 6 Y store issued, 7 pass-1 issue (MMA warp)."""
import os
import sys
from pathlib import Path

import numpy as np

out = "/tmp/tc_trace.txt"
os.environ["DCTADJ_TC_TRACE"] = out
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2505_23618_b200 import benchmark, pipeline  # noqa: E402
from paper_2505_23618_b200.transforms import TransformKind, build_transform  # noqa: E402

td = benchmark._dense_transform(build_transform(TransformKind.DST7, 32).entries)
mode = sys.argv[1] if len(sys.argv) > 1 else "linear"
if mode == "fused":  # config 5 comparison step: adjusted + exact in one kernel
    from paper_2505_23618_b200 import matio
    ta = pipeline.make_adjusted_transform(matio.load_designed("sub8_post_dct2_dst7_n32"))
    x = torch.randn(64, 2160, 3840, device="cuda")
    for _ in range(3):
        pipeline.forward_frames_exact(ta, ta, td, td, x)
elif mode == "frames":  # config 5 shape: 64 frames of 2160 x 3840 (bottom tile row zero-filled)
    x = torch.randn(64, 2160, 3840, device="cuda")
    for _ in range(3):
        pipeline.forward_frames(td, td, x)
else:
    x = torch.randn(65536, 32, 32, device="cuda")
    for _ in range(3):
        pipeline.forward_adjusted_2d(td, td, x)
torch.cuda.synchronize()
t = np.loadtxt(out, dtype=np.float64)
ctas, t = t[128:, :2], t[:128]
ctas = ctas[ctas[:, 0] > 0]
c0 = ctas[:, 0].min()
print("CTAs", len(ctas), "start spread ns", int(ctas[:, 0].max() - c0), "end ns: min",
      int(ctas[:, 1].min() - c0), "median", int(np.median(ctas[:, 1]) - c0), "max",
      int(ctas[:, 1].max() - c0), "CTA0", int(ctas[0, 1] - c0))
t0 = t[t[:, 0] > 0, 0].min()
np.set_printoptions(linewidth=200, suppress=True)
print("tile  top  landed a1  d1  a2  d2  stored  mma1  (cycles from first event)")
for k in list(range(12)) + list(range(100, len(t))):
    if t[k, 0] > 0:
        print(k, (t[k] - t0).astype(np.int64))
d = np.diff(t[:, :7], axis=1)
v = t[:, 0] > 0
print("mean phase cycles (landed-top, a1-landed, d1-a1, a2-d1, d2-a2, stored-d2):",
      d[v][8:].mean(axis=0).astype(int), "tiles", int(v.sum()), "span", int(t[v, 6].max() - t0))
print("mma1 issue - a1:", (t[v, 7] - t[v, 2])[8:].mean().astype(int), " d1 - mma1:",
      (t[v, 3] - t[v, 7])[8:].mean().astype(int))
