"""Small cases of every kernel family, for compute-sanitizer (memcheck /
racecheck / synccheck, one tool per run).  Exits 0 when all results check."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2505_23618_b200 import kernels, pipeline  # noqa: E402

torch.manual_seed(0)
dev = "cuda"
t8 = bench._post(32, "dct8")
t6 = bench._pre(32, "dst7")
x = torch.randn(37, 32, 32, device=dev)  # ragged vs the 2-4 block super-tiles
for t in (t8, t6):
    y = pipeline.forward_adjusted_2d(t, t, x)
    xr = pipeline.inverse_adjusted_2d(t, t, y)
    assert float((xr - x).abs().max()) < 1e-4
xd = x.double()
y = pipeline.forward_adjusted_2d(t6, t6, xd)
assert float((pipeline.inverse_adjusted_2d(t6, t6, y) - xd).abs().max()) < 1e-10
v = torch.randn(45, 64, device=dev)
assert float((kernels.idct2(kernels.dct2(v)) - v).abs().max()) < 1e-4
t64 = bench._pre(64, "dst7")
assert float((pipeline.inverse_adjusted(t64, pipeline.forward_adjusted(t64, v)) - v).abs().max()) < 1e-4
fr = torch.randn(2, 48, 96, device=dev)
c = pipeline.forward_frames(t8, t8, fr)
assert float((pipeline.inverse_frames(t8, t8, c, 48, 96) - fr).abs().max()) < 1e-4
b = pipeline.MixedBatch.packed(np.array([0, 2, 3, 1, 2]), np.array([1, 0, 3, 2, 2]), [16, 16, 32, 32])
tab = [bench._post(16, "dst7"), bench._post(16, "dct8"), bench._post(32, "dst7"), bench._post(32, "dct8")]
xm = torch.randn(b.total_elements, device=dev)
assert float((pipeline.mixed_inverse(b, tab, pipeline.mixed_forward(b, tab, xm)) - xm).abs().max()) < 1e-4
from paper_2505_23618_b200 import matio  # noqa: E402
s7 = matio.load_designed("sub8_post_dct2_dst7_n32")
res = pipeline.simultaneous_encoder_eval(x[:5], pipeline.EncoderContext(s7, s7))
assert len(res) == 5
torch.cuda.synchronize()
print("sanitize smoke ok")
