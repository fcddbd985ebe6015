"""Dense 32x32 fp32 through the tensor-core path vs numpy fp64 (small)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2505_23618_b200 import benchmark, pipeline  # noqa: E402
from paper_2505_23618_b200.transforms import TransformKind, build_transform  # noqa: E402

d7 = build_transform(TransformKind.DST7, 32).entries
td = benchmark._dense_transform(d7)
for nblk in (1, 5, 4, 37, 4096):
    x = torch.randn(nblk, 32, 32, device="cuda")
    y = pipeline.forward_adjusted_2d(td, td, x)
    xr = pipeline.inverse_adjusted_2d(td, td, y)
    torch.cuda.synchronize()
    xs = x.double().cpu().numpy()
    ref = np.einsum("ij,bjk,lk->bil", d7, xs, d7)
    err = np.abs(y.double().cpu().numpy() - ref).max() / np.abs(ref).max()
    err2 = np.abs(xr.double().cpu().numpy() - xs).max() / np.abs(xs).max()
    print(nblk, f"fwd rel err {err:.2e}  roundtrip {err2:.2e}")
    assert err < 1e-5 and err2 < 1e-5
print("tc smoke ok")
