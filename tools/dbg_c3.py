"""Debug: per-class non-finite / round-trip failures of the config-3 workload."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402

side = sys.argv[1] if len(sys.argv) > 1 else "pre"
w = bench.Mixed(side, 0)
for name, fn in w.launches:
    fn()
torch.cuda.synchronize()
b = w.batch
sizes = np.array([16, 16, 32, 32])
H = sizes[w.v_index]
W = sizes[w.h_index]
offs = torch.from_numpy(b.offsets).cuda()
for hs in (16, 32):
    for ws in (16, 32):
        for hk in range(2):
            for vk in range(2):
                sel = np.nonzero((H == hs) & (W == ws) & (w.h_index % 2 == hk) & (w.v_index % 2 == vk))[0]
                if len(sel) == 0:
                    continue
                idx = offs[torch.from_numpy(sel).cuda()][:, None] + torch.arange(hs * ws, device="cuda")[None, :]
                y, xr, x = w.y[idx], w.xr[idx], w.x[idx]
                ny = (~torch.isfinite(y)).any(dim=1)
                nx = (~torch.isfinite(xr)).any(dim=1)
                ex = ((xr - x).abs().amax(dim=1) > 1e-3 * x.abs().max())
                print(f"{hs}x{ws} hk{hk} vk{vk}: n={len(sel)} nonfinite fwd {int(ny.sum())} inv {int(nx.sum())} "
                      f"bad roundtrip {int(ex.sum())} first {sel[torch.nonzero(ny | nx | ex).flatten()[:3].cpu().numpy()] if (ny|nx|ex).any() else '-'}")
