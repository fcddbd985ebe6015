"""Config 5 fused step timing: the fused launch (adjusted + exact + error sums)
and the inverse, per launch, CUDA events over back-to-back launches; plus the
full-shard oracle gate (--gate).  In a DCTADJ_TUNING=1 build, DCTADJ_FX_WS=1
selects the warp-specialised variant (frames_exact.cuh)."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402

w = bench.Frames(rotate=False)
stream = torch.cuda.current_stream()
w.step(0)
torch.cuda.synchronize()
gate = w.gate(16) if "--gate" in sys.argv else None
res = {"ws": os.environ.get("DCTADJ_FX_WS", "0")}
for name, fn in w.launches + w.two_kernel:
    res[name] = bench._time_launch(stream, fn, 1, 50)
try:
    res["approx"] = w.approximation_error()
except SystemExit as e:  # diagnostics runs (DCTADJ_FX_SKIP) produce wrong sums by design
    res["approx"] = str(e)[:80]
res["fused_frac"] = w.bytes_first_launch / (res["forward_frames_exact"] / 1e3) / 1e9 / 6528.1
if gate:
    res["gate"] = {k: (v["max_err"] if isinstance(v, dict) else v) for k, v in gate.items()}
print(json.dumps(res))
