"""Config 3 by class: the fused gather round trip on HOMOGENEOUS mixed batches
(one shape, one kind pair), per-launch time and algorithmic GB/s (12 B per
coefficient pair), next to the real 16-class mix.  Usage:
python tools/prof_c3_classes.py [pre|post] [iters]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2505_23618_b200 import _lib, pipeline  # noqa: E402

side = sys.argv[1] if len(sys.argv) > 1 else "pre"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
mk = bench._pre if side == "pre" else bench._post
table = [mk(16, "dst7"), mk(16, "dct8"), mk(32, "dst7"), mk(32, "dct8")]
axes = (_lib.Axis * 4)()
keep = []
for k, tr in enumerate(table):
    ax, m = tr.axis()
    axes[k] = ax
    keep.append(m)
lib = _lib.load()
st = torch.cuda.current_stream().cuda_stream
target = 256 << 20  # elements' bytes per homogeneous batch (> 2 x L2)


def run(h_index, v_index, label):
    b = pipeline.MixedBatch.packed(h_index, v_index, bench.C3_SIZES)
    n = b.total_elements
    sets = [(torch.randn(n, device="cuda") * 16, torch.empty(n, device="cuda"), torch.empty(n, device="cuda"))
            for _ in range(2)]

    def step(i):
        x, y, xr = sets[i & 1]
        _lib.check(lib.dctadj_mixed_roundtrip(b._plan, axes, x.data_ptr(), y.data_ptr(), xr.data_ptr(), 0, st))

    for i in range(4):
        step(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(iters):
        step(i)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    print(f"{label:28s} {len(h_index):8d} blocks  {ms * 1e3:9.1f} us  {12 * n / ms / 1e6:7.0f} GB/s  "
          f"{2 * n / ms / 1e6:7.1f} G coef/s", flush=True)


for hi in range(4):
    for vi in range(4):
        if hi % 2 != vi % 2 and len(sys.argv) <= 3:
            continue  # kinds differ only in coefficient tables / mirrored pairs: the two same-kind pairs per shape
        w, h = bench.C3_SIZES[hi], bench.C3_SIZES[vi]
        nb = target // (4 * w * h)
        run(np.full(nb, hi, np.int32), np.full(nb, vi, np.int32), f"{h}x{w} h{hi} v{vi}")
gh, gv, _ = bench.c3_table()
run(gh, gv, "config-3 mix (16 classes)")
