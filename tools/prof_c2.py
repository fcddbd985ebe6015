"""Minimal driver for ncu: a few forward + inverse launches of the config-2
kernels (65,536 x 32x32 fp32, DCT-8 post).  Usage under gpurun:
    python tools/prof_c2.py [--config c2] [--iters 3]"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2505_23618_b200 import pipeline, workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
wl, nblk, n, dt, make, inputs, inverse = bench.UNIFORM[a.config]
th = tv = make()
x = getattr(workloads, inputs)("cuda", nblk)
torch.cuda.synchronize()
for _ in range(a.iters):
    y = pipeline.forward_adjusted_2d(th, tv, x)
    if inverse:
        pipeline.inverse_adjusted_2d(th, tv, y)
torch.cuda.synchronize()
print("ok")
