"""Config-1 kernels (4,096 x 32x32 fp64, DST-7 band6-pre): forward and inverse,
back-to-back launches, plus the forward on rotating buffers (L2 not resident).
Usage: python tools/prof_c1.py [iters]"""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2505_23618_b200 import _lib  # noqa: E402

w = bench.Uniform("c1", 0)
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 3
fwd = w.launches[0][1]
ref = w._ref


def inv():
    _lib.check(w._lib.dctadj_inverse_2d(ref, ref, w.y.data_ptr(), w.xr.data_ptr(), w.nblk,
                                        w._dtc, w._st))


def timed(fn, n):
    fn(0) if fn.__code__.co_argcount else fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(n):
        fn(i) if fn.__code__.co_argcount else fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


print(f"c1 fwd {timed(fwd, iters):.2f} us per launch")
print(f"c1 inv {timed(inv, iters):.2f} us per launch")
r, step = w.rotating()
rot = timed(lambda i: step(i % r), max(iters, r))
print(f"c1 fwd rotating ({r} buffers) {rot:.2f} us per launch")
err = (w.xr - w.x).abs().max().item() / w.x.abs().max().item()
print(f"c1 round-trip rel err {err:.2e}")
assert err < 1e-12, err
