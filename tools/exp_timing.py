"""Timing experiment: isolate kernel time, host launch overhead and steady-state
bandwidth for the config-2 kernels (not a bench number)."""
import ctypes
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2505_23618_b200 import _lib, workloads  # noqa: E402

EXTRA = {"pre32": ("pre32", 65536, 32, "f32", lambda: bench._pre(32, "dst7"), "c2_inputs", True)}
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
if name.startswith("shape"):  # shape<side>_<H>x<W>: uniform blocks of one C3 class
    side, hw = name[5:].split("_")
    H, W = map(int, hw.split("x"))
    mk = bench._pre if side == "pre" else bench._post
    th, tv = mk(W, "dst7"), mk(H, "dst7")
    nblk = (1 << 26) // (H * W)
    cfg = {"h": H, "w": W}
    x = workloads.ar1_blocks(nblk, H, W, 0.9, 16.0, 3)
else:
    wl, nblk, n_, dt_, make, inputs, inverse = EXTRA.get(name) or bench.UNIFORM[name]
    cfg = {"h": n_, "w": n_}
    th = tv = make()
    x = getattr(workloads, inputs)("cuda", nblk)
y = torch.empty_like(x)
xr = torch.empty_like(x)
lib = _lib.load()
(axh, kh), (axv, kv) = th.axis(), tv.axis()
dt = _lib.F32 if x.dtype == torch.float32 else _lib.F64
s = torch.cuda.current_stream()


def fwd(a, b, n=nblk):
    lib.dctadj_forward_2d(ctypes.byref(axh), ctypes.byref(axv), a.data_ptr(), b.data_ptr(), n, dt, s.cuda_stream)


def inv(a, b, n=nblk):
    lib.dctadj_inverse_2d(ctypes.byref(axh), ctypes.byref(axv), a.data_ptr(), b.data_ptr(), n, dt, s.cuda_stream)


def timed(fn, reps, trials=3):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(trials):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            fn()
        e1.record(s)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / reps * 1e3)  # us
    return best


nbytes = 2 * x.numel() * x.element_size()
print(f"bytes per launch {nbytes/1e6:.1f} MB")
t = timed(lambda: fwd(x, y), 50)
print(f"fwd x50 back-to-back: {t:.1f} us  {nbytes/t/1e3:.0f} GB/s")
t = timed(lambda: inv(y, xr), 50)
print(f"inv x50 back-to-back: {t:.1f} us  {nbytes/t/1e3:.0f} GB/s")
t = timed(lambda: (fwd(x, y), inv(y, xr)), 25)
print(f"fwd+inv x25: {t:.1f} us per pair  {2*nbytes/t/1e3:.0f} GB/s")
t = timed(lambda: lib.dctadj_copy_tiles(x.data_ptr(), y.data_ptr(), nblk, cfg["h"], cfg["w"], dt, s.cuda_stream), 50)
print(f"tile-pipeline copy x50: {t:.1f} us  {nbytes/t/1e3:.0f} GB/s")
t = timed(lambda: y.copy_(x), 50)
print(f"torch copy x50: {t:.1f} us  {nbytes/t/1e3:.0f} GB/s")
# host overhead per call (tiny batch)
xs = x[:1].clone(); ys = torch.empty_like(xs)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(2000):
    fwd(xs, ys, 1)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"host time per forward call: {(t1-t0)/2000*1e6:.1f} us")
# CUDA graph of one step
g = torch.cuda.CUDAGraph()
st = torch.cuda.Stream()
st.wait_stream(s)
with torch.cuda.stream(st):
    with torch.cuda.graph(g, stream=st):
        lib.dctadj_forward_2d(ctypes.byref(axh), ctypes.byref(axv), x.data_ptr(), y.data_ptr(), nblk, dt, st.cuda_stream)
        lib.dctadj_inverse_2d(ctypes.byref(axh), ctypes.byref(axv), y.data_ptr(), xr.data_ptr(), nblk, dt, st.cuda_stream)
s.wait_stream(st)
torch.cuda.synchronize()
t = timed(lambda: g.replay(), 25)
print(f"graph fwd+inv x25: {t:.1f} us per pair  {2*nbytes/t/1e3:.0f} GB/s")
