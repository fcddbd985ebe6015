"""HBM ceilings for the traffic patterns of the C2 step (diagnostic):
1:1 copy (the two-kernel schedule) and 1:2 read:write (the fused round trip),
268 MB read per launch like config 2.  Usage: python tools/diag/copy12.py"""
import ctypes
import subprocess
from pathlib import Path

import torch

HERE = Path(__file__).resolve().parent
so = HERE / "libcopy12.so"
if not so.exists():
    subprocess.run(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                    "-Xcompiler", "-fPIC", "-o", str(so), str(HERE / "copy12.cu")], check=True)
lib = ctypes.CDLL(str(so))
lib.diag_copy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                          ctypes.c_int, ctypes.c_void_p]
n = 65536 * 1024
x = torch.randn(n, device="cuda")
y = torch.empty_like(x)
z = torch.empty_like(x)
st = torch.cuda.current_stream().cuda_stream
sms = torch.cuda.get_device_properties(0).multi_processor_count
for name, zz, nbytes in (("1:1 copy", None, 8 * n), ("1:2 read:write", z, 12 * n)):
    best = None
    for blocks in (sms * 2, sms * 4, sms * 8, sms * 16):
        f = lambda: lib.diag_copy(x.data_ptr(), y.data_ptr(), zz.data_ptr() if zz is not None else None,  # noqa: E731
                                  n // 4, blocks, st)
        f()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(50):
            f()
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) / 50 * 1e3
        if best is None or us < best[0]:
            best = (us, blocks)
    print(f"{name}: {best[0]:.1f} us, {nbytes / best[0] / 1e3:.0f} GB/s ({best[1]} blocks of 512)")
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
y.copy_(x)
a.record()
for _ in range(50):
    y.copy_(x)
b.record()
torch.cuda.synchronize()
us = a.elapsed_time(b) / 50 * 1e3
print(f"torch copy_: {us:.1f} us, {8 * n / us / 1e3:.0f} GB/s")
