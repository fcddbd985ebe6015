"""Device plumbing for the Python mirror: numpy/torch in, device buffers to the
C-ABI, the caller's type out.  PyTorch provides device memory and the current
stream only; all arithmetic happens in libdctadj.so.

numpy inputs follow the reference's convention (cast to float64,
pipeline.py:47-57) and come back as new float64 arrays; CUDA torch tensors keep
their float32/float64 dtype and stay on the device.
"""
from __future__ import annotations

import numpy as np

from . import _lib
from .errors import CudaError

try:  # torch is plumbing only; a missing torch means no device path at all
    import torch
except ImportError:  # pragma: no cover
    torch = None


def require_cuda() -> None:
    if torch is None or not torch.cuda.is_available():
        raise CudaError("no CUDA device: this build has no CPU path (B200 / sm_100a only)")
    _lib.load()


def is_tensor(x) -> bool:
    return torch is not None and isinstance(x, torch.Tensor)


def to_device(x):
    """(contiguous CUDA tensor, returns_numpy)."""
    require_cuda()
    if is_tensor(x):
        t = x
        if t.dtype not in (torch.float32, torch.float64):
            t = t.to(torch.float64)
        if not t.is_cuda:
            return t.contiguous().to("cuda"), False
        t = t.contiguous()
        if t.data_ptr() % 16:  # TMA needs 16-byte aligned bases (a view at an odd offset)
            t = t.clone()
        return t, False
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    return torch.from_numpy(a).to("cuda"), True


def from_device(t, as_numpy: bool):
    return t.cpu().numpy() if as_numpy else t


def dtype_code(t) -> int:
    return _lib.F32 if t.dtype == torch.float32 else _lib.F64


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def empty_like(t, shape=None):
    return torch.empty(t.shape if shape is None else shape, dtype=t.dtype, device=t.device)
