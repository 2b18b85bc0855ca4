"""Array plumbing: numpy (host) or torch (CUDA device) buffers -> raw pointers.

torch is the device-memory / stream provider only; all compute is in
libnufft_b200.so.  Host (numpy) buffers are handed to the C-ABI as host
pointers and staged by the library itself.
"""

from __future__ import annotations

import numpy as np
import torch

_NP_TO_TORCH = {np.float32: torch.float32, np.float64: torch.float64,
                np.complex64: torch.complex64, np.complex128: torch.complex128,
                np.int32: torch.int32, np.int64: torch.int64}


def is_torch(x) -> bool:
    return isinstance(x, torch.Tensor)


def torch_dtype(np_dtype):
    return _NP_TO_TORCH[np.dtype(np_dtype).type]


def as_buffer(x, np_dtype, device=None):
    """Return (array, ptr, kind) with x converted to a contiguous buffer of
    np_dtype.  kind is 'cuda' for CUDA tensors, 'host' otherwise (CPU tensors
    are viewed as numpy)."""
    if is_torch(x):
        if x.is_cuda:
            t = x
            td = torch_dtype(np_dtype)
            if t.dtype != td:
                t = t.to(td)
            t = t.contiguous()
            return t, t.data_ptr(), "cuda"
        x = x.detach().numpy()
    a = np.ascontiguousarray(np.asarray(x), dtype=np_dtype)
    return a, a.ctypes.data, "host"


def empty_like_kind(kind, shape, np_dtype, device):
    if kind == "cuda":
        t = torch.empty(shape, dtype=torch_dtype(np_dtype), device=device)
        return t, t.data_ptr()
    a = np.empty(shape, dtype=np_dtype)
    return a, a.ctypes.data


def current_stream_ptr(device):
    if not torch.cuda.is_available():
        return None
    return torch.cuda.current_stream(device).cuda_stream


def numel(x):
    return x.numel() if is_torch(x) else int(np.asarray(x).size)
