"""Device plumbing: torch owns every buffer, libivk does every flop."""

import numpy as np
import torch

from . import _lib

__all__ = ["device", "upload", "ptr", "stream", "as_device_vector", "to_host", "is_device",
           "require_cuda"]


def require_cuda():
    if not torch.cuda.is_available():
        raise _lib.IvkError("a CUDA device is required: the IRK-Vanka path runs only on the GPU "
                            "(no CPU fallback)")
    _lib.load()


def device():
    require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def upload(a, dtype):
    """Host array -> contiguous device tensor of ``dtype``."""
    arr = np.ascontiguousarray(np.asarray(a), dtype=dtype)
    return torch.from_numpy(arr).to(device(), non_blocking=False)


def ptr(t):
    return None if t is None else t.data_ptr()


def stream():
    return torch.cuda.current_stream().cuda_stream


def is_device(x):
    return isinstance(x, torch.Tensor) and x.is_cuda


def as_device_vector(x, n):
    """(tensor on device, was_numpy).  Numpy input is copied up once."""
    if is_device(x):
        if x.dtype != torch.float64 or x.ndim != 1 or x.numel() != n:
            raise ValueError(f"expected a float64 device vector of length {n}")
        return x.contiguous(), False
    arr = np.asarray(x, dtype=np.float64)
    if arr.shape != (n,):
        raise ValueError(f"expected a vector of length {n}, got shape {arr.shape}")
    return upload(arr, np.float64), True


def to_host(t):
    return t.detach().cpu().numpy()
