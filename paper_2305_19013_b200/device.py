"""Device plumbing: torch owns device memory and streams; kernels come from the C ABI."""

from __future__ import annotations

import numpy as np
import torch


class NoDeviceError(RuntimeError):
    pass


def get_device(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise NoDeviceError("paper_2305_19013_b200 requires a CUDA device (no CPU fallback)")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device)
    if dev.type != "cuda":
        raise NoDeviceError(f"device {dev} is not a CUDA device (no CPU fallback)")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


def current_stream_ptr(device=None) -> int:
    return torch.cuda.current_stream(get_device(device)).cuda_stream


def as_device(x, device=None, dtype=torch.float64):
    """(tensor on the device, converter back to the caller's array type)."""
    if isinstance(x, torch.Tensor):
        dev = get_device(device if device is not None else (x.device if x.is_cuda else None))
        t = x.to(device=dev, dtype=dtype)
        if x.is_cuda:
            return t, (lambda y: y)
        return t, (lambda y: y.cpu())
    dev = get_device(device)
    arr = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    t = torch.from_numpy(arr).to(dev)
    return t, (lambda y: y.cpu().numpy())


def from_device(t):
    return t.cpu().numpy()
