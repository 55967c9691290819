"""Device plumbing: fp64 CUDA tensors, the current stream, scratch caches.

PyTorch is used only for allocation, streams and host<->device copies; every
computation on the path is a kernel of lib/libpintlab_b200.so.
"""
from __future__ import annotations

import numpy as np
import torch

_scratch: dict = {}


def device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1407_6486_b200 needs a CUDA device (B200); "
                           "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr():
    return torch.cuda.current_stream().cuda_stream


def to_device(x):
    """(tensor, was_host): fp64 contiguous CUDA tensor for x (numpy / torch)."""
    if isinstance(x, torch.Tensor):
        if x.is_cuda and x.dtype == torch.float64 and x.is_contiguous():
            return x, False
        host = not x.is_cuda
        return x.to(device=device(), dtype=torch.float64).contiguous(), host
    arr = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    return torch.from_numpy(arr).to(device()), True


def like_input(t, was_host):
    """Return t as numpy when the caller passed host data (drop-in behaviour)."""
    return t.cpu().numpy() if was_host else t


def ptr(t):
    return None if t is None else t.data_ptr()


def empty(shape):
    return torch.empty(shape, dtype=torch.float64, device=device())


def zeros(shape):
    return torch.zeros(shape, dtype=torch.float64, device=device())


def scratch(tag, nbytes):
    """Stream-ordered scratch buffer reused across calls (keyed per stream)."""
    key = (tag, stream_ptr(), torch.cuda.current_device())
    buf = _scratch.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(int(nbytes), 8), dtype=torch.uint8, device=device())
        _scratch[key] = buf
    return buf


def release_scratch():
    _scratch.clear()
