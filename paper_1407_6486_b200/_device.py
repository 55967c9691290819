"""Device plumbing: fp64 CUDA fields in the library's layout, the current
stream, scratch caches.

Device layout (include/pintlab_b200.h): a grid field of shape (N,)*d with
N = n-1 is stored with an x-row pitch of n doubles for d >= 2 (one zero pad
per row, 16-byte aligned rows for TMA); 1-D fields are unpadded.  Public
objects expose *strided views* of the logical shape, so ``states.y[m][i, j]``
indexes exactly like the reference's numpy arrays.  Nodal arrays (M+1 fields)
are one allocation with a field stride of the padded field size.  All
storage is zero-initialised and every kernel maps pad zeros to zeros.

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


def _layout(grid_shape):
    """(field strides, storage elements) of one grid field."""
    d = len(grid_shape)
    N = grid_shape[-1]
    pitch = N + 1 if d >= 2 else N
    if d == 1:
        return (1,), N
    if d == 2:
        return (pitch, 1), N * pitch
    return (N * pitch, pitch, 1), N * N * pitch


def field_elems(grid_shape):
    return _layout(tuple(grid_shape))[1]


def new_field(grid_shape, lead=()):
    """Zeroed device field(s) in the library layout; returns the strided view
    of logical shape lead + grid_shape."""
    grid_shape = tuple(grid_shape)
    lead = tuple(lead)
    strides, ns = _layout(grid_shape)
    count = int(np.prod(lead)) if lead else 1
    store = torch.zeros(count * ns, dtype=torch.float64, device=device())
    lead_strides = []
    acc = ns
    for dim in reversed(lead):
        lead_strides.insert(0, acc)
        acc *= dim
    return torch.as_strided(store, lead + grid_shape, tuple(lead_strides) + strides)


def is_field(t, grid_dim):
    """True when t is an fp64 CUDA view in the library layout."""
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64):
        return False
    shape = tuple(t.shape)
    if len(shape) < grid_dim:
        return False
    gshape = shape[len(shape) - grid_dim:]
    if len(set(gshape)) != 1:
        return False
    strides, ns = _layout(gshape)
    want = list(strides)
    acc = ns
    for dim in reversed(shape[:len(shape) - grid_dim]):
        want.insert(0, acc)
        acc *= dim
    got = list(t.stride())
    return all(g == w or s == 1 for g, w, s in zip(got, want, shape))


def require_field(t, grid_dim, what):
    """The *_into entry points take device fields in the library layout (no
    copies); anything else is an error, never a silent out-of-bounds read."""
    if not is_field(t, grid_dim):
        raise ValueError(f"{what}: expected an fp64 CUDA field in the library's row-padded "
                         "layout (use _device.to_device / new_field)")


def to_device(x, grid_dim=None):
    """(field, was_host): x as a device field in the library layout (copied
    unless it already is one).  grid_dim defaults to x.ndim."""
    if grid_dim is None:
        grid_dim = np.ndim(x) if not isinstance(x, torch.Tensor) else x.dim()
    if is_field(x, grid_dim):
        return x, False
    host = not (isinstance(x, torch.Tensor) and x.is_cuda)
    if isinstance(x, torch.Tensor):
        src = x.detach().to(dtype=torch.float64)
    else:
        src = torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64)))
    shape = tuple(src.shape)
    out = new_field(shape[len(shape) - grid_dim:], shape[:len(shape) - grid_dim])
    out.copy_(src, non_blocking=src.is_pinned() if not src.is_cuda else False)
    return out, host


def clone_field(t, grid_dim=None):
    """Copy of a device field, in the library layout."""
    if grid_dim is None:
        grid_dim = t.dim()
    shape = tuple(t.shape)
    out = new_field(shape[len(shape) - grid_dim:], shape[:len(shape) - grid_dim])
    out.copy_(t)
    return out


def flat_storage(t):
    """Contiguous 1-D view of one field's storage (pads included): the wire
    format of the time-rank hand-offs."""
    return torch.as_strided(t, (field_elems(tuple(t.shape)),), (1,), t.storage_offset())


def field_from_flat(flat, grid_shape):
    """Field view over a flat storage buffer (inverse of flat_storage)."""
    strides, ns = _layout(tuple(grid_shape))
    return torch.as_strided(flat, tuple(grid_shape), strides, flat.storage_offset())


def like_input(t, was_host):
    """Return t as a dense numpy array when the caller passed host data."""
    return t.contiguous().cpu().numpy() if was_host else t


def ptr(t):
    return None if t is None else t.data_ptr()


def zeros(shape):
    return torch.zeros(shape, dtype=torch.float64, device=device())


def scratch(tag, nbytes):
    """Zeroed, stream-ordered scratch buffer reused across calls (per stream);
    zero pads stay zero because every kernel maps zeros to zeros."""
    key = (tag, stream_ptr(), torch.cuda.current_device())
    buf = _scratch.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.zeros(max(int(nbytes), 8), dtype=torch.uint8, device=device())
        _scratch[key] = buf
    return buf


def release_scratch():
    _scratch.clear()
