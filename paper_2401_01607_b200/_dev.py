"""Host/device tensor plumbing (PyTorch is only the allocator and the handoff)."""

from __future__ import annotations

import numpy as np


def torch():
    import torch as _t

    return _t


def is_tensor(a) -> bool:
    try:
        import torch as _t
    except ImportError:  # pragma: no cover
        return False
    return isinstance(a, _t.Tensor)


def np_dtype(a):
    """numpy dtype (float32/float64) of an ndarray or tensor."""
    if is_tensor(a):
        t = torch()
        return np.float32 if a.dtype == t.float32 else np.float64
    return np.float32 if a.dtype == np.float32 else np.float64


def torch_dtype(npd):
    t = torch()
    return t.float32 if npd == np.float32 else t.float64


class device_guard:
    """`torch.cuda.device(d)` without its Python overhead: switches the current
    device only when it differs (engine calls are made on their own device
    almost always)."""

    __slots__ = ("idx", "prev")

    def __init__(self, device):
        self.idx = device.index if hasattr(device, "index") else int(device)

    def __enter__(self):
        self.prev = torch()._C._cuda_exchangeDevice(self.idx)
        return self

    def __exit__(self, *exc):
        if self.prev != self.idx:
            torch()._C._cuda_exchangeDevice(self.prev)
        return False


def as_device(a, npd, device=None):
    """Contiguous CUDA tensor of dtype npd holding a (ndarray or tensor)."""
    t = torch()
    td = torch_dtype(npd)
    if is_tensor(a) and a.is_cuda and a.dtype == td and a.is_contiguous():
        # already in place: skip the .to() dispatch (hot in fused streaming calls)
        want = device.index if isinstance(device, t.device) else (
            t.device(device).index if device is not None else t._C._cuda_getDevice())
        if a.get_device() == want:
            return a
    dev = device if device is not None else t.device("cuda", t.cuda.current_device())
    if is_tensor(a):
        return a.to(device=dev, dtype=td, non_blocking=a.device.type == "cpu" and a.is_pinned()).contiguous()
    arr = np.ascontiguousarray(a, dtype=npd)
    return t.from_numpy(arr).to(device=dev)


def as_device_many(arrays, npd, device=None):
    """as_device of every array; several host arrays go up in ONE copy
    (packed on the host, split on the device) instead of one small copy each
    (an IR-swap schedule of 19 host IRs: one ~50 us upload, not 19 dispatches)."""
    t = torch()
    td = torch_dtype(npd)
    if arrays and all(isinstance(a, t.Tensor) for a in arrays):
        # fast path: every array already a contiguous CUDA tensor of the right
        # dtype on the target device (an IR schedule held on the device)
        want = device.index if isinstance(device, t.device) else (
            t.device(device).index if device is not None else t._C._cuda_getDevice())
        if all(a.get_device() == want and a.dtype == td and a.is_contiguous() for a in arrays):
            return list(arrays)
    host = [a for a in arrays if not (is_tensor(a) and a.is_cuda)]
    if len(host) < 2 or len(host) != len(arrays) or any(np.ndim(a) == 0 for a in arrays):
        return [as_device(a, npd, device=device) for a in arrays]
    td = torch_dtype(npd)
    shapes = [tuple(a.shape) for a in arrays]
    sizes = [int(np.prod(sh)) for sh in shapes]
    if sum(sizes) * np.dtype(npd).itemsize > (64 << 10) * len(arrays):
        # large arrays: packing costs a host memcpy; one copy each is cheaper
        return [as_device(a, npd, device=device) for a in arrays]
    if all(is_tensor(a) for a in arrays):
        flat = t.empty(sum(sizes), dtype=td, pin_memory=True)
        t.cat([a.reshape(-1).to(td) for a in arrays], out=flat)
    else:
        flat = t.from_numpy(np.concatenate([np.asarray(a, dtype=npd).reshape(-1) for a in arrays]))
    dflat = as_device(flat, npd, device=device)
    return [v.view(sh) for v, sh in zip(t.split(dflat, sizes), shapes)]


PINNED_STREAM_MIN_BYTES = 1 << 24   # pinned host streams this large are pipelined in the library


def host_pipe_chunks() -> int:
    """Runs per pipelined host stream: 0 = the library's choice (2..4 by
    size); SC_HOST_PIPE_CHUNKS overrides (experiments)."""
    import os

    return int(os.environ.get("SC_HOST_PIPE_CHUNKS", "0"))


def pinned_rows(x, npd, channels: int):
    """x as a contiguous [channels, n] pinned CPU tensor of dtype npd when it
    is one (1-D allowed for one channel) and large enough to pipeline, else
    None (the caller takes the device path)."""
    if not (is_tensor(x) and x.device.type == "cpu" and x.is_pinned() and x.is_contiguous()):
        return None
    if x.dtype != torch_dtype(npd) or x.numel() * x.element_size() < PINNED_STREAM_MIN_BYTES:
        return None
    rows = x[None, :] if x.ndim == 1 and channels == 1 else x
    if rows.ndim != 2 or rows.shape[0] != channels or rows.shape[1] == 0:
        return None
    return rows


def like_input(result, *inputs):
    """Return result (a CUDA tensor) in the caller's currency: a CUDA tensor if
    any input was one, a CPU tensor if any input was a tensor, else an ndarray."""
    if any(is_tensor(a) and a.is_cuda for a in inputs):
        return result
    if any(is_tensor(a) for a in inputs):
        if any(is_tensor(a) and a.is_pinned() for a in inputs):
            # pinned in -> pinned out: one DMA at full PCIe/C2C rate
            out = torch().empty(result.shape, dtype=result.dtype, pin_memory=True)
            out.copy_(result, non_blocking=True)
            torch().cuda.current_stream(result.device).synchronize()
            return out
        return result.cpu()
    return result.cpu().numpy()
