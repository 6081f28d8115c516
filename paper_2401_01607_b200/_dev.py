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


def as_device(a, npd, device=None):
    """Contiguous CUDA tensor of dtype npd holding a (ndarray or tensor)."""
    t = torch()
    td = torch_dtype(npd)
    if is_tensor(a) and a.is_cuda and a.dtype == td and a.is_contiguous():
        # already in place: skip the .to() dispatch (hot in fused streaming calls)
        want = t.device(device).index if device is not None else t.cuda.current_device()
        if a.device.index == want:
            return a
    dev = device if device is not None else t.device("cuda", t.cuda.current_device())
    if is_tensor(a):
        return a.to(device=dev, dtype=td, non_blocking=a.device.type == "cpu" and a.is_pinned()).contiguous()
    arr = np.ascontiguousarray(a, dtype=npd)
    return t.from_numpy(arr).to(device=dev)


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
