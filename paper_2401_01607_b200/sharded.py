"""Time-sharded convolution of long signals across GPUs (north_star (4);
SURVEY.md 8(e)).

The full output [0, Ne+Nh-1) is cut into equal contiguous segments, one per
GPU.  GPU g owning outputs [a, b) needs inputs [max(0, a-Nh+1), min(Ne, b)):
its slice plus an (Nh-1)-sample halo.  Partitioning by OUTPUT means no MAC is
done twice and no partial sums cross GPUs: results simply concatenate, so
the data path has no collective.  A device-side gather (NCCL send/recv via
torch.distributed) is only used when a caller asks for the whole result on
one rank.

Two drivers:
  * ``convolve_sharded``      one process, one host thread per local GPU
  * ``distributed_convolve``  one process per GPU (torchrun), the bench path
"""

from __future__ import annotations

import threading
from dataclasses import dataclass

import numpy as np

from . import _dev
from . import _native as N


@dataclass(frozen=True)
class Shard:
    rank: int
    n_begin: int   # outputs [n_begin, n_end)
    n_end: int
    x_begin: int   # inputs [x_begin, x_end) incl. the halo
    x_end: int

    @property
    def n_out(self) -> int:
        return self.n_end - self.n_begin

    @property
    def n_in(self) -> int:
        return self.x_end - self.x_begin

    def macs(self, nh: int) -> int:
        """Metric MACs (out samples x taps) owned by this shard."""
        return self.n_out * nh


def shard_plan(ne: int, nh: int, world: int) -> list[Shard]:
    """Equal contiguous output segments with their input halos."""
    if ne < 1 or nh < 1 or world < 1:
        raise ValueError("need ne >= 1, nh >= 1, world >= 1")
    nout = ne + nh - 1
    per = -(-nout // world)
    plan = []
    for g in range(world):
        a = min(g * per, nout)
        b = min(a + per, nout)
        xb = max(0, a - nh + 1)
        xe = max(xb, min(ne, b))
        plan.append(Shard(g, a, b, xb, xe))
    return plan


def convolve_shard(x_slice, shard: Shard, h, mode=None):
    """Compute one shard on the current device: x_slice holds inputs
    [shard.x_begin, shard.x_end) (CUDA float32), h the taps (CUDA float32).
    Returns the shard's outputs [n_begin, n_end) as a CUDA tensor.
    mode: None/"fast" (kernel chosen by shape), "ffma" or "tc"."""
    from .core import mode_code

    t = _dev.torch()
    L = N.lib()
    y = t.empty(shard.n_out, dtype=t.float32, device=h.device)
    if shard.n_out:
        N.check(L.sc_fir_range(N.SC_F32, mode_code(mode), N.ptr(x_slice) if x_slice.numel() else None,
                               shard.x_begin, shard.x_end, N.ptr(h), h.shape[0], N.ptr(y),
                               shard.n_begin, shard.n_end, N.stream_ptr()))
    return y


def convolve_sharded(x, h, devices=None, gather: str | None = "host"):
    """Single-process multi-GPU driver: one host thread per device.

    x: host float32 [Ne] (pinned internally), h: float32 [Nh].  Each thread
    uploads its slice+halo, runs ``sc_fir_range`` and keeps its segment on
    its device.  gather="host" returns the concatenated ndarray,
    gather=None returns the per-device tensors, gather="cuda:K" concatenates
    on device K (peer copies over NVLink).
    """
    t = _dev.torch()
    devices = list(devices) if devices is not None else list(range(t.cuda.device_count()))
    x = np.ascontiguousarray(x, dtype=np.float32)
    h = np.ascontiguousarray(h, dtype=np.float32)
    plan = shard_plan(len(x), len(h), len(devices))
    xt = t.from_numpy(x).pin_memory()
    outs = [None] * len(devices)
    errors = []

    def work(i):
        try:
            dev = t.device("cuda", devices[i])
            with t.cuda.device(dev):
                sh = plan[i]
                xs = xt[sh.x_begin:sh.x_end].to(dev, non_blocking=True)
                hd = t.from_numpy(h).to(dev)
                outs[i] = convolve_shard(xs, sh, hd)
                t.cuda.current_stream(dev).synchronize()
        except Exception as exc:  # pragma: no cover - surfaced below
            errors.append(exc)

    threads = [threading.Thread(target=work, args=(i,)) for i in range(len(devices))]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    if errors:
        raise errors[0]
    if gather is None:
        return outs
    if gather == "host":
        return np.concatenate([o.cpu().numpy() for o in outs])
    dst = t.device(gather)
    return t.cat([o.to(dst) for o in outs])


def _pinned_1d(a, npd):
    """A contiguous pinned host tensor holding a (host array or tensor): the
    caller's own tensor when it already is one, else one staging copy (the
    library's transfers only overlap from pinned memory)."""
    t = _dev.torch()
    td = _dev.torch_dtype(npd)
    if _dev.is_tensor(a):
        if a.device.type == "cpu" and a.is_pinned() and a.dtype == td and a.is_contiguous():
            return a
        return a.detach().to(device="cpu", dtype=td).contiguous().pin_memory()
    return t.from_numpy(np.ascontiguousarray(a, dtype=npd)).pin_memory()


def fir_sharded(x, h, devices=None, *, mode=None, gather_device=None):
    """The C-ABI multi-GPU entry (``sc_fir_sharded``): host x [Ne] and h [Nh]
    (float32 or float64), outputs partitioned over ``devices`` (repeats
    allowed); each device runs the chunk-pipelined range engine (upload /
    FIR / download overlapped, persistent buffers) on its own native host
    thread.  Returns the full Ne+Nh-1 result in pinned host memory (a tensor
    when x is a tensor, else an ndarray view of it), or as a CUDA tensor on
    ``gather_device`` (filled by the shards' peer stores).  mode as
    ``scatter_convolve``: float64 defaults to ORDERED, bit-identical to the
    reference at any device count."""
    import ctypes

    from .core import _MODES, _result_dtype

    t = _dev.torch()
    devices = list(devices) if devices is not None else list(range(t.cuda.device_count()))
    npd = _result_dtype(x, h)
    if np.ndim(x) != 1 or np.ndim(h) != 1:
        raise ValueError("x and h must be 1-D")
    if len(x) == 0:
        raise ValueError("input signal is empty")
    if len(h) == 0:
        raise ValueError("impulse response is empty")
    if mode not in _MODES:
        raise ValueError(f"mode must be one of {sorted(k for k in _MODES if k)}, got {mode!r}")
    m = _MODES[mode]
    if m is None:
        m = N.SC_MODE_FAST if npd == np.float32 else N.SC_MODE_ORDERED
    xp = _pinned_1d(x, npd)
    hp = _pinned_1d(h, npd)
    nout = xp.shape[0] + hp.shape[0] - 1
    if gather_device is None:
        y = t.empty(nout, dtype=_dev.torch_dtype(npd), pin_memory=True)
        gd = -1
    else:
        gd = t.device(gather_device).index if not isinstance(gather_device, int) else gather_device
        y = t.empty(nout, dtype=_dev.torch_dtype(npd), device=t.device("cuda", gd))
        # the shards store from their own streams: the allocation (and any
        # earlier use of this memory) on the gather device's stream is done first
        t.cuda.current_stream(y.device).synchronize()
    devs = (ctypes.c_int * len(devices))(*devices)
    N.check(N.lib().sc_fir_sharded(N.dtype_code(npd), m, N.ptr(xp), xp.shape[0], N.ptr(hp), hp.shape[0],
                                   N.ptr(y), len(devices), devs, gd))
    if gather_device is None and not _dev.is_tensor(x):
        return y.numpy()
    return y


def distributed_convolve(x, h, *, rank=None, world=None, compute=None, device=None,
                         to_host=False):
    """One shard per process (torchrun / torch.distributed initialised).

    x: the FULL input on the host (ndarray, or a CPU tensor -- pinned tensors
    upload asynchronously); each rank uploads only its slice + halo.  h: taps.
    Returns (shard, y_local): y_local on this rank's device, or in pinned host
    memory with ``to_host=True``.  ``compute(x_slice, shard, h) -> y``
    defaults to the CUDA kernel; tests inject the CPU oracle to check the
    partition and gather logic under gloo.  No collective touches the data.
    """
    import torch.distributed as dist

    rank = dist.get_rank() if rank is None else rank
    world = dist.get_world_size() if world is None else world
    plan = shard_plan(len(x), len(h), world)
    sh = plan[rank]
    if compute is not None:
        return sh, compute(x[sh.x_begin:sh.x_end], sh, h)
    t = _dev.torch()
    dev = device if device is not None else t.device("cuda", t.cuda.current_device())
    dev = t.device(dev)
    if to_host:
        # the chunk-pipelined range engine: this rank's slice + halo goes up
        # chunk by chunk, overlapped with the FIR and the download of the
        # outputs into pinned host memory (csrc/sharded.cu sc_fir_range_host)
        xp = _pinned_1d(x, np.float32)
        hp = _dev.as_device(h, np.float32, device=dev) if _dev.is_tensor(h) and h.is_cuda else _pinned_1d(h, np.float32)
        y = t.empty(sh.n_out, dtype=t.float32, pin_memory=True)
        if sh.n_out:
            N.check(N.lib().sc_fir_range_host(N.SC_F32, N.SC_MODE_FAST, N.ptr(xp), xp.shape[0], N.ptr(hp),
                                              hp.shape[0], N.ptr(y), sh.n_begin, sh.n_end, dev.index, 0))
        return sh, y
    with t.cuda.device(dev):
        xs = _dev.as_device(x[sh.x_begin:sh.x_end], np.float32, device=dev)
        hd = _dev.as_device(h, np.float32, device=dev)
        y = convolve_shard(xs, sh, hd)
        return sh, y


def gather_shards(y_local, shard: Shard, plan_len: int, dst: int = 0):
    """Concatenate every rank's segment on rank `dst` (send/recv; NCCL on GPU,
    gloo on CPU).  Returns the full output on dst, None elsewhere.  This is
    the only collective and it is optional (north_star (4))."""
    import torch.distributed as dist

    t = _dev.torch()
    rank = dist.get_rank()
    world = dist.get_world_size()
    sizes = t.tensor([shard.n_out], dtype=t.int64, device=y_local.device)
    all_sizes = [t.zeros_like(sizes) for _ in range(world)]
    dist.all_gather(all_sizes, sizes)
    if rank != dst:
        dist.send(y_local.contiguous(), dst)
        return None
    parts = []
    for r in range(world):
        if r == rank:
            parts.append(y_local)
        else:
            buf = t.empty(int(all_sizes[r].item()), dtype=y_local.dtype, device=y_local.device)
            dist.recv(buf, r)
            parts.append(buf)
    return t.cat(parts)
