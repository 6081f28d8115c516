"""Streaming convolution engine -- drop-in for ``scatterconv.engine``.

Mirrors pkg/src/scatterconv/engine.py (EngineConfig, ScatterEngine with
process_sample / process_block / flush / swap_ir / swap_ir_at_next_block /
render and the ring / read_index / current_ir / samples_consumed
properties).  The state lives on the GPU inside a ``sc_engine`` handle
(csrc/engine.cu): the residue ring (kept in schedule order), the impulse
response copy, ``live``, ``cap`` and ``read_index``.  Blocks and IR swaps
never wait on the host; only calls that must return host data (flush, the
state properties, numpy-in/numpy-out blocks) synchronise.

Arithmetic is the ordered chain (csrc/k_ordered.cu): float64 engines are
bit-identical to the reference, and in both dtypes any block partition
yields the identical stream (block-size invariance, engine.py:7-9).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from operator import is_ as _is

import numpy as np

from . import _dev
from . import _native as N
from .core import Signal

TAIL_POLICIES = ("emit-on-flush", "auto-append")

# Block size sweet spot (engine.py:31-33).
DEFAULT_BLOCK_SIZE = 8192


@dataclass
class EngineConfig:
    """Knobs for a ScatterEngine (engine.py:36-57).

    block_size_nb        upper bound on samples per process_block call
    zero_skip_threshold  inputs with |x| <= threshold scatter nothing
    tail_policy          "auto-append" or "emit-on-flush" (render)
    """

    block_size_nb: int = DEFAULT_BLOCK_SIZE
    zero_skip_threshold: float = 0.0
    tail_policy: str = "emit-on-flush"

    def __post_init__(self):
        if not isinstance(self.block_size_nb, (int, np.integer)) or self.block_size_nb < 1:
            raise ValueError(f"block_size_nb must be >= 1, got {self.block_size_nb!r}")
        if self.zero_skip_threshold < 0:
            raise ValueError(f"zero_skip_threshold must be >= 0, got {self.zero_skip_threshold}")
        if self.tail_policy not in TAIL_POLICIES:
            raise ValueError(f"tail_policy must be one of {TAIL_POLICIES}, got {self.tail_policy!r}")


def _engine_mode(mode, npd) -> bool:
    """True for the FAST engine mode.  Default: FAST for float32 engines
    (tensor cores for large fused streams / blocks), ORDERED for float64
    (bit-identical to the reference).  float64 'fast' = the same chain with
    fused multiply-adds (within 1e-12, twice the FP64 throughput)."""
    if mode not in (None, "fast", "ordered"):
        raise ValueError(f"mode must be 'fast' or 'ordered', got {mode!r}")
    if mode is None:
        return npd == np.float32
    return mode == "fast"


def _signal(samples, sample_rate):
    """A Signal around samples the engine just produced (already 1-D, float,
    in the caller's currency): skips the constructor's coercion and checks."""
    sig = object.__new__(Signal)
    sig.samples = samples
    sig.sample_rate = sample_rate
    return sig


def _is_dev_ir(ir, device, npd) -> bool:
    """An IR the library can read in place: a contiguous CUDA tensor of the
    engine's dtype on its device (a Signal holding one counts)."""
    t = _dev.torch()
    a = ir.samples if isinstance(ir, Signal) else ir
    return (type(a) is t.Tensor and a.is_cuda and a.get_device() == device.index and a.is_contiguous()
            and a.dtype == _dev.torch_dtype(npd))


class ScatterEngine:
    """Stateful block- or sample-driven convolution processor on the GPU.

    One instance is single-threaded; instances are independent (one engine
    per channel, engine.py:60-66).  The engine's dtype is the impulse
    response's (float64 by default, float32 for float32 arrays/tensors).
    """

    def __init__(self, h: Signal, config: EngineConfig | None = None, *, device=None, mode=None):
        if len(h) == 0:
            raise ValueError("impulse response is empty")
        fast = _engine_mode(mode, h.dtype)
        self.config = config if config is not None else EngineConfig()
        t = _dev.torch()
        self._lib = N.lib()
        self._npd = h.dtype
        self._dt = N.dtype_code(self._npd)
        if device is None:
            device = h.samples.device if (_dev.is_tensor(h.samples) and h.samples.is_cuda) else \
                t.device("cuda", t.cuda.current_device())
        self._device = t.device(device)
        if self._device.index is None:
            self._device = t.device("cuda", t.cuda.current_device())
        self._dev_idx = self._device.index
        self._sample_rate = h.sample_rate
        self._ir_like = h.samples[:0]   # currency of returned signals (host / device / pinned)
        self._nh = len(h)
        self._pending_ir = None
        self._handle = ctypes.c_void_p()
        self._stream_val = None
        self._sched_cache = None
        self._stream_fast = None  # see _process_stream_fast
        self._ir_stage = None     # see _stage_irs
        hd = self._to_dev(h.samples)
        with _dev.device_guard(self._device):
            N.check(self._lib.sc_engine_create(self._dt, N.ptr(hd), len(h),
                                               int(self.config.block_size_nb),
                                               float(self.config.zero_skip_threshold),
                                               N.stream_ptr(), ctypes.byref(self._handle)))
            if fast:
                N.check(self._lib.sc_engine_set_mode(self._handle, N.SC_MODE_FAST))
        self.mode = "fast" if fast else "ordered"
        # per-block hot path: bound entry point, raw handle, torch dtype
        self._pb = self._lib.sc_engine_process_block
        self._hv = self._handle.value
        self._td = _dev.torch_dtype(self._npd)

    # ------------------------------------------------------------- plumbing

    def _to_dev(self, samples):
        return _dev.as_device(samples, self._npd, device=self._device)

    def _stage_irs(self, arrs):
        """(device pointer, length) of each IR of a swap schedule, for one
        call.  Host IRs are packed into an engine-owned pinned buffer and go
        up in ONE copy into an engine-owned device buffer, so their device
        addresses are the same on every call (the library's CUDA-graph cache
        keys on them: a render loop with host IRs replays one graph) while the
        data is fresh (edited-in-place IRs are seen).  Device IRs of the
        engine's dtype are read in place; others are converted (kept alive
        in the returned list's third element).  Runs under the engine's
        device guard: events record / wait on the current stream."""
        t = _dev.torch()
        td = _dev.torch_dtype(self._npd)
        ptrs = [0] * len(arrs)
        nhs = [0] * len(arrs)
        keep = []
        host = []
        for i, a in enumerate(arrs):
            if _is_dev_ir(a, self._device, self._npd):
                ptrs[i], nhs[i] = a.data_ptr(), a.shape[0]
            elif _dev.is_tensor(a) and a.is_cuda:
                d = _dev.as_device(a, self._npd, device=self._device)
                keep.append(d)
                ptrs[i], nhs[i] = d.data_ptr(), d.shape[0]
            else:
                host.append(i)
        if not host:
            return ptrs, nhs, keep
        harr = [arrs[i] for i in host]
        sizes = [len(a) for a in harr]
        total = sum(sizes)
        st = self._ir_stage
        if st is None or st[0].numel() < total:
            if st is not None:
                st[2].synchronize()
            st = (t.empty(total, dtype=td, device=self._device), t.empty(total, dtype=td, pin_memory=True),
                  t.cuda.Event(), t.cuda.Event())
            self._ir_stage = st
        dbuf, hbuf, ev_copy, ev_used = st
        ev_copy.synchronize()   # the previous call's upload has left hbuf
        # one packing op where the IRs allow it (the per-IR ops cost ~2 us
        # each in Python): torch.cat for CPU tensors of the engine's dtype,
        # np.concatenate for arrays
        if all(type(a) is t.Tensor and a.dtype == td and a.dim() == 1 and not a.requires_grad for a in harr):
            t.cat(harr, out=hbuf[:total])
        elif all(type(a) is np.ndarray and a.ndim == 1 for a in harr):
            np.concatenate(harr, out=hbuf.numpy()[:total], casting="unsafe")
        else:
            hv = hbuf.numpy()
            off = 0
            for a, n in zip(harr, sizes):
                if _dev.is_tensor(a):
                    a = a.detach().to(td).numpy()
                hv[off:off + n] = np.asarray(a, dtype=self._npd).reshape(-1)
                off += n
        ev_used.wait()   # the current stream: kernels of the previous call are done with dbuf
        dbuf[:total].copy_(hbuf[:total], non_blocking=True)
        ev_copy.record()
        base, es, off = dbuf.data_ptr(), dbuf.element_size(), 0
        for i, n in zip(host, sizes):
            ptrs[i], nhs[i] = base + off * es, n
            off += n
        return ptrs, nhs, keep

    def _staged_irs_used(self, on_dev):
        """Mark the staged IR buffer as read by the work just queued (the next
        call's upload into it waits for that work on the device)."""
        if not on_dev and self._ir_stage is not None:
            self._ir_stage[3].record()

    def _bind_stream(self):
        # the engine queues on the caller's current stream; rebinding only
        # when it changed keeps a ctypes call off the per-block path
        sp = N.stream_ptr().value or 0
        if sp != self._stream_val:
            N.check(self._lib.sc_engine_set_stream(self._handle, sp))
            self._stream_val = sp

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and h.value:
            try:
                self._lib.sc_engine_destroy(h)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            self._handle = ctypes.c_void_p()

    def _state(self):
        ri, live, cap, cons, nh = (ctypes.c_int64() for _ in range(5))
        pend = ctypes.c_int()
        t = _dev.torch()
        with _dev.device_guard(self._device):
            self._bind_stream()
            N.check(self._lib.sc_engine_state(self._handle, ctypes.byref(ri), ctypes.byref(live),
                                              ctypes.byref(cap), ctypes.byref(cons),
                                              ctypes.byref(nh), ctypes.byref(pend)))
        return {"read_index": ri.value, "live": live.value, "cap": cap.value,
                "consumed": cons.value, "nh": nh.value}

    # ----------------------------------------------------------- properties

    @property
    def ring(self) -> np.ndarray:
        """The reference's physical ring (engine.py:83-85): the schedule-order
        residue rotated by read_index.  A host copy."""
        st = self._state()
        sched = self._schedule_order()
        return np.roll(sched, st["read_index"])

    @property
    def read_index(self) -> int:
        return self._state()["read_index"]

    @property
    def current_ir(self) -> Signal:
        """The impulse response in force (engine.py:91-93): read back from the
        engine's own device copy, in the currency of the IR last given."""
        t = _dev.torch()
        with _dev.device_guard(self._device):
            buf = t.empty(self._nh, dtype=_dev.torch_dtype(self._npd), device=self._device)
            n = ctypes.c_int64()
            self._bind_stream()
            N.check(self._lib.sc_engine_current_ir(self._handle, N.ptr(buf), self._nh, ctypes.byref(n)))
        return Signal(_dev.like_input(buf[:n.value], self._ir_like), self._sample_rate)

    @property
    def samples_consumed(self) -> int:
        return self._state()["consumed"]

    @property
    def dtype(self):
        return self._npd

    # ------------------------------------------------------------- streaming

    def process_sample(self, x: float) -> float:
        """Consume one input sample, return the output sample it completes
        (engine.py:99-116; a pending swap is not applied)."""
        t = _dev.torch()
        with _dev.device_guard(self._device):
            xd = t.tensor([x], dtype=_dev.torch_dtype(self._npd), device=self._device)
            out = t.empty(1, dtype=xd.dtype, device=self._device)
            self._bind_stream()
            N.check(self._lib.sc_engine_process_sample(self._handle, N.ptr(xd), N.ptr(out)))
            return float(out.item())

    def process_block(self, block: Signal) -> Signal:
        """Consume a block of at most block_size_nb samples (engine.py:118-146).

        Order of effects as in the reference: pending swap, size check, rate
        check, then the block.  CUDA-tensor blocks return CUDA-tensor output
        without synchronising.
        """
        if self._pending_ir is not None:
            h_new, self._pending_ir = self._pending_ir, None
            self.swap_ir(h_new)
        if block.samples.shape[0] > self.config.block_size_nb:
            raise ValueError(
                f"block of {len(block)} samples exceeds block_size_nb={self.config.block_size_nb}"
            )
        if block.sample_rate != self._sample_rate:
            raise ValueError(
                f"sample rates differ: block {block.sample_rate} Hz vs engine {self._sample_rate} Hz"
            )
        samples = block.samples
        n = samples.shape[0]
        t = _dev.torch()
        C = t._C
        prev = C._cuda_exchangeDevice(self._dev_idx)
        try:
            if (type(samples) is t.Tensor and samples.is_cuda and samples.dtype is self._td
                    and samples.get_device() == self._dev_idx and samples.is_contiguous()):
                xd = samples                  # already in place: the per-block hot path
            else:
                xd = self._to_dev(samples)
            out = t.empty_like(xd)
            if n:
                sp = C._cuda_getCurrentRawStream(self._dev_idx)
                if sp != self._stream_val:
                    N.check(self._lib.sc_engine_set_stream(self._handle, sp))
                    self._stream_val = sp
                rc = self._pb(self._hv, xd.data_ptr(), n, out.data_ptr())
                if rc:
                    N.check(rc)
        finally:
            if prev != self._dev_idx:
                C._cuda_exchangeDevice(prev)
        res = out if samples is xd else _dev.like_input(out, samples)
        return _signal(res, self._sample_rate)

    def flush(self) -> Signal:
        """Emit the pending residue and reset the engine (engine.py:148-161):
        max(len(ir)-1, live) samples in emission order."""
        return self._flush_end(self._flush_begin())

    def _flush_begin(self):
        """Queue the flush's device work (tail copy, state read-back, reset);
        returns the tail buffer for _flush_end (csrc sc_engine_flush_begin)."""
        t = _dev.torch()
        with _dev.device_guard(self._device):
            self._bind_stream()
            cap = ctypes.c_int64()
            N.check(self._lib.sc_engine_tail_bound(self._handle, ctypes.byref(cap)))
            tail = t.empty(cap.value, dtype=_dev.torch_dtype(self._npd), device=self._device)
            N.check(self._lib.sc_engine_flush_begin(self._handle, N.ptr(tail), cap.value))
        return tail

    def _flush_end(self, tail) -> Signal:
        """Wait for the queued flush; the tail is max(len(ir)-1, live) long."""
        n = ctypes.c_int64()
        with _dev.device_guard(self._device):
            N.check(self._lib.sc_engine_flush_end(self._handle, ctypes.byref(n)))
        return Signal(_dev.like_input(tail[:n.value], self._ir_like), self._sample_rate)

    def swap_ir(self, h_new: Signal):
        """Replace the impulse response, effective for the very next sample
        (engine.py:163-186).  Residue keeps its schedule; no host round-trip."""
        if len(h_new) == 0:
            raise ValueError("impulse response is empty")
        if h_new.sample_rate != self._sample_rate:
            raise ValueError(
                f"sample rates differ: new impulse response {h_new.sample_rate} Hz "
                f"vs engine {self._sample_rate} Hz"
            )
        t = _dev.torch()
        with _dev.device_guard(self._device):
            hd = self._to_dev(h_new.samples)
            self._bind_stream()
            N.check(self._lib.sc_engine_swap_ir(self._handle, N.ptr(hd), len(h_new)))
        self._ir_like = h_new.samples[:0]
        self._nh = len(h_new)

    def swap_ir_at_next_block(self, h_new: Signal):
        """Defer the swap to the start of the next process_block call (engine.py:188-192)."""
        if len(h_new) == 0:
            raise ValueError("impulse response is empty")
        self._pending_ir = h_new

    def render(self, e: Signal) -> Signal:
        """Run a whole signal through in blocks (engine.py:194-209)."""
        nb = self.config.block_size_nb
        parts = []
        for start in range(0, len(e), nb):
            chunk = Signal(e.samples[start:start + nb], e.sample_rate)
            parts.append(self.process_block(chunk).samples)
        if _dev.is_tensor(e.samples):
            t = _dev.torch()
            body = t.cat(parts) if parts else e.samples[:0].to(_dev.torch_dtype(self._npd))
            if self.config.tail_policy == "auto-append":
                body = t.cat([body, self.flush().samples.to(body.device)])
        else:
            body = np.concatenate(parts) if parts else np.empty(0, dtype=self._npd)
            if self.config.tail_policy == "auto-append":
                body = np.concatenate([body, self.flush().samples])
        return Signal(body, self._sample_rate)

    def _schedule_order(self) -> np.ndarray:
        """Ring contents reordered so index 0 is the next slot to emit (engine.py:211-214)."""
        t = _dev.torch()
        with _dev.device_guard(self._device):
            st = self._state()
            buf = t.empty(max(st["cap"], 1), dtype=_dev.torch_dtype(self._npd), device=self._device)
            n = ctypes.c_int64()
            N.check(self._lib.sc_engine_schedule(self._handle, N.ptr(buf), st["cap"],
                                                 ctypes.byref(n)))
            return buf[:n.value].cpu().numpy()

    # ------------------------------------------------------ device-side extras

    def process_stream(self, x, nb: int | None = None, swaps=()):
        """Back-to-back blocks of `nb` samples with an IR-swap schedule, queued
        without host synchronisation (one C call; csrc/engine.cu).

        ``swaps`` is a sequence of (block_index, impulse_response) pairs: the
        swap_ir happens right before that block.  Ordered mode (float64
        always): bit-identical to calling swap_ir/process_block in the same
        order.  Float32 'fast' mode (the float32 default): when every IR
        segment carries >= 2^30 MACs, each segment is convolved on the
        tensor-core FIR path and the segments plus the residue are combined --
        within the FP32 tolerance of the ordered result, same engine state.
        Returns the body (device tensor if x is a CUDA tensor, else ndarray).
        """
        nb = self.config.block_size_nb if nb is None else int(nb)
        fp = self._stream_fast
        if fp is not None and self._pending_ir is None:
            out = self._process_stream_fast(fp, x, nb, swaps)
            if out is not None:
                return out
        if nb < 1 or nb > self.config.block_size_nb:
            raise ValueError(f"nb must be in [1, block_size_nb={self.config.block_size_nb}]")
        t = _dev.torch()
        with _dev.device_guard(self._device):
            xs = x.samples if isinstance(x, Signal) else x
            n_blocks = -(-len(xs) // nb)
            pending = None
            if self._pending_ir is not None and n_blocks:
                # the deferred swap acts before block 0, after any explicit
                # block-0 swap (as swap_ir + process_block would order them):
                # the library places it (csrc/engine.cu process_blocks_impl)
                pending, self._pending_ir = self._pending_ir, None
                if pending.sample_rate != self._sample_rate:
                    raise ValueError(
                        f"sample rates differ: new impulse response {pending.sample_rate} Hz "
                        f"vs engine {self._sample_rate} Hz"
                    )
                pd = self._to_dev(pending.samples)
                self._bind_stream()
                N.check(self._lib.sc_engine_swap_ir_at_next_block(self._handle, N.ptr(pd), len(pending)))
            # The prepared schedule (sorted, on the device, as C arrays) is
            # reused while the caller passes the same IR objects at the same
            # blocks -- a render loop replaying one schedule pays no
            # per-swap Python (the cache keeps the objects alive, so their
            # identities cannot be recycled).  Only for schedules whose IRs
            # are all device tensors (the library reads them in place): host
            # IRs are uploaded again on every call, so an IR edited in place
            # between calls is seen, as the reference reads it per call.
            if not isinstance(swaps, (list, tuple)):
                swaps = list(swaps)
            on_dev = all(_is_dev_ir(s[1], self._device, self._npd) for s in swaps)
            sig = (n_blocks, tuple((s[0], id(s[1])) for s in swaps)) if on_dev else None
            cached = self._sched_cache
            if sig is not None and cached is not None and cached[0] == sig:
                swaps, irs, blocks, ptrs, nhs, n = cached[1]
            else:
                keep = list(swaps)
                # swaps outside [0, n_blocks) precede no block: the library ignores them
                swaps = sorted((s for s in keep if 0 <= int(s[0]) < n_blocks), key=lambda s: s[0])
                arrs = [s[1].samples if isinstance(s[1], Signal) else s[1] for s in swaps]
                if on_dev:
                    irs = arrs
                    p_list, n_list = [ir.data_ptr() for ir in irs], [ir.shape[0] for ir in irs]
                else:
                    p_list, n_list, irs = self._stage_irs(arrs)
                n = len(swaps)
                blocks = (ctypes.c_int64 * max(n, 1))(*[int(s[0]) for s in swaps])
                ptrs = (ctypes.c_void_p * max(n, 1))(*p_list)
                nhs = (ctypes.c_int64 * max(n, 1))(*n_list)
                # host schedules are staged again on the next call: nothing to keep
                self._sched_cache = (sig, (swaps, irs, blocks, ptrs, nhs, n), keep) if on_dev else None
            self._bind_stream()
            xh = _dev.pinned_rows(xs, self._npd, 1)
            if xh is not None:
                # large pinned host stream: transfers overlap the blocks run by
                # run inside the library (sc_engine_process_blocks_host)
                out = t.empty(xh.shape[1], dtype=xh.dtype, pin_memory=True)
                N.check(self._lib.sc_engine_process_blocks_host(self._handle, N.ptr(xh), xh.shape[1], nb,
                                                                blocks, ptrs, nhs, n, N.ptr(out), _dev.host_pipe_chunks()))
                self._staged_irs_used(on_dev)
                self._note_swaps(swaps, pending)
                return out
            xd = self._to_dev(xs)
            out = xd.new_empty(xd.shape[0])
            rc = self._lib.sc_engine_process_blocks(self._handle, xd.data_ptr(), xd.shape[0], nb, blocks, ptrs,
                                                    nhs, n, out.data_ptr())
            if rc:
                N.check(rc)
            self._staged_irs_used(on_dev)
            self._note_swaps(swaps, pending)
            if xd is xs and pending is None and type(xs) is t.Tensor and xs.dim() == 1 and on_dev:
                # args[1] keeps the device IRs (and the C arrays) alive
                self._stream_fast = (nb, xs.shape[0], xs.dtype, self._device.index, self._sched_cache[2],
                                     self._sched_cache[1], (self._ir_like, self._nh) if swaps else None)
        return out if xd is xs else _dev.like_input(out, xs)

    def _process_stream_fast(self, fp, x, nb, swaps):
        """process_stream's repeat call: the same device tensor shape and
        dtype, the same nb and the same swap schedule (the very same
        (block, IR) tuples as the call that built the cached C arrays), no
        pending swap, on the same device and stream -- straight to the C call
        (~3 us of Python instead of ~12: the fused stream's GPU work starts
        that much earlier).  None when any of it differs."""
        f_nb, f_len, f_dtype, f_dev, f_keep, args, note = fp
        t = _dev.torch()
        if (nb != f_nb or type(x) is not t.Tensor or type(swaps) not in (list, tuple)
                or x.dtype is not f_dtype or x.dim() != 1
                or x.shape[0] != f_len or not x.is_cuda or x.get_device() != f_dev or not x.is_contiguous()
                or len(swaps) != len(f_keep) or not all(map(_is, swaps, f_keep))):
            return None
        C = t._C
        if C._cuda_getDevice() != f_dev or C._cuda_getCurrentRawStream(f_dev) != self._stream_val:
            return None
        _, _, blocks, ptrs, nhs, n = args
        out = x.new_empty(f_len)
        rc = self._lib.sc_engine_process_blocks(self._handle, x.data_ptr(), f_len, f_nb, blocks, ptrs, nhs, n,
                                                out.data_ptr())
        if rc:
            N.check(rc)
        if note is not None:
            self._ir_like, self._nh = note
        return out

    def _note_swaps(self, swaps, pending=None):
        """Host copy of the IR now in effect: the last swap of the timeline,
        where a pending IR follows the block-0 swaps."""
        last = swaps[-1][1] if swaps else None
        if pending is not None and (not swaps or int(swaps[-1][0]) == 0):
            last = pending
        if last is not None:
            last = last.samples if isinstance(last, Signal) else last
            self._ir_like = last[:0]
            self._nh = len(last)

    def state_dict(self) -> dict:
        """Snapshot for tests/checkpointing: ring, schedule, read_index, live, consumed."""
        st = self._state()
        sched = self._schedule_order()
        return {"read_index": st["read_index"], "ring": np.roll(sched, st["read_index"]),
                "consumed": st["consumed"], "live": st["live"], "sched": sched}
