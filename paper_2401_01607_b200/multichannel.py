"""Batched multichannel convolution (north_star (3)).

The reference has no batched path: it runs one ScatterEngine per channel,
sequentially in the CLI (cli.py:186-202) or on a thread pool in the bench
(bench.py:200-202), relying on the nogil kernel (engine.py:60-66).  Here all
channels go through ONE launch of the register-tiled FP32 kernel
(grid.z = channel), each channel with its own impulse response.
"""

from __future__ import annotations

import numpy as np

from . import _dev
from . import _native as N


def convolve_batched(x, h, mode=None):
    """y[c] = x[c] (*) h[c] for all channels in one launch.

    x: [C, Ne] float32 (ndarray or tensor), h: [C, Nh] float32 (or [Nh],
    broadcast to every channel like the CLI's mono IR, cli.py:147-155).
    Returns [C, Ne+Nh-1] float32 in the caller's currency.  A large pinned
    host input streams channel groups through upload / FIR / download on
    three overlapping streams (pinned host output).
    """
    t = _dev.torch()
    if x.ndim != 2:
        raise ValueError(f"x must be [channels, samples], got shape {tuple(x.shape)}")
    C, ne = int(x.shape[0]), int(x.shape[1])
    if ne == 0:
        raise ValueError("input signal is empty")
    pinned_in = _dev.is_tensor(x) and x.device.type == "cpu" and x.is_pinned()
    dev = t.device("cuda", t.cuda.current_device())
    xd = None if pinned_in else _dev.as_device(x, np.float32)
    hd = _dev.as_device(h, np.float32, device=xd.device if xd is not None else dev)
    if hd.ndim == 1:
        hd = hd.unsqueeze(0).expand(C, -1).contiguous()
    if hd.shape[0] != C:
        raise ValueError(f"h has {hd.shape[0]} channels, x has {C}")
    nh = int(hd.shape[1])
    if nh == 0:
        raise ValueError("impulse response is empty")
    from .core import mode_code

    L = N.lib()
    if (_dev.is_tensor(x) and x.device.type == "cpu" and x.is_pinned() and x.dtype == t.float32
            and x.is_contiguous() and mode_code(mode) != N.SC_MODE_ORDERED and C >= 2
            and C * ne * nh >= _PIPELINE_MIN_MACS):
        return _batched_host_pipelined(x, hd, mode_code(mode))
    if xd is None:
        xd = _dev.as_device(x, np.float32, device=hd.device)
    with t.cuda.device(xd.device):
        y = t.empty((C, ne + nh - 1), dtype=t.float32, device=xd.device)
        N.check(L.sc_fir_batched(N.SC_F32, mode_code(mode), N.ptr(xd), ne, N.ptr(hd), nh, N.ptr(y),
                                 ne + nh - 1, C,
                                 ne, nh, N.stream_ptr()))
    return _dev.like_input(y, x, h)


_PIPELINE_MIN_MACS = 1 << 34   # pinned-host batches this large overlap H2D / FIR / D2H


def _batched_host_pipelined(x_pin, hd, mode):
    """Pinned-host [C, Ne] input: channel groups flow through upload, FIR and
    download on three streams (event-chained), so the PCIe/C2C transfers of
    one group overlap the tensor-core work of another.  Returns a pinned host
    [C, Ne+Nh-1] tensor."""
    from .core import pipe_streams

    t = _dev.torch()
    L = N.lib()
    dev = hd.device
    C, ne = int(x_pin.shape[0]), int(x_pin.shape[1])
    nh = int(hd.shape[1])
    nout = ne + nh - 1
    out = t.empty((C, nout), dtype=t.float32, pin_memory=True)
    with t.cuda.device(dev):
        xd = t.empty((C, ne), dtype=t.float32, device=dev)
        yd = t.empty((C, nout), dtype=t.float32, device=dev)
        main = t.cuda.current_stream(dev)
        s_in, s_cmp, s_out = pipe_streams(dev)
        for s in (s_in, s_cmp, s_out):
            s.wait_stream(main)
        groups = max(2, min(C, 8, (C * ne * nh) >> 35))
        per = -(-C // groups)
        for c0 in range(0, C, per):
            c1 = min(C, c0 + per)
            with t.cuda.stream(s_in):
                xd[c0:c1].copy_(x_pin[c0:c1], non_blocking=True)
            s_cmp.wait_stream(s_in)
            N.check(L.sc_fir_batched(N.SC_F32, mode, N.ptr(xd[c0]), ne, N.ptr(hd[c0]), nh, N.ptr(yd[c0]), nout,
                                     c1 - c0, ne, nh, N.stream_ptr(s_cmp)))
            s_out.wait_stream(s_cmp)
            with t.cuda.stream(s_out):
                out[c0:c1].copy_(yd[c0:c1], non_blocking=True)
        s_out.synchronize()
    return out


class MultiChannelEngine:
    """C streaming engines that advance together, one per channel.

    The reference runs one ``ScatterEngine`` per channel and loops over them
    (engine.py:60-66; the CLI's per-channel loop, cli.py:186-202, with the
    mono-IR broadcast of cli.py:147-155).  Here all channels share one
    device engine: one launch per block for every channel, each channel with
    its own residue, ``live``, ``cap`` and ``read_index`` (SURVEY.md 8(f)
    row 1).  Semantics per channel are exactly ``ScatterEngine``'s
    (bit-identical in float64).

    h: [C, Nh] (or [Nh] with ``channels=C`` to broadcast a mono IR).
    Blocks are [C, n] arrays/tensors; outputs come back in the same currency.
    """

    def __init__(self, h, config=None, *, channels=None, device=None, mode=None):
        import ctypes

        from .engine import EngineConfig, _engine_mode

        t = _dev.torch()
        self.config = config if config is not None else EngineConfig()
        hd = h if _dev.is_tensor(h) else np.asarray(h)
        npd = _dev.np_dtype(hd) if (_dev.is_tensor(hd) or hd.dtype in (np.float32, np.float64)) else np.float64
        if hd.ndim == 1:
            if channels is None:
                raise ValueError("a 1-D impulse response needs channels=C to broadcast")
            hd = hd[None, :].repeat(channels, 0) if not _dev.is_tensor(hd) else hd[None, :].expand(channels, -1)
        if hd.shape[-1] == 0:
            raise ValueError("impulse response is empty")
        self._npd = npd
        fast = _engine_mode(mode, npd)
        self._dt = N.dtype_code(npd)
        self._device = t.device(device) if device is not None else t.device("cuda", t.cuda.current_device())
        self._lib = N.lib()
        self._C = int(hd.shape[0])
        self._pending = None
        h_dev = _dev.as_device(hd, npd, device=self._device).contiguous()
        self._handle = ctypes.c_void_p()
        with _dev.device_guard(self._device):
            N.check(self._lib.sc_engine_create_multi(self._dt, N.ptr(h_dev), h_dev.shape[1], self._C,
                                                     int(self.config.block_size_nb),
                                                     float(self.config.zero_skip_threshold),
                                                     N.stream_ptr(), ctypes.byref(self._handle)))
            if fast:
                N.check(self._lib.sc_engine_set_mode(self._handle, N.SC_MODE_FAST))
        self.mode = "fast" if fast else "ordered"

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and h.value:
            try:
                self._lib.sc_engine_destroy(h)
            except Exception:  # pragma: no cover
                pass
            self._handle = None

    @property
    def channels(self) -> int:
        return self._C

    def _bind(self):
        N.check(self._lib.sc_engine_set_stream(self._handle, N.stream_ptr()))

    def _rows(self, a, n_expected=None):
        d = _dev.as_device(a, self._npd, device=self._device)
        if d.ndim == 1 and self._C == 1:
            d = d[None, :]
        if d.ndim != 2 or d.shape[0] != self._C:
            raise ValueError(f"expected [channels={self._C}, n] samples, got shape {tuple(d.shape)}")
        return d.contiguous()

    def _ir_rows(self, h):
        hd = h if _dev.is_tensor(h) else np.asarray(h)
        if hd.ndim == 1:
            hd = hd[None, :].repeat(self._C, 0) if not _dev.is_tensor(hd) else hd[None, :].expand(self._C, -1)
        if hd.shape[-1] == 0:
            raise ValueError("impulse response is empty")
        return self._rows(hd)

    def _ir_rows_many(self, hs):
        """_ir_rows of a swap schedule, uploaded together (_dev.as_device_many)."""
        rows = []
        for h in hs:
            hd = h if _dev.is_tensor(h) else np.asarray(h)
            if hd.ndim == 1:
                hd = hd[None, :].expand(self._C, -1) if _dev.is_tensor(hd) else np.repeat(hd[None, :], self._C, 0)
            if hd.shape[-1] == 0:
                raise ValueError("impulse response is empty")
            rows.append(hd)
        return [self._rows(d) for d in _dev.as_device_many(rows, self._npd, device=self._device)]

    def process_block(self, block):
        """[C, n] in, [C, n] out (engine.py:118-146 per channel)."""
        t = _dev.torch()
        if self._pending is not None:
            h_new, self._pending = self._pending, None
            self.swap_ir(h_new)
        with _dev.device_guard(self._device):
            xd = self._rows(block)
            n = xd.shape[1]
            if n > self.config.block_size_nb:
                raise ValueError(f"block of {n} samples exceeds block_size_nb={self.config.block_size_nb}")
            out = t.empty_like(xd)
            if n:
                self._bind()
                N.check(self._lib.sc_engine_process_block(self._handle, N.ptr(xd), n, N.ptr(out)))
        return _dev.like_input(out, block)

    def process_sample(self, x):
        """One sample per channel ([C]) -> [C] outputs (engine.py:99-116)."""
        t = _dev.torch()
        with _dev.device_guard(self._device):
            xd = _dev.as_device(np.asarray(x, dtype=self._npd).reshape(self._C, 1), self._npd, device=self._device)
            out = t.empty_like(xd)
            self._bind()
            N.check(self._lib.sc_engine_process_sample(self._handle, N.ptr(xd), N.ptr(out)))
            return out[:, 0].cpu().numpy()

    def swap_ir(self, h_new):
        """Every channel swaps to its row of h_new (or a broadcast mono IR)."""
        t = _dev.torch()
        with _dev.device_guard(self._device):
            hd = self._ir_rows(h_new)
            self._bind()
            N.check(self._lib.sc_engine_swap_ir(self._handle, N.ptr(hd), hd.shape[1]))

    def swap_ir_at_next_block(self, h_new):
        self._ir_rows(h_new)  # validate now (engine.py:188-192)
        self._pending = h_new

    def flush(self, *, on_device: bool = False):
        """Per-channel tails (max(len(ir)-1, live_c) samples each) as a list of
        host arrays; with on_device=True, (tails [C, max_len] CUDA tensor,
        lengths) instead -- no device-to-host copy (row c is valid up to
        lengths[c], zero beyond)."""
        import ctypes

        t = _dev.torch()
        with _dev.device_guard(self._device):
            self._bind()
            cap = ctypes.c_int64()
            N.check(self._lib.sc_engine_tail_bound(self._handle, ctypes.byref(cap)))
            tail = t.empty((self._C, cap.value), dtype=_dev.torch_dtype(self._npd), device=self._device)
            n = (ctypes.c_int64 * self._C)()
            N.check(self._lib.sc_engine_flush(self._handle, N.ptr(tail), cap.value, n))
            if on_device:
                lengths = list(n)
                return tail[:, :max(lengths, default=0)], lengths
            host = tail.cpu().numpy()
        return [host[c, :n[c]].copy() for c in range(self._C)]

    def state(self) -> dict:
        import ctypes

        C = self._C
        ri, live, cap = (ctypes.c_int64 * C)(), (ctypes.c_int64 * C)(), (ctypes.c_int64 * C)()
        cons, nh = ctypes.c_int64(), ctypes.c_int64()
        pend = ctypes.c_int()
        t = _dev.torch()
        with _dev.device_guard(self._device):
            self._bind()
            N.check(self._lib.sc_engine_state(self._handle, ri, live, cap, ctypes.byref(cons), ctypes.byref(nh),
                                              ctypes.byref(pend)))
        return {"read_index": list(ri), "live": list(live), "cap": list(cap), "consumed": cons.value,
                "nh": nh.value}

    def process_stream(self, x, nb=None, swaps=()):
        """[C, N] through back-to-back blocks of nb with an IR-swap schedule
        ((block_index, IR) pairs, applied to every channel) in one fused
        launch per <= 31 swaps; bit-identical to the block-by-block calls in
        ordered mode (float32 'fast' mode: tensor cores for large segments, see
        ScatterEngine.process_stream)."""
        import ctypes

        t = _dev.torch()
        nb = self.config.block_size_nb if nb is None else int(nb)
        if nb < 1 or nb > self.config.block_size_nb:
            raise ValueError(f"nb must be in [1, block_size_nb={self.config.block_size_nb}]")
        n_total = x.shape[-1]
        n_blocks = -(-n_total // nb)
        with _dev.device_guard(self._device):
            if self._pending is not None and n_blocks:
                # after any explicit block-0 swap, as process_block orders it;
                # the library places it (csrc/engine.cu process_blocks_impl)
                pd, self._pending = self._ir_rows(self._pending), None
                self._bind()
                N.check(self._lib.sc_engine_swap_ir_at_next_block(self._handle, N.ptr(pd), pd.shape[1]))
            # swaps outside [0, n_blocks) precede no block: the library ignores them
            swaps = sorted((s for s in swaps if 0 <= int(s[0]) < n_blocks), key=lambda s: s[0])
            irs = self._ir_rows_many([s[1] for s in swaps])
            k = len(swaps)
            blocks = (ctypes.c_int64 * max(k, 1))(*[int(s[0]) for s in swaps])
            ptrs = (ctypes.c_void_p * max(k, 1))(*[ir.data_ptr() for ir in irs])
            nhs = (ctypes.c_int64 * max(k, 1))(*[ir.shape[1] for ir in irs])
            self._bind()
            xh = _dev.pinned_rows(x, self._npd, self._C)
            if xh is not None:
                # large pinned host stream: uploads / blocks / downloads overlap
                # run by run inside the library (sc_engine_process_blocks_host)
                out = t.empty(xh.shape, dtype=xh.dtype, pin_memory=True)
                N.check(self._lib.sc_engine_process_blocks_host(self._handle, N.ptr(xh), xh.shape[1], nb, blocks,
                                                                ptrs, nhs, k, N.ptr(out), _dev.host_pipe_chunks()))
                return out
            xd = self._rows(x)
            out = t.empty_like(xd)
            N.check(self._lib.sc_engine_process_blocks(self._handle, N.ptr(xd), xd.shape[1], nb, blocks, ptrs,
                                                       nhs, k, N.ptr(out)))
        return _dev.like_input(out, x)
