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
        ragged = None
        if isinstance(h, (list, tuple)):
            # one IR per channel, lengths may differ (one engine per channel)
            if channels is not None and channels != len(h):
                raise ValueError(f"{len(h)} impulse responses for channels={channels}")
            ragged = list(h)
            npd0 = (np.float32 if all(_dev.np_dtype(a) == np.float32 for a in ragged
                                      if _dev.is_tensor(a) or np.asarray(a).dtype in (np.float32, np.float64))
                    else np.float64)
            if any(len(a) == 0 for a in ragged):
                raise ValueError("impulse response is empty")
            h = np.zeros((len(ragged), max(len(a) for a in ragged)), dtype=npd0)
            for c, a in enumerate(ragged):
                h[c, :len(a)] = a.cpu().numpy() if _dev.is_tensor(a) else np.asarray(a)
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
        if ragged is not None and len({len(a) for a in ragged}) > 1:
            # channels start on IRs of their own lengths: a per-channel swap on
            # the fresh state is exactly a fresh engine per channel
            self.swap_ir(ragged)

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
        """[C, n] in, [C, n] out (engine.py:118-146 per channel).  A pending
        swap (uniform or per channel) is applied first, inside the library."""
        t = _dev.torch()
        with _dev.device_guard(self._device):
            xd = self._rows(block)
            n = xd.shape[1]
            out = t.empty_like(xd)
            self._bind()   # an empty block still applies a pending swap (engine.py:124-126)
            N.check(self._lib.sc_engine_process_block(self._handle, N.ptr(xd) if n else None, n,
                                                      N.ptr(out) if n else None))
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

    def _channel_irs(self, h_new, channels):
        """(rows [C, L] on the device, per-channel lengths (0 = keep)) for a
        per-channel swap.  h_new: a mono IR (1-D) for the selected channels,
        [C, n] rows, or a list of C per-channel IRs (None = keep); channels:
        indices or a boolean mask of the channels that swap (default: every
        channel given an IR)."""
        C = self._C
        if isinstance(h_new, (list, tuple)):
            if len(h_new) != C:
                raise ValueError(f"expected {C} per-channel impulse responses, got {len(h_new)}")
            per = [None if a is None else (a.cpu().numpy() if _dev.is_tensor(a) else np.asarray(a)) for a in h_new]
        else:
            hd = h_new.cpu().numpy() if _dev.is_tensor(h_new) else np.asarray(h_new)
            if hd.ndim == 1:
                per = [hd] * C
            elif hd.ndim == 2 and hd.shape[0] == C:
                per = list(hd)
            else:
                raise ValueError(f"expected a mono IR, [channels={C}, n] rows or {C} IRs, got shape {hd.shape}")
        if channels is not None:
            sel = np.zeros(C, dtype=bool)
            ch = np.asarray(channels)
            if ch.dtype == bool:
                if ch.shape != (C,):
                    raise ValueError(f"channel mask must have {C} entries")
                sel = ch
            else:
                sel[ch.astype(np.int64)] = True
            per = [a if sel[c] else None for c, a in enumerate(per)]
        if any(a is not None and len(a) == 0 for a in per):
            raise ValueError("impulse response is empty")
        lengths = np.array([0 if a is None else len(a) for a in per], dtype=np.int64)
        if not lengths.any():
            raise ValueError("no channel swaps")
        rows = np.zeros((C, int(lengths.max())), dtype=self._npd)
        for c, a in enumerate(per):
            if a is not None:
                rows[c, :len(a)] = a
        return _dev.as_device(rows, self._npd, device=self._device), lengths

    def _uniform(self, h_new, channels) -> bool:
        if channels is not None or isinstance(h_new, (list, tuple)):
            return False
        return True

    def swap_ir(self, h_new, channels=None):
        """Swap impulse responses (engine.py:163-186, per channel).  Every
        channel to its row of h_new (or a broadcast mono IR); with
        ``channels`` (indices or mask) or a list of per-channel IRs (None =
        keep), only those channels swap and lengths may differ -- the
        semantics of one engine per channel."""
        import ctypes

        with _dev.device_guard(self._device):
            self._bind()
            if self._uniform(h_new, channels):
                hd = self._ir_rows(h_new)
                N.check(self._lib.sc_engine_swap_ir(self._handle, N.ptr(hd), hd.shape[1]))
                return
            rows, lengths = self._channel_irs(h_new, channels)
            nh = (ctypes.c_int64 * self._C)(*lengths.tolist())
            N.check(self._lib.sc_engine_swap_ir_channels(self._handle, N.ptr(rows), rows.shape[1], nh))

    def swap_ir_at_next_block(self, h_new, channels=None):
        """Deferred swap applied by the next process_block (engine.py:188-192),
        for every channel or (``channels`` / per-channel list) some of them."""
        import ctypes

        with _dev.device_guard(self._device):
            self._bind()
            if self._uniform(h_new, channels):
                hd = self._ir_rows(h_new)   # validated now
                N.check(self._lib.sc_engine_swap_ir_at_next_block(self._handle, N.ptr(hd), hd.shape[1]))
                return
            rows, lengths = self._channel_irs(h_new, channels)
            nh = (ctypes.c_int64 * self._C)(*lengths.tolist())
            N.check(self._lib.sc_engine_swap_ir_at_next_block_channels(self._handle, N.ptr(rows), rows.shape[1], nh))

    @property
    def ir_lengths(self) -> list:
        """Every channel's current impulse-response length."""
        import ctypes

        nh = (ctypes.c_int64 * self._C)()
        N.check(self._lib.sc_engine_channel_nh(self._handle, nh))
        return list(nh)

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
                "nh": nh.value, "nh_per_channel": self.ir_lengths}

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
            # swaps outside [0, n_blocks) precede no block: the library ignores them
            swaps = sorted((s for s in swaps if 0 <= int(s[0]) < n_blocks), key=lambda s: s[0])
            if any(len(s) > 2 or isinstance(s[1], (list, tuple)) for s in swaps):
                return self._process_stream_channels(x, nb, swaps)
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

    def _process_stream_channels(self, x, nb, swaps):
        """Per-channel swap schedule: entries (block, IR) swap every channel,
        (block, IR, channels) or (block, [per-channel IRs]) only some; the
        library runs the blocks one launch each (sc_engine_process_blocks_channels)."""
        import ctypes

        t = _dev.torch()
        C = self._C
        rows_list, flat = [], []
        for s in swaps:
            rows, lengths = self._channel_irs(s[1], s[2] if len(s) > 2 else None)
            rows_list.append(rows)
            flat.extend(lengths.tolist())
        k = len(swaps)
        blocks = (ctypes.c_int64 * max(k, 1))(*[int(s[0]) for s in swaps])
        ptrs = (ctypes.c_void_p * max(k, 1))(*[r.data_ptr() for r in rows_list])
        lds = (ctypes.c_int64 * max(k, 1))(*[r.shape[1] for r in rows_list])
        nhs = (ctypes.c_int64 * max(k * C, 1))(*flat)
        xd = self._rows(x)
        out = t.empty_like(xd)
        self._bind()
        N.check(self._lib.sc_engine_process_blocks_channels(self._handle, N.ptr(xd), xd.shape[1], nb, blocks, ptrs,
                                                            lds, nhs, k, N.ptr(out)))
        return _dev.like_input(out, x)
