"""Whole-signal scatter convolution -- drop-in for ``scatterconv.core``.

Mirrors pkg/src/scatterconv/core.py (Signal, ConvOutput, direct_form,
scatter_convolve, commuted_convolve, scatter_convolve_skip_zeros) with the
same names, argument meaning, validation messages and return types.  The
arithmetic runs in the CUDA library (csrc/), never on the host:

* float64 signals (the reference's only type, core.py:38) use the ORDERED
  kernel: each output is a single chain over input index ascending with
  separately rounded multiply and add -- bit-identical to the reference.
* float32 signals (arrays or tensors; ``Signal`` keeps float32 instead of
  upcasting) use the FAST path, within 1e-5*max|x|*||h||_1 of the
  reference: the tcgen05 tensor-core FIR (fp16 hi/lo split, 3 MMAs) for
  filters of >= 256 taps (>= 26 on launches of >= 2^30 MACs), the CUDA-core
  short-filter kernels below that; ``mode="ffma"`` forces the FFMA2
  register-tiled kernel, ``mode="tc"`` the tensor cores, and
  ``mode="ordered"`` the ordered chain in float32.
* ``direct_form`` is exactly rounded like the reference's math.fsum.

Samples may be numpy arrays (results come back as arrays) or torch tensors
(CUDA tensors stay on the device; no host synchronisation).
"""

from __future__ import annotations

from dataclasses import dataclass

import os

import numpy as np

from . import _dev
from . import _native as N


@dataclass(eq=False)
class Signal:
    """A finite run of samples at a fixed sample rate (core.py:25-49).

    ``samples`` becomes a 1-D float64 array like the reference, except that
    float32 arrays and float32/float64 torch tensors keep their dtype (and
    CUDA tensors their device) so the FP32 path and device residency are
    reachable through the same type.
    """

    samples: object
    sample_rate: int = 44100

    def __post_init__(self):
        if _dev.is_tensor(self.samples):
            t = _dev.torch()
            if self.samples.dtype not in (t.float32, t.float64):
                self.samples = self.samples.to(t.float64)
        else:
            arr = np.asarray(self.samples)
            if arr.dtype != np.float32:
                arr = np.asarray(self.samples, dtype=np.float64)
            self.samples = arr
        if self.samples.ndim != 1:
            raise ValueError(f"samples must be 1-D, got shape {tuple(self.samples.shape)}")
        if not isinstance(self.sample_rate, (int, np.integer)) or self.sample_rate <= 0:
            raise ValueError(f"sample_rate must be a positive integer, got {self.sample_rate!r}")

    def __len__(self):
        return int(self.samples.shape[0])

    @property
    def duration_s(self) -> float:
        return len(self) / self.sample_rate

    @property
    def dtype(self):
        return _dev.np_dtype(self.samples)


@dataclass(eq=False)
class ConvOutput:
    """Body (aligned with the input) and tail (len(h)-1 samples), core.py:52-66."""

    body: Signal
    tail: Signal

    def concatenated(self) -> Signal:
        a, b = self.body.samples, self.tail.samples
        if _dev.is_tensor(a):
            joined = _dev.torch().cat([a, b.to(a.device)])
        else:
            joined = np.concatenate([a, b])
        return Signal(joined, self.body.sample_rate)


def _check_pair(e: Signal, h: Signal):
    """core.py:69-77 (same messages)."""
    if len(e) == 0:
        raise ValueError("input signal is empty")
    if len(h) == 0:
        raise ValueError("impulse response is empty")
    if e.sample_rate != h.sample_rate:
        raise ValueError(
            f"sample rates differ: input {e.sample_rate} Hz vs impulse response {h.sample_rate} Hz"
        )


def _result_dtype(*arrays):
    return np.float64 if any(_dev.np_dtype(a) == np.float64 for a in arrays) else np.float32


_MODES = {None: None, "fast": N.SC_MODE_FAST, "ordered": N.SC_MODE_ORDERED,
          "strict": N.SC_MODE_ORDERED, "ffma": N.SC_MODE_FFMA, "tc": N.SC_MODE_TC}


def mode_code(mode) -> int:
    """C-ABI mode for a float32 fast-path name (None/"fast", "ffma", "tc")."""
    if mode is None:
        return N.SC_MODE_FAST
    if mode not in ("fast", "ffma", "tc"):
        raise ValueError(f"mode must be 'fast', 'ffma' or 'tc', got {mode!r}")
    return _MODES[mode]


_PIPELINE_MIN_MACS = 1 << 36   # host-resident inputs this large are streamed in chunks (by the
_PIPELINE_MIN_BYTES = 1 << 25   # library: one per >= 2^36 MACs or 16 MiB, 2..12), as are transfer-bound ones
_PIPE_STREAMS: dict = {}


def pipe_streams(dev):
    """(upload, compute, download) streams of a device, created once: the
    library's scratch buffers are keyed by stream, so fresh streams would
    re-allocate every call."""
    t = _dev.torch()
    if dev.index not in _PIPE_STREAMS:
        _PIPE_STREAMS[dev.index] = tuple(t.cuda.Stream(dev) for _ in range(3))
    return _PIPE_STREAMS[dev.index]


def _fir_host_pipelined(x_pin, kern, mode):
    """Pinned-host float32 input: the native chunk-pipelined range engine
    (csrc/sharded.cu sc_fir_range_host) over the whole output -- upload,
    FIR and download of consecutive output chunks overlap on three persistent
    streams.  Returns a pinned host tensor with the full Ne+Nh-1 result."""
    t = _dev.torch()
    dev = t.cuda.current_device()
    h = kern if (_dev.is_tensor(kern) and kern.is_cuda and kern.get_device() == dev
                 and kern.dtype == t.float32 and kern.is_contiguous()) else None
    if h is None:
        h = _dev.as_device(kern, np.float32, device=t.device("cuda", dev))
    ne, nh = x_pin.shape[0], h.shape[0]
    out = t.empty(ne + nh - 1, dtype=t.float32, pin_memory=True)
    # h (and x, when the caller just filled it) are ordered on the current stream
    t.cuda.current_stream().synchronize()
    chunks = int(os.environ.get("SC_PIPE_CHUNKS", "0"))
    N.check(N.lib().sc_fir_range_host(N.SC_F32, mode, N.ptr(x_pin), ne, N.ptr(h), nh, N.ptr(out), 0,
                                      ne + nh - 1, dev, chunks))
    return out


def _fir(drive, kern, *, mode=None, skip_mode=N.SC_SKIP_NONE, threshold=0.0):
    """Full convolution of two 1-D sample arrays on the device (core._scatter_full
    semantics: slot n accumulates drive samples in increasing index)."""
    if mode not in _MODES:
        raise ValueError(f"mode must be one of {sorted(k for k in _MODES if k)}, got {mode!r}")
    npd = _result_dtype(drive, kern)
    m = _MODES[mode]
    if m is None:
        m = N.SC_MODE_FAST if npd == np.float32 else N.SC_MODE_ORDERED
    L = N.lib()
    t = _dev.torch()
    if (npd == np.float32 and m != N.SC_MODE_ORDERED and skip_mode == N.SC_SKIP_NONE
            and _dev.is_tensor(drive) and drive.device.type == "cpu" and drive.is_pinned()
            and drive.dtype == t.float32 and (drive.shape[0] * int(np.shape(kern)[0]) >= _PIPELINE_MIN_MACS
                                              or 4 * drive.shape[0] >= _PIPELINE_MIN_BYTES)):
        return _fir_host_pipelined(drive, kern, m)
    x = _dev.as_device(drive, npd)
    h = _dev.as_device(kern, npd, device=x.device)
    nout = x.shape[0] + h.shape[0] - 1
    with t.cuda.device(x.device):
        y = t.empty(nout, dtype=x.dtype, device=x.device)
        N.check(L.sc_fir_full(N.dtype_code(npd), m, N.ptr(x), x.shape[0], N.ptr(h), h.shape[0],
                              N.ptr(y), skip_mode, float(threshold), N.stream_ptr()))
    return _dev.like_input(y, drive, kern)


def _scatter_full(drive, kern, mode=None):
    """Scatter `drive` through `kern` into a fresh linear buffer (core.py:80-92).

    Each drive sample adds its scaled copy of `kern` in increasing tap order,
    so every output slot accumulates contributions in increasing drive-index
    order -- the ordered kernel reproduces exactly that chain.
    """
    return _fir(drive, kern, mode=mode)


def _split(full, n_body: int, sample_rate: int) -> ConvOutput:
    """core.py:95-99.  The reference copies the two slices out of its scratch
    buffer; `full` here is always a fresh buffer owned by this result, so the
    body and tail are views of it (no extra host/device copy)."""
    return ConvOutput(body=Signal(full[:n_body], sample_rate),
                      tail=Signal(full[n_body:], sample_rate))


def direct_form(e: Signal, h: Signal) -> Signal:
    """Gather-form convolution (core.py:102-119).

    The reference sums each output's individually rounded products with
    math.fsum; the device runs the same exactly rounded summation (CPython's
    fsum algorithm, one thread per output), float64 always, so the results
    are bit-identical.  Like math.fsum it raises OverflowError on an
    intermediate overflow of finite products and ValueError on -inf + inf.
    """
    _check_pair(e, h)
    L = N.lib()
    t = _dev.torch()
    x = _dev.as_device(e.samples, np.float64)
    k = _dev.as_device(h.samples, np.float64, device=x.device)
    with t.cuda.device(x.device):
        y = t.empty(len(e) + len(h) - 1, dtype=t.float64, device=x.device)
        status = t.zeros(1, dtype=t.int32, device=x.device)
        N.check(L.sc_direct_form(N.ptr(x), len(e), N.ptr(k), len(h), N.ptr(y), N.ptr(status), N.stream_ptr()))
        bad = int(status.item())
    if bad & 1:
        raise OverflowError("intermediate overflow in fsum")
    if bad & 2:
        raise ValueError("-inf + inf in fsum")
    return Signal(_dev.like_input(y, e.samples, h.samples), e.sample_rate)


def scatter_convolve(e: Signal, h: Signal, *, mode=None) -> ConvOutput:
    """Convolve by scattering one scaled, delayed copy of h per input sample
    (core.py:122-131).  ``mode``: None (float64 -> ordered, float32 -> fast),
    "fast" or "ordered"/"strict"."""
    _check_pair(e, h)
    full = _scatter_full(e.samples, h.samples, mode=mode) if mode else _scatter_full(e.samples, h.samples)
    return _split(full, len(e), e.sample_rate)


def commuted_convolve(e: Signal, h: Signal) -> ConvOutput:
    """Scatter with the shorter signal driving the loop (core.py:134-147).

    The body/tail split still follows the original argument roles.
    """
    _check_pair(e, h)
    if len(h) <= len(e):
        full = _scatter_full(h.samples, e.samples)
    else:
        full = _scatter_full(e.samples, h.samples)
    return _split(full, len(e), e.sample_rate)


def scatter_convolve_skip_zeros(e: Signal, h: Signal, threshold: float = 0.0) -> ConvOutput:
    """Scatter convolution skipping input samples with |value| <= threshold
    (core.py:150-167).  NaN inputs are not skipped (they propagate)."""
    if threshold < 0:
        raise ValueError(f"threshold must be non-negative, got {threshold}")
    _check_pair(e, h)
    full = _fir(e.samples, h.samples, mode="ordered", skip_mode=N.SC_SKIP_LE,
                threshold=threshold)
    return _split(full, len(e), e.sample_rate)
