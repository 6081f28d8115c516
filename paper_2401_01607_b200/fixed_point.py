"""Fixed-point requantisation budgets and bit-true simulation on the device
(SURVEY.md 8(f) row 4).

Drop-in for ``scatterconv.quantize`` (pkg/src/scatterconv/quantize.py): the
same names, argument meaning, validation messages and results.  The closed
forms (accumulator width, bits removed per rounding event) are plain host
arithmetic; quantisation and the exact-integer convolution under the
``ideal`` / ``mac`` schemes run in csrc/k_fixed.cu with __int128
intermediates, and the double-precision comparison runs through the device
``direct_form``.  Outputs are bit-identical to the reference's unbounded
Python-integer simulation whenever the 128-bit accumulator provably holds
every intermediate (always for word lengths up to 32 bits); otherwise a
ValueError says so instead of returning a wrapped result.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _dev
from . import _native as N
from .core import Signal, direct_form

ROUNDING_MODES = ("nearest-even",)
OVERFLOW_MODES = ("saturate",)
SCHEMES = ("ideal", "mac")
_SCHEME_CODE = {"ideal": 0, "mac": 1}


@dataclass(frozen=True)
class FixedPointFormat:
    """Two's-complement fraction: one sign bit and word_bits-1 fractional bits
    (quantize.py:34-70)."""

    word_bits: int
    rounding: str = "nearest-even"
    overflow: str = "saturate"

    def __post_init__(self):
        if not isinstance(self.word_bits, (int, np.integer)) or self.word_bits < 2:
            raise ValueError(f"word_bits must be an integer >= 2, got {self.word_bits!r}")
        if self.rounding not in ROUNDING_MODES:
            raise ValueError(f"rounding must be one of {ROUNDING_MODES}, got {self.rounding!r}")
        if self.overflow not in OVERFLOW_MODES:
            raise ValueError(f"overflow must be one of {OVERFLOW_MODES}, got {self.overflow!r}")

    fractional_bits = property(lambda self: self.word_bits - 1)
    scale = property(lambda self: 1 << (self.word_bits - 1))
    min_int = property(lambda self: -(1 << (self.word_bits - 1)))
    max_int = property(lambda self: (1 << (self.word_bits - 1)) - 1)
    ulp = property(lambda self: 1.0 / (1 << (self.word_bits - 1)))


@dataclass
class RequantReport:
    """Error statistics of one simulated scheme (quantize.py:73-100):
    rounding events per output, bits removed per event, and rms / max error
    against the exact-product result on the same quantised inputs."""

    scheme: str
    operations_count: int
    bits_removed_per_op: int
    rms_error: float
    max_error: float

    def __post_init__(self):
        if self.scheme not in SCHEMES:
            raise ValueError(f"scheme must be one of {SCHEMES}, got {self.scheme!r}")
        if self.operations_count < 0 or self.bits_removed_per_op < 0:
            raise ValueError("counts must be non-negative")
        if self.rms_error > self.max_error:
            raise ValueError(f"rms_error {self.rms_error} exceeds max_error {self.max_error}")


# ------------------------------------------------------------------ closed forms


def _check_bits(n_bits, ir_len):
    if not isinstance(n_bits, (int, np.integer)) or n_bits < 2:
        raise ValueError(f"word length must be an integer >= 2 bits, got {n_bits!r}")
    if not isinstance(ir_len, (int, np.integer)) or ir_len < 1:
        raise ValueError(f"impulse response length must be a positive integer, got {ir_len!r}")


def ideal_accumulator_bits(n_bits: int, ir_len: int) -> int:
    """Overflow-proof accumulator width, 2*n_bits + ir_len - 1 (one carry bit
    per added term: the reference's deliberately conservative budget)."""
    _check_bits(n_bits, ir_len)
    return 2 * n_bits + ir_len - 1


def ideal_bits_removed(n_bits: int, ir_len: int) -> int:
    """Bits the single final rounding of the ideal scheme drops."""
    _check_bits(n_bits, ir_len)
    return n_bits + ir_len - 1


def mac_requant_count(n_bits: int, ir_len: int) -> tuple[int, int]:
    """(rounding events, bits each) of the round-after-every-MAC scheme."""
    _check_bits(n_bits, ir_len)
    return ir_len - 1, n_bits


# ------------------------------------------------------------------ device simulation


def _quantize_device(values, fmt: FixedPointFormat):
    """-> (k int64 CUDA tensor, k/scale float64 CUDA tensor, max |k|)."""
    t = _dev.torch()
    x = _dev.as_device(values, np.float64)
    if x.ndim != 1:
        x = x.reshape(-1)
    if fmt.word_bits > 64:
        raise ValueError(f"word_bits {fmt.word_bits} exceeds the device simulation's 64-bit sample words")
    k = t.empty(x.shape[0], dtype=t.int64, device=x.device)
    xq = t.empty(x.shape[0], dtype=t.float64, device=x.device)
    stats = t.zeros(2, dtype=t.int64, device=x.device)
    with t.cuda.device(x.device):
        N.check(N.lib().sc_fixed_quantize(N.ptr(x), x.shape[0], int(fmt.word_bits), N.ptr(k), N.ptr(xq),
                                          N.ptr(stats), N.stream_ptr()))
    bad, mx = stats.cpu().numpy().view(np.uint64).tolist()
    if bad:
        raise ValueError("samples outside the representable range [-1, 1)")
    return k, xq, int(mx)


def quantize(values, fmt: FixedPointFormat):
    """Round values in [-1, 1) onto the format's grid (exact floats); returns
    the caller's currency (ndarray for host input, tensor for tensors)."""
    _, xq, _ = _quantize_device(values, fmt)
    return _dev.like_input(xq, values)


def fixed_point_convolve(e: Signal, h: Signal, fmt: FixedPointFormat, scheme: str) -> Signal:
    """Quantise both signals, convolve exactly in integers, requantise per
    scheme (quantize.py:163-195).  Float64 outputs on the format's grid."""
    if scheme not in SCHEMES:
        raise ValueError(f"scheme must be one of {SCHEMES}, got {scheme!r}")
    if len(e) == 0 or len(h) == 0:
        raise ValueError("empty signal")
    if e.sample_rate != h.sample_rate:
        raise ValueError("sample rates differ")
    y = _fixed_conv_device(e, h, fmt, scheme)[0]
    return Signal(_dev.like_input(y, e.samples, h.samples), e.sample_rate)


def _fixed_conv_device(e: Signal, h: Signal, fmt: FixedPointFormat, scheme: str):
    t = _dev.torch()
    ke, eq, me = _quantize_device(e.samples, fmt)
    kh, hq, mh = _quantize_device(h.samples, fmt)
    terms = min(len(e), len(h))
    need = me.bit_length() + mh.bit_length() + max(0, math.ceil(math.log2(terms)))
    if need > 126:
        raise ValueError(f"{fmt.word_bits}-bit simulation of {terms}-term sums needs {need} accumulator bits; "
                         "the device accumulator holds 126")
    wide = me >= (1 << 31) or mh >= (1 << 31)
    y = t.empty(len(e) + len(h) - 1, dtype=t.float64, device=ke.device)
    with t.cuda.device(ke.device):
        N.check(N.lib().sc_fixed_convolve(N.ptr(ke), len(e), N.ptr(kh), len(h), int(fmt.word_bits),
                                          _SCHEME_CODE[scheme], int(wide), N.ptr(y), N.stream_ptr()))
    return y, eq, hq


def simulate_fixed_point_conv(e: Signal, h: Signal, fmt: FixedPointFormat, scheme: str) -> RequantReport:
    """Run one scheme and measure it against direct_form on the quantised
    inputs, isolating requantisation damage (quantize.py:198-222)."""
    if scheme not in SCHEMES:
        raise ValueError(f"scheme must be one of {SCHEMES}, got {scheme!r}")
    if len(e) == 0 or len(h) == 0:
        raise ValueError("empty signal")
    if e.sample_rate != h.sample_rate:
        raise ValueError("sample rates differ")
    y, eq, hq = _fixed_conv_device(e, h, fmt, scheme)
    ref = direct_form(Signal(eq, e.sample_rate), Signal(hq, h.sample_rate)).samples
    # the two summary statistics are numpy reductions of the device results
    # (pairwise sums, as the reference computes them)
    err = y.cpu().numpy() - ref.cpu().numpy()
    nh = len(h)
    ops, bits = (1, ideal_bits_removed(fmt.word_bits, nh)) if scheme == "ideal" else (max(1, nh - 1), fmt.word_bits)
    return RequantReport(scheme=scheme, operations_count=ops, bits_removed_per_op=bits,
                         rms_error=float(np.sqrt(np.mean(err ** 2))), max_error=float(np.max(np.abs(err))))


__all__ = ["FixedPointFormat", "OVERFLOW_MODES", "ROUNDING_MODES", "RequantReport", "SCHEMES",
           "fixed_point_convolve", "ideal_accumulator_bits", "ideal_bits_removed", "mac_requant_count",
           "quantize", "simulate_fixed_point_conv"]
