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


def _int_at_least(v, lo: int) -> bool:
    return isinstance(v, (int, np.integer)) and v >= lo


def _one_of(value, allowed, what: str):
    if value not in allowed:
        raise ValueError(f"{what} must be one of {allowed}, got {value!r}")


@dataclass(frozen=True)
class FixedPointFormat:
    """Two's-complement fraction: one sign bit and word_bits-1 fractional bits
    (quantize.py:34-70).  Rounds to nearest-even; saturates where samples are
    stored."""

    word_bits: int
    rounding: str = "nearest-even"
    overflow: str = "saturate"

    def __post_init__(self):
        if not _int_at_least(self.word_bits, 2):
            raise ValueError(f"word_bits must be an integer >= 2, got {self.word_bits!r}")
        _one_of(self.rounding, ROUNDING_MODES, "rounding")
        _one_of(self.overflow, OVERFLOW_MODES, "overflow")

    @property
    def fractional_bits(self) -> int:
        return self.word_bits - 1

    @property
    def scale(self) -> int:                 # 2^fractional_bits
        return 1 << self.fractional_bits

    @property
    def min_int(self) -> int:
        return -self.scale

    @property
    def max_int(self) -> int:
        return self.scale - 1

    @property
    def ulp(self) -> float:
        return 1.0 / self.scale


@dataclass
class RequantReport:
    """What one simulated scheme did (quantize.py:73-100): rounding events
    per output sample and the bits each removes, plus rms / max deviation from
    the exact-product result on the same quantised inputs."""

    scheme: str
    operations_count: int
    bits_removed_per_op: int
    rms_error: float
    max_error: float

    def __post_init__(self):
        _one_of(self.scheme, SCHEMES, "scheme")
        if min(self.operations_count, self.bits_removed_per_op) < 0:
            raise ValueError("counts must be non-negative")
        if self.rms_error > self.max_error:
            raise ValueError(f"rms_error {self.rms_error} exceeds max_error {self.max_error}")


# ------------------------------------------------------------------ closed forms


def _budget_args(n_bits, ir_len):
    if not _int_at_least(n_bits, 2):
        raise ValueError(f"word length must be an integer >= 2 bits, got {n_bits!r}")
    if not _int_at_least(ir_len, 1):
        raise ValueError(f"impulse response length must be a positive integer, got {ir_len!r}")
    return int(n_bits), int(ir_len)


def ideal_accumulator_bits(n_bits: int, ir_len: int) -> int:
    """Overflow-proof accumulator width: two N-bit operands per product plus
    one carry bit per added term (the reference's conservative budget)."""
    n, L = _budget_args(n_bits, ir_len)
    return 2 * n + L - 1


def ideal_bits_removed(n_bits: int, ir_len: int) -> int:
    """Bits the ideal scheme's single final rounding drops."""
    n, L = _budget_args(n_bits, ir_len)
    return n + L - 1


def mac_requant_count(n_bits: int, ir_len: int) -> tuple[int, int]:
    """(rounding events, bits per event) when every MAC is rounded back."""
    n, L = _budget_args(n_bits, ir_len)
    return L - 1, n


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


def _round_shift_half_even(t, shift: int):
    """t / 2**shift rounded to nearest, ties to even (quantize.py:145-154),
    evaluated by the device's requantisation step (``sc_fixed_round_shift``).
    Scalar in, scalar out (as the reference); arrays map element-wise."""
    tt = _dev.torch()
    scalar = np.ndim(t) == 0
    v = np.asarray(t, dtype=object).reshape(-1)
    if any(not (-(1 << 63) <= int(a) < (1 << 63)) for a in v):
        raise ValueError("the device requantisation step takes 64-bit integers")
    src = tt.tensor([int(a) for a in v], dtype=tt.int64).to(tt.device("cuda", tt.cuda.current_device()))
    out = tt.empty_like(src)
    with tt.cuda.device(src.device):
        N.check(N.lib().sc_fixed_round_shift(N.ptr(src), src.shape[0], int(shift), N.ptr(out), N.stream_ptr()))
    res = [int(a) for a in out.cpu().tolist()]
    return res[0] if scalar else np.asarray(res, dtype=np.int64)


def _check_pair(e: Signal, h: Signal, scheme: str):
    _one_of(scheme, SCHEMES, "scheme")
    if min(len(e), len(h)) == 0:
        raise ValueError("empty signal")
    if e.sample_rate != h.sample_rate:
        raise ValueError("sample rates differ")


def fixed_point_convolve(e: Signal, h: Signal, fmt: FixedPointFormat, scheme: str) -> Signal:
    """Quantise both signals, convolve exactly in integers, requantise per
    scheme (quantize.py:163-195).  Float64 outputs on the format's grid."""
    _check_pair(e, h, scheme)
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
    _check_pair(e, h, scheme)
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
