"""Whole-signal convolution on the GPU vs the reference's goldens and the CPU
oracle.  Mirrors pkg/tests/test_core.py (frozen values, oracle equivalence,
algebraic properties) and adds the float32 fast path.

float64: bit-exact to the reference (ordered kernel).  float32 fast path:
max-abs error <= 1e-5 * max|x| * ||h||_1 (north_star tolerance).
"""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import oracle as O
from paper_2401_01607_b200 import core, configs
from paper_2401_01607_b200.core import (
    Signal,
    commuted_convolve,
    direct_form,
    scatter_convolve,
    scatter_convolve_skip_zeros,
)
from paper_2401_01607_b200.multichannel import convolve_batched
from paper_2401_01607_b200.sharded import convolve_shard, shard_plan
from tests import _golden as G

pytestmark = pytest.mark.gpu


def _sig(values, rate=44100):
    return Signal(np.asarray(values, dtype=np.float64), rate)


def _whole(out) -> np.ndarray:
    return np.asarray(out.concatenated().samples)


def _near(actual, expected, rtol):
    expected = np.asarray(expected)
    scale = max(1.0, float(np.max(np.abs(expected))) if expected.size else 0.0)
    np.testing.assert_allclose(actual, expected, rtol=0.0, atol=rtol * scale)


def within_tol(y, ref, x, h, dtype="f32"):
    tol = configs.tolerance(x, h, dtype)
    err = float(np.max(np.abs(np.asarray(y, np.float64) - ref))) if len(ref) else 0.0
    assert err <= tol, f"max err {err:.3e} > tol {tol:.3e}"
    return err, tol


_AMP = st.floats(min_value=-1.0, max_value=1.0, allow_nan=False, width=64)
_SEQ = st.lists(_AMP, min_size=1, max_size=64)

# ---------------------------------------------------------------- frozen values


def test_direct_form_hand_examples():
    assert np.array_equal(direct_form(_sig([1.0]), _sig([5.0, 6.0, 7.0])).samples, [5.0, 6.0, 7.0])
    assert np.array_equal(direct_form(_sig([1.0, 2.0]), _sig([3.0, 4.0])).samples, [3.0, 10.0, 8.0])
    assert np.array_equal(direct_form(_sig([0.0, 0.0, 0.0]), _sig([1.0, 1.0])).samples, np.zeros(4))


def test_scatter_hand_examples():
    out = scatter_convolve(_sig([1.0, 2.0]), _sig([3.0, 4.0]))
    assert np.array_equal(out.body.samples, [3.0, 10.0])
    assert np.array_equal(out.tail.samples, [8.0])
    out = scatter_convolve(_sig([1.0, 0.0, 0.0, 0.0]), _sig([9.0]))
    assert np.array_equal(out.body.samples, [9.0, 0.0, 0.0, 0.0]) and len(out.tail) == 0
    h = _sig([0.5, -0.25, 0.125])
    for k in (1, 3, 7):
        got = _whole(scatter_convolve(_sig([0.0] * k + [1.0]), h))
        assert np.array_equal(got[:k], np.zeros(k)) and np.array_equal(got[k:], h.samples)


def test_commuted_short_signal_drives(monkeypatch):
    lengths = []
    original = core._scatter_full

    def spy(drive, kern):
        lengths.append(len(drive))
        return original(drive, kern)

    monkeypatch.setattr(core, "_scatter_full", spy)
    e = _sig([1.0, 2.0, 3.0, 4.0, 5.0, 6.0])
    h = _sig([1.0, 2.0, 3.0])
    out = commuted_convolve(e, h)
    assert lengths == [3]
    assert len(out.body) == 6 and len(out.tail) == 2
    lengths.clear()
    commuted_convolve(h, e)
    assert lengths == [3]


def test_skip_zeros_hand_examples():
    out = scatter_convolve_skip_zeros(_sig([1.0, 0.0, 2.0]), _sig([1.0, 1.0]), threshold=0.0)
    assert np.array_equal(out.body.samples, [1.0, 1.0, 2.0]) and np.array_equal(out.tail.samples, [2.0])
    out = scatter_convolve_skip_zeros(_sig([0.0, 0.0]), _sig([4.0, 5.0, 6.0]), threshold=0.0)
    assert np.array_equal(_whole(out), np.zeros(4))
    out = scatter_convolve_skip_zeros(_sig([1.0, 1e-9, 1.0]), _sig([1.0]), threshold=1e-6)
    assert np.array_equal(out.body.samples, [1.0, 0.0, 1.0])


def test_nan_and_signed_zero_semantics():
    # scatter_convolve propagates NaN (core.py:90); -0.0 inputs still "scatter"
    got = _whole(scatter_convolve(_sig([1.0, np.nan, 2.0]), _sig([1.0, 1.0])))
    want = O.scatter_full([1.0, np.nan, 2.0], [1.0, 1.0])
    assert np.array_equal(got, want, equal_nan=True)
    got = _whole(scatter_convolve(_sig([-0.0]), _sig([-0.0, 1.0])))
    assert np.array_equal(np.signbit(got), np.signbit(O.scatter_full([-0.0], [-0.0, 1.0])))


# ---------------------------------------------------------------- reference goldens


@pytest.fixture(scope="module")
def pairs():
    return G.small_pairs()


def test_golden_scatter_commuted_skip_bit_exact(pairs):
    for p in pairs:
        E, H = _sig(p["e"]), _sig(p["h"])
        assert np.array_equal(_whole(scatter_convolve(E, H)), p["scatter"])
        assert np.array_equal(_whole(commuted_convolve(E, H)), p["commuted"])
        assert np.array_equal(_whole(scatter_convolve_skip_zeros(E, H, p["threshold"])), p["skip"])


def test_golden_direct_form(pairs):
    """Exactly rounded like math.fsum: every golden output bit-exact."""
    for p in pairs:
        got = direct_form(_sig(p["e"]), _sig(p["h"])).samples
        assert np.array_equal(got, p["direct"])


@given(e=_SEQ, h=_SEQ)
@settings(max_examples=150)
def test_direct_form_matches_fsum_oracle(e, h):
    assert np.array_equal(direct_form(_sig(e), _sig(h)).samples, O.direct_form(e, h))


def test_direct_form_cancellation_and_specials():
    """Products whose exact sum cancels far below any partial (where a
    compensated sum fails), ties that the half-even fix-up decides, and
    fsum's non-finite rules (NaN / Inf propagate; -inf + inf and an
    intermediate overflow raise like math.fsum)."""
    import math

    cases = [
        ([1e16, 1.0, -1e16, 1e-16], [1.0]),
        ([1.0, 2.0 ** -53, 2.0 ** -106], [1.0]),
        ([2.0 ** 53, 1.0, 1.0 - 2.0 ** -53], [1.0, 1.0]),
        ([1e308, 1e308, -1e308], [0.5]),
        ([3.0, -1e-300, 1e300, -1e300], [1.0, 1e-10, 7.0]),
        ([0.1] * 10 + [-1.0], [1.0]),
    ]
    for e, h in cases:
        got = direct_form(_sig(e), _sig(h)).samples
        ne, nh = len(e), len(h)
        want = [math.fsum(e[m] * h[n - m] for m in range(max(0, n - nh + 1), min(n, ne - 1) + 1))
                for n in range(ne + nh - 1)]
        assert np.array_equal(got, np.asarray(want)), (e, h)
    assert np.isnan(direct_form(_sig([1.0, float("nan")]), _sig([1.0])).samples[1])
    assert direct_form(_sig([float("inf"), 1.0]), _sig([1.0, 1.0])).samples[1] == float("inf")
    with pytest.raises(ValueError, match="inf"):
        direct_form(_sig([float("inf"), float("-inf")]), _sig([1.0, 1.0]))
    with pytest.raises(OverflowError):
        direct_form(_sig([1e308, 1e308]), _sig([1.0, 1.0]))


# ---------------------------------------------------------------- properties (float64)


@given(e=_SEQ, h=_SEQ)
@settings(max_examples=150)
def test_oracle_equivalence(e, h):
    got = _whole(scatter_convolve(_sig(e), _sig(h)))
    assert np.array_equal(got, O.scatter_full(e, h))          # reference chain, bit-exact
    _near(got, O.direct_form(e, h), 1e-12)             # exact-sum oracle


@given(e=_SEQ, h=_SEQ)
def test_length_law_and_commutativity(e, h):
    out = scatter_convolve(_sig(e), _sig(h))
    assert len(out.body) == len(e) and len(out.tail) == len(h) - 1
    _near(_whole(out), _whole(scatter_convolve(_sig(h), _sig(e))), 1e-12)
    _near(_whole(commuted_convolve(_sig(e), _sig(h))), _whole(out), 1e-12)


@given(e1=_SEQ, e2=_SEQ, h=_SEQ,
       a=st.floats(min_value=-10, max_value=10, allow_nan=False, width=64),
       b=st.floats(min_value=-10, max_value=10, allow_nan=False, width=64))
def test_linearity(e1, e2, h, a, b):
    n = max(len(e1), len(e2))
    x1 = np.zeros(n)
    x1[: len(e1)] = e1
    x2 = np.zeros(n)
    x2[: len(e2)] = e2
    mixed = _whole(scatter_convolve(_sig(a * x1 + b * x2), _sig(h)))
    separate = a * _whole(scatter_convolve(_sig(x1), _sig(h))) + b * _whole(scatter_convolve(_sig(x2), _sig(h)))
    _near(mixed, separate, 1e-10)


@given(e=_SEQ, h=_SEQ, k=st.integers(min_value=1, max_value=16))
def test_time_invariance_bit_exact(e, h, k):
    base = _whole(scatter_convolve(_sig(e), _sig(h)))
    shifted = _whole(scatter_convolve(_sig([0.0] * k + e), _sig(h)))
    assert np.array_equal(shifted[:k], np.zeros(k)) and np.array_equal(shifted[k:], base)


@given(h=_SEQ)
def test_unit_impulse_bit_exact(h):
    assert np.array_equal(_whole(scatter_convolve(_sig([1.0]), _sig(h))), np.asarray(h))


@given(e=_SEQ, h=_SEQ, threshold=st.floats(min_value=0, max_value=0.5, width=64))
def test_skip_threshold_equals_thresholded_input(e, h, threshold):
    skipped = _whole(scatter_convolve_skip_zeros(_sig(e), _sig(h), threshold=threshold))
    gated = np.where(np.abs(np.asarray(e)) <= threshold, 0.0, np.asarray(e))
    assert np.array_equal(skipped, _whole(scatter_convolve(_sig(gated), _sig(h))))


# ---------------------------------------------------------------- float32 fast path

F32_CASES = [(1, 1), (1, 5000), (5000, 1), (3, 2), (8192, 64), (8193, 65), (10000, 3000),
             (100_000, 4097), (30_000, 70_000), (20_000, 100_000), (200_000, 1023), (65, 8191)]


@pytest.mark.parametrize("ne,nh", F32_CASES)
def test_fast_f32_within_tolerance(ne, nh):
    rng = np.random.default_rng(ne * 7 + nh)
    x = rng.uniform(-1, 1, ne).astype(np.float32)
    h = (rng.standard_normal(nh) * np.exp(-np.arange(nh) / max(1.0, nh / 4))).astype(np.float32)
    y = _whole(scatter_convolve(Signal(x), Signal(h)))
    assert y.dtype == np.float32 and len(y) == ne + nh - 1
    ref = O.scatter_window(x, h, 0, ne + nh - 1)
    within_tol(y, ref, x, h)


@pytest.mark.parametrize("ne,nh", [(1, 1), (4000, 333), (20_000, 2048)])
def test_ordered_f32_within_tolerance(ne, nh):
    rng = np.random.default_rng(ne + 3 * nh)
    x = rng.uniform(-1, 1, ne).astype(np.float32)
    h = rng.standard_normal(nh).astype(np.float32)
    y = _whole(scatter_convolve(Signal(x), Signal(h), mode="ordered"))
    within_tol(y, O.scatter_full(x, h), x, h)


def test_fast_f32_is_deterministic_and_tensor_resident():
    import torch

    rng = np.random.default_rng(1)
    x = torch.from_numpy(rng.uniform(-1, 1, 50_000).astype(np.float32)).cuda()
    h = torch.from_numpy(rng.standard_normal(9000).astype(np.float32)).cuda()
    a = scatter_convolve(Signal(x), Signal(h)).concatenated().samples
    b = scatter_convolve(Signal(x), Signal(h)).concatenated().samples
    assert a.is_cuda and a.dtype == torch.float32
    assert torch.equal(a, b)


def test_fast_f32_nan_propagates_like_reference():
    x = np.zeros(20_000, np.float32)
    x[5] = np.nan
    x[100] = 1.0
    h = np.ones(300, np.float32)
    y = _whole(scatter_convolve(Signal(x), Signal(h)))
    ref = O.scatter_full(x, h)
    assert np.array_equal(np.isnan(y), np.isnan(ref))


def test_batched_matches_oracle_per_channel():
    rng = np.random.default_rng(9)
    C, ne, nh = 5, 3000, 1500
    x = rng.uniform(-1, 1, (C, ne)).astype(np.float32)
    h = rng.standard_normal((C, nh)).astype(np.float32)
    y = convolve_batched(x, h)
    assert y.shape == (C, ne + nh - 1)
    for c in range(C):
        within_tol(y[c], O.scatter_full(x[c], h[c]), x[c], h[c])
    yb = convolve_batched(x, h[0])  # mono IR broadcast
    within_tol(yb[3], O.scatter_full(x[3], h[0]), x[3], h[0])


def test_shards_reassemble_full_output():
    import torch

    rng = np.random.default_rng(4)
    x = rng.uniform(-1, 1, 40_000).astype(np.float32)
    h = rng.standard_normal(5000).astype(np.float32)
    hd = torch.from_numpy(h).cuda()
    parts = []
    for sh in shard_plan(len(x), len(h), 8):
        xs = torch.from_numpy(x[sh.x_begin:sh.x_end]).cuda()
        parts.append(convolve_shard(xs, sh, hd).cpu().numpy())
    y = np.concatenate(parts)
    within_tol(y, O.scatter_full(x, h), x, h)
