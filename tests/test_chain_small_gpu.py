"""k_chain_small (csrc/k_ordered.cu): the latency kernel for small strict
float64 convolutions of one IR (cfg1 class).  Its chains take a padded,
fixed number of steps (zero taps / zero drive outside the reference's loop
bounds), so these tests pin it bit-exact against the CPU oracle
(oracle/scatter_oracle.c, the reference's _scatter_full order,
core.py:80-92) across IR lengths that are and are not multiples of 8, the
16-chunk maximum, signals shorter than the IR, signed zeros, and non-finite
operands next to the padded steps (where a padded 0*inf would be NaN and the
kernel must take its bounded path instead).
"""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2401_01607_b200 import _native as N
from paper_2401_01607_b200.core import Signal, scatter_convolve

pytestmark = pytest.mark.gpu


def _conv(x, h):
    return np.asarray(scatter_convolve(Signal(np.asarray(x, np.float64)), Signal(np.asarray(h, np.float64)))
                      .concatenated().samples)


def _bits_equal(a, b):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape
    nan = np.isnan(a) & np.isnan(b)
    assert np.array_equal(np.isnan(a), np.isnan(b)), "NaN positions differ"
    assert np.array_equal(a.view(np.uint64)[~nan], b.view(np.uint64)[~nan]), "not bit-identical"


@pytest.mark.parametrize("ne,nh", [(1, 1), (5, 3), (100, 1), (3000, 7), (3000, 8), (3000, 9), (20_000, 1024),
                                   (48_000, 1024), (700, 2048), (10_000, 2047), (17, 2000), (9000, 129)])
def test_small_chain_bit_exact(ne, nh):
    rng = np.random.default_rng(ne * 7919 + nh)
    x = rng.uniform(-1, 1, ne)
    h = rng.standard_normal(nh) * np.exp(-np.arange(nh) / max(1.0, nh / 5))
    _bits_equal(_conv(x, h), O.scatter_full(x, h))


def test_small_chain_signed_zeros():
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, 4000)
    x[::7] = -0.0
    x[1::11] = 0.0
    h = rng.standard_normal(301)
    h[::5] = -0.0
    _bits_equal(_conv(x, h), O.scatter_full(x, h))
    # an all-(-0) drive: every reference chain is +0 + (-0) ... = +0
    _bits_equal(_conv(np.full(50, -0.0), -np.ones(13)), O.scatter_full(np.full(50, -0.0), -np.ones(13)))


@pytest.mark.parametrize("where", ["x_head", "x_tail", "x_mid", "h_head", "h_tail", "h_mid"])
@pytest.mark.parametrize("val", [np.inf, -np.inf, np.nan])
def test_small_chain_nonfinite_next_to_padding(where, val):
    rng = np.random.default_rng(11)
    ne, nh = 6000, 1021  # nh not a multiple of 8: 3 padded front steps per chain
    x = rng.uniform(-1, 1, ne)
    h = rng.standard_normal(nh)
    if where == "x_head":
        x[0] = val
    elif where == "x_tail":
        x[-1] = val
    elif where == "x_mid":
        x[ne // 2] = val
    elif where == "h_head":
        h[0] = val
    elif where == "h_tail":
        h[-1] = val
    else:
        h[nh // 2] = val
    _bits_equal(_conv(x, h), O.scatter_full(x, h))


def test_small_chain_matches_windowed_chain(tmp_path):
    """The same cfg1-shape launch with k_chain_small disabled
    (SC_CHAIN_SMALL=0: the windowed k_chain_w) gives the same bits."""
    import os
    import subprocess
    import sys

    rng = np.random.default_rng(5)
    x, h = rng.uniform(-1, 1, 48_000), rng.standard_normal(1024) * np.exp(-np.arange(1024) / 200)
    np.save(tmp_path / "x.npy", x)
    np.save(tmp_path / "h.npy", h)
    code = (
        "import numpy as np, sys; sys.path.insert(0, %r)\n"
        "from paper_2401_01607_b200.core import Signal, scatter_convolve\n"
        "x = np.load(%r); h = np.load(%r)\n"
        "np.save(%r, np.asarray(scatter_convolve(Signal(x), Signal(h)).concatenated().samples))\n"
    ) % (os.getcwd(), str(tmp_path / "x.npy"), str(tmp_path / "h.npy"), str(tmp_path / "y.npy"))
    env = dict(os.environ, SC_CHAIN_SMALL="0")
    subprocess.run([sys.executable, "-c", code], check=True, env=env)
    _bits_equal(_conv(x, h), np.load(tmp_path / "y.npy"))


@pytest.mark.parametrize("thr", [0.0, 0.3])
@pytest.mark.parametrize("case", ["plain", "x_nonfinite", "h_inf"])
def test_small_chain_skip_zeros_bit_exact(thr, case):
    """scatter_convolve_skip_zeros (core.py:150-167, skip |x| <= threshold,
    NaN not skipped) through k_chain_small: skipped samples are zeroed in the
    staged window (exact with finite taps); a non-finite tap sends every CTA
    to the bounded loop, which reads and skips the drive itself."""
    from paper_2401_01607_b200.core import scatter_convolve_skip_zeros

    rng = np.random.default_rng(17)
    ne, nh = 5000, 777
    x = rng.uniform(-1, 1, ne)
    x[::5] = 0.0
    x[1::9] = -0.0
    h = rng.standard_normal(nh)
    if case == "x_nonfinite":
        x[3] = np.inf        # |inf| > thr: scatters
        x[2500] = np.nan     # NaN is not skipped here: propagates
    if case == "h_inf":
        h[100] = np.inf
    got = np.asarray(scatter_convolve_skip_zeros(Signal(x), Signal(h), threshold=thr).concatenated().samples)
    _bits_equal(got, O.scatter_full(x, h, skip_mode=O.SKIP_LE, threshold=thr))
