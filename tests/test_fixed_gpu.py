"""Device fixed-point simulation (csrc/k_fixed.cu) against the reference's
fixed_point_convolve / simulate_fixed_point_conv outputs and the `quant`
CLI's stdout (tests/golden/ref_fixed.*), plus the C oracle at sizes the
reference's Python loops would take minutes on.  Integer work: bit-exact."""

from __future__ import annotations

import contextlib
import io
import json
import pathlib

import numpy as np
import pytest

from oracle import oracle

pytestmark = pytest.mark.gpu

GOLD = pathlib.Path(__file__).parent / "golden"
REF = np.load(GOLD / "ref_fixed.npz")
META = json.loads((GOLD / "ref_fixed.json").read_text())
CASES = sorted({k.split("/")[0] for k in REF.files})
BITS = sorted({int(k.split("/")[1]) for k in REF.files if k.count("/") == 2})


def _bits(a):
    return np.asarray(a, dtype=np.float64).view(np.int64)


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("scheme", ["ideal", "mac"])
def test_fixed_point_convolve_golden(case, scheme):
    from paper_2401_01607_b200 import fixed_point as fx
    from paper_2401_01607_b200.core import Signal

    e, h = REF[f"{case}/e"], REF[f"{case}/h"]
    for bits in BITS:
        y = fx.fixed_point_convolve(Signal(e, 48000), Signal(h, 48000), fx.FixedPointFormat(bits), scheme)
        assert isinstance(y.samples, np.ndarray) and y.sample_rate == 48000
        np.testing.assert_array_equal(_bits(y.samples), _bits(REF[f"{case}/{bits}/{scheme}"]),
                                      err_msg=f"{case} {bits}-bit {scheme}")


def test_simulate_reports_golden():
    from paper_2401_01607_b200 import fixed_point as fx
    from paper_2401_01607_b200.core import Signal

    for key, (ops, bits_removed, rms, mx) in META["reports"].items():
        case, bits, scheme = key.split("/")
        r = fx.simulate_fixed_point_conv(Signal(REF[f"{case}/e"], 48000), Signal(REF[f"{case}/h"], 48000),
                                         fx.FixedPointFormat(int(bits)), scheme)
        assert (r.scheme, r.operations_count, r.bits_removed_per_op) == (scheme, ops, bits_removed)
        assert r.rms_error == rms and r.max_error == mx, key


@pytest.mark.parametrize("name", [k for k, v in META["cli"].items() if "--simulate" in v["argv"]])
def test_quant_cli_simulate_stdout(name):
    from paper_2401_01607_b200.__main__ import main

    ref = META["cli"][name]
    o, e = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(o), contextlib.redirect_stderr(e):
        rc = main(ref["argv"])
    assert (rc, o.getvalue(), e.getvalue()) == (ref["rc"], ref["stdout"], ref["stderr"])


@pytest.mark.parametrize("bits", [8, 16, 24, 32])
@pytest.mark.parametrize("scheme", ["ideal", "mac"])
def test_large_vs_oracle(bits, scheme):
    """20k x 700 taps: minutes in the reference's Python loops, a few ms here."""
    from paper_2401_01607_b200 import fixed_point as fx
    from paper_2401_01607_b200.core import Signal

    rng = np.random.default_rng(bits * 7 + len(scheme))
    e = rng.uniform(-1, 1, 20000)
    h = rng.uniform(-1, 1, 700) * np.exp(-np.arange(700) / 150.0)
    y = fx.fixed_point_convolve(Signal(e), Signal(h), fx.FixedPointFormat(bits), scheme).samples
    np.testing.assert_array_equal(_bits(y), _bits(oracle.fixed_convolve(e, h, bits, scheme)))


def test_quantize_device_vs_oracle_and_tensor_currency():
    import torch

    from paper_2401_01607_b200 import fixed_point as fx

    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, 100_003)
    x[:6] = [-1.0, 1.0 - 2.0 ** -53, 0.5, 3 / 16, 5 / 16, -3 / 16]
    for bits in (2, 4, 16, 33, 53, 64):
        q = fx.quantize(x, fx.FixedPointFormat(bits))
        assert isinstance(q, np.ndarray)
        want = oracle.fixed_quantize(x, bits) / float(1 << (bits - 1))
        np.testing.assert_array_equal(_bits(q), _bits(want))
    qt = fx.quantize(torch.from_numpy(x).cuda(), fx.FixedPointFormat(12))
    assert qt.is_cuda
    np.testing.assert_array_equal(_bits(qt.cpu().numpy()), _bits(fx.quantize(x, fx.FixedPointFormat(12))))


def test_errors():
    from paper_2401_01607_b200 import fixed_point as fx
    from paper_2401_01607_b200.core import Signal

    f8 = fx.FixedPointFormat(8)
    with pytest.raises(ValueError, match=r"outside the representable range \[-1, 1\)"):
        fx.quantize(np.array([0.2, 1.0]), f8)
    with pytest.raises(ValueError, match=r"outside the representable range"):
        fx.fixed_point_convolve(Signal(np.array([-1.5])), Signal(np.array([0.5])), f8, "ideal")
    with pytest.raises(ValueError, match="scheme must be one of"):
        fx.fixed_point_convolve(Signal(np.array([0.5])), Signal(np.array([0.5])), f8, "exact")
    with pytest.raises(ValueError, match="empty signal"):
        fx.fixed_point_convolve(Signal(np.zeros(0)), Signal(np.array([0.5])), f8, "mac")
    with pytest.raises(ValueError, match="sample rates differ"):
        fx.fixed_point_convolve(Signal(np.array([0.5]), 8000), Signal(np.array([0.5]), 16000), f8, "mac")
    # 64-bit words over long sums exceed the 128-bit accumulator: refused, not wrapped
    with pytest.raises(ValueError, match="accumulator"):
        fx.fixed_point_convolve(Signal(np.full(64, -1.0)), Signal(np.full(64, -1.0)), fx.FixedPointFormat(64),
                                "ideal")


def test_wide_words_exact():
    """48- and 60-bit words take the 64x64->128 product path; still exact
    (checked against Python integers on a small case)."""
    from paper_2401_01607_b200 import fixed_point as fx
    from paper_2401_01607_b200.core import Signal

    rng = np.random.default_rng(9)
    e, h = rng.uniform(-1, 1, 9), rng.uniform(-1, 1, 5)
    for bits in (48, 60):
        frac = bits - 1
        ke = [int(v) for v in np.clip(np.round(e * 2.0 ** frac), -2 ** frac, 2 ** frac - 1)]
        kh = [int(v) for v in np.clip(np.round(h * 2.0 ** frac), -2 ** frac, 2 ** frac - 1)]

        def rs(t):   # half-even right shift by frac (Python ints)
            q, r = t >> frac, t & ((1 << frac) - 1)
            half = 1 << (frac - 1)
            return q + (1 if r > half or (r == half and q & 1) else 0)

        want_ideal, want_mac = [], []
        for n in range(len(ke) + len(kh) - 1):
            lo, hi = max(0, n - len(kh) + 1), min(n, len(ke) - 1)
            want_ideal.append(rs(sum(ke[m] * kh[n - m] for m in range(lo, hi + 1))) / 2 ** frac)
            if lo == hi:
                c = rs(ke[lo] * kh[n - lo])
            else:
                c = rs(ke[lo] * kh[n - lo] + ke[lo + 1] * kh[n - lo - 1])
                for m in range(lo + 2, hi + 1):
                    c = rs((c << frac) + ke[m] * kh[n - m])
            want_mac.append(c / 2 ** frac)
        f = fx.FixedPointFormat(bits)
        got_i = fx.fixed_point_convolve(Signal(e), Signal(h), f, "ideal").samples
        got_m = fx.fixed_point_convolve(Signal(e), Signal(h), f, "mac").samples
        np.testing.assert_array_equal(_bits(got_i), _bits(want_ideal))
        np.testing.assert_array_equal(_bits(got_m), _bits(want_mac))


def test_bench_cli_digests():
    """The `bench` CLI on the device harness prints the reference's output
    digests and writes the same CSV / plot-data shapes."""
    from paper_2401_01607_b200.__main__ import main

    ref = json.loads((GOLD / "ref_cli_bench.json").read_text())
    import tempfile

    with tempfile.TemporaryDirectory() as tmp:
        for name, r in ref.items():
            argv = [a.replace("{tmp}", tmp) for a in r["argv"]]
            o, e = io.StringIO(), io.StringIO()
            with contextlib.redirect_stdout(o), contextlib.redirect_stderr(e):
                rc = main(argv)
            stable = [ln.split(": wall-time")[0] for ln in o.getvalue().splitlines()
                      if "sha256" in ln or ln.startswith("wrote") or ln.startswith("nb sweep at")]
            assert rc == r["rc"], name
            assert stable == [s.replace("/tmp", tmp) for s in r["stable"]], name
            assert e.getvalue() == r["stderr"], name
        csv = (pathlib.Path(tmp) / "x.csv").read_text().splitlines()
        assert csv[0] == "ir_samples,nb,rep,wall_time_s,realtime_ratio" and len(csv) == 6
        assert (pathlib.Path(tmp) / "p.dat").read_text().startswith("# ir_samples")
