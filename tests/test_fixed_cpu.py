"""Fixed-point simulation, host side (no GPU): the C oracle pinned against the
reference's own fixed_point_convolve outputs (tests/golden/ref_fixed.npz,
written by make_golden.py from pkg/src/scatterconv/quantize.py), the closed
forms and validation of quantize.py:34-134, and the `quant` CLI lines that
need no simulation (cli.py:286-293)."""

from __future__ import annotations

import contextlib
import io
import json
import pathlib

import numpy as np
import pytest

from oracle import oracle
from paper_2401_01607_b200 import fixed_point as fx
from paper_2401_01607_b200.__main__ import main

GOLD = pathlib.Path(__file__).parent / "golden"
REF = np.load(GOLD / "ref_fixed.npz")
META = json.loads((GOLD / "ref_fixed.json").read_text())
CASES = sorted({k.split("/")[0] for k in REF.files})
BITS = sorted({int(k.split("/")[1]) for k in REF.files if k.count("/") == 2})


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("scheme", ["ideal", "mac"])
def test_oracle_matches_reference(case, scheme):
    e, h = REF[f"{case}/e"], REF[f"{case}/h"]
    for bits in BITS:
        got = oracle.fixed_convolve(e, h, bits, scheme)
        np.testing.assert_array_equal(got.view(np.int64), REF[f"{case}/{bits}/{scheme}"].view(np.int64),
                                      err_msg=f"{case} {bits}-bit {scheme}")


def test_oracle_quantize_edges():
    k = oracle.fixed_quantize([-1.0, 1.0 - 2.0 ** -40, 0.5, 3 / 16, 5 / 16, -3 / 16], 4)
    # 3/16*8 = 1.5 -> 2, 5/16*8 = 2.5 -> 2, -1.5 -> -2 (half to even); 1-eps saturates to 7
    assert k.tolist() == [-8, 7, 4, 2, 2, -2]
    with pytest.raises(ValueError, match=r"outside the representable range \[-1, 1\)"):
        oracle.fixed_quantize([0.0, 1.0], 8)


def test_closed_forms():
    assert fx.ideal_accumulator_bits(16, 32) == 63
    assert fx.ideal_bits_removed(16, 32) == 47
    assert fx.mac_requant_count(16, 32) == (31, 16)
    assert fx.mac_requant_count(2, 1) == (0, 2)
    for fn in (fx.ideal_accumulator_bits, fx.ideal_bits_removed, fx.mac_requant_count):
        with pytest.raises(ValueError, match="word length must be an integer >= 2 bits"):
            fn(1, 4)
        with pytest.raises(ValueError, match="impulse response length must be a positive integer"):
            fn(8, 0)
        with pytest.raises(ValueError, match="word length"):
            fn(8.0, 4)


def test_format_and_report_validation():
    f = fx.FixedPointFormat(16)
    assert (f.fractional_bits, f.scale, f.min_int, f.max_int, f.ulp) == (15, 32768, -32768, 32767, 1 / 32768)
    with pytest.raises(ValueError, match="word_bits must be an integer >= 2"):
        fx.FixedPointFormat(1)
    with pytest.raises(ValueError, match="rounding must be one of"):
        fx.FixedPointFormat(8, rounding="truncate")
    with pytest.raises(ValueError, match="overflow must be one of"):
        fx.FixedPointFormat(8, overflow="wrap")
    with pytest.raises(ValueError, match="scheme must be one of"):
        fx.RequantReport("exact", 1, 1, 0.0, 0.0)
    with pytest.raises(ValueError, match="counts must be non-negative"):
        fx.RequantReport("mac", -1, 1, 0.0, 0.0)
    with pytest.raises(ValueError, match="exceeds max_error"):
        fx.RequantReport("mac", 1, 1, 2.0, 1.0)


def _cli(argv):
    o, e = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(o), contextlib.redirect_stderr(e):
        rc = main(argv)
    return rc, o.getvalue(), e.getvalue()


@pytest.mark.parametrize("name", [k for k, v in META["cli"].items() if "--simulate" not in v["argv"]
                                  or v["rc"] != 0])
def test_quant_cli_without_simulation(name):
    ref = META["cli"][name]
    assert _cli(ref["argv"]) == (ref["rc"], ref["stdout"], ref["stderr"])


@pytest.mark.parametrize("argv", [
    ["bench", "--ir-sweep", "1:2"],
    ["bench", "--ir-sweep", "a:2:1"],
    ["bench", "--ir-sweep", "3:2:1"],
    ["bench", "--ir-sweep", "1:2:0"],
    ["bench", "--nb-sweep", "4,x"],
    ["bench", "--nb-sweep", "4,0"],
    ["bench", "--nb-sweep", ","],
    ["quant", "--bits", "8"],
])
def test_cli_arg_errors(argv):
    assert _cli(argv)[0] == 2


def test_ir_sweep_range_no_drift():
    from paper_2401_01607_b200.__main__ import _ms_range

    assert _ms_range("0.1:0.7:0.1") == [0.1 + i * 0.1 for i in range(7)]
    assert _ms_range("5:5:1") == [5.0]


def test_bench_cli_errors_before_gpu():
    ref = json.loads((GOLD / "ref_cli_bench.json").read_text())
    for name in ("nothing", "bad_input"):
        rc, _, err = _cli(ref[name]["argv"])
        assert (rc, err) == (ref[name]["rc"], ref[name]["stderr"])
