"""Host logic of the device measurement harness (paper_2401_01607_b200.sweeps,
the drop-in for scatterconv.bench): generators, validation, the real-time
limit, the linear fit and the report formats -- modelled on the reference's
pkg/tests/test_bench.py.  CPU only."""

import numpy as np
import pytest

from paper_2401_01607_b200.sweeps import (
    CSV_HEADER,
    BenchReport,
    BenchRow,
    SweepSpec,
    _least_squares as _fit_line,
    find_realtime_limit,
    gen_white_noise,
    ms_to_samples,
)


def test_noise_deterministic_and_in_range():
    a = gen_white_noise(1000, seed=42)
    assert np.array_equal(a.samples, gen_white_noise(1000, seed=42).samples)
    assert not np.array_equal(a.samples, gen_white_noise(1000, seed=43).samples)
    s = gen_white_noise(44100, 44100, seed=0)
    assert s.duration_s == 1.0 and np.all(s.samples >= -1.0) and np.all(s.samples < 1.0)
    with pytest.raises(ValueError, match="duration"):
        gen_white_noise(0)


def test_ms_to_samples():
    assert ms_to_samples(100, 44100) == 4410
    assert ms_to_samples(10.5, 8000) == 84
    with pytest.raises(ValueError, match="positive"):
        ms_to_samples(0, 44100)


def test_sweep_spec_validation():
    x = gen_white_noise(100, 8000)
    for bad, match in (({"ir_lengths": []}, "ir_lengths"), ({"ir_lengths": [0]}, "ir_lengths"),
                       ({"nb_values": []}, "nb_values"), ({"nb_values": [0]}, "nb_values"),
                       ({"repetitions": 0}, "repetitions")):
        kw = {"ir_lengths": [10], "input_signal": x, **bad}
        with pytest.raises(ValueError, match=match):
            SweepSpec(**kw)
    with pytest.raises(ValueError, match="input_signal"):
        SweepSpec([10], x.samples)


def synthetic(rows, d=10.0):
    return BenchReport([BenchRow(n, 8192, 0, w, w / d) for n, w in rows], d)


def test_realtime_limit_cases():
    d = 10.0
    for dur in (10.0, 2.5, 129.0):
        assert find_realtime_limit(synthetic([(1000, 0.5 * dur), (3000, 1.5 * dur)], dur), dur) == 2000.0
    assert find_realtime_limit(synthetic([(1000, 1.0), (3000, 2.0)]), d) is None
    assert find_realtime_limit(synthetic([(500, 12.0), (900, 20.0)]), d) == 500.0
    assert find_realtime_limit(synthetic([(100, 2.0), (200, 10.0), (400, 30.0)]), d) == 200.0
    rows = [BenchRow(3000, 8192, 0, 14.0, 1.4), BenchRow(1000, 8192, 0, 4.0, 0.4),
            BenchRow(3000, 8192, 1, 16.0, 1.6), BenchRow(1000, 8192, 1, 6.0, 0.6)]
    assert find_realtime_limit(BenchReport(rows, d), d) == 2000.0
    with pytest.raises(ValueError, match="distinct"):
        find_realtime_limit(synthetic([(1000, 5.0), (1000, 6.0)]), d)
    with pytest.raises(ValueError, match="input_duration"):
        find_realtime_limit(synthetic([(1000, 5.0), (2000, 6.0)]), 0.0)


def test_linear_fit():
    assert _fit_line([5, 5], [1.0, 2.0]) is None
    fit = _fit_line([1, 2, 3, 4], [2.0, 4.0, 6.0, 8.0])
    assert fit.slope == pytest.approx(2.0) and fit.intercept == pytest.approx(0.0, abs=1e-12)
    assert fit.r_squared == pytest.approx(1.0)
    noisy = _fit_line([1, 2, 3, 4], [1.0, 3.0, 2.0, 4.0])
    ref = np.polyfit([1, 2, 3, 4], [1.0, 3.0, 2.0, 4.0], 1)
    assert noisy.slope == pytest.approx(ref[0]) and 0.0 <= noisy.r_squared <= 1.0


def test_report_csv_and_plot(tmp_path):
    rep = BenchReport([BenchRow(10, 8192, 0, 0.5, 0.05), BenchRow(20, 8192, 0, 1.0, 0.1),
                       BenchRow(10, 8192, 1, 0.7, 0.07)], 10.0)
    text = rep.to_csv()
    lines = text.splitlines()
    assert lines[0] == CSV_HEADER == "ir_samples,nb,rep,wall_time_s,realtime_ratio"
    assert len(lines) == 4 and text.endswith("\n") and "\r" not in text
    assert rep.median_wall_times() == {10: pytest.approx(0.6), 20: 1.0}
    p = tmp_path / "rows.csv"
    rep.write_csv(p)
    assert p.read_bytes().decode() == text
    q = tmp_path / "curve.dat"
    rep.write_plot_data(q)
    pl = q.read_text().splitlines()
    assert pl[0].startswith("#") and len(pl) == 3 and pl[1].split()[0] == "10"
