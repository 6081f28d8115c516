"""Device measurement harness on the GPU: its outputs are the reference's
(digests of the reference's own run_ir_sweep / run_nb_sweep, tests/golden/
ref_sweeps.json) and its device timings behave like a linear-cost engine."""

import json

import numpy as np
import pytest

from paper_2401_01607_b200.sweeps import SweepSpec, gen_white_noise, run_ir_sweep, run_nb_sweep
from tests._golden import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pins():
    return json.loads((GOLDEN / "ref_sweeps.json").read_text())


def test_ir_sweep_digest_equals_reference(pins):
    p = pins["ir_sweep"]
    x = gen_white_noise(p["n"], p["rate"], seed=tuple(p["seed"]))
    rep = run_ir_sweep(SweepSpec(p["ir_lengths"], x, repetitions=1, rng_seed=p["rng_seed"]))
    assert rep.output_digest == p["digest"]
    assert len(rep.rows) == 3 and all(r.wall_time_s > 0 and r.nb == 8192 for r in rep.rows)
    assert rep.linear_fit is not None and 0.0 <= rep.linear_fit.r_squared <= 1.0
    par = run_ir_sweep(SweepSpec(p["ir_lengths"], x, repetitions=1, rng_seed=p["rng_seed"]), parallel=True)
    assert par.output_digest == p["digest"]


def test_nb_sweep_digest_equals_reference(pins):
    p = pins["nb_sweep"]
    x = gen_white_noise(3000, 8000, seed=(77, 1))
    rep = run_nb_sweep(SweepSpec(p["ir_lengths"], x, nb_values=p["nb_values"], repetitions=2,
                                 rng_seed=p["rng_seed"]))
    assert rep.output_digest == p["digest"]
    assert len(rep.rows) == 6 and rep.nb_spread_percent >= 0.0


def test_device_cost_is_linear_in_ir_length():
    # large enough that the fused stream (not the fixed flush/launch cost) dominates
    x = gen_white_noise(1_500_000, 44100, seed=12)
    rep = run_ir_sweep(SweepSpec([8000, 16000, 32000], x, repetitions=3, rng_seed=7))
    med = rep.median_wall_times()
    assert 1.5 <= med[16000] / med[8000] <= 2.5
    assert 1.5 <= med[32000] / med[16000] <= 2.5
    assert rep.linear_fit.r_squared >= 0.98
    # every length runs far faster than real time on a B200
    assert rep.limit_filter_length is None
    assert np.all([r.realtime_ratio < 1.0 for r in rep.rows])
