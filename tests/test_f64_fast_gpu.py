"""float64 FAST mode: the ordered chain with one fused multiply-add per step
(csrc/k_ordered.cu mac_step<true>).  North_star's FP64 bar: max-abs error
<= 1e-12 * max|x| * ||h||_1 against the reference (the oracle, float64,
separately rounded).  The chain order is kept, so stream == batch holds
bit-exactly inside the mode."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _tol(x, h):
    return 1e-12 * float(np.max(np.abs(x))) * float(np.sum(np.abs(h)))


@pytest.mark.parametrize("ne,nh", [(48_000, 1_024), (1, 5), (7, 300), (20_011, 4_097), (300_000, 64)])
def test_f64_fast_within_1e12(ne, nh):
    from paper_2401_01607_b200.core import Signal, scatter_convolve

    rng = np.random.default_rng(ne + nh)
    x = rng.uniform(-1, 1, ne)
    h = rng.standard_normal(nh) * np.exp(-np.arange(nh) / max(1, nh / 4))
    fast = scatter_convolve(Signal(x), Signal(h), mode="fast").concatenated().samples
    ordered = scatter_convolve(Signal(x), Signal(h)).concatenated().samples
    ref = O.scatter_full(x, h)
    assert np.array_equal(ordered, ref)                       # default stays bit-exact
    assert np.max(np.abs(fast - ref)) <= _tol(x, h)
    if ne * nh > 10_000:
        assert not np.array_equal(fast, ref)                  # really the fused kernel


def test_f64_fast_engine_stream_equals_blocks_and_oracle():
    import torch

    from paper_2401_01607_b200.core import Signal
    from paper_2401_01607_b200.engine import EngineConfig, ScatterEngine

    rng = np.random.default_rng(5)
    x = rng.uniform(-1, 1, 50_000)
    x[rng.uniform(size=50_000) < 0.2] = 0.0
    h0, h1 = rng.standard_normal(700), rng.standard_normal(1_300)
    nb = 1000
    a = ScatterEngine(Signal(h0), EngineConfig(block_size_nb=nb), mode="fast")
    assert a.mode == "fast"
    blocks = []
    for b, s in enumerate(range(0, len(x), nb)):
        if b == 20:
            a.swap_ir(Signal(h1))
        blocks.append(a.process_block(Signal(x[s:s + nb])).samples)
    blocks.append(a.flush().samples)
    by_block = np.concatenate(blocks)
    f = ScatterEngine(Signal(torch.from_numpy(h0).cuda()), EngineConfig(block_size_nb=nb), mode="fast")
    body = f.process_stream(torch.from_numpy(x).cuda(), nb, [(20, torch.from_numpy(h1).cuda())])
    fused = np.concatenate([body.cpu().numpy(), f.flush().samples.cpu().numpy()])
    assert np.array_equal(fused, by_block)                    # stream == batch within the mode
    eng = O.OracleEngine(h0, nb)
    ref = []
    for b, s in enumerate(range(0, len(x), nb)):
        if b == 20:
            eng.swap_ir(h1)
        ref.append(eng.process_block(x[s:s + nb]))
    ref.append(eng.flush())
    ref = np.concatenate(ref)
    assert len(ref) == len(by_block)
    assert np.max(np.abs(by_block - ref)) <= max(_tol(x, h0), _tol(x, h1))
