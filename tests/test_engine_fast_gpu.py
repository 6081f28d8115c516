"""Float32 FAST fused streams (csrc/engine.cu fast_stream): every IR segment
with >= 2^30 MACs is convolved on the tensor-core FIR path and combined with
the residue.  Checked against the float64 oracle engine (tolerance
1e-5 * max|x| * ||h||_1 per channel, the FP32 bar) and against the ordered
engine for the data-dependent state (live / cap / read_index, tail lengths)
and the NaN/Inf pattern."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle

pytestmark = pytest.mark.gpu


def _tol(x, h):
    return 1e-5 * float(np.max(np.abs(x))) * float(np.sum(np.abs(h)))


def _oracle_stream(x, irs_at, nb, thr=0.0):
    """float64 reference engine over blocks of nb with swaps {block: h}."""
    eng = oracle.OracleEngine(irs_at[0].astype(np.float64), nb, thr)
    out = []
    for b, s in enumerate(range(0, len(x), nb)):
        if b in irs_at and b > 0:
            eng.swap_ir(irs_at[b].astype(np.float64))
        out.append(eng.process_block(x[s:s + nb].astype(np.float64)))
    return np.concatenate(out), eng.flush()


def test_single_channel_fast_vs_oracle_and_ordered():
    import torch

    from paper_2401_01607_b200.core import Signal
    from paper_2401_01607_b200.engine import EngineConfig, ScatterEngine

    rng = np.random.default_rng(11)
    n, nh, nb = 1 << 20, 4096, 8192
    x = rng.uniform(-1, 1, n).astype(np.float32)
    x[rng.uniform(size=n) < 0.1] = 0.0           # skipped samples
    x[1000:1010] = np.nan                         # engine skips NaN
    h0 = (rng.standard_normal(nh) * np.exp(-np.arange(nh) / 700)).astype(np.float32)
    h1 = (rng.standard_normal(3000) * np.exp(-np.arange(3000) / 500)).astype(np.float32)
    swap_block = (n // nb) // 2                   # 2 segments of 2^19 x ~4k taps: > 2^30 MACs each
    outs, tails, states = {}, {}, {}
    for mode in ("fast", "ordered"):
        eng = ScatterEngine(Signal(torch.from_numpy(h0).cuda()), EngineConfig(block_size_nb=nb,
                                                                             zero_skip_threshold=0.0),
                            mode=mode)
        assert eng.mode == mode
        body = eng.process_stream(torch.from_numpy(x).cuda(), nb, [(swap_block, torch.from_numpy(h1).cuda())])
        states[mode] = eng.state_dict()["live"], eng._state()["cap"], eng._state()["read_index"]
        tails[mode] = eng.flush().samples.cpu().numpy()
        outs[mode] = body.cpu().numpy()
    ref_body, ref_tail = _oracle_stream(x, {0: h0, swap_block: h1}, nb)
    tol = max(_tol(np.nan_to_num(x), h0), _tol(np.nan_to_num(x), h1))
    assert states["fast"] == states["ordered"]
    assert len(tails["fast"]) == len(tails["ordered"]) == len(ref_tail)
    for mode in ("fast", "ordered"):
        assert np.max(np.abs(outs[mode] - ref_body)) <= tol, mode
        assert np.max(np.abs(tails[mode] - ref_tail)) <= tol, mode
    assert not np.array_equal(outs["fast"], outs["ordered"])   # really a different kernel


def test_multichannel_fast_residue_carry_and_threshold():
    import torch

    from paper_2401_01607_b200.engine import EngineConfig
    from paper_2401_01607_b200.multichannel import MultiChannelEngine

    rng = np.random.default_rng(12)
    C, n, nh, nb, thr = 8, 1 << 18, 2048, 4096, 0.05
    x = rng.uniform(-1, 1, (C, n)).astype(np.float32)
    h = (rng.standard_normal((C, nh)) * np.exp(-np.arange(nh) / 300)).astype(np.float32)
    eng = MultiChannelEngine(torch.from_numpy(h).cuda(), EngineConfig(block_size_nb=nb, zero_skip_threshold=thr))
    assert eng.mode == "fast"
    # two calls: the second continues from the residue of the first
    half = n // 2
    b1 = eng.process_stream(torch.from_numpy(x[:, :half]).cuda(), nb).cpu().numpy()
    b2 = eng.process_stream(torch.from_numpy(x[:, half:]).cuda(), nb).cpu().numpy()
    tails = eng.flush()
    for c in range(C):
        ref_body, ref_tail = _oracle_stream(x[c], {0: h[c]}, nb, thr)
        tol = _tol(x[c], h[c])
        got = np.concatenate([b1[c], b2[c]])
        assert np.max(np.abs(got - ref_body)) <= tol, c
        assert len(tails[c]) == len(ref_tail)
        assert np.max(np.abs(tails[c] - ref_tail)) <= tol, c


def test_fast_nonfinite_pattern_matches_ordered():
    import torch

    from paper_2401_01607_b200.core import Signal
    from paper_2401_01607_b200.engine import EngineConfig, ScatterEngine

    rng = np.random.default_rng(13)
    n, nh, nb = 1 << 19, 4096, 8192
    x = rng.uniform(-1, 1, n).astype(np.float32)
    x[300000] = np.inf
    h = rng.standard_normal(nh).astype(np.float32)
    h[17] = 0.0                                   # 0 * inf -> NaN at one output
    res = {}
    for mode in ("fast", "ordered"):
        eng = ScatterEngine(Signal(torch.from_numpy(h).cuda()), EngineConfig(block_size_nb=nb), mode=mode)
        res[mode] = eng.process_stream(torch.from_numpy(x).cuda(), nb).cpu().numpy()
    for f in (np.isnan, np.isposinf, np.isneginf):
        np.testing.assert_array_equal(f(res["fast"]), f(res["ordered"]))
    fin = np.isfinite(res["ordered"])
    assert np.max(np.abs(res["fast"][fin] - res["ordered"][fin])) <= _tol(np.where(np.isfinite(x), x, 0), h)


def test_small_segments_stay_ordered_and_mode_validation():
    import torch

    from paper_2401_01607_b200.core import Signal
    from paper_2401_01607_b200.engine import EngineConfig, ScatterEngine

    rng = np.random.default_rng(14)
    x = rng.uniform(-1, 1, 50000).astype(np.float32)
    h = rng.standard_normal(512).astype(np.float32)
    a = ScatterEngine(Signal(torch.from_numpy(h).cuda()), EngineConfig(block_size_nb=1024))
    b = ScatterEngine(Signal(torch.from_numpy(h).cuda()), EngineConfig(block_size_nb=1024), mode="ordered")
    ya = a.process_stream(torch.from_numpy(x).cuda(), 1024).cpu().numpy()
    yb = b.process_stream(torch.from_numpy(x).cuda(), 1024).cpu().numpy()
    np.testing.assert_array_equal(ya, yb)         # 25.6M MACs: below the FAST threshold
    with pytest.raises(ValueError, match="mode must be"):
        ScatterEngine(Signal(h), mode="tc")


@pytest.mark.parametrize("channels", [1, 3])
def test_periodic_swaps_batched_path(channels):
    """cfg2's pattern: equal segments (the last one shorter), one IR length --
    all segments in one batched tensor-core launch; vs the oracle engine."""
    import torch

    from paper_2401_01607_b200.engine import EngineConfig
    from paper_2401_01607_b200.multichannel import MultiChannelEngine

    rng = np.random.default_rng(15 + channels)
    n, nh, nb, every = 150_000 + 77, 4096, 256, 100          # 6 segments of 25,600, last 22,077
    x = rng.uniform(-1, 1, (channels, n)).astype(np.float32)
    n_blocks = -(-n // nb)
    irs = [(rng.standard_normal((channels, nh)) * np.exp(-np.arange(nh) / 800)).astype(np.float32)
           for _ in range(-(-n_blocks // every))]
    eng = MultiChannelEngine(torch.from_numpy(irs[0]).cuda(), EngineConfig(block_size_nb=nb, zero_skip_threshold=0.01))
    swaps = [(b, torch.from_numpy(irs[b // every]).cuda()) for b in range(every, n_blocks, every)]
    body = eng.process_stream(torch.from_numpy(x).cuda(), nb, swaps).cpu().numpy()
    tails = eng.flush()
    for c in range(channels):
        ref_body, ref_tail = _oracle_stream(x[c], {b: irs[b // every][c] for b in range(0, n_blocks, every)}, nb, 0.01)
        tol = max(_tol(x[c], ir[c]) for ir in irs)
        assert np.max(np.abs(body[c] - ref_body)) <= tol, c
        assert len(tails[c]) == len(ref_tail)
        assert np.max(np.abs(tails[c] - ref_tail)) <= tol, c


def test_unequal_segments_per_segment_path():
    """Large segments of different IR lengths: one FIR launch per segment."""
    import torch

    from paper_2401_01607_b200.core import Signal
    from paper_2401_01607_b200.engine import EngineConfig, ScatterEngine

    rng = np.random.default_rng(21)
    n, nb = 1 << 20, 8192
    x = rng.uniform(-1, 1, n).astype(np.float32)
    h0 = rng.standard_normal(4096).astype(np.float32) * 0.1
    h1 = rng.standard_normal(6000).astype(np.float32) * 0.1
    eng = ScatterEngine(Signal(torch.from_numpy(h0).cuda()), EngineConfig(block_size_nb=nb))
    body = eng.process_stream(torch.from_numpy(x).cuda(), nb, [(40, torch.from_numpy(h1).cuda())]).cpu().numpy()
    tail = eng.flush().samples.cpu().numpy()
    ref_body, ref_tail = _oracle_stream(x, {0: h0, 40: h1}, nb)
    tol = max(_tol(x, h0), _tol(x, h1))
    assert np.max(np.abs(body - ref_body)) <= tol
    assert len(tail) == len(ref_tail) and np.max(np.abs(tail - ref_tail)) <= tol


def test_fast_process_block_large_blocks_with_pending_swap():
    """FAST mode routes a single block with >= 2^30 MACs through the fused
    tensor-core path (pending swap applied first, as in engine.py:124-126)."""
    import torch

    from paper_2401_01607_b200.engine import EngineConfig
    from paper_2401_01607_b200.multichannel import MultiChannelEngine

    rng = np.random.default_rng(31)
    C, nb, nh = 8, 8192, 16384
    x = rng.uniform(-1, 1, (C, 5 * nb - 100)).astype(np.float32)
    h0 = (rng.standard_normal((C, nh)) * np.exp(-np.arange(nh) / 3000)).astype(np.float32)
    h1 = (rng.standard_normal((C, nh)) * np.exp(-np.arange(nh) / 2000)).astype(np.float32)
    eng = MultiChannelEngine(torch.from_numpy(h0).cuda(), EngineConfig(block_size_nb=nb))
    outs = []
    for b, s in enumerate(range(0, x.shape[1], nb)):
        if b == 3:
            eng.swap_ir_at_next_block(torch.from_numpy(h1).cuda())
        outs.append(eng.process_block(torch.from_numpy(x[:, s:s + nb]).cuda()).cpu().numpy())
    body = np.concatenate(outs, axis=1)
    tails = eng.flush()
    for c in range(C):
        ref_body, ref_tail = _oracle_stream(x[c], {0: h0[c], 3: h1[c]}, nb)
        tol = max(_tol(x[c], h0[c]), _tol(x[c], h1[c]))
        assert np.max(np.abs(body[c] - ref_body)) <= tol, c
        assert len(tails[c]) == len(ref_tail) and np.max(np.abs(tails[c] - ref_tail)) <= tol, c


def test_fast_many_swaps_chunked_calls():
    """45 IR changes: the fused call is split into launches of <= 31 events,
    each of which takes the batched tensor-core path (uniform segments)."""
    import torch

    from paper_2401_01607_b200.core import Signal
    from paper_2401_01607_b200.engine import EngineConfig, ScatterEngine

    rng = np.random.default_rng(45)
    nb, every, nh = 256, 10, 4096
    n = nb * every * 46
    x = rng.uniform(-1, 1, n).astype(np.float32)
    irs = [(rng.standard_normal(nh) * np.exp(-np.arange(nh) / 600)).astype(np.float32) for _ in range(46)]
    eng = ScatterEngine(Signal(torch.from_numpy(irs[0]).cuda()), EngineConfig(block_size_nb=nb))
    swaps = [(every * j, torch.from_numpy(irs[j]).cuda()) for j in range(1, 46)]
    body = eng.process_stream(torch.from_numpy(x).cuda(), nb, swaps).cpu().numpy()
    tail = eng.flush().samples.cpu().numpy()
    ref_body, ref_tail = _oracle_stream(x, {every * j: irs[j] for j in range(46)}, nb)
    tol = max(_tol(x, h) for h in irs)
    assert np.max(np.abs(body - ref_body)) <= tol
    assert len(tail) == len(ref_tail) and np.max(np.abs(tail - ref_tail)) <= tol


def test_unequal_segments_padded_batched_path():
    """Segments of one IR length but different lengths (44, 46, 38 blocks):
    padded to the longest and convolved in one batched launch."""
    import torch

    from paper_2401_01607_b200.engine import EngineConfig
    from paper_2401_01607_b200.multichannel import MultiChannelEngine

    rng = np.random.default_rng(52)
    C, nb, nh = 2, 4096, 4096
    n = nb * 128 - 1000
    x = rng.uniform(-1, 1, (C, n)).astype(np.float32)
    x[:, 5000:5100] = np.nan
    irs = [(rng.standard_normal((C, nh)) * np.exp(-np.arange(nh) / 900)).astype(np.float32) for _ in range(3)]
    eng = MultiChannelEngine(torch.from_numpy(irs[0]).cuda(), EngineConfig(block_size_nb=nb, zero_skip_threshold=0.02))
    swaps = [(44, torch.from_numpy(irs[1]).cuda()), (90, torch.from_numpy(irs[2]).cuda())]
    body = eng.process_stream(torch.from_numpy(x).cuda(), nb, swaps).cpu().numpy()
    tails = eng.flush()
    for c in range(C):
        ref_body, ref_tail = _oracle_stream(x[c], {0: irs[0][c], 44: irs[1][c], 90: irs[2][c]}, nb, 0.02)
        xc = np.nan_to_num(x[c])
        tol = max(_tol(xc, ir[c]) for ir in irs)
        assert np.max(np.abs(body[c] - ref_body)) <= tol, c
        assert len(tails[c]) == len(ref_tail) and np.max(np.abs(tails[c] - ref_tail)) <= tol, c


def test_fast_stream_graph_replay_identical():
    """The FAST fused stream (batched tensor-core FIR, state replay forked on a
    side stream) captured as a CUDA graph and replayed: every replay equals
    the first, direct call bit for bit, and the graph is actually used."""
    import ctypes

    import torch

    from paper_2401_01607_b200 import _native as N
    from paper_2401_01607_b200.core import Signal
    from paper_2401_01607_b200.engine import EngineConfig, ScatterEngine

    rng = np.random.default_rng(77)
    n, nh, nb, every = 256 * 600, 4096, 256, 100
    x = torch.from_numpy(rng.uniform(-1, 1, n).astype(np.float32)).cuda()
    irs = [torch.from_numpy((rng.standard_normal(nh) * np.exp(-np.arange(nh) / 800)).astype(np.float32)).cuda()
           for _ in range(6)]
    swaps = [(0, irs[0])] + [(b, irs[b // every]) for b in range(every, n // nb, every)]
    eng = ScatterEngine(Signal(irs[0]), EngineConfig(block_size_nb=nb))
    assert eng.mode == "fast"
    res = []
    for _ in range(12):
        body = eng.process_stream(x, nb, swaps)
        tail = eng.flush().samples
        res.append((body.cpu().numpy().copy(), tail.cpu().numpy().copy()))
    hits, caps, fails = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    N.check(N.lib().sc_engine_graph_stats(eng._handle, ctypes.byref(hits), ctypes.byref(caps), ctypes.byref(fails)))
    assert fails.value == 0 and caps.value >= 1 and hits.value >= 3, (hits.value, caps.value, fails.value)
    for body, tail in res[1:]:
        assert np.array_equal(body, res[0][0]) and np.array_equal(tail, res[0][1])
    # and within the FP32 tolerance of the float64 oracle engine
    ref_body, ref_tail = _oracle_stream(x.cpu().numpy(), {b: h.cpu().numpy() for b, h in swaps}, nb)
    tol = max(_tol(x.cpu().numpy(), h.cpu().numpy()) for h in irs)
    assert np.max(np.abs(res[0][0] - ref_body)) <= tol
    assert np.max(np.abs(res[0][1] - ref_tail)) <= tol
