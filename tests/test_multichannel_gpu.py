"""Multichannel streaming engine vs one reference
engine per channel (the oracle restatement of engine.py, pinned to the
reference).  float64: bit-exact per channel, including per-channel `live`
(one channel goes silent so its tail is shorter), swaps, deferred swaps,
process_sample and the fused process_stream."""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2401_01607_b200 import EngineConfig, MultiChannelEngine

pytestmark = pytest.mark.gpu


def _inputs(rng, C, n, dtype):
    x = rng.uniform(-1, 1, (C, n)).astype(dtype)
    x[rng.uniform(0, 1, (C, n)) < 0.15] = 0.0
    x[1, n // 2:] = 0.0          # channel 1 falls silent: its live drains early
    x[2, 7] = np.nan             # NaN input is skipped by the engine (_kernels.py:33)
    return x


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_blocks_swaps_flush_per_channel(dtype):
    rng = np.random.default_rng(3)
    C, nb = 4, 50
    h1 = rng.standard_normal((C, 40)).astype(dtype)
    h2 = rng.standard_normal((C, 90)).astype(dtype)
    h3 = rng.standard_normal((C, 15)).astype(dtype)
    x = _inputs(rng, C, 600, dtype)
    eng = MultiChannelEngine(h1, EngineConfig(block_size_nb=nb, zero_skip_threshold=0.05))
    refs = [O.OracleEngine(h1[c], nb, 0.05) for c in range(C)]
    got, want = [], [[] for _ in range(C)]
    for b, s in enumerate(range(0, 600, nb)):
        if b == 3:
            eng.swap_ir(h2)
            for c in range(C):
                refs[c].swap_ir(h2[c])
        if b == 7:
            eng.swap_ir_at_next_block(h3)   # applied by the next process_block
            for c in range(C):
                refs[c].swap_ir_at_next_block(h3[c])
        got.append(np.asarray(eng.process_block(x[:, s:s + nb])))
        for c in range(C):
            want[c].append(refs[c].process_block(x[c, s:s + nb]))
    st = eng.state()
    assert st["live"] == [r.live for r in refs]
    assert st["read_index"] == [r.read_index for r in refs]
    tails = eng.flush()
    body = np.concatenate(got, axis=1)
    for c in range(C):
        w = np.concatenate(want[c])
        wt = refs[c].flush()
        assert len(tails[c]) == len(wt)
        if dtype == np.float64:
            assert np.array_equal(body[c], w) and np.array_equal(tails[c], wt)
        else:
            tol = 1e-5 * np.sum(np.abs(h2[c])) * 2
            assert np.max(np.abs(body[c] - w)) <= tol and np.max(np.abs(tails[c] - wt), initial=0) <= tol


def test_fused_stream_and_samples_f64():
    import torch

    rng = np.random.default_rng(9)
    C, nb = 3, 32
    h0 = rng.standard_normal((C, 70))
    irs = [rng.standard_normal((C, n)) for n in (20, 150, 70)]
    x = _inputs(rng, C, 32 * 40 + 5, np.float64)
    swaps = [(4, irs[0]), (10, irs[1]), (10, irs[2]), (25, irs[0])]
    eng = MultiChannelEngine(h0, EngineConfig(block_size_nb=nb))
    # a few per-sample steps first (never apply pending swaps)
    s0 = [eng.process_sample(x[:, i]) for i in range(3)]
    body = eng.process_stream(torch.from_numpy(x[:, 3:]).cuda(), nb, swaps).cpu().numpy()
    tails = eng.flush()
    for c in range(C):
        ref = O.OracleEngine(h0[c], nb)
        w = [ref.process_sample(x[c, i]) for i in range(3)]
        assert np.array_equal([s[c] for s in s0], w)
        outs = []
        for b, s in enumerate(range(3, x.shape[1], nb)):
            for sb, ir in swaps:
                if sb == b:
                    ref.swap_ir(ir[c])
            outs.append(ref.process_block(x[c, s:s + nb]))
        assert np.array_equal(body[c], np.concatenate(outs))
        assert np.array_equal(tails[c], ref.flush())


def test_mono_ir_broadcast_and_errors():
    rng = np.random.default_rng(1)
    h = rng.standard_normal(33)
    eng = MultiChannelEngine(h, channels=2)
    x = rng.uniform(-1, 1, (2, 100))
    y = eng.process_block(x)
    for c in range(2):
        assert np.array_equal(y[c], O.OracleEngine(h).process_block(x[c]))
    with pytest.raises(ValueError, match="exceeds block_size_nb"):
        MultiChannelEngine(h, EngineConfig(block_size_nb=4), channels=2).process_block(np.zeros((2, 5)))
    with pytest.raises(ValueError, match="channels"):
        eng.process_block(np.zeros((3, 5)))
    with pytest.raises(ValueError, match="empty"):
        eng.swap_ir(np.zeros((2, 0)))


def test_batched_pinned_host_pipeline(monkeypatch):
    """Pinned host [C, Ne] -> channel groups overlapped over three streams."""
    import torch

    from oracle import oracle as O
    from paper_2401_01607_b200 import multichannel

    monkeypatch.setattr(multichannel, "_PIPELINE_MIN_MACS", 0)
    rng = np.random.default_rng(77)
    X = rng.uniform(-1, 1, (11, 20_011)).astype(np.float32)
    H = rng.standard_normal((11, 1_500)).astype(np.float32)
    y = multichannel.convolve_batched(torch.from_numpy(X).pin_memory(), torch.from_numpy(H))
    assert y.is_pinned() and tuple(y.shape) == (11, 20_011 + 1_499)
    for c in range(11):
        ref = O.scatter_full(X[c], H[c])
        tol = 1e-5 * np.max(np.abs(X[c])) * np.sum(np.abs(H[c]))
        assert np.max(np.abs(y[c].numpy().astype(np.float64) - ref)) <= tol


# ---------------------------------------------------------------- independent channels


def _ir(rng, n):
    return rng.standard_normal(n) * np.exp(-np.arange(n) / max(1.0, n / 4))


@pytest.mark.parametrize("nb", [37, 300, 3000])
def test_independent_channels_staggered_swaps_bit_exact(nb):
    """One engine per channel (engine.py:60-66): every channel has its own IR
    length from the start, swaps at its own blocks (some channels never),
    takes per-channel deferred swaps, and drains its own live/tail -- float64
    bit-exact against C independent oracle engines.  nb = 3000 exercises the
    multi-launch path for blocks above the one-launch kernel's limit."""
    rng = np.random.default_rng(50 + nb)
    C = 5
    n = 9000
    lens0 = [33, 700, 1, 260, 1500]
    h0 = [_ir(rng, L) for L in lens0]
    x = _inputs(rng, C, n, np.float64)
    eng = MultiChannelEngine(h0, EngineConfig(block_size_nb=nb, zero_skip_threshold=0.01))
    assert eng.ir_lengths == lens0
    refs = [O.OracleEngine(h0[c], nb, 0.01) for c in range(C)]
    n_blocks = -(-n // nb)
    plan = {}                                   # block -> [(kind, channel, ir)]
    for c in range(C):
        if c == 2:
            continue                            # channel 2 never swaps
        for b in sorted(rng.choice(np.arange(1, n_blocks), size=min(3, n_blocks - 1), replace=False)):
            kind = "now" if (c + int(b)) % 2 else "next"
            plan.setdefault(int(b), []).append((kind, c, _ir(rng, int(rng.integers(1, 2000)))))
    got, want = [], [[] for _ in range(C)]
    for b, s in enumerate(range(0, n, nb)):
        for kind, c, h in plan.get(b, []):
            per = [None] * C
            per[c] = h
            if kind == "now":
                eng.swap_ir(per)
                refs[c].swap_ir(h)
            else:
                eng.swap_ir_at_next_block(h, channels=[c])
                refs[c].swap_ir_at_next_block(h)
        got.append(np.asarray(eng.process_block(x[:, s:s + nb])))
        for c in range(C):
            want[c].append(refs[c].process_block(x[c, s:s + nb]))
        if b == n_blocks // 2:
            st = eng.state()
            assert st["live"] == [r.live for r in refs]
            assert st["read_index"] == [r.read_index for r in refs]
            assert st["nh_per_channel"] == [len(r.ir) for r in refs]
    tails = eng.flush()
    body = np.concatenate(got, axis=1)
    for c in range(C):
        assert np.array_equal(body[c], np.concatenate(want[c])), c
        wt = refs[c].flush()
        assert len(tails[c]) == len(wt) and np.array_equal(tails[c], wt), c


def test_independent_channels_stream_schedule():
    """process_stream with a per-channel schedule ((block, IR, channels) and
    (block, [per-channel IRs]) entries) equals the block-by-block calls of
    independent oracle engines, bit for bit (float64)."""
    import torch

    rng = np.random.default_rng(61)
    C, nb, n = 3, 64, 64 * 30 + 11
    h0 = [_ir(rng, L) for L in (50, 120, 7)]
    x = _inputs(rng, C, n, np.float64)
    a, b2 = _ir(rng, 300), _ir(rng, 20)
    swaps = [(3, a, [1]), (5, [b2, None, _ir(rng, 90)]), (5, _ir(rng, 40), [0]), (17, a, [0, 2]), (22, np.stack([a[:64]] * 3))]
    eng = MultiChannelEngine(h0, EngineConfig(block_size_nb=nb))
    body = eng.process_stream(torch.from_numpy(x).cuda(), nb, swaps).cpu().numpy()
    tails = eng.flush()
    for c in range(C):
        ref = O.OracleEngine(h0[c], nb)
        out = []
        for blk, s in enumerate(range(0, n, nb)):
            for sw in swaps:
                if sw[0] != blk:
                    continue
                irs = sw[1]
                if len(sw) > 2:
                    if c in sw[2]:
                        ref.swap_ir(irs)
                elif isinstance(irs, list):
                    if irs[c] is not None:
                        ref.swap_ir(irs[c])
                else:
                    ref.swap_ir(irs[c])
            out.append(ref.process_block(x[c, s:s + nb]))
        assert np.array_equal(body[c], np.concatenate(out)), c
        assert np.array_equal(tails[c], ref.flush()), c
