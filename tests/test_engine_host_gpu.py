"""Host-resident streams through the engines (sc_engine_process_blocks_host):
a large pinned [C, n] input is processed in runs of whole blocks whose
uploads, blocks and downloads overlap.  The run cut must be invisible: in
ORDERED mode body, tail and engine state are bit-identical to the device
path (which is bit-identical to block-by-block processing and, in float64,
to the reference engine); FAST mode stays within the FP32 tolerance."""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2401_01607_b200 import EngineConfig, MultiChannelEngine, ScatterEngine, Signal
from paper_2401_01607_b200 import _dev

pytestmark = pytest.mark.gpu


@pytest.fixture
def pipe_small(monkeypatch):
    """Pipeline from a few KiB so small test streams take the host path."""
    monkeypatch.setattr(_dev, "PINNED_STREAM_MIN_BYTES", 1)
    calls = []
    from paper_2401_01607_b200 import _native as N

    lib = N.lib()
    real = lib.sc_engine_process_blocks_host

    class Spy:
        def __getattr__(self, name):
            return getattr(lib, name)

        def sc_engine_process_blocks_host(self, *a):
            calls.append(a[2])
            return real(*a)

    return calls, Spy()


def _np(a):
    return a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)


def _pinned(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).pin_memory()


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_multichannel_host_stream_bit_identical(pipe_small, dtype):
    import torch

    calls, spy = pipe_small
    rng = np.random.default_rng(91)
    C, nb, n = 3, 64, 64 * 37 + 11          # ragged last block
    h1 = rng.standard_normal((C, 150)).astype(dtype)
    h2 = rng.standard_normal((C, 70)).astype(dtype)
    h3 = rng.standard_normal((C, 300)).astype(dtype)
    x = rng.uniform(-1, 1, (C, n)).astype(dtype)
    x[rng.uniform(0, 1, (C, n)) < 0.1] = 0.0
    # swaps at block 0, at the run boundary (2 runs of 19 blocks), inside run 1
    # and beyond the end (ignored by both paths)
    swaps = [(0, h2), (19, h1), (25, h3), (400, h2)]
    cfg = EngineConfig(block_size_nb=nb, zero_skip_threshold=0.02)

    dev = MultiChannelEngine(h1, cfg, mode="ordered")
    body_d = dev.process_stream(torch.from_numpy(x).cuda(), nb,
                                [(b, torch.from_numpy(h).cuda()) for b, h in swaps]).cpu().numpy()
    state_d = dev.state()
    tail_d = dev.flush()

    host = MultiChannelEngine(h1, cfg, mode="ordered")
    host._lib = spy
    body_h = host.process_stream(_pinned(x), nb, [(b, _pinned(h)) for b, h in swaps])
    assert calls == [n] and body_h.is_pinned() and tuple(body_h.shape) == (C, n)
    assert host.state() == state_d
    tail_h = host.flush()
    np.testing.assert_array_equal(body_h.numpy().view(np.uint8), body_d.view(np.uint8))
    for a, b in zip(tail_h, tail_d):
        np.testing.assert_array_equal(a.view(np.uint8), b.view(np.uint8))
    if dtype == np.float64:
        # and the reference engine per channel
        for c in range(C):
            ref = O.OracleEngine(h1[c], nb, 0.02)
            out = []
            for bi, s in enumerate(range(0, n, nb)):
                for b, h in swaps:
                    if b == bi:
                        ref.swap_ir(h[c])
                out.append(ref.process_block(x[c, s:s + nb]))
            np.testing.assert_array_equal(np.concatenate(out), body_h.numpy()[c])


def test_single_channel_host_stream_float64(pipe_small):
    import torch

    calls, spy = pipe_small
    rng = np.random.default_rng(92)
    nb, n = 128, 128 * 50
    h = rng.standard_normal(700)
    h2 = rng.standard_normal(900)
    x = rng.uniform(-1, 1, n)
    eng_d = ScatterEngine(Signal(h), EngineConfig(block_size_nb=nb))
    body_d = eng_d.process_stream(torch.from_numpy(x).cuda(), nb, [(30, torch.from_numpy(h2).cuda())]).cpu().numpy()
    eng_h = ScatterEngine(Signal(h), EngineConfig(block_size_nb=nb))
    eng_h._lib = spy
    body_h = eng_h.process_stream(_pinned(x), nb, [(30, _pinned(h2))])
    assert calls == [n] and body_h.is_pinned()
    np.testing.assert_array_equal(body_h.numpy(), body_d)
    np.testing.assert_array_equal(_np(eng_h.flush().samples), _np(eng_d.flush().samples))
    # the engine keeps working on the device afterwards (buffers reused)
    more = Signal(rng.uniform(-1, 1, 100))
    np.testing.assert_array_equal(_np(eng_h.process_block(more).samples), _np(eng_d.process_block(more).samples))


def test_multichannel_host_stream_fast_within_tolerance(pipe_small):
    """FAST mode (tensor-core segments) from a pinned host stream: within the
    FP32 tolerance of the float64 oracle, same residue for the flush."""
    calls, spy = pipe_small
    rng = np.random.default_rng(93)
    C, nb, n, nh = 2, 8192, 8192 * 48, 4096      # >= 2^30 MACs per run: the FAST path
    h = rng.standard_normal((C, nh)).astype(np.float32)
    x = rng.uniform(-1, 1, (C, n)).astype(np.float32)
    eng = MultiChannelEngine(h, EngineConfig(block_size_nb=nb), mode="fast")
    eng._lib = spy
    body = eng.process_stream(_pinned(x), nb).numpy()
    tail = eng.flush()
    assert calls == [n]
    for c in range(C):
        ref = O.scatter_window(x[c].astype(np.float64), h[c].astype(np.float64), 0, n + nh - 1)
        got = np.concatenate([body[c], tail[c]])
        tol = 1e-5 * np.max(np.abs(x[c])) * np.sum(np.abs(h[c]))
        assert np.max(np.abs(got - ref[:len(got)])) <= tol


def test_host_stream_small_or_pageable_takes_device_path(monkeypatch):
    """Below the size threshold, or from pageable memory, the device path runs."""
    import torch

    from paper_2401_01607_b200 import _native as N

    lib = N.lib()
    seen = []

    class Spy:
        def __getattr__(self, name):
            if name == "sc_engine_process_blocks_host":
                seen.append(name)
            return getattr(lib, name)

    rng = np.random.default_rng(94)
    h = rng.standard_normal((2, 50)).astype(np.float32)
    x = rng.uniform(-1, 1, (2, 1000)).astype(np.float32)
    eng = MultiChannelEngine(h, EngineConfig(block_size_nb=100), mode="ordered")
    eng._lib = Spy()
    eng.process_stream(_pinned(x), 100)           # 8 KB: below the threshold
    eng.process_stream(torch.from_numpy(x), 100)  # pageable
    assert seen == []


@pytest.mark.parametrize("kind", ["numpy", "pinned", "pageable", "mixed_cuda"])
def test_as_device_many_packs_small_host_arrays(kind):
    """A swap schedule's IRs go up in one packed copy; values, shapes and
    dtype are those of one as_device call per array."""
    import torch

    rng = np.random.default_rng(95)
    arrays = [rng.standard_normal(n) for n in (5, 300, 1)] + [rng.standard_normal((3, 40))]
    if kind == "pinned":
        arrays = [_pinned(a) for a in arrays]
    elif kind == "pageable":
        arrays = [torch.from_numpy(a) for a in arrays]
    elif kind == "mixed_cuda":
        arrays = [torch.from_numpy(a).cuda() if i == 1 else a for i, a in enumerate(arrays)]
    for npd in (np.float64, np.float32):
        got = _dev.as_device_many(arrays, npd)
        want = [_dev.as_device(a, npd) for a in arrays]
        assert len(got) == len(want)
        for g, w in zip(got, want):
            assert g.is_cuda and g.dtype == w.dtype and g.shape == w.shape and g.is_contiguous()
            assert torch.equal(g, w)
