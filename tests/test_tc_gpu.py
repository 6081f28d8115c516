"""Tensor-core (tcgen05, fp16 hi/lo split) FIR vs the CPU oracle.

Tolerance: max-abs <= 1e-5 * max|x| * ||h||_1 (north_star), on shapes that
exercise every boundary of the kernel: one/many X windows (64 shifts each),
partial H8 stages, partial last tile, tiny and huge dynamic range, shards
(output ranges with halos) and batched channels.
"""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2401_01607_b200 import configs
from paper_2401_01607_b200.core import Signal, scatter_convolve
from paper_2401_01607_b200.multichannel import convolve_batched
from paper_2401_01607_b200.sharded import convolve_shard, shard_plan

pytestmark = pytest.mark.gpu


def err_frac(y, ref, x, h):
    tol = configs.tolerance(x, h, "f32")
    return float(np.max(np.abs(np.asarray(y, np.float64) - ref))) / tol


CASES = [(20_000, 256), (20_000, 1000), (16_384, 4096), (100_000, 9_000), (50_001, 20_003),
         (3_000, 70_000), (300_000, 1_100), (1, 300), (1000, 8191), (40_000, 262_144),
         # <= 2 shifts: the 2-shift drain variant (k_tc_fir<2>)
         (50_001, 64), (20_000, 129), (7, 3), (33_333, 1), (70_000, 100)]


@pytest.mark.parametrize("ne,nh", CASES)
def test_tc_matches_oracle(ne, nh):
    rng = np.random.default_rng(ne + 17 * nh)
    x = rng.uniform(-1, 1, ne).astype(np.float32)
    h = (rng.standard_normal(nh) * np.exp(-np.arange(nh) / (nh / 5))).astype(np.float32)
    y = np.asarray(scatter_convolve(Signal(x), Signal(h), mode="tc").concatenated().samples)
    assert len(y) == ne + nh - 1
    ref = O.scatter_window(x, h, 0, ne + nh - 1)
    assert err_frac(y, ref, x, h) <= 1.0


@pytest.mark.parametrize("xscale,hscale", [(1e-6, 1.0), (1.0, 1e-9), (3e4, 7e3), (1e-30, 1e20),
                                           # scales beyond float range: the ordered fallback
                                           (1e-36, 1.0), (1.0, 1e-37), (1e25, 1e-30)])
def test_tc_scaling_is_exact_power_of_two(xscale, hscale):
    rng = np.random.default_rng(5)
    x = (rng.uniform(-1, 1, 30_000) * xscale).astype(np.float32)
    h = (rng.standard_normal(3000) * hscale).astype(np.float32)
    y = np.asarray(scatter_convolve(Signal(x), Signal(h), mode="tc").concatenated().samples)
    assert np.all(np.isfinite(y))
    assert err_frac(y, O.scatter_window(x, h, 0, len(y)), x, h) <= 1.0


def test_tc_shards_and_batched():
    import torch

    rng = np.random.default_rng(8)
    x = rng.uniform(-1, 1, 90_000).astype(np.float32)
    h = rng.standard_normal(5000).astype(np.float32)
    hd = torch.from_numpy(h).cuda()
    ref = O.scatter_window(x, h, 0, len(x) + len(h) - 1)
    parts = []
    for sh in shard_plan(len(x), len(h), 3):
        xs = torch.from_numpy(x[sh.x_begin:sh.x_end]).cuda()
        parts.append(convolve_shard(xs, sh, hd, mode="tc").cpu().numpy())
    assert err_frac(np.concatenate(parts), ref, x, h) <= 1.0
    X = rng.uniform(-1, 1, (3, 40_000)).astype(np.float32)
    H = rng.standard_normal((3, 2000)).astype(np.float32)
    H[1] *= 1e-3
    Y = convolve_batched(X, H, mode="tc")
    for c in range(3):
        assert err_frac(Y[c], O.scatter_window(X[c], H[c], 0, Y.shape[1]), X[c], H[c]) <= 1.0


@pytest.mark.parametrize("nh", [5, 200])
@pytest.mark.parametrize("where", ["x_nan", "h_inf"])
def test_short_filter_nonfinite_exact(nh, where):
    # the short-filter kernel multiplies only taps whose input exists, so
    # 0*Inf never appears at the signal edges (reference semantics)
    rng = np.random.default_rng(nh)
    x = rng.uniform(-1, 1, 10_000).astype(np.float32)
    h = rng.standard_normal(nh).astype(np.float32)
    if where == "x_nan":
        x[[0, 4000, 9999]] = np.nan
    else:
        h[nh // 2] = np.inf
    y = np.asarray(scatter_convolve(Signal(x), Signal(h)).concatenated().samples)
    ref = O.scatter_full(x, h)
    assert np.array_equal(np.isnan(y), np.isnan(ref)) and np.array_equal(np.isinf(y), np.isinf(ref))
    fin = np.isfinite(ref)
    assert np.max(np.abs(y[fin] - ref[fin])) <= 1e-5 * np.sum(np.abs(h[np.isfinite(h)])) + 1e-6


@pytest.mark.parametrize("where", ["x_nan", "x_inf", "h_inf"])
def test_fast_mode_nonfinite_reroutes_on_device(where):
    # FAST mode on a long filter runs the tensor-core kernel; NaN/Inf inputs
    # are detected on the device and the FFMA kernel produces the reference's
    # exact NaN/Inf pattern (no host synchronisation involved).
    rng = np.random.default_rng(6)
    x = rng.uniform(-1, 1, 40_000).astype(np.float32)
    h = rng.standard_normal(3000).astype(np.float32)
    if where == "x_nan":
        x[1234] = np.nan
    elif where == "x_inf":
        x[20_000] = np.inf
    else:
        h[17] = -np.inf
    y = np.asarray(scatter_convolve(Signal(x), Signal(h)).concatenated().samples)
    ref = O.scatter_window(x, h, 0, len(y))
    assert np.array_equal(np.isnan(y), np.isnan(ref))
    assert np.array_equal(np.isinf(y), np.isinf(ref))
    fin = np.isfinite(ref)
    tol = 1e-5 * np.max(np.abs(x[np.isfinite(x)])) * np.sum(np.abs(h[np.isfinite(h)]))
    assert np.max(np.abs(y[fin] - ref[fin])) <= tol


@pytest.mark.parametrize("mode", [None, "ffma"])
def test_pinned_host_pipeline(monkeypatch, mode):
    """Pinned host input -> chunked H2D / FIR / D2H overlap (core._fir_host_pipelined)."""
    import torch

    from paper_2401_01607_b200 import core

    monkeypatch.setattr(core, "_PIPELINE_MIN_MACS", 0)
    monkeypatch.setenv("SC_PIPE_CHUNKS", "5")   # the native range engine's chunk count
    rng = np.random.default_rng(44)
    x = rng.uniform(-1, 1, 70_001).astype(np.float32)
    h = rng.standard_normal(3_333).astype(np.float32)
    xp = torch.from_numpy(x).pin_memory()
    out = scatter_convolve(Signal(xp), Signal(torch.from_numpy(h)), mode=mode)
    assert out.body.samples.is_pinned() and len(out.body) == len(x) and len(out.tail) == len(h) - 1
    y = out.concatenated().samples
    assert err_frac(y.numpy(), O.scatter_window(x, h, 0, len(y)), x, h) <= 1.0



@pytest.mark.parametrize("nh", [1, 8, 40])
def test_pinned_host_pipeline_transfer_bound(monkeypatch, nh):
    """Short filters on large pinned inputs are streamed by size, not by MACs
    (upload and download of consecutive chunks overlap)."""
    import torch

    from paper_2401_01607_b200 import core

    monkeypatch.setattr(core, "_PIPELINE_MIN_BYTES", 4 * 100_000)
    monkeypatch.setenv("SC_PIPE_CHUNKS", "7")
    calls = []
    real = core._fir_host_pipelined
    monkeypatch.setattr(core, "_fir_host_pipelined", lambda *a: calls.append(1) or real(*a))
    rng = np.random.default_rng(45 + nh)
    x = rng.uniform(-1, 1, 210_007).astype(np.float32)
    h = rng.standard_normal(nh).astype(np.float32)
    out = scatter_convolve(Signal(torch.from_numpy(x).pin_memory()), Signal(torch.from_numpy(h)))
    assert calls and out.body.samples.is_pinned()
    y = out.concatenated().samples
    assert err_frac(y.numpy(), O.scatter_window(x, h, 0, len(y)), x, h) <= 1.0

def test_tc_deterministic():
    import torch

    rng = np.random.default_rng(2)
    x = torch.from_numpy(rng.uniform(-1, 1, 200_000).astype(np.float32)).cuda()
    h = torch.from_numpy(rng.standard_normal(12_000).astype(np.float32)).cuda()
    a = scatter_convolve(Signal(x), Signal(h), mode="tc").concatenated().samples
    b = scatter_convolve(Signal(x), Signal(h), mode="tc").concatenated().samples
    assert torch.equal(a, b)


@pytest.mark.parametrize("nh", [300, 4096, 40_000])
def test_tc_same_sign_inputs(nh):
    """DC (all-positive) drive through an all-positive decaying filter: no
    cancellation hides errors in the split products or the drains."""
    rng = np.random.default_rng(nh)
    x = rng.uniform(0.5, 1.0, 60_000).astype(np.float32)
    h = (rng.uniform(0, 1, nh) * np.exp(-np.arange(nh) / (nh / 3))).astype(np.float32)
    y = np.asarray(scatter_convolve(Signal(x), Signal(h), mode="tc").concatenated().samples)
    assert err_frac(y, O.scatter_window(x, h, 0, len(y)), x, h) <= 1.0


# ---------------------------------------------------------------- fused split (k_tc_fir_fs)
# Taken for filters of <= 72 padded shifts (~9,000 taps) on launches of >= 2
# tiles per SM (>= 296 tiles of 16,384 outputs): one-stage units (<= 255 taps)
# on the bulk-copy path, 3-72 shifts on the in-place cp.async path.


def _fs_check(x, h, y, seeds=6):
    n = len(x) + len(h) - 1
    wins = [0, n - 512, min(len(x) - 256, n - 512)] + [int(s) for s in np.random.default_rng(seeds).integers(0, n - 512, seeds)]
    for s in wins:
        ref = O.scatter_window(x, h, s, s + 512)
        assert err_frac(np.asarray(y[s:s + 512]), ref, x, h) <= 1.0, s


@pytest.mark.parametrize("nh", [48, 128, 255, 256, 300, 511, 512, 700, 900, 1024, 1100, 2049, 4096, 8191, 9000])
def test_fused_split_large_launch(nh):
    import torch

    rng = np.random.default_rng(900 + nh)
    ne = (1 << 23) + 12_345                       # 512+ tiles: the fused-split kernel
    x = rng.uniform(-1, 1, ne).astype(np.float32)
    h = (rng.standard_normal(nh) * np.exp(-np.arange(nh) / (nh / 4 + 1))).astype(np.float32)
    y = scatter_convolve(Signal(torch.from_numpy(x).cuda()), Signal(torch.from_numpy(h).cuda()))
    y = y.concatenated().samples.cpu().numpy()
    assert len(y) == ne + nh - 1
    _fs_check(x, h, y)


@pytest.mark.parametrize("ne,nh", [((1 << 20) + 777, 600), (1 << 21, 1024), (700_001, 1000)])
def test_fused_split_one_wave_launch(ne, nh):
    """One-wave launches (37..148 tiles) of 512-1,024-tap filters take the
    multi-stage fused-split units with shift-range splits."""
    import torch

    from paper_2401_01607_b200 import _native as N

    rng = np.random.default_rng(ne % 1000 + nh)
    x = rng.uniform(-1, 1, ne).astype(np.float32)
    h = (rng.standard_normal(nh) * np.exp(-np.arange(nh) / (nh / 4 + 1))).astype(np.float32)
    N.lib().sc_tc_stats_reset()
    y = scatter_convolve(Signal(torch.from_numpy(x).cuda()), Signal(torch.from_numpy(h).cuda()))
    y = y.concatenated().samples.cpu().numpy()
    assert N.tc_stats()["kernel"] == "k_tc_fir_fs"
    assert len(y) == ne + nh - 1
    _fs_check(x, h, y)


@pytest.mark.parametrize("nh", [26, 33, 47])
def test_fused_split_short_filters_from_26_taps(nh):
    """FAST dispatch takes the fused-split tensor cores from 26 taps on
    launches of >= 2^30 MACs (capi.cu kTcShortMinTaps)."""
    import torch

    rng = np.random.default_rng(300 + nh)
    ne = (1 << 30) // nh + 4_321
    x = rng.uniform(-1, 1, ne).astype(np.float32)
    h = rng.standard_normal(nh).astype(np.float32)
    y = scatter_convolve(Signal(torch.from_numpy(x).cuda()), Signal(torch.from_numpy(h).cuda()))
    y = y.concatenated().samples.cpu().numpy()
    assert len(y) == ne + nh - 1
    _fs_check(x, h, y)


@pytest.mark.parametrize("nh", [131, 300])
def test_fused_split_batched_channels_and_shards(nh):
    """Several channels in one launch (the one resident H8 stage is reloaded
    when the channel changes; 300 taps: 4-shift units), and shards."""
    import torch

    rng = np.random.default_rng(77)
    C, ne = 8, 700_001
    x = rng.uniform(-1, 1, (C, ne)).astype(np.float32)
    h = rng.standard_normal((C, nh)).astype(np.float32)
    y = convolve_batched(torch.from_numpy(x).cuda(), torch.from_numpy(h).cuda()).cpu().numpy()
    for c in (0, 3, 7):
        _fs_check(x[c], h[c], y[c], seeds=2)
    # a shard whose input slice starts unaligned (edge windows take the slow fill)
    xs = rng.uniform(-1, 1, 5_000_003).astype(np.float32)
    hs = rng.standard_normal(100).astype(np.float32)
    plan = shard_plan(len(xs), len(hs), 3)
    hd = torch.from_numpy(hs).cuda()
    for sh in plan[1:]:
        ys = convolve_shard(torch.from_numpy(xs[sh.x_begin:sh.x_end]).cuda(), sh, hd).cpu().numpy()
        for s in (0, sh.n_out - 300):
            ref = O.scatter_window(xs, hs, sh.n_begin + s, sh.n_begin + s + 300)
            assert err_frac(ys[s:s + 300], ref, xs, hs) <= 1.0


@pytest.mark.parametrize("nh", [128, 300, 2048])
def test_fused_split_nonfinite_falls_back(nh):
    import torch

    rng = np.random.default_rng(78)
    ne = 1 << 23
    x = rng.uniform(-1, 1, ne).astype(np.float32)
    x[4_000_000] = np.inf
    x[6_000_123] = np.nan
    h = rng.standard_normal(nh).astype(np.float32)
    y = scatter_convolve(Signal(torch.from_numpy(x).cuda()), Signal(torch.from_numpy(h).cuda()))
    y = y.concatenated().samples.cpu().numpy()
    for s in (3_999_900, 6_000_000, 100_000):
        ref = O.scatter_window(x, h, s, s + 400)
        got = y[s:s + 400].astype(np.float64)
        assert np.array_equal(np.isnan(got), np.isnan(ref)) and np.array_equal(np.isinf(got), np.isinf(ref)), s
        fin = np.isfinite(ref)
        assert np.max(np.abs(got[fin] - ref[fin]), initial=0) <= configs.tolerance(x[np.isfinite(x)], h, "f32")
    # the next (finite) call of the same shape: the launch's flag starts clear
    # again (one-channel launches store it in the H8 kernel, no memset)
    x2 = rng.uniform(-1, 1, ne).astype(np.float32)
    y2 = scatter_convolve(Signal(torch.from_numpy(x2).cuda()), Signal(torch.from_numpy(h).cuda()))
    y2 = y2.concatenated().samples.cpu().numpy()
    assert np.all(np.isfinite(y2))
    _fs_check(x2, h, y2, seeds=2)


@pytest.mark.parametrize("ne,nh,kernel", [((1 << 23) + 7, 128, "k_tc_fir_fs"), ((1 << 23) + 7, 300, "k_tc_fir_fs"), ((1 << 23) + 7, 2048, "k_tc_fir_fs"),
                                          ((1 << 23) + 7, 9300, "k_tc_fir"),
                                          (1 << 20, 4096, "k_tc_fir")])
def test_tc_last_kernel_names_the_kernel_that_ran(ne, nh, kernel):
    """sc_tc_last_kernel (bench.py's roofline label) reports which tensor-core
    kernel issued the MMAs; sc_tc_stats counts the launch."""
    import torch

    from paper_2401_01607_b200 import _native as N

    rng = np.random.default_rng(nh)
    x = torch.from_numpy(rng.uniform(-1, 1, ne).astype(np.float32)).cuda()
    h = torch.from_numpy(rng.standard_normal(nh).astype(np.float32)).cuda()
    N.lib().sc_tc_stats_reset()
    scatter_convolve(Signal(x), Signal(h))
    torch.cuda.synchronize()
    st = N.tc_stats()
    assert st["launches"] >= 1 and st["padded_macs"] >= ne * nh
    assert st["kernel"] == kernel
