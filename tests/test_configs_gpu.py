"""BASELINE.json configs at full size on the GPU, checked against the
reference's pins (sha256 of the reference's own outputs, tests/golden) and
the CPU oracle (prefixes, seeded spot windows incl. shard seams and the
tail) plus size-independent properties (moments of the full output).

Tolerances (north_star): FP32 max-abs <= 1e-5*max|x|*||h||_1, FP64 bit-exact.
"""

import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2401_01607_b200 import configs
from paper_2401_01607_b200.core import Signal, direct_form, scatter_convolve
from paper_2401_01607_b200.engine import EngineConfig, ScatterEngine
from paper_2401_01607_b200.multichannel import convolve_batched
from paper_2401_01607_b200.sharded import convolve_shard, shard_plan
from tests import _golden as G

pytestmark = pytest.mark.gpu


def check_tol(y, ref, x, h, what):
    tol = configs.tolerance(x, h, "f32")
    err = float(np.max(np.abs(np.asarray(y, np.float64) - ref)))
    assert err <= tol, f"{what}: max err {err:.3e} > tol {tol:.3e}"
    return err / tol


def check_moments(y_dev, x, h):
    """sum_n y = sum x * sum h and sum_n n*y = (sum m x)(sum h) + (sum x)(sum k h):
    size-independent checks over the whole output (f64 reductions)."""
    import torch

    y = y_dev.double()
    n = torch.arange(y.numel(), device=y.device, dtype=torch.float64)
    x64, h64 = np.asarray(x, np.float64), np.asarray(h, np.float64)
    m = np.arange(len(x64), dtype=np.float64)
    k = np.arange(len(h64), dtype=np.float64)
    s0 = float(y.sum())
    s1 = float((n * y).sum())
    w0 = x64.sum() * h64.sum()
    w1 = (m * x64).sum() * h64.sum() + x64.sum() * (k * h64).sum()
    scale = configs.tolerance(x, h, "f32") * np.sqrt(y.numel())
    assert abs(s0 - w0) <= scale, (s0, w0, scale)
    assert abs(s1 - w1) <= scale * y.numel(), (s1, w1)


def windows_for(nout, count, width, seed):
    starts = list(np.random.default_rng(seed).integers(0, nout - width, count))
    return sorted(set([0, nout - width] + [int(s) for s in starts]))


# ---------------------------------------------------------------- cfg1 float64


def test_cfg1_bit_exact_to_reference():
    pins = G.configs_pins()
    w = configs.cfg1()
    y = np.asarray(scatter_convolve(Signal(w.x), Signal(w.h)).concatenated().samples)
    assert G.sha(y) == str(pins["cfg1_sha_scatter"])
    eng = ScatterEngine(Signal(w.h), EngineConfig(block_size_nb=8192))
    ys = eng.render(Signal(w.x)).samples
    assert G.sha(np.concatenate([ys, eng.flush().samples])) == str(pins["cfg1_sha_scatter"])
    idx = pins["cfg1_idx"]
    df = np.asarray(direct_form(Signal(w.x), Signal(w.h)).samples)[idx]
    tol = configs.tolerance(w.x, w.h, "f64")
    assert np.array_equal(df, pins["cfg1_direct_at_idx"])         # the reference's math.fsum, bit for bit
    assert np.max(np.abs(y[idx] - pins["cfg1_direct_at_idx"])) <= tol


# ---------------------------------------------------------------- cfg2 streaming


def _cfg2_swaps(w):
    n_blocks = -(-w.ne // w.block)
    return [(b, w.irs[b // w.swap_every]) for b in range(w.swap_every, n_blocks, w.swap_every)]


def test_cfg2_float64_engine_bit_exact_to_reference():
    import torch

    pins = G.configs_pins()
    w = configs.cfg2()
    x64 = w.x.astype(np.float64)
    eng = ScatterEngine(Signal(w.irs[0].astype(np.float64)), EngineConfig(block_size_nb=256))
    swaps = [(b, ir.astype(np.float64)) for b, ir in _cfg2_swaps(w)]
    body = eng.process_stream(torch.from_numpy(x64).cuda(), 256, swaps).cpu().numpy()
    tail = eng.flush().samples
    assert G.sha(body) == str(pins["cfg2_sha_body"])
    assert G.sha(tail) == str(pins["cfg2_sha_tail"])


def test_cfg2_float32_engine_per_block_within_tolerance():
    pins = G.configs_pins()
    w = configs.cfg2()
    eng = ScatterEngine(Signal(w.irs[0]), EngineConfig(block_size_nb=256))
    outs = []
    for b, s in enumerate(range(0, w.ne, 256)):          # Python-level calls, block by block
        if b and b % 100 == 0:
            eng.swap_ir(Signal(w.irs[b // 100]))
        outs.append(eng.process_block(Signal(w.x[s:s + 256])).samples)
    body = np.concatenate(outs)
    tail = eng.flush().samples
    idx = pins["cfg2_idx"]
    # ||h||_1 of the IR in effect (the largest of the 19)
    tol = max(configs.tolerance(w.x, ir, "f32") for ir in w.irs)
    assert np.max(np.abs(body[idx] - pins["cfg2_body_at_idx"])) <= tol
    assert np.max(np.abs(tail - pins["cfg2_tail"])) <= tol
    ref_body, ref_tail = O.stream_with_swaps(w.x, w.irs, 256, 100)
    # every block's 256 outputs (480,000 = 1875 x 256), and the final flush
    per_block = np.abs(body.astype(np.float64) - ref_body).reshape(-1, 256).max(axis=1)
    assert per_block.max() <= tol
    assert np.max(np.abs(tail - ref_tail)) <= tol


def test_cfg2_float32_fast_fused_stream_full_shape():
    """The exact path bench.py --config cfg2 times: one float32 FAST
    process_stream over all 480,000 samples (1,875 blocks of 256) with the 19
    IRs swapped in every 100 blocks (block 0 re-selecting IR 0, as the bench
    does), then flush -- every block's 256 outputs and the tail against the
    float64 oracle engine (engine.py:118-186 restated)."""
    import torch

    w = configs.cfg2()
    h0 = torch.from_numpy(w.irs[0]).cuda()
    eng = ScatterEngine(Signal(h0), EngineConfig(block_size_nb=256))
    assert eng.mode == "fast"
    n_blocks = -(-w.ne // 256)
    swaps = [(0, h0)] + [(b, torch.from_numpy(w.irs[b // 100]).cuda()) for b in range(100, n_blocks, 100)]
    body = eng.process_stream(torch.from_numpy(w.x).cuda(), 256, swaps).cpu().numpy()
    tail = eng.flush().samples.cpu().numpy()
    ref_body, ref_tail = O.stream_with_swaps(w.x, w.irs, 256, 100)
    assert body.shape == ref_body.shape == (w.ne,)
    assert len(tail) == len(ref_tail) == w.nh - 1
    for j in range(len(w.irs)):                     # tolerance of the IR in effect per block
        blk = slice(j * 100 * 256, min(w.ne, (j + 1) * 100 * 256))
        tol = configs.tolerance(w.x, w.irs[j], "f32")
        # a block's outputs also carry the previous IR's residue
        if j:
            tol = max(tol, configs.tolerance(w.x, w.irs[j - 1], "f32"))
        per_block = np.abs(body[blk].astype(np.float64) - ref_body[blk]).reshape(-1, 256).max(axis=1)
        assert per_block.max() <= tol, (j, per_block.max(), tol)
    tol_last = max(configs.tolerance(w.x, ir, "f32") for ir in w.irs[-2:])
    assert np.max(np.abs(tail - ref_tail)) <= tol_last


# ---------------------------------------------------------------- cfg3 long reverb


def test_cfg3_full_fast_vs_oracle():
    import torch

    w = configs.cfg3()
    xd = torch.from_numpy(w.x).cuda()
    hd = torch.from_numpy(w.h).cuda()
    y = scatter_convolve(Signal(xd), Signal(hd)).concatenated().samples
    assert y.shape[0] == w.nout
    yh = y.cpu().numpy()
    pre = int(os.environ.get("SC_CFG3_PREFIX", "50000"))
    check_tol(yh[:pre], O.scatter_window(w.x, w.h, 0, pre), w.x, w.h, "cfg3 prefix")
    for s in windows_for(w.nout, 16, 256, (3, 2)):
        check_tol(yh[s:s + 256], O.scatter_window(w.x, w.h, s, s + 256), w.x, w.h, f"cfg3 win {s}")
    check_moments(y, w.x, w.h)


# ---------------------------------------------------------------- cfg4 batched


def test_cfg4_batched_full_vs_oracle():
    import torch

    w = configs.cfg4()
    y = convolve_batched(torch.from_numpy(w.x).cuda(), torch.from_numpy(w.h).cuda())
    assert tuple(y.shape) == (64, w.nout)
    yh = y.cpu().numpy()
    for c in range(64):
        xc, hc = w.x[c], w.h[c]
        wins = [0, w.nout - 256] + [int(s) for s in np.random.default_rng((4, 3, c)).integers(0, w.nout - 256, 2)]
        for s in wins:
            check_tol(yh[c, s:s + 256], O.scatter_window(xc, hc, s, s + 256), xc, hc, f"cfg4 ch{c} win{s}")
    for c in (0, 31, 63):
        check_moments(y[c], w.x[c], w.h[c])


# ---------------------------------------------------------------- cfg5 sharded


@pytest.fixture(scope="module")
def cfg5_full():
    import torch

    w = configs.cfg5()
    xd = torch.from_numpy(w.x).cuda()
    hd = torch.from_numpy(w.h).cuda()
    y = scatter_convolve(Signal(xd), Signal(hd)).concatenated().samples
    torch.cuda.synchronize()
    return w, xd, hd, y


def test_cfg5_full_single_gpu_vs_oracle(cfg5_full):
    w, _, _, y = cfg5_full
    assert y.shape[0] == w.nout
    pre = int(os.environ.get("SC_CFG5_PREFIX", "2000000"))   # BASELINE.json configs[4]: 2,000,000
    yh_pre = y[:pre].cpu().numpy()
    check_tol(yh_pre, O.scatter_window(w.x, w.h, 0, pre), w.x, w.h, "cfg5 prefix")
    for s in configs.cfg5_spot_windows(w.nout):
        s = int(s)
        check_tol(y[s:s + 256].cpu().numpy(), O.scatter_window(w.x, w.h, s, s + 256), w.x, w.h,
                  f"cfg5 spot {s}")
    s = w.nout - 256
    check_tol(y[s:].cpu().numpy(), O.scatter_window(w.x, w.h, s, w.nout), w.x, w.h, "cfg5 tail")
    check_moments(y, w.x, w.h)


@pytest.mark.parametrize("world", [2, 8])
def test_cfg5_shards_concatenate(cfg5_full, world):
    """Each shard computed from its input slice + (Nh-1) halo only; shards run
    one after another on the single GPU and concatenate to the full result."""
    import torch

    w, xd, hd, y = cfg5_full
    plan = shard_plan(w.ne, w.nh, world)
    worst = 0.0
    for sh in plan:
        xs = xd[sh.x_begin:sh.x_end].clone()     # the shard sees nothing else
        ys = convolve_shard(xs, sh, hd)
        d = (ys.double() - y[sh.n_begin:sh.n_end].double()).abs().max().item()
        worst = max(worst, d)
        # seam: oracle window straddling the shard start
        s = max(0, sh.n_begin - 128)
        if sh.n_begin > 0:
            ref = O.scatter_window(w.x, w.h, s, s + 256)
            got = torch.cat([y[s:sh.n_begin], ys[:s + 256 - sh.n_begin]]).cpu().numpy()
            check_tol(got, ref, w.x, w.h, f"seam {sh.n_begin}")
    assert worst <= 2 * configs.tolerance(w.x, w.h, "f32")
