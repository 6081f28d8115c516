"""Short-filter kernel (k_fir_short, Nh <= 256) vs the float64 oracle:
every tap-block count, ragged lengths, output ranges with halos (shards),
batched channels with a pitch, and misaligned input slices (guarded path).
Tolerance 1e-5 * max|x| * ||h||_1 (the FP32 bar)."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _tol(x, h):
    return 1e-5 * float(np.max(np.abs(x))) * float(np.sum(np.abs(h)))


@pytest.mark.parametrize("nh", [1, 2, 3, 4, 5, 8, 9, 12, 16, 17, 20, 24, 28, 31, 32, 33, 36, 47, 60, 63, 64, 65, 100, 128, 129, 200, 255])
@pytest.mark.parametrize("ne", [1, 7, 2048, 70_001])
def test_short_whole_signal(ne, nh):
    from paper_2401_01607_b200.core import Signal, scatter_convolve

    rng = np.random.default_rng(ne * 1000 + nh)
    x = rng.uniform(-1, 1, ne).astype(np.float32)
    h = rng.standard_normal(nh).astype(np.float32)
    for mode in (None, "ffma"):
        y = np.asarray(scatter_convolve(Signal(x), Signal(h), mode=mode).concatenated().samples, np.float64)
        ref = O.scatter_full(x, h)
        assert len(y) == len(ref)
        assert np.max(np.abs(y - ref)) <= _tol(x, h), mode


@pytest.mark.parametrize("nh", [8, 13, 20, 32, 64, 250])
def test_short_shards_and_misaligned_slices(nh):
    import torch

    from paper_2401_01607_b200.sharded import convolve_shard, shard_plan

    rng = np.random.default_rng(nh)
    x = rng.uniform(-1, 1, 123_457).astype(np.float32)
    h = rng.standard_normal(nh).astype(np.float32)
    hd = torch.from_numpy(h).cuda()
    ref = O.scatter_full(x, h)
    for world in (3, 7):
        parts = []
        for sh in shard_plan(len(x), len(h), world):
            xs = torch.from_numpy(x[sh.x_begin:sh.x_end]).cuda()
            parts.append(convolve_shard(xs, sh, hd).cpu().numpy())
        y = np.concatenate(parts).astype(np.float64)
        assert np.max(np.abs(y - ref)) <= _tol(x, h)


def test_short_batched_pitch():
    import torch

    from paper_2401_01607_b200.multichannel import convolve_batched

    rng = np.random.default_rng(3)
    X = rng.uniform(-1, 1, (5, 40_003)).astype(np.float32)
    H = rng.standard_normal((5, 37)).astype(np.float32)
    H[2] *= 1e-4
    Xd = torch.from_numpy(np.pad(X, ((0, 0), (0, 5)))).cuda()[:, :40_003]   # row pitch 40,008
    Y = convolve_batched(Xd, torch.from_numpy(H).cuda()).cpu().numpy()
    for c in range(5):
        ref = O.scatter_full(X[c], H[c])
        assert np.max(np.abs(Y[c].astype(np.float64) - ref)) <= _tol(X[c], H[c])


@pytest.mark.parametrize("nh", [9, 16, 30, 32])
def test_tapreg_bit_identical_to_register_window(nh, tmp_path):
    """k_fir_tapreg (9..32 taps) keeps k_fir_short's per-output chain (fmaf
    over taps ascending from +0), so both kernels give the same bits.  The
    kernel choice is read once per process (SC_SHORT_KIND), hence two
    subprocesses."""
    import os
    import subprocess
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    prog = (
        "import sys, numpy as np, torch\n"
        f"sys.path.insert(0, {repo!r})\n"
        "from paper_2401_01607_b200 import Signal, scatter_convolve\n"
        "rng = np.random.default_rng(77)\n"
        "x = rng.uniform(-1, 1, 300_001).astype(np.float32)\n"
        f"h = rng.standard_normal({nh}).astype(np.float32)\n"
        "y = scatter_convolve(Signal(torch.from_numpy(x).cuda()), Signal(torch.from_numpy(h).cuda()))\n"
        "np.save(sys.argv[1], y.concatenated().samples.cpu().numpy())\n"
    )
    outs = []
    for kind in ("0", "1"):
        f = str(tmp_path / f"y{kind}.npy")
        env = dict(os.environ, SC_SHORT_KIND=kind)
        subprocess.run([sys.executable, "-c", prog, f], check=True, env=env, timeout=300)
        outs.append(np.load(f))
    assert outs[0].dtype == np.float32 and np.array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32))
