"""Host-side logic that needs no GPU: validation (reference messages),
config generators, tolerance, the sharding plan and the multi-process
(world_size 2, gloo) sharded path with the oracle standing in for the
kernel.  CPU only."""

import os
import socket

import numpy as np
import pytest

from oracle import oracle as O
from paper_2401_01607_b200 import (
    ConvOutput,
    EngineConfig,
    Signal,
    commuted_convolve,
    configs,
    direct_form,
    scatter_convolve,
    scatter_convolve_skip_zeros,
    shard_plan,
)


def sig(values, rate=44100):
    return Signal(np.asarray(values, dtype=np.float64), rate)


# ---------------------------------------------------------------- Signal / errors


def test_signal_coerces_to_float64():
    s = sig([1, 2, 3])
    assert s.samples.dtype == np.float64
    assert Signal([1, 2, 3]).samples.dtype == np.float64
    assert len(s) == 3 and s.duration_s == 3 / 44100


def test_signal_keeps_float32():
    assert Signal(np.ones(3, np.float32)).samples.dtype == np.float32


def test_signal_rejects_2d_and_bad_rate():
    with pytest.raises(ValueError, match="1-D"):
        Signal(np.zeros((2, 2)))
    with pytest.raises(ValueError, match="sample_rate"):
        Signal(np.zeros(4), 0)
    with pytest.raises(ValueError, match="sample_rate"):
        Signal(np.zeros(4), -8000)


def test_signal_may_be_empty_and_concat():
    assert len(sig([])) == 0
    out = ConvOutput(body=sig([1.0, 2.0]), tail=sig([3.0]))
    assert np.array_equal(out.concatenated().samples, [1.0, 2.0, 3.0])


@pytest.mark.parametrize("func", [direct_form, scatter_convolve, commuted_convolve])
def test_empty_and_rate_checks_precede_device(func):
    # core.py:69-77 -- raised before any device work (so also on CPU)
    with pytest.raises(ValueError, match="empty"):
        func(sig([]), sig([1.0]))
    with pytest.raises(ValueError, match="empty"):
        func(sig([1.0]), sig([]))
    with pytest.raises(ValueError, match="sample rates differ"):
        func(sig([1.0], 44100), sig([1.0], 48000))


def test_skip_zeros_rejects_negative_threshold():
    with pytest.raises(ValueError, match="threshold"):
        scatter_convolve_skip_zeros(sig([1.0]), sig([1.0]), threshold=-1e-9)


def test_engine_config_validation():
    with pytest.raises(ValueError, match="block_size_nb"):
        EngineConfig(block_size_nb=0)
    with pytest.raises(ValueError, match="zero_skip_threshold"):
        EngineConfig(zero_skip_threshold=-0.1)
    with pytest.raises(ValueError, match="tail_policy"):
        EngineConfig(tail_policy="discard")
    assert EngineConfig().block_size_nb == 8192


# ---------------------------------------------------------------- configs


def test_configs_shapes_and_determinism():
    w1 = configs.cfg1()
    assert w1.x.dtype == np.float64 and w1.ne == 48000 and w1.nh == 1024
    assert w1.metric_macs == 49023 * 1024
    w2 = configs.cfg2()
    assert w2.x.dtype == np.float32 and w2.block == 256 and len(w2.irs) == 19
    h3 = configs.cfg3_h()
    assert h3[0] == 1.0 and len(h3) == 96000
    assert np.array_equal(configs.cfg5_x(ne=1000), configs.cfg5_x(ne=1000))
    assert configs.cfg5(ne=10).metric_macs == (10 + 262143) * 262144


def test_tolerance_formula():
    x = np.array([0.5, -1.0], np.float32)
    h = np.array([2.0, -3.0], np.float32)
    assert configs.tolerance(x, h, "f32") == pytest.approx(1e-5 * 1.0 * 5.0)
    assert configs.tolerance(x, h, "f64") == pytest.approx(1e-12 * 5.0)


# ---------------------------------------------------------------- sharding plan


@pytest.mark.parametrize("ne,nh,world", [(1, 1, 1), (10, 3, 4), (57_600_000, 262_144, 8),
                                         (5, 40, 3), (100, 1, 7), (3, 3, 8)])
def test_shard_plan_partitions_outputs(ne, nh, world):
    plan = shard_plan(ne, nh, world)
    assert len(plan) == world
    nout = ne + nh - 1
    assert plan[0].n_begin == 0 and plan[-1].n_end == nout
    for a, b in zip(plan, plan[1:]):
        assert a.n_end == b.n_begin
    for s in plan:
        if s.n_out:
            # the halo covers every input any owned output reads
            assert s.x_begin == max(0, s.n_begin - nh + 1)
            assert s.x_end == min(ne, s.n_end)
    assert sum(s.n_out for s in plan) == nout


def test_shards_concatenate_to_full_result():
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, 500)
    h = rng.standard_normal(77)
    full = O.scatter_full(x, h)
    parts = []
    for s in shard_plan(len(x), len(h), 5):
        xs = x[s.x_begin:s.x_end]
        # shard-local convolution with the halo, the kernel's sc_fir_range contract
        y = O.scatter_window(np.concatenate([np.zeros(s.x_begin), xs]), h, s.n_begin, s.n_end)
        parts.append(y)
    assert np.array_equal(np.concatenate(parts), full)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2401_01607_b200 import distributed_convolve, gather_shards

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(11)
        x = rng.uniform(-1, 1, 3000).astype(np.float32)
        h = rng.standard_normal(400).astype(np.float32)

        def compute(x_slice, shard, taps):  # oracle stands in for the CUDA kernel
            xx = np.zeros(shard.x_end)
            xx[shard.x_begin:] = x_slice
            y = O.scatter_window(xx, taps, shard.n_begin, shard.n_end)
            return torch.from_numpy(y)

        shard, y_local = distributed_convolve(x, h, compute=compute)
        full = gather_shards(y_local, shard, world, dst=0)
        if rank == 0:
            ref = O.scatter_full(x, h)
            q.put(bool(np.array_equal(full.numpy(), ref)))
    finally:
        dist.destroy_process_group()


def test_distributed_world2_gloo():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) is True


def test_fir_sharded_validation_without_gpu():
    """Argument errors surface before any device work (ValueError)."""
    from paper_2401_01607_b200.sharded import fir_sharded

    with pytest.raises(ValueError, match="input signal is empty"):
        fir_sharded(np.zeros(0), np.ones(3), devices=[0])
    with pytest.raises(ValueError, match="impulse response is empty"):
        fir_sharded(np.ones(3), np.zeros(0), devices=[0])
    with pytest.raises(ValueError, match="mode must be one of"):
        fir_sharded(np.ones(3), np.ones(3), devices=[0], mode="bogus")
