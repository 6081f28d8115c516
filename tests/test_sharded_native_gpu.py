"""sc_fir_sharded (one call, several devices, output-time partition with
halos) on the one GPU of the box: the device list repeats device 0, which
exercises the partition, per-shard threads/streams and the result
placement; float64 ORDERED must stay bit-identical to the reference."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("ndev", [1, 2, 3, 8])
def test_sharded_f64_ordered_bit_exact(ndev):
    from paper_2401_01607_b200.sharded import fir_sharded

    rng = np.random.default_rng(ndev)
    x, h = rng.uniform(-1, 1, 30_001), rng.standard_normal(1_777)
    y = fir_sharded(x, h, devices=[0] * ndev)
    assert isinstance(y, np.ndarray) and np.array_equal(y, O.scatter_full(x, h))


@pytest.mark.parametrize("ndev,nh", [(1, 300), (4, 300), (3, 5_000), (5, 20)])
def test_sharded_f32_fast_within_tol(ndev, nh):
    from paper_2401_01607_b200.sharded import fir_sharded

    rng = np.random.default_rng(10 * ndev + nh)
    x = rng.uniform(-1, 1, 123_457).astype(np.float32)
    h = rng.standard_normal(nh).astype(np.float32)
    y = fir_sharded(x, h, devices=[0] * ndev)
    ref = O.scatter_full(x, h)
    tol = 1e-5 * np.max(np.abs(x)) * np.sum(np.abs(h))
    assert y.dtype == np.float32 and np.max(np.abs(y.astype(np.float64) - ref)) <= tol


def test_sharded_gather_device_and_more_devices_than_outputs():
    import torch

    from paper_2401_01607_b200.sharded import fir_sharded

    rng = np.random.default_rng(3)
    x, h = rng.uniform(-1, 1, 5), rng.standard_normal(3)
    y = fir_sharded(x, h, devices=[0] * 16, gather_device=0)   # 7 outputs, 16 shards
    assert isinstance(y, torch.Tensor) and y.is_cuda
    assert np.array_equal(y.cpu().numpy(), O.scatter_full(x, h))
    with pytest.raises(ValueError, match="no device"):
        fir_sharded(x, h, devices=[99])


@pytest.mark.parametrize("nh", [2_500, 1_501])
@pytest.mark.parametrize("chunks", [1, 3, 7])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_range_host_chunk_pipeline(chunks, dtype, nh):
    """sc_fir_range_host: output sub-ranges of a host signal, cut into chunks
    whose upload / FIR / download overlap; float64 ORDERED bit-exact, float32
    FAST within the FP32 tolerance, pinned and pageable buffers alike.  (In
    float64, 1,501 taps run k_chain_small with a nonzero drive offset, drive
    window and first output; 2,500 taps the windowed chain.)"""
    import torch

    from paper_2401_01607_b200 import _native as N

    rng = np.random.default_rng(chunks)
    x = rng.uniform(-1, 1, 70_001).astype(dtype)
    h = rng.standard_normal(nh).astype(dtype)
    ref = O.scatter_full(x, h)
    dt = N.dtype_code(dtype)
    mode = N.SC_MODE_FAST if dtype == np.float32 else N.SC_MODE_ORDERED
    tol = 1e-5 * np.max(np.abs(x)) * np.sum(np.abs(h))
    for a, b in [(0, len(ref)), (1_234, 50_000), (60_000, len(ref))]:
        for pinned in (True, False):
            xp = torch.from_numpy(x).pin_memory() if pinned else torch.from_numpy(x)
            y = torch.empty(b - a, dtype=xp.dtype, pin_memory=pinned)
            N.check(N.lib().sc_fir_range_host(dt, mode, N.ptr(xp), len(x), N.ptr(torch.from_numpy(h)), len(h),
                                              N.ptr(y), a, b, 0, chunks))
            got = y.numpy()
            if dtype == np.float64:
                assert np.array_equal(got, ref[a:b]), (a, b, pinned)
            else:
                assert np.max(np.abs(got.astype(np.float64) - ref[a:b])) <= tol, (a, b, pinned)


def test_distributed_convolve_to_host_shards_concatenate():
    """distributed_convolve(to_host=True) per rank (rank/world given, no
    process group): each shard's pinned host segment, concatenated, is the
    full result."""
    from paper_2401_01607_b200.sharded import distributed_convolve

    rng = np.random.default_rng(9)
    x = rng.uniform(-1, 1, 200_000).astype(np.float32)
    h = rng.standard_normal(3_000).astype(np.float32)
    parts = [distributed_convolve(x, h, rank=r, world=3, to_host=True)[1].numpy() for r in range(3)]
    ref = O.scatter_full(x, h)
    tol = 1e-5 * np.max(np.abs(x)) * np.sum(np.abs(h))
    assert np.max(np.abs(np.concatenate(parts).astype(np.float64) - ref)) <= tol
