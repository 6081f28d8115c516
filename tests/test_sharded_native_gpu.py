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
