"""Seeded synthetic workloads for BASELINE.json configs[0..4] (cfg1..cfg5).

No public dataset is involved: every input is uniform white noise drawn the
way the reference's own generator draws it (``gen_white_noise``,
pkg/src/scatterconv/bench.py:43-52: ``default_rng(seed).uniform(-1, 1, n)``)
and impulse responses are decaying Gaussian noise.  The exact recipes and the
proposed seeds are SURVEY.md section 8(d); FP32 configs are cast from the
float64 draws and the oracle is fed the float32 values.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

RATE = 44100


@dataclass
class Workload:
    name: str
    dtype: str                 # "f32" | "f64"
    x: np.ndarray              # [Ne] or [C, Ne]
    h: np.ndarray              # [Nh] or [C, Nh]
    block: int | None = None   # streaming block size (cfg2)
    irs: list = field(default_factory=list)  # cfg2: IR per 100-block segment
    swap_every: int | None = None

    @property
    def channels(self) -> int:
        return 1 if self.x.ndim == 1 else self.x.shape[0]

    @property
    def ne(self) -> int:
        return self.x.shape[-1]

    @property
    def nh(self) -> int:
        return self.h.shape[-1]

    @property
    def nout(self) -> int:
        return self.ne + self.nh - 1

    @property
    def metric_macs(self) -> int:
        """BASELINE.json metric accounting: out samples x taps (x channels)."""
        return self.channels * self.nout * self.nh


def _decay(n: int, tau: float) -> np.ndarray:
    return np.exp(-np.arange(n, dtype=np.float64) / tau)


def cfg1() -> Workload:
    """Single channel whole-signal, float64: 48,000 x 1,024, seeds 0/1."""
    x = np.random.default_rng(0).uniform(-1.0, 1.0, 48000)
    h = np.random.default_rng(1).standard_normal(1024) * _decay(1024, 200.0)
    return Workload("cfg1_whole_f64_48000x1024", "f64", x, h)


def cfg2_ir(j: int) -> np.ndarray:
    return (np.random.default_rng((2, 1, j)).standard_normal(4096) * _decay(4096, 800.0)).astype(
        np.float32)


def cfg2() -> Workload:
    """Streaming B=256, float32, 480,000 x 4,096, IR replaced every 100 blocks."""
    x = np.random.default_rng((2, 0)).uniform(-1.0, 1.0, 480000).astype(np.float32)
    n_blocks = (480000 + 255) // 256
    n_irs = (n_blocks + 99) // 100
    irs = [cfg2_ir(j) for j in range(n_irs)]
    return Workload("cfg2_stream_f32_480000x4096_b256_swap100", "f32", x, irs[0], block=256,
                    irs=irs, swap_every=100)


def cfg3_h() -> np.ndarray:
    rng = np.random.default_rng((3, 1))
    n = np.arange(96000, dtype=np.float64)
    h = rng.standard_normal(96000) * np.exp(-6.91 * n / 72000.0)
    pos = rng.integers(1, 2400, 20)
    h[pos] += rng.uniform(0.2, 0.8, 20) * rng.choice([-1.0, 1.0], 20)
    h[0] = 1.0
    return h.astype(np.float32)


def cfg3(ne: int = 2_880_000) -> Workload:
    """Long reverb, float32: 2,880,000 x 96,000 (+20 early reflections, h[0]=1)."""
    x = np.random.default_rng((3, 0)).uniform(-1.0, 1.0, 2_880_000)[:ne].astype(np.float32)
    return Workload("cfg3_reverb_f32_2880000x96000", "f32", x, cfg3_h())


def cfg4(channels: int = 64, ne: int = 480000) -> Workload:
    """Batched 64 channels x 480,000, each with its own 16,384-tap IR."""
    tau = np.random.default_rng((4, 2)).uniform(1000.0, 6000.0, 64)
    x = np.stack([np.random.default_rng((4, 0, c)).uniform(-1.0, 1.0, 480000)[:ne]
                  for c in range(channels)]).astype(np.float32)
    h = np.stack([np.random.default_rng((4, 1, c)).standard_normal(16384) * _decay(16384, tau[c])
                  for c in range(channels)]).astype(np.float32)
    return Workload("cfg4_batched_f32_64x480000x16384", "f32", x, h)


CFG5_NE = 57_600_000
CFG5_NH = 262_144


def cfg5_h() -> np.ndarray:
    return (np.random.default_rng((5, 1)).standard_normal(CFG5_NH) * _decay(CFG5_NH, 40000.0)).astype(
        np.float32)


def cfg5_x(ne: int = CFG5_NE) -> np.ndarray:
    return np.random.default_rng((5, 0)).uniform(-1.0, 1.0, CFG5_NE)[:ne].astype(np.float32)


def cfg5(ne: int = CFG5_NE) -> Workload:
    """Time-sharded, float32: 57,600,000 x 262,144 (tau = 40,000)."""
    return Workload("cfg5_sharded_f32_57600000x262144", "f32", cfg5_x(ne), cfg5_h())


def cfg5_spot_windows(nout: int = CFG5_NE + CFG5_NH - 1, count: int = 32, width: int = 256):
    """Seeded spot-check window starts."""
    return np.random.default_rng((5, 2)).integers(0, nout - width, count)


def tolerance(x: np.ndarray, h: np.ndarray, dtype: str) -> float:
    """north_star: max-abs error <= 1e-5 * max|x| * ||h||_1 (FP32), 1e-12 (FP64).

    ||h||_1 is computed in float64 from the exact (already-rounded) taps.
    """
    rel = 1e-5 if dtype == "f32" else 1e-12
    xa = float(np.max(np.abs(np.asarray(x, dtype=np.float64)))) if np.size(x) else 0.0
    h1 = float(np.sum(np.abs(np.asarray(h, dtype=np.float64))))
    return rel * xa * h1


ALL = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4, "cfg5": cfg5}
