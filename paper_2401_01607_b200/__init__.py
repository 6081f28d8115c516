"""B200-native (sm_100a) scatter / taches convolution -- drop-in for the hot
path of the reference package ``scatterconv`` (arXiv 2401.01607).

Same entry points as pkg/src/scatterconv/__init__.py for the convolution
path:

  scatter_convolve / commuted_convolve / scatter_convolve_skip_zeros /
  direct_form                       whole-signal convolution (core)
  ScatterEngine / EngineConfig      block streaming engine with IR hot swap
  Signal / ConvOutput               sample containers

plus the B200 additions of the north_star: ``convolve_batched``
(multichannel in one launch) and ``convolve_sharded`` /
``distributed_convolve`` (output-time sharding across GPUs).

Everything computes in the CUDA library built in-tree under ``_lib`` and
called through its C ABI (include/scatterconv_b200.h).  There is no CPU
fallback: without the library or a CUDA device every compute call raises.
The reference's other public names (WAV I/O, fixed-point simulation, timing
sweeps; pkg/src/scatterconv/__init__.py:1-85) are re-exported here too, so
``from scatterconv import read_wav``-style code keeps working; their arithmetic
runs on the device as well (csrc/k_wav.cu, csrc/k_fixed.cu, CUDA-event sweeps).
"""

from . import configs
from .core import (
    ConvOutput,
    Signal,
    commuted_convolve,
    direct_form,
    scatter_convolve,
    scatter_convolve_skip_zeros,
)
from .engine import DEFAULT_BLOCK_SIZE, TAIL_POLICIES, EngineConfig, ScatterEngine
from .multichannel import MultiChannelEngine, convolve_batched
from .sharded import (
    Shard,
    convolve_shard,
    convolve_sharded,
    distributed_convolve,
    gather_shards,
    shard_plan,
)

from .fixed_point import (
    FixedPointFormat,
    RequantReport,
    fixed_point_convolve,
    ideal_accumulator_bits,
    ideal_bits_removed,
    mac_requant_count,
    quantize,
    simulate_fixed_point_conv,
)
from .wav import WavFormatError, WavSpec, read_wav, write_wav
from .sweeps import (
    BenchReport,
    BenchRow,
    LinearFit,
    SweepSpec,
    find_realtime_limit,
    gen_white_noise,
    ms_to_samples,
    run_ir_sweep,
    run_nb_sweep,
)

__version__ = "0.1.0"


__all__ = [
    "BenchReport",
    "BenchRow",
    "LinearFit",
    "SweepSpec",
    "find_realtime_limit",
    "run_ir_sweep",
    "run_nb_sweep",
    "ConvOutput",
    "DEFAULT_BLOCK_SIZE",
    "EngineConfig",
    "FixedPointFormat",
    "RequantReport",
    "WavFormatError",
    "WavSpec",
    "fixed_point_convolve",
    "ideal_accumulator_bits",
    "ideal_bits_removed",
    "mac_requant_count",
    "quantize",
    "read_wav",
    "simulate_fixed_point_conv",
    "write_wav",
    "MultiChannelEngine",
    "ScatterEngine",
    "Shard",
    "Signal",
    "TAIL_POLICIES",
    "commuted_convolve",
    "configs",
    "convolve_batched",
    "convolve_shard",
    "convolve_sharded",
    "direct_form",
    "distributed_convolve",
    "gather_shards",
    "gen_white_noise",
    "ms_to_samples",
    "scatter_convolve",
    "scatter_convolve_skip_zeros",
    "shard_plan",
    "__version__",
]
