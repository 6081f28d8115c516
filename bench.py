#!/usr/bin/env python
"""Benchmark: convolution GMAC/s (out samples x taps) and % of FP32 FMA peak.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg5]
    python bench.py --impl reference ...        # CPU reference arm

Default workload is BASELINE.json configs[4] (cfg5): 57,600,000 x 262,144
float32, time-sharded over the N GPUs of one node (one process per GPU under
torchrun; each rank owns an equal contiguous output segment and uploads its
input slice plus the (Nh-1)-sample halo; no collective on the data path).
A "step" is one full convolution of that workload.  Other configs
(--config cfg1..cfg4) are available for profiling; the parity tests cover
them all.

Timing: W warm-up steps, then K steps, each bracketed by CUDA events on the
launching stream, with a 256 MiB L2-flush memset before every step outside
the events (inputs are also > L2 at N=1).  Barrier + synchronize around the
region; the step time is the MAX over ranks.  `value` = total metric MACs /
step time.  `e2e` = same metric through the public API with host (pinned)
buffers, H2D + D2H inside the timed region.  `cpu_baseline` = the CPU oracle
(restatement of the reference's scatter_block engine, float64) on a bounded
sample, rank 0, N=1 only.  Rank 0 prints ONE JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import pathlib
import statistics
import sys
import threading
import time

import numpy as np

REPO = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = json.loads((REPO / "BASELINE.json").read_text())["metric"] if (REPO / "BASELINE.json").exists() \
    else "convolution GMAC/s (out samples x taps) and % of FP32 FMA peak at 1/2/4/8 GPU"
UNIT = "GMAC/s"



def _config_name(v: str) -> str:
    import argparse
    import re

    if v in ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5", "mstream") or re.fullmatch(r"short[1-9][0-9]*", v):
        return v
    raise argparse.ArgumentTypeError(f"unknown config {v!r} (cfg1..cfg5, mstream or shortN)")

def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="cfg5", type=_config_name,
                    help="cfg1..cfg5, mstream, or shortN (2^26 samples x N taps, N >= 1)")
    ap.add_argument("--mode", default="auto", choices=["auto", "fast", "ffma", "tc", "ordered"],
                    help="auto = the library default (float32: fast, tensor cores for long filters; "
                         "float64: ordered, bit-exact); fast on a float64 config = fused-FMA chain; "
                         "ordered = the sequential-chain kernel")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=20.0,
                    help="target seconds of CPU work for the cpu_baseline sample")
    # CPU test mode (SC_BENCH_COMPUTE=oracle): the multi-rank sharding, timing
    # and reporting logic with the CPU oracle standing in for the kernel, on a
    # reduced cfg5-law signal -- for tests/test_bench_cpu.py under gloo; never
    # a GPU number (its line says so)
    ap.add_argument("--test-ne", type=int, default=0, help=argparse.SUPPRESS)
    ap.add_argument("--test-nh", type=int, default=0, help=argparse.SUPPRESS)
    return ap.parse_args()


def free_port() -> int:
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` outside torchrun: re-launch this script as N ranks
    (one process per GPU) under torch.distributed.run on 127.0.0.1; rank 0
    prints the JSON line on the shared stdout."""
    import subprocess

    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), str(REPO / "bench.py"),
           *sys.argv[1:]]
    print(f"[bench] spawning {args.gpus} ranks: {' '.join(cmd[2:7])}", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def env_rank():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


# ------------------------------------------------------------------ clocks


class ClockSampler:
    """Samples SM clock + clock-event reasons via NVML during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index: int, period: float = 0.1):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._period = period
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        nv = self._nv
        get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            getattr(nv, "nvmlDeviceGetCurrentClocksThrottleReasons")
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = get_r(self._h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(self._period)

    def __enter__(self):
        if self._nv:
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._nv and self._t.is_alive():
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ------------------------------------------------------------------ workloads


def max_over_ranks(v: float, world: int, device) -> float:
    """MAX of a per-rank float over all ranks (device tensor under NCCL,
    host tensor under gloo)."""
    if world == 1:
        return float(v)
    import torch
    import torch.distributed as dist

    dev = device if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([v], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def peaks():
    p = {}
    f = REPO / "MEASURED_PEAKS.json"
    if f.exists():
        p = json.loads(f.read_text())
    return p


class Work:
    """One rank's share of a config: device inputs + a step() callable."""

    def __init__(self, cfg, rank, world, device):
        import torch

        from paper_2401_01607_b200 import configs
        from paper_2401_01607_b200.sharded import shard_plan

        self.cfg = cfg
        self.device = device
        self.kind = cfg
        if cfg in ("cfg5", "cfg3"):
            w = configs.cfg5() if cfg == "cfg5" else configs.cfg3()
            self.w = w
            self.plan = shard_plan(w.ne, w.nh, world)
            self.shard = self.plan[rank]
            self.total_macs = w.metric_macs
            self.rank_macs = self.shard.n_out * w.nh
            self.x_host = w.x
            self.h_host = w.h
            self.xs = torch.from_numpy(w.x[self.shard.x_begin:self.shard.x_end]).to(device)
            self.hd = torch.from_numpy(w.h).to(device)
            self.parallelism = f"time-sharded x{world} (output segments + {w.nh - 1}-sample halo, no collective)"
            self.scaling = "strong"
            self.dtype = "f32"
        elif cfg == "cfg4":
            w = configs.cfg4()
            self.w = w
            per = -(-64 // world)
            self.c0, self.c1 = min(64, rank * per), min(64, rank * per + per)
            self.total_macs = w.metric_macs
            self.rank_macs = (self.c1 - self.c0) * w.nout * w.nh
            self.xd = torch.from_numpy(w.x[self.c0:self.c1]).to(device)
            self.hd = torch.from_numpy(w.h[self.c0:self.c1]).to(device)
            self.parallelism = f"channel-sharded x{world} (no collective)"
            self.scaling = "strong"
            self.dtype = "f32"
        elif cfg == "cfg1":
            w = configs.cfg1()
            self.w = w
            self.total_macs = w.metric_macs * world   # replicas
            self.rank_macs = w.metric_macs
            self.xd = torch.from_numpy(w.x).to(device)
            self.hd = torch.from_numpy(w.h).to(device)
            self.parallelism = f"replicas x{world}"
            self.scaling = "weak"
            self.dtype = "f64"
        elif cfg.startswith("short"):
            # short-filter HBM sanity sweep: Ne = 2^26, Nh = 8..64
            nh = int(cfg[5:])
            rng = np.random.default_rng(77)
            x = rng.uniform(-1, 1, 1 << 26).astype(np.float32)
            h = rng.standard_normal(nh).astype(np.float32)
            self.w = configs.Workload(f"short_f32_67108864x{nh}", "f32", x, h)
            self.total_macs = self.w.metric_macs * world
            self.rank_macs = self.w.metric_macs
            self.xd = torch.from_numpy(x).to(device)
            self.hd = torch.from_numpy(h).to(device)
            self.parallelism = f"replicas x{world}"
            self.scaling = "weak"
            self.dtype = "f32"
        elif cfg == "mstream":
            # cfg4's 64 channels streamed through ONE
            # multichannel engine (blocks of 8192 = the reference default,
            # engine.py:33), ordered chain, IR swapped halfway (cli.py --swap-ir)
            w = configs.cfg4()
            self.w = w
            self.total_macs = w.metric_macs * world
            self.rank_macs = w.metric_macs
            self.xd = torch.from_numpy(w.x).to(device)
            self.hd = torch.from_numpy(w.h).to(device)
            self.hd2 = torch.flip(self.hd, dims=[1]).contiguous()
            n_blocks = -(-w.ne // 8192)
            self.swaps = [(0, self.hd), (n_blocks // 2, self.hd2)]
            from paper_2401_01607_b200.engine import EngineConfig
            from paper_2401_01607_b200.multichannel import MultiChannelEngine

            self._make_engine = lambda mode: MultiChannelEngine(self.hd, EngineConfig(block_size_nb=8192),
                                                                mode=mode)
            self.parallelism = f"replicas x{world} (one 64-channel engine per GPU)"
            self.scaling = "weak"
            self.dtype = "f32"
        elif cfg == "cfg2":
            w = configs.cfg2()
            self.w = w
            self.total_macs = (w.ne + w.nh - 1) * w.nh * world
            self.rank_macs = (w.ne + w.nh - 1) * w.nh
            self.xd = torch.from_numpy(w.x).to(device)
            n_blocks = -(-w.ne // 256)
            self.h0 = torch.from_numpy(w.irs[0]).to(device)
            # block 0 re-selects IR 0 so every step replays the identical stream
            self.swaps = [(0, self.h0)] + [(b, torch.from_numpy(w.irs[b // 100]).to(device))
                                           for b in range(100, n_blocks, 100)]
            from paper_2401_01607_b200.core import Signal
            from paper_2401_01607_b200.engine import EngineConfig, ScatterEngine

            self._make_engine = lambda mode: ScatterEngine(Signal(self.h0), EngineConfig(block_size_nb=256),
                                                           mode=mode)
            self.parallelism = f"replicas x{world} (streaming is sequential per stream)"
            self.scaling = "weak"
            self.dtype = "f32"

    def pick_kernel(self):
        """Which kernel family the library runs for this config/mode (mirrors
        capi.cu's FAST dispatch).  The tensor-core work it issues is read from
        the library itself (sc_tc_stats) around the timed region."""
        if self.cfg.startswith("short"):
            # FAST dispatch (capi.cu / k_fast_f32.cu): tensor cores from 26
            # taps at this size (the fused-split k_tc_fir_fs), the streaming
            # k_fir_short up to 8 taps and the tap-stationary k_fir_tapreg
            # below 26 (HBM-bound).  Filters of at most two 128-tap shifts on tensor
            # cores are HBM-bound too: 2 shifts of MMAs take less than moving
            # 8 B per output
            nh = self.w.nh
            use_tc = self.mode == "tc" or (self.mode in ("fast", "auto") and nh >= 26)   # capi.cu kTcShortMinTaps
            self.kernel = "k_tc_fir" if use_tc else ("k_fir_short" if nh <= 8 else "k_fir_tapreg" if nh <= 32
                                                     else "k_fir_short_smem")
            self.hbm_bound = (nh <= 32 and not use_tc) or (use_tc and nh <= 255)
            return
        if self.cfg == "cfg2":
            # float32 engine: FAST mode convolves the 19 equal IR segments in one
            # batched tensor-core launch; --mode ordered keeps the ordered chain
            fast = self.mode != "ordered"
            self.eng = self._make_engine("fast" if fast else "ordered")
            self.kernel = "k_tc_fir" if fast else "k_chain_w"
            return
        if self.cfg == "mstream":
            # float32 engine: FAST mode puts each IR segment (2 x 64 ch x 240,000
            # samples x 16,384 taps) on the tensor-core FIR (csrc/engine.cu
            # fast_stream); --mode ordered keeps the ordered chain
            fast = self.mode != "ordered"
            self.eng = self._make_engine("fast" if fast else "ordered")
            self.kernel = "k_tc_fir" if fast else "k_chain_w"
            return
        if self.dtype != "f32" or self.cfg not in ("cfg3", "cfg4", "cfg5") or self.mode == "ordered":
            # ordered chain (csrc/k_ordered.cu): strict float64 with one IR of
            # <= 2,048 taps runs the latency kernel k_chain_small
            self.kernel = "k_chain_small" if self.dtype == "f64" and self.w.nh <= 2048 else "k_chain_w"
            return
        nh = self.w.nh
        use_tc = self.mode == "tc" or (self.mode in ("fast", "auto") and nh >= 256)
        self.kernel = "k_tc_fir" if use_tc else ("k_fir_short" if nh <= 8 else "k_fir_tapreg" if nh <= 32 else
                                                 "k_fir_short_smem" if nh <= 256 else "k_fir_f32_fast")

    def step(self):
        import torch

        from paper_2401_01607_b200.core import Signal, scatter_convolve
        from paper_2401_01607_b200.engine import EngineConfig, ScatterEngine
        from paper_2401_01607_b200.multichannel import convolve_batched
        from paper_2401_01607_b200.sharded import convolve_shard

        if self.cfg in ("cfg5", "cfg3"):
            return convolve_shard(self.xs, self.shard, self.hd, mode=self.lib_mode)
        if self.cfg == "cfg4":
            return convolve_batched(self.xd, self.hd, mode=self.lib_mode)
        if self.cfg == "cfg1":
            # the full Ne+Nh-1 result (ConvOutput body/tail are views of it);
            # auto = ordered (bit-exact), --mode fast = fused-FMA chain
            return scatter_convolve(Signal(self.xd), Signal(self.hd), mode=self.lib_mode).body.samples
        if self.cfg == "cfg2":
            # 1,875 blocks of 256 with 18 IR swaps, then the flush of the tail
            # (engine.py:148-161) -- the whole stream, no host round-trip until
            # the flush (which returns the data-dependent tail length).
            body = self.eng.process_stream(self.xd, 256, self.swaps)
            self.eng.flush()
            return body
        if self.cfg.startswith("short"):
            return scatter_convolve(Signal(self.xd), Signal(self.hd), mode=self.lib_mode).body.samples
        if self.cfg == "mstream":
            body = self.eng.process_stream(self.xd, 8192, self.swaps)
            tails, _ = self.eng.flush(on_device=True)   # [64, 16383] tails stay in HBM like the body
            return body, tails
        raise ValueError(self.cfg)

    def e2e_step(self, x_pin, h_pin):
        """Public API with host (pinned) buffers; returns (h2d, d2h) bytes."""
        import torch.distributed as dist

        from paper_2401_01607_b200.core import Signal, scatter_convolve
        from paper_2401_01607_b200.multichannel import convolve_batched
        from paper_2401_01607_b200.sharded import distributed_convolve

        if self.cfg in ("cfg5", "cfg3"):
            if dist.is_available() and dist.is_initialized():
                sh, y = distributed_convolve(x_pin, h_pin, to_host=True)
                return sh.n_in * 4 + len(h_pin) * 4, y.numel() * 4
            out = scatter_convolve(Signal(x_pin), Signal(h_pin))   # body/tail: pinned host views
            return x_pin.numel() * 4 + h_pin.numel() * 4, (len(out.body) + len(out.tail)) * 4
        if self.cfg == "cfg4":
            y = convolve_batched(x_pin, h_pin)
            return x_pin.numel() * 4 + h_pin.numel() * 4, y.numel() * 4
        es = x_pin.element_size()
        if self.cfg == "cfg1" or self.cfg.startswith("short"):
            out = scatter_convolve(Signal(x_pin), Signal(h_pin), mode=self.lib_mode)
            return (x_pin.numel() + h_pin.numel()) * es, (len(out.body) + len(out.tail)) * es
        if self.cfg in ("cfg2", "mstream"):
            # the same stream and swap schedule from pinned host memory; body
            # and flushed tail come back to the host
            if not hasattr(self, "swaps_pin"):
                self.swaps_pin = [(b, ir.cpu().pin_memory()) for b, ir in self.swaps]
            body = self.eng.process_stream(x_pin, 256 if self.cfg == "cfg2" else 8192, self.swaps_pin)
            tail = self.eng.flush()
            tail_n = len(tail) if self.cfg == "cfg2" else sum(len(t) for t in tail)
            h2d = x_pin.numel() * es + sum(ir.numel() for _, ir in self.swaps_pin) * es
            return h2d, (body.numel() + tail_n) * es
        raise ValueError(f"no e2e path for {self.cfg}")


E2E_API = {
    "cfg4": "paper_2401_01607_b200.convolve_batched(pinned host [C, N], pinned host [C, Nh])",
    "cfg2": "ScatterEngine.process_stream(pinned host, 256, pinned-host swaps) + flush()",
    "mstream": "MultiChannelEngine.process_stream(pinned host [64, N], 8192, pinned-host swaps) + flush()",
}


# ------------------------------------------------------------------ CPU reference


def cpu_sample(cfg, seconds, threads):
    """Time the oracle (float64 restatement of the reference engine) on a
    bounded prefix of the workload sized to ~`seconds` of work."""
    from oracle import oracle as O
    from paper_2401_01607_b200 import configs

    if cfg in ("cfg4", "mstream"):   # mstream streams cfg4's channels
        w = configs.cfg4(channels=64, ne=480000)
        x, h = w.x, w.h
    elif cfg == "cfg3":
        x, h = configs.cfg3().x, configs.cfg3_h()
    elif cfg == "cfg1":
        w = configs.cfg1()
        x, h = w.x, w.h
    elif cfg == "cfg2":
        w = configs.cfg2()
        x, h = w.x, w.irs[0]
    else:
        x, h = configs.cfg5_x(ne=4_000_000), configs.cfg5_h()
    x = np.asarray(x, np.float64)
    h = np.asarray(h, np.float64)
    if cfg in ("cfg4", "mstream"):
        # one engine per channel on a thread pool (the reference's pattern)
        c = max(1, threads)
        ne0 = 8192
        t0 = time.perf_counter()
        O.conv_channels(x[:c, :ne0], h[:c], nb=8192, threads=threads)
        dt = time.perf_counter() - t0
        rate = c * ne0 * h.shape[1] / dt
        ne = int(min(x.shape[1], max(ne0, seconds * rate / (c * h.shape[1]))))
        t0 = time.perf_counter()
        O.conv_channels(x[:c, :ne], h[:c], nb=8192, threads=threads)
        dt = time.perf_counter() - t0
        macs = c * ne * h.shape[1]
        return macs / dt / 1e9, f"{c} channels x {ne} samples x {h.shape[1]} taps ({macs:.3e} MAC, one float64 engine per channel, {threads} threads)", dt
    nh = len(h)
    s0 = min(len(x), max(2000, 2048 * threads))   # probe big enough to amortise thread start-up
    t0 = time.perf_counter()
    O.conv_parallel(x[:s0], h, nb=8192, threads=threads)
    dt = time.perf_counter() - t0
    rate = s0 * nh / dt
    s = int(min(len(x), max(s0, seconds * rate / nh)))
    t0 = time.perf_counter()
    O.conv_parallel(x[:s], h, nb=8192, threads=threads)
    dt = time.perf_counter() - t0
    macs = s * nh
    return macs / dt / 1e9, (f"x[:{s}] x {nh} taps ({macs:.3e} MAC actually scattered), float64 "
                             f"scatter_block engine per input segment, overlap-add, {threads} threads"), dt


def workload_config(cfg: str) -> dict:
    """The `config` object of a bench line for `cfg` (same keys on both arms;
    host-only, no device)."""
    from paper_2401_01607_b200 import configs

    if cfg.startswith("short"):
        nh = int(cfg[5:])
        ne, ch, name = 1 << 26, 1, f"short_f32_67108864x{nh}"
    else:
        w = configs.ALL["cfg4" if cfg == "mstream" else cfg]()
        ne, nh, ch, name = w.ne, w.nh, w.channels, w.name
        if cfg == "mstream":
            name = "mstream_f32_64ch_480000x16384_b8192_1swap_multichannel_engine"
    return {"workload": name, "ne": int(ne), "nh": int(nh), "channels": int(ch),
            "metric_macs": int(ch * (ne + nh - 1) * nh)}


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    threads = len(os.sched_getaffinity(0))
    per_step = max(2.0, min(args.cpu_seconds, 150.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        cpu_sample(args.config, per_step / 4, threads)
    rates, samples, times = [], [], []
    for _ in range(args.steps):
        r, s, dt = cpu_sample(args.config, per_step, threads)
        rates.append(r)
        samples.append(s)
        times.append(dt)
    value = statistics.median(rates)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * statistics.median(times),
        "higher_is_better": True, "scaling": "strong" if args.config in ("cfg3", "cfg4", "cfg5") else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded PCG64, SURVEY.md 8(d))",
        "config": {**workload_config(args.config), "parallelism": f"CPU, {threads} threads"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": samples[-1]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "reference is Python+numba (no compiled C to build); timed via the C restatement "
                "of its scatter_block engine (oracle/), pinned bit-exact to the reference",
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ CPU test mode


def run_cpu_test_mode(args):
    """SC_BENCH_COMPUTE=oracle: the same rank/shard/timing/report logic as the
    GPU path, on CPU under gloo, with the oracle computing each rank's shard
    of a reduced cfg5-law signal (--test-ne x --test-nh).  Rank 0 gathers the
    shards (sharded.gather_shards) and checks they cover the full output and
    equal the oracle's single-pass result.  Test infrastructure: the line
    carries "compute": "oracle-cpu" and is never a benchmark number."""
    import torch
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2401_01607_b200.sharded import gather_shards, shard_plan

    rank, world, _ = env_rank()
    if world > 1:
        dist.init_process_group(os.environ.get("SC_DIST_BACKEND", "gloo"))
    ne = args.test_ne or 40_000
    nh = args.test_nh or 1_000
    rng = np.random.default_rng((5, 0))
    x = rng.uniform(-1, 1, ne).astype(np.float32)
    h = (np.random.default_rng((5, 1)).standard_normal(nh) * np.exp(-np.arange(nh) / (nh / 6.5))).astype(np.float32)
    plan = shard_plan(ne, nh, world)
    sh = plan[rank]

    def step():
        xx = np.zeros(sh.x_end)
        xx[sh.x_begin:] = x[sh.x_begin:sh.x_end]   # this rank sees only its slice + halo
        return torch.from_numpy(O.scatter_window(xx, h, sh.n_begin, sh.n_end))

    for _ in range(args.warmup):
        step()
    if world > 1:
        dist.barrier()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        y = step()
        times.append(time.perf_counter() - t0)
    ms_local = 1000 * sum(times) / len(times)
    if world > 1:
        t = torch.tensor([ms_local], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        full = gather_shards(y, sh, world, dst=0)
    else:
        ms, full = ms_local, y
    if rank == 0:
        ref = O.scatter_full(x, h)
        got = full.numpy()
        line = {
            "metric": METRIC, "value": (ne + nh - 1) * nh / (ms * 1e-3) / 1e9, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "compute": "oracle-cpu (SC_BENCH_COMPUTE=oracle test mode: no GPU, not a benchmark number)",
            "config": {"workload": f"cfg5-law {ne}x{nh} (test mode)", "ne": ne, "nh": nh,
                       "parallelism": f"time-sharded x{world} (output segments + {nh - 1}-sample halo)"},
            "coverage": {"outputs": int(len(ref)), "gathered": int(len(got)),
                         "shards": [[p.n_begin, p.n_end] for p in plan],
                         "max_abs_err": float(np.max(np.abs(got - ref))) if len(got) == len(ref) else None},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


# ------------------------------------------------------------------ main


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    if os.environ.get("SC_BENCH_COMPUTE") == "oracle":
        return run_cpu_test_mode(args)

    import torch
    import torch.distributed as dist

    from paper_2401_01607_b200 import _native as N

    rank, world, local = env_rank()
    if world > 1:
        local = local % torch.cuda.device_count()
        torch.cuda.set_device(local)
        # SC_DIST_BACKEND=gloo lets the multi-rank timing/sharding logic run
        # with several ranks on one GPU (NCCL refuses duplicate devices); the
        # data path has no collective either way -- only barrier/max-reduce.
        backend = os.environ.get("SC_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        # make the communicator visible (and eagerly created): one tiny
        # all-reduce, then report its rank count
        probe = torch.ones(1, device=torch.device("cuda", local) if backend == "nccl" else "cpu")
        dist.all_reduce(probe)
        comm = {"backend": dist.get_backend(), "nranks": dist.get_world_size(), "allreduce_check": int(probe.item())}
        print(f"[bench] rank {rank}: {comm['backend']} communicator nranks={comm['nranks']} "
              f"device=cuda:{local}", file=sys.stderr, flush=True)
    else:
        torch.cuda.set_device(0)
        comm = {"backend": None, "nranks": 1}
    device = torch.device("cuda", torch.cuda.current_device())
    L = N.lib()
    work = Work(args.config, rank, world, device)
    work.mode = args.mode
    work.lib_mode = None if args.mode == "auto" else args.mode
    work.pick_kernel()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=device)  # 256 MiB > L2

    def barrier():
        if world > 1:
            dist.barrier()

    # warm-up (same sequence as a timed step: L2 flush, then the step)
    for _ in range(max(args.warmup, 0)):
        flush.zero_()
        work.step()
    torch.cuda.synchronize()
    barrier()

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    dev_index = torch.cuda.current_device()
    phys = os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",")
    nvml_index = int(phys[dev_index]) if len(phys) > dev_index and phys[dev_index].strip().isdigit() else dev_index
    torch.cuda.synchronize()
    barrier()
    launches0 = L.sc_launch_count()
    L.sc_tc_stats_reset()
    with ClockSampler(nvml_index) as clocks:
        t_wall0 = time.perf_counter()
        # ~1 ms of device-side spin ahead of the first step, so the host's
        # enqueue of step 0 does not show up as idle time inside its events
        # (later steps are enqueued while the previous one runs)
        torch.cuda._sleep(2_000_000)
        for i in range(args.steps):
            flush.zero_()
            starts[i].record()
            work.step()
            ends[i].record()
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall0
    launches = L.sc_launch_count() - launches0
    tc = N.tc_stats()   # the library's own count of the tensor-core work it issued
    barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    ms_local = sum(step_ms) / len(step_ms)
    ms = max_over_ranks(ms_local, world, device)
    value = work.total_macs / (ms * 1e-3) / 1e9

    # roofline of the dominant kernel on this rank
    p = peaks()
    sms = torch.cuda.get_device_properties(device).multi_processor_count
    sm_max = float(p.get("sm_max_mhz", 1965.0))
    csum = clocks.summary()
    fp32_peak = 2 * 128 * sms * sm_max * 1e6 / 1e12  # TFLOP/s at max clock
    useful = 2 * work.rank_macs / (ms_local * 1e-3) / 1e12   # useful FP32-equivalent TFLOP/s
    med = csum["sm_mhz"] or sm_max
    traffic = None
    tf = REPO / "profiles" / "ncu_traffic.json"
    if tf.exists():
        tt = json.loads(tf.read_text())
        if work.kernel == "k_tc_fir" and tc["launches"]:
            traffic = tt.get(f"{args.config}_{tc['kernel'] or 'k_tc_fir'}<{tc['ssh']},{tc['tile_n']}>")
        else:
            traffic = tt.get(f"{args.config}_{work.kernel}")
    if getattr(work, "hbm_bound", False):
        # short filters: the kernel should stream x in and y out at HBM speed
        hbm = float(p.get("hbm_gbs", 6650.0))
        alg_bytes = 4 * (work.w.ne + work.w.nh + work.w.nout)
        gbs = alg_bytes / (ms_local * 1e-3) / 1e9
        roofline = {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                    "traffic": traffic, "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                    "alg_bytes_per_launch": alg_bytes, "kernel": work.kernel}
        if work.kernel == "k_tc_fir" and tc["launches"]:
            tc_peak = float(p.get("bf16_tflops", 1590.0))
            tflops = 2 * 3 * tc["padded_macs"] / args.steps / (ms_local * 1e-3) / 1e12
            roofline["kernel"] = (f"k_tc_fir_fs<{tc['ssh']},{tc['tile_n']}> (fused split: x read as FP32)"
                                  if tc["kernel"] == "k_tc_fir_fs" else
                                  f"k_tc_fir<{tc['ssh']},{tc['tile_n']}> (fp16 hi/lo operand image in HBM)")
            roofline["tensor"] = {"achieved_tflops": tflops, "frac": tflops / tc_peak,
                                  "note": "the tensor roof is not the binding one at <= 2 shifts"}
    elif work.kernel == "k_tc_fir" and tc["launches"]:
        # tensor work actually issued, as the library counts it (sc_tc_stats):
        # 3 fp16 MMAs (hi*hi, lo*hi, hi*lo) over the padded block-Toeplitz
        # GEMM -- whole 128 x tile_n-row tiles x 128 taps x drain-padded shifts
        tc_peak = float(p.get("bf16_tflops", 1590.0))
        padded = tc["padded_macs"] / args.steps
        achieved = 2 * 3 * padded / (ms_local * 1e-3) / 1e12
        # the library names the kernel that issued the MMAs (sc_tc_last_kernel):
        # k_tc_fir (operand image) or k_tc_fir_fs (fused split, medium filters)
        tmpl = f"{tc['kernel'] or 'k_tc_fir'}<{tc['ssh']},{tc['tile_n']}>"
        work.kernel_template = tmpl
        roofline = {
            "bound": "tensor", "achieved": achieved, "peak": tc_peak, "unit": "TFLOP/s",
            "frac": achieved / tc_peak, "traffic": traffic,
            "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst, cuBLAS bf16; fp16 MMA runs at "
                           "the same rate)" if "bf16_tflops" in p else "fallback 1.59 PFLOP/s",
            "achieved_per_launch": f"2 x 3 x {padded:.6e} padded MMA MACs per step (sc_tc_stats: "
                                   f"{tc['launches'] / args.steps:g} launches/step) / mean step time",
            "frac_of_nominal_dense_fp16": achieved / 2250.0,
            "peak_note": "frac > 1 means the kernel's MMA issue rate beats the driver's cuBLAS bf16 "
                         "measurement; the nominal dense fp16 peak is 2250 TFLOP/s",
            "useful_fp32_tflops": useful,
            "useful_frac_of_fp32_fma_peak": useful / fp32_peak,
            "kernel": f"{tmpl} (tcgen05.mma kind::f16 M128 x N{tc['tile_n']} x K16, TMEM accumulators, "
                      f"TMEM drain every {tc['ssh']} shifts, "
                      + ("x read as FP32 and split to fp16 hi/lo in shared memory)" if tc["kernel"] == "k_tc_fir_fs"
                         else "cp.async.bulk of the fp16 hi/lo operand image)"),
        }
    elif work.dtype == "f64":
        # ordered float64 chain: every MAC is a DMUL and a DADD (separately
        # rounded, the reference's arithmetic), i.e. 2 FP64-pipe lane-ops; the
        # FP64 pipe issues 64 lane-ops/clk/SM (tools/ubench/fp64_latency.cu
        # measured 62.2 for DADD at 32 warps/SM)
        dp_peak = 64 * sms * sm_max * 1e6 / 1e12  # T lane-ops/s
        ops_per_mac = 1 if args.mode == "fast" else 2   # DFMA vs DMUL + DADD
        dp_ops = ops_per_mac * work.rank_macs / (ms_local * 1e-3) / 1e12
        roofline = {
            "bound": "fp64_pipe", "achieved": dp_ops, "peak": dp_peak, "unit": "Tops/s (FP64 pipe lane-ops)",
            "frac": dp_ops / dp_peak, "traffic": traffic,
            "peak_source": f"computed: {sms} SMs x 64 FP64 lane-ops/clk x sm_max_mhz {sm_max:.0f}; "
                           "microbenchmark tools/ubench/fp64_latency.cu: 62.2 lane-ops/clk/SM",
            "achieved_per_launch": f"{ops_per_mac} x metric MACs ({'DFMA' if ops_per_mac == 1 else 'DMUL + DADD'}) / mean step time",
            "frac_at_observed_clock": dp_ops / (64 * sms * med * 1e6 / 1e12),
            "kernel": work.kernel,
        }
    else:
        roofline = {
            "bound": "fp32_fma",
            "achieved": useful, "peak": fp32_peak, "unit": "TFLOP/s", "frac": useful / fp32_peak,
            "traffic": traffic,
            "peak_source": f"computed: {sms} SMs x 128 FP32 FMA/clk x 2 FLOP x sm_max_mhz {sm_max:.0f} "
                           "(MEASURED_PEAKS.json); no FP32-FMA peak is measured by the driver",
            "frac_at_observed_clock": useful / (2 * 128 * sms * med * 1e6 / 1e12),
            "kernel": work.kernel,
        }
    roofline["achieved_from"] = "CUDA events around each step on the launching stream"

    # e2e through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        if args.config == "cfg4":
            x_pin = torch.from_numpy(work.w.x[work.c0:work.c1]).pin_memory()
            h_pin = torch.from_numpy(work.w.h[work.c0:work.c1]).pin_memory()
        elif args.config not in ("cfg3", "cfg5"):
            x_pin = work.xd.cpu().pin_memory()
            h_pin = work.hd.cpu().pin_memory() if hasattr(work, "hd") else None
        else:
            x_pin = torch.from_numpy(work.x_host).pin_memory()
            h_pin = torch.from_numpy(work.h_host).pin_memory()
        work.e2e_step(x_pin, h_pin)
        torch.cuda.synchronize()
        barrier()
        times = []
        hb = db = 0
        for _ in range(args.steps):
            barrier()
            t0 = time.perf_counter()
            hb, db = work.e2e_step(x_pin, h_pin)
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
        t_e2e = max_over_ranks(sum(times) / len(times), world, device)
        e2e = {"value": work.total_macs / t_e2e / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": int(hb), "d2h_bytes_per_step": int(db),
               "ms_per_step": 1000 * t_e2e,
               "api": E2E_API.get(args.config, "paper_2401_01607_b200.scatter_convolve(Signal(pinned host tensor))")
               if world == 1 or args.config not in ("cfg3", "cfg5")
               else "paper_2401_01607_b200.distributed_convolve(pinned host, to_host=True)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        rate, sample, dt = cpu_sample(args.config, args.cpu_seconds, threads)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample,
               "seconds": dt}

    if rank == 0:
        w = work.w
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": work.scaling, "vs_baseline": None, "dtype": work.dtype,
            "data": "synthetic (seeded numpy PCG64 recipes of SURVEY.md 8(d); no dataset)",
            "config": {"workload": ("mstream_f32_64ch_480000x16384_b8192_1swap_multichannel_engine"
                                    if args.config == "mstream" else w.name),
                       "ne": int(w.ne), "nh": int(w.nh),
                       "channels": int(w.channels), "metric_macs": int(work.total_macs),
                       "parallelism": work.parallelism,
                       "l2": "256 MiB memset before every timed step (outside the events); "
                             "inputs also exceed L2 at N=1"},
            "pct_fp32_fma_peak": 100.0 * useful / fp32_peak,
            "kernel": getattr(work, "kernel_template", work.kernel),
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "comm": comm,
            "clocks": csum,
            "wall_s_timed_region": t_wall,
            "step_ms_rank0": step_ms,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
