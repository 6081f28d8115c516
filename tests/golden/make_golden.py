"""Generate golden fixtures by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``scatterconv`` from /root/reference/pkg/src (numba cache
redirected to /tmp so nothing is written into the read-only reference tree),
runs the reference's own entry points on seeded inputs and writes:

  ref_small.npz      ragged random pairs: scatter_convolve, commuted_convolve,
                     direct_form, skip-zeros outputs (float64, bit-exact)
  ref_engine.json    scripted ScatterEngine sessions (blocks, samples,
                     swaps, deferred swaps, flush, state) with every output
                     recorded as float.hex -- bit-exact goldens
  ref_configs.npz    per-config reference pins: sha256 of the reference's
                     output on cfg1/cfg2 in full and cfg3/4/5 prefixes, plus
                     sampled values and exact direct_form (fsum) samples
  ref_sweeps.json    bench.py sweep reports (digests, row shapes)
  wav/, ref_wav.json WAV inputs + sha256 of the reference CLI `convolve`
                     outputs for four flag sets
  ref_fixed.*        quantize.py fixed_point_convolve outputs, simulate
                     reports and `quant` CLI stdout
  ref_cli_bench.json the `bench` CLI's timing-independent lines

`python tests/golden/make_golden.py NAME...` regenerates only make_NAME().
The fixtures are committed; the GPU box never needs /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import os
import pathlib
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
REPO = HERE.parent.parent
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(REPO))

from scatterconv import core as rcore  # noqa: E402  (the reference)
from scatterconv.core import Signal  # noqa: E402
from scatterconv.engine import EngineConfig, ScatterEngine  # noqa: E402

from paper_2401_01607_b200 import configs  # noqa: E402  (seeded generators only)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def full(out) -> np.ndarray:
    return out.concatenated().samples


# ----------------------------------------------------------------- small pairs


def make_small():
    rng = np.random.default_rng(20240101)
    es, hs, kinds, thr = [], [], [], []
    for i in range(400):
        ne, nh = int(rng.integers(1, 65)), int(rng.integers(1, 65))
        e = rng.uniform(-1, 1, ne)
        h = rng.uniform(-1, 1, nh)
        kind = i % 4
        if kind == 1:  # exact zeros sprinkled (skip-zeros cases)
            e[rng.uniform(0, 1, ne) < 0.3] = 0.0
        if kind == 2:  # tiny values around a threshold
            e[rng.uniform(0, 1, ne) < 0.3] *= 1e-3
        es.append(e)
        hs.append(h)
        kinds.append(kind)
        thr.append(0.0 if kind != 2 else 5e-4)
    # edge cases: single tap, single sample, -0.0, ints
    es += [np.array([1.0, 0.0, 0.0, 0.0]), np.array([-0.0, 1.0, -0.0]), np.array([1.0]),
           np.array([2.0, 3.0])]
    hs += [np.array([9.0]), np.array([0.5, -0.25, 0.125]), np.array([5.0, 6.0, 7.0]),
           np.array([1.0])]
    kinds += [0, 0, 0, 0]
    thr += [0.0, 0.0, 0.0, 0.0]

    sc, cm, df, sk = [], [], [], []
    for e, h, t in zip(es, hs, thr):
        E, H = Signal(e), Signal(h)
        sc.append(full(rcore.scatter_convolve(E, H)))
        cm.append(full(rcore.commuted_convolve(E, H)))
        df.append(rcore.direct_form(E, H).samples)
        sk.append(full(rcore.scatter_convolve_skip_zeros(E, H, t)))

    def pack(arrs):
        off = np.cumsum([0] + [len(a) for a in arrs]).astype(np.int64)
        return np.concatenate(arrs), off

    data = {}
    for name, arrs in (("e", es), ("h", hs), ("scatter", sc), ("commuted", cm), ("direct", df),
                       ("skip", sk)):
        v, off = pack(arrs)
        data[name] = v
        data[name + "_off"] = off
    data["threshold"] = np.asarray(thr)
    data["kind"] = np.asarray(kinds)
    np.savez_compressed(HERE / "ref_small.npz", **data)
    print("ref_small.npz:", len(es), "pairs")


# -------------------------------------------------------------- engine sessions


def hexlist(a) -> list:
    return [float(v).hex() for v in np.asarray(a, dtype=np.float64).ravel()]


def run_session(h, nb, threshold, ops):
    """Apply ops to a reference engine; return recorded outputs."""
    eng = ScatterEngine(Signal(h), EngineConfig(block_size_nb=nb, zero_skip_threshold=threshold))
    rec = []
    for op in ops:
        kind = op[0]
        if kind == "block":
            rec.append(hexlist(eng.process_block(Signal(np.asarray(op[1]))).samples))
        elif kind == "sample":
            rec.append(hexlist([eng.process_sample(op[1])]))
        elif kind == "swap":
            eng.swap_ir(Signal(np.asarray(op[1])))
            rec.append([])
        elif kind == "defer":
            eng.swap_ir_at_next_block(Signal(np.asarray(op[1])))
            rec.append([])
        elif kind == "flush":
            rec.append(hexlist(eng.flush().samples))
        elif kind == "state":
            rec.append({"read_index": int(eng.read_index), "ring": hexlist(eng.ring),
                        "consumed": int(eng.samples_consumed), "live": int(eng._live),
                        "sched": hexlist(eng._schedule_order())})
        else:
            raise ValueError(kind)
    return rec


def make_engine():
    rng = np.random.default_rng(20240102)
    sessions = []

    def add(h, nb, thr, ops, tag):
        ops_json = []
        for op in ops:
            if op[0] in ("block", "swap", "defer"):
                ops_json.append([op[0], hexlist(op[1])])
            elif op[0] == "sample":
                ops_json.append([op[0], float(op[1]).hex()])
            else:
                ops_json.append([op[0]])
        sessions.append({"tag": tag, "h": hexlist(h), "nb": nb, "threshold": float(thr).hex(),
                         "ops": ops_json, "expect": run_session(h, nb, thr, ops)})

    # hand scenarios (test_engine.py:67-71, :216-223, :283-294)
    add([3.0, 4.0], 8192, 0.0, [("sample", 1.0), ("sample", 2.0), ("flush",)], "hand_3_10_8")
    add([1.0, 1.0], 8192, 0.0, [("sample", 1.0), ("sample", 0.0), ("swap", [5.0, 5.0]),
                                ("sample", 0.0), ("sample", 0.0), ("sample", 1.0), ("flush",)],
        "hand_swap")
    add([1.0, 2.0, 3.0, 4.0, 5.0, 6.0], 8192, 0.0,
        [("sample", 1.0), ("swap", [9.0, 9.0]), ("state",), ("sample", 0.0), ("state",),
         ("flush",), ("state",)], "shrink_drain")
    add([3.0, 4.0, 5.0], 8192, 0.0, [("sample", 0.0), ("state",), ("sample", -0.0), ("state",)],
        "zero_untouched")
    add([1.0, 1.0], 8192, 0.0, [("block", [1.0, np.nan, 2.0]), ("flush",)], "nan_skipped")
    add([1.0, 0.5], 8192, 0.0, [("block", [np.inf, 1.0]), ("flush",)], "inf_scatters")
    add([0.5, 0.25], 4, 0.0, [("defer", [2.0, 2.0, 2.0]), ("block", [1.0, 1.0]), ("state",),
                              ("flush",), ("state",)], "deferred")

    # random sessions: blocks with random cuts, swaps (grow/shrink/same), deferred, samples
    for s in range(120):
        nh = int(rng.integers(1, 40))
        nb = int(rng.integers(1, 70))
        thr = 0.0 if s % 3 else float(rng.uniform(0, 0.3))
        h = rng.uniform(-1, 1, nh)
        ops = []
        for _ in range(int(rng.integers(1, 9))):
            r = rng.uniform()
            if r < 0.55:
                n = int(rng.integers(0, nb + 1))
                x = rng.uniform(-1, 1, n)
                x[rng.uniform(0, 1, n) < 0.2] = 0.0
                ops.append(("block", x))
            elif r < 0.7:
                ops.append(("sample", float(rng.uniform(-1, 1))))
            elif r < 0.82:
                ops.append(("swap", rng.uniform(-1, 1, int(rng.integers(1, 50)))))
            elif r < 0.9:
                ops.append(("defer", rng.uniform(-1, 1, int(rng.integers(1, 50)))))
            elif r < 0.95:
                ops.append(("state",))
            else:
                ops.append(("flush",))
        ops += [("state",), ("flush",), ("state",)]
        add(h, nb, thr, ops, f"random_{s}")
    with open(HERE / "ref_engine.json", "w", encoding="utf-8") as fh:
        json.dump(sessions, fh, separators=(",", ":"))
    print("ref_engine.json:", len(sessions), "sessions")


# ------------------------------------------------------------------- configs


def stream_reference(x64, h64, nb):
    eng = ScatterEngine(Signal(h64), EngineConfig(block_size_nb=nb))
    outs = [eng.process_block(Signal(x64[i:i + nb])).samples for i in range(0, len(x64), nb)]
    outs.append(eng.flush().samples)
    return np.concatenate(outs)


def make_configs():
    out = {}
    sample_rng = np.random.default_rng(99)

    # cfg1 (float64, full): scatter_convolve, engine and direct_form (fsum)
    w = configs.cfg1()
    E, H = Signal(w.x), Signal(w.h)
    y_sc = full(rcore.scatter_convolve(E, H))
    y_eng = stream_reference(w.x, w.h, 8192)
    assert np.array_equal(y_sc, y_eng)
    idx = np.sort(sample_rng.choice(w.nout, 2048, replace=False))
    idx[:3] = [0, 1, w.nout - 1]
    idx = np.unique(idx)
    y_df = np.array([np.float64(__import__("math").fsum(
        w.x[m] * w.h[n - m] for m in range(max(0, n - w.nh + 1), min(n, w.ne - 1) + 1)))
        for n in idx])
    out["cfg1_sha_scatter"] = sha(y_sc)
    out["cfg1_idx"] = idx
    out["cfg1_scatter_at_idx"] = y_sc[idx]
    out["cfg1_direct_at_idx"] = y_df

    # cfg2 (float32 inputs -> float64 reference): engine nb=256, swap every 100 blocks
    w = configs.cfg2()
    x64 = w.x.astype(np.float64)
    eng = ScatterEngine(Signal(w.irs[0].astype(np.float64)), EngineConfig(block_size_nb=256))
    outs = []
    j = 0
    for b, start in enumerate(range(0, len(x64), 256)):
        if b > 0 and b % 100 == 0:
            j += 1
            eng.swap_ir(Signal(w.irs[j].astype(np.float64)))
        outs.append(eng.process_block(Signal(x64[start:start + 256])).samples)
    body = np.concatenate(outs)
    tail = eng.flush().samples
    out["cfg2_sha_body"] = sha(body)
    out["cfg2_sha_tail"] = sha(tail)
    idx = np.unique(sample_rng.choice(len(body), 4096, replace=False))
    out["cfg2_idx"] = idx
    out["cfg2_body_at_idx"] = body[idx]
    out["cfg2_tail"] = tail.astype(np.float64)

    # cfg3 / cfg4 / cfg5 prefixes through the reference engine (float64 on f32 values)
    for name, x, h, n_pre in (
        ("cfg3", configs.cfg3(ne=24000).x, configs.cfg3_h(), 24000),
        ("cfg5", configs.cfg5_x(ne=6000), configs.cfg5_h(), 6000),
    ):
        x64 = x[:n_pre].astype(np.float64)
        eng = ScatterEngine(Signal(h.astype(np.float64)), EngineConfig(block_size_nb=8192))
        body = np.concatenate([eng.process_block(Signal(x64[i:i + 8192])).samples
                               for i in range(0, n_pre, 8192)])
        out[f"{name}_prefix_len"] = n_pre
        out[f"{name}_sha_prefix_body"] = sha(body)
        idx = np.unique(sample_rng.choice(n_pre, 512, replace=False))
        out[f"{name}_idx"] = idx
        out[f"{name}_body_at_idx"] = body[idx]
    w = configs.cfg4(channels=2, ne=30000)
    for c in range(2):
        y = stream_reference(w.x[c].astype(np.float64), w.h[c].astype(np.float64), 8192)
        out[f"cfg4_ch{c}_sha_full_ne30000"] = sha(y)
    np.savez_compressed(HERE / "ref_configs.npz", **out)
    print("ref_configs.npz:", sorted(out))


def make_sweeps():
    """Digests of the reference's own sweeps (bench.py:182-257): the outputs
    are deterministic, so a device harness with float64 engines must match."""
    from scatterconv.bench import SweepSpec, gen_white_noise, run_ir_sweep, run_nb_sweep

    x = gen_white_noise(3000, 8000, seed=(77, 1))
    ir = run_ir_sweep(SweepSpec([20, 45, 130], x, repetitions=1, rng_seed=5))
    nbs = run_nb_sweep(SweepSpec([64], x, nb_values=[17, 256, 4096], repetitions=1, rng_seed=6))
    out = {"ir_sweep": {"ir_lengths": [20, 45, 130], "n": 3000, "rate": 8000, "seed": [77, 1],
                        "rng_seed": 5, "digest": ir.output_digest},
           "nb_sweep": {"ir_lengths": [64], "nb_values": [17, 256, 4096], "rng_seed": 6,
                        "digest": nbs.output_digest}}
    with open(HERE / "ref_sweeps.json", "w", encoding="utf-8") as fh:
        json.dump(out, fh, indent=1)
    print("ref_sweeps.json:", out)


def make_wav():
    """Reference CLI runs (cli.py `convolve`) on small synthetic WAV files: the
    inputs are committed under tests/golden/wav/ and the sha256 of every
    output file (plus exit code) is recorded."""
    import contextlib
    import io

    from scatterconv.cli import main
    from scatterconv.wavio import WavSpec, write_wav

    d = HERE / "wav"
    d.mkdir(exist_ok=True)
    rng = np.random.default_rng(2026)
    rate = 8000
    x = rng.uniform(-0.5, 0.5, (2, 12000))
    x[0, 3000:3400] = 0.0
    write_wav(d / "in_pcm16_stereo.wav", [Signal(x[0], rate), Signal(x[1], rate)], WavSpec(rate, 2, "pcm16"))
    h = rng.standard_normal((2, 1500)) * np.exp(-np.arange(1500) / 300.0) * 0.1
    write_wav(d / "ir_f32_stereo.wav", [Signal(h[0], rate), Signal(h[1], rate)], WavSpec(rate, 2, "float32"))
    hs = rng.standard_normal(900) * np.exp(-np.arange(900) / 200.0) * 0.1
    write_wav(d / "swap_pcm24_mono.wav", [Signal(hs, rate)], WavSpec(rate, 1, "pcm24"))
    hm = rng.standard_normal(700) * 0.05
    write_wav(d / "ir_pcm16_mono.wav", [Signal(hm, rate)], WavSpec(rate, 1, "pcm16"))
    runs = {
        "default": ["in_pcm16_stereo.wav", "ir_f32_stereo.wav"],
        "swap_norm_pcm24": ["in_pcm16_stereo.wav", "ir_f32_stereo.wav", "--nb", "256", "--swap-ir",
                            "swap_pcm24_mono.wav@5000", "--normalize", "0.9", "--encoding", "pcm24"],
        "skip_notail_pcm16": ["in_pcm16_stereo.wav", "ir_pcm16_mono.wav", "--zero-skip", "0.01", "--no-tail",
                              "--encoding", "pcm16", "--nb", "1000"],
        "two_swaps_loud_pcm16": ["in_pcm16_stereo.wav", "ir_pcm16_mono.wav", "--swap-ir",
                                 "ir_f32_stereo.wav@100", "--swap-ir", "swap_pcm24_mono.wav@11999",
                                 "--encoding", "pcm16", "--nb", "4096"],
    }
    out = {}
    for name, args in runs.items():
        argv = ["convolve", str(d / args[0]), str(d / args[1]), f"/tmp/golden_{name}.wav"]
        rest = list(args[2:])
        for i, a in enumerate(rest):
            if a.endswith(".wav") or "@" in a:
                p, sep, at = a.partition("@")
                rest[i] = str(d / p) + sep + at
        buf_o, buf_e = io.StringIO(), io.StringIO()
        with contextlib.redirect_stdout(buf_o), contextlib.redirect_stderr(buf_e):
            rc = main(argv + rest)
        blob = open(f"/tmp/golden_{name}.wav", "rb").read()
        out[name] = {"args": args, "rc": rc, "sha256": hashlib.sha256(blob).hexdigest(), "bytes": len(blob),
                     "stderr": buf_e.getvalue()}
    with open(HERE / "ref_wav.json", "w", encoding="utf-8") as fh:
        json.dump(out, fh, indent=1)
    print("ref_wav.json:", {k: (v["rc"], v["bytes"]) for k, v in out.items()})


FIXED_BITS = (2, 3, 8, 12, 16, 24, 32)


def _fixed_cases():
    """(name, e, h) inputs for the fixed-point fixtures: random, grid edges
    (-1, values that round up to +1 and saturate, exact half steps) and the
    single-sample shapes the mac scheme special-cases."""
    rng = np.random.default_rng(1607)
    cases = [("rand", rng.uniform(-1, 1, 37), rng.uniform(-1, 1, 11)),
             ("ne1", rng.uniform(-1, 1, 1), rng.uniform(-1, 1, 6)),
             ("nh1", rng.uniform(-1, 1, 9), rng.uniform(-1, 1, 1)),
             ("nh2", rng.uniform(-1, 1, 13), rng.uniform(-1, 1, 2)),
             ("long_ir", rng.uniform(-1, 1, 20), rng.uniform(-1, 1, 64))]
    edge = np.array([-1.0, 1.0 - 2.0 ** -40, 0.5, -0.5, 0.0, -0.0, 0.25 + 2.0 ** -10, 0.375, -0.625, 0.999])
    cases.append(("edges", edge, edge[::-1].copy()))
    cases.append(("loud", np.full(24, 1.0 - 2.0 ** -45), np.full(24, -1.0)))
    return cases


def make_fixed():
    """Reference quantize.py runs: fixed_point_convolve outputs for every case x
    word length x scheme, simulate reports, and the `quant` CLI's stdout."""
    import contextlib
    import io

    import importlib

    q = importlib.import_module("scatterconv.quantize")  # the package re-exports a function of that name
    from scatterconv.cli import main

    arrays, meta = {}, {"reports": {}, "cli": {}}
    for name, e, h in _fixed_cases():
        arrays[f"{name}/e"] = e
        arrays[f"{name}/h"] = h
        for bits in FIXED_BITS:
            fmt = q.FixedPointFormat(bits)
            for scheme in q.SCHEMES:
                y = q.fixed_point_convolve(Signal(e, 48000), Signal(h, 48000), fmt, scheme).samples
                arrays[f"{name}/{bits}/{scheme}"] = y
                if name in ("rand", "long_ir"):
                    r = q.simulate_fixed_point_conv(Signal(e, 48000), Signal(h, 48000), fmt, scheme)
                    meta["reports"][f"{name}/{bits}/{scheme}"] = [r.operations_count, r.bits_removed_per_op,
                                                                  r.rms_error, r.max_error]
    runs = {"b16_ir32_sim": ["quant", "--bits", "16", "--ir-len", "32", "--simulate", "--seed", "3"],
            "b8_ir5": ["quant", "--bits", "8", "--ir-len", "5"],
            "b24_ir100_sim": ["quant", "--bits", "24", "--ir-len", "100", "--simulate", "--len", "64"],
            "b2_ir1_sim": ["quant", "--bits", "2", "--ir-len", "1", "--simulate", "--len", "5"],
            "b32_ir7_sim": ["quant", "--bits", "32", "--ir-len", "7", "--simulate", "--seed", "11", "--len", "300"],
            "bad_bits": ["quant", "--bits", "1", "--ir-len", "4"],
            "bad_len": ["quant", "--bits", "8", "--ir-len", "4", "--simulate", "--len", "0"],
            "bad_ir": ["quant", "--bits", "8", "--ir-len", "0"]}
    for name, argv in runs.items():
        o, e = io.StringIO(), io.StringIO()
        with contextlib.redirect_stdout(o), contextlib.redirect_stderr(e):
            rc = main(argv)
        meta["cli"][name] = {"argv": argv, "rc": rc, "stdout": o.getvalue(), "stderr": e.getvalue()}
    np.savez_compressed(HERE / "ref_fixed.npz", **arrays)
    with open(HERE / "ref_fixed.json", "w", encoding="utf-8") as fh:
        json.dump(meta, fh, indent=1)
    print("ref_fixed:", len(arrays), "arrays;", {k: v["rc"] for k, v in meta["cli"].items()})


def make_cli_bench():
    """The reference `bench` CLI: timing lines vary, the output digests and
    row counts do not."""
    import contextlib
    import io

    from scatterconv.cli import main

    runs = {"ir_nb": ["bench", "--ir-sweep", "1:3:1", "--input", "noise:0.05", "--reps", "1", "--nb-sweep",
                      "64,100", "--ir-ms", "2", "--csv", "{tmp}/x.csv", "--plot-data", "{tmp}/p.dat"],
            "ir_only_seed": ["bench", "--ir-sweep", "0.5:0.5:1", "--input", "noise:0.02", "--seed", "5",
                             "--rate", "8000", "--nb", "33", "--reps", "2"],
            "nothing": ["bench", "--input", "noise:0.01"],
            "bad_input": ["bench", "--ir-sweep", "1:2:1", "--input", "noise:abc"],
            "plot_needs_ir": ["bench", "--nb-sweep", "8", "--ir-ms", "1", "--input", "noise:0.01",
                              "--plot-data", "{tmp}/p.dat"]}
    out = {}
    for name, argv in runs.items():
        o, e = io.StringIO(), io.StringIO()
        with contextlib.redirect_stdout(o), contextlib.redirect_stderr(e):
            rc = main([a.replace("{tmp}", "/tmp") for a in argv])
        stable = [ln for ln in o.getvalue().splitlines()
                  if "sha256" in ln or ln.startswith("wrote") or ln.startswith("nb sweep at")]
        out[name] = {"argv": argv, "rc": rc, "stable": [ln.split(": wall-time")[0] for ln in stable],
                     "stderr": e.getvalue()}
    with open(HERE / "ref_cli_bench.json", "w", encoding="utf-8") as fh:
        json.dump(out, fh, indent=1)
    print("ref_cli_bench.json:", {k: v["rc"] for k, v in out.items()})


if __name__ == "__main__":
    if len(sys.argv) > 1:
        for name in sys.argv[1:]:
            globals()[f"make_{name}"]()
    else:
        make_small()
        make_engine()
        make_configs()
        make_sweeps()
        make_wav()
        make_fixed()
        make_cli_bench()
