#!/usr/bin/env python
"""Small invocations of every kernel path, for compute-sanitizer runs:

    compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
    compute-sanitizer --tool racecheck python tools/sanitize_smoke.py

Sizes are tiny so the instrumented run finishes in seconds; every result is
checked against the CPU oracle so a silent corruption also fails the run.
"""

import pathlib
import sys

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))

from oracle import oracle as O  # noqa: E402
from paper_2401_01607_b200 import (  # noqa: E402
    EngineConfig,
    ScatterEngine,
    Signal,
    configs,
    convolve_batched,
    scatter_convolve,
    scatter_convolve_skip_zeros,
)
from paper_2401_01607_b200 import _kernels  # noqa: E402
from paper_2401_01607_b200.sharded import convolve_shard, shard_plan  # noqa: E402


def check(name, y, ref, x, h, dtype="f32"):
    tol = configs.tolerance(x, h, dtype)
    err = float(np.max(np.abs(np.asarray(y, np.float64) - ref)))
    assert err <= tol, f"{name}: {err} > {tol}"
    print(f"ok {name}: err/tol {err / tol:.3g}", flush=True)


def main():
    import torch

    rng = np.random.default_rng(1)
    x = rng.uniform(-1, 1, 9000).astype(np.float32)
    for nh in (7, 300, 2100):
        h = rng.standard_normal(nh).astype(np.float32)
        ref = O.scatter_full(x, h)
        for mode in (None, "ffma", "tc", "ordered"):
            if mode == "tc" and nh < 256:
                continue
            y = scatter_convolve(Signal(x), Signal(h), mode=mode).concatenated().samples
            check(f"fir nh={nh} mode={mode}", y, ref, x, h)
    # split-K FFMA (few tiles, long filter) and TC shift-range splits
    h = rng.standard_normal(20_000).astype(np.float32)
    for mode in ("ffma", "tc"):
        y = scatter_convolve(Signal(x), Signal(h), mode=mode).concatenated().samples
        check(f"split mode={mode}", y, O.scatter_full(x, h), x, h)
    # float64 ordered + skip zeros
    x64 = rng.uniform(-1, 1, 3000)
    x64[::7] = 0.0
    h64 = rng.standard_normal(333)
    y = scatter_convolve_skip_zeros(Signal(x64), Signal(h64), 0.1).concatenated().samples
    assert np.array_equal(y, O.scatter_full(x64, h64, O.SKIP_LE, 0.1))
    print("ok f64 skip", flush=True)
    # batched + shards
    X = rng.uniform(-1, 1, (3, 5000)).astype(np.float32)
    H = rng.standard_normal((3, 700)).astype(np.float32)
    Y = convolve_batched(X, H)
    for c in range(3):
        check(f"batched ch{c}", Y[c], O.scatter_full(X[c], H[c]), X[c], H[c])
    hd = torch.from_numpy(H[0]).cuda()
    parts = [convolve_shard(torch.from_numpy(X[0][s.x_begin:s.x_end]).cuda(), s, hd).cpu().numpy()
             for s in shard_plan(5000, 700, 3)]
    check("shards", np.concatenate(parts), O.scatter_full(X[0], H[0]), X[0], H[0])
    # engine: blocks, swap, deferred swap, fused stream, flush
    for dt in (np.float64, np.float32):
        h1 = rng.standard_normal(50).astype(dt)
        h2 = rng.standard_normal(120).astype(dt)
        e = ScatterEngine(Signal(h1), EngineConfig(block_size_nb=64))
        ref = O.OracleEngine(h1, 64)
        xs = rng.uniform(-1, 1, 640).astype(dt)
        got, want = [], []
        for b in range(5):
            got.append(e.process_block(Signal(xs[64 * b:64 * b + 64])).samples)
            want.append(ref.process_block(xs[64 * b:64 * b + 64]))
        e.swap_ir(Signal(h2))
        ref.swap_ir(h2)
        body = e.process_stream(torch.from_numpy(xs[320:]).cuda(), 64, [(2, h1)]).cpu().numpy()
        for b in range(5):
            if b == 2:
                ref.swap_ir(h1)
            want.append(ref.process_block(xs[320 + 64 * b:320 + 64 * b + 64]))
        got.append(body)
        got.append(e.flush().samples)
        want.append(ref.flush())
        g, w = np.concatenate(got), np.concatenate(want)
        if dt == np.float64:
            assert np.array_equal(g, w)
        else:
            assert np.max(np.abs(g - w)) < 1e-4
        print(f"ok engine {dt.__name__}", flush=True)
    ring = rng.uniform(-1, 1, 40)
    out = np.empty(70)
    r2, o2 = ring.copy(), np.empty(70)
    blk = rng.uniform(-1, 1, 70)
    assert _kernels.scatter_block(ring, h64[:30], blk, out, 3, 5, 0.0) == \
        O.scatter_block(r2, h64[:30], blk, o2, 3, 5, 0.0)
    assert np.array_equal(ring, r2) and np.array_equal(out, o2)
    print("ok scatter_block", flush=True)
    # tensor cores with the 2-shift drain (<= 2 shifts) and the short kernels
    for nh in (3, 24, 100):
        h = rng.standard_normal(nh).astype(np.float32)
        for mode in (None, "tc"):
            y = scatter_convolve(Signal(x), Signal(h), mode=mode).concatenated().samples
            check(f"short nh={nh} mode={mode}", y, O.scatter_full(x, h), x, h)
    # FAST fused stream through the batched tensor-core path (thresholds lowered)
    from paper_2401_01607_b200.engine import ScatterEngine as _SE

    hf = rng.standard_normal(300).astype(np.float32)
    xf = rng.uniform(-1, 1, 256 * 40).astype(np.float32)
    ef = _SE(Signal(torch.from_numpy(hf).cuda()), EngineConfig(block_size_nb=256), mode="fast")
    bf = ef.process_stream(torch.from_numpy(xf).cuda(), 256, [(10 * j, torch.from_numpy(hf).cuda()) for j in (1, 2, 3)])
    full = np.concatenate([bf.cpu().numpy(), ef.flush().samples.cpu().numpy()])
    check("fast stream (ordered below threshold)", full, O.scatter_full(xf, hf), xf, hf)
    # fixed point, WAV codecs, native sharded call
    from paper_2401_01607_b200 import fixed_point as fx
    from paper_2401_01607_b200.sharded import fir_sharded

    e16, k16 = rng.uniform(-1, 1, 200), rng.uniform(-1, 1, 30)
    for scheme in ("ideal", "mac"):
        yq = fx.fixed_point_convolve(Signal(e16), Signal(k16), fx.FixedPointFormat(16), scheme).samples
        assert np.array_equal(yq, O.fixed_convolve(e16, k16, 16, scheme))
    print("ok fixed point", flush=True)
    assert np.array_equal(fir_sharded(x64, h64, devices=[0, 0, 0]), O.scatter_full(x64, h64))
    print("ok sharded", flush=True)
    import tempfile

    from paper_2401_01607_b200 import wav

    with tempfile.TemporaryDirectory() as tmp:
        for enc in wav.ENCODINGS:
            path = pathlib.Path(tmp) / f"{enc}.wav"
            wav.write_wav(path, [Signal(np.clip(x64[:500], -0.9, 0.9), 8000)], wav.WavSpec(8000, 1, enc))
            back, spec = wav.read_wav(path)
            assert spec.encoding == enc and len(back[0]) == 500
    print("ok wav", flush=True)
    torch.cuda.synchronize()
    print("SANITIZE SMOKE PASSED", flush=True)


if __name__ == "__main__":
    main()
