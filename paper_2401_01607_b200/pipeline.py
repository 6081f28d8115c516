"""WAV -> device -> WAV convolution pipeline.

``convolve_files`` is the device version of the reference CLI's
``scatterconv convolve`` (pkg/src/scatterconv/cli.py:158-219): decode both
files on the GPU, run every channel through ONE multichannel streaming
engine (instead of the CLI's sequential per-channel engines, cli.py:186-202),
hot-swap IRs at exact sample indices, append the tails, normalise with a
device peak reduction and encode on the device.  Engines are float64, so the
output file is byte-identical to the reference CLI's for the same flags.
"""

from __future__ import annotations

import sys


from . import _dev
from .engine import DEFAULT_BLOCK_SIZE, EngineConfig
from .multichannel import MultiChannelEngine
from .wav import WavSpec, peak_abs, read_wav_device, write_wav_device


def _map_channels(ir, n_channels: int, path):
    """Mono IRs broadcast to every input channel; otherwise the counts must
    match (cli.py:147-155)."""
    if ir.shape[0] == 1:
        return ir.expand(n_channels, -1).contiguous()
    if ir.shape[0] == n_channels:
        return ir
    raise ValueError(f"{path}: {ir.shape[0]} IR channels cannot map onto {n_channels} input channels "
                     "(must be 1 or equal)")


def convolve_files(input_path, ir_path, output_path, *, nb: int = DEFAULT_BLOCK_SIZE, zero_skip: float = 0.0,
                   swap_ir=(), normalize: float | None = None, no_tail: bool = False,
                   encoding: str = "float32", log=None, err=None) -> dict:
    """Convolve input_path with ir_path into output_path.  swap_ir is a list of
    (path, sample_index) hot swaps.  Returns {"frames", "channels", "clipped"}."""
    log = sys.stdout if log is None else log
    err = sys.stderr if err is None else err
    t = _dev.torch()
    x, in_spec = read_wav_device(input_path)
    h, ir_spec = read_wav_device(ir_path)
    if in_spec.sample_rate != ir_spec.sample_rate:
        raise ValueError(f"sample rates differ: {input_path} is {in_spec.sample_rate} Hz, "
                         f"{ir_path} is {ir_spec.sample_rate} Hz")
    n_in = int(x.shape[1])
    if n_in == 0:
        raise ValueError(f"{input_path}: no samples")
    if h.shape[1] == 0:
        raise ValueError(f"{ir_path}: no samples")
    C = in_spec.channels
    h = _map_channels(h, C, ir_path)
    swaps = []
    for path, at in swap_ir:
        hs, sw_spec = read_wav_device(path)
        if sw_spec.sample_rate != in_spec.sample_rate:
            raise ValueError(f"sample rates differ: {input_path} is {in_spec.sample_rate} Hz, "
                             f"{path} is {sw_spec.sample_rate} Hz")
        if at > n_in:
            raise ValueError(f"--swap-ir {path}@{at}: index past the input's {n_in} samples")
        swaps.append((at, _map_channels(hs, C, path)))
    swaps.sort(key=lambda s: s[0])

    engine = MultiChannelEngine(h, EngineConfig(block_size_nb=nb, zero_skip_threshold=zero_skip))
    body = t.empty_like(x)
    pos = 0
    # blocks restart at every swap point so the IR changes on the exact sample
    for at, hs in swaps:
        if at > pos:
            body[:, pos:at] = engine.process_stream(x[:, pos:at], nb)
            pos = at
        engine.swap_ir(hs)
    if n_in > pos:
        body[:, pos:] = engine.process_stream(x[:, pos:], nb)
    if no_tail:
        y = body
    else:
        tail, lengths = engine.flush(on_device=True)
        if len(set(lengths)) > 1:   # write_wav's own check (wavio.py:148-151)
            bad = next(c for c in range(C) if lengths[c] != lengths[0])
            raise ValueError(f"channel lengths differ: channel 0 has {n_in + lengths[0]}, channel {bad} has "
                             f"{n_in + lengths[bad]}")
        y = t.cat([body, tail[:, :lengths[0]]], dim=1)

    gain = 1.0
    if normalize is not None:
        peak = peak_abs(y)
        if peak > 0.0:
            gain = normalize / peak
        else:
            print("output is all zeros; --normalize left it unchanged", file=err)
    out_spec = WavSpec(in_spec.sample_rate, C, encoding)
    clipped = write_wav_device(output_path, y, out_spec, gain=gain)
    frames = int(y.shape[1])
    print(f"wrote {output_path}: {frames} frames x {C} ch, {encoding}", file=log)
    if clipped:
        print(f"warning: {clipped} samples clipped to full scale; consider --normalize", file=err)
    return {"frames": frames, "channels": C, "clipped": clipped}
