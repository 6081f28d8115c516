"""WAV -> device -> WAV pipeline parity.

The reference CLI (pkg/src/scatterconv/cli.py:158-219) was run by
tests/golden/make_golden.py on the committed inputs under tests/golden/wav/;
ref_wav.json holds the sha256 of every output file, the exit code and the
stderr text.  The device pipeline must write byte-identical files."""

from __future__ import annotations

import contextlib
import hashlib
import io
import json
import pathlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = pathlib.Path(__file__).parent / "golden"
REF = json.loads((GOLD / "ref_wav.json").read_text())


def _run(argv):
    from paper_2401_01607_b200.__main__ import main

    o, e = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(o), contextlib.redirect_stderr(e):
        rc = main(argv)
    return rc, o.getvalue(), e.getvalue()


def _argv(name, out):
    args = REF[name]["args"]
    rest = []
    for a in args[2:]:
        if a.endswith(".wav") or "@" in a:
            p, sep, at = a.partition("@")
            a = str(GOLD / "wav" / p) + sep + at
        rest.append(a)
    return ["convolve", str(GOLD / "wav" / args[0]), str(GOLD / "wav" / args[1]), str(out)] + rest


@pytest.mark.parametrize("name", sorted(REF))
def test_cli_byte_identical(name, tmp_path):
    out = tmp_path / "o.wav"
    rc, so, se = _run(_argv(name, out))
    ref = REF[name]
    assert rc == ref["rc"]
    assert se == ref["stderr"]
    blob = out.read_bytes()
    assert len(blob) == ref["bytes"]
    assert hashlib.sha256(blob).hexdigest() == ref["sha256"]
    assert so.startswith(f"wrote {out}: ")


def test_read_wav_matches_numpy_decode():
    from paper_2401_01607_b200 import wav

    for name in ("in_pcm16_stereo.wav", "swap_pcm24_mono.wav", "ir_f32_stereo.wav"):
        path = GOLD / "wav" / name
        sigs, spec = wav.read_wav(path)
        _, payload = wav._parse(path.read_bytes(), name)
        if spec.encoding == "pcm16":
            v = np.frombuffer(payload, "<i2").astype(np.float64) / 32768.0
        elif spec.encoding == "pcm24":
            b = np.frombuffer(payload, np.uint8).reshape(-1, 3).astype(np.int32)
            i = b[:, 0] | (b[:, 1] << 8) | (b[:, 2] << 16)
            v = np.where(i & 0x800000, i - (1 << 24), i).astype(np.float64) / float(1 << 23)
        else:
            v = np.frombuffer(payload, "<f4").astype(np.float64)
        v = v.reshape(-1, spec.channels)
        for c, s in enumerate(sigs):
            assert s.sample_rate == 8000
            np.testing.assert_array_equal(s.samples, v[:, c])


@pytest.mark.parametrize("enc", ["pcm16", "pcm24", "float32"])
def test_write_wav_encode_and_clip_count(enc, tmp_path):
    """Round-half-even, saturation and the clip count against a numpy
    restatement of wavio.write_wav (wavio.py:133-198)."""
    from paper_2401_01607_b200 import wav
    from paper_2401_01607_b200.core import Signal

    rng = np.random.default_rng(7)
    x = rng.uniform(-1.3, 1.3, (2, 1001))
    bits = {"pcm16": 16, "pcm24": 24}.get(enc)
    if bits:   # exact half-steps to exercise half-to-even
        s = float(1 << (bits - 1))
        x[0, :8] = (np.arange(8) - 3.5) / s
    clipped = wav.write_wav(tmp_path / "w.wav", [Signal(x[0], 8000), Signal(x[1], 8000)], wav.WavSpec(8000, 2, enc))
    spec, payload = wav._parse((tmp_path / "w.wav").read_bytes(), "w")
    inter = x.T.reshape(-1)
    if enc == "float32":
        assert clipped == 0 and payload == inter.astype("<f4").tobytes()
        return
    q = np.round(inter * s)
    ref_clip = int(np.count_nonzero((q < -s) | (q > s - 1)))
    q = np.clip(q, -s, s - 1).astype(np.int32)
    if bits == 16:
        want = q.astype("<i2").tobytes()
    else:
        u = q.astype(np.uint32)
        want = np.stack([u & 0xFF, (u >> 8) & 0xFF, (u >> 16) & 0xFF], 1).astype(np.uint8).tobytes()
    assert clipped == ref_clip > 0
    assert payload == want


def test_peak_abs_and_gain(tmp_path):
    import torch

    from paper_2401_01607_b200 import wav

    y = torch.randn(3, 4097, dtype=torch.float64, device="cuda")
    y[1, 77] = -9.5
    assert wav.peak_abs(y) == 9.5
    assert wav.peak_abs(y.float()) == 9.5
    assert wav.peak_abs(torch.zeros(2, 5, dtype=torch.float64, device="cuda")) == 0.0
    n = wav.write_wav_device(tmp_path / "g.wav", y, wav.WavSpec(8000, 3, "float32"), gain=0.5)
    _, payload = wav._parse((tmp_path / "g.wav").read_bytes(), "g")
    want = (y.cpu().numpy() * 0.5).T.reshape(-1).astype("<f4").tobytes()
    assert n == 0 and payload == want


def test_cli_domain_errors(tmp_path):
    from paper_2401_01607_b200 import wav
    from paper_2401_01607_b200.core import Signal

    w = GOLD / "wav"
    other = tmp_path / "r16k.wav"
    wav.write_wav(other, [Signal(np.ones(4), 16000)], wav.WavSpec(16000, 1, "pcm16"))
    rc, _, se = _run(["convolve", str(w / "in_pcm16_stereo.wav"), str(other), str(tmp_path / "o.wav")])
    assert rc == 2 and se.startswith("error: sample rates differ")
    tri = tmp_path / "tri.wav"
    wav.write_wav(tri, [Signal(np.ones(4), 8000)] * 3, wav.WavSpec(8000, 3, "pcm16"))
    rc, _, se = _run(["convolve", str(w / "in_pcm16_stereo.wav"), str(tri), str(tmp_path / "o.wav")])
    assert rc == 2 and "3 IR channels cannot map onto 2 input channels" in se
    rc, _, se = _run(["convolve", str(w / "in_pcm16_stereo.wav"), str(w / "ir_pcm16_mono.wav"),
                      str(tmp_path / "o.wav"), "--swap-ir", f"{w / 'ir_pcm16_mono.wav'}@12001"])
    assert rc == 2 and "index past the input's 12000 samples" in se
    empty = tmp_path / "empty.wav"
    wav.write_wav(empty, [Signal(np.zeros(0), 8000)], wav.WavSpec(8000, 1, "pcm16"))
    rc, _, se = _run(["convolve", str(empty), str(w / "ir_pcm16_mono.wav"), str(tmp_path / "o.wav")])
    assert rc == 2 and "no samples" in se


def test_cli_delta_ir_reproduces_input(tmp_path):
    """Convolving with a unit impulse writes the input back (float32 out)."""
    from paper_2401_01607_b200 import wav
    from paper_2401_01607_b200.core import Signal

    d = tmp_path / "d.wav"
    wav.write_wav(d, [Signal(np.r_[1.0, np.zeros(10)], 8000)], wav.WavSpec(8000, 1, "float32"))
    src = GOLD / "wav" / "in_pcm16_stereo.wav"
    rc, _, _ = _run(["convolve", str(src), str(d), str(tmp_path / "o.wav"), "--no-tail", "--encoding", "pcm16"])
    assert rc == 0
    assert (tmp_path / "o.wav").read_bytes() == src.read_bytes()
