"""WAV container + CLI host logic (no GPU).  Mirrors the reference's
tests/test_wavio.py / test_cli.py error cases: pkg/src/scatterconv/wavio.py
:51-114 (parsing and messages), cli.py:87-103 (flags) and the exit-code
mapping of cli.py main()."""

from __future__ import annotations

import pathlib
import struct

import numpy as np
import pytest

from paper_2401_01607_b200 import wav
from paper_2401_01607_b200.__main__ import main, make_parser

GOLD = pathlib.Path(__file__).parent / "golden" / "wav"


def _blob(name):
    return (GOLD / name).read_bytes()


@pytest.mark.parametrize("name,rate,ch,enc", [
    ("in_pcm16_stereo.wav", 8000, 2, "pcm16"),
    ("ir_f32_stereo.wav", 8000, 2, "float32"),
    ("swap_pcm24_mono.wav", 8000, 1, "pcm24"),
    ("ir_pcm16_mono.wav", 8000, 1, "pcm16"),
])
def test_parse_golden_headers(name, rate, ch, enc):
    blob = _blob(name)
    spec, payload = wav._parse(blob, name)
    assert spec == wav.WavSpec(rate, ch, enc)
    frames = len(payload) // (spec.bytes_per_sample * ch)
    assert len(payload) == frames * spec.bytes_per_sample * ch
    # our header writer reproduces the reference writer's header bytes
    hdr = wav._header(spec, frames, len(payload))
    assert blob[:len(hdr)] == hdr
    assert len(blob) == len(hdr) + len(payload) + (len(payload) & 1)


def test_wavspec_validation():
    with pytest.raises(ValueError, match="sample_rate must be a positive integer"):
        wav.WavSpec(0, 1)
    with pytest.raises(ValueError, match="sample_rate must be a positive integer"):
        wav.WavSpec(44100.0, 1)
    with pytest.raises(ValueError, match="channels must be >= 1"):
        wav.WavSpec(8000, 0)
    with pytest.raises(ValueError, match="encoding must be one of"):
        wav.WavSpec(8000, 1, "pcm8")
    assert wav.WavSpec(8000, 2, "pcm24").bytes_per_sample == 3
    assert issubclass(wav.WavFormatError, OSError)


def _fmt(tag=1, ch=1, rate=8000, bits=16, size=16):
    body = struct.pack("<HHIIHH", tag, ch, rate, rate * ch * bits // 8, ch * bits // 8, bits)
    body = body[:size] if size < 16 else body + b"\0" * (size - 16)
    return struct.pack("<4sI", b"fmt ", len(body)) + body


def _riff(*chunks):
    inner = b"WAVE" + b"".join(chunks)
    return b"RIFF" + struct.pack("<I", len(inner)) + inner


def _data(payload):
    return struct.pack("<4sI", b"data", len(payload)) + payload


@pytest.mark.parametrize("blob,msg", [
    (b"RIFF", "truncated RIFF header"),
    (b"RIFX" + b"\0" * 8, "not a RIFF/WAVE file"),
    (_riff(_data(b"\0\0")), "'data' chunk before 'fmt ' chunk"),
    (_riff(), "no 'fmt ' chunk"),
    (_riff(_fmt()), "no 'data' chunk"),
    (_riff(_fmt(size=14), _data(b"")), "'fmt ' chunk too short"),
    (_riff(_fmt(tag=0xFFFE), _data(b"")), "WAVE_FORMAT_EXTENSIBLE"),
    (_riff(_fmt(bits=8), _data(b"")), "unsupported 'fmt '"),
    (_riff(_fmt(tag=3, bits=64), _data(b"")), "unsupported 'fmt '"),
    (_riff(_fmt(ch=0), _data(b"")), "invalid 'fmt ' chunk: channels must be >= 1"),
    (_riff(_fmt(rate=0), _data(b"")), "invalid 'fmt ' chunk: sample_rate"),
    (_riff(_fmt(), struct.pack("<4sI", b"data", 100) + b"\0" * 10), "claims 100 bytes"),
])
def test_parse_errors(blob, msg):
    with pytest.raises(wav.WavFormatError, match=msg):
        wav._parse(blob, "f.wav")


def test_parse_skips_unknown_and_odd_chunks():
    odd = struct.pack("<4sI", b"LIST", 3) + b"abc" + b"\0"  # word-aligned pad byte
    spec, payload = wav._parse(_riff(_fmt(ch=2), odd, _data(b"\1\2\3\4")), "f.wav")
    assert spec == wav.WavSpec(8000, 2, "pcm16") and payload == b"\1\2\3\4"


def test_header_float_has_fact_and_pad():
    spec = wav.WavSpec(48000, 1, "pcm24")
    hdr = wav._header(spec, 3, 9)
    assert b"fact" not in hdr
    riff = struct.unpack_from("<I", hdr, 4)[0]
    assert riff == len(hdr) - 8 + 9 + 1
    f = wav._header(wav.WavSpec(48000, 2, "float32"), 5, 40)
    assert f[36:48] == struct.pack("<4sII", b"fact", 4, 5)


# ------------------------------------------------------------------ CLI


def test_cli_parser_defaults():
    a = make_parser().parse_args(["convolve", "a.wav", "b.wav", "c.wav"])
    assert (a.nb, a.zero_skip, a.swap_ir, a.normalize, a.no_tail, a.encoding) == (
        8192, 0.0, None, None, False, "float32")
    a = make_parser().parse_args(["convolve", "a", "b", "c", "--normalize", "--swap-ir", "d@e.wav@7",
                                  "--swap-ir", "z@0"])
    assert a.normalize == 1.0 and a.swap_ir == [("d@e.wav", 7), ("z", 0)]


@pytest.mark.parametrize("argv", [
    [],
    ["convolve", "a", "b"],
    ["convolve", "a", "b", "c", "--encoding", "pcm8"],
    ["convolve", "a", "b", "c", "--swap-ir", "noat"],
    ["convolve", "a", "b", "c", "--swap-ir", "f@x"],
    ["convolve", "a", "b", "c", "--swap-ir", "f@-3"],
    ["convolve", "a", "b", "c", "--nb", "1.5"],
])
def test_cli_usage_errors_exit_2(argv, capsys):
    assert main(argv) == 2


def test_cli_help_exit_0(capsys):
    assert main(["--help"]) == 0
    assert "convolve" in capsys.readouterr().out


def test_cli_missing_file_exit_1(tmp_path, capsys):
    rc = main(["convolve", str(tmp_path / "nope.wav"), str(GOLD / "ir_pcm16_mono.wav"), str(tmp_path / "o.wav")])
    assert rc == 1
    assert capsys.readouterr().err.startswith("error: ")


def test_cli_bad_wav_exit_1(tmp_path, capsys):
    bad = tmp_path / "bad.wav"
    bad.write_bytes(b"RIFX" + b"\0" * 8)
    rc = main(["convolve", str(bad), str(GOLD / "ir_pcm16_mono.wav"), str(tmp_path / "o.wav")])
    assert rc == 1
    assert "not a RIFF/WAVE file" in capsys.readouterr().err


def test_pcm_decode_numpy_restatement():
    """Pins the decode the device kernel implements (wavio.py:118-131):
    int / 2^(bits-1), 24-bit little-endian sign extension."""
    _, payload = wav._parse(_blob("swap_pcm24_mono.wav"), "s")
    b = np.frombuffer(payload, np.uint8).reshape(-1, 3).astype(np.int32)
    v = b[:, 0] | (b[:, 1] << 8) | (b[:, 2] << 16)
    v = np.where(v & 0x800000, v - (1 << 24), v)
    assert np.abs(v).max() < (1 << 23) and v.min() < 0 < v.max()
