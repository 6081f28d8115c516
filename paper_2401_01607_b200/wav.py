"""WAV files straight into (and out of) device memory -- SURVEY.md 8(f) row 3.

Drop-in names of ``scatterconv.wavio`` (WavFormatError, WavSpec, read_wav,
write_wav; pkg/src/scatterconv/wavio.py) plus device-resident variants.  The
RIFF container is parsed on the host (it is a few dozen bytes of headers);
the sample payload goes to the GPU as raw bytes and is decoded, encoded
(gain, round-half-even, saturation, clip count) and reduced (the
``--normalize`` peak) by the kernels in csrc/k_wav.cu.  Encodings: pcm16,
pcm24, float32; files written here are byte-identical to the reference's.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from . import _dev
from . import _native as N
from .core import Signal

ENCODINGS = ("pcm16", "pcm24", "float32")
_ENC_CODE = {"pcm16": 0, "pcm24": 1, "float32": 2}
_BYTES = {"pcm16": 2, "pcm24": 3, "float32": 4}
_TAG_PCM, _TAG_FLOAT, _TAG_EXTENSIBLE = 1, 3, 0xFFFE


class WavFormatError(OSError):
    """Malformed or unsupported WAV structure."""


@dataclass(frozen=True)
class WavSpec:
    sample_rate: int
    channels: int
    encoding: str = "float32"

    def __post_init__(self):
        if not isinstance(self.sample_rate, (int, np.integer)) or self.sample_rate <= 0:
            raise ValueError(f"sample_rate must be a positive integer, got {self.sample_rate!r}")
        if not isinstance(self.channels, (int, np.integer)) or self.channels < 1:
            raise ValueError(f"channels must be >= 1, got {self.channels!r}")
        if self.encoding not in ENCODINGS:
            raise ValueError(f"encoding must be one of {ENCODINGS}, got {self.encoding!r}")

    @property
    def bytes_per_sample(self) -> int:
        return _BYTES[self.encoding]


# ------------------------------------------------------------------ container


def _parse(blob: bytes, path) -> tuple[WavSpec, bytes]:
    """Walk the RIFF chunks; return the spec and the data-chunk payload."""
    if len(blob) < 12:
        raise WavFormatError(f"truncated RIFF header: wanted 12 bytes, file has {len(blob)}")
    if blob[0:4] != b"RIFF" or blob[8:12] != b"WAVE":
        raise WavFormatError(f"{path}: not a RIFF/WAVE file (header {blob[0:4]!r})")
    spec = None
    off = 12
    while off + 8 <= len(blob):
        cid, size = struct.unpack_from("<4sI", blob, off)
        off += 8
        payload = blob[off:off + size]
        if len(payload) < size:
            raise WavFormatError(f"{path}: chunk {cid!r} claims {size} bytes, file has {len(payload)}")
        if cid == b"fmt ":
            spec = _parse_fmt(payload, path)
        elif cid == b"data":
            if spec is None:
                raise WavFormatError(f"{path}: 'data' chunk before 'fmt ' chunk")
            return spec, payload
        off += size + (size & 1)  # RIFF chunks are word aligned
    if spec is None:
        raise WavFormatError(f"{path}: no 'fmt ' chunk")
    raise WavFormatError(f"{path}: no 'data' chunk")


def _parse_fmt(body: bytes, path) -> WavSpec:
    if len(body) < 16:
        raise WavFormatError(f"{path}: 'fmt ' chunk too short ({len(body)} bytes)")
    tag, n_ch, rate, _, _, bits = struct.unpack_from("<HHIIHH", body, 0)
    if tag == _TAG_EXTENSIBLE:
        raise WavFormatError(f"{path}: WAVE_FORMAT_EXTENSIBLE in 'fmt ' chunk is not supported")
    known = {(_TAG_PCM, 16): "pcm16", (_TAG_PCM, 24): "pcm24", (_TAG_FLOAT, 32): "float32"}
    if (tag, bits) not in known:
        raise WavFormatError(f"{path}: unsupported 'fmt ' (format tag {tag}, {bits}-bit); "
                             f"supported encodings: {', '.join(ENCODINGS)}")
    try:
        return WavSpec(int(rate), int(n_ch), known[(tag, bits)])
    except ValueError as exc:
        raise WavFormatError(f"{path}: invalid 'fmt ' chunk: {exc}") from exc


def _header(spec: WavSpec, frames: int, payload_len: int) -> bytes:
    tag = _TAG_FLOAT if spec.encoding == "float32" else _TAG_PCM
    bits = 8 * spec.bytes_per_sample
    align = spec.bytes_per_sample * spec.channels
    fmt = struct.pack("<4sIHHIIHH", b"fmt ", 16, tag, spec.channels, spec.sample_rate,
                      spec.sample_rate * align, align, bits)
    fact = struct.pack("<4sII", b"fact", 4, frames) if tag == _TAG_FLOAT else b""
    data = struct.pack("<4sI", b"data", payload_len)
    riff = 4 + len(fmt) + len(fact) + len(data) + payload_len + (payload_len & 1)
    return struct.pack("<4sI4s", b"RIFF", riff, b"WAVE") + fmt + fact + data


# ------------------------------------------------------------------ device codecs


def read_wav_device(path, dtype=np.float64, device=None):
    """Decode a WAV file into a [channels, frames] CUDA tensor.  Returns
    (samples, spec)."""
    t = _dev.torch()
    with open(path, "rb") as fh:
        blob = fh.read()
    spec, payload = _parse(blob, path)
    frame_bytes = spec.bytes_per_sample * spec.channels
    frames = len(payload) // frame_bytes
    dev = t.device(device) if device is not None else t.device("cuda", t.cuda.current_device())
    out = t.empty((spec.channels, frames), dtype=_dev.torch_dtype(dtype), device=dev)
    if frames:
        raw = t.frombuffer(bytearray(payload[:frames * frame_bytes]), dtype=t.uint8).to(dev)
        with t.cuda.device(dev):
            N.check(N.lib().sc_wav_decode(_ENC_CODE[spec.encoding], N.ptr(raw), frames, spec.channels,
                                          N.dtype_code(dtype), N.ptr(out), N.stream_ptr()))
    return out, spec


def peak_abs(y) -> float:
    """max |y| over a CUDA tensor (device reduction)."""
    t = _dev.torch()
    bits = t.zeros(1, dtype=t.int64, device=y.device)
    with t.cuda.device(y.device):
        N.check(N.lib().sc_peak_abs(N.dtype_code(_dev.np_dtype(y)), N.ptr(y.contiguous()), y.numel(),
                                    N.ptr(bits), N.stream_ptr()))
    return float(np.array([bits.item()], dtype=np.int64).view(np.float64)[0])


def write_wav_device(path, y, spec: WavSpec, gain: float = 1.0) -> int:
    """Encode y ([channels, frames] CUDA tensor) * gain on the device and write
    the file.  Returns the number of saturated samples (0 for float32)."""
    t = _dev.torch()
    if y.ndim != 2 or y.shape[0] != spec.channels:
        raise ValueError(f"spec declares {spec.channels} channels, got {y.shape[0]} signals")
    frames = int(y.shape[1])
    yc = y.contiguous()
    nbytes = frames * spec.channels * spec.bytes_per_sample
    raw = t.empty(max(nbytes, 1), dtype=t.uint8, device=y.device)
    clipped = t.zeros(1, dtype=t.int64, device=y.device)
    if frames:
        with t.cuda.device(y.device):
            N.check(N.lib().sc_wav_encode(_ENC_CODE[spec.encoding], N.dtype_code(_dev.np_dtype(yc)), N.ptr(yc),
                                          frames, frames, spec.channels, float(gain), N.ptr(raw),
                                          N.ptr(clipped), N.stream_ptr()))
    payload = raw[:nbytes].cpu().numpy().tobytes()
    with open(path, "wb") as fh:
        fh.write(_header(spec, frames, nbytes))
        fh.write(payload)
        if nbytes & 1:
            fh.write(b"\x00")
    return int(clipped.item())


# ------------------------------------------------------------------ drop-in API


def read_wav(path) -> tuple[list[Signal], WavSpec]:
    """wavio.read_wav: one float64 host Signal per channel (decoded on the GPU)."""
    y, spec = read_wav_device(path, np.float64)
    host = y.cpu().numpy()
    return [Signal(np.ascontiguousarray(host[c]), spec.sample_rate) for c in range(spec.channels)], spec


def write_wav(path, channels: list[Signal], spec: WavSpec) -> int:
    """wavio.write_wav: encode Signals (host or CUDA) on the GPU; returns the
    clipped-sample count."""
    t = _dev.torch()
    if not channels:
        raise ValueError("channel list is empty")
    if len(channels) != spec.channels:
        raise ValueError(f"spec declares {spec.channels} channels, got {len(channels)} signals")
    n = len(channels[0])
    for c, sig in enumerate(channels):
        if len(sig) != n:
            raise ValueError(f"channel lengths differ: channel 0 has {n}, channel {c} has {len(sig)}")
        if sig.sample_rate != spec.sample_rate:
            raise ValueError(f"channel {c} sample rate {sig.sample_rate} != spec rate {spec.sample_rate}")
    y = t.stack([_dev.as_device(sig.samples, np.float64) for sig in channels])
    return write_wav_device(path, y, spec)


__all__ = ["ENCODINGS", "WavFormatError", "WavSpec", "peak_abs", "read_wav", "read_wav_device", "write_wav",
           "write_wav_device"]
