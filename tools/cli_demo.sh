# End-to-end CLI demo: 60 s of 48 kHz stereo pcm24 convolved with a 2 s float32 IR
# (decode, multichannel float64 engine, normalize, encode -- all on the device).
cd /root/repo
python - <<'PY'
import numpy as np
from paper_2401_01607_b200.wav import WavSpec, write_wav
from paper_2401_01607_b200.core import Signal
rng = np.random.default_rng(0)
rate = 48000
x = [Signal(rng.uniform(-0.5, 0.5, 60 * rate), rate) for _ in range(2)]
write_wav("/tmp/in.wav", x, WavSpec(rate, 2, "pcm24"))
h = rng.standard_normal(2 * rate) * np.exp(-np.arange(2 * rate) / 20000) * 0.05
write_wav("/tmp/ir.wav", [Signal(h, rate)], WavSpec(rate, 1, "float32"))
PY
time python -m paper_2401_01607_b200 convolve /tmp/in.wav /tmp/ir.wav /tmp/out.wav --normalize 0.9 --encoding pcm24
ls -la /tmp/out.wav
