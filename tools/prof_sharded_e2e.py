"""End-to-end rate of the one-call multi-GPU entry (sharded.fir_sharded ->
sc_fir_sharded) on the devices of this box versus the device-only kernel
rate, cfg5 (57.6 M x 262,144, float32).  Pinned host input and output; the
chunk-pipelined range engine overlaps upload / FIR / download per shard.

    python tools/prof_sharded_e2e.py [reps]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2401_01607_b200 import configs  # noqa: E402
from paper_2401_01607_b200.core import Signal, scatter_convolve  # noqa: E402
from paper_2401_01607_b200.sharded import fir_sharded  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
w = configs.cfg5()
macs = w.metric_macs
xp = torch.from_numpy(w.x).pin_memory()
hp = torch.from_numpy(w.h).pin_memory()
ndev = torch.cuda.device_count()
# device-only reference: inputs resident, CUDA events
xd, hd = xp.cuda(), hp.cuda()
scatter_convolve(Signal(xd), Signal(hd))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
dev = []
for _ in range(reps):
    e0.record()
    scatter_convolve(Signal(xd), Signal(hd))
    e1.record()
    e1.synchronize()
    dev.append(e0.elapsed_time(e1) * 1e-3)
del xd
fir_sharded(xp, hp, devices=list(range(ndev)))       # warm: persistent buffers, streams
e2e = []
for _ in range(reps):
    t0 = time.perf_counter()
    y = fir_sharded(xp, hp, devices=list(range(ndev)))
    e2e.append(time.perf_counter() - t0)
ref = scatter_convolve(Signal(xp.cuda()), Signal(hd)).concatenated().samples.cpu()
err = float((y.double() - ref.double()).abs().max())
d, e = min(dev), min(e2e)
print(f"devices={ndev} device-only {d*1e3:.2f} ms = {macs/d/1e12:.1f} TMAC/s; fir_sharded e2e {e*1e3:.2f} ms = "
      f"{macs/e/1e12:.1f} TMAC/s (ratio {d/e:.3f}); max |diff| vs device path {err:.3g}")
