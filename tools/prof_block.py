"""Per-call host cost of block-by-block streaming (engine.py:118-146 contract):
Python process_block vs the bare C call, B = 256, cfg2's 4096-tap IR, device
tensors.  Diagnostic only.

    python tools/prof_block.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2401_01607_b200 import _native as N  # noqa: E402
from paper_2401_01607_b200 import configs  # noqa: E402
from paper_2401_01607_b200.core import Signal  # noqa: E402
from paper_2401_01607_b200.engine import EngineConfig, ScatterEngine  # noqa: E402

w = configs.cfg2()
L = N.lib()
for dt in (np.float32, np.float64):
    xd = torch.from_numpy(w.x.astype(dt)).cuda()
    h = torch.from_numpy(w.irs[0].astype(dt)).cuda()
    eng = ScatterEngine(Signal(h), EngineConfig(block_size_nb=256))
    blocks = [xd[s:s + 256] for s in range(0, w.ne, 256)]
    for b in blocks[:50]:
        eng.process_block(Signal(b))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for b in blocks:
        eng.process_block(Signal(b))
    torch.cuda.synchronize()
    py = (time.perf_counter() - t0) / len(blocks) * 1e6
    out = torch.empty(256, dtype=xd.dtype, device="cuda")
    hdl = eng._handle
    t0 = time.perf_counter()
    for b in blocks:
        L.sc_engine_process_block(hdl, b.data_ptr(), 256, out.data_ptr())
    torch.cuda.synchronize()
    c = (time.perf_counter() - t0) / len(blocks) * 1e6
    t0 = time.perf_counter()
    for b in blocks:
        Signal(b)
    sig = (time.perf_counter() - t0) / len(blocks) * 1e6
    t0 = time.perf_counter()
    for b in blocks:
        torch.empty(256, dtype=xd.dtype, device="cuda")
    emp = (time.perf_counter() - t0) / len(blocks) * 1e6
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(50_000_000)
    ev0.record()
    for b in blocks:
        L.sc_engine_process_block(hdl, b.data_ptr(), 256, out.data_ptr())
    ev1.record()
    torch.cuda.synchronize()
    dev = ev0.elapsed_time(ev1) * 1e3 / len(blocks)
    print(f"{np.dtype(dt).name}: python process_block {py:.2f} us/call, bare C call {c:.2f} us, "
          f"Signal() {sig:.2f} us, torch.empty {emp:.2f} us, device time {dev:.2f} us/block")
