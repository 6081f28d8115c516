"""Host-side cost breakdown of the fused streaming step (cfg2): how long the
Python + C enqueue of process_stream and the flush take, versus the device
time of the whole step (CUDA events).  Diagnostic only."""
import time

import torch

import sys
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from paper_2401_01607_b200 import configs
from paper_2401_01607_b200.core import Signal
from paper_2401_01607_b200.engine import EngineConfig, ScatterEngine

w = configs.cfg2()
dev = torch.device("cuda", 0)
xd = torch.from_numpy(w.x).to(dev)
irs = [torch.from_numpy(h).to(dev) for h in w.irs]
n_blocks = -(-w.ne // 256)
swaps = [(0, irs[0])] + [(b, irs[b // 100]) for b in range(100, n_blocks, 100)]
eng = ScatterEngine(Signal(irs[0]), EngineConfig(block_size_nb=256))
for it in range(6):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    body = eng.process_stream(xd, 256, swaps)
    t1 = time.perf_counter()
    tail = eng.flush()
    t2 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"iter {it}: enqueue process_stream {1e3*(t1-t0):.3f} ms, flush {1e3*(t2-t1):.3f} ms, "
          f"device {e0.elapsed_time(e1):.3f} ms, wall {1e3*(t3-t0):.3f} ms")
