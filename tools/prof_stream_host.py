"""Host-side cost breakdown of a fused streaming step: how long the Python +
C enqueue of process_stream and the flush take, versus the device time of
the whole step (CUDA events).  Diagnostic only.

    python tools/prof_stream_host.py [cfg2|mstream] [host] [cprofile]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2401_01607_b200 import configs  # noqa: E402
from paper_2401_01607_b200.core import Signal  # noqa: E402
from paper_2401_01607_b200.engine import EngineConfig, ScatterEngine  # noqa: E402
from paper_2401_01607_b200.multichannel import MultiChannelEngine  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
dev = torch.device("cuda", 0)
if cfg == "cfg2":
    w = configs.cfg2()
    xd = torch.from_numpy(w.x).to(dev)
    irs = [torch.from_numpy(h).to(dev) for h in w.irs]
    n_blocks = -(-w.ne // 256)
    nb = 256
    swaps = [(0, irs[0])] + [(b, irs[b // 100]) for b in range(100, n_blocks, 100)]
    eng = ScatterEngine(Signal(irs[0]), EngineConfig(block_size_nb=256))
else:
    w = configs.cfg4()
    xd = torch.from_numpy(w.x).to(dev)
    hd = torch.from_numpy(w.h).to(dev)
    nb = 8192
    n_blocks = -(-w.ne // nb)
    swaps = [(0, hd), (n_blocks // 2, torch.flip(hd, dims=[1]).contiguous())]
    eng = MultiChannelEngine(hd, EngineConfig(block_size_nb=nb))
if "host" in sys.argv[2:]:
    # the e2e path: pinned host stream and pinned host IRs
    xd = xd.cpu().pin_memory()
    swaps = [(b, h.cpu().pin_memory()) for b, h in swaps]
for it in range(6):
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    t0 = time.perf_counter()
    e0.record()
    body = eng.process_stream(xd, nb, swaps)
    e1.record()
    t1 = time.perf_counter()
    tail = eng.flush()
    t2 = time.perf_counter()
    e2.record()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"iter {it}: enqueue process_stream {1e3*(t1-t0):.3f} ms, flush {1e3*(t2-t1):.3f} ms, "
          f"device stream {e0.elapsed_time(e1):.3f} ms, device total {e0.elapsed_time(e2):.3f} ms, "
          f"wall {1e3*(t3-t0):.3f} ms")

if "cprofile" in sys.argv[2:]:
    import cProfile
    import pstats

    pr = cProfile.Profile()
    pr.enable()
    for _ in range(50):
        eng.process_stream(xd, nb, swaps)
        eng.flush()
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(14)
