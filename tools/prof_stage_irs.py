"""Line timing of ScatterEngine._stage_irs on cfg2's 19 pinned host IRs
(diagnostic only)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2401_01607_b200 import configs  # noqa: E402

w = configs.cfg2()
irs = [torch.from_numpy(h).pin_memory() for h in w.irs]
irs = irs[:1] + irs * 1
irs = irs[:19]
total = sum(len(a) for a in irs)
dbuf = torch.empty(total, device="cuda")
hbuf = torch.empty(total).pin_memory()
hplain = torch.empty(total)
ev = torch.cuda.Event()
for rep in range(5):
    T = [time.perf_counter()]
    hv = hbuf.numpy(); T.append(time.perf_counter())
    views = [a.numpy() for a in irs]; T.append(time.perf_counter())
    off = 0
    for v in views:
        hv[off:off + len(v)] = v
        off += len(v)
    T.append(time.perf_counter())
    hp = hplain.numpy(); off = 0
    for v in views:
        hp[off:off + len(v)] = v
        off += len(v)
    T.append(time.perf_counter())
    np.concatenate(views, out=hv); T.append(time.perf_counter())
    cur = torch.cuda.current_stream(); T.append(time.perf_counter())
    dbuf.copy_(hbuf, non_blocking=True); T.append(time.perf_counter())
    ev.record(cur); T.append(time.perf_counter())
    torch.cuda.synchronize(); T.append(time.perf_counter())
    names = ["numpy()", "views", "pack->pinned", "pack->pageable", "concat->pinned", "cur_stream", "h2d enqueue", "record",
             "sync"]
    print(" ".join(f"{n} {1e6*(b-a):.1f}" for n, a, b in zip(names, T, T[1:])), "us")
