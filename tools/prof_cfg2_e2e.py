"""cfg2 end to end (pinned host stream + pinned host IRs), phase by phase:
graph-cache stats of the engine and the wall time of each piece with a
device sync after it.  Diagnostic only."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2401_01607_b200 import _native as N, configs  # noqa: E402
from paper_2401_01607_b200.core import Signal  # noqa: E402
from paper_2401_01607_b200.engine import EngineConfig, ScatterEngine  # noqa: E402

w = configs.cfg2()
nb = 256
n_blocks = -(-w.ne // nb)
irs = [torch.from_numpy(h).pin_memory() for h in w.irs]
swaps = [(0, irs[0])] + [(b, irs[b // 100]) for b in range(100, n_blocks, 100)]
x = torch.from_numpy(w.x).pin_memory()
eng = ScatterEngine(Signal(irs[0].cuda()), EngineConfig(block_size_nb=nb))


def stats():
    h, c, f = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    N.check(N.lib().sc_engine_graph_stats(eng._handle, ctypes.byref(h), ctypes.byref(c), ctypes.byref(f)))
    return h.value, c.value, f.value


for it in range(12):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    body = eng.process_stream(x, nb, swaps)
    t1 = time.perf_counter()
    tail = eng.flush()
    t2 = time.perf_counter()
    print(f"iter {it}: process_stream {1e3*(t1-t0):.3f} ms, flush {1e3*(t2-t1):.3f} ms, graph hits/captures/failures {stats()}")

# pieces
torch.cuda.synchronize()
for name, fn in [("h2d x", lambda: x.to("cuda", non_blocking=True)),
                 ("stage irs", lambda: eng._stage_irs([s[1] for s in swaps]))]:
    for _ in range(3):
        t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"{name}: {1e3*dt:.3f} ms")
xd = x.cuda()
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    body = eng.process_stream(xd, nb, swaps); torch.cuda.synchronize(); t1 = time.perf_counter()
    eng.flush(); t2 = time.perf_counter()
    print(f"device x, host IRs: process_stream {1e3*(t1-t0):.3f} ms, flush {1e3*(t2-t1):.3f} ms, graphs {stats()}")

# copy primitives
d = torch.empty_like(x, device="cuda")
hp = torch.empty_like(x).pin_memory()
for name, fn in [("sync only", lambda: None),
                 ("x.to(cuda) 1.9 MB", lambda: x.to("cuda", non_blocking=True)),
                 ("d.copy_(x) 1.9 MB", lambda: d.copy_(x, non_blocking=True)),
                 ("hp.copy_(d) 1.9 MB", lambda: hp.copy_(d, non_blocking=True)),
                 ("stage irs", lambda: eng._stage_irs([s[1] for s in swaps]))]:
    ts = []
    for _ in range(20):
        torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    print(f"{name}: median {1e3*ts[10]:.3f} ms, min {1e3*ts[0]:.3f} ms")

# the library's host-stream path for this small stream too
from paper_2401_01607_b200 import _dev  # noqa: E402
_dev.PINNED_STREAM_MIN_BYTES = 1
for it in range(8):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    body = eng.process_stream(x, nb, swaps)
    t1 = time.perf_counter()
    tail = eng.flush()
    t2 = time.perf_counter()
    print(f"host-stream path iter {it}: process_stream {1e3*(t1-t0):.3f} ms, flush {1e3*(t2-t1):.3f} ms, graphs {stats()}")
