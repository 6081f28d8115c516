"""Host-side timeline of one cfg2 fused stream call: time from entering
ScatterEngine.process_stream to the C call, inside the C call, and after."""
import os, sys, time, statistics as S
sys.path.insert(0, os.getcwd())
import torch
from paper_2401_01607_b200 import configs
from paper_2401_01607_b200.core import Signal
from paper_2401_01607_b200.engine import EngineConfig, ScatterEngine
w = configs.cfg2(); dev = torch.device("cuda", 0)
xd = torch.from_numpy(w.x).to(dev); irs = [torch.from_numpy(h).to(dev) for h in w.irs]
n_blocks = -(-w.ne // 256)
swaps = [(0, irs[0])] + [(b, irs[b // 100]) for b in range(100, n_blocks, 100)]
eng = ScatterEngine(Signal(irs[0]), EngineConfig(block_size_nb=256))
lib = eng._lib
marks = {}
class Wrap:
    def __init__(s, l): s.l = l
    def __getattr__(s, name):
        f = getattr(s.l, name)
        def g(*a):
            marks[name + ":in"] = time.perf_counter(); r = f(*a); marks[name + ":out"] = time.perf_counter(); return r
        return g
eng._lib = Wrap(lib)
for _ in range(10):
    eng.process_stream(xd, 256, swaps); eng.flush()
pre, c, post = [], [], []
for _ in range(200):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng.process_stream(xd, 256, swaps)
    t1 = time.perf_counter()
    eng.flush()
    pre.append((marks["sc_engine_process_blocks:in"] - t0) * 1e6)
    c.append((marks["sc_engine_process_blocks:out"] - marks["sc_engine_process_blocks:in"]) * 1e6)
    post.append((t1 - marks["sc_engine_process_blocks:out"]) * 1e6)
print("python before C %.1f us, C call %.1f us, python after %.1f us" % (S.median(pre), S.median(c), S.median(post)))
