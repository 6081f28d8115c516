import os, sys, time
sys.path.insert(0, "/root/repo")
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
class Wrap:
    def __init__(s, l): s.l = l; s.t = {}
    def __getattr__(s, name):
        f = getattr(s.l, name)
        def g(*a):
            t0 = time.perf_counter(); r = f(*a); s.t[name] = s.t.get(name, 0) + time.perf_counter() - t0; return r
        return g
W = Wrap(lib); eng._lib = W
for it in range(30):
    if it == 10: W.t = {}; T0 = time.perf_counter()
    body = eng.process_stream(xd, 256, swaps); eng.flush()
torch.cuda.synchronize(); T = time.perf_counter() - T0
print("per iter total %.1f us" % (T / 20 * 1e6))
for k, v in W.t.items(): print(k, "%.1f us" % (v / 20 * 1e6))
