import os, sys, time
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
s = torch.cuda.current_stream()
e0, e1, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for it in range(10):
    eng.process_stream(xd, 256, swaps); eng.flush()
torch.cuda.synchronize()
ht, gt, ft, hs = [], [], [], []
for it in range(30):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record(s)
    body = eng.process_stream(xd, 256, swaps)
    t1 = time.perf_counter()
    e1.record(s)
    eng.flush()
    e2.record(s)
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    ht.append((t1 - t0) * 1e6); hs.append((t2 - t1) * 1e6)
    gt.append(e0.elapsed_time(e1) * 1e3); ft.append(e1.elapsed_time(e2) * 1e3)
import statistics as S
print("host process_stream %.1f us, host flush %.1f us, gpu stream %.1f us, gpu flush %.1f us" % (S.median(ht), S.median(hs), S.median(gt), S.median(ft)))
# GPU-only: launch while the GPU is busy so host overhead hides
torch.cuda._sleep(int(2e6))
e0.record(s)
for it in range(20):
    eng.process_stream(xd, 256, swaps)
e1.record(s)
torch.cuda.synchronize()
print("back-to-back process_stream (no flush), GPU-side: %.1f us each" % (e0.elapsed_time(e1) * 1e3 / 20))
