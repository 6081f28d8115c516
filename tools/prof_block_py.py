import os, sys, time, cProfile, pstats
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2401_01607_b200 import configs
from paper_2401_01607_b200.core import Signal
from paper_2401_01607_b200.engine import EngineConfig, ScatterEngine
w = configs.cfg2()
for dt in (np.float32, np.float64):
    xd = torch.from_numpy(w.x.astype(dt)).cuda()
    h = torch.from_numpy(w.irs[0].astype(dt)).cuda()
    eng = ScatterEngine(Signal(h), EngineConfig(block_size_nb=256))
    blocks = [Signal(xd[s:s + 256]) for s in range(0, w.ne, 256)]
    for b in blocks[:50]: eng.process_block(b)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for b in blocks: eng.process_block(b)
    torch.cuda.synchronize()
    print(dt.__name__, "process_block (Signal prebuilt) %.2f us" % ((time.perf_counter() - t0) / len(blocks) * 1e6))
    pr = cProfile.Profile(); pr.enable()
    for b in blocks: eng.process_block(b)
    pr.disable(); torch.cuda.synchronize()
    st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(6)
