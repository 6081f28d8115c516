"""Medium launches (fewer than 2 tiles per SM): fused split vs image path.
Run once per SC_FS_MIN_TILES_X2 value (static knob); prints ms per call."""
import os, sys, pathlib
import numpy as np, torch
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
from paper_2401_01607_b200.core import Signal, scatter_convolve
from paper_2401_01607_b200 import _native as N

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for ne in (1 << 20, 1 << 21, 2_880_000, 1 << 22):
    for nh in (512, 1024, 2048, 4096, 8192):
        rng = np.random.default_rng(1)
        x = torch.from_numpy(rng.uniform(-1, 1, ne).astype(np.float32)).cuda()
        h = torch.from_numpy(rng.standard_normal(nh).astype(np.float32)).cuda()
        for _ in range(3):
            scatter_convolve(Signal(x), Signal(h))
        ts = []
        for _ in range(10):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); scatter_convolve(Signal(x), Signal(h)); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(os.environ.get("SC_FS_MIN_TILES_X2", "4"), ne, nh, round(float(np.median(ts)), 4), N.tc_stats()["kernel"], flush=True)
