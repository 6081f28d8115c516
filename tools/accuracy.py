#!/usr/bin/env python
"""Accuracy margins of every float32 kernel on the BASELINE configs.

Prints one JSON line per (config, kernel): max-abs error vs the CPU oracle
(prefix + seeded spot windows, as in tests/test_configs_gpu.py) divided by the
north_star tolerance 1e-5*max|x|*||h||_1.  Needs a GPU; the oracle runs on
the host cores.  Used to fill DESIGN.md's accuracy table.
"""

import json
import pathlib
import sys

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))

from oracle import oracle as O  # noqa: E402
from paper_2401_01607_b200 import configs  # noqa: E402
from paper_2401_01607_b200.core import Signal, scatter_convolve  # noqa: E402
from paper_2401_01607_b200.multichannel import convolve_batched  # noqa: E402


def windows(nout, seed, count=16, width=256):
    st = np.random.default_rng(seed).integers(0, nout - width, count)
    return sorted(set([0, nout - width] + [int(s) for s in st]))


def measure(y, x, h, wins, width=256, prefix=0):
    tol = configs.tolerance(x, h, "f32")
    err = 0.0
    if prefix:
        err = max(err, float(np.max(np.abs(y[:prefix].astype(np.float64) - O.scatter_window(x, h, 0, prefix)))))
    for s in wins:
        ref = O.scatter_window(x, h, s, s + width)
        err = max(err, float(np.max(np.abs(y[s:s + width].astype(np.float64) - ref))))
    return err / tol


def main():
    import torch

    for mode in ("ffma", "tc"):
        for name in ("cfg3", "cfg5"):
            w = configs.cfg3() if name == "cfg3" else configs.cfg5()
            y = scatter_convolve(Signal(torch.from_numpy(w.x).cuda()), Signal(torch.from_numpy(w.h).cuda()),
                                 mode=mode).concatenated().samples.cpu().numpy()
            frac = measure(y, w.x, w.h, windows(w.nout, (9, 1)), prefix=100_000)
            print(json.dumps({"config": name, "kernel": mode, "max_err_over_tol": frac}), flush=True)
        w = configs.cfg4()
        y = convolve_batched(torch.from_numpy(w.x).cuda(), torch.from_numpy(w.h).cuda(), mode=mode).cpu().numpy()
        frac = max(measure(y[c], w.x[c], w.h[c], windows(w.nout, (9, 2, c), count=4)) for c in range(0, 64, 7))
        print(json.dumps({"config": "cfg4", "kernel": mode, "max_err_over_tol": frac}), flush=True)


if __name__ == "__main__":
    main()
