"""Batched multichannel convolution (north_star (3)).

The reference has no batched path: it runs one ScatterEngine per channel,
sequentially in the CLI (cli.py:186-202) or on a thread pool in the bench
(bench.py:200-202), relying on the nogil kernel (engine.py:60-66).  Here all
channels go through ONE launch of the register-tiled FP32 kernel
(grid.z = channel), each channel with its own impulse response.
"""

from __future__ import annotations

import numpy as np

from . import _dev
from . import _native as N


def convolve_batched(x, h, mode=None):
    """y[c] = x[c] (*) h[c] for all channels in one launch.

    x: [C, Ne] float32 (ndarray or tensor), h: [C, Nh] float32 (or [Nh],
    broadcast to every channel like the CLI's mono IR, cli.py:147-155).
    Returns [C, Ne+Nh-1] float32 in the caller's currency.
    """
    t = _dev.torch()
    if x.ndim != 2:
        raise ValueError(f"x must be [channels, samples], got shape {tuple(x.shape)}")
    C, ne = int(x.shape[0]), int(x.shape[1])
    if ne == 0:
        raise ValueError("input signal is empty")
    xd = _dev.as_device(x, np.float32)
    hd = _dev.as_device(h, np.float32, device=xd.device)
    if hd.ndim == 1:
        hd = hd.unsqueeze(0).expand(C, -1).contiguous()
    if hd.shape[0] != C:
        raise ValueError(f"h has {hd.shape[0]} channels, x has {C}")
    nh = int(hd.shape[1])
    if nh == 0:
        raise ValueError("impulse response is empty")
    from .core import mode_code

    L = N.lib()
    with t.cuda.device(xd.device):
        y = t.empty((C, ne + nh - 1), dtype=t.float32, device=xd.device)
        N.check(L.sc_fir_batched(N.SC_F32, mode_code(mode), N.ptr(xd), ne, N.ptr(hd), nh, N.ptr(y),
                                 ne + nh - 1, C,
                                 ne, nh, N.stream_ptr()))
    return _dev.like_input(y, x, h)
