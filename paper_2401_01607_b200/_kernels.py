"""Drop-in for ``scatterconv._kernels`` (pkg/src/scatterconv/_kernels.py:14-59).

``scatter_block`` keeps the reference signature and in-place semantics on
numpy arrays (ring and out are mutated) or CUDA tensors, but runs on the
GPU through the C ABI entry ``sc_scatter_block``.  It is synchronous because
it returns the data-dependent ``live`` count, exactly like the reference;
the streaming engine (engine.py) does not use it -- it keeps its state on
the device instead.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _dev
from . import _native as N


def scatter_block(ring, ir, block, out, read_index, live, threshold):
    """Process one block of input samples through the residue ring
    (_kernels.py:15-52).  Returns the updated (read_index, live)."""
    npd = _dev.np_dtype(ring)
    t = _dev.torch()
    L = N.lib()
    ring_d = _dev.as_device(ring, npd)
    ir_d = _dev.as_device(ir, npd, device=ring_d.device)
    blk_d = _dev.as_device(block, npd, device=ring_d.device)
    n = blk_d.shape[0]
    out_d = t.empty(n, dtype=ring_d.dtype, device=ring_d.device)
    ri = ctypes.c_int64()
    lv = ctypes.c_int64()
    with t.cuda.device(ring_d.device):
        N.check(L.sc_scatter_block(N.dtype_code(npd), N.ptr(ring_d), ring_d.shape[0], N.ptr(ir_d),
                                   ir_d.shape[0], N.ptr(blk_d), n, N.ptr(out_d), int(read_index),
                                   int(live), float(threshold), ctypes.byref(ri), ctypes.byref(lv),
                                   N.stream_ptr()))
    # write back in place (the reference mutates ring and out)
    if _dev.is_tensor(ring):
        ring.copy_(ring_d)
    else:
        ring[...] = ring_d.cpu().numpy()
    if _dev.is_tensor(out):
        out.copy_(out_d)
    else:
        out[...] = out_d.cpu().numpy()
    return ri.value, lv.value


def warm_up():
    """Load the library and run one tiny launch so timed runs never include
    module load / context creation (_kernels.py:55-59)."""
    ring = np.zeros(4)
    out = np.empty(2)
    scatter_block(ring, np.ones(3), np.zeros(2), out, 0, 0, 0.0)
