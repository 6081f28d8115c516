"""CPU oracle for the scatter-convolution hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this module, and only
as the checker or the timed CPU reference -- never as the thing measured or
shipped.  The product package ``paper_2401_01607_b200`` never imports it.

It wraps ``scatter_oracle.c`` (a plain-C restatement of the reference's
``_kernels.scatter_block`` / ``core._scatter_full`` / ``core.direct_form``)
and restates the reference's engine bookkeeping (``engine.py``) in Python on
top of the C kernel.  Pinned against the reference itself: see
``tests/golden/make_golden.py`` and ``tests/test_oracle_golden.py``.
"""

from __future__ import annotations

import ctypes
import os
import pathlib

import numpy as np

_HERE = pathlib.Path(__file__).resolve().parent
_LIB = None

_i64 = ctypes.c_int64
_dp = ctypes.POINTER(ctypes.c_double)


def _host_has_avx2() -> bool:
    try:
        with open("/proc/cpuinfo", encoding="ascii", errors="ignore") as fh:
            for line in fh:
                if line.startswith("flags"):
                    flags = set(line.split(":", 1)[1].split())
                    return {"avx2", "fma", "bmi2"} <= flags
    except OSError:
        pass
    return False


def lib():
    """Load (building if needed, in the build container only) the oracle .so."""
    global _LIB
    if _LIB is not None:
        return _LIB
    names = ["liboracle_v3.so", "liboracle.so"] if _host_has_avx2() else ["liboracle.so"]
    path = None
    for name in names:
        if (_HERE / name).exists():
            path = _HERE / name
            break
    if path is None:
        import subprocess

        subprocess.run(["make", "-C", str(_HERE)], check=True, capture_output=True)
        path = _HERE / "liboracle.so"
    L = ctypes.CDLL(str(path))
    L.oracle_scatter_block.argtypes = [_dp, _i64, _dp, _i64, _dp, _i64, _dp, _i64, _i64,
                                       ctypes.c_double, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]
    L.oracle_scatter_block.restype = None
    L.oracle_scatter_full.argtypes = [_dp, _i64, _dp, _i64, _dp, ctypes.c_int, ctypes.c_double]
    L.oracle_scatter_full.restype = None
    L.oracle_direct_form.argtypes = [_dp, _i64, _dp, _i64, _dp, _i64, _i64]
    L.oracle_direct_form.restype = None
    L.oracle_conv_parallel.argtypes = [_dp, _i64, _dp, _i64, _dp, _i64, ctypes.c_int]
    L.oracle_conv_parallel.restype = ctypes.c_int
    L.oracle_conv_channels.argtypes = [_dp, _dp, _dp, _i64, _i64, _i64, _i64, ctypes.c_int]
    L.oracle_conv_channels.restype = ctypes.c_int
    L.oracle_scatter_window.argtypes = [_dp, _i64, _dp, _i64, _dp, _i64, _i64, ctypes.c_int,
                                        ctypes.c_double, ctypes.c_int]
    L.oracle_scatter_window.restype = None
    _ip = ctypes.POINTER(_i64)
    L.oracle_fixed_quantize.argtypes = [_dp, _i64, ctypes.c_int, _ip]
    L.oracle_fixed_quantize.restype = _i64
    L.oracle_fixed_conv.argtypes = [_ip, _i64, _ip, _i64, ctypes.c_int, ctypes.c_int, _dp]
    L.oracle_fixed_conv.restype = None
    _LIB = L
    return L


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _p(a: np.ndarray):
    return a.ctypes.data_as(_dp)


# ------------------------------------------------------------------ kernels


def scatter_block(ring, ir, block, out, read_index, live, threshold):
    """_kernels.scatter_block (pkg/src/scatterconv/_kernels.py:14-52); mutates ring/out."""
    assert ring.dtype == np.float64 and out.dtype == np.float64 and ring.flags.c_contiguous
    ir = _f64(ir)
    block = _f64(block)
    ri = _i64()
    lv = _i64()
    lib().oracle_scatter_block(_p(ring), len(ring), _p(ir), len(ir), _p(block), len(block),
                               _p(out), int(read_index), int(live), float(threshold),
                               ctypes.byref(ri), ctypes.byref(lv))
    return ri.value, lv.value


SKIP_NONE, SKIP_LE, SKIP_NOT_GT = 0, 1, 2


def scatter_full(drive, kern, skip_mode=SKIP_NONE, threshold=0.0) -> np.ndarray:
    """core._scatter_full (core.py:80-92), with the skip rules of core.py:163-165 / _kernels.py:33."""
    d = _f64(drive)
    k = _f64(kern)
    out = np.empty(len(d) + len(k) - 1)
    lib().oracle_scatter_full(_p(d), len(d), _p(k), len(k), _p(out), int(skip_mode), float(threshold))
    return out


def scatter_window(x, h, n_begin, n_end, skip_mode=SKIP_NONE, threshold=0.0, threads=None):
    """Outputs [n_begin, n_end) of core._scatter_full(x, h) -- bit-identical to
    those slots of the full reference result (same per-slot chain)."""
    x = _f64(x)
    h = _f64(h)
    out = np.empty(max(0, n_end - n_begin))
    threads = threads or len(os.sched_getaffinity(0))
    lib().oracle_scatter_window(_p(x), len(x), _p(h), len(h), _p(out), int(n_begin), int(n_end),
                                int(skip_mode), float(threshold), int(threads))
    return out


def direct_form(e, h, n_begin=0, n_end=None) -> np.ndarray:
    """core.direct_form (core.py:102-119): exactly rounded (fsum) gather form."""
    e = _f64(e)
    h = _f64(h)
    nout = len(e) + len(h) - 1
    if n_end is None:
        n_end = nout
    out = np.empty(n_end - n_begin)
    lib().oracle_direct_form(_p(e), len(e), _p(h), len(h), _p(out), int(n_begin), int(n_end))
    return out


def conv_parallel(x, h, nb=8192, threads=None) -> np.ndarray:
    """Full conv by one reference engine per input segment, overlap-added (see .c)."""
    x = _f64(x)
    h = _f64(h)
    y = np.empty(len(x) + len(h) - 1)
    threads = threads or len(os.sched_getaffinity(0))
    lib().oracle_conv_parallel(_p(x), len(x), _p(h), len(h), _p(y), int(nb), int(threads))
    return y


def conv_channels(x2d, h2d, nb=8192, threads=None) -> np.ndarray:
    """One reference engine per channel on a thread pool (engine.py:60-66; bench.py:200-202)."""
    x = _f64(x2d)
    h = _f64(h2d)
    C, ne = x.shape
    nh = h.shape[1]
    y = np.empty((C, ne + nh - 1))
    threads = threads or len(os.sched_getaffinity(0))
    lib().oracle_conv_channels(_p(x), _p(h), _p(y), C, ne, nh, int(nb), int(threads))
    return y


# ------------------------------------------------------------------ engine


class OracleEngine:
    """Restatement of ScatterEngine (pkg/src/scatterconv/engine.py:60-214) over the C kernel.

    Same state (ring, read_index, live, consumed, pending IR) and the same
    swap / flush bookkeeping, minus the Signal/sample-rate plumbing.
    """

    def __init__(self, h, block_size_nb=8192, zero_skip_threshold=0.0):
        h = _f64(h)
        if len(h) == 0:
            raise ValueError("impulse response is empty")
        self.nb = block_size_nb
        self.threshold = zero_skip_threshold
        self.ir = h.copy()                      # engine.py:72
        self.ring = np.zeros(len(h))            # engine.py:75
        self.read_index = 0
        self.live = 0
        self.consumed = 0
        self.pending = None

    def process_sample(self, x) -> float:      # engine.py:99-116 (no pending swap)
        out = np.empty(1)
        self.read_index, self.live = scatter_block(self.ring, self.ir, np.array([x], np.float64),
                                                   out, self.read_index, self.live, self.threshold)
        self.consumed += 1
        return float(out[0])

    def process_block(self, block) -> np.ndarray:  # engine.py:118-146
        if self.pending is not None:
            h_new, self.pending = self.pending, None
            self.swap_ir(h_new)
        block = _f64(block)
        if len(block) > self.nb:
            raise ValueError(f"block of {len(block)} samples exceeds block_size_nb={self.nb}")
        out = np.empty(len(block))
        self.read_index, self.live = scatter_block(self.ring, self.ir, block, out,
                                                   self.read_index, self.live, self.threshold)
        self.consumed += len(block)
        return out

    def schedule_order(self) -> np.ndarray:    # engine.py:211-214
        ri = self.read_index
        return np.concatenate([self.ring[ri:], self.ring[:ri]])

    def flush(self) -> np.ndarray:             # engine.py:148-161
        n_tail = max(len(self.ir) - 1, self.live)
        tail = self.schedule_order()[:n_tail].copy()
        self.ring = np.zeros(len(self.ir))
        self.read_index = 0
        self.live = 0
        self.consumed = 0
        return tail

    def swap_ir(self, h_new):                  # engine.py:163-186
        h_new = _f64(h_new)
        if len(h_new) == 0:
            raise ValueError("impulse response is empty")
        sched = self.schedule_order()
        new_cap = max(len(h_new), self.live)
        ring = np.zeros(new_cap)
        keep = min(len(sched), new_cap)
        ring[:keep] = sched[:keep]
        self.ring = ring
        self.read_index = 0
        self.ir = h_new.copy()

    def swap_ir_at_next_block(self, h_new):    # engine.py:188-192
        h_new = _f64(h_new)
        if len(h_new) == 0:
            raise ValueError("impulse response is empty")
        self.pending = h_new


def stream_with_swaps(x, irs, nb, swap_every_blocks):
    """cfg2 oracle: engine at block size nb, swap_ir to irs[j] after every
    `swap_every_blocks` blocks (engine.py:163-186); returns (per-block outputs
    concatenated, flush tail)."""
    eng = OracleEngine(irs[0], block_size_nb=nb)
    x = _f64(x)
    outs = []
    j = 0
    for b, start in enumerate(range(0, len(x), nb)):
        if b > 0 and b % swap_every_blocks == 0:
            j += 1
            eng.swap_ir(irs[j])
        outs.append(eng.process_block(x[start:start + nb]))
    tail = eng.flush()
    return np.concatenate(outs), tail


def fixed_quantize(x, word_bits):
    """quantize._quantize_ints (quantize.py:137-143): int64 grid indices;
    raises ValueError like the reference on samples outside [-1, 1)."""
    x = _f64(x)
    k = np.empty(len(x), dtype=np.int64)
    bad = lib().oracle_fixed_quantize(_p(x), len(x), int(word_bits) - 1,
                                      k.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
    if bad:
        raise ValueError("samples outside the representable range [-1, 1)")
    return k


def fixed_convolve(e, h, word_bits, scheme):
    """quantize.fixed_point_convolve (quantize.py:163-195) on raw sample arrays."""
    ke = fixed_quantize(e, word_bits)
    kh = fixed_quantize(h, word_bits)
    out = np.empty(len(ke) + len(kh) - 1)
    ip = ctypes.POINTER(ctypes.c_int64)
    lib().oracle_fixed_conv(ke.ctypes.data_as(ip), len(ke), kh.ctypes.data_as(ip), len(kh), int(word_bits) - 1,
                            {"ideal": 0, "mac": 1}[scheme], _p(out))
    return out
