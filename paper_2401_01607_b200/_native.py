"""ctypes binding of the CUDA library (include/scatterconv_b200.h).

The library is built in-tree (``python -m paper_2401_01607_b200.build`` or
``__graft_entry__.build()``) into ``paper_2401_01607_b200/_lib``.  There is
no CPU fallback: if the library or a CUDA device is missing, every entry
point raises immediately.
"""

from __future__ import annotations

import ctypes
import os
import pathlib
import threading

import numpy as np

LIB_DIR = pathlib.Path(__file__).resolve().parent / "_lib"
LIB_NAME = "libscatterconv_b200.so"

SC_F32, SC_F64 = 0, 1
SC_MODE_FAST, SC_MODE_ORDERED, SC_MODE_FFMA, SC_MODE_TC = 0, 1, 2, 3
SC_SKIP_NONE, SC_SKIP_LE, SC_SKIP_NOT_GT = 0, 1, 2
SC_ERR_ARG = -1

_i64 = ctypes.c_int64
_vp = ctypes.c_void_p
_p64 = ctypes.POINTER(ctypes.c_int64)
_pint = ctypes.POINTER(ctypes.c_int)

# name -> argtypes (restype is int for all but sc_last_error)
_SIGNATURES = {
    "sc_abi_version": [],
    "sc_fir_full": [ctypes.c_int, ctypes.c_int, _vp, _i64, _vp, _i64, _vp, ctypes.c_int,
                    ctypes.c_double, _vp],
    "sc_fir_range": [ctypes.c_int, ctypes.c_int, _vp, _i64, _i64, _vp, _i64, _vp, _i64, _i64, _vp],
    "sc_fir_batched": [ctypes.c_int, ctypes.c_int, _vp, _i64, _vp, _i64, _vp, _i64, _i64, _i64,
                       _i64, _vp],
    "sc_direct_form": [_vp, _i64, _vp, _i64, _vp, _vp, _vp],
    "sc_scatter_block": [ctypes.c_int, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _i64,
                         ctypes.c_double, _p64, _p64, _vp],
    "sc_engine_create": [ctypes.c_int, _vp, _i64, _i64, ctypes.c_double, _vp,
                         ctypes.POINTER(_vp)],
    "sc_wav_decode": [ctypes.c_int, _vp, _i64, _i64, ctypes.c_int, _vp, _vp],
    "sc_wav_encode": [ctypes.c_int, ctypes.c_int, _vp, _i64, _i64, _i64, ctypes.c_double, _vp, _vp, _vp],
    "sc_peak_abs": [ctypes.c_int, _vp, _i64, _vp, _vp],
    "sc_engine_tail_bound": [_vp, _p64],
    "sc_fir_sharded": [ctypes.c_int, ctypes.c_int, _vp, _i64, _vp, _i64, _vp, ctypes.c_int,
                       ctypes.POINTER(ctypes.c_int), ctypes.c_int],
    "sc_fir_range_host": [ctypes.c_int, ctypes.c_int, _vp, _i64, _vp, _i64, _vp, _i64, _i64, ctypes.c_int,
                          ctypes.c_int],
    "sc_engine_set_mode": [_vp, ctypes.c_int],
    "sc_fixed_quantize": [_vp, _i64, ctypes.c_int, _vp, _vp, _vp, _vp],
    "sc_fixed_round_shift": [_vp, _i64, ctypes.c_int, _vp, _vp],
    "sc_fixed_convolve": [_vp, _i64, _vp, _i64, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp, _vp],
    "sc_engine_create_multi": [ctypes.c_int, _vp, _i64, _i64, _i64, ctypes.c_double, _vp,
                               ctypes.POINTER(_vp)],
    "sc_engine_channels": [_vp, _p64],
    "sc_engine_destroy": [_vp],
    "sc_engine_set_stream": [_vp, _vp],
    "sc_engine_process_block": [_vp, _vp, _i64, _vp],
    "sc_engine_process_sample": [_vp, _vp, _vp],
    "sc_engine_swap_ir": [_vp, _vp, _i64],
    "sc_engine_swap_ir_at_next_block": [_vp, _vp, _i64],
    "sc_engine_flush": [_vp, _vp, _i64, _p64],
    "sc_engine_flush_begin": [_vp, _vp, _i64],
    "sc_engine_flush_end": [_vp, _vp],
    "sc_engine_state": [_vp, _p64, _p64, _p64, _p64, _p64, _pint],
    "sc_engine_schedule": [_vp, _vp, _i64, _p64],
    "sc_engine_current_ir": [_vp, _vp, _i64, _p64],
    "sc_engine_process_blocks": [_vp, _vp, _i64, _i64, _p64, ctypes.POINTER(_vp), _p64, _i64,
                                 _vp],
    "sc_engine_process_blocks_host": [_vp, _vp, _i64, _i64, _p64, ctypes.POINTER(_vp), _p64, _i64,
                                      _vp, ctypes.c_int],
    "sc_tc_stats": [_p64, _p64, _pint, _pint],
    "sc_engine_graph_stats": [_vp, _p64, _p64, _p64],
    "sc_engine_swap_ir_channels": [_vp, _vp, _i64, _p64],
    "sc_engine_swap_ir_at_next_block_channels": [_vp, _vp, _i64, _p64],
    "sc_engine_channel_nh": [_vp, _p64],
    "sc_engine_process_blocks_channels": [_vp, _vp, _i64, _i64, _p64, ctypes.POINTER(_vp), _p64, _p64, _i64,
                                          _vp],
}
EXPORTS = tuple(_SIGNATURES) + ("sc_last_error", "sc_launch_count", "sc_tc_stats_reset", "sc_tc_last_kernel")
TC_KERNEL_NAMES = {0: None, 1: "k_tc_fir", 2: "k_tc_fir_fs"}   # SC_TC_KERNEL_* (include/scatterconv_b200.h)

_lock = threading.Lock()
_lib = None


def library_path() -> pathlib.Path:
    # SC_B200_LIB: an alternative build of the same library (A/B timing)
    alt = os.environ.get("SC_B200_LIB")
    return pathlib.Path(alt) if alt else LIB_DIR / LIB_NAME


def load_library() -> ctypes.CDLL:
    """Load the shared library (no CUDA device needed just to load it)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = library_path()
        if not path.exists():
            raise RuntimeError(
                f"scatterconv-b200 CUDA library not built: {path} is missing "
                "(run `python -m paper_2401_01607_b200.build`). There is no CPU fallback.")
        L = ctypes.CDLL(str(path))
        for name, args in _SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        L.sc_last_error.argtypes = []
        L.sc_last_error.restype = ctypes.c_char_p
        L.sc_launch_count.argtypes = []
        L.sc_launch_count.restype = ctypes.c_int64
        L.sc_tc_stats_reset.argtypes = []
        L.sc_tc_stats_reset.restype = None
        L.sc_tc_last_kernel.argtypes = []
        L.sc_tc_last_kernel.restype = ctypes.c_int
        _lib = L
        return L


_cuda_checked = False


def lib() -> ctypes.CDLL:
    """Library handle for COMPUTE calls: also insists on a CUDA device."""
    global _cuda_checked
    L = load_library()
    if not _cuda_checked:
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("scatterconv-b200 requires a CUDA device (B200, sm_100a); "
                               "no CPU fallback exists")
        _cuda_checked = True
    return L


def check(rc: int):
    if rc == 0:
        return
    msg = load_library().sc_last_error().decode("utf-8", "replace")
    if rc == SC_ERR_ARG:
        raise ValueError(msg)
    raise RuntimeError(f"scatterconv-b200 error {rc}: {msg}")


def dtype_code(dtype) -> int:
    import torch

    if dtype in (torch.float32, np.float32):
        return SC_F32
    if dtype in (torch.float64, np.float64):
        return SC_F64
    raise TypeError(f"unsupported dtype {dtype}")


def stream_ptr(stream=None):
    """cudaStream_t of `stream`, or of the current device's current stream.
    The default path asks torch's C layer directly (~0.3 us instead of ~10 us
    through torch.cuda.current_stream(), which dominated small engine calls)."""
    import torch

    if stream is not None:
        return ctypes.c_void_p(stream.cuda_stream)
    C = torch._C
    raw = getattr(C, "_cuda_getCurrentRawStream", None)
    if raw is not None:
        return ctypes.c_void_p(raw(C._cuda_getDevice()))
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


def tc_stats() -> dict:
    """Cumulative tensor-core launch bookkeeping (sc_tc_stats)."""
    L = load_library()
    n, macs = ctypes.c_int64(), ctypes.c_int64()
    ssh, tn = ctypes.c_int(), ctypes.c_int()
    check(L.sc_tc_stats(ctypes.byref(n), ctypes.byref(macs), ctypes.byref(ssh), ctypes.byref(tn)))
    return {"launches": n.value, "padded_macs": macs.value, "ssh": ssh.value, "tile_n": tn.value,
            "kernel": TC_KERNEL_NAMES.get(L.sc_tc_last_kernel())}
