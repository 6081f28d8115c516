"""The C-ABI library loads and exports every symbol include/*.h declares;
compute entry points fail loudly without a GPU (no CPU fallback).  CPU only."""

import ctypes
import pathlib
import re

import pytest

from paper_2401_01607_b200 import _native as N
from tests.conftest import cuda_ok

HEADER = pathlib.Path(__file__).resolve().parent.parent / "include" / "scatterconv_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sc_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_expected_surface():
    syms = declared_symbols()
    assert "sc_fir_full" in syms and "sc_engine_process_block" in syms
    assert set(syms) == set(N.EXPORTS), set(syms) ^ set(N.EXPORTS)


def test_library_exports_every_declared_symbol():
    L = N.load_library()
    for name in declared_symbols():
        assert hasattr(L, name), name
    assert L.sc_abi_version() == 1


def test_library_is_sm100a():
    # the .so embeds an sm_100a cubin (cuobjdump lists the ELF arch)
    import shutil
    import subprocess

    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not pathlib.Path(exe).exists():
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", str(N.library_path())], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_argument_errors_raise_valueerror_without_device():
    # validation happens before any device work: bad sizes are rejected on CPU
    L = N.load_library()
    rc = L.sc_fir_full(N.SC_F32, 0, None, 0, None, 4, None, 0, 0.0, None)
    assert rc == N.SC_ERR_ARG
    assert "empty" in L.sc_last_error().decode()
    rc = L.sc_fir_full(7, 0, None, 4, None, 4, None, 0, 0.0, None)
    assert rc == N.SC_ERR_ARG and "dtype" in L.sc_last_error().decode()
    with pytest.raises(ValueError, match="empty"):
        N.check(L.sc_fir_batched(N.SC_F32, N.SC_MODE_FAST, None, 1, None, 1, None, 1, 1, 0, 1, None))


@pytest.mark.skipif(cuda_ok(), reason="checks the no-GPU failure mode")
def test_compute_without_gpu_fails_loudly():
    import numpy as np

    from paper_2401_01607_b200 import Signal, scatter_convolve

    with pytest.raises(RuntimeError, match="CUDA"):
        scatter_convolve(Signal(np.ones(4)), Signal(np.ones(2)))


def test_product_never_imports_oracle():
    pkg = pathlib.Path(N.__file__).resolve().parent
    for py in pkg.rglob("*.py"):
        src = py.read_text()
        mods = re.findall(r"^\s*(?:from|import)\s+(\S+)", src, flags=re.M)
        assert not any(m.lstrip(".").split(".")[0] == "oracle" for m in mods), py
        assert "liboracle" not in src, py
