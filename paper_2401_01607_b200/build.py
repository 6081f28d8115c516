"""Build the in-tree CUDA library for sm_100a (no GPU needed: nvcc cross-compiles).

    python -m paper_2401_01607_b200.build [--verbose]

Output: paper_2401_01607_b200/_lib/libscatterconv_b200.so (git-ignored; it
travels to the GPU box with the repo snapshot).
"""

from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import pathlib
import shutil
import subprocess
import sys

PKG = pathlib.Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT = PKG / "_lib" / "libscatterconv_b200.so"
SOURCES = ["capi.cu", "k_ordered.cu", "k_fast_f32.cu", "k_tc_fir.cu", "engine.cu", "k_wav.cu", "k_fixed.cu", "sharded.cu"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and pathlib.Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def needs_build() -> bool:
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "scatterconv_b200.h"]
    return any(d.stat().st_mtime > t for d in deps if d.exists())


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed: {' '.join(cmd[-3:])}")
    if verbose:
        sys.stderr.write(res.stderr)


def build(verbose: bool = False, force: bool = False) -> pathlib.Path:
    """Every translation unit compiles in parallel (they are independent: no
    relocatable device code), then one shared-library link."""
    if not force and not needs_build():
        return OUT
    OUT.parent.mkdir(parents=True, exist_ok=True)
    objdir = OUT.parent / "obj"
    objdir.mkdir(exist_ok=True)
    extra = ["-Xptxas=-v"] if verbose else []
    jobs = [[nvcc(), *NVCC_FLAGS, *extra, "-c", "-o", str(objdir / (s + ".o")), str(CSRC / s)] for s in SOURCES]
    with cf.ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 1)) as ex:
        list(ex.map(lambda c: _run(c, verbose), jobs))
    tmp = OUT.with_suffix(".so.tmp")
    _run([nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(tmp),
          *[str(objdir / (s + ".o")) for s in SOURCES]], verbose)
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--force", action="store_true")
    a = ap.parse_args()
    print(build(verbose=a.verbose, force=a.force))
