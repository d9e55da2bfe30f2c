"""Build the CUDA library in-tree: ``paper_2305_02064_b200/libsar_b200.so``.

nvcc for sm_100a only (``-gencode arch=compute_100a,code=sm_100a``), host code
compiled with ``-ffp-contract=off`` (the fp64 tables must be the same IEEE
expressions the oracle evaluates), ``-lineinfo`` for ncu source attribution.
Incremental: objects are rebuilt only when a source or header is newer.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libsar_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES = ["plan.cpp", "pipeline.cu", "k1.cu", "fft_mid.cu", "k3.cu", "k4.cu", "nufft.cu", "bpa.cu"]
HEADERS = [os.path.join(CSRC, h) for h in ("plan_internal.h", "fft_tile.cuh", "fft_reg.cuh", "tma.cuh", "common.cuh")] + \
    [os.path.join(ROOT, "include", "sar_b200.h")]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
         "-Xptxas", "-v", "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]


def _newer(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, force, verbose, bdir=BUILD, defines=()):
    s = os.path.join(CSRC, src)
    o = os.path.join(bdir, src + ".o")
    if force or _newer(o, [s] + HEADERS):
        if src.endswith(".cpp"):
            cmd = [NVCC, *FLAGS, *defines, "-x", "c++", "-c", s, "-o", o]
        else:
            cmd = [NVCC, *ARCH, *FLAGS, *defines, "-x", "cu", "-c", s, "-o", o]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if verbose or r.returncode:
            sys.stderr.write(r.stdout + r.stderr)
        if r.returncode:
            raise RuntimeError(f"nvcc failed on {src}")
        with open(o + ".ptxas.txt", "w") as fh:
            fh.write(r.stderr)
    return o


def build(verbose: bool = False, force: bool = False, variant: str = "", defines=()) -> str:
    """Compile every translation unit (in parallel) and link the library.
    ``variant`` + ``defines`` (e.g. ["-DK4A_ROWS=256"]) build an experiment
    copy, ``libsar_b200_<variant>.so``, from objects of its own (A/B timing
    of compile-time alternatives; the product library is never affected)."""
    from concurrent.futures import ThreadPoolExecutor
    bdir = BUILD + ("_" + variant if variant else "")
    lib = LIB if not variant else LIB.replace(".so", "_" + variant + ".so")
    os.makedirs(bdir, exist_ok=True)
    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda src: _compile(src, force, verbose, bdir, list(defines)), SOURCES))
    if force or _newer(lib, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", lib, *objs, "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link failed")
    return lib


if __name__ == "__main__":
    var = [a.split("=", 1)[1] for a in sys.argv if a.startswith("--variant=")]
    defs = [a for a in sys.argv if a.startswith("-D")]
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv, variant=var[0] if var else "", defines=defs))
