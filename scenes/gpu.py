"""GPU echo synthesis (``scenes/csrc/scene_gen.cu``) -- an INPUT GENERATOR,
not part of the reconstruction path.  Same sum as ``scenes.synthesize_cpu``
(Eq. (9)) and the same counter-based noise (``scenes/rng.py``)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(_HERE, "csrc", "scene_gen.cu")
LIB = os.path.join(_HERE, "libscene_gen.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
_lib = None


def build(force=False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(SRC) > os.path.getmtime(LIB):
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-shared",
               "-Xcompiler", "-fPIC", "-o", LIB, SRC]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError("nvcc failed for scene_gen.cu:\n" + r.stdout + r.stderr)
    return LIB


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise ImportError(f"{LIB} not built (scenes.gpu.build())")
        _lib = C.CDLL(LIB)
        vp = C.c_void_p
        _lib.scene_echo.restype = C.c_int
        _lib.scene_echo.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, vp, vp, C.c_int,
                                    C.c_double, C.c_double, C.c_ulonglong, C.c_double, vp]
    return _lib


def synthesize_gpu(sc, device=0, noise=True, out=None):
    """Return a complex64 CUDA tensor s[F, n_tx, n_rx, P, n_k] for scene ``sc``."""
    import torch
    lib = _load()
    dev = torch.device("cuda", device)
    F, nt, nr, P, nk = sc.data_shape
    if out is None:
        out = torch.empty(sc.data_shape, dtype=torch.complex64, device=dev)
    nsc = max(len(q) for q in sc.scat_pos) if F else 0
    scat = np.zeros((F, max(nsc, 1), 5))
    for f in range(F):
        n = len(sc.scat_pos[f])
        scat[f, :n, :3] = sc.scat_pos[f]
        scat[f, :n, 3] = np.real(sc.scat_amp[f])
        scat[f, :n, 4] = np.imag(sc.scat_amp[f])   # padded entries have zero amplitude
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=dev)  # noqa: E731
    tx, rx, scan, sq = t(sc.tx), t(sc.rx), t(sc.scan), t(scat)
    k = sc.k
    k0 = float(k[0])
    dk = float((k[-1] - k[0]) / (nk - 1))
    sigma = float(sc.noise_sigma) if noise else 0.0
    stream = torch.cuda.current_stream(dev).cuda_stream
    err = lib.scene_echo(C.c_void_p(out.data_ptr()), F, nt, nr, P, nk, C.c_void_p(tx.data_ptr()),
                         C.c_void_p(rx.data_ptr()), C.c_void_p(scan.data_ptr()), C.c_void_p(sq.data_ptr()),
                         max(nsc, 1) if nsc else 0, k0, dk, C.c_ulonglong(sc.noise_key & 0xFFFFFFFFFFFFFFFF),
                         sigma, C.c_void_p(stream))
    if err:
        raise RuntimeError(f"scene_echo failed with CUDA error {err}")
    torch.cuda.synchronize(dev)
    return out
