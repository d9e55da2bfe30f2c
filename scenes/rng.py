"""Counter-based random numbers shared (by re-implementation, not by code) with
the CUDA scene generator in ``scenes/csrc/scene_gen.cu``.

This module holds NO arithmetic of the paper's method: it only draws the
additive receiver noise of the synthetic echoes.  The same generator is written
twice (here in NumPy, there in CUDA) so that large scenes can be synthesised on
the GPU while small ones are synthesised on the CPU, bit-compatible in the
integer stream and equal to rounding in the Gaussian values.

Generator: splitmix64 (Steele, Lea & Flood 2014) over the counter
``key + 2*n`` / ``key + 2*n + 1``; the two 53-bit uniforms feed Box-Muller.
"""
from __future__ import annotations

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser applied elementwise to a uint64 array."""
    with np.errstate(over="ignore"):
        z = (x + _GOLDEN).astype(np.uint64)
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def uniform53(bits: np.ndarray) -> np.ndarray:
    """Map 64 random bits to a float64 uniform in (0, 1)."""
    return ((bits >> np.uint64(11)).astype(np.float64) + 0.5) * (1.0 / 9007199254740992.0)


def complex_normal(key: int, start: int, count: int, sigma: float) -> np.ndarray:
    """Circular complex Gaussian samples n with E|n|^2 = sigma^2.

    Sample ``start + i`` uses counters ``2*(start+i)`` and ``2*(start+i)+1``
    offset by ``key``.  Returns complex128.
    """
    idx = np.arange(start, start + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        c0 = np.uint64(key) + idx * np.uint64(2)
        c1 = c0 + np.uint64(1)
    u1 = uniform53(splitmix64(c0))
    u2 = uniform53(splitmix64(c1))
    r = np.sqrt(-2.0 * np.log(u1)) * (sigma / np.sqrt(2.0))
    th = 2.0 * np.pi * u2
    return r * np.cos(th) + 1j * (r * np.sin(th))
