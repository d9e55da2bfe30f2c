"""Oracle for the NUFFT placement mode: the forward spatial
transform of Eq. (14) evaluated on the TRUE non-uniform planar positions
(x', y') left after the multi-planar compensation, "a non-uniform FFT (NUFFT)
approach employing fast Gaussian gridding (FGG)" (Greengard & Lee,
cited as greengard2006nufft).

TEST INFRASTRUCTURE ONLY -- never imported by the product path.

Positions are expressed in lattice units of the FFT grid (reading R19): the
virtual element of pair (t,r) at pose p sits at
    u = (x_p - x0)/dx + j^x_tr,   v = (y_p - y0)/dy + j^y_tr
(x_p, y_p the ACTUAL pose position; with zero in-plane jitter u, v are exactly
the RASTER nodes of reading R7).  The type-1 transform on the FFT index grid is
    S[b, a] = sum_m c_m exp(-2 pi i (a_s u_m / N_x + b_s v_m / N_y))
(a_s the signed index), periodic in (u, v) like the modular placement (R6).

FGG (written out step by step):
  1. fine grid R = sigma*N per axis (sigma = 2), Gaussian phi(t) = exp(-t^2/(2 s2))
     in fine cells, truncated to |t| <= W; s2 = W / (2 pi (1 - 1/(2 sigma)))
     balances truncation exp(-W^2/(2 s2)) against aliasing
  2. spread: f[jy, jx] += c_m phi(jx - sigma u_m) phi(jy - sigma v_m) (indices mod R)
  3. FFT of the fine grid (numpy sign)
  4. keep |a_s| < N/2 and divide by the kernel's continuous transform
     Phi(a) = sqrt(2 pi s2) exp(-2 pi^2 s2 a^2 / R^2) per axis
"""
from __future__ import annotations

import os

import numpy as np
import scipy.fft

from . import rma

SIGMA = 2
WIDTH = 6


def fgg_params(sigma: int = SIGMA, width: int = WIDTH):
    """(s2, width) of the Gaussian for the requested oversampling and half width."""
    return width / (2.0 * np.pi * (1.0 - 1.0 / (2.0 * sigma))), width


def signed(n: int) -> np.ndarray:
    a = np.arange(n)
    return np.where(a < n // 2, a, a - n)


def direct_dft2(u, v, c, nx: int, ny: int) -> np.ndarray:
    """Exact non-uniform sum S[b, a, ...] = sum_m c_m e^{-2 pi i (a_s u_m/nx + b_s v_m/ny)}.
    u, v: [M]; c: [M, ...].  Returns complex128 [ny, nx, ...]."""
    u = np.asarray(u, float)
    v = np.asarray(v, float)
    c = np.asarray(c, complex)
    ex = np.exp(-2j * np.pi * np.outer(signed(nx), u) / nx)      # [nx, M]
    ey = np.exp(-2j * np.pi * np.outer(signed(ny), v) / ny)      # [ny, M]
    out = np.einsum("bm,am,m...->ba...", ey, ex, c)
    # back to the FFT index order (row a holds frequency a_s)
    return out


def nufft2_type1(u, v, c, nx: int, ny: int, sigma: int = SIGMA, width: int = WIDTH) -> np.ndarray:
    """FGG type-1 transform (steps 1-4 above).  u, v: [M]; c: [M, K].
    Returns complex128 [ny, nx, K] on the FFT index grid."""
    u = np.asarray(u, float)
    v = np.asarray(v, float)
    c = np.asarray(c, complex).reshape(u.size, -1)
    s2, W = fgg_params(sigma, width)
    Rx, Ry = sigma * nx, sigma * ny
    grid = np.zeros((Ry, Rx, c.shape[1]), complex)
    cx, cy = sigma * u, sigma * v
    bx, by = np.floor(cx).astype(np.int64), np.floor(cy).astype(np.int64)
    for ty in range(-W, W + 2):
        jy = by + ty
        wy = np.exp(-(jy - cy) ** 2 / (2.0 * s2)) * (np.abs(jy - cy) <= W)
        for tx in range(-W, W + 2):
            jx = bx + tx
            wx = np.exp(-(jx - cx) ** 2 / (2.0 * s2)) * (np.abs(jx - cx) <= W)
            w = wx * wy
            np.add.at(grid, (jy % Ry, jx % Rx), w[:, None] * c)
    G = scipy.fft.fft2(grid, axes=(0, 1), workers=os.cpu_count())
    ax, ay = signed(nx), signed(ny)
    phx = np.sqrt(2.0 * np.pi * s2) * np.exp(-2.0 * np.pi ** 2 * s2 * ax ** 2 / Rx ** 2)
    phy = np.sqrt(2.0 * np.pi * s2) * np.exp(-2.0 * np.pi ** 2 * s2 * ay ** 2 / Ry ** 2)
    crop = G[np.ix_(ay % Ry, ax % Rx)]
    return crop / (phy[:, None, None] * phx[None, :, None])


def positions(geo: rma.Geometry, scan, x0: float, y0: float):
    """Lattice-unit positions (u, v) [F, n_tx, n_rx, P] of every virtual element
    (reading R19)."""
    scan = np.asarray(scan, float)
    px = (scan[:, :, 0] - x0) / geo.dx                          # [F, P]
    py = (scan[:, :, 1] - y0) / geo.dy
    u = px[:, None, None, :] + geo.jx[None, :, :, None]
    v = py[:, None, None, :] + geo.jy[None, :, :, None]
    return u, v


def compensate_values(s, geo: rma.Geometry, no_compensation=False) -> np.ndarray:
    """O2 without the placement: s_hat = s exp(+j k beta) per (f, t, r, p, k)."""
    F, nt, nr, P, nk = s.shape
    out = np.empty(s.shape, complex)
    for f in range(F):
        for t in range(nt):
            for r in range(nr):
                b = np.zeros(P) if no_compensation else rma.beta(geo, f, t, r)
                out[f, t, r] = s[f, t, r].astype(complex) * np.exp(1j * geo.k[None, :] * b[:, None])
    return out


def spectrum_nufft(s, sc, direct=False, no_compensation=False):
    """O2 + O3 of the NUFFT mode: compensated samples transformed from their
    true positions.  Returns (S [F, ny, nx, n_k], geometry)."""
    geo = rma.geometry_of(sc)
    shat = compensate_values(s, geo, no_compensation)
    u, v = positions(geo, sc.scan, sc.x0, sc.y0)
    F = shat.shape[0]
    S = np.zeros((F, geo.ny, geo.nx, geo.k.size), complex)
    for f in range(F):
        uu, vv = u[f].ravel(), v[f].ravel()
        cc = shat[f].reshape(-1, geo.k.size)
        S[f] = direct_dft2(uu, vv, cc, geo.nx, geo.ny) if direct else nufft2_type1(uu, vv, cc, geo.nx, geo.ny)
    return S, geo


def reconstruct_nufft(s, sc, direct=False, complex_out=False):
    """Whole path with NUFFT placement: O1, compensation, type-1 NUFFT from the
    true positions, then O4-O7 unchanged."""
    S, geo = spectrum_nufft(s, sc, direct)
    img = rma.magnitude_image(rma.ifft3(rma.stolt(rma.rma_filter(S, geo), geo)), geo, complex_out)
    return img, geo
