"""Oracle for the NUFFT Stolt step (reading R21, "a 1-D NUFFT
for Stolt"; "a non-uniform FFT (NUFFT) approach employing fast
Gaussian gridding (FGG) ... for the Fourier transforms and Stolt
interpolation step in (14)").

TEST INFRASTRUCTURE ONLY -- never imported by the product path.

Eq. (14) resamples every filtered column F(k_x, k_y, k) onto a uniform
k_z grid (the operator S, O5 of the default path: linear pull) and then
inverse-transforms along k_z (part of O6).  Written as one operation, the
k_z part of the inverse transform is a Riemann sum over k_z; changing the
integration variable from k_z to the measured wavenumbers k turns it into a
sum over the measured samples at their NON-uniform k_z,i, which a type-1
NUFFT evaluates without interpolating:

    o_col(m) = (1/n_z) sum_{i in band} F_i w_i exp(+j (k_z,i - k_z,0) m dz),
    k_z,i = sqrt(4 k_i^2 - k_r^2)                      (Eq. (13))
    w_i   = (dk_z/dk)_i dk / dk_z = 4 k_i dk / (k_z,i dk_z)   (Jacobian)
    band  : 4 k_i^2 > k_r^2 and k_z,i >= k_z,0          (k_z,i <= 2 k_max always)

for the signed depth index m = -n_z/2 .. n_z/2 - 1 (z = z_ref + m dz, the same
window as O7), stored at m mod n_z so that O7's roll applies unchanged.  The
uniform path computes (1/n_z) sum_j O_j exp(+j (k_z,j - k_z,0) m dz) with
O_j ~ F(k_z,j): the same integral sampled on the k_z grid; w_i makes the two
sums agree (sum of w_i over one k_z bin ~ 1).  Then O6's inverse transform over
(k_y, k_x) (1/(N_x N_y)) and O7.

FGG (as oracle/nufft.py, 1-D): fine grid of R = sigma n_z cells (sigma = 2),
sample i at t_i = sigma (k_z,i - k_z,0)/dk_z cells, Gaussian
phi(t) = exp(-t^2/(2 s2)) truncated to |t| <= W = 6, s2 = W/(2 pi (1 - 1/(2 sigma)));
spread, inverse DFT of the fine grid (exp(+2 pi j l m / R)), keep the n_z
signed outputs and divide by Phi(m) = sqrt(2 pi s2) exp(-2 pi^2 s2 m^2 / R^2).
"""
from __future__ import annotations

import os

import numpy as np
import scipy.fft

from . import rma
from .nufft import SIGMA, WIDTH, fgg_params


def signed_depths(nz: int) -> np.ndarray:
    """m = -nz/2 .. nz/2 - 1 in the storage order of the uniform path: row
    q holds m = q for q < nz/2 and m = q - nz otherwise."""
    q = np.arange(nz)
    return np.where(q < nz // 2, q, q - nz)


def type1_direct(c, t, nz: int) -> np.ndarray:
    """o[q] = (1/nz) sum_i c_i exp(+2 pi j t_i m_q / nz), m_q = signed_depths(nz)[q].
    c: [M, ...]; t: [M] (real, in k_z-grid units).  The definition."""
    c = np.asarray(c, complex)
    t = np.asarray(t, float)
    E = np.exp(2j * np.pi * np.outer(signed_depths(nz), t) / nz)    # [nz, M]
    return np.tensordot(E, c, axes=(1, 0)) / nz


def type1_fgg(c, t, nz: int, sigma: int = SIGMA, width: int = WIDTH) -> np.ndarray:
    """FGG version of type1_direct (steps in the module docstring)."""
    c = np.asarray(c, complex).reshape(np.size(t), -1)
    t = np.asarray(t, float)
    s2, W = fgg_params(sigma, width)
    R = sigma * nz
    g = np.zeros((R, c.shape[1]), complex)
    ct = sigma * t
    b = np.floor(ct).astype(np.int64)
    for d in range(-W, W + 2):
        j = b + d
        w = np.exp(-(j - ct) ** 2 / (2.0 * s2)) * (np.abs(j - ct) <= W)
        np.add.at(g, j % R, w[:, None] * c)
    G = scipy.fft.ifft(g, axis=0, workers=os.cpu_count()) * R        # sum_l g_l e^{+2 pi j l m / R}
    m = signed_depths(nz)
    ph = np.sqrt(2.0 * np.pi * s2) * np.exp(-2.0 * np.pi ** 2 * s2 * m ** 2 / R ** 2)
    return G[m % R] / ph[:, None] / nz


def row_terms(geo: rma.Geometry, b: int):
    """Terms of the columns (a, b), a = 0..nx-1 of spectral row b:
    positions t [nx, nk] in k_z-grid units, Jacobian weights w [nx, nk] and
    the in-band mask ok [nx, nk] (out-of-band samples carry w = 0)."""
    k = geo.k[None, :]
    kr2 = geo.kx[:, None] * geo.kx[:, None] + geo.ky[b] * geo.ky[b]         # [nx, 1]
    q = 4.0 * k * k - kr2
    ok = q > 0.0
    kz = np.sqrt(np.where(ok, q, 1.0))
    ok &= kz >= geo.kz[0]
    dkz = 2.0 * np.pi / (geo.nz * geo.dz)
    t = np.where(ok, (kz - geo.kz[0]) / dkz, 0.0)
    w = np.where(ok, 4.0 * k * geo.dk / (kz * dkz), 0.0)
    return t, w, ok


def stolt_nufft(Fk: np.ndarray, geo: rma.Geometry, direct: bool = False) -> np.ndarray:
    """O5 + the k_z part of O6 as one type-1 NUFFT per column (reading R21).
    Fk: filtered spectrum [F, ny, nx, nk] (O4).  Returns the columns already
    transformed along z, [F, ny, nx, nz] (row m mod nz holds depth m),
    scaled 1/nz.  Vectorised over the columns of a spectral row."""
    Fr, ny, nx, nk = Fk.shape
    nz = geo.nz
    out = np.zeros((Fr, ny, nx, nz), complex)
    m = signed_depths(nz)
    s2, W = fgg_params(SIGMA, WIDTH)
    R = SIGMA * nz
    ph = np.sqrt(2.0 * np.pi * s2) * np.exp(-2.0 * np.pi ** 2 * s2 * m ** 2 / R ** 2)
    for b in range(ny):
        t, w, ok = row_terms(geo, b)
        c = Fk[:, b] * w[None]                                          # [F, nx, nk]
        if direct:
            E = np.exp(2j * np.pi * t[:, None, :] * m[None, :, None] / nz)   # [nx, nz, nk]
            out[:, b] = np.einsum("amk,fak->fam", E, c) / nz
            continue
        g = np.zeros((Fr, nx, R), complex)
        ct = SIGMA * t
        b0 = np.floor(ct).astype(np.int64)
        rows = np.broadcast_to(np.arange(nx)[:, None], ct.shape)
        for d in range(-W, W + 2):
            j = b0 + d
            wg = np.exp(-(j - ct) ** 2 / (2.0 * s2)) * (np.abs(j - ct) <= W) * ok
            for f in range(Fr):
                np.add.at(g[f], (rows, j % R), wg * c[f])
        G = scipy.fft.ifft(g, axis=-1, workers=os.cpu_count()) * R
        out[:, b] = G[:, :, m % R] / ph[None, None, :] / nz
    return out


def reconstruct_stolt_nufft(s, sc, direct: bool = False, complex_out: bool = False,
                            no_compensation: bool = False, return_stages: bool = False):
    """Whole path with the NUFFT Stolt step: O1-O4, stolt_nufft, the (k_y, k_x)
    inverse FFT of O6 (1/(N_x N_y)), O7."""
    geo = rma.geometry_of(sc)
    S = rma.fft2(rma.compensate(s, geo, no_compensation))
    Fk = rma.rma_filter(S, geo)
    Oz = stolt_nufft(Fk, geo, direct)
    o = scipy.fft.ifft2(Oz, axes=(1, 2), workers=os.cpu_count())
    img = rma.magnitude_image(o, geo, complex_out)
    if return_stages:
        return img, geo, dict(spectrum=S, filtered=Fk, zcols=Oz, volume=o)
    return img, geo
