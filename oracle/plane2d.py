"""Oracle for the 2-D single-plane image (the "2-D Proposed"
rows of Table I; a 2-D x-y image recovered on the known target
plane).

TEST INFRASTRUCTURE ONLY -- never imported by the product path.

Steps O1-O4 are those of the 3-D path (``oracle.rma``).  Then, instead of the
Stolt step and the k_z inverse transform, every filtered spectral column is
back-propagated from the reference plane to the chosen plane z_s and summed
over the measured frequencies (reading R18):

    O5'  P[f, s, b, a] = sum_i F[f, b, a, i] * exp(+j k_z,i (z_s - z_ref))
         with F = S k_z exp(+j k_z R_ref)/P(f) from O4, so the total phase is
         exp(+j k_z,i (z_s - Z_0)); k_z,i = sqrt(4 k_i^2 - k_x^2 - k_y^2), 0 if
         evanescent (Eq. (13))
    O6'  o[f, s] = IFT_2D over (b, a), numpy normalisation 1/(N_x N_y)
    O7'  img[f, s, iy, ix] = |o[f, s, (iy + r_y) mod N_y, (ix + r_x) mod N_x]|
         (the x/y rolls of O7; no z roll)
"""
from __future__ import annotations

import os

import numpy as np
import scipy.fft

from . import rma


def plane_sum(Fk: np.ndarray, geo: rma.Geometry, z_planes) -> np.ndarray:
    """O5': [F, ny, nx, n_k] filtered spectrum -> [F, n_s, ny, nx] plane spectra."""
    z_planes = np.atleast_1d(np.asarray(z_planes, float))
    z_ref = geo.axes[2] + (geo.nz // 2) * geo.dz
    kr2 = geo.kx[None, :] * geo.kx[None, :] + geo.ky[:, None] * geo.ky[:, None]   # [ny, nx]
    out = np.zeros((Fk.shape[0], z_planes.size, geo.ny, geo.nx), complex)
    for i in range(Fk.shape[-1]):
        q = 4.0 * geo.k[i] * geo.k[i] - kr2
        kz = np.sqrt(np.maximum(q, 0.0))
        for s, zs in enumerate(z_planes):
            out[:, s] += Fk[:, :, :, i] * np.where(q > 0, np.exp(1j * kz * (zs - z_ref)), 0.0)
    return out


def ifft2_planes(P: np.ndarray) -> np.ndarray:
    """O6': IFT_2D over (b, a), normalised 1/(N_x N_y)."""
    return scipy.fft.ifft2(P, axes=(-2, -1), workers=os.cpu_count())


def magnitude_planes(o: np.ndarray, geo: rma.Geometry, complex_out=False) -> np.ndarray:
    """O7': x/y rolls of reading R8 (no z roll)."""
    yi = (np.arange(geo.ny) + geo.roll_y) % geo.ny
    xi = (np.arange(geo.nx) + geo.roll_x) % geo.nx
    v = o[:, :, yi][:, :, :, xi]
    return v if complex_out else np.abs(v)


def reconstruct_planes(s, sc_or_geo, z_planes, no_compensation=False, complex_out=False):
    """Whole 2-D path O1-O4, O5'-O7' on the complex64 input s[F, n_tx, n_rx, P, n_k].
    Returns (image [F, n_s, ny, nx], geometry)."""
    geo = sc_or_geo if isinstance(sc_or_geo, rma.Geometry) else rma.geometry_of(sc_or_geo)
    planar = rma.compensate(s, geo, no_compensation)
    S = rma.fft2(planar)
    Fk = rma.rma_filter(S, geo)
    img = magnitude_planes(ifft2_planes(plane_sum(Fk, geo, z_planes)), geo, complex_out)
    return img, geo
