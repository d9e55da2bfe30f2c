"""Oracle steps O1-O7 (see ``oracle/__init__.py``).  Plain NumPy/SciPy fp64.

TEST INFRASTRUCTURE ONLY -- never imported by the product path.
"""
from __future__ import annotations

import dataclasses
import os

import numpy as np
import scipy.fft

C0 = 299_792_458.0
# Band-edge tolerance of the Stolt pull, in samples (reading R9):
# the top k_z bin is 2*k_max by construction, so u = n_k-1 up to one rounding.
BAND_EPS = 1e-9


@dataclasses.dataclass
class Geometry:
    """Output of O1 for all frames."""

    n_frames: int
    n_tx: int
    n_rx: int
    npx: int
    npy: int
    nx: int
    ny: int
    nz: int
    dx: float
    dy: float
    dz: float
    k: np.ndarray          # [n_k]
    k0: float
    dk: float
    jx: np.ndarray         # [n_tx, n_rx] int, lattice offsets after min-subtraction
    jy: np.ndarray
    jx_min: int
    jy_min: int
    nvx: int               # virtual aperture extent (nodes)
    nvy: int
    z0: np.ndarray         # [F]
    r_ref: np.ndarray      # [F]  R_ref = z_ref - Z_0
    beta_mimo: np.ndarray  # [F, n_tx, n_rx]  (d_x^2 + d_y^2)/(4 R_ref)
    d_z: np.ndarray        # [F, P]  z_l - Z_0
    kx: np.ndarray         # [nx]
    ky: np.ndarray         # [ny]
    kz: np.ndarray         # [nz]  uniform Stolt grid
    roll_x: int
    roll_y: int
    axes: tuple            # (x_first, y_first, z_first, dx, dy, dz)
    pulse: np.ndarray      # [n_k] complex P(f)


def _pow2(n):
    return n >= 1 and (n & (n - 1)) == 0


def decompose(tx, rx, scan, npx, npy, x0, y0, dx, dy, z0, k, nx, ny, nz, dz_img, z_ref,
              pulse=None) -> Geometry:
    """O1: geometry decomposition.

    * Virtual element at the Tx/Rx midpoint, baseline d = rx - tx
      (Eq. (3)).  Midpoints must lie on the lambda/4 lattice; the
      lattice offset of pair (t,r) is j = rint(m/pitch) (reading R7: RASTER
      placement -- pose (ix,iy) is node (ix,iy), in-plane jitter dropped).
    * Plane displacement d_z = z_l - Z_0 (Eq. (4)).
    * beta = -2 d_z + (d_x^2 + d_y^2)/(4 R_ref), R_ref = z_ref - Z_0
      (Eq. (7) P:149-153 / Eq. (12) P:189-191 in the world frame with the scene
      on the +z side of the reference plane -- reading R1).
    * k_x[a] = 2*pi*a_s/(N_x*dx) with a_s the signed FFT index (numpy
      convention, reading R2); k_z grid (reading R5).
    """
    tx = np.asarray(tx, float)
    rx = np.asarray(rx, float)
    scan = np.asarray(scan, float)
    k = np.asarray(k, float)
    F = scan.shape[0]
    nt, nr, nk = tx.shape[0], rx.shape[0], k.shape[0]
    if not (_pow2(nx) and _pow2(ny) and _pow2(nz)):
        raise ValueError("nx, ny, nz must be powers of two")
    if npx > nx or npy > ny:
        raise ValueError("raster larger than the FFT grid")
    if nk < 2:
        raise ValueError("need at least two frequencies")
    # O0: uniform k grid
    k0 = float(k[0])
    dk = (k[nk - 1] - k[0]) / (nk - 1)
    if np.max(np.abs(k - (k0 + np.arange(nk) * dk))) > 1e-9 * k0:
        raise ValueError("k grid not uniform")
    # Eq. (3): midpoint and baseline of every pair
    mid = (tx[:, None, :] + rx[None, :, :]) / 2.0        # [nt, nr, 3]
    base = rx[None, :, :] - tx[:, None, :]               # [nt, nr, 3]
    if np.any(tx[:, None, 2] != rx[None, :, 2]):
        raise ValueError("Tx and Rx must share the z plane (P:111)")
    fx = mid[..., 0] / dx
    fy = mid[..., 1] / dy
    jx_raw = np.rint(fx).astype(np.int64)
    jy_raw = np.rint(fy).astype(np.int64)
    if np.max(np.abs(fx - jx_raw)) > 1e-6 or np.max(np.abs(fy - jy_raw)) > 1e-6:
        raise ValueError("Tx/Rx midpoints are not on the virtual lattice")
    jx_min, jy_min = int(jx_raw.min()), int(jy_raw.min())
    jx = jx_raw - jx_min
    jy = jy_raw - jy_min
    nvx = npx + int(jx.max())
    nvy = npy + int(jy.max())
    # Eq. (4): Z_0 and the plane displacement of each pose
    if z0 is None:
        z0 = scan[:, :, 2].mean(axis=1)
    z0 = np.asarray(z0, float).reshape(F)
    m_z = float(tx[0, 2])
    d_z = scan[:, :, 2] + m_z - z0[:, None]              # [F, P]
    r_ref = z_ref - z0
    if np.any(r_ref <= 0):
        raise ValueError("z_ref must lie beyond the reference plane")
    # Eq. (12) MIMO term with Z_0 read as the reference range (reading R1)
    bm = (base[..., 0] * base[..., 0] + base[..., 1] * base[..., 1])   # [nt, nr]
    beta_mimo = bm[None, :, :] / (4.0 * r_ref[:, None, None])
    # wavenumber tables (reading R2: numpy FFT index convention)
    ax = np.arange(nx)
    ax = np.where(ax < nx // 2, ax, ax - nx)
    ay = np.arange(ny)
    ay = np.where(ay < ny // 2, ay, ay - ny)
    kx = 2.0 * np.pi * ax / (nx * dx)
    ky = 2.0 * np.pi * ay / (ny * dy)
    dkz = 2.0 * np.pi / (nz * dz_img)
    kz = 2.0 * k[nk - 1] - (nz - 1 - np.arange(nz)) * dkz
    # O7 rolls: aperture centre and z_ref at the index centre (reading R8)
    roll_x = nvx // 2 - nx // 2
    roll_y = nvy // 2 - ny // 2
    axes = (x0 + (jx_min + roll_x) * dx, y0 + (jy_min + roll_y) * dy,
            z_ref - (nz // 2) * dz_img, dx, dy, dz_img)
    if pulse is None:
        pulse = np.ones(nk, complex)
    return Geometry(F, nt, nr, npx, npy, nx, ny, nz, dx, dy, dz_img, k, k0, dk,
                    jx, jy, jx_min, jy_min, nvx, nvy, z0, r_ref, beta_mimo, d_z,
                    kx, ky, kz, roll_x, roll_y, axes, np.asarray(pulse, complex))


def beta(geo: Geometry, f: int, t: int, r: int) -> np.ndarray:
    """Residual path length beta_l for every pose of pair (t,r), frame f
    (Eq. (12), reading R1): beta = -2 d_z + (d_x^2+d_y^2)/(4 R_ref)."""
    return -2.0 * geo.d_z[f] + geo.beta_mimo[f, t, r]


def nearest_nodes(scan, x0, y0, dx, dy):
    """NEAREST placement (reading R20; SURVEY 8(b) SAR_GRID_NEAREST, the
    in-plane irregularity of P:239 snapped to the lambda/4 lattice instead of
    interpolated): the planar node of pose p is the lattice point nearest to
    its TRUE in-plane position,
        ix = rint((x_p - x0)/dx),  iy = rint((y_p - y0)/dy)
    (fp64, the division first, round-half-even).  Returns int64 [F, P] arrays
    (ix, iy); they may be negative or beyond the raster (placement is modulo
    the FFT grid, reading R6)."""
    scan = np.asarray(scan, float)
    ix = np.rint((scan[:, :, 0] - x0) / dx).astype(np.int64)
    iy = np.rint((scan[:, :, 1] - y0) / dy).astype(np.int64)
    return ix, iy


def compensate(s, geo: Geometry, no_compensation=False, rows_per_chunk=None, nodes=None) -> np.ndarray:
    """O2: s_hat = s * exp(+j k beta) (Eq. (11)), accumulated onto the
    virtual planar lattice (reading R6: coherent sum of every (t,r,p) landing
    on a node; placement modulo the FFT grid).  Empty nodes stay 0 (the zero
    padding).  ``nodes`` = (ix, iy) [F, P] from ``nearest_nodes`` selects the
    NEAREST placement (reading R20: several poses may land on one node, their
    samples are summed; nodes no pose reaches stay 0); default RASTER
    (pose (ix, iy) -> node (ix, iy), reading R7).  Returns complex128
    [F, ny, nx, n_k]."""
    F, nt, nr, P, nk = s.shape
    assert P == geo.npx * geo.npy
    out = np.zeros((F, geo.ny, geo.nx, nk), complex)
    iy_r, ix_r = np.divmod(np.arange(P), geo.npx)
    chunk = rows_per_chunk or max(1, (1 << 22) // max(nk, 1))
    for f in range(F):
        ix, iy = (ix_r, iy_r) if nodes is None else (nodes[0][f], nodes[1][f])
        for t in range(nt):
            for r in range(nr):
                vy = (iy + geo.jy[t, r]) % geo.ny
                vx = (ix + geo.jx[t, r]) % geo.nx
                b = np.zeros(P) if no_compensation else beta(geo, f, t, r)
                for p0 in range(0, P, chunk):
                    sl = slice(p0, p0 + chunk)
                    val = s[f, t, r, sl].astype(complex)
                    val = val * np.exp(1j * geo.k[None, :] * b[sl, None])
                    if nodes is None:
                        # nodes are distinct within one pair (npx<=nx, npy<=ny)
                        out[f, vy[sl], vx[sl]] += val
                    else:
                        # NEAREST: poses of one pair may share a node
                        np.add.at(out[f], (vy[sl], vx[sl]), val)
    return out


def fft2(planar: np.ndarray) -> np.ndarray:
    """O3: FT_2D over (y', x') (Eq. (14)); numpy sign e^{-j}, unnormalised."""
    return scipy.fft.fft2(planar, axes=(-3, -2), workers=os.cpu_count())


def rma_filter(S: np.ndarray, geo: Geometry) -> np.ndarray:
    """O4: F = S * k_z * exp(+j k_z R_ref) / P(f) on the source (kx, ky, k_i)
    grid, k_z = sqrt(4k^2 - kx^2 - ky^2) (Eq. (13); filter of P:217 with
    Z_0 -> Z_0 - z_ref, reading R2; applied before Stolt, reading R3); zero
    where 4k^2 <= kx^2 + ky^2 (evanescent, reading R4)."""
    out = np.empty_like(S)
    kr2 = geo.kx[None, :] * geo.kx[None, :] + geo.ky[:, None] * geo.ky[:, None]   # [ny, nx]
    for f in range(S.shape[0]):
        for i in range(S.shape[-1]):
            q = 4.0 * geo.k[i] * geo.k[i] - kr2
            kz = np.sqrt(np.maximum(q, 0.0))
            H = np.where(q > 0, kz * np.exp(1j * kz * geo.r_ref[f]) / geo.pulse[i], 0.0)
            out[f, :, :, i] = S[f, :, :, i] * H
    return out


def stolt_index_table(geo: Geometry, a: np.ndarray, b: np.ndarray):
    """Stolt pull indices for columns (a[c], b[c]) at every output bin j
    (reading R4/R5/R9).  Returns (i0 [C, nz] int64 with -1 = zero, tau [C, nz]).

    Operation order (fp64, no fused multiply-add):
        kr2 = kx*kx + ky*ky;  ks = kz_j*kz_j + kr2;  kk = 0.5*sqrt(ks)
        u = (kk - k0)/dk;  in band iff -eps <= u <= (n_k-1)+eps and kz_j > 0
        u = clip(u, 0, n_k-1);  i0 = min(floor(u), n_k-2);  tau = u - i0
    """
    nk = geo.k.shape[0]
    kx = geo.kx[a][:, None]
    ky = geo.ky[b][:, None]
    kz = geo.kz[None, :]
    kr2 = kx * kx + ky * ky
    ks = kz * kz + kr2
    kk = 0.5 * np.sqrt(ks)
    u = (kk - geo.k0) / geo.dk
    ok = (kz > 0) & (u >= -BAND_EPS) & (u <= (nk - 1) + BAND_EPS)
    uc = np.clip(u, 0.0, nk - 1.0)
    i0 = np.minimum(np.floor(uc), nk - 2).astype(np.int64)
    tau = uc - i0
    i0 = np.where(ok, i0, -1)
    tau = np.where(ok, tau, 0.0)
    return i0, tau


def stolt(Fk: np.ndarray, geo: Geometry) -> np.ndarray:
    """O5: Stolt pull-interpolation of each (kx, ky) column from the source k
    grid onto the uniform k_z grid (operator S of Eq. (14)), linear
    in k (reading R4).  Returns complex128 [F, ny, nx, nz]."""
    Fr, ny, nx, nk = Fk.shape
    out = np.zeros((Fr, ny, nx, geo.nz), complex)
    a = np.arange(nx)
    for bb in range(ny):
        i0, tau = stolt_index_table(geo, a, np.full(nx, bb))
        ok = i0 >= 0
        i0c = np.where(ok, i0, 0)
        for f in range(Fr):
            col = Fk[f, bb]                                   # [nx, nk]
            lo = np.take_along_axis(col, i0c, axis=1)
            hi = np.take_along_axis(col, i0c + 1, axis=1)
            out[f, bb] = np.where(ok, (1.0 - tau) * lo + tau * hi, 0.0)
    return out


def ifft3(O: np.ndarray) -> np.ndarray:
    """O6: IFT_3D over (ky, kx, kz) (Eq. (14)), normalised 1/(nx ny nz)."""
    return scipy.fft.ifftn(O, axes=(-3, -2, -1), workers=os.cpu_count())


def magnitude_image(o: np.ndarray, geo: Geometry, complex_out=False) -> np.ndarray:
    """O7: img[f, m, iy, ix] = |o[f, (iy+ry) % ny, (ix+rx) % nx, (m - nz/2) % nz]|
    (reading R8).  Returns float64 [F, nz, ny, nx] (complex128 if complex_out)."""
    yi = (np.arange(geo.ny) + geo.roll_y) % geo.ny
    xi = (np.arange(geo.nx) + geo.roll_x) % geo.nx
    zi = (np.arange(geo.nz) - geo.nz // 2) % geo.nz
    v = o[:, yi][:, :, xi][:, :, :, zi]                       # [F, ny, nx, nz]
    v = np.transpose(v, (0, 3, 1, 2))
    return v if complex_out else np.abs(v)


def reconstruct(s, sc_or_geo, no_compensation=False, complex_out=False, return_stages=False, nearest=False):
    """Whole path O1..O7 for a ``scenes.Scene`` (or an explicit Geometry).

    ``s`` is the complex64 input s[F, n_tx, n_rx, P, n_k] (the same bytes the
    GPU receives).  ``nearest`` (a Scene only): NEAREST placement (reading
    R20) instead of RASTER.  Returns (image, geometry[, stages]).
    """
    geo = sc_or_geo if isinstance(sc_or_geo, Geometry) else geometry_of(sc_or_geo)
    nodes = None
    if nearest:
        sc = sc_or_geo
        nodes = nearest_nodes(sc.scan, sc.x0, sc.y0, sc.dx, sc.dy)
    planar = compensate(s, geo, no_compensation, nodes=nodes)
    S = fft2(planar)
    Fk = rma_filter(S, geo)
    O = stolt(Fk, geo)
    o = ifft3(O)
    img = magnitude_image(o, geo, complex_out)
    if return_stages:
        return img, geo, dict(planar=planar, spectrum=S, filtered=Fk, stolt=O, volume=o)
    return img, geo


def geometry_of(sc) -> Geometry:
    """O1 for a ``scenes.Scene``."""
    return decompose(sc.tx, sc.rx, sc.scan, sc.npx, sc.npy, sc.x0, sc.y0, sc.dx, sc.dy,
                     sc.z0, sc.k, sc.nx, sc.ny, sc.nz, sc.dz_img, sc.z_ref)
