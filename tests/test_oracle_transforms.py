"""Pins for oracle steps O3-O7 (FFTs, filter, Stolt, magnitude/rolls).

Pinned against brute-force DFT sums, the dispersion relation of Eq. (13)
 solved by root finding, and the flat-plate closed form.
"""
import numpy as np
import pytest
from scipy.optimize import brentq

import oracle
import scenes


def _dft_matrix(n, sign):
    j = np.arange(n)
    return np.exp(sign * 2j * np.pi * np.outer(j, j) / n)


def test_fft2_matches_bruteforce_dft():
    rng = np.random.default_rng(0)
    x = rng.normal(size=(2, 4, 8, 3)) + 1j * rng.normal(size=(2, 4, 8, 3))
    got = oracle.fft2(x)
    Wy, Wx = _dft_matrix(4, -1), _dft_matrix(8, -1)
    want = np.einsum("by,ax,fyxk->fbak", Wy, Wx, x)
    assert np.allclose(got, want, atol=1e-12)


def test_ifft3_matches_bruteforce_and_roundtrip():
    rng = np.random.default_rng(1)
    x = rng.normal(size=(1, 4, 8, 16)) + 1j * rng.normal(size=(1, 4, 8, 16))
    got = oracle.ifft3(x)
    Wy, Wx, Wz = _dft_matrix(4, +1), _dft_matrix(8, +1), _dft_matrix(16, +1)
    want = np.einsum("yb,xa,zj,fbaj->fyxz", Wy, Wx, Wz, x) / (4 * 8 * 16)
    assert np.allclose(got, want, atol=1e-12)
    # Parseval and round trip
    X = oracle.fft2(x)
    assert np.isclose(np.sum(np.abs(X) ** 2), 4 * 8 * np.sum(np.abs(x) ** 2))
    back = np.fft.ifft2(X, axes=(1, 2))
    assert np.allclose(back, x, atol=1e-12)


def _geo(nk=32, nx=16, ny=8, nz=32, dz=5e-3, z_ref=0.25, dxy=None):
    tx, rx = scenes.monostatic_layout()
    dxy = dxy or scenes.DELTA
    scan = np.zeros((1, 4 * 4, 3))
    return oracle.decompose(tx, rx, scan, 4, 4, 0.0, 0.0, dxy, dxy, np.zeros(1),
                            scenes.wavenumbers(nk), nx, ny, nz, dz, z_ref)


def _k_star(kz, kr2, lo, hi):
    """Root of the dispersion relation 4k^2 - kr^2 = kz^2 (Eq. (13))
    by bracketing -- independent of the oracle's closed-form pull."""
    return brentq(lambda k: 4 * k * k - kr2 - kz * kz, lo, hi, xtol=1e-14, rtol=1e-15)


@pytest.mark.parametrize("dz", [5e-3, 2e-3])
def test_stolt_exact_on_affine_spectra(dz):
    """Linear interpolation is exact for a spectrum affine in k: the Stolt pull
    must return alpha + gamma*k* at every in-band bin, with k* solving the
    dispersion relation (root finding), and exactly 0 elsewhere."""
    geo = _geo(dz=dz, nz=64)
    rng = np.random.default_rng(2)
    nk = geo.k.size
    al = rng.normal(size=(1, geo.ny, geo.nx, 1)) + 1j * rng.normal(size=(1, geo.ny, geo.nx, 1))
    ga = rng.normal(size=(1, geo.ny, geo.nx, 1)) + 1j * rng.normal(size=(1, geo.ny, geo.nx, 1))
    Fk = al + ga * geo.k[None, None, None, :]
    O = oracle.stolt(Fk, geo)
    kmin, kmax = geo.k[0], geo.k[-1]
    n_in = 0
    for b in range(geo.ny):
        for a in range(geo.nx):
            kr2 = geo.kx[a] ** 2 + geo.ky[b] ** 2
            for j in range(geo.nz):
                kz = geo.kz[j]
                lo_ok = kz > 0 and 4 * kmin * kmin - kr2 <= kz * kz * (1 + 1e-12)
                hi_ok = 4 * kmax * kmax - kr2 >= kz * kz * (1 - 1e-12)
                if kz > 0 and lo_ok and hi_ok:
                    ks = _k_star(kz, kr2, 0.5 * np.sqrt(max(kr2, 1e-30)), 2 * kmax)
                    want = al[0, b, a, 0] + ga[0, b, a, 0] * ks
                    assert abs(O[0, b, a, j] - want) <= 1e-9 * abs(want), (b, a, j)
                    n_in += 1
                elif kz <= 0 or 4 * kmin * kmin - kr2 > kz * kz * (1 + 1e-9) or 4 * kmax * kmax - kr2 < kz * kz * (1 - 1e-9):
                    assert O[0, b, a, j] == 0
    assert n_in > 100


def test_stolt_top_bin_in_band_at_dc():
    """k_z grid anchored at 2 k_max (reading R5): the top bin of the DC column
    maps to the last source sample (needs the band-edge epsilon, reading R9)."""
    for nk in (16, 64, 128, 256, 512):
        geo = _geo(nk=nk)
        i0, tau = oracle.stolt_index_table(geo, np.array([0]), np.array([0]))
        assert i0[0, -1] == nk - 2 and tau[0, -1] == pytest.approx(1.0, abs=1e-6)


def test_filter_evanescent_zero_and_magnitude():
    """Reading R4: H = 0 where 4k^2 <= kx^2+ky^2; elsewhere |H| = k_z (P:217
    with P(f) = 1)."""
    geo = _geo(dxy=scenes.DELTA / 2, nx=32, ny=32)   # Nyquist 2*pi/DELTA > 2 k_max
    S = np.ones((1, geo.ny, geo.nx, geo.k.size), complex)
    Fk = oracle.rma_filter(S, geo)
    kr2 = geo.kx[None, :, None] ** 2 + geo.ky[:, None, None] ** 2
    ev = 4 * geo.k[None, None, :] ** 2 <= kr2
    assert ev.any() and (~ev).any()
    assert np.all(Fk[0][ev] == 0)
    kz = np.sqrt(4 * geo.k[None, None, :] ** 2 - kr2, where=~ev, out=np.zeros(ev.shape))
    assert np.allclose(np.abs(Fk[0][~ev]), kz[~ev], rtol=1e-12)


@pytest.mark.parametrize("nz,dz", [(32, 5e-3), (64, 2.5e-3)])
def test_flat_plate_closed_form(nz, dz):
    """End-to-end closed form for O3-O7.  Monostatic array fully populating the
    FFT grid, no displacement, echo of a flat plate at range R_ref:
    s = exp(-j 2 k R_ref) at every node.  Then S is N_x N_y exp(-j 2 k R_ref) at
    DC and 0 elsewhere, F = N_x N_y * 2k (affine), and the image is constant in
    (x, y) with |o(m)| = |(1/n_z) sum_{j in band} k_z,j exp(2 pi i j m'/n_z)|,
    m' = (m - n_z/2) mod n_z (band from the dispersion relation at k_r = 0)."""
    nx = ny = 8
    tx, rx = scenes.monostatic_layout()
    k = scenes.wavenumbers(24)
    z_ref = 0.3
    scan = np.zeros((1, nx * ny, 3))
    geo = oracle.decompose(tx, rx, scan, nx, ny, 0.0, 0.0, scenes.DELTA, scenes.DELTA,
                           np.zeros(1), k, nx, ny, nz, dz, z_ref)
    s = np.broadcast_to(np.exp(-2j * k * z_ref), (1, 1, 1, nx * ny, k.size)).astype(np.complex128)
    img, _ = oracle.reconstruct(s, geo, complex_out=True)
    band = (geo.kz > 0) & (geo.kz >= 2 * k[0] * (1 - 1e-12)) & (geo.kz <= 2 * k[-1] * (1 + 1e-12))
    j = np.arange(nz)
    want = np.array([np.sum(geo.kz[band] * np.exp(2j * np.pi * j[band] * ((m - nz // 2) % nz) / nz)) / nz
                     for m in range(nz)])
    got = img[0]
    assert np.allclose(got, want[:, None, None] * np.ones((1, ny, nx)), atol=1e-9 * np.abs(want).max())
    # the plate focuses at z_ref (index n_z/2)
    assert np.argmax(np.abs(want)) == nz // 2


def test_phase_ramp_formulation_of_lattice_placement():
    """Reading R6 (modular placement): the FFT of the wrapped virtual lattice
    equals the sum over pairs of each pair's UNSHIFTED pose grid spectrum times
    the shift-theorem ramp exp(-2 pi i (a j_x/N_x + b j_y/N_y))."""
    sc = scenes.make_scene("tiny")
    sc.ny = 16                       # 16 + 7 virtual rows -> wraps 7 rows
    s = scenes.synthesize_cpu(sc)
    geo = oracle.rma.geometry_of(sc)
    assert geo.nvy > geo.ny
    got = oracle.fft2(oracle.compensate(s, geo, no_compensation=True))[0]
    a = np.arange(geo.nx)
    b = np.arange(geo.ny)
    want = np.zeros_like(got)
    for t in range(sc.n_tx):
        for r in range(sc.n_rx):
            g = np.zeros((geo.ny, geo.nx, geo.k.size), complex)
            g[:sc.npy, :sc.npx] = s[0, t, r].reshape(sc.npy, sc.npx, -1)
            ramp = np.exp(-2j * np.pi * (b[:, None] * geo.jy[t, r] / geo.ny + a[None, :] * geo.jx[t, r] / geo.nx))
            want += np.fft.fft2(g, axes=(0, 1)) * ramp[:, :, None]
    assert np.allclose(got, want, atol=1e-9 * np.abs(want).max())
