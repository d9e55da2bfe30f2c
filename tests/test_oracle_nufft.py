"""Pins for the NUFFT-mode oracle (oracle/nufft.py, the
FGG-NUFFT of P:239-242): the direct non-uniform DFT against closed forms and
numpy's FFT, the FGG algorithm against the direct sum, and the whole NUFFT
path against the RASTER path at zero in-plane jitter."""
import numpy as np
import pytest

import oracle
from oracle import nufft
import scenes


def test_direct_dft_delta_and_lattice():
    # unit value at the origin -> all-ones spectrum
    S = nufft.direct_dft2([0.0], [0.0], np.ones((1, 2)), 8, 4)
    assert np.allclose(S, 1.0, atol=1e-14)
    # integer positions -> numpy's FFT of the placed grid (positions wrap mod N)
    rng = np.random.default_rng(0)
    nx, ny = 8, 4
    u = rng.integers(-8, 16, 20).astype(float)
    v = rng.integers(-4, 8, 20).astype(float)
    c = rng.normal(size=(20, 3)) + 1j * rng.normal(size=(20, 3))
    grid = np.zeros((ny, nx, 3), complex)
    np.add.at(grid, (v.astype(int) % ny, u.astype(int) % nx), c)
    assert np.allclose(nufft.direct_dft2(u, v, c, nx, ny), np.fft.fft2(grid, axes=(0, 1)), atol=1e-11)


def test_direct_dft_single_point_is_a_phasor_plane():
    S = nufft.direct_dft2([2.3], [-1.7], np.full((1, 1), 2.0 - 1.0j), 16, 8)
    assert np.allclose(np.abs(S), abs(2.0 - 1.0j), rtol=1e-13)


def _rel(a, b):
    return np.abs(a - b).max() / np.abs(b).max()


def test_fgg_matches_direct_sum_random_points():
    rng = np.random.default_rng(1)
    nx, ny, m = 16, 32, 256
    u = rng.uniform(-3, 20, m)
    v = rng.uniform(0, 32, m)
    c = rng.normal(size=(m, 3)) + 1j * rng.normal(size=(m, 3))
    want = nufft.direct_dft2(u, v, c, nx, ny)
    assert _rel(nufft.nufft2_type1(u, v, c, nx, ny), want) <= 1e-5
    # accuracy improves with the spreading width (width monotonicity)
    e4 = _rel(nufft.nufft2_type1(u, v, c, nx, ny, width=4), want)
    e6 = _rel(nufft.nufft2_type1(u, v, c, nx, ny, width=6), want)
    assert e6 < e4 < 1e-3


def test_fgg_delta_uniform_grid_and_translation():
    nx, ny = 16, 8
    assert _rel(nufft.nufft2_type1([0.0], [0.0], np.ones((1, 1)), nx, ny), np.ones((ny, nx, 1))) <= 1e-5
    yy, xx = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    rng = np.random.default_rng(2)
    c = rng.normal(size=(nx * ny, 2)) + 1j * rng.normal(size=(nx * ny, 2))
    want = np.fft.fft2(c.reshape(ny, nx, 2), axes=(0, 1))
    assert _rel(nufft.nufft2_type1(xx.ravel(), yy.ravel(), c, nx, ny), want) <= 1e-5
    # translation: shifting every position by (du, dv) multiplies by a phase ramp
    u = rng.uniform(0, nx, 50)
    v = rng.uniform(0, ny, 50)
    c = rng.normal(size=(50, 1)) + 0j
    a0 = nufft.nufft2_type1(u, v, c, nx, ny)
    a1 = nufft.nufft2_type1(u + 0.37, v - 1.21, c, nx, ny)
    ramp = np.exp(-2j * np.pi * (nufft.signed(nx)[None, :] * 0.37 / nx - nufft.signed(ny)[:, None] * 1.21 / ny))
    assert _rel(a1, a0 * ramp[:, :, None]) <= 2e-5


def test_nufft_path_equals_raster_path_without_inplane_jitter(tiny_scene):
    """Zero in-plane jitter: the true positions ARE the lattice nodes, so the
    NUFFT spectrum equals the FFT of the RASTER placement (readings R7, R19)."""
    sc = scenes.with_geometry(tiny_scene, jitter_xy=0.0)
    s = scenes.synthesize_cpu(sc)
    S, geo = nufft.spectrum_nufft(s, sc)
    want = oracle.fft2(oracle.compensate(s, geo))
    assert _rel(S, want) <= 1e-5
    Sd, _ = nufft.spectrum_nufft(s, sc, direct=True)
    assert _rel(Sd, want) <= 1e-10


def test_fgg_spectrum_matches_direct_on_jittered_tiny(tiny_scene, tiny_data):
    S, _ = nufft.spectrum_nufft(tiny_data, tiny_scene)
    Sd, _ = nufft.spectrum_nufft(tiny_data, tiny_scene, direct=True)
    assert _rel(S, Sd) <= 1e-5


def test_nufft_focuses_inplane_jitter_better_than_raster():
    """With strong in-plane jitter (2 mm rms at 0.08 m) the RASTER placement
    (which drops it, reading R7) defocuses a point scatterer; the NUFFT
    placement restores the peak to that of the same scene without in-plane
    jitter (the purpose of P:239-242) and keeps it on its voxel."""
    sc = scenes.raster_scene(48, 48, 64, 64, 32, 32, 5e-3, 0.08, jitter_xy=2e-3, jitter_z=0.5e-3, seed=7)
    geo = oracle.rma.geometry_of(sc)
    x0, y0, z0, dx, dy, dz = geo.axes
    sc.scat_pos = [np.array([[x0 + 32 * dx, y0 + 32 * dy, z0 + 16 * dz]])]
    sc.scat_amp = [np.ones(1, complex)]
    s = scenes.synthesize_cpu(sc, noise=False)
    raster, _ = oracle.reconstruct(s, sc)
    nu, _ = nufft.reconstruct_nufft(s, sc)
    sc0 = scenes.with_geometry(sc, jitter_xy=0.0)
    ideal, _ = oracle.reconstruct(scenes.synthesize_cpu(sc0, noise=False), sc0)
    assert nu.max() > 1.5 * raster.max()
    assert abs(nu.max() / ideal.max() - 1.0) < 0.05
    assert np.unravel_index(np.argmax(nu[0]), nu[0].shape) == (16, 32, 32)
