"""Pins for the 2-D single-plane oracle (oracle/plane2d.py; SURVEY §8(f) #2,
Table I 2-D rows P:602-609, plane imaging P:394): a flat-plate closed form,
a point scatterer on its pixel, the focusing sign, back-projection brute force
on Tiny, and agreement with the 3-D path's slice on the same plane."""
import numpy as np
import pytest

import oracle
import scenes


def _ncc(a, b):
    a = np.abs(a).ravel() - np.abs(a).mean()
    b = np.abs(b).ravel() - np.abs(b).mean()
    return float(a @ b / np.linalg.norm(a) / np.linalg.norm(b))


def test_plane_flat_plate_closed_form():
    """Monostatic array filling the FFT grid, no displacement, plate echo
    s = exp(-j 2 k z_ref) (Z_0 = 0): S is N exp(-j 2k z_ref) at DC only, the
    filter at DC is 2k exp(+j 2k R_ref), so the plane image is constant in
    (x, y) and equals sum_i 2 k_i exp(+j 2 k_i (z_s - z_ref))."""
    nx = ny = 8
    tx, rx = scenes.monostatic_layout()
    k = scenes.wavenumbers(24)
    z_ref = 0.3
    scan = np.zeros((1, nx * ny, 3))
    geo = oracle.decompose(tx, rx, scan, nx, ny, 0.0, 0.0, scenes.DELTA, scenes.DELTA, np.zeros(1), k,
                           nx, ny, 16, 5e-3, z_ref)
    s = np.broadcast_to(np.exp(-2j * k * z_ref), (1, 1, 1, nx * ny, k.size)).astype(np.complex128)
    zs = np.array([z_ref, z_ref + 0.01, z_ref - 0.023])
    img, _ = oracle.reconstruct_planes(s, geo, zs, complex_out=True)
    for m, z in enumerate(zs):
        want = sum(2 * k[i] * np.exp(2j * k[i] * (z - z_ref)) for i in range(k.size))
        assert np.allclose(img[0, m], want, rtol=1e-10, atol=1e-10 * abs(want))
    # the plate focuses on its own plane
    assert np.argmax(np.abs(img[0, :, 0, 0])) == 0


def _wide_scene(ixy, z, jitter_xy=0.0, jitter_z=0.0):
    sc = scenes.raster_scene(160, 152, 256, 256, 64, 64, 2.5e-3, 0.12, jitter_xy=jitter_xy, jitter_z=jitter_z,
                             seed=5)
    geo = oracle.rma.geometry_of(sc)
    x0, y0, _, dx, dy, _ = geo.axes
    iy, ix = ixy
    sc.scat_pos = [np.array([[x0 + ix * dx, y0 + iy * dy, z]])]
    sc.scat_amp = [np.ones(1, complex)]
    return sc


@pytest.mark.parametrize("ixy,z", [((128, 128), 0.12), ((131, 123), 0.135)])
def test_plane_point_scatterer_on_its_pixel(ixy, z):
    sc = _wide_scene(ixy, z, jitter_xy=0.0, jitter_z=1e-3)
    s = scenes.synthesize_cpu(sc, noise=False)
    img, _ = oracle.reconstruct_planes(s, sc, [z])
    assert np.unravel_index(np.argmax(img[0, 0]), img[0, 0].shape) == ixy


def test_plane_focusing_sign():
    """The back-propagation phase has the right sign: the plane through the
    scatterer is brighter than planes 15 mm before or behind it."""
    z = 0.13
    sc = _wide_scene((128, 128), z)
    s = scenes.synthesize_cpu(sc, noise=False)
    img, _ = oracle.reconstruct_planes(s, sc, [z - 0.015, z, z + 0.015])
    peaks = img[0].reshape(3, -1).max(axis=1)
    assert peaks[1] > 1.5 * peaks[0] and peaks[1] > 1.5 * peaks[2]


def test_plane_matches_bpa_tiny(tiny_scene, tiny_data):
    """Back-projection brute force on the Tiny 3-point scene,
    evaluated on the same (x, y) pixels of the plane z = 0.25 m."""
    sc, s = tiny_scene, tiny_data
    img, geo = oracle.reconstruct_planes(s, sc, [0.25])
    x0, y0, _, dx, dy, _ = geo.axes
    yy, xx = np.meshgrid(y0 + dy * np.arange(sc.ny), x0 + dx * np.arange(sc.nx), indexing="ij")
    vox = np.stack([xx.ravel(), yy.ravel(), np.full(xx.size, 0.25)], axis=1)
    txw, rxw = scenes.element_positions(sc, 0)
    b = oracle.bpa(s[0], txw, rxw, sc.k, vox).reshape(sc.ny, sc.nx)
    assert _ncc(img[0, 0], b) >= 0.9


def test_plane_agrees_with_3d_slice_small():
    """On a plane of the 3-D grid the 2-D image and the 3-D path's slice (Stolt
    + k_z inverse transform) are the same physics: NCC >= 0.9."""
    sc = scenes.make_scene("small")
    s = scenes.synthesize_cpu(sc)
    img3, geo = oracle.reconstruct(s, sc)
    m = 40
    z = geo.axes[2] + m * geo.axes[5]
    img2, _ = oracle.reconstruct_planes(s, sc, [z])
    assert _ncc(img2[0, 0], img3[0, m]) >= 0.9
