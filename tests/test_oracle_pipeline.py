"""End-to-end pins for the oracle: point scatterers land on their voxel, the
back-projection gold standard agrees, the compensation is
what focuses jittered data (the RMA-vs-proposed contrast of P:244-245),
and the path is linear (Eq. (9) is linear in o)."""
import numpy as np
import pytest

import oracle
import scenes


def _voxel_scene(ijk, jitter_xy=0.0, jitter_z=0.0, seed=5, monostatic=False):
    """A wide-aperture raster (160 x 152 poses, ~150 mm at 0.1-0.15 m) so that
    the aperture spans many Fresnel zones (sqrt(lambda R/2) ~ 17 mm): with
    Tiny's 15 mm aperture the z point-spread function is shaped by the
    aperture edges and its argmax is not a property of the method."""
    sc = scenes.raster_scene(160, 152, 256, 256, 64, 64, 2.5e-3, 0.12, monostatic=monostatic,
                             jitter_xy=jitter_xy, jitter_z=jitter_z, seed=seed)
    geo = oracle.rma.geometry_of(sc)
    x0, y0, z0, dx, dy, dz = geo.axes
    m, iy, ix = ijk
    sc.scat_pos = [np.array([[x0 + ix * dx, y0 + iy * dy, z0 + m * dz]])]
    sc.scat_amp = [np.ones(1, complex)]
    return sc


@pytest.mark.parametrize("ijk", [(32, 128, 128), (36, 131, 123), (25, 120, 140)])
def test_single_scatterer_exact_voxel_zero_jitter(ijk):
    sc = _voxel_scene(ijk)
    s = scenes.synthesize_cpu(sc, noise=False)
    img, geo = oracle.reconstruct(s, sc)
    assert np.unravel_index(np.argmax(img[0]), img[0].shape) == ijk


@pytest.mark.parametrize("ijk", [(32, 128, 128), (36, 131, 123)])
def test_single_scatterer_with_jitter_within_one_voxel(ijk):
    sc = _voxel_scene(ijk, jitter_xy=0.5e-3, jitter_z=1e-3)
    s = scenes.synthesize_cpu(sc, noise=False)
    img, geo = oracle.reconstruct(s, sc)
    got = np.unravel_index(np.argmax(img[0]), img[0].shape)
    assert max(abs(a - b) for a, b in zip(got, ijk)) <= 1


def test_integer_shift_moves_the_peak():
    """Moving the scatterer by an integer number of voxels moves the image
    peak by exactly that many voxels."""
    for shift in (2, -3):
        b = _voxel_scene((32, 128, 128 + shift))
        ib, _ = oracle.reconstruct(scenes.synthesize_cpu(b, noise=False), b)
        assert np.unravel_index(np.argmax(ib[0]), ib[0].shape) == (32, 128, 128 + shift)


def test_zero_in_zero_out(tiny_scene):
    s = np.zeros(tiny_scene.data_shape, np.complex64)
    img, _ = oracle.reconstruct(s, tiny_scene)
    assert not img.any()


def test_superposition_complex(tiny_scene, tiny_data):
    """Linearity of the whole path (Eq. (9) linear in o)."""
    rng = np.random.default_rng(3)
    other = (rng.normal(size=tiny_data.shape) + 1j * rng.normal(size=tiny_data.shape)).astype(np.complex64)
    ia, _ = oracle.reconstruct(tiny_data, tiny_scene, complex_out=True)
    ib, _ = oracle.reconstruct(other, tiny_scene, complex_out=True)
    ic, _ = oracle.reconstruct(tiny_data.astype(complex) + 2.0 * other, tiny_scene, complex_out=True)
    assert np.allclose(ic, ia + 2.0 * ib, atol=1e-10 * np.abs(ic).max())


def test_compensation_is_what_focuses_jittered_data():
    """P:244-245 / P:586: plain RMA on multi-planar data defocuses; the
    proposed compensation restores the peak."""
    sc = _voxel_scene((32, 128, 128), jitter_z=4e-3)
    s = scenes.synthesize_cpu(sc, noise=False)
    good, _ = oracle.reconstruct(s, sc)
    bad, _ = oracle.reconstruct(s, sc, no_compensation=True)
    assert good.max() > 2.0 * bad.max()


def _slab_voxels(geo, ms):
    x0, y0, z0, dx, dy, dz = geo.axes
    m, iy, ix = np.meshgrid(ms, np.arange(geo.ny), np.arange(geo.nx), indexing="ij")
    return np.stack([x0 + ix * dx, y0 + iy * dy, z0 + m * dz], axis=-1).reshape(-1, 3)


def _bpa_slab(sc, s, geo, ms):
    txw, rxw = scenes.element_positions(sc, 0)
    vox = _slab_voxels(geo, ms)
    return np.abs(oracle.bpa(s[0], txw, rxw, sc.k, vox)).reshape(len(ms), geo.ny, geo.nx)


def test_bpa_bruteforce_single_scatterer():
    """BPA gold standard with the ACTUAL jittered positions and
    exact Eq. (2) distances, on a 9x9x5 voxel box around a point target: its
    peak and the oracle's peak agree within one voxel."""
    sc = scenes.raster_scene(64, 56, 128, 128, 32, 32, 2.5e-3, 0.10, jitter_xy=0.5e-3,
                             jitter_z=1e-3, seed=9)
    geo = oracle.rma.geometry_of(sc)
    x0, y0, z0, dx, dy, dz = geo.axes
    ijk = (17, 62, 66)
    sc.scat_pos = [np.array([[x0 + ijk[2] * dx + 0.3e-3, y0 + ijk[1] * dy - 0.2e-3, z0 + ijk[0] * dz]])]
    sc.scat_amp = [np.ones(1, complex)]
    s = scenes.synthesize_cpu(sc)
    img, geo = oracle.reconstruct(s, sc)
    ms, ys, xs = (np.arange(ijk[0] - 2, ijk[0] + 3), np.arange(ijk[1] - 4, ijk[1] + 5),
                  np.arange(ijk[2] - 4, ijk[2] + 5))
    m, iy, ix = np.meshgrid(ms, ys, xs, indexing="ij")
    vox = np.stack([x0 + ix * dx, y0 + iy * dy, z0 + m * dz], axis=-1).reshape(-1, 3)
    txw, rxw = scenes.element_positions(sc, 0)
    b = np.abs(oracle.bpa(s[0], txw, rxw, sc.k, vox)).reshape(m.shape)
    pb = np.unravel_index(np.argmax(b), b.shape)
    pr = np.unravel_index(np.argmax(img[0][np.ix_(ms, ys, xs)]), b.shape)
    assert max(abs(u - v) for u, v in zip(pb, pr)) <= 1, (pb, pr)
    assert pb == (2, 4, 4) or max(abs(u - v) for u, v in zip(pb, (2, 4, 4))) <= 1


@pytest.mark.slow
def test_bpa_bruteforce_ncc_three_scatterers_tiny(tiny_scene, tiny_data):
    """Tiny config (3 scatterers, jittered): normalised cross-correlation of the
    oracle and BPA magnitude slabs >= 0.9 (threshold is SPEC's own)."""
    img, geo = oracle.reconstruct(tiny_data, tiny_scene)
    m = geo.nz // 2            # z_ref = 0.25 = scatterer depth -> index nz/2
    ms = np.arange(m - 1, m + 2)
    b = _bpa_slab(tiny_scene, tiny_data, geo, ms)
    a = img[0, ms]
    ncc = np.sum(a * b) / np.sqrt(np.sum(a * a) * np.sum(b * b))
    assert ncc >= 0.9, ncc
