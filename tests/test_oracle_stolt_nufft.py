"""Pins for the NUFFT Stolt step of the oracle (oracle/stolt_nufft.py; reading
R21).

The type-1 sum is pinned to numpy's inverse FFT on integer positions (its sign,
its 1/n_z, the signed depth order); the FGG evaluation to the direct sum; the
Jacobian weights and the sign of the z phase by point scatterers landing on
their voxel with the same peak as the linear Stolt path (a missing Jacobian
changes the level by dk_z/(2 dk) ~ 5-20x, a wrong sign mirrors the depth);
and the whole path by its agreement with the default (linear pull) image."""
import numpy as np
import pytest

import oracle
import scenes
from oracle import stolt_nufft as sn

from test_oracle_pipeline import _voxel_scene


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def test_type1_on_integer_positions_is_the_inverse_fft():
    rng = np.random.default_rng(0)
    nz = 16
    t = rng.integers(-40, 40, 25)
    c = rng.normal(size=(25, 3)) + 1j * rng.normal(size=(25, 3))
    seq = np.zeros((nz, 3), complex)
    np.add.at(seq, t % nz, c)
    want = np.fft.ifft(seq, axis=0)[sn.signed_depths(nz) % nz]
    assert np.abs(sn.type1_direct(c, t.astype(float), nz) - want).max() < 1e-14
    assert list(sn.signed_depths(8)) == [0, 1, 2, 3, -4, -3, -2, -1]


def test_fgg_matches_direct_and_improves_with_width():
    rng = np.random.default_rng(1)
    t = rng.uniform(0, 63, 200)
    c = rng.normal(size=(200, 2)) + 1j * rng.normal(size=(200, 2))
    d = sn.type1_direct(c, t, 64)
    assert _rel(sn.type1_fgg(c, t, 64), d) <= 1e-5
    assert _rel(sn.type1_fgg(c, t, 64, width=3), d) > _rel(sn.type1_fgg(c, t, 64), d)


def test_fgg_path_matches_direct_path_small():
    sc = scenes.make_scene("tiny")
    s = scenes.synthesize_cpu(sc)
    a, _ = sn.reconstruct_stolt_nufft(s, sc)
    b, _ = sn.reconstruct_stolt_nufft(s, sc, direct=True)
    assert _rel(a, b) <= 1e-5


@pytest.mark.parametrize("ijk", [(32, 128, 128), (36, 131, 123)])
def test_point_scatterer_on_its_voxel_with_the_linear_paths_peak(ijk):
    sc = _voxel_scene(ijk)
    s = scenes.synthesize_cpu(sc, noise=False)
    img, _ = sn.reconstruct_stolt_nufft(s, sc)
    lin, _ = oracle.reconstruct(s, sc)
    assert np.unravel_index(np.argmax(img[0]), img[0].shape) == ijk
    assert 0.9 < img.max() / lin.max() < 1.2


def test_agrees_with_the_linear_stolt_image():
    sc = scenes.make_scene("small")
    s = scenes.synthesize_cpu(sc)
    img, _ = sn.reconstruct_stolt_nufft(s, sc)
    lin, _ = oracle.reconstruct(s, sc)
    ncc = np.sum(img * lin) / (np.linalg.norm(img) * np.linalg.norm(lin))
    assert ncc >= 0.98
