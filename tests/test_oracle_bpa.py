"""Pins of the back-projection oracle ``oracle.bpa`` (the paper's gold standard,
P:199-200; the matched filter of Eq. (9), with the exact
Eq. (2) distances) against values the mathematics fixes, so that a
wrong sign, a Tx/Rx or index mix-up or a dropped term fails one of them.
It is the reference the GPU BPA baseline is compared with."""
import math

import numpy as np

import oracle
import scenes


def _mini(seed=3, nk=12):
    sc = scenes.raster_scene(8, 6, 16, 16, nk, 8, 2.5e-3, 0.12, jitter_xy=0.6e-3, jitter_z=1.5e-3, seed=seed)
    txw, rxw = scenes.element_positions(sc, 0)
    return sc, txw, rxw


def test_single_sample_closed_form():
    """Data with ONE non-zero sample s[t0,r0,p0,i0] = a: o(v) = a exp(+j k_i0 (|v-T|+|v-R|)),
    evaluated here with scalar math.dist / cmath on hand-picked voxels."""
    sc, txw, rxw = _mini()
    nt, nr, P, nk = sc.data_shape[1:]
    rng = np.random.default_rng(0)
    vox = np.array([[0.01, -0.02, 0.11], [-0.03, 0.015, 0.2], [0.0, 0.0, 0.15]])
    for _ in range(4):
        t0, r0, p0, i0 = (int(rng.integers(n)) for n in (nt, nr, P, nk))
        a = complex(rng.normal(), rng.normal())
        s = np.zeros((nt, nr, P, nk), complex)
        s[t0, r0, p0, i0] = a
        got = oracle.bpa(s, txw, rxw, sc.k, vox)
        for n, v in enumerate(vox):
            R = math.dist(v, txw[t0, p0]) + math.dist(v, rxw[r0, p0])
            ph = float(sc.k[i0]) * R
            want = a * complex(math.cos(ph), math.sin(ph))
            assert abs(got[n] - want) <= 1e-9 * abs(a), (t0, r0, p0, i0, n)


def test_matched_filter_peak_equals_sample_count():
    """Noise-free unit scatterer at q (Eq. (9) without the amplitude term, as in
    BASELINE.json's recipe): every term of o(q) has phase 0, so o(q) = n_tx n_rx P n_k
    exactly, and |o(v)| < that everywhere else (triangle inequality)."""
    sc, txw, rxw = _mini(seed=5)
    q = np.array([[0.004, -0.003, 0.125]])
    sc.scat_pos = [q]
    sc.scat_amp = [np.ones(1, complex)]
    s = scenes.synthesize_cpu(sc, noise=False)[0]
    n = s.size
    vox = np.concatenate([q, q + [[1.0e-3, 0, 0]], q + [[0, 0, 2.0e-3]], q + [[0, -3.0e-3, 1.0e-3]]])
    o = oracle.bpa(s, txw, rxw, sc.k, vox)
    assert abs(o[0] - n) <= 2e-6 * n          # complex64 rounding of s only
    assert abs(o[0].imag) <= 2e-6 * n
    assert np.all(np.abs(o[1:]) < 0.999 * n)


def test_linear_and_chunk_independent():
    sc, txw, rxw = _mini(seed=7, nk=9)
    rng = np.random.default_rng(1)
    shp = sc.data_shape[1:]
    s1 = rng.normal(size=shp) + 1j * rng.normal(size=shp)
    s2 = rng.normal(size=shp) + 1j * rng.normal(size=shp)
    vox = rng.uniform([-0.03, -0.03, 0.1], [0.03, 0.03, 0.2], size=(7, 3))
    a, b = 0.3 - 1.1j, -0.7 + 0.2j
    o1, o2 = oracle.bpa(s1, txw, rxw, sc.k, vox), oracle.bpa(s2, txw, rxw, sc.k, vox)
    o12 = oracle.bpa(a * s1 + b * s2, txw, rxw, sc.k, vox)
    assert np.allclose(o12, a * o1 + b * o2, rtol=0, atol=1e-9 * np.abs(o12).max())
    oc = oracle.bpa(s1, txw, rxw, sc.k, vox, voxel_chunk=2)
    assert np.allclose(oc, o1, rtol=0, atol=1e-10 * np.abs(o1).max())


def test_direct_quadruple_loop_tiny():
    """Brute force: the literal quadruple sum with one complex exponential per
    term (no recurrence), 2 x 2 x 6 x 5 samples, 3 voxels."""
    sc = scenes.raster_scene(3, 2, 8, 8, 5, 4, 2.5e-3, 0.1, jitter_xy=0.4e-3, jitter_z=1e-3, seed=11)
    txw, rxw = scenes.element_positions(sc, 0)
    rng = np.random.default_rng(2)
    shp = sc.data_shape[1:]
    s = rng.normal(size=shp) + 1j * rng.normal(size=shp)
    vox = rng.uniform([-0.01, -0.01, 0.08], [0.01, 0.01, 0.12], size=(3, 3))
    want = np.zeros(3, complex)
    for n, v in enumerate(vox):
        for t in range(shp[0]):
            for r in range(shp[1]):
                for p in range(shp[2]):
                    R = math.dist(v, txw[t, p]) + math.dist(v, rxw[r, p])
                    for i in range(shp[3]):
                        ph = float(sc.k[i]) * R
                        want[n] += s[t, r, p, i] * complex(math.cos(ph), math.sin(ph))
    got = oracle.bpa(s, txw, rxw, sc.k, vox)
    assert np.allclose(got, want, rtol=0, atol=1e-10 * np.abs(want).max())
