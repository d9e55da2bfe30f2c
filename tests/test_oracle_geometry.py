"""Pins for oracle step O1/O2 (geometry decomposition and compensation).

Each pin is tied to something other than the oracle itself: values printed in
the paper (tests/golden/paper_constants.json), the exact round-trip distance of
Eq. (2), and finite differences of Eq. (22).
"""
import json
import os

import numpy as np
import pytest

import oracle
import scenes

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_constants.json")))
C0 = 299_792_458.0


def test_paper_constants():
    lam = scenes.LAMBDA_C
    assert abs(lam * 1e3 - GOLD["lambda_c_mm"]["value"]) < GOLD["lambda_c_mm"]["tol"]
    prf = 4 * 1.0 / lam / 1e3
    assert abs(prf - GOLD["prf_min_khz_1mps"]["value"]) < GOLD["prf_min_khz_1mps"]["tol"]
    f = scenes.wavenumbers(5) * C0 / (2 * np.pi)
    assert np.allclose(f[[0, -1]] / 1e9, GOLD["band_ghz"]["value"])
    tx, rx = scenes.awr1443_layout(2)
    assert np.isclose(tx[1, 1] - tx[0, 1], GOLD["tx_spacing_lambda"]["value"] * lam)
    assert np.allclose(np.diff(rx[:, 1]), GOLD["rx_spacing_lambda"]["value"] * lam)


def _decompose_simple(tx, rx, scan, z0, z_ref, pitch, npx=1, npy=1, nx=4, ny=4):
    k = scenes.wavenumbers(4)
    return oracle.decompose(np.array(tx, float), np.array(rx, float), np.array(scan, float),
                            npx, npy, 0.0, 0.0, pitch, pitch, np.array([z0]), k,
                            nx, ny, 4, 5e-3, z_ref)


def test_spec_expand_channels_example():
    g = GOLD["spec_expand_channels"]
    geo = _decompose_simple([g["tx"]], [g["rx"]], [[g["pose"]]], g["z0"], 0.3, 0.00379 / 4)
    # baseline d_x = rx - tx (Eq. (3)); midpoint on node 0; d_z = z_l - Z_0 (Eq. (4))
    d_x = g["rx"][0] - g["tx"][0]
    assert abs(d_x * 1e3 - g["d_x_mm"]) < 1e-9
    assert geo.jx[0, 0] == 0 and geo.jy[0, 0] == 0 and geo.jx_min == 0 and geo.jy_min == 0
    assert abs(geo.d_z[0, 0] * 1e3 - g["d_z_mm"]) < 1e-9


def test_spec_mimo_term():
    g = GOLD["spec_mimo_term_um"]
    d = g["d_x_mm"] * 1e-3
    geo = _decompose_simple([[-d / 2, 0, 0]], [[d / 2, 0, 0]], [[[0, 0, 0]]], 0.0, g["r_ref_m"], d / 2)
    assert abs(geo.beta_mimo[0, 0, 0] * 1e6 - g["value"]) < g["tol"]


def test_awr1443_virtual_lattice():
    """2 Tx spaced 2*lambda, 4 Rx spaced lambda/2 -> 8 distinct virtual
    elements on a lambda/4 column (brute force over all pairs)."""
    sc = scenes.make_scene("tiny")
    geo = oracle.rma.geometry_of(sc)
    mids = sorted(((sc.tx[t, 1] + sc.rx[r, 1]) / 2) for t in range(2) for r in range(4))
    assert np.allclose(np.diff(mids), scenes.LAMBDA_C / 4)
    assert sorted(geo.jy.ravel().tolist()) == list(range(8))
    assert np.all(geo.jx == 0)
    assert geo.nvy == sc.npy + 7 and geo.nvx == sc.npx


def test_off_lattice_rejected():
    with pytest.raises(ValueError):
        _decompose_simple([[0, 0, 0]], [[0.3e-3, 0, 0]], [[[0, 0, 0]]], 0.0, 0.3, 1e-3)


def _exact_R(d, xp, yp, Z0, tgt):
    """Eq. (22): exact round trip as a function of (d_x, d_y, d_z)."""
    dx_, dy_, dz_ = d
    x, y, z = tgt
    RT = np.sqrt((xp - dx_ / 2 - x) ** 2 + (yp - dy_ / 2 - y) ** 2 + (Z0 + dz_ - z) ** 2)
    RR = np.sqrt((xp + dx_ / 2 - x) ** 2 + (yp + dy_ / 2 - y) ** 2 + (Z0 + dz_ - z) ** 2)
    return RT + RR


@pytest.mark.parametrize("tgt", [(0.0, 0.0, 0.3), (0.02, -0.01, 0.25), (-0.05, 0.03, 0.45)])
def test_appendix_derivatives_finite_difference(tgt):
    """Eqs. (20)-(21), with the two typos corrected (reading R13):
    the d_z first derivative is written d/dd_y on P:673 and the Hessian (3,3)
    entry f_vv on P:654.  Central differences of Eq. (22)."""
    xp, yp, Z0 = 0.004, -0.002, 0.0
    x, y, z = tgt
    R0 = np.sqrt((xp - x) ** 2 + (yp - y) ** 2 + (Z0 - z) ** 2)
    h = 1e-5
    e = np.eye(3) * h
    f = lambda d: _exact_R(d, xp, yp, Z0, tgt)  # noqa: E731
    zero = np.zeros(3)
    grad = np.array([(f(e[i]) - f(-e[i])) / (2 * h) for i in range(3)])
    assert np.allclose(grad, [0.0, 0.0, 2 * (Z0 - z) / R0], atol=1e-8)
    H = np.empty((3, 3))
    for i in range(3):
        for j in range(3):
            H[i, j] = (f(e[i] + e[j]) - f(e[i] - e[j]) - f(-e[i] + e[j]) + f(-e[i] - e[j])) / (4 * h * h)
    Hp = np.array([
        [(1 - (xp - x) ** 2 / R0 ** 2) / (2 * R0), -(xp - x) * (yp - y) / (2 * R0 ** 3), 0.0],
        [-(xp - x) * (yp - y) / (2 * R0 ** 3), (1 - (yp - y) ** 2 / R0 ** 2) / (2 * R0), 0.0],
        [0.0, 0.0, 2 * (1 - (Z0 - z) ** 2 / R0 ** 2) / R0]])
    assert np.allclose(H, Hp, atol=2e-4 * np.abs(Hp).max())
    assert f(zero) == pytest.approx(2 * R0, rel=1e-15)


def test_quadratic_expansion_third_order():
    """Eq. (23) approximates Eq. (22) to third order: the error
    shrinks ~cubically with the displacement scale (reading R12)."""
    xp, yp, Z0 = 0.01, 0.005, 0.0
    tgt = (0.0, 0.0, 0.3)
    x, y, z = tgt
    R0 = np.sqrt((xp - x) ** 2 + (yp - y) ** 2 + (Z0 - z) ** 2)
    errs = []
    scales = [1, 0.5, 0.25, 0.125]
    for s_ in scales:
        dxx, dyy, dzz = 2 * scenes.LAMBDA_C * s_, 0.5 * scenes.LAMBDA_C * s_, 0.01 * s_
        quad = (2 * R0 + 2 * (Z0 - z) * dzz / R0 + (dxx ** 2 + dyy ** 2 + 4 * dzz ** 2) / (4 * R0)
                - (((xp - x) * dxx + (yp - y) * dyy) ** 2 + 4 * (Z0 - z) ** 2 * dzz ** 2) / (4 * R0 ** 3))
        errs.append(abs(quad - _exact_R((dxx, dyy, dzz), xp, yp, Z0, tgt)))
    slope = np.polyfit(np.log(scales), np.log(errs), 1)[0]
    assert slope >= 2.5


def test_spec_round_trip_exact():
    g = GOLD["spec_round_trip_exact_m"]
    R = (np.linalg.norm(np.subtract(g["tx"], g["target"])) + np.linalg.norm(np.subtract(g["rx"], g["target"])))
    assert abs(R - g["value"]) < g["tol"]


def _single_scatterer_scene(jitter_z_mm, tgt_offset=(0.0, 0.0), z_t=0.25):
    sc = scenes.make_scene("tiny")
    sc = scenes.with_geometry(sc, jitter_xy=0, jitter_z=0)
    rng = np.random.default_rng(11)
    sc.scan[0, :, 2] = rng.uniform(-jitter_z_mm, jitter_z_mm, sc.n_pos) * 1e-3
    sc.z0 = sc.scan[:, :, 2].mean(axis=1)
    geo = oracle.rma.geometry_of(sc)
    X0 = sc.x0 + geo.jx_min * sc.dx
    Y0 = sc.y0 + geo.jy_min * sc.dy
    # scatterer on the axis of virtual node (8, 11)
    q = np.array([[X0 + 8 * sc.dx + tgt_offset[0], Y0 + 11 * sc.dy + tgt_offset[1], z_t]])
    sc.scat_pos = [q]
    sc.scat_amp = [np.ones(1, complex)]
    sc.noise_sigma = 0.0
    sc.z_ref = z_t
    return sc, X0, Y0, q[0]


def test_compensation_matches_exact_round_trip():
    """Pins the sign and magnitude of every term of beta (Eqs. (7), (11), (12)):
    the compensated EXACT echo (Eq. (2) distances, scenes generator) must equal
    the ideal virtual planar monostatic response exp(-j 2 k R_0) (Eq. (10),
    P:176-182) at near-axis nodes, up to the dropped higher-order terms.
    Wrong d_z sign -> ~13 rad; dropped or mis-scaled MIMO term -> ~0.1 rad."""
    sc, X0, Y0, q = _single_scatterer_scene(2.0)
    s = scenes.synthesize_cpu(sc, noise=False)
    geo = oracle.rma.geometry_of(sc)
    planar = oracle.compensate(s, geo)[0]
    vy, vx = np.meshgrid(np.arange(geo.ny), np.arange(geo.nx), indexing="ij")
    xn = X0 + vx * sc.dx
    yn = Y0 + vy * sc.dy
    R0 = np.sqrt((xn - q[0]) ** 2 + (yn - q[1]) ** 2 + (geo.z0[0] - q[2]) ** 2)
    near = (np.abs(xn - q[0]) <= 5e-3) & (np.abs(yn - q[1]) <= 5e-3)
    # nodes reached by exactly one (t,r,p): MIMO column nodes overlap, so
    # compare each pair separately via a one-pair input
    worst = 0.0
    for t in range(sc.n_tx):
        for r in range(sc.n_rx):
            one = np.zeros_like(s)
            one[:, t, r] = s[:, t, r]
            pl = oracle.compensate(one, geo)[0]
            hit = near & (np.abs(pl[..., 0]) > 0.5)
            ideal = np.exp(-2j * geo.k[None, :] * R0[hit][:, None])
            err = np.angle(pl[hit] * np.conj(ideal))
            worst = max(worst, np.abs(err).max())
            assert hit.sum() > 50
    assert worst < 0.01, worst
    assert planar.shape == (geo.ny, geo.nx, geo.k.size)


def test_no_compensation_identity_when_planar_monostatic():
    """Zero displacement + monostatic layout: beta == 0 so the compensated data
    equal the raw data placed on the lattice, bit for bit."""
    sc = scenes.with_geometry(scenes.make_scene("tiny"), jitter_xy=0, jitter_z=0,
                              layout=scenes.monostatic_layout())
    s = scenes.synthesize_cpu(sc)
    geo = oracle.rma.geometry_of(sc)
    a = oracle.compensate(s, geo)
    b = oracle.compensate(s, geo, no_compensation=True)
    assert np.array_equal(a, b)
    img1, _ = oracle.reconstruct(s, geo)
    img2, _ = oracle.reconstruct(s, geo, no_compensation=True)
    assert np.array_equal(img1, img2)


def test_compensation_preserves_magnitude_and_is_linear_in_k(tiny_scene, tiny_data):
    """|s_hat| = |s| (pure phase rotation) and the applied phase is
    linear in k through the origin."""
    geo = oracle.rma.geometry_of(tiny_scene)
    one = np.zeros_like(tiny_data)
    one[:, 1, 2] = tiny_data[:, 1, 2]
    raw = oracle.compensate(one, geo, no_compensation=True)
    cor = oracle.compensate(one, geo)
    m = np.abs(raw) > 0
    assert np.allclose(np.abs(cor[m]), np.abs(raw[m]), rtol=1e-12)
    rot = (cor[m] / raw[m]).reshape(-1, geo.k.size)
    dk = geo.k[1] - geo.k[0]
    beta_est = np.angle(rot[:, 1:] * np.conj(rot[:, :-1])).mean(axis=1) / dk
    resid = np.angle(rot * np.exp(-1j * geo.k[None, :] * beta_est[:, None]))
    assert np.abs(resid).max() < 1e-9
