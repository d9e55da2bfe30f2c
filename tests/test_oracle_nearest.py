"""Pins for the NEAREST placement of the oracle (oracle.nearest_nodes and
oracle.compensate(..., nodes=...); reading R20, SURVEY 8(b) SAR_GRID_NEAREST;
the in-plane irregularity of P:239 snapped to the lambda/4 lattice).

What fixes it without an implementation to compare against: with the poses
on (or within half a pitch of) their raster nodes it must reduce EXACTLY to
the RASTER placement; moving every pose by whole pitches must roll the planar
lattice by the same number of nodes; a pose moved onto another pose's node
must add its samples there and leave a hole; and on a point scatterer whose
poses are jittered by more than a pitch it must focus better than RASTER
(which drops the in-plane jitter, reading R7)."""
import numpy as np

import oracle
import scenes


def _nodes(sc):
    return oracle.nearest_nodes(sc.scan, sc.x0, sc.y0, sc.dx, sc.dy)


def test_zero_inplane_jitter_is_the_raster_placement(tiny_scene):
    sc = scenes.with_geometry(tiny_scene, jitter_xy=0.0)
    s = scenes.synthesize_cpu(sc)
    geo = oracle.rma.geometry_of(sc)
    ix, iy = _nodes(sc)
    iy_r, ix_r = np.divmod(np.arange(sc.n_pos), sc.npx)
    assert np.array_equal(ix[0], ix_r) and np.array_equal(iy[0], iy_r)
    assert np.array_equal(oracle.compensate(s, geo, nodes=(ix, iy)), oracle.compensate(s, geo))


def test_sub_half_pitch_jitter_rounds_to_the_raster_node():
    # |jitter| < pitch/2 in x and y: rint (not floor / ceil) gives the raster node
    sc = scenes.raster_scene(12, 9, 16, 16, 8, 8, 5e-3, 0.1, seed=3)
    rng = np.random.default_rng(11)
    sc.scan[:, :, 0] += rng.uniform(-0.49, 0.49, sc.scan.shape[:2]) * sc.dx
    sc.scan[:, :, 1] += rng.uniform(-0.49, 0.49, sc.scan.shape[:2]) * sc.dy
    ix, iy = _nodes(sc)
    iy_r, ix_r = np.divmod(np.arange(sc.n_pos), sc.npx)
    assert np.array_equal(ix[0], ix_r) and np.array_equal(iy[0], iy_r)
    # 0.51 pitch to the right lands one node over
    sc.scan[0, 5, 0] = sc.x0 + (5 + 0.51) * sc.dx
    assert _nodes(sc)[0][0, 5] == 6


def test_whole_pitch_shift_rolls_the_lattice(tiny_scene):
    # every pose moved by (+3, -2) pitches: the planar lattice is the RASTER
    # lattice rolled by (+3, -2) nodes (mod the FFT grid, reading R6)
    sc = scenes.with_geometry(tiny_scene, jitter_xy=0.0)
    s = scenes.synthesize_cpu(sc)
    geo = oracle.rma.geometry_of(sc)
    sh = sc.scan.copy()
    sh[:, :, 0] += 3 * sc.dx
    sh[:, :, 1] -= 2 * sc.dy
    nodes = oracle.nearest_nodes(sh, sc.x0, sc.y0, sc.dx, sc.dy)
    got = oracle.compensate(s, geo, nodes=nodes)
    want = np.roll(oracle.compensate(s, geo), (-2, 3), axis=(1, 2))
    assert np.array_equal(got, want)


def test_collision_sums_and_leaves_a_hole():
    # monostatic layout: pose 7 moved onto pose 9's node adds its compensated
    # samples to node 9 and leaves node 7 empty; every other node unchanged
    sc = scenes.raster_scene(6, 4, 8, 8, 5, 8, 5e-3, 0.1, monostatic=True, jitter_z=1e-3, seed=5)
    sc.scat_pos = [np.array([[0.001, 0.002, 0.1]])]
    sc.scat_amp = [np.ones(1, complex)]
    s = scenes.synthesize_cpu(sc, noise=False)
    geo = oracle.rma.geometry_of(sc)
    raster = oracle.compensate(s, geo)
    sc2 = scenes.with_geometry(sc)
    sc2.scan[0, 7, :2] = sc.scan[0, 9, :2] + np.array([0.2, -0.3]) * sc.dx
    nodes = oracle.nearest_nodes(sc2.scan, sc.x0, sc.y0, sc.dx, sc.dy)
    got = oracle.compensate(s, geo, nodes=nodes)
    (y7, x7), (y9, x9) = divmod(7, 6), divmod(9, 6)
    want = raster.copy()
    want[0, y9, x9] = raster[0, y9, x9] + raster[0, y7, x7]
    want[0, y7, x7] = 0.0
    assert np.allclose(got, want, rtol=1e-14, atol=1e-15)
    # conservation: the sum over the lattice is the sum of the compensated samples
    assert np.allclose(got.sum(axis=(1, 2)), raster.sum(axis=(1, 2)), rtol=1e-13)


def test_nearest_focuses_large_inplane_jitter_better_than_raster():
    """In-plane jitter of 2 mm rms (> the 0.95 mm pitch): RASTER drops it and
    defocuses a point scatterer; NEAREST snaps each pose to the lattice node
    nearest its true position (residual error <= pitch/2), which restores most
    of the peak and keeps it on the scatterer's voxel."""
    sc = scenes.raster_scene(48, 48, 64, 64, 32, 32, 5e-3, 0.08, jitter_xy=2e-3, jitter_z=0.5e-3, seed=7)
    geo = oracle.rma.geometry_of(sc)
    x0, y0, z0, dx, dy, dz = geo.axes
    sc.scat_pos = [np.array([[x0 + 32 * dx, y0 + 32 * dy, z0 + 16 * dz]])]
    sc.scat_amp = [np.ones(1, complex)]
    s = scenes.synthesize_cpu(sc, noise=False)
    raster, _ = oracle.reconstruct(s, sc)
    near, _ = oracle.reconstruct(s, sc, nearest=True)
    sc0 = scenes.with_geometry(sc, jitter_xy=0.0)
    ideal, _ = oracle.reconstruct(scenes.synthesize_cpu(sc0, noise=False), sc0)
    assert near.max() > 2.0 * raster.max()
    assert near.max() > 0.9 * ideal.max()
    assert np.unravel_index(np.argmax(near[0]), near[0].shape) == (16, 32, 32)
