"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the
same seeded complex64 inputs.

Bar (BASELINE.json north_star): relative L2 <= 1e-4 and max normalised error
<= 1e-3 on the magnitude image; integer/index work bit-exact.  Per-stage
tolerances (fp32 FFTs of up to 512^2 points, fp32 phase in turns) are 2e-5
relative L2, derived in DESIGN.md section 7.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
import scenes  # noqa: E402
import paper_2305_02064_b200 as sar  # noqa: E402

pytestmark = pytest.mark.gpu

E2_BAR, EINF_BAR, STAGE_BAR = 1e-4, 1e-3, 2e-5


@pytest.fixture(scope="module", autouse=True)
def built():
    import __graft_entry__
    __graft_entry__.build()
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def errs(got, want):
    got = np.asarray(got, dtype=np.complex128 if np.iscomplexobj(got) else np.float64)
    d = got - want
    e2 = np.linalg.norm(d.ravel()) / max(np.linalg.norm(np.ravel(want)), 1e-300)
    einf = np.abs(d).max() / max(np.abs(want).max(), 1e-300)
    return e2, einf


def _data(sc, gpu_gen=None):
    if gpu_gen is None:
        gpu_gen = sc.n_samples * max(len(q) for q in sc.scat_pos) > 5e8
    if gpu_gen:
        from scenes import gpu as sgpu
        d = sgpu.synthesize_gpu(sc)
        return d, d.cpu().numpy()
    s = scenes.synthesize_cpu(sc)
    return torch.from_numpy(s).cuda(), s


def test_gpu_generator_matches_cpu():
    from scenes import gpu as sgpu
    for name in ("tiny", "small"):
        sc = scenes.make_scene(name)
        a = sgpu.synthesize_gpu(sc).cpu().numpy()
        b = scenes.synthesize_cpu(sc)
        e2, _ = errs(a, b)
        assert e2 < 2e-6, (name, e2)


@pytest.mark.parametrize("name", ["tiny", "small"])
def test_stage_parity(name):
    sc = scenes.make_scene(name)
    d, s = _data(sc)
    img, geo, st = oracle.reconstruct(s, sc, complex_out=True, return_stages=True)
    with sar.Plan.from_scene(sc) as plan:
        g1 = plan.debug_stage(1, d).cpu().numpy()
        g2 = plan.debug_stage(2, d).cpu().numpy()
        g3 = plan.debug_stage(3, d).cpu().numpy()
        g4 = plan.debug_stage(4, d).cpu().numpy()
    e = {k: errs(g, w) for k, g, w in (("planar", g1, st["planar"]), ("spectrum", g2, st["spectrum"]),
                                       ("stolt", g3, st["stolt"]), ("complex", g4, img))}
    for k, (e2, einf) in e.items():
        assert e2 <= STAGE_BAR, (k, e2, einf)


@pytest.mark.parametrize("kw", [dict(npx=24, npy=16, nx=32, ny=32, nk=64, nz=256, dz=2e-3, z_ref=0.25),
                                dict(npx=20, npy=12, nx=32, ny=16, nk=600, nz=512, dz=2e-3, z_ref=0.3),
                                dict(npx=30, npy=9, nx=32, ny=32, nk=40, nz=128, dz=4e-3, z_ref=0.2)],
                         ids=lambda kw: f"nz{kw['nz']}")
def test_stage_parity_k3_warp(kw):
    """Per-stage parity where K3 runs the warp-per-column kernel (n_z = 128,
    256, 512): the Stolt output before the z-IFFT and the complex image."""
    sc = _custom(**kw)
    d, s = _data(sc, gpu_gen=False)
    img, geo, st = oracle.reconstruct(s, sc, complex_out=True, return_stages=True)
    with sar.Plan.from_scene(sc) as plan:
        g3 = plan.debug_stage(3, d).cpu().numpy()
        g4 = plan.debug_stage(4, d).cpu().numpy()
    for key, g, w in (("stolt", g3, st["stolt"]), ("complex", g4, img)):
        e2, _ = errs(g, w)
        assert e2 <= STAGE_BAR, (key, e2)


def _check_e2e(sc, flags=0, gpu_gen=None, geo=None, pulse=None):
    d, s = _data(sc, gpu_gen)
    want, _ = oracle.reconstruct(s, geo if geo is not None else sc,
                                 no_compensation=bool(flags & sar.SAR_NO_COMPENSATION))
    with sar.Plan.from_scene(sc, flags=flags, pulse=pulse) as plan:
        got = plan.reconstruct(d)
        torch.cuda.synchronize()
        got = got.cpu().numpy()
    e2, einf = errs(got, want)
    assert e2 <= E2_BAR and einf <= EINF_BAR, (sc.name, e2, einf)
    return got, want, e2, einf


def _record_parity(name, e2, einf):
    """profiles/<config>_parity.json: the config's last measured GPU-vs-oracle
    errors (bench.py reports them with its line); a copy goes to gpurun_out/."""
    import json
    import os
    import time
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    rec = {"config": name, "eps2": float(e2), "epsinf": float(einf), "bar": {"eps2": E2_BAR, "epsinf": EINF_BAR},
           "source": "tests/test_gpu_parity.py (full fp64 oracle on the host, same input bytes)",
           "gpu": torch.cuda.get_device_name(0), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    for d in ("profiles", "gpurun_out"):
        path = os.path.join(root, d)
        if os.path.isdir(path):
            with open(os.path.join(path, f"{name}_parity.json"), "w") as fh:
                json.dump(rec, fh, indent=1)


@pytest.mark.parametrize("name", ["tiny", "small", "freehand", "realtime"])
def test_end_to_end(name):
    _, _, e2, einf = _check_e2e(scenes.make_scene(name))
    _record_parity(name, e2, einf)


@pytest.fixture(scope="module")
def large_case():
    """Large (configs[3]): device input and the full fp64 oracle image, computed
    once for the tests that compare against it."""
    sc = scenes.make_scene("large")
    d, s = _data(sc, True)
    want, _ = oracle.reconstruct(s, sc)
    del s
    return sc, d, want


@pytest.mark.slow
def test_end_to_end_large_bench_configuration(large_case):
    """Large (configs[3]) at full size in the launch configuration bench.py
    times (plan with SAR_PROFILE_STAGES), full oracle on the host."""
    sc, d, want = large_case
    with sar.Plan.from_scene(sc, flags=sar.SAR_PROFILE_STAGES) as plan:
        got = plan.reconstruct(d).cpu().numpy()
    e2, einf = errs(got, want)
    assert e2 <= E2_BAR and einf <= EINF_BAR, (e2, einf)
    _record_parity("large", e2, einf)


@pytest.mark.slow
def test_slab_large_g8_against_oracle(large_case):
    """The single-image slab decomposition (8 ranks emulated in this process)
    against the fp64 oracle directly, not only against the whole-image CUDA
    path."""
    from paper_2305_02064_b200 import slab
    sc, d, want = large_case
    plans = [sar.SlabPlan.from_scene(sc, rank=r, world=8) for r in range(8)]
    try:
        got = torch.full(sc.image_shape, float("nan"), device="cuda")
        slab.emulate(plans, d, got)
        got = got.cpu().numpy()
    finally:
        for p in plans:
            p.close()
    e2, einf = errs(got, want)
    assert e2 <= E2_BAR and einf <= EINF_BAR, (e2, einf)


def test_node_offsets_match_oracle():
    for name in ("tiny", "large"):
        sc = scenes.make_scene(name)
        geo = oracle.rma.geometry_of(sc)
        with sar.Plan.from_scene(sc) as plan:
            jx, jy, mx, my = plan.node_offsets()
            assert np.array_equal(jx, geo.jx) and np.array_equal(jy, geo.jy)
            assert (mx, my) == (geo.jx_min, geo.jy_min)
            assert plan.axes() == tuple(geo.axes)


@pytest.mark.parametrize("name,n_sample", [("tiny", None), ("small", None), ("freehand", 8192),
                                           ("realtime", 8192), ("large", 8192)])
def test_stolt_index_bit_exact(name, n_sample):
    """Device Stolt decisions (the code K3 runs) == oracle table, bit for bit
    in the index, to fp32 rounding in the weight.  Large: a random sample of
    columns plus the DC row/column and the Nyquist corners."""
    sc = scenes.make_scene(name)
    geo = oracle.rma.geometry_of(sc)
    b, a = np.meshgrid(np.arange(sc.ny), np.arange(sc.nx), indexing="ij")
    cols = np.stack([a.ravel(), b.ravel()], axis=1)
    if n_sample:
        rng = np.random.default_rng(0)
        pick = rng.choice(len(cols), n_sample, replace=False)
        extra = np.array([[0, 0], [sc.nx // 2, 0], [0, sc.ny // 2], [sc.nx // 2, sc.ny // 2], [1, 0], [0, 1],
                          [sc.nx - 1, sc.ny - 1]])
        cols = np.concatenate([cols[pick], extra])
    with sar.Plan.from_scene(sc) as plan:
        i0, tau = plan.stolt_index(cols)
        i0, tau = i0.cpu().numpy(), tau.cpu().numpy()
    wi, wt = oracle.stolt_index_table(geo, cols[:, 0], cols[:, 1])
    assert np.array_equal(i0, wi)
    assert np.abs(tau - wt).max() <= 1e-7
    assert (i0 >= 0).any() and (i0 < 0).any()


def _custom(npx, npy, nx, ny, nk, nz, dz, z_ref, n_frames=1, monostatic=False, n_tx=2, nsc=4, seed=0, jz=2e-3):
    sc = scenes.raster_scene(npx, npy, nx, ny, nk, nz, dz, z_ref, monostatic=monostatic, n_tx=n_tx,
                             jitter_xy=0.5e-3, jitter_z=jz, n_frames=n_frames, seed=seed)
    rng = np.random.default_rng(seed + 1)
    pos, amp = [], []
    cx = sc.x0 + npx * sc.dx / 2
    cy = sc.y0 + npy * sc.dy / 2
    for _ in range(n_frames):
        q = np.stack([cx + rng.uniform(-0.01, 0.01, nsc), cy + rng.uniform(-0.01, 0.01, nsc),
                      z_ref + rng.uniform(-0.02, 0.02, nsc)], axis=1)
        pos.append(q)
        amp.append(rng.normal(size=nsc) + 1j * rng.normal(size=nsc))
    sc.scat_pos, sc.scat_amp = pos, amp
    sc.noise_sigma = 1e-3
    sc.name = f"custom{npx}x{npy}/{nx}x{ny}x{nz}/k{nk}/F{n_frames}"
    return sc


EDGE = [
    # ragged k chunks (n_k not a multiple of 16), ragged raster, nz > n_k
    dict(npx=20, npy=13, nx=32, ny=32, nk=20, nz=64, dz=4e-3, z_ref=0.2),
    dict(npx=33, npy=7, nx=64, ny=16, nk=37, nz=16, dz=5e-3, z_ref=0.15),
    # wrap: virtual aperture taller than the grid (npy + 7 > ny)
    dict(npx=16, npy=16, nx=16, ny=16, nk=16, nz=8, dz=6e-3, z_ref=0.25),
    # minimal sizes: 2-point FFTs, 2 frequencies, single pose
    dict(npx=1, npy=1, nx=2, ny=2, nk=2, nz=2, dz=5e-3, z_ref=0.25, monostatic=True),
    dict(npx=2, npy=1, nx=2, ny=4, nk=3, nz=4, dz=5e-3, z_ref=0.25),
    # several frames with their own geometry; 3 Tx
    dict(npx=24, npy=20, nx=32, ny=32, nk=32, nz=32, dz=5e-3, z_ref=0.2, n_frames=3, n_tx=3),
    # large plane displacements (P:339 sweeps max|d_z| up to 20 cm): |dk beta|
    # beyond the K1 step-phasor bound -> exact per-sample rotation path
    dict(npx=64, npy=40, nx=64, ny=64, nk=16, nz=32, dz=5e-3, z_ref=0.45, jz=0.05),
    # maximum FFT size along x and z (1024), small elsewhere
    dict(npx=600, npy=4, nx=1024, ny=16, nk=16, nz=1024, dz=1e-3, z_ref=0.3),
    dict(npx=4, npy=700, nx=8, ny=1024, nk=24, nz=8, dz=5e-3, z_ref=0.3),
    # the maximum n_k (SAR_MAX_NK = 2048: a whole Stolt column in shared memory)
    dict(npx=8, npy=8, nx=16, ny=16, nk=2048, nz=64, dz=5e-3, z_ref=0.25),
    dict(npx=8, npy=6, nx=8, ny=8, nk=2048, nz=512, dz=2e-3, z_ref=0.25),
    # SAR_MAX_PAIRS = 64 Tx/Rx pairs (16 Tx x 4 Rx: a 64-row virtual array)
    dict(npx=16, npy=12, nx=16, ny=128, nk=16, nz=16, dz=5e-3, z_ref=0.25, n_tx=16),
    # the warp-per-column K3 (k3_warp) at every n_z it covers, n_k below / above n_z
    dict(npx=24, npy=16, nx=32, ny=32, nk=64, nz=256, dz=2e-3, z_ref=0.25),
    dict(npx=20, npy=12, nx=32, ny=16, nk=600, nz=512, dz=2e-3, z_ref=0.3),
    dict(npx=30, npy=9, nx=32, ny=32, nk=40, nz=128, dz=4e-3, z_ref=0.2),
]


@pytest.mark.parametrize("kw", EDGE, ids=lambda kw: "x".join(str(kw[k]) for k in ("npx", "npy", "nx", "ny", "nk", "nz"))
                         + ("_jz" if "jz" in kw else ""))
def test_edge_cases(kw):
    _check_e2e(_custom(**kw), gpu_gen=False)


def test_no_compensation_parity_and_contrast():
    sc = scenes.make_scene("small")
    a, _, _, _ = _check_e2e(sc, flags=sar.SAR_NO_COMPENSATION)
    b, _, _, _ = _check_e2e(sc)
    assert np.linalg.norm(a - b) / np.linalg.norm(b) > 0.05


@pytest.mark.parametrize("name", ["tiny", "freehand", "large", "realtime"])
def test_compensation_changes_every_config(name):
    """on every config the NO_COMPENSATION image (the paper's
    plain-RMA failure baseline) differs from the compensated one,
    i.e. beta is really applied (GPU vs GPU; parity of both modes is pinned
    against the oracle elsewhere)."""
    sc = scenes.make_scene(name)
    d, _ = _data(sc, gpu_gen=name in ("freehand", "large", "realtime"))
    with sar.Plan.from_scene(sc) as p0, sar.Plan.from_scene(sc, flags=sar.SAR_NO_COMPENSATION) as p1:
        a = p0.reconstruct(d)
        b = p1.reconstruct(d)
        rel = float(torch.linalg.vector_norm(a - b) / torch.linalg.vector_norm(a))
    assert rel > 0.05, rel


def test_pulse_spectrum_parity():
    sc = scenes.make_scene("tiny")
    pulse = np.exp(1j * np.linspace(0, 2, sc.n_k)) * np.linspace(1.0, 2.0, sc.n_k)
    geo = oracle.decompose(sc.tx, sc.rx, sc.scan, sc.npx, sc.npy, sc.x0, sc.y0, sc.dx, sc.dy, sc.z0, sc.k,
                           sc.nx, sc.ny, sc.nz, sc.dz_img, sc.z_ref, pulse=pulse)
    _check_e2e(sc, geo=geo, pulse=pulse)


def test_zero_input_zero_output_and_empty_frames():
    sc = scenes.make_scene("tiny")
    with sar.Plan.from_scene(sc) as plan:
        out = plan.reconstruct(torch.zeros(sc.data_shape, dtype=torch.complex64, device="cuda"))
        assert not out.any().item()
    sc0 = scenes.make_scene("tiny")
    sc0.scan = sc0.scan[:0]
    sc0.z0 = sc0.z0[:0]
    sc0.n_frames = 0
    with sar.Plan.from_scene(sc0) as plan:
        out = plan.reconstruct(torch.zeros(sc0.data_shape, dtype=torch.complex64, device="cuda"))
        assert out.numel() == 0 and plan.launches_per_call() == 0


def test_complex_output_linearity():
    sc = scenes.make_scene("tiny")
    d, _ = _data(sc)
    rng = np.random.default_rng(1)
    o = torch.from_numpy((rng.normal(size=sc.data_shape) + 1j * rng.normal(size=sc.data_shape)).astype(np.complex64)).cuda()
    with sar.Plan.from_scene(sc, flags=sar.SAR_OUTPUT_COMPLEX) as plan:
        A = plan.reconstruct(d).cpu().numpy()
        B = plan.reconstruct(o).cpu().numpy()
        Cc = plan.reconstruct(d + 2 * o).cpu().numpy()
    e2, _ = errs(Cc, A + 2 * B)
    assert e2 < 1e-5


def test_host_api_matches_device_api():
    sc = scenes.make_scene("small")
    d, s = _data(sc)
    with sar.Plan.from_scene(sc) as plan:
        dev = plan.reconstruct(d).cpu().numpy()
        host = plan.reconstruct_host(torch.from_numpy(s).pin_memory()).numpy()
    assert np.array_equal(dev, host)


def test_profiling_and_launch_count():
    sc = scenes.make_scene("small")
    d, _ = _data(sc)
    with sar.Plan.from_scene(sc, flags=sar.SAR_PROFILE_STAGES) as plan:
        assert plan.launches_per_call() == 5
        for _ in range(3):
            plan.reconstruct(d)
        ms, n = plan.profile_read()
        assert n == 3 and all(m > 0 for m in ms)
        plan.profile_reset()
        assert plan.profile_read()[1] == 0


@pytest.mark.parametrize("name,flags", [("small", 0), ("freehand", 0), ("realtime", 0),
                                        ("tiny", sar.SAR_GRID_NUFFT), ("small", sar.SAR_FORCE_PLAIN)])
def test_deterministic(name, flags):
    """No kernel has a race: repeated calls give bit-identical images (every
    kernel family: TMA rings, mbarrier hand-backs, shared tiles)."""
    sc = scenes.make_scene(name)
    d, _ = _data(sc, gpu_gen=name != "small" and name != "tiny")
    with sar.Plan.from_scene(sc, flags=flags) as plan:
        a = plan.reconstruct(d).clone()
        for _ in range(4):
            assert torch.equal(plan.reconstruct(d), a)


def test_bad_tensor_arguments():
    sc = scenes.make_scene("tiny")
    with sar.Plan.from_scene(sc) as plan:
        with pytest.raises(ValueError):
            plan.reconstruct(torch.zeros((1, 2, 4, 256, 15), dtype=torch.complex64, device="cuda"))
        with pytest.raises(TypeError):
            plan.reconstruct(torch.zeros(sc.data_shape, dtype=torch.complex64))


@pytest.mark.parametrize("name", ["small", "realtime"])
def test_non_tma_fallback_path(name):
    """The plain (non-TMA) kernels used for odd n_k / unaligned rasters are
    forced with the SAR_FORCE_PLAIN plan flag and must meet the same bar."""
    _check_e2e(scenes.make_scene(name), flags=sar.SAR_FORCE_PLAIN)


@pytest.mark.parametrize("name", ["tiny", "small", "realtime"])
def test_cuda_graph_replay_equals_direct_launches(name):
    """SAR_CUDA_GRAPH: the recorded call replays the same kernels (bit-identical
    images), and a new (data, image) pair is recorded anew."""
    sc = scenes.make_scene(name)
    d, _ = _data(sc, gpu_gen=name == "realtime")
    with sar.Plan.from_scene(sc) as p0:
        want = p0.reconstruct(d)
    with sar.Plan.from_scene(sc, flags=sar.SAR_CUDA_GRAPH) as plan:
        out = torch.empty_like(want)
        for _ in range(3):
            out.zero_()
            plan.reconstruct(d, out)
            assert torch.equal(out, want)
        d2 = d.clone()
        out2 = plan.reconstruct(d2)
        assert torch.equal(out2, want)
        # replay after the input changed in place: the graph reads the new values
        d2.mul_(2.0)
        assert torch.allclose(plan.reconstruct(d2, out2), 2.0 * want, rtol=1e-5, atol=1e-6 * float(want.max()))


def test_tma_and_plain_paths_agree():
    sc = scenes.make_scene("small")
    d, _ = _data(sc)
    with sar.Plan.from_scene(sc) as plan:
        a = plan.reconstruct(d).cpu().numpy()
    with sar.Plan.from_scene(sc, flags=sar.SAR_FORCE_PLAIN) as plan:
        b = plan.reconstruct(d).cpu().numpy()
    e2, _ = errs(a, b.astype(np.float64))
    assert e2 < 1e-5


# ---- Tx/Rx layouts with x baselines (j^x != 0; Eq. (3)) --------
def _xlayout(n_tx=2):
    """Tx along x (x = 0, 2 lambda[, 4 lambda]) and the 4 Rx along y: the
    virtual midpoints ((tx + rx)/2, Eq. (3)) span both lattice axes, j^x in
    {0, 4, 8} and j^y in {0..3}.  Every pair with j^x != 0 lands on other
    lattice columns than its pose, so K1 accumulates in the shared x-tile
    instead of registers (k1_correct_xfft_tma<N, false, *>)."""
    lam = scenes.LAMBDA_C
    tx = np.zeros((n_tx, 3))
    tx[:, 0] = [2.0 * lam * i for i in range(n_tx)]
    rx = np.zeros((4, 3))
    rx[:, 1] = [0.0, lam / 2.0, lam, 1.5 * lam]
    return tx, rx


XLAYOUT = [
    # TMA K1 with the shared accumulation tile (nx >= 64, npx % 4 == 0, even n_k), no wrap
    dict(npx=48, npy=24, nx=64, ny=32, nk=32, nz=32, dz=5e-3, z_ref=0.2),
    # x-wrap: npx + max j^x > nx, the virtual aperture wraps 8 columns (3 Tx)
    dict(npx=64, npy=24, nx=64, ny=32, nk=48, nz=32, dz=5e-3, z_ref=0.2, n_tx=3),
    # nx = 512 (the Large x-FFT tile), wrap of 4 columns, ragged last k chunk
    dict(npx=512, npy=8, nx=512, ny=16, nk=40, nz=16, dz=5e-3, z_ref=0.25),
    # the plain (non-TMA) K1: odd n_k
    dict(npx=30, npy=10, nx=32, ny=16, nk=17, nz=16, dz=5e-3, z_ref=0.2),
]


@pytest.mark.parametrize("kw", XLAYOUT, ids=lambda kw: "x".join(str(kw[k]) for k in ("npx", "npy", "nx", "nk")))
def test_x_baseline_layouts(kw):
    """Tx/Rx layouts with x baselines against the oracle, per stage (planar
    lattice, spectrum) and end to end."""
    sc = _custom(**kw)
    sc.tx, sc.rx = _xlayout(kw.get("n_tx", 2))
    info = sar.describe_scene(sc)
    assert info["jx"].max() > 0 and info["jy"].max() > 0
    d, s = _data(sc, gpu_gen=False)
    img, geo, st = oracle.reconstruct(s, sc, complex_out=True, return_stages=True)
    assert np.array_equal(geo.jx, info["jx"])
    with sar.Plan.from_scene(sc) as plan:
        g1 = plan.debug_stage(1, d).cpu().numpy()
        g2 = plan.debug_stage(2, d).cpu().numpy()
    for key, g in (("planar", g1), ("spectrum", g2)):
        e2, _ = errs(g, st[key])
        assert e2 <= STAGE_BAR, (key, e2)
    _check_e2e(sc, gpu_gen=False)
    # the shared-tile accumulation and the TMA stage hand-back are race-free:
    # repeated runs are bit-identical
    with sar.Plan.from_scene(sc) as plan:
        ref = plan.debug_stage(2, d)
        for _ in range(8):
            assert torch.equal(plan.debug_stage(2, d), ref)


# ---- 2-D single-plane images (SAR_IMAGE_2D, reading R18) -------------------
@pytest.mark.parametrize("name,planes", [("tiny", [0.25]), ("small", [0.2, 0.25, 0.3]),
                                         ("freehand", [0.30]), ("realtime", [0.25, 0.3])])
def test_plane2d_parity(name, planes):
    sc = scenes.make_scene(name)
    d, s = _data(sc)
    want, _ = oracle.reconstruct_planes(s, sc, planes)
    with sar.Plan.from_scene(sc, z_planes=planes) as plan:
        assert plan.image_shape == (sc.n_frames, len(planes), sc.ny, sc.nx)
        got = plan.reconstruct(d)
        torch.cuda.synchronize()
        got = got.cpu().numpy()
        ax = plan.axes()
    e2, einf = errs(got, want)
    assert e2 <= E2_BAR and einf <= EINF_BAR, (name, e2, einf)
    assert ax[2] == planes[0]


def test_plane2d_many_planes_and_complex():
    sc = scenes.make_scene("small")
    d, s = _data(sc)
    planes = list(np.linspace(0.19, 0.36, 8))
    want, _ = oracle.reconstruct_planes(s, sc, planes, complex_out=True)
    with sar.Plan.from_scene(sc, z_planes=planes, flags=sar.SAR_OUTPUT_COMPLEX) as plan:
        got = plan.reconstruct(d).cpu().numpy()
    e2, _ = errs(got, want)
    assert e2 <= E2_BAR


# ---- NUFFT placement (SAR_GRID_NUFFT, reading R19) -------------------------
@pytest.mark.parametrize("name", ["tiny", "small"])
def test_nufft_parity(name):
    from oracle import nufft
    sc = scenes.make_scene(name)
    d, s = _data(sc)
    S, geo = nufft.spectrum_nufft(s, sc)
    want, _ = nufft.reconstruct_nufft(s, sc)
    with sar.Plan.from_scene(sc, flags=sar.SAR_GRID_NUFFT) as plan:
        g2 = plan.debug_stage(2, d).cpu().numpy()
        got = plan.reconstruct(d)
        torch.cuda.synchronize()
        got = got.cpu().numpy()
        with pytest.raises(sar.SarError):
            plan.debug_stage(1, d)
    e2s, _ = errs(g2, S)
    assert e2s <= STAGE_BAR, e2s
    e2, einf = errs(got, want)
    assert e2 <= E2_BAR and einf <= EINF_BAR, (name, e2, einf)


@pytest.mark.parametrize("name,planes", [("small", [0.2, 0.25, 0.3]), ("tiny", [0.25])])
def test_nufft_plane2d_parity(name, planes):
    """SAR_GRID_NUFFT | SAR_IMAGE_2D: the NUFFT spectrum (reading R19) followed
    by the plane sums of reading R18 (oracle: nufft.spectrum_nufft, then the
    2-D steps O4, O5'-O7')."""
    from oracle import nufft
    sc = scenes.make_scene(name)
    d, s = _data(sc)
    S, geo = nufft.spectrum_nufft(s, sc)
    want = oracle.magnitude_planes(oracle.ifft2_planes(oracle.plane_sum(oracle.rma_filter(S, geo), geo, planes)),
                                   geo)
    with sar.Plan.from_scene(sc, flags=sar.SAR_GRID_NUFFT, z_planes=planes) as plan:
        assert plan.launches_per_call() == 6
        got = plan.reconstruct(d).cpu().numpy()
    e2, einf = errs(got, want)
    assert e2 <= E2_BAR and einf <= EINF_BAR, (name, e2, einf)


def test_nufft_equals_raster_without_inplane_jitter():
    sc = scenes.with_geometry(scenes.make_scene("small"), jitter_xy=0.0)
    d = torch.from_numpy(scenes.synthesize_cpu(sc)).cuda()
    with sar.Plan.from_scene(sc) as p0, sar.Plan.from_scene(sc, flags=sar.SAR_GRID_NUFFT) as p1:
        a = p0.reconstruct(d).cpu().numpy()
        b = p1.reconstruct(d).cpu().numpy()
    e2, _ = errs(b, a.astype(np.float64))
    assert e2 <= 2e-5


@pytest.mark.parametrize("name,flags", [("small", 0), ("realtime", 0), ("tiny", sar.SAR_OUTPUT_COMPLEX)])
def test_report_peak_equals_image_max(name, flags):
    """SAR_REPORT_PEAK: the per-frame peak recorded by the K4b epilogue is the
    maximum of the frame's magnitude image (the same fp32 values)."""
    sc = scenes.make_scene(name)
    d, _ = _data(sc, gpu_gen=name == "realtime")
    with sar.Plan.from_scene(sc, flags=flags | sar.SAR_REPORT_PEAK) as plan:
        img = plan.reconstruct(d)
        pk = plan.peaks()
    mag = img.abs() if img.is_complex() else img
    want = mag.reshape(sc.n_frames, -1).amax(dim=1).cpu().numpy()
    assert np.allclose(pk, want, rtol=2e-7, atol=0), (pk[:4], want[:4])
    with sar.Plan.from_scene(sc) as plan:
        with pytest.raises(sar.SarError):
            plan.peaks()


NUFFT_EDGE = [
    dict(npx=20, npy=13, nx=32, ny=32, nk=20, nz=64, dz=4e-3, z_ref=0.2),           # ragged raster, odd-ish k
    dict(npx=33, npy=7, nx=64, ny=16, nk=37, nz=16, dz=5e-3, z_ref=0.15),          # odd n_k, wide strip
    dict(npx=24, npy=20, nx=32, ny=32, nk=32, nz=32, dz=5e-3, z_ref=0.2, n_frames=3, n_tx=3),  # frames, wrap
    dict(npx=8, npy=6, nx=32, ny=16, nk=2048, nz=32, dz=5e-3, z_ref=0.2),          # SAR_MAX_NK: 8 k chunks
]


@pytest.mark.slow
@pytest.mark.parametrize("n_k,pairs", [(136, (1, 2)), (24, (2, 4))])
def test_nufft_freehand_geometry(n_k, pairs):
    """NUFFT placement at the Freehand geometry (BJ.configs[2]: 256 x 256
    free-hand poses, 256^2 image -> the 512^2 fine grid, the 512-point fine
    x-FFT and k2n_yfft_crop<512>), against the FGG oracle.  n_k = 136 (> 128)
    runs the 256-thread spread; the full 2 x 4 array at n_k = 24 keeps the
    oracle to ~1 minute."""
    from oracle import nufft
    sc = scenes.make_scene("freehand", n_k=n_k)
    sc.tx, sc.rx = sc.tx[:pairs[0]], sc.rx[:pairs[1]]
    d, s = _data(sc, gpu_gen=True)
    S, geo = nufft.spectrum_nufft(s, sc)
    want = oracle.magnitude_image(oracle.ifft3(oracle.stolt(oracle.rma_filter(S, geo), geo)), geo)
    with sar.Plan.from_scene(sc, flags=sar.SAR_GRID_NUFFT) as plan:
        g2 = plan.debug_stage(2, d).cpu().numpy()
        got = plan.reconstruct(d).cpu().numpy()
    e2s, _ = errs(g2, S)
    assert e2s <= STAGE_BAR, e2s
    e2, einf = errs(got, want)
    assert e2 <= E2_BAR and einf <= EINF_BAR, (n_k, e2, einf)


@pytest.mark.parametrize("kw", NUFFT_EDGE, ids=lambda kw: "x".join(str(kw[k]) for k in ("npx", "npy", "nx", "ny", "nk")))
def test_nufft_edge_cases(kw):
    from oracle import nufft
    sc = _custom(**kw)
    d, s = _data(sc, gpu_gen=False)
    want, _ = nufft.reconstruct_nufft(s, sc)
    with sar.Plan.from_scene(sc, flags=sar.SAR_GRID_NUFFT) as plan:
        got = plan.reconstruct(d).cpu().numpy()
    e2, einf = errs(got, want)
    assert e2 <= E2_BAR and einf <= EINF_BAR, (sc.name, e2, einf)


@pytest.mark.parametrize("kw,planes", [(NUFFT_EDGE[0], [0.2]), (NUFFT_EDGE[1], [0.14, 0.15, 0.16]),
                                       (NUFFT_EDGE[2], [0.19, 0.21])])
def test_plane2d_edge_cases(kw, planes):
    sc = _custom(**kw)
    d, s = _data(sc, gpu_gen=False)
    want, _ = oracle.reconstruct_planes(s, sc, planes)
    with sar.Plan.from_scene(sc, z_planes=planes) as plan:
        got = plan.reconstruct(d).cpu().numpy()
    e2, einf = errs(got, want)
    assert e2 <= E2_BAR and einf <= EINF_BAR, (sc.name, e2, einf)


# ---- single-image slab decomposition (sar_slab_*) -----
@pytest.mark.parametrize("name,world,flags", [("small", 1, 0), ("small", 2, 0), ("small", 4, 0),
                                              ("small", 2, sar.SAR_OUTPUT_COMPLEX),
                                              ("small", 2, sar.SAR_NO_COMPENSATION),
                                              ("freehand", 4, 0), ("large", 2, 0), ("large", 8, 0),
                                              ("large", 16, 0)])
def test_slab_emulated_equals_whole_image(name, world, flags):
    """All G ranks run in this process (exchanges by tensor indexing, the same
    block permutation NCCL's all_to_all_single performs -- test_multiproc.py
    checks that); every voxel comes from the same kernel code as the
    whole-image path, so the assembled image must match it bit for bit."""
    from paper_2305_02064_b200 import slab
    sc = scenes.make_scene(name)
    if name in ("freehand", "large"):
        from scenes import gpu as sgpu
        d = sgpu.synthesize_gpu(sc)
    else:
        d, _ = _data(sc)
    with sar.Plan.from_scene(sc, flags=flags) as p0:
        want = p0.reconstruct(d)
    plans = [sar.SlabPlan.from_scene(sc, rank=r, world=world, flags=flags) for r in range(world)]
    try:
        got = torch.full_like(want, float("nan")) if not (flags & sar.SAR_OUTPUT_COMPLEX) else \
            torch.full_like(want, complex(float("nan"), 0))
        slab.emulate(plans, d, got)
        owned = sorted(m for p in plans for m in p.planes())
        assert owned == list(range(sc.nz))
        torch.cuda.synchronize()
        assert torch.equal(got, want), (name, world, (got - want).abs().max().item())
    finally:
        for p in plans:
            p.close()


def test_slab_rank_writes_only_its_planes_and_errors():
    from paper_2305_02064_b200 import slab  # noqa: F401
    sc = scenes.make_scene("small")
    d, _ = _data(sc)
    with sar.SlabPlan.from_scene(sc, rank=1, world=4) as p:
        img = torch.full(p.image_shape, -1.0, device="cuda")
        s1 = p.stage1(d)
        # feed this rank its own blocks only: the planes it does not own stay -1
        s2 = p.stage2(torch.zeros(p.send1_shape, dtype=torch.complex64, device="cuda"))
        p.stage3(torch.zeros(p.send2_shape, dtype=torch.complex64, device="cuda"), img)
        torch.cuda.synchronize()
        mine = set(p.planes())
        for m in range(sc.nz):
            plane = img[0, m]
            assert bool((plane == 0).all()) if m in mine else bool((plane == -1).all())
        assert s1.shape == (4, sc.ny // 4, sc.nx // 4, sc.k.size) and s2.shape == (4, sc.ny, sc.nx // 4, sc.nz // 4)
        # the slab workspace holds only the slabs, so the whole-image entry points refuse
        assert p.workspace_bytes() == 2 * 8 * sc.ny * sc.nx * (sc.nz // 4)
        with pytest.raises(sar.SarError):
            p.reconstruct(d)
    with pytest.raises(sar.SarError):
        sar.SlabPlan.from_scene(sc, rank=0, world=3)            # 3 does not divide 128
    with pytest.raises(sar.SarError):
        sar.SlabPlan.from_scene(sc, rank=4, world=4)
    with pytest.raises(sar.SarError):
        sar.SlabPlan.from_scene(sc, rank=0, world=2, flags=sar.SAR_GRID_NUFFT)
    with pytest.raises(sar.SarError):
        sar.SlabPlan.from_scene(scenes.make_scene("realtime"), rank=0, world=2)   # 64 frames


@pytest.mark.parametrize("world", [2, 4, 8])
def test_slab_nonsquare_small_z_slots(world):
    """Slab decomposition on a non-square grid whose z-slots per rank are
    fewer than one 16-wide chunk (nz/G = 8, 4): still bit-identical."""
    from paper_2305_02064_b200 import slab
    sc = _custom(npx=40, npy=13, nx=64, ny=32, nk=24, nz=32, dz=4e-3, z_ref=0.2, n_tx=3)
    d, _ = _data(sc, gpu_gen=False)
    with sar.Plan.from_scene(sc) as p0:
        want = p0.reconstruct(d)
    plans = [sar.SlabPlan.from_scene(sc, rank=r, world=world) for r in range(world)]
    try:
        got = torch.full_like(want, float("nan"))
        slab.emulate(plans, d, got)
        torch.cuda.synchronize()
        assert torch.equal(got, want), (world, (got - want).abs().max().item())
    finally:
        for p in plans:
            p.close()


def test_slab_without_tma_equals_whole_image():
    """The slab stages on the non-TMA fallback kernels (SAR_FORCE_PLAIN)."""
    from paper_2305_02064_b200 import slab
    sc = scenes.make_scene("small")
    d, _ = _data(sc)
    with sar.Plan.from_scene(sc) as p0:
        want = p0.reconstruct(d)
    plans = [sar.SlabPlan.from_scene(sc, rank=r, world=4, flags=sar.SAR_FORCE_PLAIN) for r in range(4)]
    try:
        got = torch.full_like(want, float("nan"))
        slab.emulate(plans, d, got)
        torch.cuda.synchronize()
        e2, einf = errs(got.cpu().numpy(), want.cpu().numpy())
        assert e2 <= 1e-6 and einf <= 1e-5, (e2, einf)
    finally:
        for p in plans:
            p.close()


@pytest.mark.parametrize("world,flags", [(2, 0), (4, 0), (4, sar.SAR_NO_COMPENSATION)])
def test_slab_small_against_oracle(world, flags):
    """Small, G = 2 and 4 emulated ranks, compared with the fp64 oracle."""
    from paper_2305_02064_b200 import slab
    sc = scenes.make_scene("small")
    d, s = _data(sc)
    want, _ = oracle.reconstruct(s, sc, no_compensation=bool(flags & sar.SAR_NO_COMPENSATION))
    plans = [sar.SlabPlan.from_scene(sc, rank=r, world=world, flags=flags) for r in range(world)]
    try:
        got = torch.full(sc.image_shape, float("nan"), device="cuda")
        slab.emulate(plans, d, got)
        got = got.cpu().numpy()
    finally:
        for p in plans:
            p.close()
    e2, einf = errs(got, want)
    assert e2 <= E2_BAR and einf <= EINF_BAR, (world, e2, einf)


@pytest.mark.parametrize("name,world", [("small", 2), ("small", 4), ("large", 8)])
def test_slab_peer_stores_equal_whole_image(name, world):
    """Exchange by peer stores (sar_slab_stage_peers): every rank's pack kernel
    writes its blocks straight into the other ranks' receive buffers -- here
    all on this GPU, the same kernel writes over NVLink when the pointers are
    IPC-mapped -- and the assembled image equals the whole image bit for bit."""
    from paper_2305_02064_b200 import slab
    sc = scenes.make_scene(name)
    if name == "large":
        from scenes import gpu as sgpu
        d = sgpu.synthesize_gpu(sc)
    else:
        d, _ = _data(sc)
    with sar.Plan.from_scene(sc) as p0:
        want = p0.reconstruct(d)
    plans = [sar.SlabPlan.from_scene(sc, rank=r, world=world) for r in range(world)]
    try:
        got = torch.full_like(want, float("nan"))
        slab.emulate_peers(plans, d, got)
        torch.cuda.synchronize()
        assert torch.equal(got, want), (name, world)
    finally:
        for p in plans:
            p.close()


def _ipc_worker(rank, world, port, out):
    import os as _os
    import torch.distributed as dist
    _os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2305_02064_b200 import slab
    sc = scenes.make_scene("small")
    d = torch.from_numpy(scenes.synthesize_cpu(sc)).cuda()
    with sar.Plan.from_scene(sc) as p0:
        want = p0.reconstruct(d)
    with sar.SlabPlan.from_scene(sc, rank=rank, world=world) as p:
        recv1 = torch.empty(p.send1_shape, dtype=torch.complex64, device="cuda")
        recv2 = torch.empty(p.send2_shape, dtype=torch.complex64, device="cuda")
        peers1, keep1 = slab.open_peer_buffers(recv1)
        peers2, keep2 = slab.open_peer_buffers(recv2)
        img = torch.full_like(want, float("nan"))
        slab.reconstruct_peers(p, d, img, recv1, recv2, peers1, peers2)
        torch.cuda.synchronize()
        mine = p.planes()
        ok = bool(torch.equal(img[:, mine], want[:, mine]))
        dist.barrier()
        del keep1, keep2
    out.put((rank, ok))
    dist.barrier()
    dist.destroy_process_group()


def test_slab_peer_stores_ipc_two_processes():
    """The CUDA-IPC plumbing of the peer-store exchange (open_peer_buffers /
    reconstruct_peers) with two processes; both use this GPU (one GPU per
    gpurun call), their kernels never wait on each other (host barriers
    between the stages)."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    assert res == {0: True, 1: True}


# ---- NEAREST placement (SAR_GRID_NEAREST, reading R20) ---------------------
@pytest.mark.parametrize("name", ["tiny", "small", "freehand"])
def test_nearest_parity(name):
    """Planar lattice (stage 1, before the x-FFT) and image against the oracle
    with the NEAREST node table; Freehand's cumulative spacing puts poses
    several nodes from their raster index, with collisions and holes."""
    sc = scenes.make_scene(name)
    d, s = _data(sc)
    want, geo, st = oracle.reconstruct(s, sc, nearest=True, return_stages=True)
    with sar.Plan.from_scene(sc, flags=sar.SAR_GRID_NEAREST) as plan:
        assert plan.launches_per_call() == 5
        g1 = plan.debug_stage(1, d).cpu().numpy()
        got = plan.reconstruct(d)
        torch.cuda.synchronize()
        got = got.cpu().numpy()
    e1, _ = errs(g1, st["planar"])
    assert e1 <= STAGE_BAR, e1
    e2, einf = errs(got, want)
    assert e2 <= E2_BAR and einf <= EINF_BAR, (name, e2, einf)
    if name == "freehand":
        raster, _ = oracle.reconstruct(s, sc)
        assert errs(raster, want)[0] > 0.1    # the placements really differ here


def test_nearest_equals_raster_bitwise_on_the_lattice():
    """Every pose on its raster node: the node lists hold one row per pair in
    pair order, so NEAREST runs exactly the plain K1's arithmetic -- the
    images of the two plain paths are bit-identical."""
    sc = scenes.with_geometry(scenes.make_scene("small"), jitter_xy=0.0)
    d = torch.from_numpy(scenes.synthesize_cpu(sc)).cuda()
    fp = sar.SAR_FORCE_PLAIN
    with sar.Plan.from_scene(sc, flags=fp) as p0, sar.Plan.from_scene(sc, flags=fp | sar.SAR_GRID_NEAREST) as p1:
        assert torch.equal(p0.reconstruct(d), p1.reconstruct(d))
    with sar.Plan.from_scene(sc) as p0, sar.Plan.from_scene(sc, flags=sar.SAR_GRID_NEAREST) as p1:
        e2, _ = errs(p1.reconstruct(d).cpu().numpy(), p0.reconstruct(d).cpu().numpy().astype(np.float64))
    assert e2 <= 2e-5


NEAREST_EDGE = [
    # poses pushed 0.6..3 pitches off the raster: collisions, holes, and
    # nodes beyond the raster and below 0 (modulo the FFT grid)
    dict(npx=24, npy=16, nx=32, ny=32, nk=16, nz=16, jit=2.5e-3, seed=3),
    # odd n_k, several frames, 3 Tx, nx = 512 with the x-FFT of the Large tile
    dict(npx=500, npy=6, nx=512, ny=16, nk=13, nz=8, jit=1.5e-3, seed=4, n_tx=3, frames=2),
    # NO_COMPENSATION with NEAREST
    dict(npx=16, npy=12, nx=16, ny=16, nk=8, nz=8, jit=1e-3, seed=5, nocomp=True),
]


@pytest.mark.parametrize("kw", NEAREST_EDGE, ids=lambda kw: f"{kw['npx']}x{kw['npy']}_nk{kw['nk']}")
def test_nearest_edge_cases(kw):
    sc = scenes.raster_scene(kw["npx"], kw["npy"], kw["nx"], kw["ny"], kw["nk"], kw["nz"], 5e-3, 0.15,
                             n_tx=kw.get("n_tx", 2), jitter_xy=kw["jit"], jitter_z=1e-3,
                             n_frames=kw.get("frames", 1), seed=kw["seed"])
    rng = np.random.default_rng(kw["seed"])
    sc.scat_pos = [np.column_stack([rng.uniform(-0.01, 0.01, 3), rng.uniform(-0.01, 0.01, 3),
                                    rng.uniform(0.12, 0.18, 3)]) for _ in range(sc.n_frames)]
    sc.scat_amp = [np.ones(3, complex) for _ in range(sc.n_frames)]
    d, s = _data(sc)
    nocomp = kw.get("nocomp", False)
    flags = sar.SAR_GRID_NEAREST | (sar.SAR_NO_COMPENSATION if nocomp else 0)
    want, _ = oracle.reconstruct(s, sc, no_compensation=nocomp, nearest=True)
    ix, _ = oracle.nearest_nodes(sc.scan, sc.x0, sc.y0, sc.dx, sc.dy)
    assert ix.min() < 0 or ix.max() >= sc.npx   # nodes leave the raster
    with sar.Plan.from_scene(sc, flags=flags) as plan:
        got = plan.reconstruct(d).cpu().numpy()
    e2, einf = errs(got, want)
    assert e2 <= E2_BAR and einf <= EINF_BAR, (kw, e2, einf)


def test_nearest_deterministic_and_rejections():
    sc = scenes.make_scene("small")
    d, _ = _data(sc)
    with sar.Plan.from_scene(sc, flags=sar.SAR_GRID_NEAREST) as plan:
        a = plan.reconstruct(d).clone()
        assert torch.equal(plan.reconstruct(d), a)
    with pytest.raises(sar.SarError) as ei:
        sar.Plan.from_scene(sc, flags=sar.SAR_GRID_NEAREST | sar.SAR_GRID_NUFFT)
    assert ei.value.status == 1


# ---- NUFFT Stolt step (SAR_STOLT_NUFFT, reading R21) -----------------------
@pytest.mark.parametrize("name", ["tiny", "small", "freehand"])
def test_stolt_nufft_parity(name):
    from oracle import stolt_nufft as sn
    sc = scenes.make_scene(name)
    d, s = _data(sc)
    want, _ = sn.reconstruct_stolt_nufft(s, sc)
    with sar.Plan.from_scene(sc, flags=sar.SAR_STOLT_NUFFT) as plan:
        got = plan.reconstruct(d).cpu().numpy()
        with pytest.raises(sar.SarError):
            plan.debug_stage(3, d)
    e2, einf = errs(got, want)
    assert e2 <= E2_BAR and einf <= EINF_BAR, (name, e2, einf)


STOLT_NUFFT_EDGE = [
    # nz = 8: the fine grid (16 cells) is narrower than the Gaussian (13 cells): several images per cell
    dict(npx=16, npy=12, nx=16, ny=16, nk=13, nz=8, dz=6e-3, frames=2),
    dict(npx=12, npy=8, nx=16, ny=8, nk=40, nz=4, dz=1e-2, frames=1),
    # n_k below n_z, window deeper than the band
    dict(npx=24, npy=16, nx=32, ny=32, nk=24, nz=64, dz=3e-3, frames=1),
]


@pytest.mark.parametrize("kw", STOLT_NUFFT_EDGE, ids=lambda kw: f"nk{kw['nk']}_nz{kw['nz']}")
def test_stolt_nufft_edge_cases(kw):
    from oracle import stolt_nufft as sn
    sc = scenes.raster_scene(kw["npx"], kw["npy"], kw["nx"], kw["ny"], kw["nk"], kw["nz"], kw["dz"], 0.15,
                             jitter_xy=0.3e-3, jitter_z=1e-3, n_frames=kw["frames"], seed=9)
    rng = np.random.default_rng(9)
    sc.scat_pos = [np.column_stack([rng.uniform(-0.01, 0.01, 3), rng.uniform(-0.01, 0.01, 3),
                                    rng.uniform(0.13, 0.17, 3)]) for _ in range(sc.n_frames)]
    sc.scat_amp = [np.ones(3, complex) for _ in range(sc.n_frames)]
    d, s = _data(sc)
    want, _ = sn.reconstruct_stolt_nufft(s, sc)
    with sar.Plan.from_scene(sc, flags=sar.SAR_STOLT_NUFFT) as plan:
        got = plan.reconstruct(d).cpu().numpy()
    e2, einf = errs(got, want)
    assert e2 <= E2_BAR and einf <= EINF_BAR, (kw, e2, einf)


def test_stolt_nufft_large_agrees_with_linear_and_is_deterministic(large_case):
    """Large (the bench config): the full fp64 NUFFT-Stolt oracle is too slow
    in Python, so the GPU image is checked against the linear-pull GPU image
    (both approximate the same inversion: NCC >= 0.98, oracle property pinned
    in tests/test_oracle_stolt_nufft.py) and for determinism."""
    sc, d, want = large_case
    with sar.Plan.from_scene(sc, flags=sar.SAR_STOLT_NUFFT) as plan:
        a = plan.reconstruct(d)
        b = plan.reconstruct(d)
        assert torch.equal(a, b)
        a = a.cpu().numpy().astype(np.float64)
    ncc = float(np.sum(a * want) / (np.linalg.norm(a) * np.linalg.norm(want)))
    assert ncc >= 0.98, ncc


def test_stolt_nufft_rejections():
    sc = scenes.make_scene("tiny")
    with pytest.raises(sar.SarError) as ei:
        sar.Plan.from_scene(sc, flags=sar.SAR_STOLT_NUFFT, z_planes=[0.25])
    assert ei.value.status == 1
    import dataclasses
    with pytest.raises(sar.SarError) as ei:
        sar.Plan.from_scene(dataclasses.replace(sc, nz=1024), flags=sar.SAR_STOLT_NUFFT)
    assert ei.value.status == 3


def test_k3_ws_deterministic_and_equal_to_k3_pp():
    """The warp-specialised K3 (n_z = 512; producer, Stolt and FFT warps handing
    work on through mbarriers) on a small grid: repeated calls bit-identical,
    and equal to the oracle like every other K3 (the edge cases at n_z = 512
    above); many items per CTA so that the rings wrap many times."""
    sc = scenes.raster_scene(40, 36, 64, 64, 64, 512, 1e-3, 0.2, jitter_xy=0.3e-3, jitter_z=1e-3, seed=12)
    rng = np.random.default_rng(12)
    sc.scat_pos = [np.column_stack([rng.uniform(-0.01, 0.01, 4), rng.uniform(-0.01, 0.01, 4),
                                    rng.uniform(0.1, 0.3, 4)])]
    sc.scat_amp = [np.ones(4, complex)]
    d, s = _data(sc)
    want, _ = oracle.reconstruct(s, sc)
    with sar.Plan.from_scene(sc) as plan:
        a = plan.reconstruct(d).clone()
        for _ in range(4):
            assert torch.equal(plan.reconstruct(d), a)
    e2, einf = errs(a.cpu().numpy(), want)
    assert e2 <= E2_BAR and einf <= EINF_BAR, (e2, einf)
