"""Host-side tests of the C ABI (no GPU): the library loads, exports every
entry point include/sar_b200.h declares, validates its arguments, and its fp64
host decomposition (sar_plan_describe) reproduces the oracle's integer tables
and k tables bit for bit (the inputs of every index decision, reading R9)."""
import os
import re
import subprocess

import numpy as np
import pytest

import oracle
import scenes
import paper_2305_02064_b200 as sar
from paper_2305_02064_b200 import sar as sarmod

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sar_b200.h")


@pytest.fixture(scope="module", autouse=True)
def built():
    import __graft_entry__
    __graft_entry__.build()


def _declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(sar_[a-z_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    declared = _declared()
    assert len(declared) >= 15
    out = subprocess.run(["nm", "-D", "--defined-only", sar.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (sar_\w+)", out))
    missing = [d for d in declared if d not in exported]
    assert not missing, missing
    lib = sar.load_library()
    for d in declared:
        assert hasattr(lib, d)
    assert sorted(sarmod.exported_symbols()) == declared
    assert lib.sar_version() == 6


def test_library_has_no_unresolved_own_symbols():
    """Every symbol the library needs comes from libc/libstdc++/libdl (the CUDA
    runtime is linked statically): a C/C++ linkage mismatch between two
    translation units would otherwise only fail at load time on the GPU box."""
    out = subprocess.run(["nm", "-D", "--undefined-only", sar.LIB_PATH], capture_output=True, text=True).stdout
    bad = [ln.split()[-1] for ln in out.splitlines()
           if ln.strip() and not ln.strip().startswith("w ") and "@" not in ln.split()[-1]]
    assert not bad, bad


def test_no_oracle_in_product_path():
    """The product package never imports the oracle (test infrastructure)."""
    pkg = os.path.join(ROOT, "paper_2305_02064_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cpp", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, fn)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", txt, flags=re.M), fn
                assert "scipy" not in txt, fn


@pytest.mark.parametrize("name", ["tiny", "small", "freehand", "large", "realtime"])
def test_describe_matches_oracle_bit_exact(name):
    sc = scenes.make_scene(name)
    d = sar.describe_scene(sc)
    geo = oracle.rma.geometry_of(sc)
    assert np.array_equal(d["jx"], geo.jx) and np.array_equal(d["jy"], geo.jy)
    assert (d["jx_min"], d["jy_min"], d["nvx"], d["nvy"]) == (geo.jx_min, geo.jy_min, geo.nvx, geo.nvy)
    assert (d["roll_x"], d["roll_y"]) == (geo.roll_x, geo.roll_y)
    # bit-exact fp64 tables feeding the Stolt decisions
    assert np.array_equal(d["kx"], geo.kx) and np.array_equal(d["ky"], geo.ky)
    assert np.array_equal(d["kz"], geo.kz)
    assert d["k0"] == geo.k0 and d["dk"] == geo.dk
    assert d["axes"] == tuple(geo.axes)
    # fp32 beta terms: the fp64 oracle values rounded once
    bet = -2.0 * geo.d_z
    assert np.array_equal(d["apose"], bet.astype(np.float32))
    assert np.array_equal(d["bpair"], geo.beta_mimo.astype(np.float32))
    # the workspace holds one frame wave (waves are off in this build: all F frames)
    assert d["workspace_bytes"] == sc.n_frames * sc.ny * sc.nx * (sc.n_k + sc.nz) * 8


def test_describe_no_compensation_zero_beta():
    sc = scenes.make_scene("tiny")
    d = sar.describe_scene(sc, flags=sar.SAR_NO_COMPENSATION)
    assert not d["apose"].any() and not d["bpair"].any()


def _args(**over):
    sc = scenes.make_scene("tiny")
    a = dict(tx=sc.tx, rx=sc.rx, scan=sc.scan, npx=sc.npx, npy=sc.npy, x0=sc.x0, y0=sc.y0, dx=sc.dx,
             dy=sc.dy, z0=sc.z0, k=sc.k, nx=sc.nx, ny=sc.ny, nz=sc.nz, dz=sc.dz_img, z_ref=sc.z_ref)
    a.update(over)
    return a


@pytest.mark.parametrize("over,status", [
    (dict(nx=48), 1), (dict(nz=1), 1), (dict(ny=2048), 1), (dict(npx=65, nx=64), 1),
    (dict(k=scenes.wavenumbers(16)[:1]), 1), (dict(dz=0.0), 1),
    (dict(k=np.sort(np.random.default_rng(0).uniform(1600, 1700, 16))), 2),
    (dict(z_ref=-1.0), 2),
    (dict(rx=np.array([[0.0, 0.3e-3, 0.0]] * 4)), 2),
    (dict(rx=np.array([[0.0, 0.0, 1e-3]] * 4)), 2),
    (dict(tx=np.zeros((9, 3)), rx=np.zeros((8, 3))), 3),
])
def test_validation_errors(over, status):
    with pytest.raises(sar.SarError) as ei:
        sar.describe(**_args(**over))
    assert ei.value.status == status
    assert sar.load_library().sar_last_error().decode()


def test_empty_frames_describe_ok():
    sc = scenes.make_scene("tiny")
    d = sar.describe(**_args(scan=np.zeros((0, sc.n_pos, 3)), z0=np.zeros(0)))
    assert d["workspace_bytes"] == 0


def test_plan_create_without_gpu_fails_loudly():
    """No CPU fallback: without a B200 the plan refuses (UNSUPPORTED)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(sar.SarError) as ei:
        sar.Plan.from_scene(scenes.make_scene("tiny"))
    assert ei.value.status == 3


@pytest.mark.parametrize("name,n_sample", [("tiny", None), ("small", None), ("freehand", None),
                                           ("realtime", None), ("large", 8192)])
def test_stolt_ranges_cover_every_oracle_in_band_bin(name, n_sample):
    """The k_z bin range K3 evaluates per spectral column (the host class table
    it uploads, sar_plan_describe_stolt_ranges) contains every bin the oracle's
    pull puts in band (oracle.stolt_index_table, readings R5/R9), so the bins
    outside it -- and the columns the plan skips, (0, -1) -- are exactly zero
    in the oracle too.  Large: a random sample of columns plus the DC and
    Nyquist rows/columns, where the range widens to the whole axis."""
    sc = scenes.make_scene(name)
    geo = oracle.rma.geometry_of(sc)
    rng_tab = sar.describe_stolt_ranges_scene(sc)
    b, a = np.meshgrid(np.arange(sc.ny), np.arange(sc.nx), indexing="ij")
    a, b = a.ravel(), b.ravel()
    if n_sample:
        pick = np.random.default_rng(1).choice(a.size, n_sample, replace=False)
        extra_a = np.concatenate([np.arange(sc.nx), np.zeros(sc.ny, int), np.full(sc.ny, sc.nx // 2)])
        extra_b = np.concatenate([np.zeros(sc.nx, int), np.arange(sc.ny), np.arange(sc.ny)])
        a, b = np.concatenate([a[pick], extra_a]), np.concatenate([b[pick], extra_b])
    i0, _ = oracle.stolt_index_table(geo, a, b)
    lo, hi = rng_tab[b, a, 0], rng_tab[b, a, 1]
    j = np.arange(sc.nz)[None, :]
    inband = i0 >= 0
    inside = (j >= lo[:, None]) & (j <= hi[:, None])
    assert not (inband & ~inside).any(), np.argwhere(inband & ~inside)[:5]
    skipped = hi < lo
    assert not inband[skipped].any()
    # the range is a tight superset: at most 2 bins of margin on each side of
    # the in-band run (reading R9's widening), except where an edge nears k_z = 0
    live = inband.any(axis=1)
    first = np.where(live, inband.argmax(axis=1), 0)
    last = np.where(live, sc.nz - 1 - inband[:, ::-1].argmax(axis=1), 0)
    tight = live & (hi - lo < sc.nz - 1)
    assert (first[tight] - lo[tight] <= 3).all() and (hi[tight] - last[tight] <= 3).all()
    if name in ("freehand", "large", "realtime"):
        # the evanescent corners of the (k_x, k_y) plane (~18% of the columns at
        # lambda/4 sampling) and, with a shallow k_z window (Realtime), the
        # columns whose band lies below it are skipped
        frac = (rng_tab[:, :, 1] < rng_tab[:, :, 0]).mean()
        assert 0.17 < frac < 0.5, frac


@pytest.mark.parametrize("name", ["tiny", "small", "freehand", "large", "realtime"])
def test_nearest_nodes_match_oracle_bit_exact(name):
    """SAR_GRID_NEAREST node table (reading R20): the host's fp64 rint of the
    true in-plane position equals the oracle's for every pose of every frame
    (integer work, bit-exact); Freehand's cumulative spacing walks poses
    several nodes away from their raster index, which this exercises."""
    sc = scenes.make_scene(name)
    ix, iy = sar.describe_nearest_scene(sc)
    ox, oy = oracle.nearest_nodes(sc.scan, sc.x0, sc.y0, sc.dx, sc.dy)
    assert np.array_equal(ix, ox) and np.array_equal(iy, oy)
    if name == "freehand":
        iy_r, ix_r = np.divmod(np.arange(sc.n_pos), sc.npx)
        assert np.abs(ix[0] - ix_r).max() >= 3


def test_nearest_with_nufft_is_rejected():
    with pytest.raises(sar.SarError) as ei:
        sar.describe(**_args(), flags=sar.SAR_GRID_NEAREST | sar.SAR_GRID_NUFFT)
    assert ei.value.status == 1


def test_bpa_host_side_validation():
    """sar_bpa (the BPA baseline) checks its arguments on the host before it
    touches a device: an empty voxel list is a no-op, NULL buffers, a frame out
    of range and a non-uniform k are rejected with their status codes."""
    import ctypes as C
    lib = sar.load_library()
    sc = scenes.make_scene("tiny")

    def call(k=sc.k, frame=0, nvox=3, data=True, g_null=False):
        g, _, keep = sarmod._descriptors(sc.tx, sc.rx, sc.scan, sc.npx, sc.npy, 0.0, 0.0, 1.0, 1.0, None, k,
                                         2, 2, 2, 1.0, 1.0, None, 0)
        vox = np.zeros((max(nvox, 1), 3))
        dummy = np.zeros(4)
        ms = C.c_float(-1.0)
        st = lib.sar_bpa(None if g_null else C.byref(g), C.c_int32(frame),
                         C.c_void_p(dummy.ctypes.data) if data else None, C.c_void_p(vox.ctypes.data),
                         C.c_int64(nvox), C.c_void_p(dummy.ctypes.data), None, C.byref(ms))
        del keep
        return st, ms.value

    assert call(nvox=0) == (0, 0.0)
    assert call(g_null=True)[0] == 1
    assert call(frame=1)[0] == 1 and call(frame=-1)[0] == 1
    assert call(nvox=-1)[0] == 1
    assert call(data=False)[0] == 1
    kbad = sc.k.copy()
    kbad[5] *= 1.0 + 1e-6
    assert call(k=kbad)[0] == 2
    assert b"uniform" in lib.sar_last_error()
