"""Seeded synthetic inputs for the MIMO-SAR reconstruction path.

This package is the ONLY code shared by the CUDA path's tests/bench and the
oracle: it produces geometry (Tx/Rx layout, jittered scan positions), the
point-scatterer scene and the frequency-domain echo of Eq. (9) (PAPER.md
P:165-170, without the 1/(R_T R_R) amplitude as BASELINE.json's configs state).
It holds none of the method's arithmetic (no compensation, no FFT, no Stolt).

Workloads follow BASELINE.json ``configs[0..4]`` and the recipe in DESIGN.md
("Input recipe"):

* band 77-81 GHz, ``f = linspace(77e9, 81e9, n_k)``, ``k = 2*pi*f/c``;
* TI AWR1443 layout: 2 Tx spaced 2*lambda_c, 4 Rx spaced lambda_c/2;
  the 3-Tx Large config adds a Tx at 4*lambda_c;
* nominal raster at lambda_c/4 pitch, jittered in x/y/z;
* point targets at 0.2-0.5 m, a cut-out planar target.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional

import numpy as np

from . import rng as _rng

C0 = 299_792_458.0
F_LO, F_HI = 77e9, 81e9
F_C = 79e9
LAMBDA_C = C0 / F_C
DELTA = LAMBDA_C / 4.0  # raster / virtual lattice pitch
NOISE_SIGMA = 1e-3      # E|n|^2 = (1e-3)^2  ("N(0, 1e-3) complex noise", configs[0])


@dataclasses.dataclass
class Scene:
    """One synthetic workload (all frames).  Arrays are float64 unless noted."""

    name: str
    n_frames: int
    tx: np.ndarray          # [n_tx, 3] body frame (m)
    rx: np.ndarray          # [n_rx, 3] body frame (m)
    npx: int
    npy: int
    x0: float               # nominal raster origin / pitch (m)
    y0: float
    dx: float
    dy: float
    scan: np.ndarray        # [F, npy*npx, 3] actual (jittered) radar positions, world (m)
    z0: np.ndarray          # [F] reference plane Z_0 per frame (mean of scan z)
    k: np.ndarray           # [n_k] wavenumbers (rad/m)
    nx: int                 # image / FFT grid
    ny: int
    nz: int
    dz_img: float
    z_ref: float
    scat_pos: List[np.ndarray]    # per frame [n, 3]
    scat_amp: List[np.ndarray]    # per frame [n] complex128
    noise_key: int
    noise_sigma: float = NOISE_SIGMA

    @property
    def n_tx(self):
        return self.tx.shape[0]

    @property
    def n_rx(self):
        return self.rx.shape[0]

    @property
    def n_k(self):
        return self.k.shape[0]

    @property
    def n_pos(self):
        return self.npx * self.npy

    @property
    def n_samples(self):
        return self.n_frames * self.n_tx * self.n_rx * self.n_pos * self.n_k

    @property
    def data_shape(self):
        return (self.n_frames, self.n_tx, self.n_rx, self.n_pos, self.n_k)

    @property
    def image_shape(self):
        return (self.n_frames, self.nz, self.ny, self.nx)

    def raw_bytes(self):
        return 8 * self.n_samples

    def image_bytes(self):
        return 4 * self.n_frames * self.nz * self.ny * self.nx

    def alg_bytes(self):
        """Algorithmic bytes: every raw complex64 sample read once, every
        float32 voxel written once ('Algorithmic bytes')."""
        return self.raw_bytes() + self.image_bytes()


def wavenumbers(n_k: int) -> np.ndarray:
    f = np.linspace(F_LO, F_HI, n_k)
    return 2.0 * np.pi * f / C0


def awr1443_layout(n_tx: int = 2):
    """Tx at y = 0, 2*lambda (, 4*lambda); Rx at y = 0, lambda/2, lambda, 3*lambda/2.

    Midpoints land on 0..(4*n_tx-1)*DELTA: a contiguous lambda/4 virtual column
    (P:289 'two Tx elements spaced by 2 lambda_c and four Rx elements spaced by
    lambda_c/2')."""
    lam = LAMBDA_C
    tx = np.zeros((n_tx, 3))
    tx[:, 1] = [2.0 * lam * i for i in range(n_tx)]
    rx = np.zeros((4, 3))
    rx[:, 1] = [0.0, lam / 2.0, lam, 1.5 * lam]
    return tx, rx


def monostatic_layout():
    return np.zeros((1, 3)), np.zeros((1, 3))


def _raster_origin(npx, npy, n_virt_rows):
    x0 = -(npx // 2) * DELTA
    y0 = -((npy + n_virt_rows - 1) // 2) * DELTA
    return x0, y0


def _aperture_centre(x0, y0, npx, npy, tx, rx):
    mid = (tx[:, None, :] + rx[None, :, :]) / 2.0
    cx = x0 + (npx - 1) / 2.0 * DELTA + mid[..., 0].mean()
    cy = y0 + (npy - 1) / 2.0 * DELTA + mid[..., 1].mean()
    return cx, cy


def _nominal_xy(npx, npy, x0, y0):
    iy, ix = np.meshgrid(np.arange(npy), np.arange(npx), indexing="ij")
    return x0 + ix.ravel() * DELTA, y0 + iy.ravel() * DELTA


def _noise_key(seed: int) -> int:
    return int(_rng.splitmix64(np.array([seed * 7919 + 17], dtype=np.uint64))[0])


def make_scene(name: str, *, n_k: Optional[int] = None) -> Scene:
    """Build one of the five BASELINE.json configs by name (geometry + scene,
    no echo).  ``n_k`` may override the frequency count for test variants."""
    builders = {
        "tiny": _tiny, "small": _small, "freehand": _freehand,
        "large": _large, "realtime": _realtime,
    }
    sc = builders[name.lower()]()
    if n_k is not None:
        sc.k = wavenumbers(n_k)
    return sc


def _tiny() -> Scene:
    rng = np.random.default_rng(1)
    tx, rx = awr1443_layout(2)
    npx = npy = 16
    x0, y0 = _raster_origin(npx, npy, 8)
    nx_, ny_ = _nominal_xy(npx, npy, x0, y0)
    P = npx * npy
    scan = np.empty((1, P, 3))
    scan[0, :, 0] = nx_ + rng.normal(0, 0.5e-3, P)
    scan[0, :, 1] = ny_ + rng.normal(0, 0.5e-3, P)
    scan[0, :, 2] = rng.normal(0, 1e-3, P)
    cx, cy = _aperture_centre(x0, y0, npx, npy, tx, rx)
    pos = np.empty((3, 3))
    pos[:, 0] = cx + rng.uniform(-20e-3, 20e-3, 3)
    pos[:, 1] = cy + rng.uniform(-20e-3, 20e-3, 3)
    pos[:, 2] = 0.25
    return Scene("tiny", 1, tx, rx, npx, npy, x0, y0, DELTA, DELTA, scan,
                 scan[:, :, 2].mean(axis=1), wavenumbers(16), 64, 64, 16, 5e-3, 0.25,
                 [pos], [np.ones(3, complex)], _noise_key(1))


def _small() -> Scene:
    rng = np.random.default_rng(2)
    tx, rx = awr1443_layout(2)
    npx, npy = 64, 32
    x0, y0 = _raster_origin(npx, npy, 8)
    nx_, ny_ = _nominal_xy(npx, npy, x0, y0)
    P = npx * npy
    scan = np.empty((1, P, 3))
    scan[0, :, 0] = nx_ + rng.normal(0, 1e-3, P)
    scan[0, :, 1] = ny_ + rng.normal(0, 1e-3, P)
    scan[0, :, 2] = 3e-3 * np.sin(2 * np.pi * np.arange(P) / P) + rng.normal(0, 1e-3, P)
    cx, cy = _aperture_centre(x0, y0, npx, npy, tx, rx)
    n = 20
    pos = np.empty((n, 3))
    pos[:, 0] = cx + rng.uniform(-30e-3, 30e-3, n)
    pos[:, 1] = cy + rng.uniform(-30e-3, 30e-3, n)
    pos[:, 2] = rng.uniform(0.2, 0.35, n)
    amp = rng.uniform(0.5, 1.0, n).astype(complex)
    return Scene("small", 1, tx, rx, npx, npy, x0, y0, DELTA, DELTA, scan,
                 scan[:, :, 2].mean(axis=1), wavenumbers(64), 128, 128, 64, 5e-3, 0.275,
                 [pos], [amp], _noise_key(2))


# Cut-outs of the planar target, (x_lo, x_hi, y_lo, y_hi) in metres relative to
# the target centre (P:392 'rectangular strip with cutouts of various sizes').
_CUTOUTS = [(-0.060, -0.045, -0.035, 0.035), (-0.020, 0.000, -0.040, -0.015),
            (0.010, 0.045, 0.010, 0.022), (0.052, 0.064, -0.030, 0.040)]


def _freehand() -> Scene:
    rng = np.random.default_rng(3)
    tx, rx = awr1443_layout(2)
    npx = npy = 256
    x0, y0 = _raster_origin(npx, npy, 8)
    P = npx * npy
    # x_{l,j} = x0 + sum_{j'<j} DELTA*U(0.6,1.4); y_l = y0 + sum_{l'<l} DELTA*U(0.6,1.4)
    stepx = DELTA * rng.uniform(0.6, 1.4, (npy, npx))
    xs = x0 + np.concatenate([np.zeros((npy, 1)), np.cumsum(stepx[:, :-1], axis=1)], axis=1)
    stepy = DELTA * rng.uniform(0.6, 1.4, npy)
    ys = y0 + np.concatenate([[0.0], np.cumsum(stepy[:-1])])
    # z: random walk in raster order, step N(0, 0.5 mm), clipped to +-10 mm
    z = np.empty(P)
    zz = 0.0
    steps = rng.normal(0, 0.5e-3, P)
    for i in range(P):
        zz = min(max(zz + steps[i], -10e-3), 10e-3)
        z[i] = zz
    scan = np.empty((1, P, 3))
    scan[0, :, 0] = xs.ravel()
    scan[0, :, 1] = np.repeat(ys, npx)
    scan[0, :, 2] = z
    cx, cy = _aperture_centre(x0, y0, npx, npy, tx, rx)
    n = 2000
    pts = []
    while len(pts) < n:
        u = rng.uniform(-0.080, 0.080)
        v = rng.uniform(-0.050, 0.050)
        if any(a <= u <= b and c <= v <= d for a, b, c, d in _CUTOUTS):
            continue
        pts.append((cx + u, cy + v, 0.30))
    pos = np.array(pts)
    return Scene("freehand", 1, tx, rx, npx, npy, x0, y0, DELTA, DELTA, scan,
                 scan[:, :, 2].mean(axis=1), wavenumbers(256), 256, 256, 128, 2.5e-3, 0.30,
                 [pos], [np.ones(n, complex)], _noise_key(3))


def _large() -> Scene:
    rng = np.random.default_rng(4)
    tx, rx = awr1443_layout(3)
    npx = npy = 512
    x0, y0 = _raster_origin(npx, npy, 12)
    nx_, ny_ = _nominal_xy(npx, npy, x0, y0)
    P = npx * npy
    scan = np.empty((1, P, 3))
    scan[0, :, 0] = nx_ + rng.normal(0, 1.5e-3, P)
    scan[0, :, 1] = ny_ + rng.normal(0, 1.5e-3, P)
    scan[0, :, 2] = rng.normal(0, 4e-3, P)
    cx, cy = _aperture_centre(x0, y0, npx, npy, tx, rx)
    n = 10_000
    pos = np.empty((n, 3))
    pos[:, 0] = cx + rng.uniform(-0.120, 0.120, n)
    pos[:, 1] = cy + rng.uniform(-0.120, 0.120, n)
    pos[:, 2] = rng.uniform(0.2, 0.5, n)
    amp = (rng.normal(0, 1, n) + 1j * rng.normal(0, 1, n)) / math.sqrt(2.0)  # Rayleigh |amp|
    return Scene("large", 1, tx, rx, npx, npy, x0, y0, DELTA, DELTA, scan,
                 scan[:, :, 2].mean(axis=1), wavenumbers(512), 512, 512, 512, 2e-3, 0.35,
                 [pos], [amp], _noise_key(4))


def _realtime(n_frames: int = 64) -> Scene:
    tx, rx = awr1443_layout(2)
    npx = npy = 128
    x0, y0 = _raster_origin(npx, npy, 8)
    nx_, ny_ = _nominal_xy(npx, npy, x0, y0)
    P = npx * npy
    cx, cy = _aperture_centre(x0, y0, npx, npy, tx, rx)
    scan = np.empty((n_frames, P, 3))
    poss, amps = [], []
    for f, ss in enumerate(np.random.SeedSequence(5).spawn(n_frames)):
        rng = np.random.default_rng(ss)
        scan[f, :, 0] = nx_ + rng.normal(0, 1e-3, P)
        scan[f, :, 1] = ny_ + rng.normal(0, 1e-3, P)
        scan[f, :, 2] = rng.normal(0, 1e-3, P)
        n = 50
        pos = np.empty((n, 3))
        pos[:, 0] = cx + rng.uniform(-0.040, 0.040, n)
        pos[:, 1] = cy + rng.uniform(-0.040, 0.040, n)
        pos[:, 2] = rng.uniform(0.2, 0.35, n)
        poss.append(pos)
        amps.append(np.ones(n, complex))
    return Scene("realtime", n_frames, tx, rx, npx, npy, x0, y0, DELTA, DELTA, scan,
                 scan[:, :, 2].mean(axis=1), wavenumbers(128), 128, 128, 64, 5e-3, 0.275,
                 poss, amps, _noise_key(5))


# ---------------------------------------------------------------------------
# Echo synthesis, Eq. (9) with Eq. (2) distances.
# ---------------------------------------------------------------------------

def element_positions(sc: Scene, f: int):
    """World Tx/Rx positions for every pose of frame f: [n_tx, P, 3], [n_rx, P, 3]."""
    p = sc.scan[f]
    return p[None, :, :] + sc.tx[:, None, :], p[None, :, :] + sc.rx[:, None, :]


def synthesize_cpu(sc: Scene, noise: bool = True, chunk: int = 64) -> np.ndarray:
    """s[f,t,r,p,i] = sum_n amp_n * exp(-j k_i (|tx-q_n| + |rx-q_n|)) + noise.

    float64 distances and phases, rounded once to complex64.  Feasible for the
    Tiny/Small configs (and small test variants); large configs use the CUDA
    generator in ``scenes.gpu`` which implements the same sum.
    """
    F, nt, nr, P, nk = sc.data_shape
    out = np.empty(sc.data_shape, np.complex64)
    k = sc.k
    for f in range(F):
        txw, rxw = element_positions(sc, f)
        q = sc.scat_pos[f]
        a = sc.scat_amp[f]
        for t in range(nt):
            for r in range(nr):
                acc = np.zeros((P, nk), complex)
                for n0 in range(0, q.shape[0], chunk):
                    qq = q[n0:n0 + chunk]
                    R = (np.linalg.norm(txw[t][:, None, :] - qq[None], axis=-1)
                         + np.linalg.norm(rxw[r][:, None, :] - qq[None], axis=-1))  # [P, n]
                    ph = np.exp(-1j * R[:, :, None] * k[None, None, :])            # [P, n, nk]
                    acc += np.einsum("n,pnk->pk", a[n0:n0 + chunk], ph)
                if noise and sc.noise_sigma > 0:
                    start = (((f * nt + t) * nr + r) * P) * nk
                    acc += _rng.complex_normal(sc.noise_key, start, P * nk, sc.noise_sigma).reshape(P, nk)
                out[f, t, r] = acc
    return out


def with_geometry(sc: Scene, *, jitter_xy=None, jitter_z=None, layout=None) -> Scene:
    """Return a copy with modified geometry (test variants: zero jitter,
    monostatic layout, ...)."""
    sc = dataclasses.replace(sc)
    if layout is not None:
        sc.tx, sc.rx = layout
    nx_, ny_ = _nominal_xy(sc.npx, sc.npy, sc.x0, sc.y0)
    scan = sc.scan.copy()
    if jitter_xy == 0:
        scan[:, :, 0] = nx_[None]
        scan[:, :, 1] = ny_[None]
    if jitter_z == 0:
        scan[:, :, 2] = 0.0
    sc.scan = scan
    sc.z0 = scan[:, :, 2].mean(axis=1)
    return sc


def raster_scene(npx, npy, nx, ny, n_k, nz, dz_img, z_ref, *, n_tx=2, monostatic=False,
                 jitter_xy=0.0, jitter_z=0.0, n_frames=1, seed=0, name="custom") -> Scene:
    """A custom raster workload for tests (no scatterers yet; set
    ``scat_pos``/``scat_amp``).  Same construction as the named configs."""
    tx, rx = monostatic_layout() if monostatic else awr1443_layout(n_tx)
    J = 1 if monostatic else 4 * n_tx
    x0, y0 = _raster_origin(npx, npy, J)
    nx_, ny_ = _nominal_xy(npx, npy, x0, y0)
    P = npx * npy
    rng = np.random.default_rng(seed)
    scan = np.zeros((n_frames, P, 3))
    for f in range(n_frames):
        scan[f, :, 0] = nx_ + (rng.normal(0, jitter_xy, P) if jitter_xy else 0.0)
        scan[f, :, 1] = ny_ + (rng.normal(0, jitter_xy, P) if jitter_xy else 0.0)
        scan[f, :, 2] = rng.normal(0, jitter_z, P) if jitter_z else 0.0
    return Scene(name, n_frames, tx, rx, npx, npy, x0, y0, DELTA, DELTA, scan,
                 scan[:, :, 2].mean(axis=1), wavenumbers(n_k), nx, ny, nz, dz_img, z_ref,
                 [np.zeros((0, 3))] * n_frames, [np.zeros(0, complex)] * n_frames,
                 _noise_key(1000 + seed), 0.0)


def frame_subset(sc: Scene, lo: int, hi: int) -> Scene:
    """Frames [lo, hi) of a multi-frame scene as a scene of its own, with the
    noise counter shifted so that its echo equals frames lo..hi-1 of the full
    scene's echo (sample n of the subset uses counter key + 2*(n + offset))."""
    lo, hi = max(0, lo), min(sc.n_frames, hi)
    per_frame = sc.n_tx * sc.n_rx * sc.n_pos * sc.n_k
    key = (int(sc.noise_key) + 2 * lo * per_frame) & 0xFFFFFFFFFFFFFFFF
    return dataclasses.replace(sc, n_frames=hi - lo, scan=sc.scan[lo:hi], z0=sc.z0[lo:hi],
                               scat_pos=sc.scat_pos[lo:hi], scat_amp=sc.scat_amp[lo:hi], noise_key=key)
