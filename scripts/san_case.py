"""One small reconstruction per named case, for compute-sanitizer runs:
    compute-sanitizer --tool racecheck python scripts/san_case.py xbase
Cases: tiny, small, xbase (x-baseline Tx/Rx layout, shared-tile K1), ragged
(odd n_k, plain kernels), nufft, plane2d, slab (G = 2 emulated), k3w (n_z = 512)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import scenes  # noqa: E402
import paper_2305_02064_b200 as sar  # noqa: E402


def custom(npx, npy, nx, ny, nk, nz, dz, z_ref, n_tx=2, seed=0):
    sc = scenes.raster_scene(npx, npy, nx, ny, nk, nz, dz, z_ref, n_tx=n_tx, jitter_xy=0.5e-3, jitter_z=2e-3,
                             seed=seed)
    rng = np.random.default_rng(seed + 1)
    cx, cy = sc.x0 + npx * sc.dx / 2, sc.y0 + npy * sc.dy / 2
    q = np.stack([cx + rng.uniform(-0.01, 0.01, 4), cy + rng.uniform(-0.01, 0.01, 4),
                  z_ref + rng.uniform(-0.02, 0.02, 4)], axis=1)
    sc.scat_pos, sc.scat_amp = [q], [rng.normal(size=4) + 1j * rng.normal(size=4)]
    sc.noise_sigma = 1e-3
    return sc


def xlayout(sc, n_tx=2):
    lam = scenes.LAMBDA_C
    tx = np.zeros((n_tx, 3))
    tx[:, 0] = [2.0 * lam * i for i in range(n_tx)]
    rx = np.zeros((4, 3))
    rx[:, 1] = [0.0, lam / 2.0, lam, 1.5 * lam]
    sc.tx, sc.rx = tx, rx
    return sc


case = sys.argv[1] if len(sys.argv) > 1 else "small"
flags, planes = 0, None
if case in ("tiny", "small"):
    sc = scenes.make_scene(case)
elif case == "xbase":
    sc = xlayout(custom(512, 8, 512, 16, 40, 16, 5e-3, 0.25))
elif case == "xbase64":
    sc = xlayout(custom(64, 24, 64, 32, 48, 32, 5e-3, 0.2, n_tx=3), 3)
elif case == "ragged":
    sc = custom(30, 10, 32, 16, 17, 16, 5e-3, 0.2)
elif case == "nufft":
    sc, flags = scenes.make_scene("tiny"), sar.SAR_GRID_NUFFT
elif case == "plane2d":
    sc, planes = scenes.make_scene("small"), [0.2, 0.25, 0.3]
elif case == "k3w":
    sc = custom(20, 12, 32, 16, 600, 512, 2e-3, 0.3)
else:
    sc = scenes.make_scene("small")
d = torch.from_numpy(scenes.synthesize_cpu(sc)).cuda()
if case == "slab":
    from paper_2305_02064_b200 import slab
    plans = [sar.SlabPlan.from_scene(sc, rank=r, world=2) for r in range(2)]
    img = torch.zeros(sc.image_shape, device="cuda")
    slab.emulate(plans, d, img)
    for p in plans:
        p.close()
else:
    with sar.Plan.from_scene(sc, flags=flags, z_planes=planes) as plan:
        for st in ((2, 3, 4) if flags == 0 else (2, 4)):
            plan.debug_stage(st, d)
        img = plan.reconstruct(d)
torch.cuda.synchronize()
print(case, "ok", float(img.abs().max()))
