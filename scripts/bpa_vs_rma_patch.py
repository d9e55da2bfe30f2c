"""Large-config physics check: NCC of |BPA| and the RMA image on a W x W patch
of one z plane, per placement (the whole plane would take ~80 s of BPA):
    python scripts/bpa_vs_rma_patch.py [CONFIG] [W]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import scenes  # noqa: E402
from scenes import gpu as sgpu  # noqa: E402
import paper_2305_02064_b200 as sar  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "large"
W = int(sys.argv[2]) if len(sys.argv) > 2 else 64
sc = scenes.make_scene(name)
sgpu.build()
d = sgpu.synthesize_gpu(sc)
m = sc.nz // 2
ys = np.arange(sc.ny // 2 - W // 2, sc.ny // 2 + W // 2)
xs = np.arange(sc.nx // 2 - W // 2, sc.nx // 2 + W // 2)
imgs = {}
for tag, fl in (("raster", 0), ("nearest", sar.SAR_GRID_NEAREST), ("nufft", sar.SAR_GRID_NUFFT)):
    try:
        with sar.Plan.from_scene(sc, flags=fl) as plan:
            imgs[tag] = plan.reconstruct(d)[0, m].cpu().numpy().astype(np.float64)[np.ix_(ys, xs)]
            x0, y0, z0, dx, dy, dz = plan.axes()
    except sar.SarError as e:
        print(tag, "not available:", e)
iy, ix = np.meshgrid(ys, xs, indexing="ij")
vox = np.stack([x0 + ix * dx, y0 + iy * dy, np.full(ix.shape, z0 + m * dz)], axis=-1).reshape(-1, 3)
out, ms = sar.bpa_scene(sc, d, vox)
b = np.abs(out.cpu().numpy()).reshape(W, W).astype(np.float64)
print(f"{name} plane {m}, central {W}x{W} patch: BPA {ms:.0f} ms; NCC(|BPA|, RMA image) " +
      "  ".join(f"{k} {float((b * v).sum() / np.sqrt((b * b).sum() * (v * v).sum())):.4f}" for k, v in imgs.items()),
      flush=True)
