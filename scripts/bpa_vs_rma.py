"""Physics check with the GPU back-projection baseline (the paper's gold
standard): normalised cross-correlation between the BPA magnitude
and the RMA image on one z plane of a configuration, for the RASTER, NEAREST
and NUFFT placements:  python scripts/bpa_vs_rma.py CONFIG [PLANE_INDEX]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import scenes  # noqa: E402
from scenes import gpu as sgpu  # noqa: E402
import paper_2305_02064_b200 as sar  # noqa: E402


def ncc(a, b):
    return float((a * b).sum() / np.sqrt((a * a).sum() * (b * b).sum()))


def plane_ncc(sc, d, m, flags_list):
    """NCC of |BPA| and the RMA magnitude on image plane m for each flag set."""
    imgs = {}
    for name, fl in flags_list:
        with sar.Plan.from_scene(sc, flags=fl) as plan:
            imgs[name] = plan.reconstruct(d)[0, m].cpu().numpy().astype(np.float64)
            x0, y0, z0, dx, dy, dz = plan.axes()
    iy, ix = np.meshgrid(np.arange(sc.ny), np.arange(sc.nx), indexing="ij")
    vox = np.stack([x0 + ix * dx, y0 + iy * dy, np.full(ix.shape, z0 + m * dz)], axis=-1).reshape(-1, 3)
    out, ms = sar.bpa_scene(sc, d, vox)
    b = np.abs(out.cpu().numpy()).reshape(sc.ny, sc.nx).astype(np.float64)
    return {k: ncc(b, v) for k, v in imgs.items()}, ms


if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "freehand"
    sc = scenes.make_scene(name)
    sgpu.build()
    d = sgpu.synthesize_gpu(sc)
    m = int(sys.argv[2]) if len(sys.argv) > 2 else sc.nz // 2
    res, ms = plane_ncc(sc, d, m, [("raster", 0), ("nearest", sar.SAR_GRID_NEAREST), ("nufft", sar.SAR_GRID_NUFFT)])
    print(f"{name} plane {m}: BPA {ms:.1f} ms for {sc.nx * sc.ny} voxels; NCC(|BPA|, RMA image) " +
          "  ".join(f"{k} {v:.4f}" for k, v in res.items()), flush=True)
