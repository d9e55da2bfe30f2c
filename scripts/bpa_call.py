"""A few sar_bpa calls for profiling: python scripts/bpa_call.py CONFIG NVOX [CALLS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import scenes  # noqa: E402
from scenes import gpu as sgpu  # noqa: E402
import paper_2305_02064_b200 as sar  # noqa: E402

name, nvox = sys.argv[1], int(sys.argv[2])
calls = int(sys.argv[3]) if len(sys.argv) > 3 else 2
sc = scenes.make_scene(name)
sgpu.build()
d = sgpu.synthesize_gpu(sc)
with sar.Plan.from_scene(sc) as plan:
    x0, y0, z0, dx, dy, dz = plan.axes()
m, iy, ix = np.meshgrid(np.arange(sc.nz // 2, sc.nz), np.arange(sc.ny), np.arange(sc.nx), indexing="ij")
vox = np.stack([x0 + ix * dx, y0 + iy * dy, z0 + m * dz], axis=-1).reshape(-1, 3)[:nvox]
for _ in range(calls):
    out, ms = sar.bpa_scene(sc, d, vox)
    print(f"{name} {vox.shape[0]} voxels: kernel {ms:.3f} ms", flush=True)
