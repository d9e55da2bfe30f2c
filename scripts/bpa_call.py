"""A few sar_bpa calls for profiling / A-B timing:
    python scripts/bpa_call.py CONFIG NVOX [CALLS] [LIBPATH ...]"""
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
from paper_2305_02064_b200 import sar as sarmod  # noqa: E402

terms = vox.shape[0] * sc.n_tx * sc.n_rx * sc.n_pos * sc.n_k
ref = None
for lib in (sys.argv[4:] or [sarmod.LIB_PATH]):
    sarmod._lib = None
    sarmod.load_library(lib)
    for _ in range(calls):
        out, ms = sar.bpa_scene(sc, d, vox)
        if ref is None:
            ref = out.clone()
        dev = ((out - ref).norm() / ref.norm()).item()
        print(f"{os.path.basename(lib)} {name} {vox.shape[0]} voxels: kernel {ms:.3f} ms  "
              f"{terms / ms / 1e6:.0f} Gterms/s  frac {8 * terms / (ms * 1e-3) / 74.45e12:.3f}  "
              f"rel-diff-vs-first {dev:.1e}", flush=True)
