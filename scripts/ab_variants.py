"""A/B timing of compile-time variants of the library (experiments only):
    python scripts/ab_variants.py CONFIG NAME[:LIBPATH] ...
Per-kernel CUDA-event times (5 calls after 3 warm-ups) of each library on one
config; NAME alone means the product library."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import scenes  # noqa: E402
from scenes import gpu as sgpu  # noqa: E402
import paper_2305_02064_b200 as sar  # noqa: E402
from paper_2305_02064_b200 import sar as sarmod  # noqa: E402

name, _, mode = sys.argv[1].partition(":")   # CONFIG or CONFIG:nufft
sc = scenes.make_scene(name)
mflags = sar.SAR_GRID_NUFFT if mode == "nufft" else 0
sgpu.build()
d = sgpu.synthesize_gpu(sc)
ref = None
for spec in sys.argv[2:]:
    tag, _, path = spec.partition(":")
    sarmod._lib = None
    sarmod.load_library(path or sarmod.LIB_PATH)
    with sar.Plan.from_scene(sc, flags=sar.SAR_PROFILE_STAGES | mflags) as plan:
        for _ in range(3):
            img = plan.reconstruct(d)
        torch.cuda.synchronize()
        if ref is None:
            ref = img.clone()
        dev = ((img - ref).norm() / ref.norm()).item()
        plan.profile_reset()
        for _ in range(5):
            plan.reconstruct(d)
        ms, n = plan.profile_read()
    print(f"{name} {tag:>10} " + " ".join(f"{s.split()[0]}={m / n:.3f}" for s, m in zip(sar.STAGE_NAMES, ms)) +
          f" total={sum(ms) / n:.3f}ms  rel-diff-vs-first={dev:.2e}", flush=True)
