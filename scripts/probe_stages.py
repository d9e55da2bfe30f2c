"""Per-kernel CUDA-event times of the path on one config, with and without
the compensation (isolates the phase-rotation cost of K1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import scenes  # noqa: E402
from scenes import gpu as sgpu  # noqa: E402
import paper_2305_02064_b200 as sar  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "large"
sc = scenes.make_scene(name)
sgpu.build()
d = sgpu.synthesize_gpu(sc)
for flags in (sar.SAR_PROFILE_STAGES, sar.SAR_PROFILE_STAGES | sar.SAR_NO_COMPENSATION):
    with sar.Plan.from_scene(sc, flags=flags) as plan:
        for _ in range(3):
            plan.reconstruct(d)
        torch.cuda.synchronize()
        plan.profile_reset()
        for _ in range(5):
            plan.reconstruct(d)
        ms, n = plan.profile_read()
        print(name, "nocomp" if flags & 1 else "comp  ", " ".join(f"{s}={m / n:.3f}ms" for s, m in zip(sar.STAGE_NAMES, ms)),
              f"total={sum(ms) / n:.3f}ms", flush=True)
