"""Back-to-back sar_reconstruct loop time (CUDA events around K calls) for
plans with and without per-kernel profiling events, per library:
    python scripts/loop_time.py CONFIG NAME[:LIBPATH] ..."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import scenes  # noqa: E402
from scenes import gpu as sgpu  # noqa: E402
import paper_2305_02064_b200 as sar  # noqa: E402
from paper_2305_02064_b200 import sar as sarmod  # noqa: E402

name = sys.argv[1]
sc = scenes.make_scene(name)
sgpu.build()
d = sgpu.synthesize_gpu(sc)
out = torch.empty(sc.image_shape, dtype=torch.float32, device="cuda")
K = 20
for spec in sys.argv[2:]:
    tag, _, path = spec.partition(":")
    sarmod._lib = None
    sarmod.load_library(path or sarmod.LIB_PATH)
    for flags in (0, sar.SAR_PROFILE_STAGES):
        with sar.Plan.from_scene(sc, flags=flags) as plan:
            for _ in range(3):
                plan.reconstruct(d, out)
            torch.cuda.synchronize()
            if flags:
                plan.profile_reset()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            t0 = time.perf_counter()
            for _ in range(K):
                plan.reconstruct(d, out)
            t1 = time.perf_counter()
            e1.record()
            torch.cuda.synchronize()
            print(f"{name} {tag:>8} {'profiled' if flags else 'plain   '} {e0.elapsed_time(e1) / K:.4f} ms/call"
                  f" (host enqueue {(t1 - t0) * 1e3 / K:.4f} ms/call)", flush=True)
            if flags:
                ms, n = plan.profile_read()
                print("   stages over the loop:", " ".join(f"{m / n:.3f}" for m in ms), f"sum {sum(ms) / n:.4f} ms (n={n})")
