"""Per-call time and per-stage times as a function of the back-to-back loop
length (sustained-load behaviour): python scripts/loop_len.py CONFIG"""
import os
import subprocess
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
out = torch.empty(sc.image_shape, dtype=torch.float32, device="cuda")


def smi():
    q = "clocks.sm,clocks.mem,power.draw,temperature.gpu,temperature.memory,clocks_event_reasons.active"
    return subprocess.run(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader"], capture_output=True,
                          text=True).stdout.strip()


with sar.Plan.from_scene(sc, flags=sar.SAR_PROFILE_STAGES) as plan:
    for K in (5, 10, 20, 40, 80, 5, 20):
        for _ in range(3):
            plan.reconstruct(d, out)
        torch.cuda.synchronize()
        plan.profile_reset()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(K):
            plan.reconstruct(d, out)
        e1.record()
        torch.cuda.synchronize()
        ms, n = plan.profile_read()
        print(f"K={K:3d} loop {e0.elapsed_time(e1) / K:.4f} ms/call  stages " +
              " ".join(f"{m / n:.3f}" for m in ms) + f"  sum {sum(ms) / n:.4f}   smi: {smi()}", flush=True)
