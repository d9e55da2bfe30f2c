"""Sustained-load A/B of library variants (the GPU's power cap lowers the SM
clock after a few tens of milliseconds of back-to-back calls): per library,
K back-to-back calls after 3 warm-ups, loop time, per-stage times and the
nvidia-smi clocks / power / throttle reasons right after the loop.
    python scripts/sustained_ab.py CONFIG K NAME[:LIBPATH] ..."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import scenes  # noqa: E402
from scenes import gpu as sgpu  # noqa: E402
import paper_2305_02064_b200 as sar  # noqa: E402
from paper_2305_02064_b200 import sar as sarmod  # noqa: E402

name, K = sys.argv[1], int(sys.argv[2])
sc = scenes.make_scene(name)
sgpu.build()
d = sgpu.synthesize_gpu(sc)
out = torch.empty(sc.image_shape, dtype=torch.float32, device="cuda")


try:
    import pynvml
    pynvml.nvmlInit()
    _h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())

    def energy_mj():
        return pynvml.nvmlDeviceGetTotalEnergyConsumption(_h)
except Exception:  # noqa: BLE001
    def energy_mj():
        return float("nan")


def smi():
    q = "clocks.sm,power.draw,power.limit,clocks_event_reasons.active"
    return subprocess.run(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader"], capture_output=True,
                          text=True).stdout.strip()


for rep in range(2):
    for spec in sys.argv[3:]:
        tag, _, rest = spec.partition(":")
        path, _, fl = rest.partition(":")
        flags = int(fl) if fl else 0
        sarmod._lib = None
        sarmod.load_library(path or sarmod.LIB_PATH)
        with sar.Plan.from_scene(sc, flags=sar.SAR_PROFILE_STAGES | flags) as plan:
            for _ in range(3):
                plan.reconstruct(d, out)
            torch.cuda.synchronize()
            plan.profile_reset()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            j0 = energy_mj()
            e0.record()
            for _ in range(K):
                plan.reconstruct(d, out)
            e1.record()
            torch.cuda.synchronize()
            j1 = energy_mj()
            s = smi()
            ms, n = plan.profile_read()
        print(f"{name} {tag:>8} K={K} loop {e0.elapsed_time(e1) / K:.4f} ms/call  stages " +
              " ".join(f"{m / n:.3f}" for m in ms) + f"  {(j1 - j0) / K:.0f} mJ/call  smi: {s}", flush=True)
