"""Does the GPU's recent power history decide when the SW power cap hits the
bench loop?  Synthesise the Large scene (a long, power-hungry GPU job), then
for each rest period: sleep, run the bench's 5 warm-up + 20 timed calls with a
CUDA event around every call, and print the per-call times and the loop mean:
    python scripts/power_rest.py [CONFIG]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import scenes  # noqa: E402
from scenes import gpu as sgpu  # noqa: E402
import paper_2305_02064_b200 as sar  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "large"
sc = scenes.make_scene(name)
sgpu.build()
t0 = time.time()
d = sgpu.synthesize_gpu(sc)
torch.cuda.synchronize()
print(f"synthesis {time.time() - t0:.2f} s", flush=True)
out = torch.empty(sc.image_shape, dtype=torch.float32, device="cuda")
with sar.Plan.from_scene(sc) as plan:
    for rest in (0.0, 2.0, 0.0, 5.0, 0.5, 2.0):
        time.sleep(rest)
        for _ in range(5):
            plan.reconstruct(d, out)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(21)]
        ev[0].record()
        for i in range(20):
            plan.reconstruct(d, out)
            ev[i + 1].record()
        torch.cuda.synchronize()
        per = [ev[i].elapsed_time(ev[i + 1]) for i in range(20)]
        print(f"rest {rest:3.1f} s: mean {ev[0].elapsed_time(ev[20]) / 20:.4f} ms/call  per call " +
              " ".join(f"{p:.3f}" for p in per), flush=True)
