"""Per-call latency of the small, launch-bound configs: K back-to-back calls
between CUDA events, with and without SAR_CUDA_GRAPH."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import scenes  # noqa: E402
import paper_2305_02064_b200 as sar  # noqa: E402

K = 200
for name in sys.argv[1:] or ["tiny", "small"]:
    sc = scenes.make_scene(name)
    d = torch.from_numpy(scenes.synthesize_cpu(sc)).cuda()
    out = torch.empty(sc.image_shape, device="cuda")
    s = torch.cuda.Stream()
    for flags, tag in ((0, "launches"), (sar.SAR_CUDA_GRAPH, "graph")):
        with torch.cuda.stream(s), sar.Plan.from_scene(sc, flags=flags) as plan:
            for _ in range(10):
                plan.reconstruct(d, out)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record()
            for _ in range(K):
                plan.reconstruct(d, out)
            e1.record()
            torch.cuda.synchronize()
            wall = (time.perf_counter() - t0) / K
            print(f"{name:6s} {tag:9s} {e0.elapsed_time(e1) / K * 1e3:7.1f} us/call (device)  {wall * 1e6:7.1f} us/call (host wall)",
                  flush=True)
