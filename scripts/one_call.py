"""A few reconstructions of one config (for ncu captures: -s/-c pick the call)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import scenes  # noqa: E402
from scenes import gpu as sgpu  # noqa: E402
import paper_2305_02064_b200 as sar  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "large"
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 3
if len(sys.argv) > 3 and sys.argv[3] != "-":   # a library variant (scripts/ab_variants.py)
    from paper_2305_02064_b200 import sar as sarmod
    sarmod.load_library(sys.argv[3])
flags = int(sys.argv[4]) if len(sys.argv) > 4 else 0
sc = scenes.make_scene(name)
sgpu.build()
d = sgpu.synthesize_gpu(sc)
with sar.Plan.from_scene(sc, flags=flags) as plan:
    for _ in range(calls):
        plan.reconstruct(d)
    torch.cuda.synchronize()
print("ok", name, calls)
