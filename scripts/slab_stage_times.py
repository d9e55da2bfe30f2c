"""CUDA-event times of the three slab stages (one rank of a G-way split, the
exchanges replaced by local copies of this rank's own blocks)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import scenes  # noqa: E402
from scenes import gpu as sgpu  # noqa: E402
import paper_2305_02064_b200 as sar  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "large"
G = int(sys.argv[2]) if len(sys.argv) > 2 else 8
sc = scenes.make_scene(name)
sgpu.build()
d = sgpu.synthesize_gpu(sc)
with sar.SlabPlan.from_scene(sc, rank=0, world=G) as p:
    img = torch.empty(p.image_shape, device="cuda")
    s1 = torch.empty(p.send1_shape, dtype=torch.complex64, device="cuda")
    s2 = torch.empty(p.send2_shape, dtype=torch.complex64, device="cuda")
    r1, r2 = torch.empty_like(s1), torch.empty_like(s2)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    acc = [0.0, 0.0, 0.0]
    for it in range(13):
        ev[0].record()
        p.stage1(d, s1)
        ev[1].record()
        p.stage2(r1, s2)
        ev[2].record()
        p.stage3(r2, img)
        ev[3].record()
        torch.cuda.synchronize()
        if it >= 3:
            for i in range(3):
                acc[i] += ev[i].elapsed_time(ev[i + 1]) / 10
    print(name, f"G={G}", " ".join(f"stage{i + 1}={a:.3f}ms" for i, a in enumerate(acc)), f"sum={sum(acc):.3f}ms")
