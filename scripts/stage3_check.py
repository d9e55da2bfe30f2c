"""Stage-3 (Stolt output) error against the oracle for the n_z = 512,
n_k = 600 edge case, per library, repeated (nondeterminism hunt)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2305_02064_b200 as sar  # noqa: E402
from paper_2305_02064_b200 import sar as sarmod  # noqa: E402
from test_gpu_parity import _custom, errs  # noqa: E402

kw = dict(npx=20, npy=12, nx=32, ny=16, nk=600, nz=512, dz=2e-3, z_ref=0.3)
sc = _custom(**kw)
import scenes  # noqa: E402
s = scenes.synthesize_cpu(sc)
d = torch.from_numpy(s).cuda()
img, geo, st = oracle.reconstruct(s, sc, complex_out=True, return_stages=True)
for spec in sys.argv[1:]:
    tag, _, path = spec.partition(":")
    sarmod._lib = None
    sarmod.load_library(path or sarmod.LIB_PATH)
    for rep in range(3):
        with sar.Plan.from_scene(sc) as plan:
            g3 = plan.debug_stage(3, d).cpu().numpy()
            g2 = plan.debug_stage(2, d).cpu().numpy()
        print(tag, rep, "stolt e2 %.3e" % errs(g3, st["stolt"])[0], "spectrum e2 %.3e" % errs(g2, st["spectrum"])[0],
              flush=True)
