"""Run debug stages of one small case repeatedly and report run-to-run bit
differences (race hunting):  python scripts/det_case.py CASE STAGE REPS [LIB]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.argv, args = sys.argv[:2], sys.argv[1:]
import torch  # noqa: E402

import san_case  # noqa: E402,F401  (builds the scene `sc` and data `d`)
from paper_2305_02064_b200 import sar as sarmod  # noqa: E402

case, stage, reps = args[0], int(args[1]), int(args[2])
if len(args) > 3:
    sarmod._lib = None
    sarmod.load_library(args[3])
import paper_2305_02064_b200 as sar  # noqa: E402
sc, d = san_case.sc, san_case.d
with sar.Plan.from_scene(sc) as plan:
    ref = plan.debug_stage(stage, d).clone()
    nbad = 0
    for i in range(reps):
        g = plan.debug_stage(stage, d)
        diff = (g != ref)
        if diff.any():
            nbad += 1
            idx = diff.nonzero()
            print("rep", i, "differs at", int(diff.sum()), "elements; first", idx[:6].tolist(),
                  "unique dims:", [sorted(set(idx[:, k].tolist()))[:12] for k in range(idx.shape[1])])
    print(case, "stage", stage, "reps", reps, "runs differing:", nbad)
