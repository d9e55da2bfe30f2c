"""Write tests/golden/tiny_oracle.json: statistics of the fp64 oracle's Tiny
reconstructions (BASELINE.json configs[0]), used as a regression pin for the
oracle (tests/test_oracle_golden.py).  Calls only oracle/ and the seeded scene
generator; no value comes from the CUDA path."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import scenes  # noqa: E402


def stats(img):
    a = np.asarray(img, float)[0]
    idx = np.unravel_index(np.argmax(a), a.shape)
    flat = a.ravel()
    picks = np.linspace(0, flat.size - 1, 16).astype(int)
    return {"shape": list(a.shape), "argmax": [int(i) for i in idx], "max": float(a.max()),
            "l2": float(np.linalg.norm(flat)), "samples_at": picks.tolist(), "samples": flat[picks].tolist()}


def main():
    sc = scenes.make_scene("tiny")
    s = scenes.synthesize_cpu(sc)
    out = {"source": "scripts/make_golden.py (oracle only), scene tiny (BASELINE.json configs[0], seed 1)"}
    out["rma3d"] = stats(oracle.reconstruct(s, sc)[0])
    out["rma3d_no_compensation"] = stats(oracle.reconstruct(s, sc, no_compensation=True)[0])
    out["plane2d_z0.25"] = stats(oracle.reconstruct_planes(s, sc, [0.25])[0])
    out["nufft3d"] = stats(oracle.nufft.reconstruct_nufft(s, sc)[0])
    with open(os.path.join(ROOT, "tests", "golden", "tiny_oracle.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
