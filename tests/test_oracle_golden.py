"""Regression pin of the oracle itself: its Tiny reconstructions must keep the
statistics stored in tests/golden/tiny_oracle.json (written by
scripts/make_golden.py, which calls only oracle/).  A change to the oracle's
arithmetic that moves them must be justified by a paper passage or a DESIGN.md
reading (and the golden file regenerated in the same commit)."""
import json
import os

import numpy as np
import pytest

import oracle
import scenes

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "tiny_oracle.json")))


def _check(img, g):
    a = np.asarray(img, float)[0]
    assert list(a.shape) == g["shape"]
    assert list(np.unravel_index(np.argmax(a), a.shape)) == g["argmax"]
    assert np.isclose(a.max(), g["max"], rtol=1e-9)
    assert np.isclose(np.linalg.norm(a.ravel()), g["l2"], rtol=1e-9)
    assert np.allclose(a.ravel()[g["samples_at"]], g["samples"], rtol=1e-8, atol=1e-12 * g["max"])


@pytest.fixture(scope="module")
def tiny():
    sc = scenes.make_scene("tiny")
    return sc, scenes.synthesize_cpu(sc)


def test_golden_rma3d(tiny):
    sc, s = tiny
    _check(oracle.reconstruct(s, sc)[0], GOLD["rma3d"])
    _check(oracle.reconstruct(s, sc, no_compensation=True)[0], GOLD["rma3d_no_compensation"])


def test_golden_plane2d_and_nufft(tiny):
    sc, s = tiny
    _check(oracle.reconstruct_planes(s, sc, [0.25])[0], GOLD["plane2d_z0.25"])
    _check(oracle.nufft.reconstruct_nufft(s, sc)[0], GOLD["nufft3d"])
