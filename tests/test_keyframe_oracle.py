"""Keyframe-preparation oracle (oracle/keyframe_oracle.py) pinned to the live reference's
make_keyframe images (tests/golden/golden_keyframe.npz, made by tests/golden/make_golden.py)."""
import os

import numpy as np
import pytest

from oracle import keyframe_oracle as KO

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_keyframe.npz"))


@pytest.mark.parametrize("case", ["full", "part"])
def test_keyframe_oracle_matches_reference(case):
    cloud = G[f"{case}_cloud"]
    cam = tuple(G[f"{case}_cam"])
    W, H = int(cam[0]), int(cam[1])
    est = KO.estimate_camera(cloud, W, H)
    assert np.allclose(est[2:], cam[2:], rtol=0, atol=0)
    assert bool(KO.full_circle(cam)) == bool(G[f"{case}_full_circle"])
    rng, valid = KO.build_range_image(cam, cloud)
    assert np.array_equal(valid, G[f"{case}_valid"]) and np.array_equal(rng, G[f"{case}_range"])
    sm = KO.smooth_range_image(rng, valid, KO.full_circle(cam))
    assert np.array_equal(sm, G[f"{case}_smooth"])  # the median is one of the inputs: bit-exact
    n, ok = KO.range_image_normals(cam, sm, valid)
    assert np.array_equal(ok, G[f"{case}_nvalid"])
    assert np.abs(n - G[f"{case}_normals"]).max() <= 1e-12
