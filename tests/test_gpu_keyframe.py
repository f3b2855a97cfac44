"""Device keyframe preparation (ss_range_image, ss_smooth_range_image,
ss_range_image_normals) against the live reference's make_keyframe images
(tests/golden/golden_keyframe.npz): range image and smoothing bit-exact, normal
mask exact, normals within 1e-12 (float64; CUDA's cos/sin may differ from
libm's in the last bit of a pixel direction)."""
import os

import numpy as np
import pytest
import torch

from oracle import keyframe_oracle as KO
from paper_2503_17491_b200 import SE3Pose, SphericalCamera
from paper_2503_17491_b200 import keyframe as KF
from paper_2503_17491_b200 import mapping as MP

pytestmark = pytest.mark.gpu

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_keyframe.npz"))
CASES = ["full", "part"]


def _cam(case):
    c = G[f"{case}_cam"]
    return SphericalCamera(int(c[0]), int(c[1]), *[float(x) for x in c[2:]])


@pytest.mark.parametrize("case", CASES)
def test_range_and_smoothing_bit_exact(cuda, case):
    cam = _cam(case)
    rimg = KF.build_range_image(cam, G[f"{case}_cloud"])
    assert np.array_equal(rimg.valid, G[f"{case}_valid"]) and np.array_equal(rimg.range, G[f"{case}_range"])
    sm = KF.smooth_range_image(rimg, cam.full_circle)
    assert np.array_equal(sm.range, G[f"{case}_smooth"])
    assert np.array_equal(sm.valid, rimg.valid)


@pytest.mark.parametrize("case", CASES)
def test_normals(cuda, case):
    cam = _cam(case)
    sm = KF.RangeImage(G[f"{case}_smooth"], G[f"{case}_valid"])
    n = KF.range_image_normals(cam, sm)
    assert np.array_equal(n.valid, G[f"{case}_nvalid"])
    assert np.abs(n.normals - G[f"{case}_normals"]).max() <= 1e-12


@pytest.mark.parametrize("case", CASES)
def test_make_keyframe(cuda, case):
    c = G[f"{case}_cam"]
    kf = KF.make_keyframe(3, G[f"{case}_cloud"], SE3Pose.identity(), int(c[0]), int(c[1]))
    assert (kf.camera.az_min, kf.camera.az_max, kf.camera.el_min, kf.camera.el_max) == tuple(float(x) for x in c[2:])
    assert np.array_equal(kf.range_image.range, G[f"{case}_range"])
    assert np.array_equal(kf.normal_image.valid, G[f"{case}_nvalid"])
    assert np.abs(kf.normal_image.normals - G[f"{case}_normals"]).max() <= 1e-12
    dk = MP.DeviceKeyframe.from_cloud(torch.as_tensor(G[f"{case}_cloud"], device="cuda"), SE3Pose.identity(),
                                      int(c[0]), int(c[1]), camera=kf.camera)
    assert np.array_equal(dk.nvalid.cpu().numpy().astype(bool), G[f"{case}_nvalid"])
    assert np.array_equal(dk.range.cpu().numpy(), G[f"{case}_range"].astype(np.float32))


def test_no_wrap_edges_and_sparse_windows(cuda):
    """Unwrapped columns clamp like ndimage's 'nearest'; windows with five or more
    invalid pixels keep the original range (oracle comparison, random sparse image)."""
    rng = np.random.default_rng(4)
    H, W = 20, 37
    r = rng.uniform(1.0, 30.0, (H, W))
    v = rng.random((H, W)) > 0.45
    r[~v] = 0.0
    for wrap in (False, True):
        got = KF.smooth_range_image(KF.RangeImage(r, v), wrap)
        assert np.array_equal(got.range, KO.smooth_range_image(r, v, wrap))
