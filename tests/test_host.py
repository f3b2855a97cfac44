"""Host-side logic without a GPU: camera constants, workloads, error mapping."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2503_17491_b200 import (BlendRecords, GeometryError, PixelGradients, RasterConfig, SE3Pose, SplatModel,
                                   SphericalCamera, rasterize_backward, se3_exp)
from paper_2503_17491_b200 import workloads as W
from paper_2503_17491_b200._lib import check


@pytest.mark.parametrize("cam", [W.synth_camera(1024, 64), W.synth_camera(2048, 128),
                                 SphericalCamera(64, 16, -np.pi, np.pi, -0.349, 0.262),
                                 SphericalCamera(96, 24, -1.0, 0.7, -0.35, 0.25)])
def test_camera_constants_match_oracle(cam):
    k = O.intrinsics((cam.width, cam.height, cam.az_min, cam.az_max, cam.el_min, cam.el_max))
    assert np.array_equal(k, [cam.fx, cam.fy, cam.cx, cam.cy, *cam.grid_offset])
    d, _, _, _ = O.pixel_planes((cam.width, cam.height, cam.az_min, cam.az_max, cam.el_min, cam.el_max))
    assert np.abs(d - cam.pixel_directions).max() < 1e-15


def test_raster_config_defaults():
    c = RasterConfig()
    assert (c.tile_size, c.chunk_size, c.alpha_cutoff, c.alpha_clamp, c.min_transmittance, c.denom_eps) == \
        (8, 256, 1 / 255, 0.99, 1e-4, 1e-12)
    assert abs(c.cutoff_sigma - np.sqrt(2 * np.log(255))) < 1e-15
    assert c.bbox_pad_px == 0.5


def test_workloads_deterministic_and_float32():
    a = W.random_splats(1000, 5)
    b = W.random_splats(1000, 5)
    for k in a:
        assert a[k].dtype == np.float32
        assert np.array_equal(a[k], b[k])
    assert a["centers"][:, 2].min() >= -2.0 and a["centers"][:, 2].max() <= 6.0
    r = np.linalg.norm(a["centers"][:, :2], axis=1)
    assert r.max() <= 50.0 + 1e-3


def test_stale_records_raise_geometry_error():
    m = SplatModel(np.zeros((3, 3)) + 5.0)
    rec = BlendRecords(W.synth_camera(64, 16), SE3Pose.identity(), RasterConfig(), 3, m.version, 8, 2)
    m.touch()
    with pytest.raises(GeometryError):
        rasterize_backward(m, rec, None, PixelGradients(None, None, None))


def test_status_mapping():
    check(0)
    with pytest.raises(GeometryError):
        check(2, "x")
    with pytest.raises(RuntimeError):
        check(4, "x")


def test_se3_exp_round_trip():
    d = np.array([0.1, -0.2, 0.3, 0.01, 0.02, -0.03])
    T = se3_exp(d)
    assert np.allclose(T.rotation.T @ T.rotation, np.eye(3), atol=1e-12)
    assert np.allclose(SE3Pose.identity().retract(d).translation, T.translation)


def test_device_cache_key_sees_inplace_edits():
    """The float32 device copy of a model is reused only while the parameter arrays are
    unchanged: in-place edits without touch() (which the reference's version counter
    would not see) and array reassignment both change the key."""
    import numpy as np
    from paper_2503_17491_b200 import SplatModel
    from paper_2503_17491_b200 import workloads as W
    from paper_2503_17491_b200.rasterizer import _cache_key
    m = SplatModel.from_params(W.random_splats(1000, 3))
    k0 = _cache_key(m)
    assert _cache_key(m) == k0
    m.centers[5, 1] += 1e-3
    k1 = _cache_key(m)
    assert k1 != k0
    m.log_scales[[0, 1]] = m.log_scales[[1, 0]]  # a row swap keeps sums: position-sensitive key
    assert _cache_key(m) != k1
    k2 = _cache_key(m)
    m.logit_opacity = m.logit_opacity.copy()  # same values, new array
    assert _cache_key(m) != k2
    m.touch()
    assert _cache_key(m)[0][0] == m.version
