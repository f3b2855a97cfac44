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


def test_host_stage_rounding_and_fingerprints():
    """ss_host_stage_f64 (host only): float32 staging equals numpy's round-to-nearest cast bit
    for bit (subnormals, huge values, NaN/inf included), the float64 copy is exact, and the
    fingerprint is chunk-invariant and sees a one-ulp edit."""
    import ctypes

    import numpy as np

    from paper_2503_17491_b200 import engine
    from paper_2503_17491_b200._lib import lib

    rng = np.random.default_rng(3)
    a = np.concatenate([rng.normal(size=100_001) * 10.0 ** rng.integers(-50, 50, 100_001),
                        [1e-45, 3e-39, 1e39, -0.0, np.inf, -np.inf, np.nan, 2.0 ** -149, 1.0 + 2.0 ** -24]])
    f32 = np.empty(a.size, np.float32)
    f64 = np.empty(a.size, np.float64)
    fp = ctypes.c_uint64()
    assert lib().ss_host_stage_f64(a.ctypes.data, f32.ctypes.data, 1, a.size, 0, ctypes.byref(fp)) == 0
    with np.errstate(over="ignore"):
        assert np.array_equal(f32.view(np.uint32), a.astype(np.float32).view(np.uint32))
    assert lib().ss_host_stage_f64(a.ctypes.data, f64.ctypes.data, 0, a.size, 0, ctypes.byref(fp)) == 0
    assert np.array_equal(f64.view(np.uint64), a.view(np.uint64))
    whole = fp.value
    parts = 0
    for b in range(0, a.size, 7_777):
        e = min(b + 7_777, a.size)
        lib().ss_host_stage_f64(a[b:].ctypes.data, None, 0, e - b, b, ctypes.byref(fp))
        parts += fp.value
    assert parts % 2 ** 64 == whole == engine.fingerprints([a])[0]
    b = a.copy()
    b[5] = np.nextafter(b[5], np.inf)
    assert engine.fingerprints([b])[0] != whole
    c = a.copy()
    c[[10, 11]] = c[[11, 10]]
    assert engine.fingerprints([c])[0] != whole
