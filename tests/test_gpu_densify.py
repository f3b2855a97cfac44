"""Device map growth (DeviceMap.start / add_keyframe: spawn weights, densify mask, prune,
spawn) against the live reference (tests/golden/golden_densify.npz): LocalMap.start on
keyframe 0 and add_keyframe with keyframe 1, same numpy RNG stream."""
import ctypes
import os

import numpy as np
import pytest
import torch

from paper_2503_17491_b200 import SE3Pose, SphericalCamera, engine
from paper_2503_17491_b200 import mapping as MP
from paper_2503_17491_b200._lib import check, lib
from paper_2503_17491_b200.geometry import pose_rt

pytestmark = pytest.mark.gpu

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_densify.npz"))
NAMES = ("centers", "raw_t_alpha", "raw_t_beta", "log_scales", "logit_opacity")


def _kf(i):
    c = G[f"kf{i}_cam"]
    cam = SphericalCamera(int(c[0]), int(c[1]), *[float(x) for x in c[2:]])
    return MP.DeviceKeyframe(cam, SE3Pose(G[f"kf{i}_R"], G[f"kf{i}_t"]), G[f"kf{i}_range"], G[f"kf{i}_valid"],
                             G[f"kf{i}_normal"], G[f"kf{i}_nvalid"], i)


def _close(dm, prefix):
    for k in NAMES:
        got = dm.params[k].cpu().numpy().astype(np.float64).reshape(G[f"{prefix}_{k}"].shape)
        ref = G[f"{prefix}_{k}"].astype(np.float32).astype(np.float64)
        assert got.shape == ref.shape, (k, got.shape, ref.shape)
        assert np.abs(got - ref).max() <= 1e-6 * max(1.0, np.abs(ref).max()), k


def test_spawn_weights(cuda):
    for i in (0, 1):
        kf = _kf(i)
        w = torch.empty_like(kf.range64)
        check(lib().ss_spawn_weights(kf.camera.width, kf.camera.height, int(bool(kf.camera.full_circle)),
                                     ctypes.c_void_p(kf.range64.data_ptr()), ctypes.c_void_p(kf.valid.data_ptr()),
                                     ctypes.c_void_p(w.data_ptr()), ctypes.c_void_p(engine.stream_ptr())), "w")
        ref = G[f"kf{i}_gradw"]
        assert np.abs(w.cpu().numpy() - ref).max() <= 1e-12 * max(1.0, ref.max())


def test_start_and_add_keyframe(cuda):
    cfg = MP.MappingConfig(n_spawn=1000)
    rng = np.random.default_rng(21)
    dm = MP.DeviceMap.start(_kf(0), cfg, rng)
    assert dm.scene_scale == pytest.approx(float(G["scene_scale"]), rel=1e-15)
    _close(dm, "s")
    dm.params["logit_opacity"][7] = -8.0  # as the golden run, so the add prunes one splat
    kf1 = _kf(1)
    # the densify mask of the float32 render against the reference's float64 one
    D, N, O = engine.forward(kf1.camera, pose_rt(kf1.pose), dm.params, MP.RasterConfig(), dm.rec)
    mask = torch.empty_like(kf1.valid)
    check(lib().ss_densify_mask(int(kf1.valid.numel()), ctypes.c_void_p(kf1.range64.data_ptr()),
                                ctypes.c_void_p(kf1.valid.data_ptr()), ctypes.c_void_p(D.data_ptr()),
                                ctypes.c_void_p(O.data_ptr()), cfg.densify_opacity, cfg.densify_range_err,
                                ctypes.c_void_p(mask.data_ptr()), ctypes.c_void_p(engine.stream_ptr())), "mask")
    diff = int((mask.cpu().numpy().astype(bool) != G["mask1"]).sum())
    print("densify mask pixels differing from the reference:", diff, "of", int(G["mask1"].sum()))
    assert diff == 0
    stats = dm.add_keyframe(kf1, cfg, rng)
    assert stats == {"pruned": int(G["pruned"]), "spawned": int(G["spawned"])}
    _close(dm, "a")
    assert np.array_equal(dm.epochs.cpu().numpy(), G["epochs"].astype(np.int32))
    assert dm.m.shape[0] == dm.n and not dm.m.any()
