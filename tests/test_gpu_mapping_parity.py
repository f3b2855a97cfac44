"""Config-2 mapping parity against the oracle (oracle/mapping_oracle.py restates
mapping.py:128-196 and :342-379, 474-497; oracle.c the rasterizer).

1. The fused loss kernels term by term: ``ss_mapping_loss`` pixel gradients
   dD / dN / dO and loss parts, ``ss_scale_loss`` gradient and hinge value, on a
   config-2 render, against the numpy restatement evaluated on the same images.
2. Three refine iterations of the config-2 map (grown by DeviceMap.start + 9
   add_keyframe, 200k surfels, 64x1024): at every iteration the device raw
   gradient against the C oracle's (render, mapping loss, backward, raw chain)
   at the device's current parameters, per class within 1e-3 norm-wise
   (BASELINE north star), and the fused Adam update against numpy Adam on the
   device gradient.
"""
import ctypes

import numpy as np
import pytest
import torch

from oracle import mapping_oracle as MO
from oracle import oracle as O
from paper_2503_17491_b200 import engine
from paper_2503_17491_b200 import mapping as MP
from paper_2503_17491_b200 import workloads as W
from paper_2503_17491_b200._lib import check, lib
from paper_2503_17491_b200.geometry import pose_rt

pytestmark = pytest.mark.gpu

CLASSES = {"centers": slice(0, 3), "raw_t_alpha": slice(3, 6), "raw_t_beta": slice(6, 9), "log_scales": slice(9, 11),
           "logit_opacity": slice(11, 12)}


@pytest.fixture(scope="module")
def config2(cuda):
    targets = W.keyframe_targets(10, 0, 1024, 64)
    dkfs = W.device_keyframes(targets)
    dm = W.build_local_map(dkfs, 20_000, 0)
    return targets, dkfs, dm


def _kf_host(tg):
    return {"range": tg["range"].astype(np.float64), "valid": tg["valid"].astype(bool),
            "normal": tg["normal"].astype(np.float64), "nvalid": tg["nvalid"].astype(bool)}


def test_config2_map_size(config2):
    _, _, dm = config2
    assert dm.n == 200_000  # the spawn cap of 20k per keyframe gives exactly 200,000


def test_mapping_loss_terms_match_oracle(config2):
    targets, dkfs, dm = config2
    cfg = MP.MappingConfig()
    for k in (0, 6):
        kf = dkfs[k]
        D, N, Op = engine.forward(kf.camera, pose_rt(kf.pose), dm.params, MP.RasterConfig(), dm.rec)
        dD, dN, dO, parts = engine.mapping_loss(D, N, Op, kf.range, kf.valid, kf.normal, kf.nvalid,
                                                w_opacity=cfg.w_opacity, w_normal=cfg.w_normal,
                                                range_floor=cfg.range_weight_floor)
        ds = torch.empty((dm.n, 2), dtype=torch.float32, device="cuda")
        check(lib().ss_scale_loss(ctypes.c_void_p(dm.params["log_scales"].data_ptr()), dm.n, float(cfg.scale_cap),
                                  float(cfg.w_scale), ctypes.c_void_p(ds.data_ptr()),
                                  ctypes.c_void_p(parts.data_ptr() + 3 * 8), ctypes.c_void_p(engine.stream_ptr())),
              "scale_loss")
        Dh, Nh, Oh = (x.cpu().numpy().astype(np.float64) for x in (D, N, Op))
        ls = dm.params["log_scales"].cpu().numpy().astype(np.float64)
        total, gD, gN, gO, gS, ref = MO.mapping_loss(Dh, Nh, Oh, _kf_host(targets[k][2]), ls, cfg)
        got = parts.cpu().numpy()
        for i, name in enumerate(("range", "opacity", "normal", "scale")):
            assert abs(got[i] - ref[name]) <= 1e-9 * max(abs(ref[name]), 1.0), (name, got[i], ref[name])
        # pixel gradients: same support, float32 rounding of the float64 values
        for a, b in ((dD, gD), (dN, gN), (dO, gO)):
            a = a.cpu().numpy().astype(np.float64)
            assert np.array_equal(a != 0, b != 0)
            assert np.abs(a - b).max() <= 1e-6 * max(np.abs(b).max(), 1e-30)
        assert np.array_equal(ds.cpu().numpy().astype(np.float64), gS)
        print(f"kf {k}: parts {got} total {total}")


def test_three_refine_iterations_match_oracle(config2):
    targets, dkfs, dm0 = config2
    cfg = MP.MappingConfig()
    dm = MP.DeviceMap({k: v.clone() for k, v in dm0.params.items()}, dkfs, dm0.scene_scale)
    x = MO.flat({k: v.cpu().numpy().astype(np.float64) for k, v in dm.params.items()})
    opt = MO.Adam(x.shape[0], cfg, dm.scene_scale)
    rng = np.random.default_rng(3)
    for it in range(3):
        k = MP.sample_keyframe_index(len(dkfs), cfg.kf_sample_p, rng)
        g_dev, parts = dm.raw_gradient(k, cfg)
        g_dev = g_dev.cpu().numpy().astype(np.float64)
        # the oracle at the device's current parameters (float32 values promoted)
        xd = MO.flat({kk: v.cpu().numpy().astype(np.float64) for kk, v in dm.params.items()})
        p = MO.unflat(xd)
        cam, pose, tg = targets[k]
        ct = (cam.width, cam.height, cam.az_min, cam.az_max, cam.el_min, cam.el_max)
        r = O.render(ct, pose.rotation, pose.translation, p)
        total, gD, gN, gO, gS, _ = MO.mapping_loss(r["range"], r["normal"], r["opacity"], _kf_host(tg),
                                                   p["log_scales"], cfg)
        plain = O.backward_lists(ct, r["arr"], pose.rotation, r["tile_ptr"], r["pair_splats"], r["range"],
                                 r["normal"], r["opacity"], gD, gN, gO)
        g_ref = O.raw_gradients(p, plain, gS)
        w = np.array([1.0, cfg.w_opacity, cfg.w_normal, cfg.w_scale])
        loss_dev = float(parts.cpu().numpy() @ w)
        assert abs(loss_dev - total) <= 1e-4 * abs(total), (it, loss_dev, total)
        for name, sl in CLASSES.items():
            rel = np.linalg.norm(g_dev[:, sl] - g_ref[:, sl]) / max(np.linalg.norm(g_ref[:, sl]), 1e-30)
            print(f"iter {it} kf {k} {name}: gradient rel err {rel:.2e}")
            assert rel <= 1e-3, (it, name, rel)
        # fused Adam == numpy Adam on the same (device) gradient
        before = xd.copy()
        dm.apply_adam(torch.tensor(g_dev, dtype=torch.float32, device="cuda"), cfg)
        opt.step(xd, g_dev.astype(np.float32).astype(np.float64))
        after = MO.flat({kk: v.cpu().numpy().astype(np.float64) for kk, v in dm.params.items()})
        # per element: float32 storage (a few ulp of the parameter) + float32 step arithmetic
        allow = 3 * np.spacing(np.abs(xd).astype(np.float32)).astype(np.float64) + 1e-5 * np.abs(xd - before) + 1e-12
        bad = np.abs(after - xd) > allow
        assert bad.sum() <= 1e-5 * bad.size, (it, int(bad.sum()))
