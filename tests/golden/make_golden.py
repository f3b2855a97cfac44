"""Generate golden vectors from the LIVE reference (run in the build container).

The reference package `splatscan` is importable here from
/root/reference/pkg/src; it does not exist on the GPU box, so its outputs are
frozen into small .npz fixtures committed next to this script.  The fixtures
pin the CPU oracle (oracle/) and, through it, the CUDA path.

Cases (inputs are float32-rounded values promoted to float64, exactly what the
GPU path consumes):
  full      64x16 full-circle camera of pkg/tests/conftest.py:15-17, 300 splats
            on a 2-8 m shell with 25% forced behind the sensor, random pose
  synth     128x32 synth-grid camera (synth.py:277-281), config-0-style draw of
            2000 splats, identity pose, extra splats on the seam
  partial   96x24 partial field of view, 400 splats, random pose
  tile16    the `full` inputs rendered with tile_size=16
Each case stores the reference's tile lists, images, plain-space gradients for
seeded pixel gradients, and raw-space gradients (mapping.py:479-494).
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from splatscan.geometry import SphericalCamera  # noqa: E402
from splatscan.rasterizer import (PixelGradients, RasterConfig, rasterize_backward,  # noqa: E402
                                  rasterize_forward, reference_rasterize)
from splatscan.se3 import SE3Pose, so3_exp  # noqa: E402
from splatscan.splats import SplatModel, tangent_raw_gradients  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def quat_frames(q):
    q = q / np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    ta = np.stack([1 - 2 * (y * y + z * z), 2 * (x * y + w * z), 2 * (x * z - w * y)], axis=1)
    tb = np.stack([2 * (x * y - w * z), 1 - 2 * (x * x + z * z), 2 * (y * z + w * x)], axis=1)
    return ta, tb


def shell_model(rng, n, rmin, rmax, behind=0.0, zclip=None, mean_log_s=np.log(0.05), sig=0.5):
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    if behind > 0:
        k = int(n * behind)
        d[:k, 0] = -np.abs(d[:k, 0])
    c = d * rng.uniform(rmin, rmax, n)[:, None]
    if zclip is not None:
        c[:, 2] = np.clip(c[:, 2], *zclip)
    ls = rng.normal(mean_log_s, sig, (n, 2))
    ta, tb = quat_frames(rng.normal(size=(n, 4)))
    lo = rng.normal(0.0, 1.0, n)
    return dict(centers=c, raw_t_alpha=ta, raw_t_beta=tb, log_scales=ls, logit_opacity=lo)


def to_model(p):
    p = {k: f32(v) for k, v in p.items()}
    m = SplatModel(p["centers"], p["raw_t_alpha"], p["raw_t_beta"], p["log_scales"], p["logit_opacity"])
    return m, p


def random_pose(rng, rot_deg=20.0, trans=0.5):
    R = so3_exp(np.deg2rad(rot_deg) * rng.normal(size=3) / np.sqrt(3))
    return SE3Pose(R, rng.normal(size=3) * trans)


def make_case(name, cam, model, params, pose, cfg, rng):
    render, rec = rasterize_forward(cam, pose, model, cfg)
    H, W = cam.height, cam.width
    gD = rng.choice([-1.0, 1.0], size=(H, W)) * (render.opacity > 0)
    gN = 0.1 * rng.normal(size=(H, W, 3))
    gO = 0.05 * rng.normal(size=(H, W))
    g = rasterize_backward(model, rec, render, PixelGradients(gD, gN, gO))
    plain = np.concatenate([g.d_centers, g.d_t_alpha, g.d_t_beta, g.d_normal, g.d_scales,
                            g.d_opacity[:, None]], axis=1)
    ga, gb = tangent_raw_gradients(model.raw_t_alpha, model.raw_t_beta, g.d_t_alpha, g.d_t_beta, g.d_normal)
    s = model.scales
    o = model.opacities
    raw = np.concatenate([g.d_centers, ga, gb, g.d_scales * s, (g.d_opacity * o * (1 - o))[:, None]], axis=1)
    brute = reference_rasterize(cam, pose, model, cfg) if W * H <= 4096 else None
    bz = np.zeros(0)
    np.savez_compressed(
        os.path.join(OUT, f"golden_{name}.npz"),
        cam=np.array([cam.width, cam.height, cam.az_min, cam.az_max, cam.el_min, cam.el_max]),
        tile_size=cfg.tile_size, R=pose.rotation, t=pose.translation,
        fx=cam.fx, fy=cam.fy, cx=cam.cx, cy=cam.cy, grid_offset=cam.grid_offset,
        dirs=cam.pixel_directions if W * H <= 2048 else np.zeros(0),
        **{f"p_{k}": v for k, v in params.items()},
        tile_ptr=rec.tile_ptr, pair_splats=rec.pair_splats, tiles_x=rec.tiles_x, tiles_y=rec.tiles_y,
        range=render.range, normal=render.normal, opacity=render.opacity,
        brute_range=brute.range if brute else bz, brute_normal=brute.normal if brute else bz,
        brute_opacity=brute.opacity if brute else bz,
        gD=gD, gN=gN, gO=gO, plain=plain, raw=raw,
    )
    print(name, "pairs", rec.pair_splats.shape[0], "covered px", int((render.opacity > 0).sum()))


def main():
    rng = np.random.default_rng(20251019)
    # full-circle conftest camera, behind-sensor splats, random pose
    cam = SphericalCamera(64, 16, -np.pi, np.pi, -np.deg2rad(20.0), np.deg2rad(15.0))
    p = shell_model(rng, 300, 2.0, 8.0, behind=0.25, mean_log_s=np.log(0.15), sig=0.4)
    m, p = to_model(p)
    pose = random_pose(rng)
    make_case("full", cam, m, p, pose, RasterConfig(), rng)
    make_case("tile16", cam, m, p, pose, RasterConfig(tile_size=16), rng)
    # synth-grid camera, config-0 style draw, seam splats
    W, H = 128, 32
    cam = SphericalCamera(W, H, -np.pi, np.pi - 2 * np.pi / W, -np.deg2rad(22.5), np.deg2rad(22.5))
    p = shell_model(rng, 2000, 2.0, 50.0, zclip=(-2.0, 6.0), mean_log_s=np.log(0.3))
    k = 60  # centres straddling the azimuth seam
    az = np.pi + rng.normal(0, 0.02, k)
    r = rng.uniform(3, 20, k)
    p["centers"][:k] = np.stack([r * np.cos(az), r * np.sin(az), rng.uniform(-1, 2, k)], axis=1)
    m, p = to_model(p)
    make_case("synth", cam, m, p, SE3Pose.identity(), RasterConfig(), rng)
    # partial field of view
    cam = SphericalCamera(96, 24, -1.0, 0.7, -0.35, 0.25)
    p = shell_model(rng, 400, 2.0, 12.0, mean_log_s=np.log(0.2), sig=0.4)
    p["centers"][:, 0] = np.abs(p["centers"][:, 0])
    m, p = to_model(p)
    make_case("partial", cam, m, p, random_pose(rng, 5.0, 0.2), RasterConfig(), rng)


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def make_registration_case():
    """Photometric registration on a small room scene (registration.py:387-524)."""
    from splatscan import registration as REG
    from splatscan.registration import RegistrationConfig, register
    from splatscan.synth import ScanSpec, raycast_scan, room_with_boxes

    rng = np.random.default_rng(7)
    scene = room_with_boxes(n_boxes=4, seed=0)
    spec = ScanSpec(width=256, height=32)
    truth = SE3Pose(so3_exp(np.deg2rad([0.0, 0.0, 10.0])), np.array([0.3, -0.2, 0.1]))
    sc = raycast_scan(scene, truth, spec)
    scan_pts = f32(sc.cloud)
    # splats on the visible surfaces (pkg/tests/conftest.py:38-51), float32-rounded
    pts, normals = scene.visible_surface_points(9000, np.zeros((1, 3)), rng)
    idx = rng.choice(pts.shape[0], min(3000, pts.shape[0]), replace=False)
    pts, normals = pts[idx], normals[idx]
    ref = np.where(np.abs(normals[:, 2:3]) < 0.9, [[0.0, 0.0, 1.0]], [[1.0, 0.0, 0.0]])
    ta = np.cross(normals, ref)
    ta /= np.linalg.norm(ta, axis=1, keepdims=True)
    tb = np.cross(normals, ta)
    p = dict(centers=pts, raw_t_alpha=ta, raw_t_beta=tb, log_scales=np.full((len(pts), 2), np.log(0.12)),
             logit_opacity=np.full(len(pts), np.log(0.95 / 0.05)))
    model, p = to_model(p)
    initial = truth.compose(SE3Pose(so3_exp(np.deg2rad([1.0, -1.5, 2.0])), np.array([0.12, -0.08, 0.05])))
    cfg = RegistrationConfig(mode="photometric", max_iters=15)
    cam = sc.camera
    # one linearisation at a pose off the anchor grid (at `initial` itself the
    # anchors re-project exactly onto scan grid lines, where floor() is decided
    # by the last ulp of numpy's own atan2)
    T0 = initial.retract(np.array([2e-3, -1e-3, 1e-3, 1e-3, 2e-3, -1e-3]))
    geo_cam = SphericalCamera(cam.width * 2, cam.height * 2, cam.az_min, cam.az_max, cam.el_min, cam.el_max)
    model_pts, _, _ = REG.sample_model(model, geo_cam, initial, cfg)
    X_w = model_pts[::4]
    scan_img = REG.build_range_image(cam, scan_pts)
    sysr = REG._photo_system(X_w, scan_img, cam, T0, cfg, max(cfg.trim_floor_photo, 0.5))
    r, J = sysr
    w = REG._huber_weights(r, cfg.huber_photo)
    H0 = (J.T * w) @ J
    b0 = J.T @ (w * r)
    res = register(model, scan_pts, cam, initial, cfg)
    np.savez_compressed(
        os.path.join(OUT, "golden_register.npz"),
        cam=np.array([cam.width, cam.height, cam.az_min, cam.az_max, cam.el_min, cam.el_max]),
        **{f"p_{k}": np.asarray(v, np.float32) for k, v in p.items()},
        scan=np.asarray(scan_pts, np.float32), initial_R=initial.rotation, initial_t=initial.translation,
        T0_R=T0.rotation, T0_t=T0.translation,
        truth_R=truth.rotation, truth_t=truth.translation, n_model_pts=model_pts.shape[0], X_w=X_w,
        scan_range=scan_img.range, scan_valid=scan_img.valid, H0=H0, b0=b0, m0=r.shape[0],
        huber0=REG._huber_value(r, cfg.huber_photo), sum_r2_0=float(r @ r),
        final_R=res.pose.rotation, final_t=res.pose.translation, iterations=res.iterations,
        converged=res.converged, photo_rms=res.photo_rms, n_photo=res.n_photo,
    )
    err_t = np.linalg.norm(res.pose.translation - truth.translation)
    print("register: anchors", X_w.shape[0], "m0", r.shape[0], "iters", res.iterations, "err_t", err_t)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "register":
    make_registration_case()


def make_refine_case():
    """Three refine() iterations of a small two-keyframe local map (mapping.py:455-498)."""
    from splatscan.mapping import LocalMap, MappingConfig, add_keyframe, make_keyframe, refine
    from splatscan.synth import ScanSpec, raycast_scan, room_with_boxes

    scene = room_with_boxes(n_boxes=3, seed=1)
    spec = ScanSpec(width=128, height=16)
    cfg = MappingConfig(n_spawn=1200)
    rng = np.random.default_rng(11)
    poses = [SE3Pose.identity(), SE3Pose(so3_exp(np.deg2rad([0, 0, 4.0])), np.array([0.4, 0.1, 0.0]))]
    kfs = [make_keyframe(i, raycast_scan(scene, p, spec).cloud, p, spec.width, spec.height) for i, p in enumerate(poses)]
    lmap = LocalMap.start(kfs[0], cfg, rng)
    add_keyframe(lmap, kfs[1], cfg, rng)
    m = lmap.model
    for k in ("centers", "raw_t_alpha", "raw_t_beta", "log_scales", "logit_opacity"):
        getattr(m, k)[...] = f32(getattr(m, k))
    # the device consumes float32 images: make the reference's float64 ones exactly representable
    for kf in kfs:
        kf.range_image.range[...] = f32(kf.range_image.range)
        kf.normal_image.normals[...] = f32(kf.normal_image.normals)
    before = {k: getattr(m, k).copy() for k in ("centers", "raw_t_alpha", "raw_t_beta", "log_scales", "logit_opacity")}
    rng_state = np.random.default_rng(99)
    losses = refine(lmap, cfg, 3, rng_state)
    after = {k: getattr(m, k).copy() for k in before}
    out = {f"b_{k}": v for k, v in before.items()}
    out.update({f"a_{k}": v for k, v in after.items()})
    for i, kf in enumerate(kfs):
        c = kf.camera
        out[f"kf{i}_cam"] = np.array([c.width, c.height, c.az_min, c.az_max, c.el_min, c.el_max])
        out[f"kf{i}_R"] = kf.pose.rotation
        out[f"kf{i}_t"] = kf.pose.translation
        out[f"kf{i}_range"] = kf.range_image.range.astype(np.float32)
        out[f"kf{i}_valid"] = kf.range_image.valid
        out[f"kf{i}_normal"] = kf.normal_image.normals.astype(np.float32)
        out[f"kf{i}_nvalid"] = kf.normal_image.valid
    np.savez_compressed(os.path.join(OUT, "golden_refine.npz"), scene_scale=lmap.scene_scale, losses=np.array(losses),
                        adam_t=lmap.optimizer.t, **out)
    print("refine: splats", len(m), "losses", losses)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "refine":
    make_refine_case()


def make_keyframe_case():
    """make_keyframe's images (mapping.py:106-114): range image, 3x3 median smoothing and
    normals, for a full-circle scan (seam wrap) and a noisy partial-field-of-view crop."""
    from splatscan.geometry import build_range_image, estimate_camera, range_image_normals, smooth_range_image
    from splatscan.synth import ScanSpec, raycast_scan, room_with_boxes

    rng = np.random.default_rng(5)
    scene = room_with_boxes(n_boxes=5, seed=2)
    spec = ScanSpec(width=256, height=32)
    pose = SE3Pose(so3_exp(np.deg2rad([0.0, 0.0, 25.0])), np.array([0.5, -0.3, 0.2]))
    full = f32(raycast_scan(scene, pose, spec).cloud)
    noisy = full * (1.0 + 0.003 * rng.normal(size=(full.shape[0], 1)))
    az = np.arctan2(noisy[:, 1], noisy[:, 0])
    part = f32(noisy[(az > -1.2) & (az < 1.7)])
    out = {}
    for name, cloud, (W, H) in (("full", full, (256, 32)), ("part", part, (118, 32))):
        cam = estimate_camera(cloud, W, H)
        rimg = build_range_image(cam, cloud)
        sm = smooth_range_image(rimg, cam.full_circle)
        nimg = range_image_normals(cam, sm)
        out[f"{name}_cloud"] = cloud
        out[f"{name}_cam"] = np.array([cam.width, cam.height, cam.az_min, cam.az_max, cam.el_min, cam.el_max])
        out[f"{name}_full_circle"] = np.array(cam.full_circle)
        out[f"{name}_range"] = rimg.range
        out[f"{name}_valid"] = rimg.valid
        out[f"{name}_smooth"] = sm.range
        out[f"{name}_normals"] = nimg.normals
        out[f"{name}_nvalid"] = nimg.valid
        print(name, "points", cloud.shape[0], "valid", int(rimg.valid.sum()), "normals", int(nimg.valid.sum()),
              "full circle", cam.full_circle, "smoothed changed", int((sm.range != rimg.range).sum()))
    np.savez_compressed(os.path.join(OUT, "golden_keyframe.npz"), **out)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "keyframe":
    make_keyframe_case()


def make_geometric_case():
    """The geometric half of registration (registration.py:98-164, 231-274, 387-524) on the
    inputs of golden_register.npz: the leaf tree of the model points, one _geo_system
    linearisation, and register() in the geometric, joint and sequential modes."""
    from splatscan import registration as REG
    from splatscan.registration import RegistrationConfig, register

    G = np.load(os.path.join(OUT, "golden_register.npz"))
    c = G["cam"]
    cam = SphericalCamera(int(c[0]), int(c[1]), *[float(x) for x in c[2:]])
    p = {k[2:]: G[k].astype(np.float64) for k in G.files if k.startswith("p_")}
    model, _ = to_model(p)
    scan = G["scan"].astype(np.float64)
    initial = SE3Pose(G["initial_R"], G["initial_t"])
    T0 = SE3Pose(G["T0_R"], G["T0_t"])
    cfg = RegistrationConfig()
    geo_cam = SphericalCamera(cam.width * 2, cam.height * 2, cam.az_min, cam.az_max, cam.el_min, cam.el_max)
    model_pts, _, _ = REG.sample_model(model, geo_cam, initial, cfg)
    tree = REG.build_leaf_tree(model_pts, initial.translation, cfg.leaf_size, cfg.flatness_tau)
    sel = np.random.default_rng(0).choice(scan.shape[0], cfg.max_geo_points, replace=False)
    geo_scan = scan[sel]
    r, J = REG._geo_system(tree, geo_scan, T0, cfg, max(cfg.trim_floor_geo, 0.5))
    w = REG._huber_weights(r, cfg.huber_geo)
    out = dict(model_pts=model_pts, point_leaf=tree.point_leaf, leaf_centroids=tree.centroids,
               leaf_normals=tree.normals, leaf_sizes=tree.sizes, leaf_usable=tree.usable, geo_sel=sel,
               geo_H0=(J.T * w) @ J, geo_b0=J.T @ (w * r), geo_m0=r.shape[0],
               geo_huber0=REG._huber_value(r, cfg.huber_geo), geo_r0=r)
    for mode, iters in (("geometric", 15), ("joint", 15), ("sequential", 30)):
        res = register(model, scan, cam, initial, RegistrationConfig(mode=mode, max_iters=iters))
        out.update({f"{mode}_R": res.pose.rotation, f"{mode}_t": res.pose.translation,
                    f"{mode}_iterations": res.iterations, f"{mode}_converged": res.converged,
                    f"{mode}_geo_rms": res.geo_rms, f"{mode}_photo_rms": res.photo_rms,
                    f"{mode}_n_geo": res.n_geo, f"{mode}_n_photo": res.n_photo})
        print(mode, "iters", res.iterations, "converged", res.converged, "n_geo", res.n_geo, "n_photo", res.n_photo,
              "err_t", np.linalg.norm(res.pose.translation - G["truth_t"]))
    print("model_pts", model_pts.shape[0], "leaves", tree.sizes.shape[0], "usable", int(tree.usable.sum()),
          "geo m0", r.shape[0])
    np.savez_compressed(os.path.join(OUT, "golden_register_geo.npz"), **out)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "geometric":
    make_geometric_case()


def make_densify_case():
    """Map growth (mapping.py:202-311, 383-438): LocalMap.start on keyframe 0 (spawn at every
    valid pixel, capped: weighted draw without replacement), then add_keyframe with keyframe 1
    (render, densify mask, prune, spawn), float64 keyframe images kept as they were used."""
    from splatscan.mapping import LocalMap, MappingConfig, _range_gradient_weights, add_keyframe, densify_mask, \
        make_keyframe
    from splatscan.rasterizer import rasterize_forward as rf
    from splatscan.synth import ScanSpec, raycast_scan, room_with_boxes

    scene = room_with_boxes(n_boxes=4, seed=3)
    spec = ScanSpec(width=128, height=16)
    cfg = MappingConfig(n_spawn=1000)
    poses = [SE3Pose.identity(), SE3Pose(so3_exp(np.deg2rad([0, 0, 6.0])), np.array([0.5, 0.2, 0.0]))]
    kfs = [make_keyframe(i, raycast_scan(scene, p, spec).cloud, p, spec.width, spec.height) for i, p in enumerate(poses)]
    rng = np.random.default_rng(21)
    lmap = LocalMap.start(kfs[0], cfg, rng)
    m0 = lmap.model
    after_start = {k: getattr(m0, k).copy() for k in ("centers", "raw_t_alpha", "raw_t_beta", "log_scales",
                                                         "logit_opacity")}
    # make one splat prunable so add_keyframe exercises the compaction
    lmap.model.logit_opacity[7] = -8.0
    render, _ = rf(kfs[1].camera, kfs[1].pose, lmap.model)
    mask1 = densify_mask(render, kfs[1], cfg)
    stats = add_keyframe(lmap, kfs[1], cfg, rng)
    out = {f"s_{k}": v for k, v in after_start.items()}
    out.update({f"a_{k}": getattr(lmap.model, k).copy() for k in after_start})
    for i, kf in enumerate(kfs):
        c = kf.camera
        out[f"kf{i}_cam"] = np.array([c.width, c.height, c.az_min, c.az_max, c.el_min, c.el_max])
        out[f"kf{i}_R"], out[f"kf{i}_t"] = kf.pose.rotation, kf.pose.translation
        out[f"kf{i}_range"], out[f"kf{i}_valid"] = kf.range_image.range, kf.range_image.valid
        out[f"kf{i}_normal"], out[f"kf{i}_nvalid"] = kf.normal_image.normals, kf.normal_image.valid
        out[f"kf{i}_gradw"] = _range_gradient_weights(kf)
    out.update(scene_scale=lmap.scene_scale, mask1=mask1, pruned=stats["pruned"], spawned=stats["spawned"],
               render1_range=render.range, render1_opacity=render.opacity, epochs=lmap.model.epochs)
    np.savez_compressed(os.path.join(OUT, "golden_densify.npz"), **out)
    print("densify: start", after_start["centers"].shape[0], "after add", len(lmap.model), stats)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "densify":
    make_densify_case()


def depth_rmse_ref(lmap, kfs):
    """Depth RMSE of a local map over its keyframes: rendered range D against the keyframe
    range on valid pixels, and D / O against it on pixels with O > 0.5 (sample_model's
    depth, registration.py:190-213)."""
    se = cnt = se2 = cnt2 = 0.0
    for kf in kfs:
        r, _ = rasterize_forward(kf.camera, kf.pose, lmap.model)
        v = kf.range_image.valid
        se += float(((r.range - kf.range_image.range)[v] ** 2).sum())
        cnt += int(v.sum())
        c = v & (r.opacity > 0.5)
        se2 += float(((r.range / np.maximum(r.opacity, 1e-12) - kf.range_image.range)[c] ** 2).sum())
        cnt2 += int(c.sum())
    return float(np.sqrt(se / max(cnt, 1))), float(np.sqrt(se2 / max(cnt2, 1))), cnt2 / max(cnt, 1)


def make_quality_case(iters=30):
    """A reduced config-2 run of the reference (SURVEY 8(d) config 2 at 512x32, 4 keyframes
    1 m apart, n_spawn 3000): LocalMap.start + add_keyframe (mapping.py:392-438), then
    `iters` refine iterations (mapping.py:455-498); depth RMSE and losses before/after, the
    reference-side quality number bench.py's config-2 line is reported beside."""
    import time

    from splatscan.mapping import LocalMap, MappingConfig, add_keyframe, make_keyframe, refine
    from splatscan.synth import ScanSpec, raycast_scan, room_with_boxes

    scene = room_with_boxes(n_boxes=4, seed=5)
    spec = ScanSpec(width=512, height=32)
    cfg = MappingConfig(n_spawn=3000)
    rng0 = np.random.default_rng(3)
    poses = [SE3Pose(so3_exp([0.0, 0.0, np.deg2rad(2.0) * rng0.normal()]), np.array([0.5 * i, 0.0, 0.0]))
             for i in range(4)]
    kfs = [make_keyframe(i, raycast_scan(scene, p, spec).cloud, p, spec.width, spec.height) for i, p in enumerate(poses)]
    for kf in kfs:  # the device consumes float32 images
        kf.range_image.range[...] = f32(kf.range_image.range)
        kf.normal_image.normals[...] = f32(kf.normal_image.normals)
    rng = np.random.default_rng(17)
    t0 = time.perf_counter()
    lmap = LocalMap.start(kfs[0], cfg, rng)
    for kf in kfs[1:]:
        add_keyframe(lmap, kf, cfg, rng)
    t_build = time.perf_counter() - t0
    n_built = len(lmap.model)
    before = depth_rmse_ref(lmap, kfs)
    t0 = time.perf_counter()
    losses = refine(lmap, cfg, iters, np.random.default_rng(23))
    t_refine = time.perf_counter() - t0
    after = depth_rmse_ref(lmap, kfs)
    out = {}
    for i, kf in enumerate(kfs):
        c = kf.camera
        out[f"kf{i}_cam"] = np.array([c.width, c.height, c.az_min, c.az_max, c.el_min, c.el_max])
        out[f"kf{i}_R"], out[f"kf{i}_t"] = kf.pose.rotation, kf.pose.translation
        out[f"kf{i}_range"] = kf.range_image.range.astype(np.float32)
        out[f"kf{i}_valid"] = kf.range_image.valid
        out[f"kf{i}_normal"] = kf.normal_image.normals.astype(np.float32)
        out[f"kf{i}_nvalid"] = kf.normal_image.valid
    np.savez_compressed(os.path.join(OUT, "golden_quality.npz"), n_keyframes=len(kfs), n_spawn=cfg.n_spawn,
                        build_seed=17, refine_seed=23, iters=iters, n_built=n_built, n_final=len(lmap.model),
                        losses=np.array(losses), rmse_before=np.array(before), rmse_after=np.array(after),
                        ref_build_s=t_build, ref_refine_s_per_iter=t_refine / iters, **out)
    print("quality: splats", n_built, "rmse before", before, "after", after, "loss", losses[0], losses[-1],
          "refine s/iter", t_refine / iters)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "quality":
    make_quality_case()
