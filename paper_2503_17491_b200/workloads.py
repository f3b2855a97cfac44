"""Seeded synthetic workloads (BASELINE.json configs 0-4).

The paper's datasets are not available; these generators stand in for them
with the shapes, sizes and value distributions BASELINE.json names.  Inputs
are drawn in numpy with ``default_rng(seed)`` and rounded to float32; the CPU
oracle receives the same float32 values promoted to float64.

Pinned choices (BASELINE leaves them open; recorded in DESIGN.md):
  * "uniform in a spherical shell" = uniform RADIUS in [2, 50] m.
  * rotations: unit quaternion q ~ N(0, I4) normalised, (w, x, y, z); the raw
    tangents stored are the first two columns of R(q).
  * scene: ground z = -1.7 m (60 m half extent); four walls at x, y = +-30 m,
    z in [-1.7, 6.3]; 20 boxes, centre xy ~ U(-25, 25), half sizes ~ U(0.5, 2.5),
    resting on the ground; all drawn with default_rng(0).
"""
from __future__ import annotations

import numpy as np

from .geometry import SE3Pose, SphericalCamera, so3_exp


def synth_camera(width: int, height: int, el_deg: float = 22.5) -> SphericalCamera:
    """Camera on the raycast_scan grid: az in [-pi, pi - 2pi/W] (synth.py:277-281)."""
    return SphericalCamera(width, height, -np.pi, np.pi - 2.0 * np.pi / width, -np.deg2rad(el_deg),
                           np.deg2rad(el_deg))


def quat_tangents(q: np.ndarray):
    q = q / np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    ta = np.stack([1 - 2 * (y * y + z * z), 2 * (x * y + w * z), 2 * (x * z - w * y)], axis=1)
    tb = np.stack([2 * (x * y - w * z), 1 - 2 * (x * x + z * z), 2 * (y * z + w * x)], axis=1)
    return ta, tb


def random_splats(n: int, seed: int, rmin: float = 2.0, rmax: float = 50.0, zclip=(-2.0, 6.0),
                  mean_log_scale: float = float(np.log(0.05)), sigma_log_scale: float = 0.5,
                  draw: str = "uniform-radius") -> dict:
    """Config 0/1 splats in the fixed draw order of SURVEY 8(d); float32 arrays."""
    rng = np.random.default_rng(seed)
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    if draw == "uniform-radius":
        r = rng.uniform(rmin, rmax, n)
    else:
        r = np.cbrt(rng.uniform(rmin ** 3, rmax ** 3, n))
    c = d * r[:, None]
    c[:, 2] = np.clip(c[:, 2], *zclip)
    ls = rng.normal(mean_log_scale, sigma_log_scale, (n, 2))
    ta, tb = quat_tangents(rng.normal(size=(n, 4)))
    lo = rng.normal(0.0, 1.0, n)
    f = lambda a: np.ascontiguousarray(a, dtype=np.float32)  # noqa: E731
    return {"centers": f(c), "raw_t_alpha": f(ta), "raw_t_beta": f(tb), "log_scales": f(ls), "logit_opacity": f(lo)}


# --- procedural scene and ray casting -------------------------------------------------


class Scene:
    """Axis-aligned rectangles and boxes (ground, four walls, boxes)."""

    def __init__(self, seed: int = 0, n_boxes: int = 20):
        rng = np.random.default_rng(seed)
        # rectangles: (axis of the normal, offset, centre of the other two coords, half extents)
        self.rects = [(2, -1.7, (0.0, 0.0), (60.0, 60.0))]
        for ax, off in ((0, 30.0), (0, -30.0), (1, 30.0), (1, -30.0)):
            # in-plane coords: the other horizontal axis (half 30) and z (centre 2.3, half 4)
            self.rects.append((ax, off, (0.0, 2.3), (30.0, 4.0)))
        xy = rng.uniform(-25.0, 25.0, (n_boxes, 2))
        half = rng.uniform(0.5, 2.5, (n_boxes, 3))
        self.box_lo = np.concatenate([xy - half[:, :2], (-1.7) * np.ones((n_boxes, 1))], axis=1)
        self.box_hi = np.concatenate([xy + half[:, :2], (-1.7 + 2 * half[:, 2:3])], axis=1)

    def raycast(self, origin: np.ndarray, dirs: np.ndarray):
        """Nearest hit distance (inf if none) and world normal per ray."""
        o = np.asarray(origin, dtype=float).reshape(1, 3)
        d = np.asarray(dirs, dtype=float).reshape(-1, 3)
        n = d.shape[0]
        best = np.full(n, np.inf)
        nrm = np.zeros((n, 3))
        with np.errstate(divide="ignore", invalid="ignore"):
            for ax, off, cen, half in self.rects:
                others = [a for a in range(3) if a != ax]
                t = (off - o[0, ax]) / d[:, ax]
                hit = o[0, None, :] + t[:, None] * d
                ok = (t > 1e-9) & (np.abs(hit[:, others[0]] - cen[0]) <= half[0]) & \
                     (np.abs(hit[:, others[1]] - cen[1]) <= half[1])
                closer = ok & (t < best)
                best = np.where(closer, t, best)
                nn = np.zeros(3)
                nn[ax] = 1.0
                nrm[closer] = nn
            inv = 1.0 / d
            for lo, hi in zip(self.box_lo, self.box_hi):
                t1 = (lo[None, :] - o) * inv
                t2 = (hi[None, :] - o) * inv
                tmin = np.minimum(t1, t2)
                tmax = np.maximum(t1, t2)
                tn = np.max(tmin, axis=1)
                tf = np.min(tmax, axis=1)
                ok = (tn <= tf) & (tf > 1e-9)
                t = np.where(tn > 1e-9, tn, tf)
                closer = ok & (t < best)
                ax = np.argmax(tmin, axis=1)
                best = np.where(closer, t, best)
                nn = np.zeros((n, 3))
                nn[np.arange(n), ax] = 1.0
                nrm[closer] = nn[closer]
        return best, nrm


def target_images(scene: Scene, cam: SphericalCamera, pose: SE3Pose | None = None, max_range: float = 100.0):
    """Ray-cast range image of ``scene`` on ``cam``'s sample rays plus smoothed-range normals.

    Normals follow make_keyframe (mapping.py:110-113): 3x3 median of the valid
    ranges (seam wrap), central differences with four valid neighbours,
    oriented toward the sensor (geometry.py:271-338)."""
    from scipy import ndimage

    pose = pose or SE3Pose.identity()
    H, W = cam.height, cam.width
    dirs = cam.pixel_directions.reshape(-1, 3)
    t, _ = scene.raycast(pose.translation, dirs @ pose.rotation.T)
    valid = np.isfinite(t) & (t <= max_range)
    rng = np.where(valid, t, 0.0).reshape(H, W)
    valid = valid.reshape(H, W)
    filled = np.pad(np.where(valid, rng, np.inf), ((0, 0), (1, 1)), mode="wrap")
    sm = ndimage.median_filter(filled, size=3, mode="nearest")[:, 1:-1]
    sm = np.where(valid & np.isfinite(sm), sm, rng)
    pts = sm[..., None] * cam.pixel_directions
    wrap = cam.full_circle
    left, right = np.roll(pts, 1, axis=1), np.roll(pts, -1, axis=1)
    lv, rv = np.roll(valid, 1, axis=1), np.roll(valid, -1, axis=1)
    if not wrap:
        lv[:, 0] = False
        rv[:, -1] = False
    up = np.zeros_like(pts); up[1:] = pts[:-1]
    dn = np.zeros_like(pts); dn[:-1] = pts[1:]
    uv = np.zeros_like(valid); uv[1:] = valid[:-1]
    dv = np.zeros_like(valid); dv[:-1] = valid[1:]
    ok = valid & lv & rv & uv & dv
    nrm = np.cross(right - left, dn - up)
    nn = np.linalg.norm(nrm, axis=-1)
    ok &= nn > 1e-12
    nrm = nrm / np.maximum(nn, 1e-12)[..., None]
    flip = np.sum(nrm * cam.pixel_directions, axis=-1) > 0
    nrm[flip] = -nrm[flip]
    nrm[~ok] = 0.0
    return {"range": rng.astype(np.float32), "valid": valid, "normal": nrm.astype(np.float32), "nvalid": ok}


def config(index: int) -> dict:
    """Camera, splats and loss target of BASELINE.json configs 0 and 1."""
    if index == 0:
        cam, n, seed = synth_camera(1024, 64), 50_000, 0
    elif index == 1:
        cam, n, seed = synth_camera(2048, 128), 500_000, 1
    else:
        raise ValueError("configs 0 and 1 are single renders; see bench.py for 2-4")
    return {"camera": cam, "splats": random_splats(n, seed), "pose": SE3Pose.identity(), "seed": seed}


def random_pose(rng, rot_deg: float, trans: float) -> SE3Pose:
    return SE3Pose(so3_exp(np.deg2rad(rot_deg) * rng.normal(size=3)), rng.normal(size=3) * trans)


# --- configs 2 and 3 ----------------------------------------------------------------

def _complete_frames(n: np.ndarray):
    """Orthonormal tangents with t_alpha x t_beta = n (mapping.py:242-251 construction)."""
    ref = np.tile([0.0, 0.0, 1.0], (n.shape[0], 1))
    ref[np.abs(n[:, 2]) > 0.9] = [1.0, 0.0, 0.0]
    ta = np.cross(n, ref)
    ta /= np.linalg.norm(ta, axis=1, keepdims=True)
    return ta, np.cross(n, ta)


def keyframe_poses(n: int = 10, seed: int = 0):
    """Straight 1 m/frame trajectory with yaw noise N(0, 2 deg) (BASELINE config 2)."""
    rng = np.random.default_rng(seed)
    return [SE3Pose(so3_exp([0.0, 0.0, np.deg2rad(2.0) * rng.normal()]), np.array([float(i), 0.0, 0.0]))
            for i in range(n)]


def config2_map(n_keyframes: int = 10, per_keyframe: int = 20_000, seed: int = 0, width: int = 1024,
                height: int = 64):
    """Local map of BASELINE config 2: keyframes of the procedural scene and surfels
    back-projected from them (spawn_splats construction, mapping.py:254-303: keyframe
    normal or facing the sensor, pixel-footprint scales, opacity 0.5), 20k per keyframe."""
    rng = np.random.default_rng(seed)
    scene = Scene(0)
    cam = synth_camera(width, height)
    kfs, cents, tas, tbs, ls = [], [], [], [], []
    for pose in keyframe_poses(n_keyframes, seed):
        tg = target_images(scene, cam, pose)
        kfs.append((cam, pose, tg))
        idx = np.flatnonzero(tg["valid"].ravel())
        idx = rng.choice(idx, size=min(per_keyframe, idx.size), replace=False)
        rows, cols = np.unravel_index(idx, tg["valid"].shape)
        d = tg["range"][rows, cols].astype(np.float64)
        dirs = cam.pixel_directions[rows, cols]
        pts = d[:, None] * dirs
        n_s = np.where(tg["nvalid"][rows, cols][:, None], tg["normal"][rows, cols], -dirs)
        n_s /= np.linalg.norm(n_s, axis=1, keepdims=True)
        ta, tb = _complete_frames(n_s @ pose.rotation.T)
        cents.append(pose.apply(pts))
        tas.append(ta)
        tbs.append(tb)
        pa, pe = 1.0 / abs(cam.fx), 1.0 / abs(cam.fy)
        ls.append(np.log(np.maximum(np.stack([d * pa, d * pe], axis=1), 1e-4)))
    f = lambda a: np.ascontiguousarray(np.concatenate(a), dtype=np.float32)  # noqa: E731
    n = sum(c.shape[0] for c in cents)
    params = {"centers": f(cents), "raw_t_alpha": f(tas), "raw_t_beta": f(tbs), "log_scales": f(ls),
              "logit_opacity": np.zeros(n, dtype=np.float32)}
    ranges = np.concatenate([k[2]["range"][k[2]["valid"]] for k in kfs[:1]])
    return params, kfs, float(np.median(ranges))


def surface_samples(scene: Scene, n: int, rng, inside: float = 30.0):
    """Area-weighted uniform samples on the scene's rectangles (clipped to the walled
    area |x|, |y| <= inside, the only part a sensor inside can see) and box faces."""
    faces = []  # (origin, e_u, e_v, half_u, half_v, normal)
    for ax, off, cen, half in scene.rects:
        half = (min(half[0], inside), min(half[1], inside))
        others = [a for a in range(3) if a != ax]
        o = np.zeros(3); o[ax] = off; o[others[0]] = cen[0]; o[others[1]] = cen[1]
        eu = np.zeros(3); eu[others[0]] = 1.0
        ev = np.zeros(3); ev[others[1]] = 1.0
        nn = np.zeros(3); nn[ax] = 1.0
        faces.append((o, eu, ev, half[0], half[1], nn))
    for lo, hi in zip(scene.box_lo, scene.box_hi):
        c, h = 0.5 * (lo + hi), 0.5 * (hi - lo)
        for ax in range(3):
            others = [a for a in range(3) if a != ax]
            for sgn in (-1.0, 1.0):
                o = c.copy(); o[ax] += sgn * h[ax]
                eu = np.zeros(3); eu[others[0]] = 1.0
                ev = np.zeros(3); ev[others[1]] = 1.0
                nn = np.zeros(3); nn[ax] = sgn
                faces.append((o, eu, ev, h[others[0]], h[others[1]], nn))
    area = np.array([4 * f[3] * f[4] for f in faces])
    cnt = rng.multinomial(n, area / area.sum())
    pts, nrm = [], []
    for f, k in zip(faces, cnt):
        if k == 0:
            continue
        u = rng.uniform(-1, 1, k)[:, None] * f[3]
        v = rng.uniform(-1, 1, k)[:, None] * f[4]
        pts.append(f[0] + u * f[1] + v * f[2])
        nrm.append(np.tile(f[5], (k, 1)))
    return np.concatenate(pts), np.concatenate(nrm)


def config3_problem(n_surfels: int = 300_000, seed: int = 0, width: int = 1024, height: int = 64):
    """BASELINE config 3: a map of surfels on the visible surfaces of the procedural scene
    (scale 0.08 m, opacity 0.95; conftest.surface_model construction), a scan ray-cast at
    the true pose, and an initial pose perturbed by N(0, 0.2 m) / N(0, 2 deg) per axis."""
    rng = np.random.default_rng(seed)
    scene = Scene(0)
    pts, nrm = surface_samples(scene, 3 * n_surfels, rng)
    seen = np.zeros(pts.shape[0], dtype=bool)
    for vp in (np.zeros(3), np.array([2.0, 0, 0]), np.array([-2.0, 0, 0])):
        rest = np.flatnonzero(~seen)
        vec = pts[rest] - vp
        dist = np.linalg.norm(vec, axis=1)
        t, _ = scene.raycast(vp, vec / np.maximum(dist, 1e-9)[:, None])
        seen[rest[t >= dist - 1e-4]] = True
    idx = np.flatnonzero(seen)
    idx = rng.choice(idx, size=min(n_surfels, idx.size), replace=False)
    pts, nrm = pts[idx], nrm[idx]
    ta, tb = _complete_frames(nrm)
    m = pts.shape[0]
    f = lambda a: np.ascontiguousarray(a, dtype=np.float32)  # noqa: E731
    params = {"centers": f(pts), "raw_t_alpha": f(ta), "raw_t_beta": f(tb),
              "log_scales": np.full((m, 2), np.log(0.08), np.float32),
              "logit_opacity": np.full(m, np.log(0.95 / 0.05), np.float32)}
    truth = SE3Pose.identity()
    cam = synth_camera(width, height)
    tg = target_images(scene, cam, truth)
    scan = (tg["range"][tg["valid"]][:, None].astype(np.float64) * cam.pixel_directions[tg["valid"]])
    initial = truth.compose(SE3Pose(so3_exp(np.deg2rad(2.0) * rng.normal(size=3)), 0.2 * rng.normal(size=3)))
    return params, cam, scan, truth, initial


# --- device-built local maps (configs 2 and 4) ---------------------------------------

_KF_CACHE: dict = {}


def keyframe_targets(n: int = 10, seed: int = 0, width: int = 1024, height: int = 64):
    """[(camera, pose, target images)] along the config-2 trajectory (keyframe_poses) over
    the procedural scene; cached per process (the numpy ray cast is the slow part)."""
    key = (n, seed, width, height)
    if key not in _KF_CACHE:
        scene = Scene(0)
        cam = synth_camera(width, height)
        _KF_CACHE[key] = [(cam, pose, target_images(scene, cam, pose)) for pose in keyframe_poses(n, seed)]
    return _KF_CACHE[key]


def device_keyframes(targets) -> list:
    """DeviceKeyframe per (camera, pose, targets) entry, indexed in order."""
    from .mapping import DeviceKeyframe
    return [DeviceKeyframe(cam, pose, tg["range"], tg["valid"], tg["normal"], tg["nvalid"], i)
            for i, (cam, pose, tg) in enumerate(targets)]


def build_local_map(dkfs: list, n_spawn: int, seed: int, raster=None):
    """A local map grown the reference's way: LocalMap.start on the first keyframe, then
    add_keyframe with each further one (mapping.py:392-438: render, densify mask, prune,
    weighted spawn of up to n_spawn surfels), on the device.  SURVEY 8(d) config 2:
    10 keyframes x 20k at 64x1024 gives 200,000 surfels."""
    from .mapping import DeviceMap, MappingConfig
    cfg = MappingConfig(n_spawn=n_spawn)
    rng = np.random.default_rng(seed)
    dm = DeviceMap.start(dkfs[0], cfg, rng, raster)
    for kf in dkfs[1:]:
        dm.add_keyframe(kf, cfg, rng, raster)
    return dm


def merge_maps(maps: list, keyframes: list):
    """One DeviceMap holding the union of the given maps' surfels (config 4b's shared map)."""
    import torch

    from .engine import PARAM_NAMES
    from .mapping import DeviceMap
    params = {k: torch.cat([m.params[k] for m in maps]) for k in PARAM_NAMES}
    return DeviceMap(params, keyframes, maps[0].scene_scale)


def config3_frames(n_frames: int = 8, seed: int = 0, width: int = 1024, height: int = 64, step: float = 0.25):
    """Frames for batched registration against the config-3 map: true poses along x (``step``
    m apart), a scan ray-cast at each, initial poses perturbed by N(0, 0.2 m) / N(0, 2 deg) per
    axis.  Returns (map params, camera, scans, truths, initials)."""
    params, cam, _, _, _ = config3_problem(seed=seed, width=width, height=height)
    rng = np.random.default_rng(1000 + seed)
    scene = Scene(0)
    scans, truths, initials = [], [], []
    for f in range(n_frames):
        truth = SE3Pose(so3_exp([0.0, 0.0, np.deg2rad(1.0) * rng.normal()]), np.array([step * f, 0.0, 0.0]))
        tg = target_images(scene, cam, truth)
        scans.append(tg["range"][tg["valid"]][:, None].astype(np.float64) * cam.pixel_directions[tg["valid"]])
        truths.append(truth)
        initials.append(truth.compose(SE3Pose(so3_exp(np.deg2rad(2.0) * rng.normal(size=3)), 0.2 * rng.normal(size=3))))
    return params, cam, scans, truths, initials


def map_depth_rmse(dm, dkfs, raster=None) -> tuple:
    """Depth RMSE of a device map over keyframes: rendered range D vs the keyframe range on
    valid pixels, and D / O vs it where O > 0.5 (sample_model's depth); plus the fraction
    of valid pixels that are confident."""
    from . import engine
    from .geometry import pose_rt
    from .mapping import RasterConfig
    se = cnt = se2 = cnt2 = 0.0
    for kf in dkfs:
        D, _, O = engine.forward(kf.camera, pose_rt(kf.pose), dm.params, raster or RasterConfig(), dm.rec)
        v = kf.valid.bool()
        se += float(((D.double() - kf.range64)[v] ** 2).sum())
        cnt += int(v.sum())
        c = v & (O > 0.5)
        se2 += float(((D.double() / O.double().clamp_min(1e-12) - kf.range64)[c] ** 2).sum())
        cnt2 += int(c.sum())
    return float(np.sqrt(se / max(cnt, 1))), float(np.sqrt(se2 / max(cnt2, 1))), cnt2 / max(cnt, 1)


def quality_run(fx) -> dict:
    """The reduced config-2 run of tests/golden/golden_quality.npz (made by the reference:
    LocalMap.start + add_keyframe, then refine) repeated on the device with the same
    keyframe images, configuration and seeds: the depth RMSE the reference reached beside
    ours.  ``fx`` is the loaded npz."""
    from .geometry import SE3Pose, SphericalCamera
    from .mapping import DeviceKeyframe, DeviceMap, MappingConfig
    dkfs = []
    for i in range(int(fx["n_keyframes"])):
        w, h, a0, a1, e0, e1 = fx[f"kf{i}_cam"]
        cam = SphericalCamera(int(w), int(h), float(a0), float(a1), float(e0), float(e1))
        dkfs.append(DeviceKeyframe(cam, SE3Pose(fx[f"kf{i}_R"], fx[f"kf{i}_t"]), fx[f"kf{i}_range"],
                                   fx[f"kf{i}_valid"], fx[f"kf{i}_normal"], fx[f"kf{i}_nvalid"], i))
    cfg = MappingConfig(n_spawn=int(fx["n_spawn"]))
    rng = np.random.default_rng(int(fx["build_seed"]))
    dm = DeviceMap.start(dkfs[0], cfg, rng)
    for kf in dkfs[1:]:
        dm.add_keyframe(kf, cfg, rng)
    n_built = dm.n
    before = map_depth_rmse(dm, dkfs)
    losses = dm.refine(cfg, int(fx["iters"]), np.random.default_rng(int(fx["refine_seed"])))
    after = map_depth_rmse(dm, dkfs)
    return {"splats": n_built, "rmse_before": before, "rmse_after": after,
            "loss_first": float(losses[0]), "loss_last": float(losses[-1])}
