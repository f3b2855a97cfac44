"""CPU oracle (TEST INFRASTRUCTURE ONLY) for keyframe preparation: a numpy
restatement of the reference's image functions, pinned to the live reference's
outputs in tests/golden/golden_keyframe.npz (tests/test_keyframe_oracle.py).

  build_range_image     pkg/src/splatscan/geometry.py:252-268
  smooth_range_image    pkg/src/splatscan/geometry.py:271-287 (size 3; the
                        median of each 3x3 window is computed by sorting the
                        nine shifted copies instead of scipy.ndimage)
  range_image_normals   pkg/src/splatscan/geometry.py:290-338
  estimate_camera       pkg/src/splatscan/geometry.py:198-215

Only tests/ may import this module; the product path is libsplatb200.so.
"""
from __future__ import annotations

import numpy as np


def spherical_coords(p):  # geometry.py:52-57
    az = np.arctan2(p[..., 1], p[..., 0])
    el = np.arctan2(p[..., 2], np.hypot(p[..., 0], p[..., 1]))
    return az, el


def camera_constants(cam):
    """fx, fy, cx, cy, grid offsets (geometry.py:95-109, 160-174)."""
    W, H, az_min, az_max, el_min, el_max = cam
    fov_h, fov_v = az_max - az_min, el_max - el_min
    fx, fy = -(W - 1) / fov_h, -(H - 1) / fov_v
    cx = 0.5 * W * (1.0 + (az_max + az_min) / fov_h)
    cy = 0.5 * H * (1.0 + (el_max + el_min) / fov_v)
    first_u, first_v = fx * az_max + cx, fy * el_max + cy
    off_u = np.mod(first_u + 0.5, 1.0) - 0.5
    off_v = np.mod(first_v + 0.5, 1.0) - 0.5
    return fx, fy, cx, cy, off_u, off_v


def full_circle(cam):  # geometry.py:117-121
    W, fov = cam[0], cam[3] - cam[2]
    pitch = fov / (W - 1)
    return fov + pitch >= 2.0 * np.pi - 0.5 * pitch


def pixel_directions(cam):  # geometry.py:176-185, 60-65
    W, H = int(cam[0]), int(cam[1])
    fx, fy, cx, cy, ou, ov = camera_constants(cam)
    v, u = np.mgrid[0:H, 0:W].astype(float)
    az = ((u + ou) - cx) / fx
    el = ((v + ov) - cy) / fy
    ce = np.cos(el)
    return np.stack([ce * np.cos(az), ce * np.sin(az), np.sin(el)], axis=-1)


def estimate_camera(points, W, H):
    p = np.asarray(points, float).reshape(-1, 3)
    p = p[np.linalg.norm(p, axis=1) > 1e-9]
    az, el = spherical_coords(p)
    return (W, H, float(az.min()), float(az.max()), float(el.min()), float(el.max()))


def build_range_image(cam, points):
    W, H = int(cam[0]), int(cam[1])
    fx, fy, cx, cy, _, _ = camera_constants(cam)
    p = np.asarray(points, float).reshape(-1, 3)
    r = np.linalg.norm(p, axis=1)
    keep = r > 1e-9
    p, r = p[keep], r[keep]
    az, el = spherical_coords(p)
    cols = np.floor(fx * az + cx + 0.5).astype(int)
    rows = np.floor(fy * el + cy + 0.5).astype(int)
    ok = (cols >= 0) & (cols < W) & (rows >= 0) & (rows < H)
    img = np.full((H, W), np.inf)
    np.minimum.at(img, (rows[ok], cols[ok]), r[ok])
    valid = np.isfinite(img)
    img[~valid] = 0.0
    return img, valid


def smooth_range_image(rng, valid, wrap):
    filled = np.where(valid, rng, np.inf)
    H, W = filled.shape
    rows = np.clip(np.arange(H)[:, None] + np.array([-1, 0, 1])[None, :], 0, H - 1)  # ndimage mode="nearest"
    if wrap:
        cols = (np.arange(W)[:, None] + np.array([-1, 0, 1])[None, :]) % W
    else:
        cols = np.clip(np.arange(W)[:, None] + np.array([-1, 0, 1])[None, :], 0, W - 1)
    win = np.stack([filled[rows[:, a]][:, cols[:, b]] for a in range(3) for b in range(3)], axis=-1)
    sm = np.sort(win, axis=-1)[..., 4]
    return np.where(valid & np.isfinite(sm), sm, rng)


def range_image_normals(cam, rng, valid):
    dirs = pixel_directions(cam)
    pts = rng[..., None] * dirs
    if full_circle(cam):
        left, right = np.roll(pts, 1, axis=1), np.roll(pts, -1, axis=1)
        lv, rv = np.roll(valid, 1, axis=1), np.roll(valid, -1, axis=1)
    else:
        left, right = np.zeros_like(pts), np.zeros_like(pts)
        left[:, 1:], right[:, :-1] = pts[:, :-1], pts[:, 1:]
        lv, rv = np.zeros_like(valid), np.zeros_like(valid)
        lv[:, 1:], rv[:, :-1] = valid[:, :-1], valid[:, 1:]
    up, down = np.zeros_like(pts), np.zeros_like(pts)
    up[1:], down[:-1] = pts[:-1], pts[1:]
    uv, dv = np.zeros_like(valid), np.zeros_like(valid)
    uv[1:], dv[:-1] = valid[:-1], valid[1:]
    ok = valid & lv & rv & uv & dv
    n = np.cross(right - left, down - up)
    norm = np.linalg.norm(n, axis=-1)
    ok &= norm > 1e-12
    n = np.divide(n, np.maximum(norm, 1e-12)[..., None], where=ok[..., None])
    flip = np.sum(n * dirs, axis=-1) > 0
    n[flip] = -n[flip]
    n[~ok] = 0.0
    return n, ok
