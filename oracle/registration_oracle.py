"""CPU restatement (numpy, float64) of the reference's photometric registration.

TEST INFRASTRUCTURE ONLY (see oracle.c): the parity checker of the device
registration path; never imported by the product package.

Restates pkg/src/splatscan/:
  registration.py:170-187  _jump_mask          registration.py:190-213  sample_model
  geometry.py:252-268      build_range_image   registration.py:277-313  _bilinear_range
  registration.py:316-362  _photo_system       registration.py:219-228  Huber weight / value
  registration.py:387-524  register (photometric phase)
Pinned against tests/golden/golden_register.npz (live reference outputs).
"""
from __future__ import annotations

import numpy as np

from . import oracle as O


def intrinsics(cam):
    fx, fy, cx, cy, ou, ov = O.intrinsics(cam)
    return fx, fy, cx, cy, ou, ov


def full_circle(cam) -> bool:
    fov = cam[3] - cam[2]
    pitch = fov / (cam[0] - 1)
    return fov + pitch >= 2.0 * np.pi - 0.5 * pitch


def _angles(q):
    az = np.arctan2(q[..., 1], q[..., 0])
    el = np.arctan2(q[..., 2], np.hypot(q[..., 0], q[..., 1]))
    return az, el


def jump_mask(depth, valid, gate, wrap):
    """Pixels whose depth differs by more than gate from a valid 4-neighbour."""
    H, W = depth.shape
    bad = np.zeros_like(valid)
    # vertical neighbours never wrap
    up = np.zeros_like(valid); up[1:] = valid[:-1]
    dn = np.zeros_like(valid); dn[:-1] = valid[1:]
    dup = np.zeros_like(depth); dup[1:] = depth[:-1]
    ddn = np.zeros_like(depth); ddn[:-1] = depth[1:]
    bad |= valid & up & (np.abs(depth - dup) > gate)
    bad |= valid & dn & (np.abs(depth - ddn) > gate)
    lv = np.roll(valid, 1, axis=1); rv = np.roll(valid, -1, axis=1)
    if not wrap:
        lv[:, 0] = False
        rv[:, -1] = False
    bad |= valid & lv & (np.abs(depth - np.roll(depth, 1, axis=1)) > gate)
    bad |= valid & rv & (np.abs(depth - np.roll(depth, -1, axis=1)) > gate)
    return bad


def sample_model(params, geo_cam, R, t, vis=0.5, gate=0.5):
    """World points of confident, jump-free rendered pixels (row-major order)."""
    r = O.render(geo_cam, R, t, params)
    D, Op = r["range"], r["opacity"]
    m = (Op > vis) & (D > 0)
    depth = np.where(m, D / np.maximum(Op, 1e-12), 0.0)
    m &= ~jump_mask(depth, m, gate, full_circle(geo_cam))
    fx, fy, cx, cy, ou, ov = intrinsics(geo_cam)
    rows, cols = np.nonzero(m)
    az = (cols + ou - cx) / fx
    el = (rows + ov - cy) / fy
    ce = np.cos(el)
    pc = depth[rows, cols][:, None] * np.stack([ce * np.cos(az), ce * np.sin(az), np.sin(el)], axis=1)
    return pc @ np.asarray(R).T + np.asarray(t)


def build_range_image(cam, pts):
    W, H = int(cam[0]), int(cam[1])
    fx, fy, cx, cy, _, _ = intrinsics(cam)
    p = np.asarray(pts, float).reshape(-1, 3)
    rr = np.linalg.norm(p, axis=1)
    p, rr = p[rr > 1e-9], rr[rr > 1e-9]
    az, el = _angles(p)
    cu = np.floor(fx * az + cx + 0.5).astype(int)
    cv = np.floor(fy * el + cy + 0.5).astype(int)
    ok = (cu >= 0) & (cu < W) & (cv >= 0) & (cv < H)
    img = np.full((H, W), np.inf)
    np.minimum.at(img, (cv[ok], cu[ok]), rr[ok])
    valid = np.isfinite(img)
    img[~valid] = 0.0
    return img, valid


def photo_system(X, rimg, valid, cam, R, t, trim_floor, trim_factor=5.0, gate=0.5):
    """(r, J) of the kept residuals at pose (R, t), or None."""
    W, H = int(cam[0]), int(cam[1])
    fx, fy, cx, cy, ou, ov = intrinsics(cam)
    q = (np.asarray(X) - t) @ R
    rho2 = q[:, 0] ** 2 + q[:, 1] ** 2
    r2 = rho2 + q[:, 2] ** 2
    az, el = _angles(q)
    u = fx * az + cx - ou
    v = fy * el + cy - ov
    i0 = np.floor(u).astype(int)
    j0 = np.floor(v).astype(int)
    ok = (i0 >= 0) & (i0 + 1 < W) & (j0 >= 0) & (j0 + 1 < H) & (rho2 > 1e-12)
    i0c, j0c = np.clip(i0, 0, W - 2), np.clip(j0, 0, H - 2)
    fu, fv = u - i0c, v - j0c
    ok &= valid[j0c, i0c] & valid[j0c, i0c + 1] & valid[j0c + 1, i0c] & valid[j0c + 1, i0c + 1]
    d00, d10 = rimg[j0c, i0c], rimg[j0c, i0c + 1]
    d01, d11 = rimg[j0c + 1, i0c], rimg[j0c + 1, i0c + 1]
    cell = np.stack([d00, d10, d01, d11])
    ok &= cell.max(axis=0) - cell.min(axis=0) <= gate
    top = d00 * (1 - fu) + d10 * fu
    bot = d01 * (1 - fu) + d11 * fu
    val = top * (1 - fv) + bot * fv
    du = (d10 - d00) * (1 - fv) + (d11 - d01) * fv
    dv = bot - top
    if not ok.any():
        return None
    res = np.sqrt(r2[ok]) - val[ok]
    keep = np.abs(res) <= max(trim_factor * np.median(np.abs(res)), trim_floor)
    if not keep.any():
        return None
    qk = q[ok][keep]
    x, y, z = qk.T
    rho2k, r2k = rho2[ok][keep], r2[ok][keep]
    rho = np.sqrt(rho2k)
    dudq = fx * np.stack([-y / rho2k, x / rho2k, np.zeros_like(x)], axis=1)
    dvdq = fy * np.stack([-x * z / (r2k * rho), -y * z / (r2k * rho), rho / r2k], axis=1)
    g = qk / np.sqrt(r2k)[:, None] - du[ok][keep][:, None] * dudq - dv[ok][keep][:, None] * dvdq
    J = np.concatenate([-g, np.cross(g, qk)], axis=1)
    return res[keep], J


def huber_w(r, d):
    a = np.abs(r)
    return np.where(a <= d, 1.0, d / np.maximum(a, 1e-12))


def huber_v(r, d):
    a = np.abs(r)
    return float(np.sum(np.where(a <= d, 0.5 * r * r, d * (a - 0.5 * d))))


def _exp(delta):
    from scipy.spatial.transform import Rotation
    rho, phi = delta[:3], delta[3:]
    a = np.linalg.norm(phi)
    K = np.array([[0, -phi[2], phi[1]], [phi[2], 0, -phi[0]], [-phi[1], phi[0], 0]])
    if a < 1e-8:
        Rm = np.eye(3) + K + 0.5 * K @ K
        Jl = np.eye(3) + 0.5 * K + K @ K / 6.0
    else:
        Rm = np.eye(3) + np.sin(a) / a * K + (1 - np.cos(a)) / a ** 2 * K @ K
        Jl = np.eye(3) + (1 - np.cos(a)) / a ** 2 * K + (a - np.sin(a)) / a ** 3 * K @ K
    return Rm, Jl @ rho


def register_photometric(X, rimg, valid, cam, R0, t0, max_iters=30, tol=1e-6, huber=0.2, trim_floor=0.02,
                         gate_assoc=1.0, damping_init=1e-6, damping_max=1e6, min_residuals=10):
    """The GN/LM loop of register() for mode='photometric'.  Returns (R, t, iters, converged, rms, m, deltas)."""
    R, t = np.array(R0, float), np.array(t0, float)
    lam = damping_init
    it = 0
    converged = False
    last = (np.zeros(0), 0)
    deltas = []
    while it < max_iters:
        it += 1
        fp = max(trim_floor, gate_assoc * 0.5 ** it)
        ph = photo_system(X, rimg, valid, cam, R, t, fp)
        if ph is None or ph[0].shape[0] < min_residuals:
            raise RuntimeError("too few residuals")
        r, J = ph
        w = huber_w(r, huber)
        s = 1.0 / r.shape[0]
        H = s * (J.T * w) @ J
        b = s * (J.T @ (w * r))
        last = (r, r.shape[0])
        obj0 = s * huber_v(r, huber)
        accepted = False
        while lam <= damping_max:
            try:
                d = np.linalg.solve(H + lam * np.eye(6), -b)
            except np.linalg.LinAlgError:
                lam = max(lam, 1e-8) * 10
                continue
            dR, dt = _exp(d)
            Rt, tt = R @ dR, R @ dt + t
            p2 = photo_system(X, rimg, valid, cam, Rt, tt, fp)
            if p2 is not None and s * huber_v(p2[0], huber) <= obj0 + 1e-12:
                R, t = Rt, tt
                lam = max(lam * 0.25, damping_init)
                accepted = True
                deltas.append(d)
                break
            lam = max(lam, 1e-8) * 10
        if not accepted:
            break
        if np.linalg.norm(d) < tol:
            converged = True
            break
    U, _, Vt = np.linalg.svd(R)
    Rn = U @ Vt
    if np.linalg.det(Rn) < 0:
        U[:, -1] *= -1
        Rn = U @ Vt
    r, m = last
    rms = float(np.sqrt(np.mean(r * r))) if m else 0.0
    return Rn, t, it, converged, rms, m, deltas
