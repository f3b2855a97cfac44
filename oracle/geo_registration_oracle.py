"""CPU restatement (numpy/scipy, float64) of the geometric half of the reference's
registration -- TEST INFRASTRUCTURE ONLY (the checker of the device path).

Restates pkg/src/splatscan/registration.py:
  :98-164   build_leaf_tree / _push_leaf  recursive PCA splits into planar leaves
  :231-274  _geo_system                   k-nearest-leaf point-to-plane residuals,
                                           median trim, Jacobian
  :219-228  Huber weights / value         :379-384 _objective (positional pairing)
  :387-524  register: geometric, joint and sequential phase schedules
Third-party arithmetic: numpy.linalg.eigh (LAPACK syevd), scipy.spatial.cKDTree
(k-NN with distance_upper_bound).  Pinned against tests/golden/golden_register_geo.npz.
"""
from __future__ import annotations

import numpy as np
from scipy.spatial import cKDTree

from . import registration_oracle as RO


def build_leaf_tree(pts, viewpoint, leaf_size=64, tau=0.02):
    """(centroids, normals, sizes, usable, point_leaf): leaves in the reference's stack order."""
    pts = np.asarray(pts, float)
    point_leaf = np.zeros(pts.shape[0], dtype=int)
    cents, norms, sizes, usable = [], [], [], []

    def leaf(idx, c, normal):
        point_leaf[idx] = len(cents)
        cents.append(c)
        if normal is not None and normal @ (viewpoint - c) < 0:
            normal = -normal
        norms.append(np.zeros(3) if normal is None else normal)
        sizes.append(idx.size)
        usable.append(normal is not None)

    work = [np.arange(pts.shape[0])]
    while work:
        idx = work.pop()
        sub = pts[idx]
        c = sub.mean(axis=0)
        if idx.size < 3:
            leaf(idx, c, None)
            continue
        lam, vec = np.linalg.eigh(np.cov(sub.T, bias=True))
        if lam[1] <= 1e-12 or lam[0] / lam[1] <= tau or idx.size <= leaf_size:
            leaf(idx, c, vec[:, 0] if lam[1] > 1e-12 else None)
            continue
        proj = (sub - c) @ vec[:, 2]
        lo = proj <= np.median(proj)
        if lo.all() or not lo.any():
            leaf(idx, c, vec[:, 0])
            continue
        work.append(idx[lo])
        work.append(idx[~lo])
    return (np.array(cents).reshape(-1, 3), np.array(norms).reshape(-1, 3), np.array(sizes),
            np.array(usable, bool), point_leaf)


class Tree:
    def __init__(self, pts, viewpoint, leaf_size=64, tau=0.02):
        self.c, self.n, self.sizes, self.usable, self.point_leaf = build_leaf_tree(pts, viewpoint, leaf_size, tau)
        self.ids = np.flatnonzero(self.usable)
        self.kd = cKDTree(self.c[self.usable]) if self.usable.any() else None


def geo_system(tree: Tree, scan, R, t, trim_floor, k=3, gate=1.0, trim_factor=5.0):
    """(r, J) of the kept scan points, or None."""
    if tree.kd is None:
        return None
    p = scan @ R.T + t
    kk = min(k, tree.kd.n)
    d, li = tree.kd.query(p, k=kk, distance_upper_bound=gate)
    if kk == 1:
        d, li = d[:, None], li[:, None]
    valid = np.isfinite(d)
    ok = valid[:, 0]
    if not ok.any():
        return None
    lg = tree.ids[np.where(valid, li, 0)]
    pd = np.abs(np.einsum("pkj,pkj->pk", tree.n[lg], p[:, None, :] - tree.c[lg]))
    pd[~valid] = np.inf
    pick = lg[np.arange(p.shape[0]), pd.argmin(axis=1)][ok]
    n, c, q = tree.n[pick], tree.c[pick], scan[ok]
    r = np.sum(n * (p[ok] - c), axis=1)
    keep = np.abs(r) <= max(trim_factor * np.median(np.abs(r)), trim_floor)
    if not keep.any():
        return None
    n, q, r = n[keep], q[keep], r[keep]
    nR = n @ R
    return r, np.concatenate([nR, np.cross(q, nR)], axis=1)


def register(mode, tree: Tree, geo_scan, X, rimg, valid, cam, R0, t0, max_iters=30, tol=1e-6, huber_geo=0.1,
             huber_photo=0.2, floor_geo=0.02, floor_photo=0.02, gate=1.0, damping_init=1e-6, damping_max=1e6,
             min_residuals=10, k=3):
    """register()'s loop for every mode.  Returns (R, t, iters, converged, geo_rms, photo_rms, n_geo, n_photo)."""
    phases = [("geometric", max_iters // 2), ("joint", max_iters)] if mode == "sequential" else [(mode, max_iters)]
    R, t = np.array(R0, float), np.array(t0, float)
    it = 0
    converged = False
    last = {"geo": (np.zeros(0), 0), "photo": (np.zeros(0), 0)}
    for phase, budget in phases:
        use_geo, use_photo = phase in ("geometric", "joint"), phase in ("photometric", "joint")
        lam = damping_init
        converged = False
        while it < budget:
            it += 1
            anneal = gate * 0.5 ** it
            fg, fp = max(floor_geo, anneal), max(floor_photo, anneal)
            H, b, terms, cur = np.zeros((6, 6)), np.zeros(6), [], []
            for fam, use in (("geo", use_geo), ("photo", use_photo)):
                sysr = None
                if use:
                    sysr = geo_system(tree, geo_scan, R, t, fg, k=k, gate=gate) if fam == "geo" else \
                        RO.photo_system(X, rimg, valid, cam, R, t, fp)
                if sysr is not None:
                    r, J = sysr
                    hub = huber_geo if fam == "geo" else huber_photo
                    w = RO.huber_w(r, hub)
                    s = 1.0 / r.shape[0]
                    H += s * (J.T * w) @ J
                    b += s * (J.T @ (w * r))
                    terms.append((hub, s))
                    cur.append(r)
                    last[fam] = (r, r.shape[0])
            if sum(r.shape[0] for r in cur) < min_residuals:
                raise RuntimeError("too few residuals")
            obj0 = sum(s * RO.huber_v(r, hub) for r, (hub, s) in zip(cur, terms))
            accepted = False
            while lam <= damping_max:
                try:
                    d = np.linalg.solve(H + lam * np.eye(6), -b)
                except np.linalg.LinAlgError:
                    lam = max(lam, 1e-8) * 10
                    continue
                if not np.all(np.isfinite(d)):
                    lam = max(lam, 1e-8) * 10
                    continue
                dR, dt = RO._exp(d)
                Rt, tt = R @ dR, R @ dt + t
                trial = []
                if use_geo:
                    g2 = geo_system(tree, geo_scan, Rt, tt, fg, k=k, gate=gate)
                    if g2 is not None:
                        trial.append(g2[0])
                if use_photo:
                    p2 = RO.photo_system(X, rimg, valid, cam, Rt, tt, fp)
                    if p2 is not None:
                        trial.append(p2[0])
                # positional pairing of residual families with the frozen terms (registration.py:379-384)
                if trial and sum(s * RO.huber_v(r, hub) for r, (hub, s) in zip(trial, terms)) <= obj0 + 1e-12:
                    R, t = Rt, tt
                    lam = max(lam * 0.25, damping_init)
                    accepted = True
                    break
                lam = max(lam, 1e-8) * 10
            if not accepted:
                break
            if np.linalg.norm(d) < tol:
                converged = True
                break
        if mode != "sequential":
            break
    U, _, Vt = np.linalg.svd(R)
    Rn = U @ Vt
    if np.linalg.det(Rn) < 0:
        U[:, -1] *= -1
        Rn = U @ Vt
    rms = lambda r: float(np.sqrt(np.mean(r * r))) if r.size else 0.0  # noqa: E731
    return Rn, t, it, converged, rms(last["geo"][0]), rms(last["photo"][0]), last["geo"][1], last["photo"][1]
