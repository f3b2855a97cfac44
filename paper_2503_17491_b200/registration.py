"""Drop-in registration (reference: pkg/src/splatscan/registration.py).

``register(model, scan, cam, initial, cfg)`` runs the reference's
Gauss-Newton / Levenberg loop (registration.py:387-524) in every mode --
photometric, geometric, joint and the default sequential schedule -- as ONE
cooperative sm_100a kernel (``ss_reg_solve``): per evaluation the geometric
point-to-plane system (k nearest leaves, closest plane, median trim;
:231-274) and / or the photometric range-warp system (:316-362), the damped
6x6 solve, the SE(3) update and the acceptance test, with no host round trip.
Around it: the model render of ``sample_model`` is the B200 rasterizer, the
PCA leaf tree (:98-164) is built level-parallel on the device
(``ss_leaf_tree_build``), the scan range image by ``ss_range_image``.  The
host only draws the reference's geometric scan subsample (same numpy RNG
call) and re-orthonormalises the final rotation (SVD).  ``PhotoProblem``
exposes single ``_photo_system`` evaluations (``ss_photo_system``) for
callers that drive their own loop.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import engine
from ._lib import SS_ERR_CAPACITY, SsRegCfg, SsRegSolveCfg, check, lib
from .errors import RegistrationError
from .geometry import SE3Pose, SphericalCamera, pose_rt
from .rasterizer import RasterConfig

__all__ = ["RegistrationConfig", "RegistrationResult", "register", "DeviceScan", "PhotoProblem"]


@dataclass
class RegistrationConfig:
    """Same fields and defaults as the reference (registration.py:41-61)."""
    mode: str = "sequential"
    huber_geo: float = 0.1
    huber_photo: float = 0.2
    assoc_gate: float = 1.0
    assoc_k: int = 3
    trim_factor: float = 5.0
    trim_floor_geo: float = 0.02
    trim_floor_photo: float = 0.02
    spread_gate: float = 0.5
    max_iters: int = 30
    tol: float = 1e-6
    visibility_opacity: float = 0.5
    leaf_size: int = 64
    flatness_tau: float = 0.02
    min_residuals: int = 10
    max_geo_points: int = 8000
    geo_supersample: int = 2
    damping_init: float = 1e-6
    damping_max: float = 1e6


@dataclass
class RegistrationResult:
    """registration.py:64-75."""
    pose: SE3Pose
    converged: bool
    iterations: int
    geo_rms: float
    photo_rms: float
    n_geo: int
    n_photo: int
    mode: str
    used_fallback: bool = False
    message: str = ""


class DeviceScan:
    """Scan range image on the device (build_range_image, geometry.py:252-268)."""

    _stage = None  # reused pinned staging buffer and the event of its last upload

    def __init__(self, cam, scan: np.ndarray):
        dev = engine.require_cuda()
        arr = np.ascontiguousarray(np.asarray(scan, dtype=np.float64).reshape(-1, 3))
        # pinned staging: the upload is stream-ordered without blocking the host (so it
        # can be prepared while a render is in flight, see register())
        st = DeviceScan._stage
        if st is None or st[0].shape[0] < arr.shape[0]:
            st = (torch.empty((max(arr.shape[0], 1), 3), dtype=torch.float64).pin_memory(), torch.cuda.Event())
            DeviceScan._stage = st
        else:
            st[1].synchronize()  # the previous upload from this buffer has finished
        host = st[0][: arr.shape[0]]
        host.numpy()[...] = arr
        pts = host.to(dev, non_blocking=True)
        st[1].record()
        self.cam = cam
        self.range = torch.empty((cam.height, cam.width), dtype=torch.float64, device=dev)
        self.valid = torch.empty((cam.height, cam.width), dtype=torch.uint8, device=dev)
        c = engine.ss_camera(cam)
        check(lib().ss_range_image(ctypes.byref(c), ctypes.c_void_p(pts.data_ptr() if pts.numel() else 0),
                                   int(pts.shape[0]), ctypes.c_void_p(self.range.data_ptr()),
                                   ctypes.c_void_p(self.valid.data_ptr()), ctypes.c_void_p(engine.stream_ptr())),
              "build_range_image")


class LeafTree:
    """registration.py:81-95 (the k-d tree over usable centroids is replaced by the
    device association; ``kdtree`` stays None).  ``dev_centroids`` / ``dev_normals``
    hold the usable leaves on the device for the association kernel; ``point_leaf``
    is copied to the host on first access."""

    kdtree = None

    def __init__(self, centroids, normals, sizes, usable, point_leaf_dev, dev_centroids, dev_normals):
        self.centroids, self.normals, self.sizes, self.usable = centroids, normals, sizes, usable
        self.point_leaf_dev = point_leaf_dev
        self.dev_centroids, self.dev_normals = dev_centroids, dev_normals
        self._point_leaf = None

    @property
    def point_leaf(self) -> np.ndarray:
        if self._point_leaf is None:
            self._point_leaf = self.point_leaf_dev.cpu().numpy().astype(int)
        return self._point_leaf


_TREE_HOST: list = []


def _tree_host_buffers(cap: int):
    """Reused host output buffers of ss_leaf_tree_build (fresh multi-MB arrays per call cost page faults)."""
    if not _TREE_HOST or _TREE_HOST[0][0].shape[0] < cap:
        _TREE_HOST[:] = [(np.zeros((cap, 3)), np.zeros((cap, 3)), np.zeros(cap, np.int32), np.zeros(cap, np.uint8))]
    return _TREE_HOST[0]


def build_leaf_tree(points, viewpoint, leaf_size: int = 64, flatness_tau: float = 0.02) -> LeafTree:
    """registration.py:98-164 on the device (level-parallel PCA median splits)."""
    dev = engine.require_cuda()
    P = points if torch.is_tensor(points) else torch.as_tensor(np.asarray(points, np.float64).reshape(-1, 3))
    P = P.to(dev, torch.float64).reshape(-1, 3).contiguous()
    n = int(P.shape[0])
    if n == 0:
        raise RegistrationError("cannot build a leaf tree from an empty cloud")
    vp = np.ascontiguousarray(np.asarray(viewpoint, np.float64).reshape(3))
    cap = n
    cent, nrm, sizes, usable = _tree_host_buffers(cap)
    pl = torch.empty(n, dtype=torch.int32, device=dev)
    nl = ctypes.c_int32(0)
    ws = torch.empty(int(lib().ss_leaf_tree_workspace_bytes(n)), dtype=torch.uint8, device=dev)
    check(lib().ss_leaf_tree_build(ctypes.c_void_p(P.data_ptr()), n, vp.ctypes.data_as(ctypes.c_void_p),
                                   int(leaf_size), float(flatness_tau), cap, cent.ctypes.data_as(ctypes.c_void_p),
                                   nrm.ctypes.data_as(ctypes.c_void_p), sizes.ctypes.data_as(ctypes.c_void_p),
                                   usable.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(pl.data_ptr()),
                                   ctypes.byref(nl), ctypes.c_void_p(ws.data_ptr()),
                                   ctypes.c_void_p(engine.stream_ptr())), "build_leaf_tree")
    k = nl.value
    use = usable[:k].astype(bool)
    return LeafTree(cent[:k].copy(), nrm[:k].copy(), sizes[:k].astype(int), use, pl,
                    torch.as_tensor(np.ascontiguousarray(cent[:k][use]), device=dev),
                    torch.as_tensor(np.ascontiguousarray(nrm[:k][use]), device=dev))


def sample_anchors(model_or_params, geo_cam, pose, cfg: RegistrationConfig, raster: RasterConfig | None = None,
                   thin: int = 1, overlap=None):
    """Device sample_model (registration.py:190-213): world anchors, thinned by ``thin``.

    Returns (X float64 [n,3] device tensor, number of confident pixels).  ``overlap``: an
    optional host callable run while the render executes (its result is returned third)."""
    raster = raster or RasterConfig()
    params = engine.as_device_params(model_or_params)
    rec = engine.Records.acquire()
    try:
        # no host wait after the render: the anchor extraction below synchronises anyway,
        # and the capacity check is read afterwards (re-run on the rare overflow)
        D, N, O = engine.forward(geo_cam, pose_rt(pose), params, raster, rec, sync=False)
        extra = overlap() if overlap is not None else None
        X, counts = _anchors(D, O, geo_cam, pose, cfg, thin)
        if rec.check(True) == SS_ERR_CAPACITY:
            D, N, O = engine.forward(geo_cam, pose_rt(pose), params, raster, rec)
            X, counts = _anchors(D, O, geo_cam, pose, cfg, thin)
        else:
            check(rec.check(True), "rasterize_forward")
    finally:
        rec.release()
    if overlap is not None:
        return X[: counts[1]], int(counts[0]), extra
    return X[: counts[1]], int(counts[0])


def _anchors(D, O, geo_cam, pose, cfg, thin):
    """ss_reg_anchors on a rendered (D, O): (X buffer, counts [confident, kept]); synchronises."""
    dev = D.device
    P = geo_cam.width * geo_cam.height
    cap = (P + thin - 1) // thin
    X = torch.empty((max(cap, 1), 3), dtype=torch.float64, device=dev)
    ws = torch.empty(int(lib().ss_anchor_workspace_bytes(geo_cam.width, geo_cam.height)), dtype=torch.uint8,
                     device=dev)
    counts = (ctypes.c_int32 * 2)()
    c = engine.ss_camera(geo_cam)
    prt = pose_rt(pose)
    check(lib().ss_reg_anchors(ctypes.byref(c), ctypes.c_void_p(D.data_ptr()), ctypes.c_void_p(O.data_ptr()),
                               prt.ctypes.data_as(ctypes.c_void_p), float(cfg.visibility_opacity),
                               float(cfg.spread_gate), int(thin), ctypes.c_void_p(X.data_ptr()), int(cap), counts,
                               ctypes.c_void_p(ws.data_ptr()), ctypes.c_void_p(engine.stream_ptr())),
          "sample_model")
    return X, counts


class PhotoProblem:
    """Repeated _photo_system evaluations (registration.py:316-362) on the device."""

    def __init__(self, X_w: torch.Tensor, scan: DeviceScan, cfg: RegistrationConfig):
        self.X = X_w.contiguous()
        self.M = int(self.X.shape[0])
        self.scan = scan
        self.cfg = SsRegCfg(float(cfg.huber_photo), float(cfg.trim_factor), float(cfg.spread_gate))
        self.ws = torch.empty(int(lib().ss_photo_workspace_bytes(max(self.M, 1))), dtype=torch.uint8,
                              device=self.X.device)
        self.cam = engine.ss_camera(scan.cam)
        self.out = np.zeros(30)
        self.calls = 0

    def evaluate(self, T, trim_floor: float, objective_only: bool = False):
        """None when no residual survives (the reference returns None), else
        (H 6x6, b 6, huber_sum, m, sum_r2) as unnormalised float64 sums."""
        if self.M == 0:
            return None
        prt = pose_rt(T)
        self.calls += 1
        check(lib().ss_photo_system(ctypes.c_void_p(self.X.data_ptr()), self.M,
                                    ctypes.c_void_p(self.scan.range.data_ptr()),
                                    ctypes.c_void_p(self.scan.valid.data_ptr()), ctypes.byref(self.cam),
                                    prt.ctypes.data_as(ctypes.c_void_p), float(trim_floor), ctypes.byref(self.cfg),
                                    int(bool(objective_only)), self.out.ctypes.data_as(ctypes.c_void_p),
                                    ctypes.c_void_p(self.ws.data_ptr()), ctypes.c_void_p(engine.stream_ptr())),
              "photo_system")
        o = self.out
        m = int(round(o[28]))
        if m == 0:
            return None
        H = np.zeros((6, 6))
        k = 0
        for a in range(6):
            for b in range(a, 6):
                H[a, b] = H[b, a] = o[k]
                k += 1
        return H, o[21:27].copy(), float(o[27]), m, float(o[29])


_MODE = {"photometric": 0, "geometric": 1, "joint": 2, "sequential": 3}


def register(model, scan, cam, initial, cfg: RegistrationConfig | None = None, raster: RasterConfig | None = None,
             rng=None) -> RegistrationResult:
    """Align a sensor-frame scan to the model (registration.py:387-524)."""
    cfg = cfg or RegistrationConfig()
    scan = np.asarray(scan, dtype=float).reshape(-1, 3)
    if scan.shape[0] == 0:
        raise RegistrationError("empty scan")
    if cfg.mode not in _MODE:
        raise RegistrationError(f"unknown registration mode {cfg.mode!r}")
    s = max(int(cfg.geo_supersample), 1)
    geo_cam = cam
    if s > 1:
        geo_cam = SphericalCamera(cam.width * s, cam.height * s, cam.az_min, cam.az_max, cam.el_min, cam.el_max)
    # model surface points (sample_model, :190-213) and the photometric anchors X_w = model_pts[::s*s] (:430)
    # the scan's upload and range image are prepared while the model renders
    model_pts, n_model, dscan = sample_anchors(model, geo_cam, initial, cfg, raster, thin=1,
                                               overlap=lambda: DeviceScan(cam, scan))
    if n_model < cfg.min_residuals:
        raise RegistrationError("model renders to too few confident pixels")
    X_w = model_pts[:: s * s].contiguous() if s > 1 else model_pts
    tree, geo_scan = None, None
    if cfg.mode != "photometric":
        geo_scan = scan
        if scan.shape[0] > cfg.max_geo_points:  # registration.py:419-421 (same numpy draw)
            r = rng or np.random.default_rng(0)
            geo_scan = scan[r.choice(scan.shape[0], cfg.max_geo_points, replace=False)]
        tree = build_leaf_tree(model_pts, initial.translation, cfg.leaf_size, cfg.flatness_tau)
        geo_scan = torch.as_tensor(np.ascontiguousarray(geo_scan), device=model_pts.device)
    return solve_device(cfg, initial, dscan, X_w if cfg.mode != "geometric" else None, tree, geo_scan)


def solve_device(cfg: RegistrationConfig, initial, scan: DeviceScan, X_w: torch.Tensor | None = None,
                 tree: LeafTree | None = None, geo_scan: torch.Tensor | None = None) -> RegistrationResult:
    """The GN/LM loop (registration.py:437-524) as one device kernel (``ss_reg_solve``)."""
    dev = engine.require_cuda()
    M = int(X_w.shape[0]) if X_w is not None else 0
    nl = int(tree.dev_centroids.shape[0]) if tree is not None else 0
    ng = int(geo_scan.shape[0]) if geo_scan is not None else 0
    ws = torch.empty(int(lib().ss_reg_solve_workspace_bytes(nl, ng, M)), dtype=torch.uint8, device=dev)
    c = engine.ss_camera(scan.cam)
    k = SsRegSolveCfg(float(cfg.huber_photo), float(cfg.huber_geo), float(cfg.trim_factor), float(cfg.spread_gate),
                      float(cfg.assoc_gate), float(cfg.trim_floor_photo), float(cfg.trim_floor_geo), float(cfg.tol),
                      float(cfg.damping_init), float(cfg.damping_max), int(cfg.max_iters), int(cfg.min_residuals),
                      int(cfg.assoc_k), _MODE[cfg.mode])
    t0 = pose_rt(initial)
    t_out = np.zeros(12)
    info = np.zeros(6, dtype=np.int32)
    r2 = np.zeros(2)
    ptr = lambda t: ctypes.c_void_p(t.data_ptr() if t is not None and t.numel() else 0)  # noqa: E731
    check(lib().ss_reg_solve(ptr(tree.dev_centroids if tree is not None else None),
                             ptr(tree.dev_normals if tree is not None else None), nl, ptr(geo_scan), ng, ptr(X_w), M,
                             ctypes.c_void_p(scan.range.data_ptr()), ctypes.c_void_p(scan.valid.data_ptr()),
                             ctypes.byref(c), t0.ctypes.data_as(ctypes.c_void_p), ctypes.byref(k),
                             t_out.ctypes.data_as(ctypes.c_void_p), info.ctypes.data_as(ctypes.c_void_p),
                             r2.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(ws.data_ptr()),
                             ctypes.c_void_p(engine.stream_ptr())), "register")
    T = SE3Pose(t_out[:9].reshape(3, 3), t_out[9:]).orthonormalized()
    n_geo, n_photo = int(info[2]), int(info[3])
    rms = lambda s2, m: float(np.sqrt(s2 / m)) if m else 0.0  # noqa: E731
    res = RegistrationResult(T, bool(info[1]), int(info[0]), rms(r2[0], n_geo), rms(r2[1], n_photo), n_geo,
                             n_photo, cfg.mode)
    res.n_evaluations = int(info[4])  # residual evaluations the device loop ran (diagnostic)
    return res


def _solve_device(X_w: torch.Tensor, scan: DeviceScan, initial, cfg: RegistrationConfig) -> RegistrationResult:
    """Photometric device loop on given anchors (kept for the parity tests)."""
    if int(X_w.shape[0]) == 0:
        raise RegistrationError("too few residuals survive association")
    return solve_device(cfg, initial, scan, X_w.contiguous())
