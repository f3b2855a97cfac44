"""Drop-in photometric registration (reference: pkg/src/splatscan/registration.py).

``register(model, scan, cam, initial, cfg)`` with ``cfg.mode == "photometric"``
follows the reference's Gauss-Newton / Levenberg loop (registration.py:387-524)
line for line on the host (a 6x6 solve per step), while every residual,
Jacobian, median trim and normal-equation reduction runs in the sm_100a
kernels (libsplatb200.so, ``ss_photo_system``), the model render of
``sample_model`` is the B200 rasterizer and the scan range image is built on
the device (``ss_range_image``).  By default the whole GN/LM loop runs in one
cooperative kernel (``ss_reg_photo_solve``: no host round trip per
evaluation); ``register(..., device_loop=False)`` runs it on the host over
``ss_photo_system`` evaluations instead (the two agree to rounding).

The geometric / joint / sequential modes need the PCA leaf tree and k-d tree
association (registration.py:98-274), which SURVEY.md 8(f) lists as the next
item and are not on this path: they raise ``RegistrationError``.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import engine
from ._lib import SsRegCfg, SsRegSolveCfg, check, lib
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

    def __init__(self, cam, scan: np.ndarray):
        dev = engine.require_cuda()
        pts = torch.as_tensor(np.ascontiguousarray(np.asarray(scan, dtype=np.float64).reshape(-1, 3)), device=dev)
        self.cam = cam
        self.range = torch.empty((cam.height, cam.width), dtype=torch.float64, device=dev)
        self.valid = torch.empty((cam.height, cam.width), dtype=torch.uint8, device=dev)
        c = engine.ss_camera(cam)
        check(lib().ss_range_image(ctypes.byref(c), ctypes.c_void_p(pts.data_ptr() if pts.numel() else 0),
                                   int(pts.shape[0]), ctypes.c_void_p(self.range.data_ptr()),
                                   ctypes.c_void_p(self.valid.data_ptr()), ctypes.c_void_p(engine.stream_ptr())),
              "build_range_image")


def sample_anchors(model_or_params, geo_cam, pose, cfg: RegistrationConfig, raster: RasterConfig | None = None,
                   thin: int = 1):
    """Device sample_model (registration.py:190-213): world anchors, thinned by ``thin``.

    Returns (X float64 [n,3] device tensor, number of confident pixels)."""
    raster = raster or RasterConfig()
    params = engine.as_device_params(model_or_params)
    rec = engine.Records.acquire()
    try:
        D, N, O = engine.forward(geo_cam, pose_rt(pose), params, raster, rec)
    finally:
        rec.release()
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
    return X[: counts[1]], int(counts[0])


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


def register(model, scan, cam, initial, cfg: RegistrationConfig | None = None, raster: RasterConfig | None = None,
             rng=None, device_loop: bool = True) -> RegistrationResult:
    """Align a sensor-frame scan to the model (registration.py:387-524, photometric mode)."""
    cfg = cfg or RegistrationConfig()
    scan = np.asarray(scan, dtype=float).reshape(-1, 3)
    if scan.shape[0] == 0:
        raise RegistrationError("empty scan")
    if cfg.mode not in ("geometric", "photometric", "joint", "sequential"):
        raise RegistrationError(f"unknown registration mode {cfg.mode!r}")
    if cfg.mode != "photometric":
        raise RegistrationError(f"mode {cfg.mode!r} needs the leaf-tree association, which is not on the B200 "
                                "path (SURVEY 8(f)); use mode='photometric'")
    s = max(int(cfg.geo_supersample), 1)
    geo_cam = cam
    if s > 1:
        geo_cam = SphericalCamera(cam.width * s, cam.height * s, cam.az_min, cam.az_max, cam.el_min, cam.el_max)
    # anchors: the confident surface points thinned back to scan resolution
    X_w, n_model = sample_anchors(model, geo_cam, initial, cfg, raster, thin=s * s if s > 1 else 1)
    if n_model < cfg.min_residuals:
        raise RegistrationError("model renders to too few confident pixels")
    dscan = DeviceScan(cam, scan)
    if device_loop:
        return _solve_device(X_w, dscan, initial, cfg)
    prob = PhotoProblem(X_w, dscan, cfg)
    return _solve(prob, initial, cfg)


def _solve_device(X_w: torch.Tensor, scan: DeviceScan, initial, cfg: RegistrationConfig) -> RegistrationResult:
    """The GN/LM loop (registration.py:437-524, photometric phase) as one device kernel."""
    X = X_w.contiguous()
    M = int(X.shape[0])
    if M == 0:
        raise RegistrationError("too few residuals survive association")
    ws = torch.empty(int(lib().ss_reg_solve_workspace_bytes(M)), dtype=torch.uint8, device=X.device)
    c = engine.ss_camera(scan.cam)
    k = SsRegSolveCfg(float(cfg.huber_photo), float(cfg.trim_factor), float(cfg.spread_gate), float(cfg.assoc_gate),
                      float(cfg.trim_floor_photo), float(cfg.tol), float(cfg.damping_init), float(cfg.damping_max),
                      int(cfg.max_iters), int(cfg.min_residuals))
    t0 = pose_rt(initial)
    t_out = np.zeros(12)
    info = np.zeros(4, dtype=np.int32)
    r2 = ctypes.c_double(0.0)
    check(lib().ss_reg_photo_solve(ctypes.c_void_p(X.data_ptr()), M, ctypes.c_void_p(scan.range.data_ptr()),
                                   ctypes.c_void_p(scan.valid.data_ptr()), ctypes.byref(c),
                                   t0.ctypes.data_as(ctypes.c_void_p), ctypes.byref(k),
                                   t_out.ctypes.data_as(ctypes.c_void_p), info.ctypes.data_as(ctypes.c_void_p),
                                   ctypes.byref(r2), ctypes.c_void_p(ws.data_ptr()),
                                   ctypes.c_void_p(engine.stream_ptr())), "register")
    T = SE3Pose(t_out[:9].reshape(3, 3), t_out[9:]).orthonormalized()
    m = int(info[2])
    rms = float(np.sqrt(r2.value / m)) if m else 0.0
    return RegistrationResult(T, bool(info[1]), int(info[0]), 0.0, rms, 0, m, cfg.mode)


def _solve(prob: PhotoProblem, initial, cfg: RegistrationConfig) -> RegistrationResult:
    """The reference's GN/LM loop (registration.py:437-524), photometric phase only."""
    T = initial.copy()
    it_total = 0
    converged = False
    last = (0.0, 0)
    lam = cfg.damping_init
    budget = cfg.max_iters
    while it_total < budget:
        it_total += 1
        anneal = cfg.assoc_gate * 0.5 ** it_total
        fp = max(cfg.trim_floor_photo, anneal)
        photo = prob.evaluate(T, fp)
        n_photo = 0
        if photo is not None:
            Hs, bs, hub, m, r2 = photo
            s = 1.0 / m
            H = s * Hs
            b = s * bs
            n_photo = m
            last = (r2, m)
        if n_photo < cfg.min_residuals:
            raise RegistrationError("too few residuals survive association")
        obj0 = s * hub
        accepted = False
        delta = np.zeros(6)
        while lam <= cfg.damping_max:
            try:
                delta = np.linalg.solve(H + lam * np.eye(6), -b)
            except np.linalg.LinAlgError:
                lam = max(lam, 1e-8) * 10.0
                continue
            if not np.all(np.isfinite(delta)):
                lam = max(lam, 1e-8) * 10.0
                continue
            T_try = T.retract(delta)
            p2 = prob.evaluate(T_try, fp, objective_only=True)
            if p2 is not None and s * p2[2] <= obj0 + 1e-12:
                T = T_try
                lam = max(lam * 0.25, cfg.damping_init)
                accepted = True
                break
            lam = max(lam, 1e-8) * 10.0
        if not accepted:
            break
        if np.linalg.norm(delta) < cfg.tol:
            converged = True
            break
    T = T.orthonormalized()
    r2, m = last
    rms = float(np.sqrt(r2 / m)) if m else 0.0
    return RegistrationResult(T, converged, it_total, 0.0, rms, 0, int(m), cfg.mode)
