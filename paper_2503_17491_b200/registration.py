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
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import engine
from ._lib import SS_ERR_CAPACITY, SsRegCfg, SsRegOut, SsRegSolveCfg, check, lib
from .errors import RegistrationError
from .geometry import SE3Pose, SphericalCamera, pose_rt
from .rasterizer import RasterConfig

__all__ = ["RegistrationConfig", "RegistrationResult", "register", "register_batch", "DeviceScan", "PhotoProblem"]


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


# --- frame batches ------------------------------------------------------------------------

class _BatchSlot:
    """Per-frame resources of register_batch, reused across calls: a stream, blend
    records, pinned scan staging, the pinned result record and the loop's workspace."""

    def __init__(self):
        self.stream = torch.cuda.Stream()
        self.rec = engine.Records()
        self.stage = torch.empty((1, 3), dtype=torch.float64).pin_memory()
        self.out_pinned = torch.empty(ctypes.sizeof(SsRegOut), dtype=torch.uint8).pin_memory()
        self.ws = torch.empty(0, dtype=torch.uint8, device=engine.require_cuda())

    def scan_to_device(self, scan: np.ndarray):
        n = scan.shape[0]
        if self.stage.shape[0] < n:
            self.stage = torch.empty((n, 3), dtype=torch.float64).pin_memory()
        self.stage[:n].numpy()[...] = scan
        return self.stage[:n].to(engine.require_cuda(), non_blocking=True)

    def workspace(self, nbytes: int) -> torch.Tensor:
        if self.ws.numel() < nbytes:
            self.ws = torch.empty(nbytes, dtype=torch.uint8, device=self.ws.device)
        return self.ws


_SLOTS: list = []
TIMELINE = None  # a list to collect per-frame (render start, loop launch, loop end) ms (diagnostics)


# cooperative loop blocks per SM in frame batches (k_reg_solve<2>'s launch bounds)
_RS_BLOCKS_PER_SM = int(os.environ.get("SS_RS_BPS", "2"))


def register_batch(model, scans, cam, initials, cfg: RegistrationConfig | None = None,
                   raster: RasterConfig | None = None, rng=None) -> list:
    """B independent registrations at once, each exactly ``register`` (registration.py:
    387-524) on its own scan and initial pose against the same model.

    Every frame gets its own CUDA stream: the B model renders and anchor extractions
    (sample_model, :190-213) are enqueued together, then the B GN/LM loops run as
    concurrent cooperative kernels with num_SMs / B blocks each (``ss_reg_solve_async``)
    -- a single loop is bound by its grid barriers, not by the GPU's width (DESIGN 5b).
    The results equal B calls of ``register`` (the geometric subsample draws take ``rng``
    frame by frame, or a fresh default_rng(0) per frame as ``register`` does)."""
    cfg = cfg or RegistrationConfig()
    B = len(scans)
    if len(initials) != B:
        raise ValueError("one initial pose per scan")
    if B == 0:
        return []
    if cfg.mode not in _MODE:
        raise RegistrationError(f"unknown registration mode {cfg.mode!r}")
    on_dev = all(torch.is_tensor(sc) and sc.is_cuda for sc in scans)  # device-resident scans: no upload
    if on_dev:
        scans = [sc.to(torch.float64).reshape(-1, 3) for sc in scans]
    else:
        scans = [np.asarray(sc.cpu().numpy() if torch.is_tensor(sc) else sc, dtype=float).reshape(-1, 3)
                 for sc in scans]
    if any(sc.shape[0] == 0 for sc in scans):
        raise RegistrationError("empty scan")
    if on_dev and (cfg.mode != "photometric" or TIMELINE is not None):
        scans = [sc.cpu().numpy() for sc in scans]
    dev = engine.require_cuda()
    raster = raster or RasterConfig()
    s = max(int(cfg.geo_supersample), 1)
    geo_cam = cam if s == 1 else SphericalCamera(cam.width * s, cam.height * s, cam.az_min, cam.az_max,
                                                 cam.el_min, cam.el_max)
    params = engine.as_device_params(model)
    while len(_SLOTS) < B:
        _SLOTS.append(_BatchSlot())
    slots = _SLOTS[:B]
    main = torch.cuda.current_stream()
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    blocks = max(1, (nsm * (_RS_BLOCKS_PER_SM if B > 1 else 1)) // B)
    if cfg.mode == "photometric" and TIMELINE is None:
        # (one frame: 0 = one block per SM, the single-registration build of the loop)
        return _photo_batch_native(params, scans, cam, geo_cam, initials, cfg, raster, s, slots, blocks if B > 1 else 0)
    # 1. every frame's model render and scan range image, each on its own stream
    renders, dscans = [], []
    ev = [] if TIMELINE is not None else None
    for b, slot in enumerate(slots):
        slot.stream.wait_stream(main)
        with torch.cuda.stream(slot.stream):
            if ev is not None:
                ev.append([torch.cuda.Event(enable_timing=True) for _ in range(4)])
                ev[b][0].record()
            D, _, O = engine.forward(geo_cam, pose_rt(initials[b]), params, raster, slot.rec, sync=False)
            renders.append((D, O))
            pts = slot.scan_to_device(scans[b])
            ds = DeviceScan.__new__(DeviceScan)
            ds.cam = cam
            ds.range = torch.empty((cam.height, cam.width), dtype=torch.float64, device=dev)
            ds.valid = torch.empty((cam.height, cam.width), dtype=torch.uint8, device=dev)
            c = engine.ss_camera(cam)
            check(lib().ss_range_image(ctypes.byref(c), ctypes.c_void_p(pts.data_ptr()), int(pts.shape[0]),
                                       ctypes.c_void_p(ds.range.data_ptr()), ctypes.c_void_p(ds.valid.data_ptr()),
                                       ctypes.c_void_p(engine.stream_ptr())), "build_range_image")
            dscans.append(ds)
    # 2. per frame: anchors (waits for its own stream only), leaf tree, the loop (enqueued)
    keep = []
    for b, slot in enumerate(slots):
        with torch.cuda.stream(slot.stream):
            D, O = renders[b]
            X, counts = _anchors(D, O, geo_cam, initials[b], cfg, 1)
            if slot.rec.check(True) == SS_ERR_CAPACITY:  # rare: re-render with the exact capacity
                D, _, O = engine.forward(geo_cam, pose_rt(initials[b]), params, raster, slot.rec)
                X, counts = _anchors(D, O, geo_cam, initials[b], cfg, 1)
            model_pts, n_model = X[: counts[1]], int(counts[0])
            if n_model < cfg.min_residuals:
                raise RegistrationError(f"frame {b}: model renders to too few confident pixels")
            X_w = model_pts[:: s * s].contiguous() if s > 1 else model_pts
            tree, geo_scan = None, None
            if cfg.mode != "photometric":
                geo = scans[b]
                if geo.shape[0] > cfg.max_geo_points:
                    r = rng or np.random.default_rng(0)
                    geo = geo[r.choice(geo.shape[0], cfg.max_geo_points, replace=False)]
                tree = build_leaf_tree(model_pts, initials[b].translation, cfg.leaf_size, cfg.flatness_tau)
                geo_scan = torch.as_tensor(np.ascontiguousarray(geo), device=dev)
            Xp = X_w if cfg.mode != "geometric" else None
            M = int(Xp.shape[0]) if Xp is not None else 0
            nl = int(tree.dev_centroids.shape[0]) if tree is not None else 0
            ng = int(geo_scan.shape[0]) if geo_scan is not None else 0
            ws = slot.workspace(int(lib().ss_reg_solve_workspace_bytes(nl, ng, M)))
            # one scan point per thread in the geometric family: at least ng / 256 blocks
            nblk = max(blocks, -(-ng // 256)) if ng else blocks
            c = engine.ss_camera(cam)
            k = _solve_cfg(cfg)
            t0 = pose_rt(initials[b])
            ptr = lambda t: ctypes.c_void_p(t.data_ptr() if t is not None and t.numel() else 0)  # noqa: E731
            if ev is not None:
                ev[b][1].record()
            check(lib().ss_reg_solve_async(ptr(tree.dev_centroids if tree is not None else None),
                                           ptr(tree.dev_normals if tree is not None else None), nl, ptr(geo_scan), ng,
                                           ptr(Xp), M, ctypes.c_void_p(dscans[b].range.data_ptr()),
                                           ctypes.c_void_p(dscans[b].valid.data_ptr()), ctypes.byref(c),
                                           t0.ctypes.data_as(ctypes.c_void_p), ctypes.byref(k), nblk,
                                           ctypes.c_void_p(slot.out_pinned.data_ptr()), ctypes.c_void_p(ws.data_ptr()),
                                           ctypes.c_void_p(engine.stream_ptr())), "register")
            keep.append((X, tree, geo_scan, t0))  # alive until the loops finished
            if ev is not None:
                ev[b][2].record()
    # 3. collect
    results = []
    failed = None
    for b, slot in enumerate(slots):
        slot.stream.synchronize()
        if ev is not None:
            TIMELINE.append([ev[0][0].elapsed_time(e) for e in ev[b][:3]])
        main.wait_stream(slot.stream)
        out = SsRegOut.from_buffer_copy(slot.out_pinned.numpy().tobytes())
        info = list(out.info)
        if info[5] and failed is None:
            failed = b
        T = SE3Pose(np.array(out.T[:9]).reshape(3, 3), np.array(out.T[9:])).orthonormalized()
        rms = lambda s2, m: float(np.sqrt(s2 / m)) if m else 0.0  # noqa: E731
        res = RegistrationResult(T, bool(info[1]), int(info[0]), rms(out.r2[0], info[2]), rms(out.r2[1], info[3]),
                                 int(info[2]), int(info[3]), cfg.mode)
        res.n_evaluations = int(info[4])
        results.append(res)
    if failed is not None:
        raise RegistrationError(f"frame {failed}: too few residuals survive association")
    return results


def _solve_cfg(cfg: RegistrationConfig) -> SsRegSolveCfg:
    return SsRegSolveCfg(float(cfg.huber_photo), float(cfg.huber_geo), float(cfg.trim_factor), float(cfg.spread_gate),
                         float(cfg.assoc_gate), float(cfg.trim_floor_photo), float(cfg.trim_floor_geo), float(cfg.tol),
                         float(cfg.damping_init), float(cfg.damping_max), int(cfg.max_iters), int(cfg.min_residuals),
                         int(cfg.assoc_k), _MODE[cfg.mode])


_NATIVE: dict = {}


def _photo_batch_native(params, scans, cam, geo_cam, initials, cfg, raster, s, slots, blocks):
    """register_batch's photometric path: one C-ABI call enqueues every frame's render,
    range image, anchors and loop (ss_register_photo_batch)."""
    dev = engine.require_cuda()
    B = len(scans)
    Pg, P = geo_cam.width * geo_cam.height, cam.width * cam.height
    thin = s * s
    cap = (Pg + thin - 1) // thin
    a_stride = (int(lib().ss_anchor_workspace_bytes(geo_cam.width, geo_cam.height)) + 255) // 256 * 256
    s_stride = (int(lib().ss_reg_solve_workspace_bytes(0, 0, cap)) + 255) // 256 * 256
    offs = np.zeros(B + 1, dtype=np.int32)
    offs[1:] = np.cumsum([sc.shape[0] for sc in scans])
    key = (B, Pg, P, cap)
    bufs = _NATIVE.get(key)
    if bufs is None:
        _NATIVE.clear()
        bufs = {"render": torch.empty(B * 5 * Pg, dtype=torch.float32, device=dev),
                "range": torch.empty(B * P, dtype=torch.float64, device=dev),
                "valid": torch.empty(B * P, dtype=torch.uint8, device=dev),
                "anchors": torch.empty(B * cap * 3, dtype=torch.float64, device=dev),
                "aws": torch.empty(B * a_stride, dtype=torch.uint8, device=dev),
                "sws": torch.empty(B * s_stride, dtype=torch.uint8, device=dev),
                "out": torch.empty(B * ctypes.sizeof(SsRegOut), dtype=torch.uint8).pin_memory(),
                "pts_host": torch.empty((1, 3), dtype=torch.float64).pin_memory()}
        _NATIVE[key] = bufs
    n = int(offs[-1])
    main = torch.cuda.current_stream()
    if torch.is_tensor(scans[0]):
        pts = torch.cat(scans).contiguous()
    else:
        if bufs["pts_host"].shape[0] < n:
            bufs["pts_host"] = torch.empty((n, 3), dtype=torch.float64).pin_memory()
        host = bufs["pts_host"][:n]
        np.concatenate(scans, out=host.numpy())
        pts = host.to(dev, non_blocking=True)  # on the caller's stream; the frame streams wait for it
    for slot in slots:
        slot.stream.wait_stream(main)
    recs = (ctypes.c_void_p * B)(*[slot.rec.ptr.value for slot in slots])
    streams = (ctypes.c_void_p * B)(*[slot.stream.cuda_stream for slot in slots])
    poses = np.ascontiguousarray(np.stack([pose_rt(p) for p in initials]))
    gc, c = engine.ss_camera(geo_cam), engine.ss_camera(cam)
    sp, rk, k = engine.ss_splats(params), engine.ss_cfg(raster), _solve_cfg(cfg)
    st = lib().ss_register_photo_batch(B, ctypes.byref(gc), ctypes.byref(c), ctypes.byref(sp), ctypes.byref(rk),
                                       recs, streams, poses.ctypes.data_as(ctypes.c_void_p),
                                       ctypes.c_void_p(pts.data_ptr()), offs.ctypes.data_as(ctypes.c_void_p), thin,
                                       float(cfg.visibility_opacity), float(cfg.spread_gate), ctypes.byref(k), blocks,
                                       ctypes.c_void_p(bufs["render"].data_ptr()),
                                       ctypes.c_void_p(bufs["range"].data_ptr()),
                                       ctypes.c_void_p(bufs["valid"].data_ptr()),
                                       ctypes.c_void_p(bufs["anchors"].data_ptr()), cap,
                                       ctypes.c_void_p(bufs["aws"].data_ptr()), a_stride,
                                       ctypes.c_void_p(bufs["sws"].data_ptr()), s_stride,
                                       ctypes.c_void_p(bufs["out"].data_ptr()))
    check(st, "register")
    for slot in slots:
        main.wait_stream(slot.stream)
    raw = bufs["out"].numpy().tobytes()
    results, failed = [], None
    for b in range(B):
        out = SsRegOut.from_buffer_copy(raw[b * ctypes.sizeof(SsRegOut):(b + 1) * ctypes.sizeof(SsRegOut)])
        info = list(out.info)
        if info[5] and failed is None:
            failed = (b, info[5])
        T = SE3Pose(np.array(out.T[:9]).reshape(3, 3), np.array(out.T[9:])).orthonormalized()
        rms = lambda s2, m: float(np.sqrt(s2 / m)) if m else 0.0  # noqa: E731
        res = RegistrationResult(T, bool(info[1]), int(info[0]), rms(out.r2[0], info[2]), rms(out.r2[1], info[3]),
                                 int(info[2]), int(info[3]), cfg.mode)
        res.n_evaluations = int(info[4])
        results.append(res)
    if failed is not None:
        b, code = failed
        raise RegistrationError(f"frame {b}: " + ("model renders to too few confident pixels" if code == 2 else
                                                  "too few residuals survive association"))
    return results
