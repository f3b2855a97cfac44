"""Device-resident map refinement (reference: pkg/src/splatscan/mapping.py:342-498).

``refine(lmap, cfg, iters, rng)`` runs the reference's refine loop -- sample a
keyframe (same numpy draw), render, mapping loss, backward to the raw
parameters, Adam with per-group learning rates, log-scale clamp -- with every
per-pixel and per-splat operation in the sm_100a kernels: the rasterizer,
``ss_mapping_loss``, ``ss_scale_loss`` and the fused ``ss_adam_step``.  The
map's parameters and Adam moments stay on the device between iterations
(SURVEY 8(f) item 1); ``refine`` on a reference ``LocalMap`` uploads, runs
and writes parameters and optimiser state back.

Keyframe creation, densification and pruning (RNG-driven, host-side) are
not on this path.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import engine
from ._lib import check, lib
from .geometry import pose_rt
from .rasterizer import RasterConfig

__all__ = ["MappingConfig", "DeviceKeyframe", "DeviceMap", "refine", "sample_keyframe_index"]


@dataclass
class MappingConfig:
    """Same fields and defaults as the reference (mapping.py:69-93)."""
    n_spawn: int = 20000
    refine_iters: int = 10
    w_opacity: float = 0.05
    w_normal: float = 0.1
    w_scale: float = 1.0
    scale_cap: float = 0.5
    densify_opacity: float = 0.5
    densify_range_err: float = 0.1
    kf_sample_p: float = 0.4
    max_keyframes: int = 100
    prune_opacity: float = 0.005
    coverage_min: float = 0.3
    reset_radius: float = 50.0
    lr_centers: float = 1e-3
    lr_tangents: float = 1e-3
    lr_log_scales: float = 5e-3
    lr_logit_opacity: float = 5e-2
    scale_floor: float = 1e-4
    opacity_init: float = 0.5
    footprint_gain: float = 1.0
    range_weight_floor: float = 1.0


def sample_keyframe_index(n: int, p: float, rng) -> int:
    """Truncated geometric draw over keyframe ages (mapping.py:441-452), same numpy call."""
    if n <= 0:
        raise ValueError("no keyframes to sample")
    w = p * (1.0 - p) ** np.arange(n)
    w /= w.sum()
    return n - 1 - int(rng.choice(n, p=w))


class DeviceKeyframe:
    """Camera, pose and target images of one keyframe on the device."""

    def __init__(self, camera, pose, range_img, valid, normals, nvalid, index: int = 0):
        dev = engine.require_cuda()
        self.camera = camera
        self.pose = pose
        self.index = index
        # float64 images drive spawning (exact reference arithmetic); float32 copies feed the loss
        self.range64 = torch.as_tensor(np.ascontiguousarray(range_img, np.float64), device=dev)
        self.normal64 = torch.as_tensor(np.ascontiguousarray(normals, np.float64), device=dev)
        self.range = self.range64.float().contiguous()
        self.valid = torch.as_tensor(np.asarray(valid, np.uint8), device=dev).contiguous()
        self.normal = self.normal64.float().contiguous()
        self.nvalid = torch.as_tensor(np.asarray(nvalid, np.uint8), device=dev).contiguous()

    @classmethod
    def from_cloud(cls, cloud, pose, width: int, height: int, camera=None, index: int = 0) -> "DeviceKeyframe":
        """make_keyframe (mapping.py:106-114) on the device: the target images never leave HBM."""
        from . import keyframe as KF
        cam = camera if camera is not None else KF.estimate_camera(
            cloud.cpu().numpy() if torch.is_tensor(cloud) else cloud, width, height)
        im = KF.keyframe_images(cam, cloud)
        kf = cls.__new__(cls)
        kf.camera, kf.pose, kf.index = cam, pose, index
        kf.range64, kf.normal64 = im["range"], im["normal"]
        kf.range = im["range"].float().contiguous()
        kf.valid = im["valid"]
        kf.normal = im["normal"].float().contiguous()
        kf.nvalid = im["nvalid"]
        return kf

    @classmethod
    def from_reference(cls, kf) -> "DeviceKeyframe":
        return cls(kf.camera, kf.pose, kf.range_image.range, kf.range_image.valid, kf.normal_image.normals,
                   kf.normal_image.valid, int(getattr(kf, "index", 0)))


class DeviceMap:
    """Splat parameters + Adam state + keyframes resident on the device."""

    def __init__(self, params: dict, keyframes: list, scene_scale: float = 1.0, t: int = 0, m=None, v=None):
        dev = engine.require_cuda()
        self.params = {k: torch.as_tensor(np.asarray(params[k], np.float32) if not torch.is_tensor(params[k])
                                          else params[k], device=dev).contiguous().float()
                       for k in engine.PARAM_NAMES}
        self.params["logit_opacity"] = self.params["logit_opacity"].reshape(-1)
        n = self.n
        self.m = torch.zeros((n, 12), dtype=torch.float32, device=dev) if m is None else m
        self.v = torch.zeros((n, 12), dtype=torch.float32, device=dev) if v is None else v
        self.t = t
        self.keyframes = keyframes
        self.scene_scale = scene_scale
        self.rec = engine.Records()
        self.d_scales = torch.zeros((n, 2), dtype=torch.float32, device=dev)
        self.losses = torch.zeros((0, 4), dtype=torch.float64, device=dev)
        self.epochs = torch.zeros(n, dtype=torch.int32, device=dev)  # keyframe that spawned each splat

    # --- map growth (mapping.py:383-438) ---------------------------------------------
    @classmethod
    def start(cls, kf: DeviceKeyframe, cfg: MappingConfig, rng, raster: RasterConfig | None = None) -> "DeviceMap":
        """LocalMap.start (mapping.py:392-400): an empty map seeded from one keyframe."""
        ranges = kf.range64[kf.valid.bool()].cpu().numpy()
        scale = float(np.median(ranges)) if ranges.size else 1.0
        empty = {k: np.zeros((0, engine.PARAM_WIDTH[k]) if engine.PARAM_WIDTH[k] > 1 else 0, np.float32)
                 for k in engine.PARAM_NAMES}
        dm = cls(empty, [], max(scale, 1e-3))
        dm.add_keyframe(kf, cfg, rng, raster)
        return dm

    def _resize(self, n_new: int, keep_prefix: int):
        """Per-splat arrays grown to n_new rows (the first keep_prefix rows kept)."""
        dev = self.m.device
        for k in engine.PARAM_NAMES:
            w = engine.PARAM_WIDTH[k]
            t = torch.empty((n_new, w) if w > 1 else (n_new,), dtype=torch.float32, device=dev)
            t[:keep_prefix] = self.params[k][:keep_prefix]
            self.params[k] = t
        for name in ("m", "v"):
            t = torch.zeros((n_new, 12), dtype=torch.float32, device=dev)
            t[:keep_prefix] = getattr(self, name)[:keep_prefix]
            setattr(self, name, t)
        e = torch.zeros(n_new, dtype=torch.int32, device=dev)
        e[:keep_prefix] = self.epochs[:keep_prefix]
        self.epochs = e
        self.d_scales = torch.zeros((n_new, 2), dtype=torch.float32, device=dev)

    def prune(self, prune_opacity: float) -> int:
        """SplatModel.prune + _Adam.prune (splats.py:266-279, mapping.py:363-365) on the device."""
        n = self.n
        if n == 0:
            return 0
        dev = self.m.device
        ws = torch.empty(int(lib().ss_prune_workspace_bytes(n)), dtype=torch.uint8, device=dev)
        kept = ctypes.c_int32(0)
        check(lib().ss_prune_flags(n, ctypes.c_void_p(self.params["logit_opacity"].data_ptr()), float(prune_opacity),
                                   ctypes.byref(kept), ctypes.c_void_p(ws.data_ptr()),
                                   ctypes.c_void_p(engine.stream_ptr())), "prune")
        k = kept.value
        if k == n:
            return 0
        arrays = [(self.params, name, engine.PARAM_WIDTH[name]) for name in engine.PARAM_NAMES]
        for holder, name, w in arrays + [(self.__dict__, "m", 12), (self.__dict__, "v", 12)]:
            src = holder[name]
            dst = torch.empty((k,) + tuple(src.shape[1:]), dtype=torch.float32, device=dev)
            check(lib().ss_prune_compact(n, w, ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(dst.data_ptr()),
                                         ctypes.c_void_p(ws.data_ptr()), ctypes.c_void_p(engine.stream_ptr())),
                  "prune")
            holder[name] = dst
        e = torch.empty(k, dtype=torch.int32, device=dev)
        check(lib().ss_prune_compact(n, 1, ctypes.c_void_p(self.epochs.data_ptr()), ctypes.c_void_p(e.data_ptr()),
                                     ctypes.c_void_p(ws.data_ptr()), ctypes.c_void_p(engine.stream_ptr())), "prune")
        self.epochs = e
        self.d_scales = torch.zeros((k, 2), dtype=torch.float32, device=dev)
        return n - k

    def spawn(self, kf: DeviceKeyframe, mask: torch.Tensor, n_max: int, cfg: MappingConfig, rng) -> int:
        """spawn_splats (mapping.py:254-303): the weighted draw without replacement is numpy's own
        call on the host; weights, back-projection and frames are computed on the device."""
        cam = kf.camera
        idx = np.flatnonzero((mask.bool() & kf.valid.bool()).cpu().numpy().ravel())
        if idx.size == 0:
            return 0
        if idx.size > n_max:
            w_img = torch.empty_like(kf.range64)
            check(lib().ss_spawn_weights(cam.width, cam.height, int(bool(cam.full_circle)),
                                         ctypes.c_void_p(kf.range64.data_ptr()), ctypes.c_void_p(kf.valid.data_ptr()),
                                         ctypes.c_void_p(w_img.data_ptr()), ctypes.c_void_p(engine.stream_ptr())),
                  "spawn weights")
            w = w_img.cpu().numpy().ravel()[idx]
            total = w.sum()
            p = w / total if total > 0 else None
            idx = rng.choice(idx, size=n_max, replace=False, p=p)
        m = int(idx.size)
        n0 = self.n
        self._resize(n0 + m, n0)
        pix = torch.as_tensor(np.ascontiguousarray(idx, np.int64), device=self.m.device)
        c = engine.ss_camera(cam)
        prt = pose_rt(kf.pose)
        ptr = lambda name: ctypes.c_void_p(self.params[name][n0:].data_ptr())  # noqa: E731
        check(lib().ss_spawn_splats(ctypes.byref(c), ctypes.c_void_p(kf.range64.data_ptr()),
                                    ctypes.c_void_p(kf.normal64.data_ptr()), ctypes.c_void_p(kf.nvalid.data_ptr()),
                                    prt.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(pix.data_ptr()), m,
                                    float(cfg.footprint_gain), float(cfg.scale_floor), float(cfg.opacity_init),
                                    ptr("centers"), ptr("raw_t_alpha"), ptr("raw_t_beta"), ptr("log_scales"),
                                    ptr("logit_opacity"), ctypes.c_void_p(engine.stream_ptr())), "spawn")
        self.epochs[n0:] = int(getattr(kf, "index", 0))
        return m

    def add_keyframe(self, kf: DeviceKeyframe, cfg: MappingConfig, rng, raster: RasterConfig | None = None) -> dict:
        """add_keyframe (mapping.py:412-438): prune dead splats, densify where the keyframe is unexplained."""
        stats = {"pruned": 0, "spawned": 0}
        if self.n == 0:
            mask = kf.valid
        else:
            raster = raster or RasterConfig()
            D, N, O = engine.forward(kf.camera, pose_rt(kf.pose), self.params, raster, self.rec)
            mask = torch.empty_like(kf.valid)
            check(lib().ss_densify_mask(int(kf.valid.numel()), ctypes.c_void_p(kf.range64.data_ptr()),
                                        ctypes.c_void_p(kf.valid.data_ptr()), ctypes.c_void_p(D.data_ptr()),
                                        ctypes.c_void_p(O.data_ptr()), float(cfg.densify_opacity),
                                        float(cfg.densify_range_err), ctypes.c_void_p(mask.data_ptr()),
                                        ctypes.c_void_p(engine.stream_ptr())), "densify_mask")
            stats["pruned"] = self.prune(cfg.prune_opacity)
        stats["spawned"] = self.spawn(kf, mask, cfg.n_spawn, cfg, rng)
        self.keyframes.append(kf)
        return stats

    @property
    def n(self) -> int:
        return int(self.params["centers"].shape[0])

    def lrs(self, cfg: MappingConfig) -> np.ndarray:
        return np.array([cfg.lr_centers * self.scene_scale, cfg.lr_tangents, cfg.lr_tangents, cfg.lr_log_scales,
                         cfg.lr_logit_opacity], dtype=np.float64)

    def _render_loss(self, kf_index: int, cfg: MappingConfig, raster: RasterConfig | None, sync: bool,
                     scale_loss: bool = True):
        """Render keyframe ``kf_index`` and its mapping loss: (dD, dN, dO, parts); the scale-loss
        gradient lands in ``self.d_scales`` (scale_loss=False: left to the fused finalize)."""
        raster = raster or RasterConfig()
        kf = self.keyframes[kf_index]
        sp = self.params
        D, N, O = engine.forward(kf.camera, pose_rt(kf.pose), sp, raster, self.rec, sync=sync)
        dD, dN, dO, parts = engine.mapping_loss(D, N, O, kf.range, kf.valid, kf.normal, kf.nvalid,
                                                w_opacity=cfg.w_opacity, w_normal=cfg.w_normal,
                                                range_floor=cfg.range_weight_floor)
        if scale_loss:
            check(lib().ss_scale_loss(ctypes.c_void_p(sp["log_scales"].data_ptr()), self.n, float(cfg.scale_cap),
                                      float(cfg.w_scale), ctypes.c_void_p(self.d_scales.data_ptr()),
                                      ctypes.c_void_p(parts.data_ptr() + 3 * 8), ctypes.c_void_p(engine.stream_ptr())),
                  "scale_loss")
        return dD, dN, dO, parts

    def raw_gradient(self, kf_index: int, cfg: MappingConfig, raster: RasterConfig | None = None,
                     sync: bool = True):
        """Render keyframe ``kf_index``, mapping loss, backward: (n x 12 raw gradient, loss parts
        [range, opacity, normal, scale] float64) on the device."""
        dD, dN, dO, parts = self._render_loss(kf_index, cfg, raster, sync)
        g = engine.backward(self.rec, self.params, dD, dN, dO, raw_space=True, d_scales_extra=self.d_scales)
        return g, parts

    def blend_gradient(self, kf_index: int, cfg: MappingConfig, raster: RasterConfig | None = None,
                       sync: bool = True):
        """``raw_gradient`` up to the per-splat accumulators (render, loss, blend backward);
        ``finalize_rows`` then produces the raw gradient rows.  Returns the loss parts."""
        dD, dN, dO, parts = self._render_loss(kf_index, cfg, raster, sync)
        engine.backward_blend(self.rec, self.params, dD, dN, dO)
        return parts

    def finalize_rows(self, begin: int, end: int, out: torch.Tensor) -> None:
        """Raw gradient rows [begin, end) of the last ``blend_gradient`` into ``out``."""
        engine.finalize(self.rec, self.params, out, begin, end, raw_space=True, d_scales_extra=self.d_scales)

    def apply_adam(self, g: torch.Tensor, cfg: MappingConfig) -> None:
        """Fused Adam step + log-scale clamp (mapping.py:367-379, 495-496)."""
        self.t += 1
        lrs = self.lrs(cfg)
        check(lib().ss_adam_step(*(ctypes.c_void_p(self.params[k].data_ptr()) for k in engine.PARAM_NAMES),
                                 ctypes.c_void_p(g.data_ptr()), ctypes.c_void_p(self.m.data_ptr()),
                                 ctypes.c_void_p(self.v.data_ptr()), self.n, self.t,
                                 lrs.ctypes.data_as(ctypes.c_void_p), 0.9, 0.999, 1e-8,
                                 float(np.log(cfg.scale_floor)), float(np.log(10.0 * cfg.scale_cap)),
                                 ctypes.c_void_p(engine.stream_ptr())), "adam_step")

    def step(self, kf_index: int, cfg: MappingConfig, raster: RasterConfig | None = None) -> torch.Tensor:
        """One refine iteration on keyframe ``kf_index``; returns the device loss parts."""
        g, parts = self.raw_gradient(kf_index, cfg, raster)
        self.apply_adam(g, cfg)
        return parts

    def refine(self, cfg: MappingConfig, iters: int, rng, raster: RasterConfig | None = None,
               graphs: bool = True) -> list:
        """mapping.py:455-498 on the device; returns the per-iteration loss totals.

        With ``graphs`` (default) each keyframe's whole step (render, loss,
        backward, Adam) is captured once as a CUDA graph and replayed, so the
        host only draws the keyframe index: the eager loop is host-bound
        (~0.7 ms of Python and launches per iteration at config 2)."""
        if self.n == 0 or not self.keyframes:
            return []
        if graphs:
            out = self._refine_graphs(cfg, iters, rng, raster or RasterConfig())
            if out is not None:
                return out
        parts = []
        for _ in range(iters):
            idx = sample_keyframe_index(len(self.keyframes), cfg.kf_sample_p, rng)
            parts.append(self.step(idx, cfg, raster))
        P = torch.stack(parts).cpu().numpy()
        w = np.array([1.0, cfg.w_opacity, cfg.w_normal, cfg.w_scale])
        return [float(x) for x in P @ w]

    # --- CUDA-graph refine -----------------------------------------------------------
    _HIST = 4096

    def _graph_key(self, cfg, raster):
        # the graphs hold raw device pointers: the parameter / moment tensors and every
        # buffer of the shared records (whose generation moves when an eager forward or
        # backward reallocated one of them)
        return (self.n, len(self.keyframes), tuple(self.params[k].data_ptr() for k in engine.PARAM_NAMES),
                self.m.data_ptr(), self.v.data_ptr(), self.d_scales.data_ptr(), self.rec.generation(),
                tuple(sorted(vars(cfg).items())), tuple(sorted(vars(raster).items())), self.scene_scale)

    def _graph_step(self, kf_index, cfg, raster):
        # render, loss, blend backward; then the finalize fused with the scale hinge and the
        # Adam step (the raw gradient never leaves the kernel: the same arithmetic as
        # step()'s separate kernels)
        dD, dN, dO, parts = self._render_loss(kf_index, cfg, raster, False, scale_loss=False)
        engine.backward_blend(self.rec, self.params, dD, dN, dO)
        check(lib().ss_records_sticky_overflow(self.rec.ptr, ctypes.c_void_p(self._sticky.data_ptr()),
                                               ctypes.c_void_p(engine.stream_ptr())), "overflow flag")
        lrs = self.lrs(cfg)
        sp = engine.ss_splats(self.params)
        check(lib().ss_render_finalize_adam_dev(self.rec.ptr, ctypes.byref(sp), ctypes.c_void_p(self.d_scales.data_ptr()),
                                                ctypes.c_void_p(self.m.data_ptr()), ctypes.c_void_p(self.v.data_ptr()),
                                                ctypes.c_void_p(self._t_dev.data_ptr()),
                                                ctypes.c_void_p(self._bias.data_ptr()),
                                                lrs.ctypes.data_as(ctypes.c_void_p), 0.9, 0.999, 1e-8,
                                                float(np.log(cfg.scale_floor)), float(np.log(10.0 * cfg.scale_cap)),
                                                float(cfg.scale_cap), float(cfg.w_scale),
                                                ctypes.c_void_p(parts.data_ptr() + 3 * 8),
                                                ctypes.c_void_p(engine.stream_ptr())), "finalize + adam")
        check(lib().ss_store_loss_parts(ctypes.c_void_p(parts.data_ptr()), ctypes.c_void_p(self._hist.data_ptr()),
                                        ctypes.c_void_p(self._it.data_ptr()), self._HIST,
                                        ctypes.c_void_p(engine.stream_ptr())), "loss history")

    def capture_graphs(self, cfg: MappingConfig, raster: RasterConfig | None = None) -> None:
        """Capture the refine step of every keyframe as a CUDA graph now (capture runs nothing:
        no side effect on the map), so that refine() replays only."""
        raster = raster or RasterConfig()
        self._prepare_graphs(cfg, raster)
        for idx in range(len(self.keyframes)):
            self._graph_for(idx, cfg, raster)

    def _graph_for(self, idx, cfg, raster):
        gr = self._graphs.get(idx)
        if gr is None:
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.stream(side):
                with torch.cuda.graph(gr, stream=side):
                    self._graph_step(idx, cfg, raster)
            torch.cuda.current_stream().wait_stream(side)
            self._graphs[idx] = gr
        return gr

    def _prepare_graphs(self, cfg, raster):
        dev = self.m.device
        key = self._graph_key(cfg, raster)
        if getattr(self, "_gkey", None) != key:
            # size the shared records for every keyframe (2x headroom: the step moves the splats)
            most = 0
            for kf in self.keyframes:
                engine.forward(kf.camera, pose_rt(kf.pose), self.params, raster, self.rec)
                most = max(most, self.rec.counts()[0])
            lib().ss_records_reserve(self.rec.ptr, 2 * most + 65536)
            # allocate at that size, backward buffers included (nothing may be allocated under capture)
            self.raw_gradient(len(self.keyframes) - 1, cfg, raster)
            self._graphs = {}
            self._gkey = self._graph_key(cfg, raster)  # after the allocations above
            self._t_dev = torch.zeros(1, dtype=torch.int32, device=dev)
            self._bias = torch.ones(2, dtype=torch.float32, device=dev)
            self._it = torch.zeros(1, dtype=torch.int32, device=dev)
            self._sticky = torch.zeros(1, dtype=torch.int32, device=dev)
            self._hist = torch.zeros((self._HIST, 4), dtype=torch.float64, device=dev)

    # Step-by-step replay for callers that interleave several maps (parallel.LocalMapShard):
    # begin_replay(), then replay_step(k) per iteration, then end_replay().
    def begin_replay(self, cfg: MappingConfig, raster: RasterConfig | None = None) -> None:
        """Capture (or reuse) the per-keyframe step graphs and reset the on-device step state."""
        raster = raster or RasterConfig()
        self.capture_graphs(cfg, raster)  # every keyframe's graph now: no capture inside a timed loop
        self._t_dev.fill_(self.t)
        self._it.zero_()
        self._sticky.zero_()
        self._replay = (cfg, raster)

    def replay_step(self, kf_index: int) -> None:
        """One refine iteration on keyframe ``kf_index`` (graph replay, no host synchronisation)."""
        cfg, raster = self._replay
        self._graph_for(kf_index, cfg, raster).replay()

    def end_replay(self) -> bool:
        """Synchronise; False if a replay overflowed its pair capacity (its results are invalid)."""
        ok = not int(self._sticky.item())
        self.t = int(self._t_dev.item())
        if not ok:
            self._gkey = None
        return ok

    def _refine_graphs(self, cfg, iters, rng, raster):
        """Graph-replayed refine; None when it cannot be used (the eager loop runs instead)."""
        if iters > self._HIST or bool(getattr(raster, "deterministic", False)):
            return None
        self._prepare_graphs(cfg, raster)
        snapshot = ({k: v.clone() for k, v in self.params.items()}, self.m.clone(), self.v.clone(), self.t,
                    rng.bit_generator.state)
        self._t_dev.fill_(self.t)
        self._it.zero_()
        self._sticky.zero_()
        for _ in range(iters):
            idx = sample_keyframe_index(len(self.keyframes), cfg.kf_sample_p, rng)
            self._graph_for(idx, cfg, raster).replay()
        if int(self._sticky.item()):  # a replay overflowed its pair capacity: redo eagerly
            params, m, v, t, state = snapshot
            for k in engine.PARAM_NAMES:
                self.params[k].copy_(params[k])
            self.m.copy_(m)
            self.v.copy_(v)
            self.t = t
            rng.bit_generator.state = state
            self._gkey = None
            return None
        self.t = int(self._t_dev.item())
        P = self._hist[:iters].cpu().numpy()
        w = np.array([1.0, cfg.w_opacity, cfg.w_normal, cfg.w_scale])
        return [float(x) for x in P @ w]

    # --- reference LocalMap interop -------------------------------------------------
    @classmethod
    def from_local_map(cls, lmap) -> "DeviceMap":
        model = lmap.model
        params = {k: getattr(model, k) for k in engine.PARAM_NAMES}
        kfs = [DeviceKeyframe.from_reference(kf) for kf in lmap.keyframes]
        dm = cls(params, kfs, float(lmap.scene_scale))
        opt = getattr(lmap, "optimizer", None)
        if opt is not None and getattr(opt, "slots", None) is not None:
            dm.t = int(opt.t)
            cols = [opt.slots[k] for k in engine.PARAM_NAMES]
            m = np.concatenate([c[0].reshape(dm.n, -1) for c in cols], axis=1)
            v = np.concatenate([c[1].reshape(dm.n, -1) for c in cols], axis=1)
            dm.m = torch.as_tensor(m.astype(np.float32), device=dm.m.device).contiguous()
            dm.v = torch.as_tensor(v.astype(np.float32), device=dm.v.device).contiguous()
        return dm

    def write_back(self, lmap, touches: int = 1) -> None:
        model = lmap.model
        for k in engine.PARAM_NAMES:
            getattr(model, k)[...] = self.params[k].cpu().numpy().astype(np.float64).reshape(getattr(model, k).shape)
        opt = getattr(lmap, "optimizer", None)
        if opt is not None and getattr(opt, "slots", None) is not None:
            opt.t = self.t
            m = self.m.cpu().numpy().astype(np.float64)
            v = self.v.cpu().numpy().astype(np.float64)
            c = 0
            for k in engine.PARAM_NAMES:
                w = engine.PARAM_WIDTH[k]
                shape = opt.slots[k][0].shape
                opt.slots[k] = (m[:, c:c + w].reshape(shape).copy(), v[:, c:c + w].reshape(shape).copy())
                c += w
        for _ in range(max(touches, 1)):  # the reference bumps the version once per Adam step
            model.touch()


def refine(lmap, cfg, iters: int, rng, raster: RasterConfig | None = None) -> list:
    """Drop-in for mapping.refine (mapping.py:455-498) on a reference LocalMap."""
    if len(lmap.model) == 0 or not lmap.keyframes:
        return []
    dm = DeviceMap.from_local_map(lmap)
    losses = dm.refine(cfg, iters, rng, raster)
    dm.write_back(lmap, touches=iters)
    return losses
