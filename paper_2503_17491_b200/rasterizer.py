"""Drop-in replacement of the reference rasterizer API (pkg/src/splatscan/rasterizer.py).

Same names, argument meaning and error behaviour as the reference:
  RasterConfig        rasterizer.py:69-78
  RenderOutput        rasterizer.py:81-87   (host float64 images, like the reference)
  PixelGradients      rasterizer.py:90-96
  SplatGradients      rasterizer.py:99-124
  BlendRecords        rasterizer.py:136-148 (tile_ptr / pair_splats materialise lazily)
  rasterize_forward   rasterizer.py:455-499
  rasterize_backward  rasterizer.py:534-701 (GeometryError on stale records, zeros when empty)

All arithmetic runs in the sm_100a kernels (engine.py -> libsplatb200.so).
Device tensors of every result stay attached (``.device``) so GPU callers
never pay the host copies.
"""
from __future__ import annotations

import weakref
from dataclasses import dataclass, field

import numpy as np
import torch

from . import engine
from .errors import GeometryError
from .geometry import pose_rt

__all__ = ["RasterConfig", "RenderOutput", "PixelGradients", "SplatGradients", "BlendRecords",
           "rasterize_forward", "rasterize_backward"]


@dataclass(frozen=True)
class RasterConfig:
    tile_size: int = 8
    chunk_size: int = 256
    alpha_cutoff: float = 1.0 / 255.0
    alpha_clamp: float = 0.99
    min_transmittance: float = 1e-4
    denom_eps: float = 1e-12
    cutoff_sigma: float = engine.CUTOFF_SIGMA
    bbox_pad_px: float = 0.5
    # not in the reference (rasterizer.py:69-78): fixed-order, run-to-run bit-identical
    # gradient reduction in the backward of renders made with this config
    deterministic: bool = False


class _Lazy:
    """Host view of a device tensor, copied on first access."""

    def __init__(self, t: torch.Tensor, dtype=np.float64):
        self.t = t
        self.dtype = dtype
        self._host = None

    def host(self) -> np.ndarray:
        if self._host is None:
            self._host = self.t.detach().cpu().numpy().astype(self.dtype)
        return self._host


class RenderOutput:
    """Blended range, camera-frame normal and opacity images (rasterizer.py:81-87)."""

    def __init__(self, range=None, normal=None, opacity=None, device: dict | None = None):
        self._dev = device or {}
        self._host = {"range": range, "normal": normal, "opacity": opacity}

    def _get(self, k):
        if self._host[k] is None:
            self._host[k] = self._dev[k].detach().cpu().numpy().astype(np.float64)  # float32 over PCIe
        return self._host[k]

    range = property(lambda self: self._get("range"), lambda self, v: self._host.__setitem__("range", v))
    normal = property(lambda self: self._get("normal"), lambda self, v: self._host.__setitem__("normal", v))
    opacity = property(lambda self: self._get("opacity"), lambda self, v: self._host.__setitem__("opacity", v))

    @property
    def device(self) -> dict:
        return self._dev


@dataclass
class PixelGradients:
    d_range: np.ndarray
    d_normal: np.ndarray
    d_opacity: np.ndarray


@dataclass
class SplatGradients:
    d_centers: np.ndarray
    d_t_alpha: np.ndarray
    d_t_beta: np.ndarray
    d_normal: np.ndarray
    d_scales: np.ndarray
    d_opacity: np.ndarray

    @classmethod
    def zeros(cls, n: int) -> "SplatGradients":
        return cls(np.zeros((n, 3)), np.zeros((n, 3)), np.zeros((n, 3)), np.zeros((n, 3)), np.zeros((n, 2)),
                   np.zeros(n))

    @classmethod
    def from_device(cls, g: torch.Tensor) -> "SplatGradients":
        """From the (n, 15) float32 device gradients: laid out field by field on the device,
        each field copied into a reused pinned buffer in ~0.5 M-value pieces, each behind its
        own event, and widened into a new float64 array on a host thread as soon as it lands (numpy's casts release
        the GIL), so the download and the widening overlap."""
        n = g.shape[0]
        cols = ((0, 3), (3, 6), (6, 9), (9, 12), (12, 14), (14, 15))
        flat = torch.cat([g[:, a:b].reshape(-1) for a, b in cols])
        buf = _pinned_f32(flat.numel())
        host = buf.numpy()
        outs, jobs, off = [], [], 0
        rows = max(1, (1 << 19) // 3)  # ~0.5 M values per piece
        for a, b in cols:
            w = b - a
            o = np.empty((n, w) if w > 1 else (n,), dtype=np.float64)
            for r0 in range(0, n, rows):
                r1 = min(n, r0 + rows)
                p0, p1 = off + r0 * w, off + r1 * w
                buf[p0:p1].copy_(flat[p0:p1], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record()
                jobs.append((ev, o[r0:r1], host[p0:p1].reshape(o[r0:r1].shape)))
            outs.append(o)
            off += n * w

        def widen(j):
            j[0].synchronize()
            np.copyto(j[1], j[2])

        list(_pool().map(widen, jobs))
        return cls(*outs)

    @classmethod
    def from_packed(cls, g: np.ndarray) -> "SplatGradients":
        g = np.asarray(g, dtype=np.float64)
        return cls(g[:, 0:3].copy(), g[:, 3:6].copy(), g[:, 6:9].copy(), g[:, 9:12].copy(), g[:, 12:14].copy(),
                   g[:, 14].copy())


class BlendRecords:
    """Binning and identity snapshot for replaying a render (rasterizer.py:136-148)."""

    def __init__(self, cam, pose, config, n_splats, model_version, tiles_x, tiles_y, handle=None,
                 tile_ptr=None, pair_splats=None):
        self.cam = cam
        self.pose = pose
        self.config = config
        self.n_splats = n_splats
        self.model_version = model_version
        self.tiles_x = tiles_x
        self.tiles_y = tiles_y
        self._handle = handle
        self._tile_ptr = tile_ptr
        self._pair_splats = pair_splats

    def _export(self):
        if self._tile_ptr is None:
            tp, ps = self._handle.export()
            self._tile_ptr = tp.cpu().numpy()
            self._pair_splats = ps.cpu().numpy()

    @property
    def tile_ptr(self) -> np.ndarray:
        self._export()
        return self._tile_ptr

    @property
    def pair_splats(self) -> np.ndarray:
        self._export()
        return self._pair_splats


_PINNED: dict = {}
_POOL = None


def _pinned_f32(n: int) -> torch.Tensor:
    """A reused pinned host buffer of at least n float32 (grown as needed)."""
    t = _PINNED.get("f32")
    if t is None or t.numel() < n:
        t = torch.empty(max(n, 1), dtype=torch.float32, pin_memory=True)
        _PINNED["f32"] = t
    return t[:n]


def _pool():
    global _POOL
    if _POOL is None:
        from concurrent.futures import ThreadPoolExecutor
        _POOL = ThreadPoolExecutor(max_workers=8, thread_name_prefix="splat-host")
    return _POOL


# float32 device copies of models, keyed by object identity, version, the parameter
# arrays' identities and buffers, and a content fingerprint of each array
_dev_cache: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def _identity_key(model) -> tuple:
    key = [int(getattr(model, "version", 0)), len(model)]
    for k in engine.PARAM_NAMES:
        a = getattr(model, k)
        key.append((id(a), a.ctypes.data if isinstance(a, np.ndarray) else 0))
    return tuple(key)


def _fingerprints(model) -> tuple:
    """Content fingerprints of the parameter arrays (``engine.fingerprints``: a position-
    weighted wrapping sum of the float64 bit patterns, one pass on host threads).  Any
    in-place edit the reference's version counter would not see (``model.centers[i] = ...``
    without ``touch()``) changes them; the reference itself re-reads the arrays every call."""
    return engine.fingerprints([getattr(model, k) for k in engine.PARAM_NAMES])


def _cache_key(model) -> tuple:
    """(identity key: version, length, the arrays' identities and buffers; content fingerprints)."""
    return _identity_key(model), _fingerprints(model)


def _device_params(model) -> dict:
    """float32 device copy of ``model``'s parameters, reused while the model is unchanged.
    The content fingerprints are only computed when everything else matches (a changed
    version or array already forces the upload, whose staging pass fingerprints them)."""
    ident = _identity_key(model)
    try:
        hit = _dev_cache.get(model)
    except TypeError:
        hit = None
    if hit is not None and hit[0][0] == ident:
        fp = _fingerprints(model)
        if hit[0][1] == fp:
            return hit[1]
    t, fp = engine.splats_to_device(model, want_fingerprints=True)
    try:
        _dev_cache[model] = ((ident, fp), t)
    except TypeError:
        pass
    return t


def rasterize_forward(cam, pose, model, cfg: RasterConfig | None = None):
    """Render ``model`` from ``pose`` onto ``cam`` (rasterizer.py:455-499)."""
    cfg = cfg or RasterConfig()
    H, W = cam.height, cam.width
    T = cfg.tile_size
    tx, ty = (W + T - 1) // T, (H + T - 1) // T
    pose_c = pose.copy()
    if len(model) == 0:
        rec = BlendRecords(cam, pose_c, cfg, 0, model.version, tx, ty,
                           tile_ptr=np.zeros(tx * ty + 1, dtype=np.int64), pair_splats=np.zeros(0, dtype=np.int64))
        return RenderOutput(np.zeros((H, W)), np.zeros((H, W, 3)), np.zeros((H, W))), rec
    params = _device_params(model)
    handle = engine.Records.acquire()
    D, N, O = engine.forward(cam, pose_rt(pose), params, cfg, handle)
    out = RenderOutput(device={"range": D, "normal": N, "opacity": O})
    rec = BlendRecords(cam, pose_c, cfg, len(model), model.version, tx, ty, handle=handle)
    rec._params = params
    # the records' device buffers go back to the pool when the caller drops them
    # (stream-ordered reuse; no free / malloc per render)
    weakref.finalize(rec, handle.release)
    return out, rec


def _pixel_grads_to_device(pg, H: int, W: int):
    """The three pixel-gradient images as float32 device tensors: rounded to float32 on host
    threads into one reused pinned buffer, one upload (a pageable float64 upload per image
    cost ~1 ms at config 1).  Device tensors pass through."""
    xs, shapes = (pg.d_range, pg.d_normal, pg.d_opacity), ((H, W), (H, W, 3), (H, W))
    if any(isinstance(x, torch.Tensor) for x in xs):
        return tuple(_dev(x, sh) for x, sh in zip(xs, shapes))
    arrs = []
    for x, sh in zip(xs, shapes):
        a = np.asarray(x)
        if a.size != int(np.prod(sh)):
            raise ValueError(f"pixel gradient of {a.size} values, expected {int(np.prod(sh))}")
        arrs.append(a)
    dev32, offs, _ = engine.stage_upload_f32(arrs)
    return tuple(dev32[offs[j]:offs[j + 1]].view(shapes[j]) for j in range(3))


def _dev(x, like_shape):
    if isinstance(x, torch.Tensor):
        return x.to(engine.require_cuda(), torch.float32).contiguous()
    a = np.ascontiguousarray(x)
    if a.dtype not in (np.float32, np.float64):
        a = a.astype(np.float64)
    return torch.from_numpy(a.reshape(like_shape)).to(engine.require_cuda()).to(torch.float32).contiguous()


def rasterize_backward(model, records: BlendRecords, render: RenderOutput, pixel_grads: PixelGradients):
    """Gradients of a pixel-space loss w.r.t. plain splat parameters (rasterizer.py:534-701)."""
    if records.n_splats != len(model) or records.model_version != model.version:
        raise GeometryError("blend records are stale for this model")
    n = len(model)
    if n == 0 or records._handle is None:
        return SplatGradients.zeros(n)
    H, W = records.cam.height, records.cam.width
    params = getattr(records, "_params", None) or _device_params(model)
    gD, gN, gO = _pixel_grads_to_device(pixel_grads, H, W)
    g = engine.backward(records._handle, params, gD, gN, gO, raw_space=False)
    out = SplatGradients.from_device(g)
    out.device = g
    return out
