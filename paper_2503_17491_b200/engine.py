"""Device engine: torch-owned device memory + the C-ABI kernels.

PyTorch provides device memory and the current CUDA stream (plumbing only);
all hot-path arithmetic runs in the sm_100a kernels of libsplatb200.so.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import SsCamera, SsRasterCfg, SsSplats, check, lib

CUTOFF_SIGMA = float(np.sqrt(2.0 * np.log(255.0)))  # rasterizer.py:66

PARAM_NAMES = ("centers", "raw_t_alpha", "raw_t_beta", "log_scales", "logit_opacity")
PARAM_WIDTH = {"centers": 3, "raw_t_alpha": 3, "raw_t_beta": 3, "log_scales": 2, "logit_opacity": 1}


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2503_17491_b200 needs a CUDA device (sm_100a); no CPU fallback exists")
    lib()
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def ss_camera(cam) -> SsCamera:
    return SsCamera(int(cam.width), int(cam.height), float(cam.az_min), float(cam.az_max), float(cam.el_min),
                    float(cam.el_max))


def ss_cfg(cfg) -> SsRasterCfg:
    return SsRasterCfg(int(cfg.tile_size), int(getattr(cfg, "chunk_size", 256)), float(cfg.alpha_cutoff),
                       float(cfg.alpha_clamp), float(cfg.min_transmittance), float(cfg.denom_eps),
                       float(cfg.cutoff_sigma), float(cfg.bbox_pad_px))


def ss_splats(t: dict) -> SsSplats:
    n = int(t["centers"].shape[0])
    for k in PARAM_NAMES:
        x = t[k]
        if x.dtype != torch.float32 or not x.is_cuda or not x.is_contiguous() or x.shape[0] != n:
            raise ValueError(f"{k}: expected contiguous float32 CUDA tensor with {n} rows")
    return SsSplats(n, *(t[k].data_ptr() for k in PARAM_NAMES))


_STAGE: dict = {}


def _host_pool():
    pool = _STAGE.get("pool")
    if pool is None:
        from concurrent.futures import ThreadPoolExecutor
        pool = _STAGE["pool"] = ThreadPoolExecutor(max_workers=8, thread_name_prefix="splat-upload")
    return pool


_CHUNK = 1 << 19  # float64 values per host staging job (and per pipelined upload)


def _stage_chunks(src: np.ndarray, dst, fp: bool = True) -> list:
    """``ss_host_stage_f64`` jobs (src, dst, begin, end, fp) over chunks of the flat float64
    array ``src``: copied into ``dst`` (float64 or float32, rounded to nearest) unless it is
    None, and fingerprinted when ``fp``."""
    return [(src, dst, b, min(b + _CHUNK, src.size), fp) for b in range(0, max(src.size, 1), _CHUNK)]


def _run_stage(job) -> int:
    src, dst, b, e, want = job
    if e <= b:
        return 0
    fp = ctypes.c_uint64(0)
    f32 = dst is not None and dst.dtype == np.float32
    dptr = None if dst is None else dst.ctypes.data + dst.itemsize * b
    check(lib().ss_host_stage_f64(src.ctypes.data + 8 * b, dptr, int(f32), e - b, b,
                                  ctypes.byref(fp) if want or dst is None else None))
    return fp.value


def fingerprints(arrays) -> tuple:
    """Content fingerprints of host arrays (float64 values; ``ss_host_stage_f64``, host threads):
    any in-place edit changes them.  Equal to the ones ``splats_to_device`` reports."""
    flats = [np.ascontiguousarray(np.asarray(a, dtype=np.float64)).reshape(-1) for a in arrays]
    return _sum_fps([_stage_chunks(f, None) for f in flats])


def _sum_fps(job_lists) -> tuple:
    flat = [j for jl in job_lists for j in jl]
    fps = list(_host_pool().map(_run_stage, flat))
    out, q = [], 0
    for jl in job_lists:
        out.append(sum(fps[q:q + len(jl)]) & 0xFFFFFFFFFFFFFFFF)
        q += len(jl)
    return tuple(out)


def _pinned_stage(key, n: int):
    """A reused pinned float32 staging buffer of >= n values and its upload event (waited
    on: the previous upload from it has left)."""
    st = _STAGE.get(key)
    if st is None or st[0].numel() < n:
        st = (torch.empty(max(n, 1), dtype=torch.float32).pin_memory(), torch.cuda.Event())
        _STAGE[key] = st
    else:
        st[1].synchronize()
    return st


def stage_upload_f32(arrays, device=None, want_fingerprints: bool = False):
    """Host arrays -> one float32 device tensor (their concatenation) through a reused pinned
    buffer: float64 arrays are rounded to float32 on host threads in the same pass that
    fingerprints them (``ss_host_stage_f64``; the same rounding as a device conversion, half
    the PCIe bytes), other dtypes are cast by numpy.  Each ~1M-value chunk is uploaded as soon
    as it is staged, so the host pass and the DMA overlap.  Returns (device tensor, offsets,
    fingerprints or None)."""
    device = device or require_cuda()
    arrs = [np.ascontiguousarray(a).reshape(-1) for a in arrays]
    arrs = [a if a.dtype in (np.float32, np.float64) else a.astype(np.float64) for a in arrs]
    offs = np.concatenate([[0], np.cumsum([a.size for a in arrs])]).astype(int)
    total = int(offs[-1])
    st = _pinned_stage(("stage32", len(arrs)), total)
    host = st[0].numpy()
    dev = torch.empty(max(total, 1), dtype=torch.float32, device=device)[:total]
    pool = _host_pool()
    pending = []  # (future, global begin, global end, array index or -1)
    for j, a in enumerate(arrs):
        o = int(offs[j])
        if a.dtype == np.float64:
            for job in _stage_chunks(a, host[o:int(offs[j + 1])], want_fingerprints):
                pending.append((pool.submit(_run_stage, job), o + job[2], o + job[3], j))
        else:
            pending.append((pool.submit(np.copyto, host[o:int(offs[j + 1])], a), o, int(offs[j + 1]), -1))
    fps = [0] * len(arrs)
    for fut, b, e, j in pending:
        r = fut.result()
        if j >= 0:
            fps[j] = (fps[j] + r) & 0xFFFFFFFFFFFFFFFF
        if e > b:
            dev[b:e].copy_(st[0][b:e], non_blocking=True)
    st[1].record()
    if want_fingerprints:
        casts = [j for j, a in enumerate(arrs) if a.dtype != np.float64]
        fx = fingerprints([arrs[j] for j in casts]) if casts else ()
        for q, j in enumerate(casts):
            fps[j] = fx[q]
    return dev, offs, (tuple(fps) if want_fingerprints else None)


def splats_to_device(model, device=None, want_fingerprints: bool = False):
    """float32 device copies of a SplatModel's raw parameters (reference or ours).

    The host arrays go through one reused pinned staging buffer (``stage_upload_f32``:
    float64 rounded to float32 and fingerprinted on host threads in one pass) and one DMA.
    With ``want_fingerprints`` the arrays' content fingerprints (``fingerprints``) come back
    too, so a cache keyed on them costs no second read of the model."""
    n = len(model)
    dev, offs, fps = stage_upload_f32([getattr(model, k) for k in PARAM_NAMES], device, want_fingerprints)
    out = {}
    for j, k in enumerate(PARAM_NAMES):
        t = dev[offs[j]:offs[j + 1]]
        out[k] = t if k == "logit_opacity" else t.view(n, PARAM_WIDTH[k])
    return (out, fps) if want_fingerprints else out


def as_device_params(x) -> dict:
    """float32 CUDA tensors from a SplatModel, a dict of numpy arrays, or a dict of tensors."""
    if not isinstance(x, dict):
        return splats_to_device(x)
    dev = require_cuda()
    out = {}
    for k in PARAM_NAMES:
        v = x[k]
        t = v if torch.is_tensor(v) else torch.from_numpy(np.ascontiguousarray(np.asarray(v, dtype=np.float32)))
        t = t.to(dev, torch.float32).contiguous()
        out[k] = t.reshape(-1) if k == "logit_opacity" else t.reshape(-1, PARAM_WIDTH[k])
    return out


class Records:
    """Owner of one ss_records handle (tile lists + per-pixel blend state)."""

    _pool: list = []

    def __init__(self):
        ptr = lib().ss_records_create()
        if not ptr:
            raise RuntimeError("ss_records_create failed")
        self.ptr = ctypes.c_void_p(ptr)

    @classmethod
    def acquire(cls) -> "Records":
        return cls._pool.pop() if cls._pool else cls()

    def release(self) -> None:
        """Return the handle (and its device buffers) for reuse; beyond a few pooled
        handles it is destroyed instead."""
        if len(Records._pool) < 8:
            Records._pool.append(self)

    def check(self, wait: bool = True) -> int:
        """Status of the last forward (SS_ERR_CAPACITY means: re-run it)."""
        return int(lib().ss_records_check(self.ptr, int(bool(wait))))

    def generation(self) -> int:
        """Buffer generation (bumped when a forward / backward reallocated a device buffer)."""
        g = ctypes.c_uint64(0)
        check(lib().ss_records_generation(self.ptr, ctypes.byref(g)), "records")
        return int(g.value)

    def counts(self):
        n = ctypes.c_int64(0)
        tx = ctypes.c_int32(0)
        ty = ctypes.c_int32(0)
        check(lib().ss_records_counts(self.ptr, ctypes.byref(n), ctypes.byref(tx), ctypes.byref(ty)), "records")
        return int(n.value), int(tx.value), int(ty.value)

    def export(self):
        """(tile_ptr int64, pair_splats int64) as device tensors (BlendRecords layout)."""
        n, tx, ty = self.counts()
        dev = require_cuda()
        tp = torch.empty(tx * ty + 1, dtype=torch.int64, device=dev)
        ps = torch.empty(n, dtype=torch.int64, device=dev)
        check(lib().ss_records_export(self.ptr, ctypes.c_void_p(tp.data_ptr()),
                                      ctypes.c_void_p(ps.data_ptr() if n else 0), ctypes.c_void_p(stream_ptr())),
              "records export")
        return tp, ps

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            if _lib._lib is not None and self.ptr:
                _lib._lib.ss_records_destroy(self.ptr, ctypes.c_void_p(stream_ptr()))
        except Exception:
            pass


def forward(cam, pose_rt: np.ndarray, splats: dict, cfg, records: Records, sync: bool = True, out=None):
    """Render; returns (range [H,W], normal [H,W,3], opacity [H,W]) float32 device tensors.

    The C-ABI forward is fully stream-ordered with a speculative pair
    capacity.  With ``sync`` (default) the call waits for completion and
    transparently re-runs when the capacity was too small; with
    ``sync=False`` the caller must call ``records.check()`` before trusting
    the outputs (bench / CUDA-graph loops)."""
    dev = require_cuda()
    H, W = int(cam.height), int(cam.width)
    if out is None:
        D = torch.empty((H, W), dtype=torch.float32, device=dev)
        N = torch.empty((H, W, 3), dtype=torch.float32, device=dev)
        O = torch.empty((H, W), dtype=torch.float32, device=dev)
    else:
        D, N, O = out
    c = ss_camera(cam)
    sp = ss_splats(splats)
    k = ss_cfg(cfg)
    prt = np.ascontiguousarray(pose_rt, dtype=np.float64)
    lib().ss_records_set_deterministic(records.ptr, int(bool(getattr(cfg, "deterministic", False))))
    for _attempt in range(4):
        st = lib().ss_render_forward(ctypes.byref(c), prt.ctypes.data_as(ctypes.c_void_p), ctypes.byref(sp),
                                     ctypes.byref(k), ctypes.c_void_p(D.data_ptr()), ctypes.c_void_p(N.data_ptr()),
                                     ctypes.c_void_p(O.data_ptr()), records.ptr, ctypes.c_void_p(stream_ptr()))
        check(st, "rasterize_forward")
        if not sync:
            break
        st = records.check(wait=True)
        if st != _lib.SS_ERR_CAPACITY:
            check(st, "rasterize_forward")
            break
    return D, N, O


def backward(records: Records, splats: dict, dD, dN, dO, raw_space: bool, d_scales_extra=None, out=None):
    """Splat gradients: (n, 15) plain-space or (n, 12) raw-space float32 device tensor
    (written into ``out`` when given: a contiguous float32 tensor of that shape)."""
    dev = require_cuda()
    n = int(splats["centers"].shape[0])
    shape = (n, 12 if raw_space else 15)
    if out is None:
        out = torch.empty(shape, dtype=torch.float32, device=dev)
    elif tuple(out.shape) != shape or out.dtype != torch.float32 or not out.is_contiguous():
        raise ValueError(f"out must be a contiguous float32 tensor of shape {shape}")
    dD = dD.contiguous().float()
    dN = dN.contiguous().float()
    dO = dO.contiguous().float()
    ex = 0
    if d_scales_extra is not None:
        d_scales_extra = d_scales_extra.contiguous().float()
        ex = d_scales_extra.data_ptr()
    sp = ss_splats(splats)
    st = lib().ss_render_backward(records.ptr, ctypes.byref(sp), ctypes.c_void_p(dD.data_ptr()),
                                  ctypes.c_void_p(dN.data_ptr()), ctypes.c_void_p(dO.data_ptr()), ctypes.c_void_p(ex),
                                  ctypes.c_void_p(out.data_ptr()), int(bool(raw_space)),
                                  ctypes.c_void_p(stream_ptr()))
    check(st, "rasterize_backward")
    return out


FINALIZE_ALIGN = 128  # ss_render_finalize row chunks start on multiples of this


def backward_blend(records: Records, splats: dict, dD, dN, dO) -> None:
    """First half of ``backward``: the blend backward into the records' accumulators."""
    require_cuda()
    sp = ss_splats(splats)
    dD, dN, dO = (x.contiguous().float() for x in (dD, dN, dO))
    st = lib().ss_render_backward_blend(records.ptr, ctypes.byref(sp), ctypes.c_void_p(dD.data_ptr()),
                                        ctypes.c_void_p(dN.data_ptr()), ctypes.c_void_p(dO.data_ptr()),
                                        ctypes.c_void_p(stream_ptr()))
    check(st, "rasterize_backward")
    records._pix_grads = (dD, dN, dO)  # alive until the stream consumed them


def finalize(records: Records, splats: dict, out, begin: int, end: int, raw_space: bool = True,
             d_scales_extra=None) -> None:
    """Second half of ``backward`` for splats [begin, end) into rows begin..end-1 of ``out``."""
    sp = ss_splats(splats)
    ex = 0 if d_scales_extra is None else d_scales_extra.data_ptr()
    st = lib().ss_render_finalize(records.ptr, ctypes.byref(sp), ctypes.c_void_p(ex),
                                  ctypes.c_void_p(out.data_ptr()), int(bool(raw_space)), int(begin), int(end),
                                  ctypes.c_void_p(stream_ptr()))
    check(st, "rasterize_backward")


def mapping_loss(D, N, O, kf_range, kf_valid, kf_normal, kf_nvalid, w_opacity=0.05, w_normal=0.1,
                 range_floor=1.0):
    """Fused loss (mapping.py:128-163 terms): returns (dD, dN, dO, parts[3] float64 device)."""
    H, W = D.shape
    dD = torch.empty_like(D)
    dN = torch.empty_like(N)
    dO = torch.empty_like(O)
    parts = torch.zeros(4, dtype=torch.float64, device=D.device)
    st = lib().ss_mapping_loss(W, H, D.data_ptr(), N.data_ptr(), O.data_ptr(), kf_range.data_ptr(),
                               kf_valid.data_ptr(), kf_normal.data_ptr(), kf_nvalid.data_ptr(), float(w_opacity),
                               float(w_normal), float(range_floor), dD.data_ptr(), dN.data_ptr(), dO.data_ptr(),
                               parts.data_ptr(), stream_ptr())
    check(st, "mapping_loss")
    return dD, dN, dO, parts
