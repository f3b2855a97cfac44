"""ctypes front end of the CPU oracle (liboracle.so, built from oracle.c).

TEST INFRASTRUCTURE ONLY: this is the parity checker for the CUDA product
path.  Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline /
``--impl reference`` leg may import it.  The product package
(paper_2503_17491_b200) never imports anything from oracle/.

Every function restates the reference (pkg/src/splatscan/) in float64; see the
header of oracle.c for the file:line map.  Parity of the restatement is pinned
against golden vectors generated from the live reference
(tests/golden/make_golden.py).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "liboracle.so")

_P = ctypes.POINTER
_D = _P(ctypes.c_double)
_I64 = _P(ctypes.c_int64)
_U8 = _P(ctypes.c_uint8)

CUTOFF_SIGMA = float(np.sqrt(2.0 * np.log(255.0)))  # rasterizer.py:66


class _Cam(ctypes.Structure):
    _fields_ = [("width", ctypes.c_int), ("height", ctypes.c_int), ("az_min", ctypes.c_double),
                ("az_max", ctypes.c_double), ("el_min", ctypes.c_double), ("el_max", ctypes.c_double)]


class _Cfg(ctypes.Structure):
    _fields_ = [("tile_size", ctypes.c_int), ("alpha_cutoff", ctypes.c_double),
                ("alpha_clamp", ctypes.c_double), ("min_transmittance", ctypes.c_double),
                ("denom_eps", ctypes.c_double), ("cutoff_sigma", ctypes.c_double),
                ("bbox_pad_px", ctypes.c_double)]


@dataclass(frozen=True)
class OracleCfg:
    """RasterConfig defaults (rasterizer.py:69-78)."""
    tile_size: int = 8
    alpha_cutoff: float = 1.0 / 255.0
    alpha_clamp: float = 0.99
    min_transmittance: float = 1e-4
    denom_eps: float = 1e-12
    cutoff_sigma: float = CUTOFF_SIGMA
    bbox_pad_px: float = 0.5


def build() -> str:
    """Compile liboracle.so with the committed Makefile (gcc only)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(os.path.join(_HERE, "oracle.c")):
            build()
        L = ctypes.CDLL(_LIB)
        L.orc_count_pairs.restype = ctypes.c_int64
        L.orc_splat_arrays.restype = ctypes.c_int
        L.orc_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _cam(cam) -> _Cam:
    w, h, a0, a1, e0, e1 = cam
    return _Cam(int(w), int(h), float(a0), float(a1), float(e0), float(e1))


def _cfg(cfg: OracleCfg) -> _Cfg:
    return _Cfg(cfg.tile_size, cfg.alpha_cutoff, cfg.alpha_clamp, cfg.min_transmittance,
                cfg.denom_eps, cfg.cutoff_sigma, cfg.bbox_pad_px)


def _d(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a, t=_D):
    return a.ctypes.data_as(t)


def intrinsics(cam):
    """(fx, fy, cx, cy, off_u, off_v) of a camera tuple (W, H, az_min, az_max, el_min, el_max)."""
    out = np.empty(6)
    lib().orc_camera_intrinsics(ctypes.byref(_cam(cam)), _ptr(out))
    return out


def pixel_planes(cam):
    W, H = int(cam[0]), int(cam[1])
    dirs = np.empty((H, W, 3)); hx = np.empty((H, W, 3)); hy = np.empty((H, W, 3))
    ok = np.empty((H, W), dtype=np.uint8)
    lib().orc_pixel_planes(ctypes.byref(_cam(cam)), _ptr(dirs), _ptr(hx), _ptr(hy), _ptr(ok, _U8))
    return dirs, hx, hy, ok.astype(bool)


def splat_arrays(params: dict, R, t) -> np.ndarray:
    """(N, 22) float64 camera-frame arrays; see oracle.c for the column layout."""
    c = _d(params["centers"]); n = c.shape[0]
    arr = np.zeros((n, 22))
    rc = lib().orc_splat_arrays(n, _ptr(c), _ptr(_d(params["raw_t_alpha"])), _ptr(_d(params["raw_t_beta"])),
                                _ptr(_d(params["log_scales"])), _ptr(_d(params["logit_opacity"])),
                                _ptr(_d(R)), _ptr(_d(t)), _ptr(arr))
    if rc != 0:
        raise ValueError("degenerate raw tangents")
    return arr


def tile_hits(cam, arr, cfg: OracleCfg = OracleCfg()):
    T = cfg.tile_size
    tx = (int(cam[0]) + T - 1) // T
    ty = (int(cam[1]) + T - 1) // T
    n = arr.shape[0]
    rh = np.zeros((n, ty), dtype=np.uint8); ch = np.zeros((n, tx), dtype=np.uint8)
    lib().orc_tile_hits(ctypes.byref(_cam(cam)), ctypes.byref(_cfg(cfg)), n, _ptr(_d(arr)), _ptr(rh, _U8), _ptr(ch, _U8))
    return rh.astype(bool), ch.astype(bool), tx, ty


def bin_splats(cam, arr, cfg: OracleCfg = OracleCfg()):
    """(tile_ptr int64[tiles+1], pair_splats int64[P], tiles_x, tiles_y)."""
    rh, ch, tx, ty = tile_hits(cam, arr, cfg)
    rh8 = np.ascontiguousarray(rh, dtype=np.uint8); ch8 = np.ascontiguousarray(ch, dtype=np.uint8)
    n = arr.shape[0]
    total = lib().orc_count_pairs(n, tx, ty, _ptr(rh8, _U8), _ptr(ch8, _U8))
    tile_ptr = np.zeros(tx * ty + 1, dtype=np.int64)
    pairs = np.zeros(max(total, 1), dtype=np.int64)
    lib().orc_bin(n, tx, ty, _ptr(rh8, _U8), _ptr(ch8, _U8), _ptr(_d(arr)), _ptr(tile_ptr, _I64), _ptr(pairs, _I64))
    return tile_ptr, pairs[:total], tx, ty


def forward_lists(cam, arr, tile_ptr, pairs, cfg: OracleCfg = OracleCfg(), margins: bool = False):
    """Blend pre-binned lists; returns (D, N, O, stats[evaluated, use, contributing]) and, with
    ``margins``, the per-pixel threshold margin of the parity protocol as a fifth element."""
    W, H = int(cam[0]), int(cam[1])
    D = np.zeros((H, W)); N = np.zeros((H, W, 3)); O = np.zeros((H, W))
    M = np.full((H, W), np.inf) if margins else None
    stats = np.zeros(3, dtype=np.int64)
    tp = np.ascontiguousarray(tile_ptr, dtype=np.int64); ps = np.ascontiguousarray(pairs, dtype=np.int64)
    lib().orc_forward_lists(ctypes.byref(_cam(cam)), ctypes.byref(_cfg(cfg)), _ptr(_d(arr)), _ptr(tp, _I64),
                            _ptr(ps, _I64), _ptr(D), _ptr(N), _ptr(O), _ptr(stats, _I64),
                            _ptr(M) if margins else None)
    return (D, N, O, stats, M) if margins else (D, N, O, stats)


def backward_lists(cam, arr, R, tile_ptr, pairs, D, N, O, gD, gN, gO, cfg: OracleCfg = OracleCfg(),
                   max_threads: int = 16):
    """Plain-space SplatGradients as an (N, 15) array:
    d_centers[0:3] d_t_alpha[3:6] d_t_beta[6:9] d_normal[9:12] d_scales[12:14] d_opacity[14]."""
    n = arr.shape[0]
    out = np.zeros((n, 15))
    tp = np.ascontiguousarray(tile_ptr, dtype=np.int64); ps = np.ascontiguousarray(pairs, dtype=np.int64)
    lib().orc_backward_lists(ctypes.byref(_cam(cam)), ctypes.byref(_cfg(cfg)), n, _ptr(_d(arr)), _ptr(_d(R)),
                             _ptr(tp, _I64), _ptr(ps, _I64), _ptr(_d(D)), _ptr(_d(N)), _ptr(_d(O)),
                             _ptr(_d(gD)), _ptr(_d(gN)), _ptr(_d(gO)), _ptr(out), int(max_threads))
    return out


def raw_gradients(params: dict, plain, d_scales_extra=None):
    """(N, 12) raw-parameter gradients: centers 3, raw_t_alpha 3, raw_t_beta 3, log_scales 2, logit 1."""
    n = plain.shape[0]
    out = np.zeros((n, 12))
    ex = None if d_scales_extra is None else _d(d_scales_extra)
    lib().orc_raw_gradients(n, _ptr(_d(params["raw_t_alpha"])), _ptr(_d(params["raw_t_beta"])),
                            _ptr(_d(params["log_scales"])), _ptr(_d(params["logit_opacity"])), _ptr(_d(plain)),
                            _ptr(ex) if ex is not None else None, _ptr(out))
    return out


def render(cam, R, t, params, cfg: OracleCfg = OracleCfg(), margins: bool = False):
    """Full forward: arrays, binning, blend.  Returns dict with images and lists."""
    arr = splat_arrays(params, R, t)
    tile_ptr, pairs, tx, ty = bin_splats(cam, arr, cfg)
    out = forward_lists(cam, arr, tile_ptr, pairs, cfg, margins=margins)
    res = {"arr": arr, "tile_ptr": tile_ptr, "pair_splats": pairs, "tiles_x": tx, "tiles_y": ty,
           "range": out[0], "normal": out[1], "opacity": out[2], "stats": out[3]}
    if margins:
        res["margin"] = out[4]
    return res


def num_threads() -> int:
    return int(lib().orc_num_threads())
