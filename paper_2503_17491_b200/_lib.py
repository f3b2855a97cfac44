"""Loader and ctypes bindings of the sm_100a C-ABI library (libsplatb200.so).

The declarations mirror include/splat_b200.h.  There is no fallback: if the
library or a CUDA device is missing, every entry point raises.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPLAT_B200_LIB", os.path.join(_HERE, "libsplatb200.so"))  # env: A/B builds
CSRC = os.path.join(_HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(_HERE), "include")

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared"]


def build_library(verbose: bool = False) -> str:
    """Compile libsplatb200.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    cmd = [nvcc, *NVCC_FLAGS, "-o", LIB_PATH, os.path.join(CSRC, "capi.cu")]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.run(cmd, check=True)
    return LIB_PATH


class SsCamera(ctypes.Structure):
    _fields_ = [("width", ctypes.c_int32), ("height", ctypes.c_int32), ("az_min", ctypes.c_double),
                ("az_max", ctypes.c_double), ("el_min", ctypes.c_double), ("el_max", ctypes.c_double)]


class SsRasterCfg(ctypes.Structure):
    _fields_ = [("tile_size", ctypes.c_int32), ("chunk_size", ctypes.c_int32), ("alpha_cutoff", ctypes.c_double),
                ("alpha_clamp", ctypes.c_double), ("min_transmittance", ctypes.c_double),
                ("denom_eps", ctypes.c_double), ("cutoff_sigma", ctypes.c_double), ("bbox_pad_px", ctypes.c_double)]


class SsSplats(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("centers", ctypes.c_void_p), ("raw_t_alpha", ctypes.c_void_p),
                ("raw_t_beta", ctypes.c_void_p), ("log_scales", ctypes.c_void_p),
                ("logit_opacity", ctypes.c_void_p)]


class SsRegSolveCfg(ctypes.Structure):
    _fields_ = [("huber_photo", ctypes.c_double), ("huber_geo", ctypes.c_double), ("trim_factor", ctypes.c_double),
                ("spread_gate", ctypes.c_double), ("assoc_gate", ctypes.c_double),
                ("trim_floor_photo", ctypes.c_double), ("trim_floor_geo", ctypes.c_double), ("tol", ctypes.c_double),
                ("damping_init", ctypes.c_double), ("damping_max", ctypes.c_double), ("max_iters", ctypes.c_int32),
                ("min_residuals", ctypes.c_int32), ("assoc_k", ctypes.c_int32), ("mode", ctypes.c_int32)]


class SsRegCfg(ctypes.Structure):
    _fields_ = [("huber_photo", ctypes.c_double), ("trim_factor", ctypes.c_double), ("spread_gate", ctypes.c_double)]


class SsRegOut(ctypes.Structure):
    _fields_ = [("T", ctypes.c_double * 12), ("r2", ctypes.c_double * 2), ("info", ctypes.c_int32 * 6)]


SS_OK = 0
SS_ERR_INVALID_ARGUMENT = 1
SS_ERR_STALE_RECORDS = 2
SS_ERR_UNSUPPORTED = 3
SS_ERR_CUDA = 4
SS_ERR_CAPACITY = 5
SS_ERR_DEGENERATE = 6
SS_ERR_REGISTRATION = 7

_lib = None


def lib() -> ctypes.CDLL:
    """The loaded library; raises if it is missing (no CPU fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, d = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    L.ss_version.restype = ctypes.c_char_p
    L.ss_records_create.restype = vp
    L.ss_records_destroy.argtypes = [vp, vp]
    L.ss_render_forward.argtypes = [ctypes.POINTER(SsCamera), vp, ctypes.POINTER(SsSplats),
                                    ctypes.POINTER(SsRasterCfg), vp, vp, vp, vp, vp]
    L.ss_records_counts.argtypes = [vp, ctypes.POINTER(i64), ctypes.POINTER(i32), ctypes.POINTER(i32)]
    L.ss_records_export.argtypes = [vp, vp, vp, vp]
    L.ss_records_pixel_state.argtypes = [vp, vp, vp, vp]
    L.ss_records_pixel_state.restype = ctypes.c_int
    L.ss_render_backward.argtypes = [vp, ctypes.POINTER(SsSplats), vp, vp, vp, vp, vp, ctypes.c_int, vp]
    L.ss_render_backward_blend.argtypes = [vp, ctypes.POINTER(SsSplats), vp, vp, vp, vp]
    L.ss_render_backward_blend.restype = ctypes.c_int
    L.ss_render_finalize.argtypes = [vp, ctypes.POINTER(SsSplats), vp, vp, ctypes.c_int, i32, i32, vp]
    L.ss_render_finalize.restype = ctypes.c_int
    L.ss_fp32_peak_tflops.argtypes = [ctypes.POINTER(d), vp]
    L.ss_fp32_peak_tflops.restype = ctypes.c_int
    L.ss_host_stage_f64.argtypes = [vp, vp, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(ctypes.c_uint64)]
    L.ss_host_stage_f64.restype = ctypes.c_int
    L.ss_records_set_deterministic.argtypes = [vp, i32]
    L.ss_records_set_deterministic.restype = ctypes.c_int
    L.ss_records_generation.argtypes = [vp, ctypes.POINTER(ctypes.c_uint64)]
    L.ss_records_generation.restype = ctypes.c_int
    L.ss_records_reserve.argtypes = [vp, i64]
    L.ss_records_reserve.restype = ctypes.c_int
    L.ss_records_sticky_overflow.argtypes = [vp, vp, vp]
    L.ss_records_sticky_overflow.restype = ctypes.c_int
    L.ss_records_check.argtypes = [vp, ctypes.c_int]
    L.ss_records_check.restype = ctypes.c_int
    L.ss_records_work.argtypes = [vp, ctypes.POINTER(i64), ctypes.POINTER(i64), vp]
    L.ss_records_profile.argtypes = [vp, ctypes.c_int]
    L.ss_records_stage_times.argtypes = [vp, ctypes.POINTER(d), ctypes.POINTER(i32), i32]
    L.ss_mapping_loss.argtypes = [i32, i32, vp, vp, vp, vp, vp, vp, vp, d, d, d, vp, vp, vp, vp, vp]
    L.ss_photo_workspace_bytes.argtypes = [i32]
    L.ss_photo_workspace_bytes.restype = ctypes.c_size_t
    L.ss_photo_system.argtypes = [vp, i32, vp, vp, ctypes.POINTER(SsCamera), vp, d, ctypes.POINTER(SsRegCfg),
                                  i32, vp, vp, vp]
    L.ss_anchor_workspace_bytes.argtypes = [i32, i32]
    L.ss_anchor_workspace_bytes.restype = ctypes.c_size_t
    L.ss_reg_anchors.argtypes = [ctypes.POINTER(SsCamera), vp, vp, vp, d, d, i32, vp, i32, vp, vp, vp]
    L.ss_reg_anchors.restype = ctypes.c_int
    L.ss_scale_loss.argtypes = [vp, i32, d, d, vp, vp, vp]
    L.ss_scale_loss.restype = ctypes.c_int
    L.ss_adam_step.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, i32, i32, vp, d, d, d, d, d, vp]
    L.ss_adam_step.restype = ctypes.c_int
    L.ss_adam_step_dev.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, i32, vp, vp, vp, d, d, d, d, d, vp]
    L.ss_adam_step_dev.restype = ctypes.c_int
    L.ss_render_finalize_adam_dev.argtypes = [vp, ctypes.POINTER(SsSplats), vp, vp, vp, vp, vp, vp, d, d, d, d, d, d, d,
                                              vp, vp]
    L.ss_render_finalize_adam_dev.restype = ctypes.c_int
    L.ss_store_loss_parts.argtypes = [vp, vp, vp, i32, vp]
    L.ss_store_loss_parts.restype = ctypes.c_int
    L.ss_range_image.argtypes = [ctypes.POINTER(SsCamera), vp, i32, vp, vp, vp]
    L.ss_range_image.restype = ctypes.c_int
    L.ss_smooth_range_image.argtypes = [i32, i32, i32, vp, vp, vp, vp]
    L.ss_smooth_range_image.restype = ctypes.c_int
    L.ss_range_image_normals.argtypes = [ctypes.POINTER(SsCamera), vp, vp, vp, vp, vp]
    L.ss_range_image_normals.restype = ctypes.c_int
    L.ss_leaf_tree_workspace_bytes.argtypes = [i32]
    L.ss_leaf_tree_workspace_bytes.restype = ctypes.c_size_t
    L.ss_leaf_tree_build.argtypes = [vp, i32, vp, i32, d, i32, vp, vp, vp, vp, vp, vp, vp, vp]
    L.ss_leaf_tree_build.restype = ctypes.c_int
    L.ss_spawn_weights.argtypes = [i32, i32, i32, vp, vp, vp, vp]
    L.ss_densify_mask.argtypes = [i32, vp, vp, vp, vp, d, d, vp, vp]
    L.ss_spawn_splats.argtypes = [ctypes.POINTER(SsCamera), vp, vp, vp, vp, vp, i32, d, d, d, vp, vp, vp, vp, vp, vp]
    L.ss_prune_workspace_bytes.argtypes = [i32]
    L.ss_prune_workspace_bytes.restype = ctypes.c_size_t
    L.ss_prune_flags.argtypes = [i32, vp, d, ctypes.POINTER(i32), vp, vp]
    L.ss_prune_compact.argtypes = [i32, i32, vp, vp, vp, vp]
    for name in ("ss_spawn_weights", "ss_densify_mask", "ss_spawn_splats", "ss_prune_flags", "ss_prune_compact"):
        getattr(L, name).restype = ctypes.c_int
    L.ss_reg_solve_workspace_bytes.argtypes = [i32, i32, i32]
    L.ss_reg_solve_workspace_bytes.restype = ctypes.c_size_t
    L.ss_reg_solve.argtypes = [vp, vp, i32, vp, i32, vp, i32, vp, vp, ctypes.POINTER(SsCamera), vp,
                               ctypes.POINTER(SsRegSolveCfg), vp, vp, vp, vp, vp]
    L.ss_reg_solve.restype = ctypes.c_int
    L.ss_reg_solve_async.argtypes = [vp, vp, i32, vp, i32, vp, i32, vp, vp, ctypes.POINTER(SsCamera), vp,
                                     ctypes.POINTER(SsRegSolveCfg), i32, vp, vp, vp]
    L.ss_reg_solve_async.restype = ctypes.c_int
    L.ss_register_photo_batch.argtypes = [i32, ctypes.POINTER(SsCamera), ctypes.POINTER(SsCamera),
                                          ctypes.POINTER(SsSplats), ctypes.POINTER(SsRasterCfg), vp, vp, vp, vp, vp,
                                          i32, d, d, ctypes.POINTER(SsRegSolveCfg), i32, vp, vp, vp, vp, i32, vp,
                                          ctypes.c_size_t, vp, ctypes.c_size_t, vp]
    L.ss_register_photo_batch.restype = ctypes.c_int
    for name in ("ss_records_work", "ss_records_profile", "ss_records_stage_times", "ss_render_forward", "ss_records_counts", "ss_records_export", "ss_render_backward",
                 "ss_mapping_loss", "ss_photo_system"):
        getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


EXPORTED = ["ss_version", "ss_records_create", "ss_records_destroy", "ss_render_forward", "ss_records_counts",
            "ss_records_export", "ss_records_pixel_state", "ss_records_check", "ss_records_work", "ss_records_profile", "ss_records_stage_times", "ss_fp32_peak_tflops", "ss_host_stage_f64",
            "ss_render_backward", "ss_mapping_loss", "ss_photo_workspace_bytes",
            "ss_photo_system", "ss_anchor_workspace_bytes", "ss_reg_anchors", "ss_range_image", "ss_scale_loss",
            "ss_adam_step", "ss_reg_solve_workspace_bytes", "ss_reg_solve",
            "ss_smooth_range_image", "ss_range_image_normals", "ss_leaf_tree_workspace_bytes", "ss_leaf_tree_build",
            "ss_records_set_deterministic", "ss_spawn_weights", "ss_densify_mask", "ss_spawn_splats",
            "ss_prune_workspace_bytes", "ss_prune_flags", "ss_prune_compact", "ss_adam_step_dev", "ss_render_finalize_adam_dev",
            "ss_store_loss_parts", "ss_records_sticky_overflow", "ss_records_reserve", "ss_records_generation",
            "ss_render_backward_blend", "ss_render_finalize", "ss_reg_solve_async",
            "ss_register_photo_batch"]


def check(status: int, what: str = "") -> None:
    """Map a C-ABI status onto the reference's exception classes (errors.py)."""
    from .errors import GeometryError, RegistrationError
    if status == SS_OK:
        return
    if status == SS_ERR_REGISTRATION:
        raise RegistrationError(f"{what}: too few residuals survive association")
    msg = {SS_ERR_INVALID_ARGUMENT: "invalid argument", SS_ERR_STALE_RECORDS: "blend records are stale for this model",
           SS_ERR_UNSUPPORTED: "unsupported configuration", SS_ERR_CUDA: "CUDA error",
           SS_ERR_CAPACITY: "pair capacity exceeded", SS_ERR_DEGENERATE: "degenerate raw tangents"}.get(status, "error")
    if status in (SS_ERR_CUDA, SS_ERR_CAPACITY):
        raise RuntimeError(f"{what}: {msg} (status {status})")
    raise GeometryError(f"{what}: {msg}")
