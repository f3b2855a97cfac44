"""Keyframe preparation on the device (reference: pkg/src/splatscan/geometry.py:198-338,
mapping.py:97-114).

Drop-ins with the reference's names and return types:

* ``build_range_image(cam, points) -> RangeImage``      geometry.py:252-268
* ``smooth_range_image(rimg, wrap, size=3) -> RangeImage`` geometry.py:271-287
* ``range_image_normals(cam, rimg) -> NormalImage``      geometry.py:290-338
* ``estimate_camera(points, width, height)``             geometry.py:198-215 (host)
* ``make_keyframe(index, cloud, pose, width, height) -> Keyframe``  mapping.py:106-114

Each runs the sm_100a kernels of libsplatb200.so (``ss_range_image``,
``ss_smooth_range_image``, ``ss_range_image_normals``); the host only
estimates the camera (four angular extremes) and converts the results back to
numpy for reference consumers.  ``keyframe_images`` is the device-resident
path: cloud tensor in, target images as device tensors out, no host sync, which
``mapping.DeviceKeyframe.from_cloud`` uses.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import engine
from ._lib import check, lib
from .errors import GeometryError
from .geometry import SE3Pose, SphericalCamera

__all__ = ["RangeImage", "NormalImage", "Keyframe", "build_range_image", "smooth_range_image",
           "range_image_normals", "estimate_camera", "keyframe_images", "make_keyframe"]

_MIN_RANGE = 1e-9  # geometry.py:49


@dataclass
class RangeImage:
    """geometry.py:218-233."""
    range: np.ndarray
    valid: np.ndarray

    def __post_init__(self):
        self.range = np.asarray(self.range, dtype=float)
        self.valid = np.asarray(self.valid, dtype=bool)
        if self.range.shape != self.valid.shape or self.range.ndim != 2:
            raise GeometryError("range and valid must be matching H x W arrays")

    @property
    def shape(self):
        return self.range.shape


@dataclass
class NormalImage:
    """geometry.py:236-249."""
    normals: np.ndarray
    valid: np.ndarray

    def __post_init__(self):
        self.normals = np.asarray(self.normals, dtype=float)
        self.valid = np.asarray(self.valid, dtype=bool)
        if self.normals.ndim != 3 or self.normals.shape[2] != 3:
            raise GeometryError("normals must be H x W x 3")
        if self.normals.shape[:2] != self.valid.shape:
            raise GeometryError("normals and valid shapes disagree")


@dataclass
class Keyframe:
    """mapping.py:96-103."""
    index: int
    cloud: np.ndarray
    pose: SE3Pose
    camera: SphericalCamera
    range_image: RangeImage
    normal_image: NormalImage


def estimate_camera(points, width: int, height: int) -> SphericalCamera:
    """geometry.py:198-215: bounds are the cloud's angular extremes (host, float64)."""
    p = np.asarray(points, dtype=float).reshape(-1, 3)
    p = p[np.linalg.norm(p, axis=1) > _MIN_RANGE]
    if p.shape[0] == 0:
        raise GeometryError("no usable points for camera estimation")
    az = np.arctan2(p[:, 1], p[:, 0])
    el = np.arctan2(p[:, 2], np.hypot(p[:, 0], p[:, 1]))
    az_min, az_max = float(az.min()), float(az.max())
    el_min, el_max = float(el.min()), float(el.max())
    if az_max - az_min < 1e-12 or el_max - el_min < 1e-12:
        raise GeometryError("cloud has zero angular extent")
    return SphericalCamera(width, height, az_min, az_max, el_min, el_max)


def _dev_points(points) -> torch.Tensor:
    dev = engine.require_cuda()
    if torch.is_tensor(points):
        return points.to(dev, torch.float64).reshape(-1, 3).contiguous()
    return torch.as_tensor(np.ascontiguousarray(np.asarray(points, dtype=np.float64).reshape(-1, 3)), device=dev)


def _range_dev(cam, pts: torch.Tensor):
    dev = pts.device
    rng = torch.empty((cam.height, cam.width), dtype=torch.float64, device=dev)
    val = torch.empty((cam.height, cam.width), dtype=torch.uint8, device=dev)
    c = engine.ss_camera(cam)
    check(lib().ss_range_image(ctypes.byref(c), ctypes.c_void_p(pts.data_ptr() if pts.numel() else 0),
                               int(pts.shape[0]), ctypes.c_void_p(rng.data_ptr()), ctypes.c_void_p(val.data_ptr()),
                               ctypes.c_void_p(engine.stream_ptr())), "build_range_image")
    return rng, val


def _smooth_dev(rng: torch.Tensor, val: torch.Tensor, wrap: bool) -> torch.Tensor:
    H, W = rng.shape
    out = torch.empty_like(rng)
    check(lib().ss_smooth_range_image(W, H, int(bool(wrap)), ctypes.c_void_p(rng.data_ptr()),
                                      ctypes.c_void_p(val.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                      ctypes.c_void_p(engine.stream_ptr())), "smooth_range_image")
    return out


def _normals_dev(cam, rng: torch.Tensor, val: torch.Tensor):
    H, W = rng.shape
    if (H, W) != (cam.height, cam.width):
        raise GeometryError("range image and camera disagree")
    nrm = torch.empty((H, W, 3), dtype=torch.float64, device=rng.device)
    ok = torch.empty((H, W), dtype=torch.uint8, device=rng.device)
    c = engine.ss_camera(cam)
    check(lib().ss_range_image_normals(ctypes.byref(c), ctypes.c_void_p(rng.data_ptr()),
                                       ctypes.c_void_p(val.data_ptr()), ctypes.c_void_p(nrm.data_ptr()),
                                       ctypes.c_void_p(ok.data_ptr()), ctypes.c_void_p(engine.stream_ptr())),
          "range_image_normals")
    return nrm, ok


def _img_dev(rimg: RangeImage):
    dev = engine.require_cuda()
    rng = torch.as_tensor(np.ascontiguousarray(rimg.range, dtype=np.float64), device=dev)
    val = torch.as_tensor(np.ascontiguousarray(rimg.valid, dtype=np.uint8), device=dev)
    return rng, val


def build_range_image(cam, points) -> RangeImage:
    """geometry.py:252-268 on the device."""
    rng, val = _range_dev(cam, _dev_points(points))
    return RangeImage(rng.cpu().numpy(), val.cpu().numpy().astype(bool))


def smooth_range_image(rimg: RangeImage, wrap: bool = False, size: int = 3) -> RangeImage:
    """geometry.py:271-287 on the device (the 3x3 window of make_keyframe)."""
    if size != 3:
        raise GeometryError("the device smoothing implements size=3 (make_keyframe's window) only")
    rng, val = _img_dev(rimg)
    out = _smooth_dev(rng, val, wrap)
    return RangeImage(out.cpu().numpy(), rimg.valid.copy())


def range_image_normals(cam, rimg: RangeImage) -> NormalImage:
    """geometry.py:290-338 on the device."""
    rng, val = _img_dev(rimg)
    nrm, ok = _normals_dev(cam, rng, val)
    return NormalImage(nrm.cpu().numpy(), ok.cpu().numpy().astype(bool))


def keyframe_images(cam, cloud) -> dict:
    """Device path of make_keyframe's images: {range, valid, normal, nvalid} device tensors
    (float64 / uint8), stream-ordered, no host synchronisation."""
    rng, val = _range_dev(cam, _dev_points(cloud))
    nrm, ok = _normals_dev(cam, _smooth_dev(rng, val, cam.full_circle), val)
    return {"range": rng, "valid": val, "normal": nrm, "nvalid": ok}


def make_keyframe(index: int, cloud, pose, width: int, height: int) -> Keyframe:
    """mapping.py:106-114: camera from the cloud, range image, normals of the smoothed ranges."""
    cloud = np.asarray(cloud, dtype=float)
    cam = estimate_camera(cloud, width, height)
    im = keyframe_images(cam, cloud)
    return Keyframe(index, cloud, pose.copy(), cam,
                    RangeImage(im["range"].cpu().numpy(), im["valid"].cpu().numpy().astype(bool)),
                    NormalImage(im["normal"].cpu().numpy(), im["nvalid"].cpu().numpy().astype(bool)))
