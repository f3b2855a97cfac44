"""Spherical camera and SE(3) pose used by the drop-in API.

Mirrors the reference's ``SphericalCamera`` (geometry.py:68-185) and
``SE3Pose`` (se3.py:74-157) closely enough that reference objects and these
are interchangeable at the API boundary (same attribute names and formulas).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from functools import cached_property

import numpy as np

from .errors import GeometryError


def _py_mod(a, b):
    return np.mod(a, b)


@dataclass(eq=False)
class SphericalCamera:
    """W x H spherical grid over [az_min, az_max] x [el_min, el_max] (geometry.py:68-115)."""

    width: int
    height: int
    az_min: float
    az_max: float
    el_min: float
    el_max: float

    def __post_init__(self):
        if self.width < 2 or self.height < 2:
            raise GeometryError("image must be at least 2 x 2")
        if not (self.az_max > self.az_min and self.el_max > self.el_min):
            raise GeometryError("angular bounds must have positive extent")

    @property
    def fx(self) -> float:
        return -(self.width - 1) / (self.az_max - self.az_min)

    @property
    def fy(self) -> float:
        return -(self.height - 1) / (self.el_max - self.el_min)

    @property
    def cx(self) -> float:
        return 0.5 * self.width * (1.0 + (self.az_max + self.az_min) / (self.az_max - self.az_min))

    @property
    def cy(self) -> float:
        return 0.5 * self.height * (1.0 + (self.el_max + self.el_min) / (self.el_max - self.el_min))

    @property
    def full_circle(self) -> bool:
        fov = self.az_max - self.az_min
        pitch = fov / (self.width - 1)
        return fov + pitch >= 2.0 * np.pi - 0.5 * pitch

    @property
    def grid_offset(self) -> np.ndarray:
        first = np.array([self.fx * self.az_max + self.cx, self.fy * self.el_max + self.cy])
        return _py_mod(first + 0.5, 1.0) - 0.5

    def angles_of(self, uv):
        uv = np.asarray(uv, dtype=float)
        return (uv[..., 0] - self.cx) / self.fx, (uv[..., 1] - self.cy) / self.fy

    def project(self, points) -> np.ndarray:
        p = np.asarray(points, dtype=float)
        az = np.arctan2(p[..., 1], p[..., 0])
        el = np.arctan2(p[..., 2], np.hypot(p[..., 0], p[..., 1]))
        return np.stack([self.fx * az + self.cx, self.fy * el + self.cy], axis=-1)

    def back_project(self, uv, ranges) -> np.ndarray:
        az, el = self.angles_of(uv)
        ce = np.cos(el)
        d = np.stack([ce * np.cos(az), ce * np.sin(az), np.sin(el)], axis=-1)
        return np.asarray(ranges, dtype=float)[..., None] * d

    @cached_property
    def sample_grid(self) -> np.ndarray:
        uu, vv = np.meshgrid(np.arange(self.width, dtype=float), np.arange(self.height, dtype=float))
        return np.stack([uu, vv], axis=-1) + self.grid_offset

    @cached_property
    def pixel_directions(self) -> np.ndarray:
        az, el = self.angles_of(self.sample_grid)
        ce = np.cos(el)
        return np.stack([ce * np.cos(az), ce * np.sin(az), np.sin(el)], axis=-1)


def skew(v) -> np.ndarray:
    x, y, z = v
    return np.array([[0.0, -z, y], [z, 0.0, -x], [-y, x, 0.0]])


def so3_exp(phi) -> np.ndarray:
    """Rodrigues (se3.py:29-39)."""
    phi = np.asarray(phi, dtype=float)
    a = float(np.linalg.norm(phi))
    K = skew(phi)
    if a < 1e-8:
        return np.eye(3) + K + 0.5 * (K @ K)
    return np.eye(3) + (np.sin(a) / a) * K + ((1.0 - np.cos(a)) / (a * a)) * (K @ K)


def _left_jacobian(phi) -> np.ndarray:
    a = float(np.linalg.norm(phi))
    K = skew(phi)
    if a < 1e-8:
        return np.eye(3) + 0.5 * K + (K @ K) / 6.0
    return np.eye(3) + ((1.0 - np.cos(a)) / (a * a)) * K + ((a - np.sin(a)) / (a ** 3)) * (K @ K)


@dataclass
class SE3Pose:
    """Sensor-in-world pose, p_w = R p_s + t, right updates (se3.py:3-7, 74-141)."""

    rotation: np.ndarray = field(default_factory=lambda: np.eye(3))
    translation: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def __post_init__(self):
        self.rotation = np.asarray(self.rotation, dtype=float).reshape(3, 3)
        self.translation = np.asarray(self.translation, dtype=float).reshape(3)

    @classmethod
    def identity(cls) -> "SE3Pose":
        return cls()

    def compose(self, other) -> "SE3Pose":
        return SE3Pose(self.rotation @ other.rotation, self.rotation @ other.translation + self.translation)

    def inverse(self) -> "SE3Pose":
        Rt = self.rotation.T
        return SE3Pose(Rt, -Rt @ self.translation)

    def apply(self, points) -> np.ndarray:
        return np.asarray(points, dtype=float) @ self.rotation.T + self.translation

    def retract(self, delta) -> "SE3Pose":
        return self.compose(se3_exp(delta))

    def orthonormalized(self) -> "SE3Pose":
        U, _, Vt = np.linalg.svd(self.rotation)
        R = U @ Vt
        if np.linalg.det(R) < 0:
            U[:, -1] = -U[:, -1]
            R = U @ Vt
        return SE3Pose(R, self.translation.copy())

    def copy(self) -> "SE3Pose":
        return SE3Pose(self.rotation.copy(), self.translation.copy())


def se3_exp(delta) -> SE3Pose:
    """Twist (rho, phi) -> pose (se3.py:144-150)."""
    d = np.asarray(delta, dtype=float).reshape(6)
    return SE3Pose(so3_exp(d[3:]), _left_jacobian(d[3:]) @ d[:3])


def pose_rt(pose) -> np.ndarray:
    """Row-major R then t as 12 float64 (the C-ABI pose layout)."""
    return np.ascontiguousarray(np.concatenate([np.asarray(pose.rotation, float).reshape(9),
                                                np.asarray(pose.translation, float).reshape(3)]))
