"""Splat model storage used by the drop-in API (splats.py:166-279 of the reference).

Same raw parameterisation: centers, raw tangent pair, log scales, logit
opacity, epochs and a ``version`` counter bumped on mutation so that stale
blend records are detected (rasterizer.py:546-547).
"""
from __future__ import annotations

import numpy as np

from .errors import GeometryError


def _sigmoid(x):
    x = np.asarray(x, dtype=float)
    e = np.exp(-np.abs(x))
    return np.where(x >= 0, 1.0 / (1.0 + e), e / (1.0 + e))


class SplatModel:
    def __init__(self, centers=None, raw_t_alpha=None, raw_t_beta=None, log_scales=None, logit_opacity=None,
                 epochs=None):
        self.centers = np.array(centers if centers is not None else np.zeros((0, 3)), dtype=float).reshape(-1, 3)
        n = self.centers.shape[0]
        self.raw_t_alpha = np.array(raw_t_alpha if raw_t_alpha is not None else np.tile([1.0, 0, 0], (n, 1)),
                                    dtype=float).reshape(-1, 3)
        self.raw_t_beta = np.array(raw_t_beta if raw_t_beta is not None else np.tile([0.0, 1, 0], (n, 1)),
                                   dtype=float).reshape(-1, 3)
        self.log_scales = np.array(log_scales if log_scales is not None else np.zeros((n, 2)), dtype=float).reshape(-1, 2)
        self.logit_opacity = np.array(logit_opacity if logit_opacity is not None else np.zeros(n),
                                      dtype=float).reshape(-1)
        self.epochs = np.array(epochs if epochs is not None else np.zeros(n, dtype=int)).reshape(-1).astype(int)
        if {a.shape[0] for a in (self.raw_t_alpha, self.raw_t_beta, self.log_scales, self.logit_opacity,
                                 self.epochs)} != {n}:
            raise GeometryError("splat arrays have inconsistent lengths")
        self.version = 0

    def __len__(self) -> int:
        return self.centers.shape[0]

    @property
    def scales(self) -> np.ndarray:
        return np.exp(self.log_scales)

    @property
    def opacities(self) -> np.ndarray:
        return _sigmoid(self.logit_opacity)

    def touch(self) -> None:
        self.version += 1

    @classmethod
    def from_params(cls, params: dict) -> "SplatModel":
        return cls(params["centers"], params["raw_t_alpha"], params["raw_t_beta"], params["log_scales"],
                   params["logit_opacity"])
