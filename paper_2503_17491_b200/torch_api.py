"""Differentiable torch entry point (the north-star ``render`` API).

``render(splats, pose, camera)`` -> (range, normal, opacity) float32 images,
differentiable w.r.t. the raw parameters of the splats (centres, raw tangent
pair, log scales, logit opacity).  The backward pass is the fused sm_100a
backward + finalize kernel in raw space: it equals the reference's
``rasterize_backward`` (rasterizer.py:534-701) chained through
``tangent_raw_gradients`` (splats.py:133-163) and the activation derivatives
of ``refine`` (mapping.py:479-494).
"""
from __future__ import annotations

import numpy as np
import torch

from . import engine
from .geometry import pose_rt
from .rasterizer import RasterConfig


class _Render(torch.autograd.Function):
    @staticmethod
    def forward(ctx, centers, raw_t_alpha, raw_t_beta, log_scales, logit_opacity, pose12, cam, cfg):
        splats = {"centers": centers.detach().contiguous(), "raw_t_alpha": raw_t_alpha.detach().contiguous(),
                  "raw_t_beta": raw_t_beta.detach().contiguous(), "log_scales": log_scales.detach().contiguous(),
                  "logit_opacity": logit_opacity.detach().contiguous()}
        rec = engine.Records.acquire()
        D, N, O = engine.forward(cam, pose12, splats, cfg, rec)
        ctx.rec = rec
        ctx.splats = splats
        ctx.mark_non_differentiable()
        return D, N, O

    @staticmethod
    def backward(ctx, gD, gN, gO):
        H, W = gD.shape if gD is not None else gO.shape
        dev = ctx.splats["centers"].device
        z = lambda *s: torch.zeros(s, dtype=torch.float32, device=dev)  # noqa: E731
        gD = gD if gD is not None else z(H, W)
        gN = gN if gN is not None else z(H, W, 3)
        gO = gO if gO is not None else z(H, W)
        g = engine.backward(ctx.rec, ctx.splats, gD, gN, gO, raw_space=True)
        ctx.rec.release()
        ctx.rec = None
        return (g[:, 0:3], g[:, 3:6], g[:, 6:9], g[:, 9:11], g[:, 11], None, None, None)


def render(splats: dict, pose, camera, cfg: RasterConfig | None = None):
    """Render a splat set; ``splats`` maps the raw parameter names to float32 CUDA tensors.

    ``pose``: SE3Pose-like (rotation, translation) sensor-in-world, or a 12-vector [R row-major, t].
    Returns (range [H,W], normal [H,W,3], opacity [H,W]).
    """
    cfg = cfg or RasterConfig()
    p12 = np.asarray(pose, dtype=np.float64).reshape(12) if not hasattr(pose, "rotation") else pose_rt(pose)
    return _Render.apply(splats["centers"], splats["raw_t_alpha"], splats["raw_t_beta"], splats["log_scales"],
                         splats["logit_opacity"], p12, camera, cfg)
