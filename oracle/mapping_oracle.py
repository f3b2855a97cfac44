"""CPU restatement (numpy, float64) of the reference's mapping objective and optimiser.

TEST INFRASTRUCTURE ONLY (see oracle.c): the parity checker of the device
loss / Adam kernels and the CPU baseline of the mapping step; never imported
by the product package.

Restates pkg/src/splatscan/mapping.py:
  :128-137  range_loss     range-weighted L1 over the keyframe's valid mask
  :140-151  normal_loss    1 - n.N where range and normal are valid
  :154-163  opacity_loss   -log max(O, eps) over valid pixels
  :166-178  scale_loss     hinge on the larger scale above the cap
  :181-196  mapping_loss   weighted total, pixel gradients, scale gradient
  :342-379  _Adam.step     per-group learning rates, bias correction
  :474-497  refine         one iteration: render, loss, backward, raw chain, Adam, clamp
"""
from __future__ import annotations

import numpy as np

from . import oracle as O

PARAM_W = (("centers", 3), ("raw_t_alpha", 3), ("raw_t_beta", 3), ("log_scales", 2), ("logit_opacity", 1))


def range_loss(D, kf_range, kf_valid, floor=1.0):
    M = kf_valid
    w = 1.0 / np.maximum(kf_range, floor)
    diff = D - kf_range
    return float(np.sum(w[M] * np.abs(diff[M]))), np.where(M, w * np.sign(diff), 0.0)


def normal_loss(N, kf_valid, kf_normal, kf_nvalid):
    M = kf_valid & kf_nvalid
    dots = np.sum(N * kf_normal, axis=-1)
    return float(np.sum(1.0 - dots[M])), np.where(M[..., None], -kf_normal, 0.0)


def opacity_loss(Op, kf_valid, eps=1e-6):
    M = kf_valid
    clamped = np.maximum(Op, eps)
    return float(np.sum(-np.log(clamped[M]))), np.where(M & (Op > eps), -1.0 / clamped, 0.0)


def scale_loss(log_scales, cap):
    s = np.exp(np.asarray(log_scales, dtype=np.float64))
    if s.shape[0] == 0:
        return 0.0, np.zeros((0, 2))
    mx = s.max(axis=1)
    over = mx - cap
    g = np.zeros_like(s)
    hot = over > 0
    arg = s.argmax(axis=1)
    g[hot, arg[hot]] = 1.0
    return float(np.sum(np.maximum(over, 0.0))), g


def mapping_loss(D, N, Op, kf, log_scales, cfg):
    """kf: dict(range, valid, normal, nvalid) host arrays.  Returns
    (total, gD, gN, gO, d_scales, parts{range, opacity, normal, scale})."""
    L_d, g_d = range_loss(D, kf["range"], kf["valid"], cfg.range_weight_floor)
    L_o, g_o = opacity_loss(Op, kf["valid"])
    L_n, g_n = normal_loss(N, kf["valid"], kf["normal"], kf["nvalid"])
    L_s, g_s = scale_loss(log_scales, cfg.scale_cap)
    total = L_d + cfg.w_opacity * L_o + cfg.w_normal * L_n + cfg.w_scale * L_s
    parts = {"range": L_d, "opacity": L_o, "normal": L_n, "scale": L_s}
    return total, g_d, cfg.w_normal * g_n, cfg.w_opacity * g_o, cfg.w_scale * g_s, parts


def flat(params) -> np.ndarray:
    n = len(params["centers"])
    return np.concatenate([np.asarray(params[k], dtype=np.float64).reshape(n, -1) for k, _ in PARAM_W], axis=1)


def unflat(x) -> dict:
    out, c = {}, 0
    for k, w in PARAM_W:
        out[k] = x[:, c:c + w] if w > 1 else x[:, c]
        c += w
    return out


class Adam:
    """_Adam.step (mapping.py:367-379) on the flattened (n, 12) layout, then the log-scale
    clamp of refine (mapping.py:496)."""

    def __init__(self, n, cfg, scene_scale=1.0):
        self.m = np.zeros((n, 12))
        self.v = np.zeros((n, 12))
        self.t = 0
        self.lr = np.array([cfg.lr_centers * scene_scale] * 3 + [cfg.lr_tangents] * 6 + [cfg.lr_log_scales] * 2 +
                           [cfg.lr_logit_opacity])
        self.lo, self.hi = np.log(cfg.scale_floor), np.log(10.0 * cfg.scale_cap)

    def step(self, x, g):
        self.t += 1
        self.m = 0.9 * self.m + 0.1 * g
        self.v = 0.999 * self.v + 0.001 * g * g
        x -= self.lr * (self.m / (1 - 0.9 ** self.t)) / (np.sqrt(self.v / (1 - 0.999 ** self.t)) + 1e-8)
        np.clip(x[:, 9:11], self.lo, self.hi, out=x[:, 9:11])


def refine_iteration(x, opt: Adam, cam, R, t, kf, cfg, max_threads: int = 64):
    """One refine iteration (mapping.py:474-497) on the flattened float64 parameters ``x``
    (updated in place) with the C oracle's render and backward.  Returns the loss total."""
    p = unflat(x)
    r = O.render(cam, R, t, p)
    total, gD, gN, gO, gS, _ = mapping_loss(r["range"], r["normal"], r["opacity"], kf, p["log_scales"], cfg)
    plain = O.backward_lists(cam, r["arr"], R, r["tile_ptr"], r["pair_splats"], r["range"], r["normal"],
                             r["opacity"], gD, gN, gO, max_threads=max_threads)
    g = O.raw_gradients(p, plain, gS)
    opt.step(x, g)
    return total
