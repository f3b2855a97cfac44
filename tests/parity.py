"""Parity gates of SURVEY.md 7.3 (images) and 7.3 item 4 (gradients)."""
import numpy as np

IMG_REL = 1e-4      # BASELINE: depth, normal, alpha within 1e-4 relative
GRAD_REL = 1e-3     # BASELINE: gradients within 1e-3 relative
MARGIN = 1e-5       # pixels closer than this to a discrete threshold are flagged, not gated


def image_report(gpu: dict, ref: dict, margin: np.ndarray) -> dict:
    """Strict per-pixel 1e-4 check on pixels with threshold margin > 1e-5; norm-wise 1e-4 per channel.

    Normals are compared as vectors against max(|n_ref|, O_ref)."""
    safe = margin > MARGIN
    out = {"flagged": int((~safe).sum()), "pixels": int(margin.size)}
    for k in ("range", "opacity"):
        a, b = gpu[k].astype(np.float64), ref[k]
        err = np.abs(a - b)
        scale = np.maximum(np.abs(b), 1e-6)
        bad = (err > IMG_REL * scale) & safe
        out[f"{k}_bad"] = int(bad.sum())
        out[f"{k}_norm"] = float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))
        out[f"{k}_max_rel_safe"] = float((err / scale)[safe].max()) if safe.any() else 0.0
    a, b = gpu["normal"].astype(np.float64), ref["normal"]
    err = np.linalg.norm(a - b, axis=-1)
    scale = np.maximum(np.maximum(np.linalg.norm(b, axis=-1), ref["opacity"]), 1e-6)
    out["normal_bad"] = int(((err > IMG_REL * scale) & safe).sum())
    out["normal_norm"] = float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))
    return out


def assert_images(rep: dict, max_flagged_frac: float = 1e-3):
    for k in ("range", "opacity", "normal"):
        assert rep[f"{k}_bad"] == 0, rep
        assert rep[f"{k}_norm"] <= IMG_REL, rep
    assert rep["flagged"] <= max(3, max_flagged_frac * rep["pixels"]), rep


CLASSES = {"d_centers": slice(0, 3), "d_t_alpha": slice(3, 6), "d_t_beta": slice(6, 9), "d_normal": slice(9, 12),
           "d_scales": slice(12, 14), "d_opacity": slice(14, 15)}
RAW_CLASSES = {"centers": slice(0, 3), "raw_t_alpha": slice(3, 6), "raw_t_beta": slice(6, 9),
               "log_scales": slice(9, 11), "logit_opacity": slice(11, 12)}


def grad_report(gpu: np.ndarray, ref: np.ndarray, classes=CLASSES) -> dict:
    out = {}
    for name, sl in classes.items():
        a, b = gpu[:, sl].astype(np.float64), ref[:, sl]
        nb = np.linalg.norm(b)
        out[f"{name}_norm"] = float(np.linalg.norm(a - b) / max(nb, 1e-30))
        pn = np.linalg.norm(b, axis=1)
        sig = pn > 1e-3 * max(pn.max(), 1e-30)
        rel = np.linalg.norm(a - b, axis=1)[sig] / pn[sig]
        out[f"{name}_splat_ok_frac"] = float((rel <= GRAD_REL).mean()) if sig.any() else 1.0
        out[f"{name}_splat_max"] = float(rel.max()) if sig.any() else 0.0
    return out


def assert_grads(rep: dict, classes=CLASSES, min_ok_frac: float = 0.995):
    for name in classes:
        assert rep[f"{name}_norm"] <= GRAD_REL, rep
        assert rep[f"{name}_splat_ok_frac"] >= min_ok_frac, rep
