"""Pin the CPU oracle (oracle/) against golden vectors of the live reference.

CPU only.  The fixtures were produced by tests/golden/make_golden.py from the
reference package itself; the oracle must reproduce its tile lists bit for bit
and its float64 images/gradients to round-off.
"""
import numpy as np
import pytest

from golden import CASES, load
from oracle import oracle as O


@pytest.fixture(scope="module", params=CASES)
def case(request):
    g = load(request.param)
    cfg = O.OracleCfg(tile_size=int(g["tile_size"]))
    r = O.render(g["cam_tuple"], g["R"], g["t"], g["params"], cfg)
    return g, cfg, r


def test_intrinsics(case):
    g, _, _ = case
    k = O.intrinsics(g["cam_tuple"])
    assert np.array_equal(k[:4], [g["fx"], g["fy"], g["cx"], g["cy"]])
    assert np.array_equal(k[4:], g["grid_offset"])
    if g["dirs"].size:
        assert np.abs(O.pixel_planes(g["cam_tuple"])[0] - g["dirs"]).max() < 1e-15


def test_tile_lists_bit_exact(case):
    g, _, r = case
    assert r["tiles_x"] == int(g["tiles_x"]) and r["tiles_y"] == int(g["tiles_y"])
    assert np.array_equal(r["tile_ptr"], g["tile_ptr"])
    assert np.array_equal(r["pair_splats"], g["pair_splats"])


def test_images(case):
    g, _, r = case
    for k in ("range", "normal", "opacity"):
        assert np.abs(r[k] - g[k]).max() <= 1e-11 * max(1.0, np.abs(g[k]).max()), k
    if g["brute_range"].size:  # the reference's own brute-force renderer agrees too
        assert np.abs(g["brute_range"] - g["range"]).max() < 1e-10


def test_backward_plain_and_raw(case):
    g, cfg, r = case
    pl = O.backward_lists(g["cam_tuple"], r["arr"], g["R"], r["tile_ptr"], r["pair_splats"], r["range"],
                          r["normal"], r["opacity"], g["gD"], g["gN"], g["gO"], cfg)
    scale = np.abs(g["plain"]).max(axis=0) + 1e-30
    assert (np.abs(pl - g["plain"]).max(axis=0) / scale).max() < 1e-10
    raw = O.raw_gradients(g["params"], pl)
    scale = np.abs(g["raw"]).max(axis=0) + 1e-30
    assert (np.abs(raw - g["raw"]).max(axis=0) / scale).max() < 1e-10


def test_oracle_gradients_match_finite_differences():
    """The restated backward is the derivative of the restated forward (raw space)."""
    g = load("full")
    cam, R, t = g["cam_tuple"], g["R"], g["t"]
    params = {k: v[:60].copy() for k, v in g["params"].items()}
    rng = np.random.default_rng(3)
    H, W = cam[1], cam[0]
    gD, gN, gO = rng.normal(size=(H, W)), 0.1 * rng.normal(size=(H, W, 3)), 0.05 * rng.normal(size=(H, W))

    def loss(p):
        r = O.render(cam, R, t, p)
        return float((gD * r["range"]).sum() + (gN * r["normal"]).sum() + (gO * r["opacity"]).sum()), r

    L0, r = loss(params)
    pl = O.backward_lists(cam, r["arr"], R, r["tile_ptr"], r["pair_splats"], r["range"], r["normal"], r["opacity"],
                          gD, gN, gO)
    raw = O.raw_gradients(params, pl)
    cols = {"centers": (0, 3), "raw_t_alpha": (3, 6), "raw_t_beta": (6, 9), "log_scales": (9, 11),
            "logit_opacity": (11, 12)}
    h = 1e-6
    checked = 0
    for name, (a, b) in cols.items():
        for i in rng.choice(60, 6, replace=False):
            for c in range(b - a):
                if abs(raw[i, a + c]) < 1e-6:
                    continue
                p1 = {k: v.copy() for k, v in params.items()}
                p2 = {k: v.copy() for k, v in params.items()}
                if name == "logit_opacity":
                    p1[name][i] += h; p2[name][i] -= h
                else:
                    p1[name][i, c] += h; p2[name][i, c] -= h
                fd = (loss(p1)[0] - loss(p2)[0]) / (2 * h)
                assert abs(fd - raw[i, a + c]) <= 1e-4 * max(1.0, abs(raw[i, a + c])), (name, i, c, fd, raw[i, a + c])
                checked += 1
    assert checked > 20
