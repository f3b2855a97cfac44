"""Pin the numpy registration oracle against the live reference's golden outputs (CPU)."""
import numpy as np
import pytest

from oracle import registration_oracle as RO

G = np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "golden_register.npz"))
CAM = tuple([int(G["cam"][0]), int(G["cam"][1])] + [float(x) for x in G["cam"][2:]])
PARAMS = {k[2:]: G[k].astype(np.float64) for k in G.files if k.startswith("p_")}


def test_sample_model_anchors():
    geo = (CAM[0] * 2, CAM[1] * 2) + CAM[2:]
    pts = RO.sample_model(PARAMS, geo, G["initial_R"], G["initial_t"])
    assert pts.shape[0] == int(G["n_model_pts"])
    assert np.abs(pts[::4] - G["X_w"]).max() < 1e-12


def test_range_image_exact():
    img, valid = RO.build_range_image(CAM, G["scan"].astype(np.float64))
    assert np.array_equal(valid, G["scan_valid"])
    assert np.array_equal(img, G["scan_range"])


def test_photo_system():
    r, J = RO.photo_system(G["X_w"], G["scan_range"], G["scan_valid"], CAM, G["T0_R"], G["T0_t"], 0.5)
    assert r.shape[0] == int(G["m0"])
    w = RO.huber_w(r, 0.2)
    H = (J.T * w) @ J
    b = J.T @ (w * r)
    assert np.abs(H - G["H0"]).max() <= 1e-12 * np.abs(G["H0"]).max()
    assert np.abs(b - G["b0"]).max() <= 1e-12 * np.abs(G["b0"]).max()
    assert abs(RO.huber_v(r, 0.2) - float(G["huber0"])) <= 1e-12 * abs(float(G["huber0"]))


def test_register_photometric_final_pose():
    R, t, it, conv, rms, m, _ = RO.register_photometric(G["X_w"], G["scan_range"], G["scan_valid"], CAM,
                                                        G["initial_R"], G["initial_t"], max_iters=15)
    assert np.abs(t - G["final_t"]).max() < 1e-9
    assert np.abs(R - G["final_R"]).max() < 1e-9
    assert it == int(G["iterations"]) and conv == bool(G["converged"]) and m == int(G["n_photo"])
    assert abs(rms - float(G["photo_rms"])) < 1e-9
