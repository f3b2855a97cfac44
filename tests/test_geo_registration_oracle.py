"""Pin the numpy oracle of the geometric registration half against the live reference
(tests/golden/golden_register_geo.npz, made by tests/golden/make_golden.py geometric)."""
import os

import numpy as np
import pytest

from oracle import geo_registration_oracle as GO

D = os.path.join(os.path.dirname(__file__), "golden")
G = np.load(os.path.join(D, "golden_register.npz"))
GG = np.load(os.path.join(D, "golden_register_geo.npz"))
CAM = tuple([int(G["cam"][0]), int(G["cam"][1])] + [float(x) for x in G["cam"][2:]])


@pytest.fixture(scope="module")
def tree():
    return GO.Tree(GG["model_pts"], G["initial_t"])


def test_leaf_tree_identical(tree):
    assert np.array_equal(tree.point_leaf, GG["point_leaf"])
    assert np.array_equal(tree.sizes, GG["leaf_sizes"]) and np.array_equal(tree.usable, GG["leaf_usable"])
    assert np.abs(tree.c - GG["leaf_centroids"]).max() <= 1e-12
    assert np.abs(tree.n - GG["leaf_normals"]).max() <= 1e-12


def test_geo_system(tree):
    scan = G["scan"].astype(np.float64)[GG["geo_sel"]]
    r, J = GO.geo_system(tree, scan, G["T0_R"], G["T0_t"], 0.5)
    assert r.shape[0] == int(GG["geo_m0"])
    assert np.abs(r - GG["geo_r0"]).max() <= 1e-12
    w = GO.RO.huber_w(r, 0.1)
    assert np.abs((J.T * w) @ J - GG["geo_H0"]).max() <= 1e-12 * np.abs(GG["geo_H0"]).max()
    assert np.abs(J.T @ (w * r) - GG["geo_b0"]).max() <= 1e-12 * np.abs(GG["geo_b0"]).max()


@pytest.mark.parametrize("mode,iters", [("geometric", 15), ("joint", 15), ("sequential", 30)])
def test_register_modes(tree, mode, iters):
    scan = G["scan"].astype(np.float64)[GG["geo_sel"]]
    R, t, it, conv, grms, prms, ng, nph = GO.register(mode, tree, scan, G["X_w"], G["scan_range"], G["scan_valid"],
                                                      CAM, G["initial_R"], G["initial_t"], max_iters=iters)
    assert it == int(GG[f"{mode}_iterations"]) and conv == bool(GG[f"{mode}_converged"])
    assert ng == int(GG[f"{mode}_n_geo"]) and nph == int(GG[f"{mode}_n_photo"])
    assert np.abs(t - GG[f"{mode}_t"]).max() < 1e-9 and np.abs(R - GG[f"{mode}_R"]).max() < 1e-9
    assert abs(grms - float(GG[f"{mode}_geo_rms"])) < 1e-9 and abs(prms - float(GG[f"{mode}_photo_rms"])) < 1e-9
