"""Device geometric registration half vs the live reference (golden_register_geo.npz).

The leaf tree is built level-parallel with Jacobi eigenvectors: the partition of
the model points into leaves must agree with the reference's except for single
median points of odd-sized splits (whose side depends on the sign LAPACK gives
the principal axis)."""
import os

import numpy as np
import pytest
import torch

from paper_2503_17491_b200 import registration as REG

pytestmark = pytest.mark.gpu

D = os.path.join(os.path.dirname(__file__), "golden")
G = np.load(os.path.join(D, "golden_register.npz"))
GG = np.load(os.path.join(D, "golden_register_geo.npz"))


def _match_leaves(ours, ref_point_leaf, ref_sizes):
    """Fraction of points whose leaf (as a point set) differs from the reference's."""
    n = ref_point_leaf.shape[0]
    # map every reference leaf to the device leaf holding most of its points
    pairs = ref_point_leaf.astype(np.int64) * (ours.max() + 1) + ours
    uniq, cnt = np.unique(pairs, return_counts=True)
    best = {}
    for u, c in zip(uniq, cnt):
        r, o = divmod(int(u), int(ours.max() + 1))
        if c > best.get(r, (0, -1))[0]:
            best[r] = (c, o)
    agree = sum(c for c, _ in best.values())
    return 1.0 - agree / n


def test_leaf_tree_matches_reference(cuda):
    tree = REG.build_leaf_tree(GG["model_pts"], G["initial_t"])
    print("leaves", tree.sizes.shape[0], "ref", GG["leaf_sizes"].shape[0], "usable", int(tree.usable.sum()))
    moved = _match_leaves(tree.point_leaf, GG["point_leaf"], GG["leaf_sizes"])
    print("points in a different leaf:", moved)
    assert abs(tree.sizes.shape[0] - GG["leaf_sizes"].shape[0]) <= max(2, 0.02 * GG["leaf_sizes"].shape[0])
    assert moved <= 0.01
    # every usable reference leaf has a device leaf with nearly the same centroid and plane
    ref_c, ref_n = GG["leaf_centroids"][GG["leaf_usable"]], GG["leaf_normals"][GG["leaf_usable"]]
    c, nn = tree.centroids[tree.usable], tree.normals[tree.usable]
    d = np.linalg.norm(ref_c[:, None, :] - c[None, :, :], axis=-1)
    j = d.argmin(axis=1)
    dist = d[np.arange(len(ref_c)), j]
    cosang = np.abs(np.sum(ref_n * nn[j], axis=1))
    print("centroid offset: median", np.median(dist), "max", dist.max(), "worst normal angle (deg)",
          np.degrees(np.arccos(np.clip(cosang.min(), -1, 1))))
    assert np.mean(dist < 0.05) >= 0.95 and np.mean(cosang > np.cos(np.deg2rad(2.0))) >= 0.95


@pytest.mark.parametrize("mode,iters", [("geometric", 15), ("joint", 15), ("sequential", 30)])
def test_register_modes_vs_reference(cuda, mode, iters):
    from paper_2503_17491_b200 import SE3Pose, SphericalCamera, SplatModel
    c = G["cam"]
    cam = SphericalCamera(int(c[0]), int(c[1]), *[float(x) for x in c[2:]])
    params = {k[2:]: G[k].astype(np.float64) for k in G.files if k.startswith("p_")}
    res = REG.register(SplatModel.from_params(params), G["scan"].astype(np.float64), cam,
                       SE3Pose(G["initial_R"], G["initial_t"]), REG.RegistrationConfig(mode=mode, max_iters=iters))
    dt = np.abs(res.pose.translation - GG[f"{mode}_t"]).max()
    dR = np.abs(res.pose.rotation - GG[f"{mode}_R"]).max()
    print(mode, "dt", dt, "dR", dR, "iters", res.iterations, int(GG[f"{mode}_iterations"]), "n_geo", res.n_geo,
          int(GG[f"{mode}_n_geo"]), "n_photo", res.n_photo, int(GG[f"{mode}_n_photo"]), "geo_rms", res.geo_rms,
          float(GG[f"{mode}_geo_rms"]))
    # The photometric anchors come from the float32 render, where a handful of pixels near the
    # O > 0.5 threshold differ from the reference's float64 one (test_gpu_registration); the
    # joint problem of this scene is ill-conditioned (the reference itself ends 3.7 cm from the
    # truth after 15 iterations) and amplifies that into a different iterate path.  With the
    # reference's own inputs every mode matches to 1e-16 (test below).
    tol = {"geometric": 1e-6, "sequential": 1e-6, "joint": 2e-2}[mode]
    assert dt <= tol and dR <= tol
    assert res.converged == bool(GG[f"{mode}_converged"])
    if mode != "joint":
        assert res.iterations == int(GG[f"{mode}_iterations"]) and res.n_geo == int(GG[f"{mode}_n_geo"])


@pytest.mark.parametrize("mode,iters", [("geometric", 15), ("joint", 15), ("sequential", 30)])
def test_device_loop_matches_reference_on_reference_inputs(cuda, mode, iters):
    """Same model points, anchors and scan subsample as the reference: the device loop
    reproduces the reference's iterations and pose (isolates the loop from the render)."""
    from paper_2503_17491_b200 import SE3Pose, SphericalCamera
    c = G["cam"]
    cam = SphericalCamera(int(c[0]), int(c[1]), *[float(x) for x in c[2:]])
    tree = REG.build_leaf_tree(GG["model_pts"], G["initial_t"])
    scan = REG.DeviceScan(cam, G["scan"].astype(np.float64))
    geo_scan = torch.as_tensor(G["scan"].astype(np.float64)[GG["geo_sel"]], device="cuda")
    X = torch.as_tensor(G["X_w"], device="cuda")
    cfg = REG.RegistrationConfig(mode=mode, max_iters=iters)
    res = REG.solve_device(cfg, SE3Pose(G["initial_R"], G["initial_t"]), scan, X if mode != "geometric" else None,
                           tree, geo_scan)
    dt = np.abs(res.pose.translation - GG[f"{mode}_t"]).max()
    print(mode, "same-inputs dt", dt, "iters", res.iterations, int(GG[f"{mode}_iterations"]), res.n_geo, res.n_photo)
    assert res.iterations == int(GG[f"{mode}_iterations"]) and res.converged == bool(GG[f"{mode}_converged"])
    assert res.n_geo == int(GG[f"{mode}_n_geo"]) and res.n_photo == int(GG[f"{mode}_n_photo"])
    assert dt <= 1e-7 and np.abs(res.pose.rotation - GG[f"{mode}_R"]).max() <= 1e-7


class _Leaves:
    """The oracle's usable leaves in the device layout solve_device reads."""

    def __init__(self, t):
        self.dev_centroids = torch.as_tensor(np.ascontiguousarray(t.c[t.usable]), device="cuda")
        self.dev_normals = torch.as_tensor(np.ascontiguousarray(t.n[t.usable]), device="cuda")


@pytest.mark.parametrize("gate,k", [(0.12, 3), (0.4, 1), (0.4, 5), (2.5, 8), (1e4, 3), (-0.4, 3)])
def test_association_gate_and_k_vs_oracle(cuda, gate, k):
    """The hashed-grid association (cells of edge |assoc_gate|) against the oracle's
    cKDTree query with distance_upper_bound, over gates from a few leaves per query to
    one cell holding every leaf, and k from 1 to the device maximum of 8."""
    from oracle import geo_registration_oracle as GO
    from paper_2503_17491_b200 import SE3Pose, SphericalCamera
    c = G["cam"]
    cam = SphericalCamera(int(c[0]), int(c[1]), *[float(x) for x in c[2:]])
    ot = GO.Tree(GG["model_pts"], G["initial_t"])
    scan_np = G["scan"].astype(np.float64)[GG["geo_sel"]]
    R, t, it, conv, grms, _, ng, _ = GO.register("geometric", ot, scan_np, None, None, None, None, G["initial_R"],
                                                 G["initial_t"], max_iters=6, gate=gate, k=k)
    cfg = REG.RegistrationConfig(mode="geometric", max_iters=6, assoc_gate=gate, assoc_k=k)
    res = REG.solve_device(cfg, SE3Pose(G["initial_R"], G["initial_t"]), REG.DeviceScan(cam, G["scan"].astype(np.float64)),
                           None, _Leaves(ot), torch.as_tensor(scan_np, device="cuda"))
    print(gate, k, "iters", res.iterations, it, "n_geo", res.n_geo, ng, "dt", np.abs(res.pose.translation - t).max())
    assert res.iterations == it and res.converged == conv and res.n_geo == ng
    assert np.abs(res.pose.translation - t).max() <= 1e-9 and np.abs(res.pose.rotation - R).max() <= 1e-9
    assert abs(res.geo_rms - grms) <= 1e-9


def test_leaf_tree_deterministic(cuda):
    """Two builds of the same cloud give bit-identical leaves (cooperative top levels
    sum block partials in a fixed order)."""
    a = REG.build_leaf_tree(GG["model_pts"], G["initial_t"])
    b = REG.build_leaf_tree(GG["model_pts"], G["initial_t"])
    assert np.array_equal(a.centroids, b.centroids) and np.array_equal(a.normals, b.normals)
    assert np.array_equal(a.sizes, b.sizes) and np.array_equal(a.point_leaf, b.point_leaf)


def _cloud(kind, n, rng):
    if kind == "random":
        return rng.normal(size=(n, 3)) * [5.0, 3.0, 1.0]
    if kind == "plane":
        p = rng.uniform(-5, 5, size=(n, 3))
        p[:, 2] = 0.3 * p[:, 0] - 0.1 * p[:, 1] + 1.0
        return p
    if kind == "line":
        t = rng.uniform(-5, 5, size=(n, 1))
        return np.hstack([t, 2 * t, -t]) + 1.0
    if kind == "duplicates":
        return np.repeat(rng.normal(size=(max(n // 50, 1), 3)), 50, axis=0)[:n]
    raise ValueError(kind)


@pytest.mark.parametrize("kind,n", [("random", 1), ("random", 2), ("random", 3), ("random", 65), ("random", 3000),
                                    ("random", 40000), ("plane", 5000), ("line", 5000), ("duplicates", 6000)])
def test_leaf_tree_edge_clouds_vs_oracle(cuda, kind, n):
    """Degenerate and tiny clouds through both the cooperative top levels and the per-node
    levels: the same leaves (sizes, usability, centroids) as the oracle's recursion."""
    from oracle import geo_registration_oracle as GO
    rng = np.random.default_rng(n)
    pts = _cloud(kind, n, rng)
    vp = np.array([0.5, -0.25, 2.0])
    c, nn, sizes, usable, pl = GO.build_leaf_tree(pts, vp)
    tree = REG.build_leaf_tree(pts, vp)
    assert tree.sizes.shape[0] == sizes.shape[0]
    assert np.array_equal(np.sort(tree.sizes), np.sort(sizes))
    assert int(tree.usable.sum()) == int(usable.sum())
    # leaf order differs (level order vs the reference's stack order): match by point sets
    for leaf in range(sizes.shape[0]):
        members = np.flatnonzero(pl == leaf)
        ours = np.unique(tree.point_leaf[members])
        assert ours.shape[0] == 1, (leaf, ours)
        o = int(ours[0])
        assert tree.sizes[o] == sizes[leaf] and bool(tree.usable[o]) == bool(usable[leaf])
        assert np.abs(tree.centroids[o] - c[leaf]).max() <= 1e-9 * max(1.0, np.abs(c[leaf]).max())
        if usable[leaf]:
            assert abs(abs(np.dot(tree.normals[o], nn[leaf])) - 1.0) <= 1e-9
