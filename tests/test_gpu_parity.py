"""GPU parity of the sm_100a path against the oracle and the golden fixtures.

Gates (BASELINE.json north_star):
  * tile_ptr / pair_splats bit-exact;
  * range/normal/opacity within 1e-4 relative per pixel for pixels farther
    than 1e-5 from any discrete threshold (flagged pixels counted), and
    within 1e-4 norm-wise per channel;
  * gradients within 1e-3 norm-wise per parameter class, and per splat on
    >= 99.5 % of splats with non-negligible gradient.
"""
import numpy as np
import pytest
import torch

from golden import CASES, load
from oracle import oracle as O
from parity import RAW_CLASSES, assert_grads, assert_images, grad_report, image_report
from paper_2503_17491_b200 import (PixelGradients, RasterConfig, SE3Pose, SplatModel, SphericalCamera,
                                   rasterize_backward, rasterize_forward)
from paper_2503_17491_b200 import torch_api
from paper_2503_17491_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _cam(t):
    return SphericalCamera(*t)


@pytest.fixture(scope="module", params=CASES)
def gcase(request, cuda):
    g = load(request.param)
    cam = _cam(g["cam_tuple"])
    pose = SE3Pose(g["R"], g["t"])
    model = SplatModel.from_params(g["params"])
    cfg = RasterConfig(tile_size=int(g["tile_size"]))
    out, rec = rasterize_forward(cam, pose, model, cfg)
    torch.cuda.synchronize()
    ocfg = O.OracleCfg(tile_size=cfg.tile_size)
    ref = O.render(g["cam_tuple"], g["R"], g["t"], g["params"], ocfg, margins=True)
    return g, cam, pose, model, cfg, out, rec, ref


def test_golden_tile_lists_bit_exact(gcase):
    g, cam, pose, model, cfg, out, rec, ref = gcase
    assert (rec.tiles_x, rec.tiles_y) == (int(g["tiles_x"]), int(g["tiles_y"]))
    assert np.array_equal(rec.tile_ptr, g["tile_ptr"])
    assert np.array_equal(rec.pair_splats, g["pair_splats"])


def test_golden_images(gcase):
    g, cam, pose, model, cfg, out, rec, ref = gcase
    rep = image_report({"range": out.range, "normal": out.normal, "opacity": out.opacity},
                       {"range": g["range"], "normal": g["normal"], "opacity": g["opacity"]}, ref["margin"])
    assert_images(rep)


def test_golden_backward_plain(gcase):
    g, cam, pose, model, cfg, out, rec, ref = gcase
    sg = rasterize_backward(model, rec, out, PixelGradients(g["gD"], g["gN"], g["gO"]))
    got = np.concatenate([sg.d_centers, sg.d_t_alpha, sg.d_t_beta, sg.d_normal, sg.d_scales, sg.d_opacity[:, None]],
                         axis=1)
    assert_grads(grad_report(got, g["plain"]))


def test_golden_torch_api_raw_gradients(gcase):
    g, cam, pose, model, cfg, out, rec, ref = gcase
    dev = torch.device("cuda")
    p = {k: torch.tensor(np.asarray(v, np.float32), device=dev, requires_grad=True) for k, v in g["params"].items()}
    D, N, Op = torch_api.render(p, pose, cam, cfg)
    loss = (D * torch.tensor(g["gD"], dtype=torch.float32, device=dev)).sum() + \
        (N * torch.tensor(g["gN"], dtype=torch.float32, device=dev)).sum() + \
        (Op * torch.tensor(g["gO"], dtype=torch.float32, device=dev)).sum()
    loss.backward()
    got = torch.cat([p["centers"].grad, p["raw_t_alpha"].grad, p["raw_t_beta"].grad, p["log_scales"].grad,
                     p["logit_opacity"].grad[:, None]], dim=1).cpu().numpy()
    assert_grads(grad_report(got, g["raw"], RAW_CLASSES), RAW_CLASSES)


def test_empty_and_invisible_models(cuda):
    cam = W.synth_camera(128, 32)
    out, rec = rasterize_forward(cam, SE3Pose.identity(), SplatModel())
    assert rec.pair_splats.shape == (0,) and np.all(out.range == 0)
    # one splat far outside the vertical field of view: no pairs, zero images and gradients
    m = SplatModel(np.array([[0.0, 0.0, 40.0]]), log_scales=np.full((1, 2), np.log(0.05)))
    out, rec = rasterize_forward(cam, SE3Pose.identity(), m)
    assert rec.pair_splats.shape == (0,) and np.all(out.opacity == 0)
    sg = rasterize_backward(m, rec, out, PixelGradients(np.ones((32, 128)), np.ones((32, 128, 3)), np.ones((32, 128))))
    assert np.all(sg.d_centers == 0)


def _config0_loss_grads(out, tgt):
    """range_loss + 0.1 normal_loss pixel gradients (mapping.py:128-151), float64 host."""
    M = tgt["valid"]
    w = 1.0 / np.maximum(tgt["range"].astype(np.float64), 1.0)
    gD = np.where(M, w * np.sign(out["range"] - tgt["range"]), 0.0)
    Mn = M & tgt["nvalid"]
    gN = np.where(Mn[..., None], -0.1 * tgt["normal"].astype(np.float64), 0.0)
    return gD, gN, np.zeros_like(gD)


@pytest.mark.parametrize("index", [0, 1])
def test_config_full_size_parity(cuda, index):
    """BASELINE configs 0 (64x1024, 50k splats) and 1 (the headline 128x2048, 500k splats)
    against the float64 C oracle (all host threads; ~2 s per config-1 render on the box)."""
    c = W.config(index)
    cam, params = c["camera"], c["splats"]
    ct = (cam.width, cam.height, cam.az_min, cam.az_max, cam.el_min, cam.el_max)
    R, t = np.eye(3), np.zeros(3)
    ref = O.render(ct, R, t, params, margins=True)
    model = SplatModel.from_params(params)
    out, rec = rasterize_forward(cam, SE3Pose.identity(), model)
    assert np.array_equal(rec.tile_ptr, ref["tile_ptr"])
    assert np.array_equal(rec.pair_splats, ref["pair_splats"])
    rep = image_report({"range": out.range, "normal": out.normal, "opacity": out.opacity}, ref, ref["margin"])
    print("image parity", rep)
    assert_images(rep)
    tgt = W.target_images(W.Scene(0), cam)
    gD, gN, gO = _config0_loss_grads(ref, tgt)
    sg = rasterize_backward(model, rec, out, PixelGradients(gD, gN, gO))
    got = np.concatenate([sg.d_centers, sg.d_t_alpha, sg.d_t_beta, sg.d_normal, sg.d_scales, sg.d_opacity[:, None]],
                         axis=1)
    plain = O.backward_lists(ct, ref["arr"], R, ref["tile_ptr"], ref["pair_splats"], ref["range"], ref["normal"],
                             ref["opacity"], gD, gN, gO)
    rep = grad_report(got, plain)
    print("grad parity", rep)
    assert_grads(rep)


def _crowded_params(n: int, n_tie: int, seed: int) -> dict:
    """Splats crowded into a narrow cone ahead of the sensor (tile lists of thousands, past the
    8-warp and 32-warp shared-memory sorts) plus a block of splats at exactly one range (runs of
    equal sort keys longer than the insertion-sort limit)."""
    rng = np.random.default_rng(seed)
    az = rng.uniform(-0.15, 0.15, n)
    el = rng.uniform(-0.1, 0.1, n)
    r = rng.uniform(4.0, 12.0, n)
    r[:n_tie] = 7.0
    d = np.stack([np.cos(el) * np.cos(az), np.cos(el) * np.sin(az), np.sin(el)], 1)
    c = d * r[:, None]
    ta, tb = W.quat_tangents(rng.normal(size=(n, 4)))
    ls = rng.normal(np.log(0.25), 0.3, (n, 2))
    lo = rng.normal(0.0, 1.0, n)
    f = lambda a: np.ascontiguousarray(a, dtype=np.float32)  # noqa: E731
    return {"centers": f(c), "raw_t_alpha": f(ta), "raw_t_beta": f(tb), "log_scales": f(ls), "logit_opacity": f(lo)}


@pytest.mark.parametrize("n,n_tie", [(6000, 0), (30000, 400)])
def test_long_lists_and_tie_runs_bit_exact(cuda, n, n_tie):
    cam = W.synth_camera(512, 64)
    params = _crowded_params(n, n_tie, 3)
    ct = (cam.width, cam.height, cam.az_min, cam.az_max, cam.el_min, cam.el_max)
    ref = O.render(ct, np.eye(3), np.zeros(3), params)
    out, rec = rasterize_forward(cam, SE3Pose.identity(), SplatModel.from_params(params))
    lens = np.diff(ref["tile_ptr"])
    print("max list", lens.max(), "lists > 2048:", int((lens > 2048).sum()), "> 8192:", int((lens > 8192).sum()))
    assert lens.max() > 2048
    assert np.array_equal(rec.tile_ptr, ref["tile_ptr"])
    assert np.array_equal(rec.pair_splats, ref["pair_splats"])
    rep = image_report({"range": out.range, "normal": out.normal, "opacity": out.opacity}, ref,
                       np.full(out.range.shape, 1.0))
    assert rep["range_norm"] < 1e-4 and rep["opacity_norm"] < 1e-4, rep


def test_many_tiles_with_tail_lists(cuda):
    """4,096 tiles (more than resident warps) with a crowded cone: lists of >= 1,536
    entries go to the block-per-tile forward alongside the warp kernel; tile lists
    bit-exact and images within the 1e-4 protocol."""
    cam = W.synth_camera(2048, 128)
    params = _crowded_params(40000, 0, 7)
    ct = (cam.width, cam.height, cam.az_min, cam.az_max, cam.el_min, cam.el_max)
    ref = O.render(ct, np.eye(3), np.zeros(3), params)
    out, rec = rasterize_forward(cam, SE3Pose.identity(), SplatModel.from_params(params))
    lens = np.diff(ref["tile_ptr"])
    print("tiles", lens.shape[0], "max list", lens.max(), "lists >= 1536:", int((lens >= 1536).sum()))
    assert lens.shape[0] == 4096 and int((lens >= 1536).sum()) > 0
    assert np.array_equal(rec.tile_ptr, ref["tile_ptr"])
    assert np.array_equal(rec.pair_splats, ref["pair_splats"])
    rep = image_report({"range": out.range, "normal": out.normal, "opacity": out.opacity}, ref,
                       np.full(out.range.shape, 1.0))
    assert rep["range_norm"] < 1e-4 and rep["opacity_norm"] < 1e-4, rep
    # backward over the same records (warp-per-tile slots; the block kernel's contribution words)
    rng = np.random.default_rng(11)
    gD = rng.normal(size=(cam.height, cam.width))
    gN = 0.1 * rng.normal(size=(cam.height, cam.width, 3))
    gO = 0.05 * rng.normal(size=(cam.height, cam.width))
    model = SplatModel.from_params(params)
    sg = rasterize_backward(model, rec, out, PixelGradients(gD, gN, gO))
    got = np.concatenate([sg.d_centers, sg.d_t_alpha, sg.d_t_beta, sg.d_normal, sg.d_scales, sg.d_opacity[:, None]],
                         axis=1)
    plain = O.backward_lists(ct, ref["arr"], np.eye(3), ref["tile_ptr"], ref["pair_splats"], ref["range"],
                             ref["normal"], ref["opacity"], gD, gN, gO)
    rep = grad_report(got, plain)
    print("tail-list grad parity", rep)
    assert_grads(rep)


def test_tie_runs_in_shared_memory_sized_lists_bit_exact(cuda):
    """Lists short enough for the 8-warp shared-memory sort but holding a run of equal
    ranges longer than its insertion limit: the block merge-sorts that tile in place."""
    cam = W.synth_camera(512, 64)
    params = _crowded_params(1600, 300, 5)
    ct = (cam.width, cam.height, cam.az_min, cam.az_max, cam.el_min, cam.el_max)
    ref = O.render(ct, np.eye(3), np.zeros(3), params)
    out, rec = rasterize_forward(cam, SE3Pose.identity(), SplatModel.from_params(params))
    lens = np.diff(ref["tile_ptr"])
    print("max list", lens.max())
    assert 64 < lens.max() <= 2048
    assert np.array_equal(rec.tile_ptr, ref["tile_ptr"])
    assert np.array_equal(rec.pair_splats, ref["pair_splats"])


@pytest.mark.parametrize("group", [12, 40, 90])
def test_medium_tie_runs_bit_exact(cuda, group):
    """Groups of splats at one range (and exact duplicates of a centre): per tile, runs of equal
    16-bit sort keys of roughly the group's size -- one thread's insertion sort (<= 8), the
    warp ranking (9-64) and the block bitonic sort (> 64) -- all put in the reference's
    (range, index) order."""
    params = _crowded_params(4000, 0, 13)
    rng = np.random.default_rng(group)
    c = params["centers"].astype(np.float64)
    d = c / np.linalg.norm(c, axis=1, keepdims=True)
    ng = 1200 // group
    for g in range(ng):
        sl = slice(g * group, (g + 1) * group)
        c[sl] = d[sl] * rng.uniform(4.0, 12.0)
    c[1200:1260] = c[1200]  # exact duplicates: equal float64 ranges, ordered by index
    params["centers"] = np.ascontiguousarray(c, dtype=np.float32)
    cam = W.synth_camera(512, 64)
    ct = (cam.width, cam.height, cam.az_min, cam.az_max, cam.el_min, cam.el_max)
    ref = O.render(ct, np.eye(3), np.zeros(3), params)
    _, rec = rasterize_forward(cam, SE3Pose.identity(), SplatModel.from_params(params))
    assert np.array_equal(rec.tile_ptr, ref["tile_ptr"])
    assert np.array_equal(rec.pair_splats, ref["pair_splats"])


def test_deterministic_backward_bit_identical(cuda):
    """RasterConfig(deterministic=True): fixed-order reduction, bit-identical gradients run to run,
    within the 1e-3 gate of the oracle; the default (atomic) path agrees to float rounding."""
    c = W.config(0)
    cam, params = c["camera"], c["splats"]
    model = SplatModel.from_params(params)
    rng = np.random.default_rng(3)
    gD = rng.normal(size=(cam.height, cam.width))
    gN = 0.1 * rng.normal(size=(cam.height, cam.width, 3))
    gO = 0.05 * rng.normal(size=(cam.height, cam.width))
    runs = []
    for det in (True, True, False):
        out, rec = rasterize_forward(cam, SE3Pose.identity(), model, RasterConfig(deterministic=det))
        sg = rasterize_backward(model, rec, out, PixelGradients(gD, gN, gO))
        runs.append(np.concatenate([sg.d_centers, sg.d_t_alpha, sg.d_t_beta, sg.d_normal, sg.d_scales,
                                    sg.d_opacity[:, None]], axis=1))
    assert np.array_equal(runs[0], runs[1])
    ref = np.linalg.norm(runs[2])
    assert np.linalg.norm(runs[0] - runs[2]) <= 1e-5 * ref
    ct = (cam.width, cam.height, cam.az_min, cam.az_max, cam.el_min, cam.el_max)
    o = O.render(ct, np.eye(3), np.zeros(3), params)
    plain = O.backward_lists(ct, o["arr"], np.eye(3), o["tile_ptr"], o["pair_splats"], o["range"], o["normal"],
                             o["opacity"], gD, gN, gO)
    assert_grads(grad_report(runs[0], plain))


def test_backward_twice_same_records(cuda):
    """Two backward passes over one forward (different pixel gradients) are independent:
    the device accumulators are cleared by each pass (rasterizer.py:534 allows repeated calls)."""
    c = W.config(0)
    cam, model = c["camera"], SplatModel.from_params(c["splats"])
    out, rec = rasterize_forward(cam, SE3Pose.identity(), model)
    rng = np.random.default_rng(5)
    g1 = PixelGradients(rng.normal(size=(cam.height, cam.width)), np.zeros((cam.height, cam.width, 3)),
                        np.zeros((cam.height, cam.width)))
    g2 = PixelGradients(np.zeros((cam.height, cam.width)), np.zeros((cam.height, cam.width, 3)),
                        rng.normal(size=(cam.height, cam.width)))
    a = rasterize_backward(model, rec, out, g1).d_centers
    b = rasterize_backward(model, rec, out, g2).d_centers
    a2 = rasterize_backward(model, rec, out, g1).d_centers
    assert np.abs(a2 - a).max() <= 1e-6 * np.abs(a).max()
    assert np.abs(b).max() > 0 and not np.allclose(a, b)


def test_pair_capacity_overflow_rerun(cuda):
    """A few huge splats near the sensor cover every tile: more (tile, splat) pairs than the
    speculative capacity (max(8 n, 65536)), so the first forward overflows on the device and
    rasterize_forward transparently re-runs with the exact capacity (ss_records_check)."""
    rng = np.random.default_rng(8)
    n = 120
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    params = {"centers": (d * rng.uniform(1.0, 3.0, (n, 1))).astype(np.float32),
              "raw_t_alpha": rng.normal(size=(n, 3)).astype(np.float32),
              "raw_t_beta": rng.normal(size=(n, 3)).astype(np.float32),
              "log_scales": np.full((n, 2), np.log(1.5), np.float32),
              "logit_opacity": rng.normal(size=n).astype(np.float32)}
    cam = W.synth_camera(1024, 64)
    ct = (cam.width, cam.height, cam.az_min, cam.az_max, cam.el_min, cam.el_max)
    ref = O.render(ct, np.eye(3), np.zeros(3), params)
    assert ref["pair_splats"].shape[0] > 65536
    out, rec = rasterize_forward(cam, SE3Pose.identity(), SplatModel.from_params(params))
    assert np.array_equal(rec.tile_ptr, ref["tile_ptr"]) and np.array_equal(rec.pair_splats, ref["pair_splats"])
    rep = image_report({"range": out.range, "normal": out.normal, "opacity": out.opacity}, ref,
                       np.full(out.range.shape, 1.0))
    assert rep["range_norm"] < 1e-4 and rep["opacity_norm"] < 1e-4, rep


def test_cuda_graph_capture_replay(cuda):
    """The forward / loss / backward sequence is stream-ordered with no host synchronisation,
    so it captures into a CUDA graph; replays match eager execution (float-atomic rounding)."""
    from paper_2503_17491_b200 import engine
    c = W.config(0)
    cam = c["camera"]
    sp = {k: torch.from_numpy(v).cuda() for k, v in c["splats"].items()}
    tgt = W.target_images(W.Scene(0), cam)
    kr, kn = torch.from_numpy(tgt["range"]).cuda(), torch.from_numpy(tgt["normal"]).cuda()
    kv = torch.from_numpy(tgt["valid"].astype(np.uint8)).cuda()
    knv = torch.from_numpy(tgt["nvalid"].astype(np.uint8)).cuda()
    rec, cfg = engine.Records(), RasterConfig()
    pose = np.concatenate([np.eye(3).reshape(9), np.zeros(3)])

    def step():
        D, N, O = engine.forward(cam, pose, sp, cfg, rec, sync=False)
        dD, dN, dO, parts = engine.mapping_loss(D, N, O, kr, kv, kn, knv, 0.0, 0.1)
        return engine.backward(rec, sp, dD, dN, dO, raw_space=True)

    engine.forward(cam, pose, sp, cfg, rec)  # sizes the pair buffers
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2):
            eager = step()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    eager = eager.clone()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        out = step()
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    assert rec.check(True) == 0
    assert torch.allclose(out, eager, rtol=1e-4, atol=1e-6 * float(eager.abs().max()))


def test_config2_long_lists_parity(cuda):
    """BASELINE config 2 (64x1024 keyframe of the 200k-surfel local map: lists up to ~3,900
    entries, fewer tiles than resident warps): exercises the block-per-tile forward for the
    longest lists and the pixel-half backward slots; tile lists bit-exact, images and
    gradients against the oracle under the same gates as configs 0/1."""
    params, kfs, _ = W.config2_map()
    cam, pose, tgt = kfs[-1]
    p64 = {k: np.asarray(v, np.float64) for k, v in params.items()}
    ct = (cam.width, cam.height, cam.az_min, cam.az_max, cam.el_min, cam.el_max)
    ref = O.render(ct, pose.rotation, pose.translation, p64, margins=True)
    assert np.diff(ref["tile_ptr"]).max() > 768
    model = SplatModel.from_params(params)
    out, rec = rasterize_forward(cam, pose, model)
    assert np.array_equal(rec.tile_ptr, ref["tile_ptr"])
    assert np.array_equal(rec.pair_splats, ref["pair_splats"])
    rep = image_report({"range": out.range, "normal": out.normal, "opacity": out.opacity}, ref, ref["margin"])
    print("config2 image parity", rep)
    assert_images(rep)
    gD, gN, gO = _config0_loss_grads(ref, tgt)
    sg = rasterize_backward(model, rec, out, PixelGradients(gD, gN, gO))
    got = np.concatenate([sg.d_centers, sg.d_t_alpha, sg.d_t_beta, sg.d_normal, sg.d_scales, sg.d_opacity[:, None]],
                         axis=1)
    plain = O.backward_lists(ct, ref["arr"], pose.rotation, ref["tile_ptr"], ref["pair_splats"], ref["range"],
                             ref["normal"], ref["opacity"], gD, gN, gO)
    rep = grad_report(got, plain)
    print("config2 grad parity", rep)
    assert_grads(rep)


def test_segment_forward_with_early_cutoffs(cuda):
    """Few tiles (512x64: 512 tiles < resident warps, so the segment-parallel forward runs)
    with long lists of nearly opaque splats: most pixels reach the transmittance cut-off in
    some middle segment, so every pass of the segment forward is exercised (partial blends,
    the combine that finds the cut-off segment, the sequential re-blend of that segment).
    Images under the 1e-4 protocol with the oracle's threshold margins, gradients under the
    1e-3 gates, and the cut-off pixels' final transmittance below min_T as in the oracle."""
    import ctypes

    import torch

    from paper_2503_17491_b200 import engine
    from paper_2503_17491_b200._lib import lib

    cam = W.synth_camera(512, 64)
    params = _crowded_params(20000, 0, 5)
    params["logit_opacity"] = np.full_like(params["logit_opacity"], 3.0)  # opacity ~0.95
    p64 = {k: np.asarray(v, np.float64) for k, v in params.items()}
    ct = (cam.width, cam.height, cam.az_min, cam.az_max, cam.el_min, cam.el_max)
    ref = O.render(ct, np.eye(3), np.zeros(3), p64, margins=True)
    lens = np.diff(ref["tile_ptr"])
    assert lens.max() > 4 * 128  # several 128-entry segments per list
    model = SplatModel.from_params(params)
    out, rec = rasterize_forward(cam, SE3Pose.identity(), model)
    assert np.array_equal(rec.tile_ptr, ref["tile_ptr"])
    assert np.array_equal(rec.pair_splats, ref["pair_splats"])
    rep = image_report({"range": out.range, "normal": out.normal, "opacity": out.opacity}, ref, ref["margin"])
    print("segment-forward image parity", rep)
    assert_images(rep)
    P = cam.width * cam.height
    T = torch.empty(P, dtype=torch.float32, device="cuda")
    last = torch.empty(P, dtype=torch.int32, device="cuda")
    assert lib().ss_records_pixel_state(rec._handle.ptr, ctypes.c_void_p(T.data_ptr()), ctypes.c_void_p(last.data_ptr()),
                                        ctypes.c_void_p(engine.stream_ptr())) == 0
    torch.cuda.synchronize()
    T = T.cpu().numpy().reshape(cam.height, cam.width)
    last = last.cpu().numpy().reshape(cam.height, cam.width)
    covered = last > 0  # (the crowded cone covers a small part of the full-circle image)
    cut = (T < 1e-4) & covered
    deep = (last[cut] > 128).mean() if cut.any() else 0.0
    print("covered pixels past the cut-off", cut.sum() / covered.sum(), "of which beyond the first segment", deep)
    assert cut.sum() > 0.3 * covered.sum() and deep > 0.05
    rng = np.random.default_rng(4)
    gD = rng.normal(size=(cam.height, cam.width))
    gN = 0.1 * rng.normal(size=(cam.height, cam.width, 3))
    gO = 0.05 * rng.normal(size=(cam.height, cam.width))
    sg = rasterize_backward(model, rec, out, PixelGradients(gD, gN, gO))
    got = np.concatenate([sg.d_centers, sg.d_t_alpha, sg.d_t_beta, sg.d_normal, sg.d_scales, sg.d_opacity[:, None]],
                         axis=1)
    plain = O.backward_lists(ct, ref["arr"], np.eye(3), ref["tile_ptr"], ref["pair_splats"], ref["range"],
                             ref["normal"], ref["opacity"], gD, gN, gO)
    grep = grad_report(got, plain)
    print("segment-forward grad parity", grep)
    assert_grads(grep)
