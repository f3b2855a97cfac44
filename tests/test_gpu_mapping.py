"""Device refine loop (mapping.py:455-498) vs the reference's golden run, and the
fused Adam / scale-hinge kernels vs their numpy restatement."""
import os

import numpy as np
import pytest
import torch

from paper_2503_17491_b200 import SE3Pose, SphericalCamera, engine
from paper_2503_17491_b200 import mapping as MP

pytestmark = pytest.mark.gpu
G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_refine.npz"))
NAMES = ("centers", "raw_t_alpha", "raw_t_beta", "log_scales", "logit_opacity")


def test_adam_kernel_matches_numpy(cuda):
    rng = np.random.default_rng(0)
    n = 1000
    params = {"centers": rng.normal(size=(n, 3)), "raw_t_alpha": rng.normal(size=(n, 3)),
              "raw_t_beta": rng.normal(size=(n, 3)), "log_scales": rng.normal(-3, 0.5, size=(n, 2)),
              "logit_opacity": rng.normal(size=n)}
    dm = MP.DeviceMap({k: v.astype(np.float32) for k, v in params.items()}, [], 2.0)
    cfg = MP.MappingConfig()
    lrs = dm.lrs(cfg)
    ref = {k: params[k].astype(np.float32).astype(np.float64) for k in NAMES}
    m = np.zeros((n, 12)); v = np.zeros((n, 12))
    import ctypes
    from paper_2503_17491_b200._lib import lib
    for t in range(1, 4):
        g = rng.normal(size=(n, 12)).astype(np.float32)
        gd = torch.tensor(g, device="cuda")
        lib().ss_adam_step(*(ctypes.c_void_p(dm.params[k].data_ptr()) for k in NAMES), ctypes.c_void_p(gd.data_ptr()),
                           ctypes.c_void_p(dm.m.data_ptr()), ctypes.c_void_p(dm.v.data_ptr()), n, t,
                           lrs.ctypes.data_as(ctypes.c_void_p), 0.9, 0.999, 1e-8, float(np.log(1e-4)),
                           float(np.log(5.0)), ctypes.c_void_p(engine.stream_ptr()))
        m = 0.9 * m + 0.1 * g
        v = 0.999 * v + 0.001 * g.astype(np.float64) ** 2
        upd = (m / (1 - 0.9 ** t)) / (np.sqrt(v / (1 - 0.999 ** t)) + 1e-8)
        c = 0
        for i, k in enumerate(NAMES):
            w = engine.PARAM_WIDTH[k]
            ref[k] = ref[k] - lrs[i] * upd[:, c:c + w].reshape(ref[k].shape)
            c += w
        ref["log_scales"] = np.clip(ref["log_scales"], np.log(1e-4), np.log(5.0))
    for k in NAMES:
        got = dm.params[k].cpu().numpy().reshape(ref[k].shape)
        assert np.abs(got - ref[k]).max() <= 1e-5 * max(1.0, np.abs(ref[k]).max()), k


def _golden_map():
    kfs = []
    for i in range(2):
        c = G[f"kf{i}_cam"]
        cam = SphericalCamera(int(c[0]), int(c[1]), *[float(x) for x in c[2:]])
        kfs.append(MP.DeviceKeyframe(cam, SE3Pose(G[f"kf{i}_R"], G[f"kf{i}_t"]), G[f"kf{i}_range"], G[f"kf{i}_valid"],
                                     G[f"kf{i}_normal"], G[f"kf{i}_nvalid"]))
    return MP.DeviceMap({k: G[f"b_{k}"] for k in NAMES}, kfs, float(G["scene_scale"]))


def test_refine_matches_reference(cuda):
    dm = _golden_map()
    cfg = MP.MappingConfig(n_spawn=1200)
    losses = dm.refine(cfg, 3, np.random.default_rng(99))
    ref_losses = G["losses"]
    print("losses", losses, ref_losses)
    assert abs(losses[0] - ref_losses[0]) <= 1e-4 * abs(ref_losses[0])
    assert np.allclose(losses, ref_losses, rtol=2e-3)
    assert dm.t == int(G["adam_t"])
    for k in NAMES:
        before = G[f"b_{k}"].reshape(-1)
        d_ref = G[f"a_{k}"].reshape(-1) - before
        d_got = dm.params[k].cpu().numpy().astype(np.float64).reshape(-1) - before
        rel = np.linalg.norm(d_got - d_ref) / max(np.linalg.norm(d_ref), 1e-30)
        print(k, "update rel err", rel)
        # Adam normalises each component.  The raw tangent gradient is orthogonal to
        # the raw vector (Gram-Schmidt is scale invariant), so its radial component is
        # round-off (1e-17 in the float64 reference, 1e-8 in float32) that Adam turns
        # into +-lr steps of random sign: those classes get a looser gate.  The
        # observable, the loss, agrees to 1e-5 above.
        gate = 6e-2 if k.startswith("raw_t") else 2e-2
        assert rel <= gate, (k, rel)


def test_graph_refine_matches_eager(cuda):
    """refine() replaying one CUDA graph per keyframe equals the eager loop (same keyframe
    draws; float-atomic rounding only), Adam step counter included."""
    cfg = MP.MappingConfig(n_spawn=1200)
    a, b = _golden_map(), _golden_map()
    la = a.refine(cfg, 6, np.random.default_rng(5), graphs=True)
    lb = b.refine(cfg, 6, np.random.default_rng(5), graphs=False)
    assert a.t == b.t == 6
    # step 1 agrees to float64 atomics order; later steps drift by Adam-amplified float32 rounding
    assert abs(la[0] - lb[0]) <= 1e-9 * abs(lb[0]) and np.allclose(la, lb, rtol=1e-4)
    la2 = a.refine(cfg, 4, np.random.default_rng(6), graphs=True)  # graphs reused, counter continues
    lb2 = b.refine(cfg, 4, np.random.default_rng(6), graphs=False)
    assert a.t == b.t == 10 and np.allclose(la2, lb2, rtol=5e-4)
    # Adam normalises components whose gradient is round-off into +-lr steps, so a few entries
    # differ by up to lr x steps between any two summation orders; the bulk agrees
    for k in NAMES:
        x, y = a.params[k].cpu().numpy(), b.params[k].cpu().numpy()
        assert np.linalg.norm(x - y) <= 2e-3 * np.linalg.norm(y), k


def test_split_backward_equals_full(cuda):
    """ss_render_backward_blend + ss_render_finalize over row chunks == ss_render_backward."""
    from paper_2503_17491_b200.parallel import row_chunks
    cfg = MP.MappingConfig(n_spawn=1200)
    dm = _golden_map()
    g_full, p_full = dm.raw_gradient(1, cfg)
    dm.blend_gradient(1, cfg)
    out = torch.full_like(g_full, float("nan"))
    for b, e in row_chunks(dm.n, 5):
        dm.finalize_rows(b, e, out)
    torch.cuda.synchronize()
    diff = (out - g_full).abs().max().item()
    scale = g_full.abs().max().item()
    assert diff <= 1e-6 * scale, (diff, scale)  # same kernels; float-atomic order only


def test_shared_map_device_ops_world1(cuda):
    """parallel.device_ops + SharedMapTrainer at world size 1 (an NCCL communicator of one
    rank): one trainer step equals DeviceMap.step on the keyframe the sampler draws."""
    import socket

    import torch.distributed as dist

    from paper_2503_17491_b200.parallel import SharedMapTrainer, device_ops
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        cfg = MP.MappingConfig(n_spawn=1200)
        a, b = _golden_map(), _golden_map()
        tr = SharedMapTrainer(device_ops(a, cfg), len(a.keyframes), cfg, seed=7, chunks=4)
        picks = [tr.step() for _ in range(3)]
        rng = np.random.default_rng(7)
        ref_picks = [MP.sample_keyframe_index(len(b.keyframes), cfg.kf_sample_p, rng) for _ in range(3)]
        assert picks == ref_picks
        for k in ref_picks:
            b.step(k, cfg)
        assert a.t == b.t == 3
        for k in NAMES:
            x, y = a.params[k].cpu().numpy(), b.params[k].cpu().numpy()
            assert np.linalg.norm(x - y) <= 2e-3 * np.linalg.norm(y), k
    finally:
        dist.destroy_process_group()


def test_local_map_shard_replay_matches_refine(cuda):
    """parallel.LocalMapShard (graph replay, maps interleaved round robin) equals each map's
    own refine() with the same sampler seeds."""
    from paper_2503_17491_b200.parallel import LocalMapShard
    cfg = MP.MappingConfig(n_spawn=1200)
    maps = [_golden_map(), _golden_map()]
    sh = LocalMapShard(maps, cfg, seed=11)
    sh.begin()
    for _ in range(6):
        sh.step()
    assert sh.end()
    for i, dm in enumerate(maps):
        ref = _golden_map()
        ref.refine(cfg, 3, np.random.default_rng(11 + i), graphs=False)
        assert dm.t == ref.t == 3
        for k in NAMES:
            x, y = dm.params[k].cpu().numpy(), ref.params[k].cpu().numpy()
            assert np.linalg.norm(x - y) <= 2e-3 * np.linalg.norm(y), k


@pytest.mark.gpu
def test_reduced_run_quality_vs_reference(cuda):
    """The reference's reduced config-2 run (tests/golden/golden_quality.npz: LocalMap.start +
    3 add_keyframe at 512x32, then 30 refine iterations) repeated on the device with the same
    images and seeds: same map size, and the depth RMSE before and after refinement within
    5 % of the reference's (the runs differ by float32 rounding only, so the weighted spawn
    draws and the refine trajectory stay close)."""
    from paper_2503_17491_b200 import workloads as W
    fx = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_quality.npz"))
    r = W.quality_run(fx)
    assert abs(r["splats"] - int(fx["n_built"])) <= 0.01 * int(fx["n_built"])
    for k in ("rmse_before", "rmse_after"):
        ours, ref = np.array(r[k][:2]), fx[k][:2]
        assert np.all(np.abs(ours - ref) <= 0.05 * ref), (k, ours, ref)
    assert r["rmse_after"][0] < r["rmse_before"][0]
    assert abs(r["loss_first"] - float(fx["losses"][0])) <= 1e-3 * float(fx["losses"][0])
