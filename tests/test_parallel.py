"""Multi-process logic of the multi-GPU paths on CPU (gloo, world size 2).

The shared-map trainer's sampler / chunked all-reduce / optimiser sequence
is run with CPU gradient ops (the float64 oracle's raw gradients of small
renders) and the reference's Adam (mapping.py:342-379, numpy restatement),
checking that both ranks hold identical parameters, that the summed
gradient equals the sum of the per-keyframe oracle gradients, and that the
parameters equal a single-process Adam on the summed gradients.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_problem():
    sys.path.insert(0, ROOT)
    from oracle import oracle as O
    from paper_2503_17491_b200 import workloads as W
    cam = W.synth_camera(128, 16)
    ct = (cam.width, cam.height, cam.az_min, cam.az_max, cam.el_min, cam.el_max)
    params = {k: v.astype(np.float64) for k, v in W.random_splats(400, 3, rmin=2, rmax=10,
                                                                  mean_log_scale=float(np.log(0.2))).items()}
    poses = [(np.eye(3), np.array([0.1 * k, 0.0, 0.0])) for k in range(4)]
    rng = np.random.default_rng(5)
    pix = [(rng.normal(size=(16, 128)), 0.1 * rng.normal(size=(16, 128, 3)), 0.05 * rng.normal(size=(16, 128)))
           for _ in poses]

    def grad_of(p, k):
        R, t = poses[k]
        r = O.render(ct, R, t, p)
        gD, gN, gO = pix[k]
        pl = O.backward_lists(ct, r["arr"], R, r["tile_ptr"], r["pair_splats"], r["range"], r["normal"],
                              r["opacity"], gD, gN, gO, max_threads=1)
        return O.raw_gradients(p, pl)

    return params, grad_of, len(poses)


PARAM_W = (("centers", 3), ("raw_t_alpha", 3), ("raw_t_beta", 3), ("log_scales", 2), ("logit_opacity", 1))


def _flat(params):
    n = len(params["centers"])
    return np.concatenate([np.asarray(params[k]).reshape(n, -1) for k, _ in PARAM_W], axis=1)


def _unflat(x):
    out, c = {}, 0
    for k, w in PARAM_W:
        out[k] = x[:, c:c + w] if w > 1 else x[:, c]
        c += w
    return out


class _Adam:
    """The reference optimiser step (mapping.py:342-379: per-group learning rates, bias
    correction) + the log-scale clamp of refine (mapping.py:496), in float64 on the
    flattened (n, 12) layout the fused device step uses."""

    def __init__(self, n, cfg, scene_scale=1.0):
        self.m = np.zeros((n, 12))
        self.v = np.zeros((n, 12))
        self.t = 0
        lr = [cfg.lr_centers * scene_scale] * 3 + [cfg.lr_tangents] * 6 + [cfg.lr_log_scales] * 2 + \
             [cfg.lr_logit_opacity]
        self.lr = np.array(lr)
        self.lo, self.hi = np.log(cfg.scale_floor), np.log(10.0 * cfg.scale_cap)

    def step(self, x, g):
        self.t += 1
        self.m = 0.9 * self.m + 0.1 * g
        self.v = 0.999 * self.v + 0.001 * g * g
        upd = self.lr * (self.m / (1 - 0.9 ** self.t)) / (np.sqrt(self.v / (1 - 0.999 ** self.t)) + 1e-8)
        x -= upd
        np.clip(x[:, 9:11], self.lo, self.hi, out=x[:, 9:11])


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, ROOT)
    from paper_2503_17491_b200.mapping import MappingConfig
    from paper_2503_17491_b200.parallel import GradOps, SharedMapTrainer, shard_maps

    params, grad_of, nkf = _oracle_problem()
    cfg = MappingConfig()
    state = {"x": _flat(params), "summed": [], "full": None}
    opt = _Adam(state["x"].shape[0], cfg)
    grad = torch.zeros((state["x"].shape[0], 12), dtype=torch.float64)

    def blend(k):  # the oracle's whole backward; finalize hands out its rows chunk by chunk
        state["full"] = torch.tensor(grad_of(_unflat(state["x"]), k), dtype=torch.float64)
        return None

    def finalize(b, e):
        grad[b:e] = state["full"][b:e]

    def adam(g):
        state["summed"].append(g.numpy().copy())
        opt.step(state["x"], g.numpy())

    tr = SharedMapTrainer(GradOps(blend, finalize, grad, adam, align=128), nkf, cfg, seed=123, chunks=3)
    picks = [tr.step() for _ in range(2)]
    out[rank] = {"x": state["x"], "picks": picks, "summed": state["summed"], "maps": shard_maps(8, rank, world)}
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_shared_map_allreduce_gloo():
    """Two ranks, three finalize/all-reduce chunks per step, the reference's Adam."""
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    a, b = out[0], out[1]
    assert np.array_equal(a["x"], b["x"])  # replicas stay identical
    assert a["maps"] == [0, 2, 4, 6] and b["maps"] == [1, 3, 5, 7]
    # first iteration: the summed gradient is the sum of the two ranks' keyframe gradients
    params, grad_of, nkf = _oracle_problem()
    k0, k1 = a["picks"][0], b["picks"][0]
    ref = grad_of(params, k0) + grad_of(params, k1)
    assert np.abs(a["summed"][0] - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())
    # two Adam steps on the summed gradients, single process, give the ranks' parameters
    from paper_2503_17491_b200.mapping import MappingConfig
    x = _flat(params)
    opt = _Adam(x.shape[0], MappingConfig())
    for it in range(2):
        if it == 1:
            g = grad_of(_unflat(x), a["picks"][1]) + grad_of(_unflat(x), b["picks"][1])
            assert np.abs(a["summed"][1] - g).max() <= 1e-12 * max(1.0, np.abs(g).max())
        opt.step(x, ref if it == 0 else g)
    assert np.abs(a["x"] - x).max() <= 1e-12


def test_row_chunks_and_shards():
    from paper_2503_17491_b200.parallel import row_chunks, shard_maps
    for n, c in ((1, 8), (127, 8), (128, 8), (1000, 3), (2_000_000, 8), (500_000, 16)):
        ch = row_chunks(n, c)
        assert ch[0][0] == 0 and ch[-1][1] == n
        assert all(b % 128 == 0 for b, _ in ch)
        assert all(ch[i][1] == ch[i + 1][0] for i in range(len(ch) - 1))
        assert len(ch) <= max(c, 1)
    assert sorted(sum((shard_maps(8, r, 3) for r in range(3)), [])) == list(range(8))
    with pytest.raises(ValueError):
        shard_maps(8, 3, 3)
