"""Multi-process logic of the multi-GPU paths on CPU (gloo, world size 2).

The shared-map trainer's sampler / all-reduce / optimiser sequence is run
with CPU gradient ops (the float64 oracle's raw gradients of small renders),
checking that both ranks hold identical parameters and that the summed
gradient equals the sum of the per-keyframe oracle gradients.
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


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, ROOT)
    from paper_2503_17491_b200.mapping import MappingConfig
    from paper_2503_17491_b200.parallel import GradOps, SharedMapTrainer, shard_maps

    params, grad_of, nkf = _oracle_problem()
    flat = np.concatenate([params[k].reshape(len(params["centers"]), -1) for k in
                           ("centers", "raw_t_alpha", "raw_t_beta", "log_scales", "logit_opacity")], axis=1)
    state = {"x": flat.copy(), "summed": []}

    def unflat(x):
        return {"centers": x[:, 0:3], "raw_t_alpha": x[:, 3:6], "raw_t_beta": x[:, 6:9], "log_scales": x[:, 9:11],
                "logit_opacity": x[:, 11]}

    def grad(k):
        return torch.tensor(grad_of(unflat(state["x"]), k), dtype=torch.float64)

    def sgd(g):  # a deterministic optimiser stand-in: the point is the collective sequence
        state["summed"].append(g.numpy().copy())
        state["x"] -= 1e-3 * g.numpy()

    tr = SharedMapTrainer(GradOps(grad, sgd), nkf, MappingConfig(), seed=123)
    picks = [tr.step() for _ in range(2)]
    out[rank] = {"x": state["x"], "picks": picks, "summed": state["summed"], "maps": shard_maps(8, rank, world)}
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_shared_map_allreduce_gloo():
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
