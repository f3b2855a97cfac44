"""Time the pieces of one config-3 photometric registration (device loop)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_17491_b200 import registration as REG
from paper_2503_17491_b200 import SphericalCamera
from paper_2503_17491_b200 import workloads as W

params, cam, scan_pts, truth, initial = W.config3_problem()
cfg = REG.RegistrationConfig(mode="photometric", max_iters=20, tol=0.0)
geo = SphericalCamera(cam.width * 2, cam.height * 2, cam.az_min, cam.az_max, cam.el_min, cam.el_max)
from paper_2503_17491_b200 import engine
dp = engine.as_device_params(params)
def t(fn, n=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): r = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3, r
ta, (X, n) = t(lambda: REG.sample_anchors(dp, geo, initial, cfg, thin=4))
ts, scan = t(lambda: REG.DeviceScan(cam, scan_pts))
tl, res = t(lambda: REG._solve_device(X, scan, initial, cfg))
tr, _ = t(lambda: REG.register(dp, scan_pts, cam, initial, cfg))
tp, _ = t(lambda: engine.as_device_params(params))
print(f"anchors {ta:.3f} ms  scan {ts:.3f} ms  device loop {tl:.3f} ms ({res.iterations} it)  register() {tr:.3f} ms  params upload {tp:.3f} ms")
scfg = REG.RegistrationConfig()
X1, n1 = REG.sample_anchors(dp, geo, initial, scfg, thin=1)
tt, tree = t(lambda: REG.build_leaf_tree(X1, initial.translation))
ts2, _ = t(lambda: REG.register(dp, scan_pts, cam, initial, scfg))
print(f"model points {n1}: leaf tree {tt:.3f} ms ({tree.sizes.shape[0]} leaves); sequential register() {ts2:.3f} ms")
X1, n1 = REG.sample_anchors(dp, geo, initial, scfg, thin=1)
tree = REG.build_leaf_tree(X1, initial.translation)
scan = REG.DeviceScan(cam, scan_pts)
sel = np.random.default_rng(0).choice(scan_pts.shape[0], scfg.max_geo_points, replace=False) if scan_pts.shape[0] > scfg.max_geo_points else np.arange(scan_pts.shape[0])
gs = torch.as_tensor(np.ascontiguousarray(scan_pts[sel]), device="cuda")
Xw = X1[::4].contiguous()
for mode in ("geometric", "photometric", "joint", "sequential"):
    c = REG.RegistrationConfig(mode=mode, max_iters=20, tol=0.0)
    tm, res = t(lambda: REG.solve_device(c, initial, scan, Xw if mode != "geometric" else None, tree if mode != "photometric" else None, gs if mode != "photometric" else None))
    print(f"{mode}: loop {tm:.3f} ms, {res.iterations} it, {res.n_evaluations} evals, {tm / max(res.iterations, 1) * 1e3:.0f} us/it, {tm / max(res.n_evaluations, 1) * 1e3:.0f} us/eval")
