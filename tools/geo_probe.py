"""One geometric-mode registration loop at config 3 (for ncu)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_17491_b200 import registration as REG, engine, SphericalCamera
from paper_2503_17491_b200 import workloads as W
params, cam, scan_pts, truth, initial = W.config3_problem()
geo = SphericalCamera(cam.width * 2, cam.height * 2, cam.az_min, cam.az_max, cam.el_min, cam.el_max)
dp = engine.as_device_params(params)
c = REG.RegistrationConfig(mode="geometric", max_iters=20, tol=0.0)
X1, n1 = REG.sample_anchors(dp, geo, initial, c, thin=1)
tree = REG.build_leaf_tree(X1, initial.translation)
scan = REG.DeviceScan(cam, scan_pts)
sel = np.random.default_rng(0).choice(scan_pts.shape[0], c.max_geo_points, replace=False)
gs = torch.as_tensor(np.ascontiguousarray(scan_pts[sel]), device="cuda")
for _ in range(2):
    res = REG.solve_device(c, initial, scan, None, tree, gs)
torch.cuda.synchronize()
print(res.iterations, res.n_geo)
