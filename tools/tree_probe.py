"""Leaf tree of the config-3 model points (for ncu launch lists)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_17491_b200 import registration as REG, engine, SphericalCamera
from paper_2503_17491_b200 import workloads as W
params, cam, scan_pts, truth, initial = W.config3_problem()
geo = SphericalCamera(cam.width * 2, cam.height * 2, cam.az_min, cam.az_max, cam.el_min, cam.el_max)
dp = engine.as_device_params(params)
X1, n1 = REG.sample_anchors(dp, geo, initial, REG.RegistrationConfig(), thin=1)
for _ in range(2):
    tree = REG.build_leaf_tree(X1, initial.translation)
torch.cuda.synchronize()
print("leaves", tree.sizes.shape[0])
