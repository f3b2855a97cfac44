"""Minimal config-1 step loop for ncu captures: W warm-up + S steps (fwd, loss, bwd)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_17491_b200 import engine  # noqa: E402
from paper_2503_17491_b200 import workloads as W  # noqa: E402
from paper_2503_17491_b200.rasterizer import RasterConfig  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfgi = int(sys.argv[2]) if len(sys.argv) > 2 else 1
c = W.config(cfgi)
cam = c["camera"]
dev = torch.device("cuda")
sp = {k: torch.from_numpy(v).to(dev) for k, v in c["splats"].items()}
tgt = W.target_images(W.Scene(0), cam)
kr = torch.from_numpy(tgt["range"]).to(dev)
kv = torch.from_numpy(tgt["valid"].astype(np.uint8)).to(dev)
kn = torch.from_numpy(tgt["normal"]).to(dev)
knv = torch.from_numpy(tgt["nvalid"].astype(np.uint8)).to(dev)
rec = engine.Records()
pose12 = np.concatenate([np.eye(3).reshape(9), np.zeros(3)])
for _ in range(3 + steps):
    D, N, O = engine.forward(cam, pose12, sp, RasterConfig(), rec, sync=False)
    dD, dN, dO, parts = engine.mapping_loss(D, N, O, kr, kv, kn, knv, 0.0, 0.1)
    g = engine.backward(rec, sp, dD, dN, dO, raw_space=True)
torch.cuda.synchronize()
print("ok", float(parts[0]), float(g.abs().sum()))
