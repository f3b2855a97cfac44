"""A few config-1 steps (forward + mapping loss + backward), for ncu captures."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_17491_b200 import engine  # noqa: E402
from paper_2503_17491_b200 import workloads as W  # noqa: E402
from paper_2503_17491_b200.rasterizer import RasterConfig  # noqa: E402

cam = W.synth_camera(2048, 128)
sp = {k: torch.from_numpy(v).cuda() for k, v in W.random_splats(500_000, 1).items()}
tgt = W.target_images(W.Scene(0), cam)
kf = [torch.from_numpy(np.asarray(tgt[k]).astype(t)).cuda()
      for k, t in (("range", np.float32), ("valid", np.uint8), ("normal", np.float32), ("nvalid", np.uint8))]
pose12 = np.concatenate([np.eye(3).reshape(9), np.zeros(3)])
rec = engine.Records()
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    D, N, O = engine.forward(cam, pose12, sp, RasterConfig(), rec)
    dD, dN, dO, parts = engine.mapping_loss(D, N, O, *kf, w_opacity=0.0, w_normal=0.1)
    g = engine.backward(rec, sp, dD, dN, dO, raw_space=True)
torch.cuda.synchronize()
print("ok", rec.counts()[0])
