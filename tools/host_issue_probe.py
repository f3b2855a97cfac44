"""Host issue time of the config-1 bench step (forward + loss + backward through engine.*)
against its device time: is the GPU ever waiting for the host?"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_17491_b200 import engine  # noqa: E402
from paper_2503_17491_b200 import workloads as W  # noqa: E402
from paper_2503_17491_b200.rasterizer import RasterConfig  # noqa: E402

c = W.config(1)
cam = c["camera"]
dev = torch.device("cuda")
sp = {k: torch.from_numpy(v).to(dev) for k, v in c["splats"].items()}
tgt = W.target_images(W.Scene(0), cam)
kf = [torch.from_numpy(np.asarray(tgt[k]).astype(t)).to(dev)
      for k, t in (("range", np.float32), ("valid", np.uint8), ("normal", np.float32), ("nvalid", np.uint8))]
rec = engine.Records()
pose12 = np.concatenate([np.eye(3).reshape(9), np.zeros(3)])
cfg = RasterConfig()


def step():
    D, N, O = engine.forward(cam, pose12, sp, cfg, rec, sync=False)
    dD, dN, dO, parts = engine.mapping_loss(D, N, O, *kf, w_opacity=0.0, w_normal=0.1)
    return engine.backward(rec, sp, dD, dN, dO, raw_space=True)


engine.forward(cam, pose12, sp, cfg, rec)
for _ in range(10):
    step()
torch.cuda.synchronize()
n = 100
t0 = time.perf_counter()
for _ in range(n):
    step()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host issue {1e3 * (t1 - t0) / n:.3f} ms/step; wall incl. drain {1e3 * (t2 - t0) / n:.3f} ms/step")
