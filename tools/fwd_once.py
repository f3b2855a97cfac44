"""A few config-1 forwards (for ncu launch lists of the binning kernels)."""
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
pose12 = np.concatenate([np.eye(3).reshape(9), np.zeros(3)])
rec = engine.Records()
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    engine.forward(cam, pose12, sp, RasterConfig(), rec)
torch.cuda.synchronize()
print("pairs", rec.counts()[0])
