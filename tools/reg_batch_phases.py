"""Phase timestamps of one register_batch(B=8) call (SS_BATCH_TIMING=1 prints them from C)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_17491_b200 import engine  # noqa: E402
from paper_2503_17491_b200 import registration as REG  # noqa: E402
from paper_2503_17491_b200 import workloads as W  # noqa: E402

params, cam, scans, truths, initials = W.config3_frames(8)
dp = engine.as_device_params(params)
scans = [torch.as_tensor(sc, device="cuda") for sc in scans]
cfg = REG.RegistrationConfig(mode="photometric", max_iters=20, tol=0.0)
for _ in range(6):
    REG.register_batch(dp, scans, cam, initials, cfg)
    torch.cuda.synchronize()
