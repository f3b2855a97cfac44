"""register() (photometric, config 3) wall time per call, after warm-up."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_17491_b200 import engine  # noqa: E402
from paper_2503_17491_b200 import registration as REG  # noqa: E402
from paper_2503_17491_b200 import workloads as W  # noqa: E402

params, cam, scans, truths, initials = W.config3_frames(4)
dp = engine.as_device_params(params)
cfg = REG.RegistrationConfig(mode="photometric", max_iters=20, tol=0.0)
for _ in range(5):
    REG.register(dp, scans[0], cam, initials[0], cfg)
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(20):
    REG.register(dp, scans[i % 4], cam, initials[i % 4], cfg)
torch.cuda.synchronize()
print(f"register: {(time.perf_counter() - t0) / 20 * 1e3:.3f} ms per call")
