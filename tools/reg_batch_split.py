"""register_batch(B=8) with max_iters 0 (renders + scan images + anchors + an empty loop)
against the full 20-iteration batch: how the batch time splits (device-synchronised wall clock)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_17491_b200 import engine  # noqa: E402
from paper_2503_17491_b200 import registration as REG  # noqa: E402
from paper_2503_17491_b200 import workloads as W  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
params, cam, scans, truths, initials = W.config3_frames(B)
dp = engine.as_device_params(params)
scans = [torch.as_tensor(sc, device="cuda") for sc in scans]
for iters in (0, 20, 0, 20):
    cfg = REG.RegistrationConfig(mode="photometric", max_iters=iters, tol=0.0)
    for _ in range(3):
        REG.register_batch(dp, scans, cam, initials, cfg)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(10):
        REG.register_batch(dp, scans, cam, initials, cfg)
    torch.cuda.synchronize()
    print(f"B={B} max_iters={iters}: {(time.perf_counter() - t) / 10 * 1e3:.3f} ms per batch")
scans0 = scans[0].cpu().numpy()
for iters in (0, 20):
    cfg = REG.RegistrationConfig(mode="photometric", max_iters=iters, tol=0.0)
    for _ in range(3):
        REG.register(dp, scans0, cam, initials[0], cfg)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(10):
        REG.register(dp, scans0, cam, initials[0], cfg)
    torch.cuda.synchronize()
    print(f"single max_iters={iters}: {(time.perf_counter() - t) / 10 * 1e3:.3f} ms")
