"""Registrations/s: register() one frame at a time against register_batch(B frames)."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_17491_b200 import engine  # noqa: E402
from paper_2503_17491_b200 import registration as REG  # noqa: E402
from paper_2503_17491_b200 import workloads as W  # noqa: E402

params, cam, scans, truths, initials = W.config3_frames(16)
dp = engine.as_device_params(params)
host_scans = scans
if os.environ.get("DEVICE_SCANS"):  # device-resident scans (the bench's value); host scans: e2e-like
    scans = [torch.as_tensor(sc, device="cuda") for sc in scans]
cfg = REG.RegistrationConfig(mode="photometric", max_iters=20, tol=0.0)
out = {}
for B in (1, 2, 4, 8, 16):
    for _ in range(2):
        REG.register_batch(dp, scans[:B], cam, initials[:B], cfg)
    torch.cuda.synchronize()
    reps = max(2, 32 // B)
    t0 = time.perf_counter()
    for _ in range(reps):
        res = REG.register_batch(dp, scans[:B], cam, initials[:B], cfg)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    out[B] = {"registrations_per_s": B / dt, "ms_per_batch": dt * 1e3,
              "max_err_m": max(float(np.abs(r.pose.translation - t.translation).max()) for r, t in zip(res, truths))}
    print(B, out[B], flush=True)
for _ in range(2):
    REG.register(dp, host_scans[0], cam, initials[0], cfg)
torch.cuda.synchronize()
t0 = time.perf_counter()
for f in range(16):
    REG.register(dp, host_scans[f], cam, initials[f], cfg)
torch.cuda.synchronize()
out["single"] = {"registrations_per_s": 16 / (time.perf_counter() - t0)}
print(json.dumps(out))
