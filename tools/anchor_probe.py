"""Split of the registration's model render + anchor extraction (config 3): device stage
times of the render and wall times of the pieces."""
import ctypes, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_17491_b200 import registration as REG, engine, SphericalCamera
from paper_2503_17491_b200 import workloads as W
from paper_2503_17491_b200._lib import lib
from paper_2503_17491_b200.geometry import pose_rt
params, cam, scan_pts, truth, initial = W.config3_problem()
geo = SphericalCamera(cam.width * 2, cam.height * 2, cam.az_min, cam.az_max, cam.el_min, cam.el_max)
dp = engine.as_device_params(params)
cfg = REG.RegistrationConfig()
for _ in range(3):
    REG.sample_anchors(dp, geo, initial, cfg, thin=1)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    REG.sample_anchors(dp, geo, initial, cfg, thin=1)
torch.cuda.synchronize()
print(f"sample_anchors {(time.perf_counter() - t0) / 20 * 1e3:.3f} ms")
rec = engine.Records.acquire()
engine.forward(geo, pose_rt(initial), dp, REG.RasterConfig(), rec)
lib().ss_records_profile(rec.ptr, 1)
t0 = time.perf_counter()
for _ in range(20):
    engine.forward(geo, pose_rt(initial), dp, REG.RasterConfig(), rec)
torch.cuda.synchronize()
print(f"forward (sync) {(time.perf_counter() - t0) / 20 * 1e3:.3f} ms")
lib().ss_records_profile(rec.ptr, 0)
ms = (ctypes.c_double * 8)(); nn = (ctypes.c_int32 * 8)()
lib().ss_records_stage_times(rec.ptr, ms, nn, 8)
names = ["preprocess", "emit", "bucket", "tile_sort", "unused", "forward", "backward", "finalize"]
print("stages (us):", " ".join(f"{n}={ms[i]/max(nn[i],1)*1000:.1f}" for i, n in enumerate(names) if nn[i]))
print("pairs", rec.counts())
