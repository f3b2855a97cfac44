"""Config-2 mapping iterations: per-stage times of the render inside refine (stage timers)."""
import ctypes, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_17491_b200 import mapping as MP, engine
from paper_2503_17491_b200 import workloads as W
from paper_2503_17491_b200._lib import lib
params, kfs, scale = W.config2_map()
dkf = [MP.DeviceKeyframe(cam, pose, tg["range"], tg["valid"], tg["normal"], tg["nvalid"]) for cam, pose, tg in kfs]
dm = MP.DeviceMap(params, dkf, scale)
cfg = MP.MappingConfig(w_opacity=0.05, w_normal=0.1)
rng = np.random.default_rng(0)
dm.capture_graphs(cfg)
dm.refine(cfg, 5, rng)
torch.cuda.synchronize()
lib().ss_records_profile(dm.rec.ptr, 1)
t0 = time.perf_counter()
dm.refine(cfg, 50, rng)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 50
lib().ss_records_profile(dm.rec.ptr, 0)
ms = (ctypes.c_double * 8)(); nn = (ctypes.c_int32 * 8)()
lib().ss_records_stage_times(dm.rec.ptr, ms, nn, 8)
names = ["preprocess", "emit", "bucket", "tile_sort", "unused", "forward", "backward", "finalize"]
print(f"{1/dt:.0f} frames/s ({dt*1e3:.3f} ms/iter); stages (us):",
      " ".join(f"{n}={ms[i]/max(nn[i],1)*1000:.1f}" for i, n in enumerate(names) if nn[i]))
t0 = time.perf_counter()
for _ in range(50):
    idx = MP.sample_keyframe_index(len(dm.keyframes), cfg.kf_sample_p, rng)
    dm.step(idx, cfg)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host issue {1e3 * (t1 - t0) / 50:.3f} ms/iter, device drained {1e3 * (t2 - t1):.1f} ms after issue ended")
