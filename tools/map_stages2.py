"""Config-2 mapping as bench.py builds it (DeviceMap.start + 9 add_keyframe): per-stage device
times of eager refine steps (stage timers), then graph-replay time per iteration."""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_17491_b200 import mapping as MP  # noqa: E402
from paper_2503_17491_b200 import workloads as W  # noqa: E402
from paper_2503_17491_b200._lib import lib  # noqa: E402

dkfs = W.device_keyframes(W.keyframe_targets(10, 0, 1024, 64))
dm = W.build_local_map(dkfs, 20_000, 0)
cfg = MP.MappingConfig(w_opacity=0.05, w_normal=0.1)
rng = np.random.default_rng(0)
dm.refine(cfg, 5, rng, graphs=False)
torch.cuda.synchronize()
lib().ss_records_profile(dm.rec.ptr, 1)
for _ in range(30):
    dm.step(MP.sample_keyframe_index(len(dm.keyframes), cfg.kf_sample_p, rng), cfg)
torch.cuda.synchronize()
lib().ss_records_profile(dm.rec.ptr, 0)
ms = (ctypes.c_double * 8)()
nn = (ctypes.c_int32 * 8)()
lib().ss_records_stage_times(dm.rec.ptr, ms, nn, 8)
names = ["preprocess", "emit", "bucket", "tile_sort", "unused", "forward", "backward", "finalize"]
print("splats", dm.n, "stages (us):", " ".join(f"{n}={ms[i] / max(nn[i], 1) * 1000:.1f}" for i, n in enumerate(names) if nn[i]))
dm.capture_graphs(cfg)
dm.refine(cfg, 5, rng)
torch.cuda.synchronize()
t0 = time.perf_counter()
dm.refine(cfg, 200, rng)
torch.cuda.synchronize()
print(f"graph refine: {(time.perf_counter() - t0) / 200 * 1e3:.3f} ms/iter")
