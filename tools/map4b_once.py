"""Config 4b's shared 2M-surfel map (four config-4a maps merged): eager refine steps with
stage timers, and list statistics."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_17491_b200 import mapping as MP  # noqa: E402
from paper_2503_17491_b200 import workloads as W  # noqa: E402
from paper_2503_17491_b200._lib import lib  # noqa: E402

dkfs = W.device_keyframes(W.keyframe_targets(10, 0, 2048, 128))
dm = W.merge_maps([W.build_local_map(dkfs, 50_000, m) for m in range(4)], dkfs)
cfg = MP.MappingConfig(w_opacity=0.05, w_normal=0.1)
rng = np.random.default_rng(0)
dm.refine(cfg, 3, rng, graphs=False)
torch.cuda.synchronize()
lib().ss_records_profile(dm.rec.ptr, 1)
for _ in range(10):
    dm.step(MP.sample_keyframe_index(len(dm.keyframes), cfg.kf_sample_p, rng), cfg)
torch.cuda.synchronize()
lib().ss_records_profile(dm.rec.ptr, 0)
ms = (ctypes.c_double * 8)()
nn = (ctypes.c_int32 * 8)()
lib().ss_records_stage_times(dm.rec.ptr, ms, nn, 8)
names = ["preprocess", "emit", "bucket", "tile_sort", "unused", "forward", "backward", "finalize"]
print("splats", dm.n, "stages (us):", " ".join(f"{n}={ms[i] / max(nn[i], 1) * 1000:.1f}" for i, n in enumerate(names) if nn[i]))
tp, _ = dm.rec.export()
L = np.diff(tp.cpu().numpy())
print("tiles", L.size, "list mean", L.mean(), "max", L.max(), "> 2048:", int((L > 2048).sum()), "> 8192:", int((L > 8192).sum()))
