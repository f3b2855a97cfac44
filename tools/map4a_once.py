"""One config-4a map (128x2048, start + 9 add_keyframe, 50k spawned per keyframe): eager refine
steps with stage timers, for a per-stage split and ncu launch lists."""
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
dm = W.build_local_map(dkfs, 50_000, 0)
cfg = MP.MappingConfig(w_opacity=0.05, w_normal=0.1)
rng = np.random.default_rng(0)
dm.refine(cfg, 3, rng, graphs=False)
torch.cuda.synchronize()
if len(sys.argv) > 1 and sys.argv[1] == "stages":
    lib().ss_records_profile(dm.rec.ptr, 1)
    for _ in range(20):
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
    print("tiles", L.size, "list mean", L.mean(), "max", L.max(), "> 2048:", int((L > 2048).sum()), ">= 1536:", int((L >= 1536).sum()))
print("ok")
