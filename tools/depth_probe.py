"""How deep into its tile list does each pixel keep contributing?  Config 2 (as bench builds
it, after 100 refine iterations) and config 1: per tile, max and mean over its pixels of the
last contributing list position, as a fraction of the list length (weighted by length)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_17491_b200 import engine  # noqa: E402
from paper_2503_17491_b200 import mapping as MP  # noqa: E402
from paper_2503_17491_b200 import workloads as W  # noqa: E402
from paper_2503_17491_b200._lib import lib  # noqa: E402
from paper_2503_17491_b200.geometry import pose_rt  # noqa: E402


def depth(cam, pose, params, tag):
    rec = engine.Records()
    D, N, O = engine.forward(cam, pose_rt(pose), params, MP.RasterConfig(), rec)
    tp, ps = rec.export()
    tp = tp.cpu().numpy()
    H, Wd = cam.height, cam.width
    T = torch.empty(H * Wd, dtype=torch.float32, device="cuda")
    last = torch.empty(H * Wd, dtype=torch.int32, device="cuda")
    lib().ss_records_pixel_state(rec.ptr, ctypes.c_void_p(T.data_ptr()), ctypes.c_void_p(last.data_ptr()),
                                 ctypes.c_void_p(engine.stream_ptr()))
    torch.cuda.synchronize()
    last = last.cpu().numpy().reshape(H, Wd)
    T = T.cpu().numpy().reshape(H, Wd)
    ts = 8
    tx, ty = (Wd + ts - 1) // ts, (H + ts - 1) // ts
    L = np.diff(tp)
    lt = last.reshape(ty, ts, tx, ts).transpose(0, 2, 1, 3).reshape(ty * tx, ts * ts)
    mx = lt.max(1)
    mn = lt.mean(1)
    ok = L > 0
    print(f"{tag}: tiles {ok.sum()}, list mean {L[ok].mean():.0f} max {L.max()}, "
          f"max-last/L weighted {np.sum(mx[ok]) / np.sum(L[ok]):.3f}, mean-last/L weighted {np.sum(mn[ok]) / np.sum(L[ok]):.3f}, "
          f"pixels terminated (T < 1e-4) {np.mean(T < 1e-4):.3f}")


dkfs = W.device_keyframes(W.keyframe_targets(10, 0, 1024, 64))
dm = W.build_local_map(dkfs, 20_000, 0)
cfg = MP.MappingConfig(w_opacity=0.05, w_normal=0.1)
depth(dkfs[0].camera, dkfs[0].pose, dm.params, "config2 before refine")
dm.refine(cfg, 100, np.random.default_rng(0))
torch.cuda.synchronize()
for i in (0, 5, 9):
    depth(dkfs[i].camera, dkfs[i].pose, dm.params, f"config2 after 100 iterations, keyframe {i}")
c = W.config(1)
depth(c["camera"], c["pose"], engine.as_device_params(c["splats"]), "config1")
