"""Config-2 map render (few tiles, segment forward): per tile, the list length L against the
largest last-contributing position over its pixels, and how many pixels never saturate --
the share of the list a forward that stopped at saturation could skip."""
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
from paper_2503_17491_b200.rasterizer import RasterConfig  # noqa: E402

dkfs = W.device_keyframes(W.keyframe_targets(10, 0, 1024, 64))
dm = W.build_local_map(dkfs, 20_000, 0)
cfg = MP.MappingConfig(w_opacity=0.05, w_normal=0.1)
rng = np.random.default_rng(0)
dm.refine(cfg, 20, rng, graphs=False)
kf = dm.keyframes[0]
D, N, O = engine.forward(kf.camera, pose_rt(kf.pose), dm.params, RasterConfig(), dm.rec, sync=True)
cam = kf.camera
P = cam.width * cam.height
T = torch.empty(P, dtype=torch.float32, device="cuda")
last = torch.empty(P, dtype=torch.int32, device="cuda")
s = ctypes.c_void_p(engine.stream_ptr())
lib().ss_records_pixel_state(dm.rec.ptr, ctypes.c_void_p(T.data_ptr()), ctypes.c_void_p(last.data_ptr()), s)
npairs = ctypes.c_int64(0)
tx = ctypes.c_int32(0)
ty = ctypes.c_int32(0)
lib().ss_records_counts(dm.rec.ptr, ctypes.byref(npairs), ctypes.byref(tx), ctypes.byref(ty))
tp = torch.empty(tx.value * ty.value + 1, dtype=torch.int64, device="cuda")
ps = torch.empty(max(1, npairs.value), dtype=torch.int64, device="cuda")
lib().ss_records_export(dm.rec.ptr, ctypes.c_void_p(tp.data_ptr()), ctypes.c_void_p(ps.data_ptr()), s)
torch.cuda.synchronize()
tp = tp.cpu().numpy()
L = np.diff(tp)
la = last.cpu().numpy().reshape(cam.height, cam.width)
Tf = T.cpu().numpy().reshape(cam.height, cam.width)
TS = 8
ntx, nty = tx.value, ty.value
ml = np.zeros(ntx * nty, dtype=np.int64)
unsat = np.zeros(ntx * nty, dtype=np.int64)
for t in range(ntx * nty):
    r, c = divmod(t, ntx)
    blk = la[r * TS:(r + 1) * TS, c * TS:(c + 1) * TS]
    ml[t] = blk.max()
    unsat[t] = int((Tf[r * TS:(r + 1) * TS, c * TS:(c + 1) * TS] >= 1e-4).sum())
seg = 128
nseg = (L + seg - 1) // seg
need = np.minimum(nseg, (ml + seg - 1) // seg + 1)
print(f"tiles {L.size}, pairs {L.sum()}, mean L {L.mean():.0f}, max L {L.max()}")
print(f"entries up to the last contribution: {ml.sum() / L.sum():.3f} of all; segments needed (last + 1): "
      f"{need.sum() / nseg.sum():.3f} of {nseg.sum()}")
print(f"tiles with every pixel saturated (T < 1e-4): {(unsat == 0).mean():.3f}; mean unsaturated pixels per tile "
      f"{unsat.mean():.1f}")
sat = unsat == 0
print(f"segments needed on saturated tiles only: {(np.where(sat, need, nseg)).sum() / nseg.sum():.3f}")
