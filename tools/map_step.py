"""A few config-2 refine iterations (for ncu launch lists)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_17491_b200 import mapping as MP
from paper_2503_17491_b200 import workloads as W
params, kfs, scale = W.config2_map()
dkf = [MP.DeviceKeyframe(cam, pose, tg["range"], tg["valid"], tg["normal"], tg["nvalid"]) for cam, pose, tg in kfs]
dm = MP.DeviceMap(params, dkf, scale)
cfg = MP.MappingConfig(w_opacity=0.05, w_normal=0.1)
dm.refine(cfg, int(sys.argv[1]) if len(sys.argv) > 1 else 3, np.random.default_rng(0))
torch.cuda.synchronize()
print("ok")
