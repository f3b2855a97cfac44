"""Config-2 refine by CUDA-graph replay (as bench.py's mapping line), a few iterations, for
an ncu launch list of the kernels inside the graphs."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_17491_b200 import mapping as MP  # noqa: E402
from paper_2503_17491_b200 import workloads as W  # noqa: E402

dkfs = W.device_keyframes(W.keyframe_targets(10, 0, 1024, 64))
dm = W.build_local_map(dkfs, 20_000, 0)
cfg = MP.MappingConfig(w_opacity=0.05, w_normal=0.1)
rng = np.random.default_rng(0)
dm.capture_graphs(cfg)
dm.refine(cfg, int(sys.argv[1]) if len(sys.argv) > 1 else 5, rng)
torch.cuda.synchronize()
print("ok")
