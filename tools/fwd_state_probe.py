"""Config-0 forward: contributions counted from the bitmask (ss_records_work) and the
per-pixel last-contributor statistics, to compare library variants."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_17491_b200 import engine  # noqa: E402
from paper_2503_17491_b200 import workloads as W  # noqa: E402
from paper_2503_17491_b200._lib import lib  # noqa: E402
from paper_2503_17491_b200.geometry import pose_rt  # noqa: E402
from paper_2503_17491_b200.rasterizer import RasterConfig  # noqa: E402

for cfgi in [int(a) for a in (sys.argv[1:] or ["0", "1"])]:
    c = W.config(cfgi)
    cam = c["camera"]
    rec = engine.Records()
    D, N, O = engine.forward(cam, pose_rt(c["pose"]), engine.as_device_params(c["splats"]), RasterConfig(), rec)
    e = ctypes.c_int64(0)
    u = ctypes.c_int64(0)
    lib().ss_records_work(rec.ptr, ctypes.byref(e), ctypes.byref(u), ctypes.c_void_p(engine.stream_ptr()))
    P = cam.width * cam.height
    T = torch.empty(P, dtype=torch.float32, device="cuda")
    last = torch.empty(P, dtype=torch.int32, device="cuda")
    lib().ss_records_pixel_state(rec.ptr, ctypes.c_void_p(T.data_ptr()), ctypes.c_void_p(last.data_ptr()),
                                 ctypes.c_void_p(engine.stream_ptr()))
    torch.cuda.synchronize()
    la = last.cpu().numpy()
    print(f"config {cfgi}: E {e.value} U {u.value} last>0 {np.mean(la > 0):.3f} mean last {la.mean():.1f} "
          f"D sum {float(D.double().sum()):.6e} T mean {float(T.mean()):.4f}")
