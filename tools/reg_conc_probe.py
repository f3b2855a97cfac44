"""Do B cooperative GN/LM loops run concurrently?  One loop at 148 and at 148/B blocks, and B
loops at 148/B blocks on B streams (ss_reg_solve_async), device time by CUDA events."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_17491_b200 import engine  # noqa: E402
from paper_2503_17491_b200 import registration as REG  # noqa: E402
from paper_2503_17491_b200 import workloads as W  # noqa: E402
from paper_2503_17491_b200._lib import SsRegOut, lib  # noqa: E402
from paper_2503_17491_b200.geometry import SphericalCamera, pose_rt  # noqa: E402

params, cam, scans, truths, initials = W.config3_frames(8)
dp = engine.as_device_params(params)
cfg = REG.RegistrationConfig(mode="photometric", max_iters=20, tol=0.0)
geo = SphericalCamera(cam.width * 2, cam.height * 2, cam.az_min, cam.az_max, cam.el_min, cam.el_max)
probs = []
for b in range(8):
    X, n = REG.sample_anchors(dp, geo, initials[b], cfg, thin=4)
    probs.append((X.contiguous(), REG.DeviceScan(cam, scans[b]), pose_rt(initials[b])))
torch.cuda.synchronize()
k = REG._solve_cfg(cfg)
c = engine.ss_camera(cam)
streams = [torch.cuda.Stream() for _ in range(8)]
outs = [torch.empty(ctypes.sizeof(SsRegOut), dtype=torch.uint8).pin_memory() for _ in range(8)]
wss = [torch.empty(int(lib().ss_reg_solve_workspace_bytes(0, 0, int(p[0].shape[0]))) + 1024, dtype=torch.uint8,
                   device="cuda") for p in probs]


def launch(b, blocks, stream):
    X, ds, t0 = probs[b]
    lib().ss_reg_solve_async(None, None, 0, None, 0, ctypes.c_void_p(X.data_ptr()), int(X.shape[0]),
                             ctypes.c_void_p(ds.range.data_ptr()), ctypes.c_void_p(ds.valid.data_ptr()),
                             ctypes.byref(c), t0.ctypes.data_as(ctypes.c_void_p), ctypes.byref(k), blocks,
                             ctypes.c_void_p(outs[b].data_ptr()), ctypes.c_void_p(wss[b].data_ptr()),
                             ctypes.c_void_p(stream.cuda_stream))


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


res = {}
for blocks in (148, 74, 37, 18, 9):
    res[f"one_loop_{blocks}_blocks_ms"] = timed(lambda: (streams[0].wait_stream(torch.cuda.current_stream()),
                                                         launch(0, blocks, streams[0])))
for B in (2, 4, 8):
    def many():
        for b in range(B):
            streams[b].wait_stream(torch.cuda.current_stream())
            launch(b, 148 // B, streams[b])
    res[f"{B}_loops_{148 // B}_blocks_ms"] = timed(many)
print(json.dumps(res))
