"""Wall-clock stages of the reference-signature e2e step at config 1 (host side of the drop-in)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2503_17491_b200 import PixelGradients, SE3Pose, SplatModel, engine  # noqa: E402
from paper_2503_17491_b200 import rasterizer as R  # noqa: E402
from paper_2503_17491_b200 import workloads as W  # noqa: E402

c = W.config(1)
cam = c["camera"]
model = SplatModel.from_params({k: v.astype(np.float64) for k, v in c["splats"].items()})
pose = SE3Pose.identity()
rng = np.random.default_rng(0)
pg = PixelGradients(np.sign(rng.normal(size=(cam.height, cam.width))), 0.1 * rng.normal(size=(cam.height, cam.width, 3)),
                    0.05 * rng.normal(size=(cam.height, cam.width)))
acc = {}
dp = R._device_params


def tick(name, t0):
    t1 = time.perf_counter()
    acc[name] = acc.get(name, 0.0) + (t1 - t0)
    return t1


for it in range(23):
    if it == 3:
        acc.clear()
    t = time.perf_counter()
    model.touch()
    params = R._device_params(model)
    t = tick("params (stage + upload issue)", t)
    torch.cuda.current_stream().synchronize()
    t = tick("  wait upload", t)
    R._device_params = lambda m, _p=params: _p  # (the cache lookup was timed above)
    out, rec = R.rasterize_forward(cam, pose, model)
    R._device_params = dp
    t = tick("forward (incl. capacity check)", t)
    _ = out.range
    t = tick("range image to host", t)
    gD, gN, gO = R._pixel_grads_to_device(pg, cam.height, cam.width)
    t = tick("pixel grads stage + upload", t)
    g = engine.backward(rec._handle, rec._params, gD, gN, gO, raw_space=False)
    torch.cuda.current_stream().synchronize()
    t = tick("backward (device)", t)
    sg = R.SplatGradients.from_device(g)
    t = tick("gradients to host float64", t)
for k, v in acc.items():
    print(f"{k:34s} {v / 20 * 1e3:7.3f} ms")
print(f"{'total':34s} {sum(acc.values()) / 20 * 1e3:7.3f} ms")
