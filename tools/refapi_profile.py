"""cProfile of the reference-signature e2e step (bench.e2e_reference_api's loop)."""
import cProfile
import pstats
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2503_17491_b200 import PixelGradients, SE3Pose, SplatModel, rasterize_backward, rasterize_forward  # noqa: E402
from paper_2503_17491_b200 import workloads as W  # noqa: E402

c = W.config(1)
cam = c["camera"]
model = SplatModel.from_params({k: v.astype(np.float64) for k, v in c["splats"].items()})
pose = SE3Pose.identity()
rng = np.random.default_rng(0)
pg = PixelGradients(np.sign(rng.normal(size=(cam.height, cam.width))), 0.1 * rng.normal(size=(cam.height, cam.width, 3)),
                    0.05 * rng.normal(size=(cam.height, cam.width)))


def one():
    model.touch()
    out, rec = rasterize_forward(cam, pose, model)
    g = rasterize_backward(model, rec, out, pg)
    return out.range, g.d_centers


for _ in range(3):
    one()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    one()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
