"""Time the config-1 step eagerly and as a captured CUDA graph."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_17491_b200 import engine
from paper_2503_17491_b200 import workloads as W
from paper_2503_17491_b200.rasterizer import RasterConfig

c = W.config(1); cam = c["camera"]
dev = torch.device("cuda")
sp = {k: torch.from_numpy(v).to(dev) for k, v in c["splats"].items()}
tg = W.target_images(W.Scene(0), cam)
kr = torch.from_numpy(tg["range"]).to(dev); kv = torch.from_numpy(tg["valid"].astype(np.uint8)).to(dev)
kn = torch.from_numpy(tg["normal"]).to(dev); knv = torch.from_numpy(tg["nvalid"].astype(np.uint8)).to(dev)
rec = engine.Records(); cfg = RasterConfig(); pose = np.concatenate([np.eye(3).reshape(9), np.zeros(3)])
def step():
    D, N, O = engine.forward(cam, pose, sp, cfg, rec, sync=False)
    dD, dN, dO, parts = engine.mapping_loss(D, N, O, kr, kv, kn, knv, 0.0, 0.1)
    return engine.backward(rec, sp, dD, dN, dO, raw_space=True)
engine.forward(cam, pose, sp, cfg, rec)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(3): g_e = step()
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
assert rec.check(True) == 0
def timeit(fn, n=20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn(); torch.cuda.synchronize()
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
eager = timeit(step)
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph):
    g_out = step()
torch.cuda.synchronize()
gt = timeit(graph.replay)
g_ref = step(); torch.cuda.synchronize()
print(f"eager {eager*1000:.1f} us/step  graph {gt*1000:.1f} us/step  graph-vs-eager grad max diff {float((g_out - g_ref).abs().max()):.3e} (atomics order)")
