"""Where does the e2e step go?  Times, per step: H2D alone, D2H alone, both directions
concurrently, the device step alone, and the double-buffered e2e loop (bench.py's)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_17491_b200 import engine
from paper_2503_17491_b200 import workloads as W
from paper_2503_17491_b200.rasterizer import RasterConfig

c = W.config(1); cam = c["camera"]; dev = torch.device("cuda")
host = {k: torch.from_numpy(v).pin_memory() for k, v in c["splats"].items()}
d = {k: v.to(dev) for k, v in host.items()}
gh = torch.empty((500_000, 12), dtype=torch.float32).pin_memory()
gd = torch.empty((500_000, 12), dtype=torch.float32, device=dev)
tg = W.target_images(W.Scene(0), cam)
kr = torch.from_numpy(tg["range"]).to(dev); kv = torch.from_numpy(tg["valid"].astype(np.uint8)).to(dev)
kn = torch.from_numpy(tg["normal"]).to(dev); knv = torch.from_numpy(tg["nvalid"].astype(np.uint8)).to(dev)
rec = engine.Records(); cfg = RasterConfig(); pose = np.concatenate([np.eye(3).reshape(9), np.zeros(3)])
def step(sp):
    D, N, O = engine.forward(cam, pose, sp, cfg, rec, sync=False)
    dD, dN, dO, parts = engine.mapping_loss(D, N, O, kr, kv, kn, knv, 0.0, 0.1)
    return engine.backward(rec, sp, dD, dN, dO, raw_space=True)
engine.forward(cam, pose, d, cfg, rec)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn, n=20):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / n * 1e3
def h2d():
    with torch.cuda.stream(s1):
        for k in host: d[k].copy_(host[k], non_blocking=True)
def d2h():
    with torch.cuda.stream(s2):
        gh.copy_(gd, non_blocking=True)
def both():
    h2d(); d2h()
print(f"H2D 24MB {timed(h2d):.3f} ms  D2H 24MB {timed(d2h):.3f} ms  both {timed(both):.3f} ms")
print(f"device step {timed(lambda: step(d)):.3f} ms")
t0 = time.perf_counter()
for _ in range(20): step(d)
t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"host issue time per step {(t1 - t0) / 20 * 1e3:.3f} ms (device drained {(t2 - t1) * 1e3:.1f} ms later)")
def overlapped():
    h2d(); d2h(); step(d)
print(f"step + both copies on side streams {timed(overlapped):.3f} ms")
print(f"step + H2D {timed(lambda: (h2d(), step(d))):.3f} ms   step + D2H {timed(lambda: (d2h(), step(d))):.3f} ms")
sc = torch.cuda.Stream()
def on_sc():
    h2d(); d2h()
    with torch.cuda.stream(sc):
        step(d)
print(f"step on a side stream + both copies {timed(on_sc):.3f} ms; default stream handle {torch.cuda.current_stream().cuda_stream}")
