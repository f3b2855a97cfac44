"""Config-2 mapping: per-stage device times of eager refine steps (stage timers on)."""
import ctypes, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_17491_b200 import mapping as MP, engine
from paper_2503_17491_b200 import workloads as W
from paper_2503_17491_b200._lib import lib
params, kfs, scale = W.config2_map()
dkf = [MP.DeviceKeyframe(cam, pose, tg["range"], tg["valid"], tg["normal"], tg["nvalid"]) for cam, pose, tg in kfs]
dm = MP.DeviceMap(params, dkf, scale)
cfg = MP.MappingConfig(w_opacity=0.05, w_normal=0.1)
rng = np.random.default_rng(0)
dm.refine(cfg, 5, rng, graphs=False)
torch.cuda.synchronize()
lib().ss_records_profile(dm.rec.ptr, 1)
for _ in range(30):
    dm.step(MP.sample_keyframe_index(len(dm.keyframes), cfg.kf_sample_p, rng), cfg)
torch.cuda.synchronize()
lib().ss_records_profile(dm.rec.ptr, 0)
ms = (ctypes.c_double * 8)(); nn = (ctypes.c_int32 * 8)()
lib().ss_records_stage_times(dm.rec.ptr, ms, nn, 8)
names = ["preprocess", "emit", "bucket", "tile_sort", "unused", "forward", "backward", "finalize"]
print("stages (us):", " ".join(f"{n}={ms[i]/max(nn[i],1)*1000:.1f}" for i, n in enumerate(names) if nn[i]))
c = dm.rec.counts()
print("records counts", c, "splats", dm.n)
# replay timing
dm.capture_graphs(cfg)
dm.refine(cfg, 5, rng)
torch.cuda.synchronize()
for iters in (50, 200):
    t0 = time.perf_counter()
    dm.refine(cfg, iters, rng)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / iters
    print(f"graph refine x{iters}: {dt*1e3:.3f} ms/iter")
g = dm._graphs[0]
torch.cuda.synchronize()
st = torch.cuda.Event(enable_timing=True); en = torch.cuda.Event(enable_timing=True)
st.record()
for _ in range(50):
    g.replay()
en.record()
torch.cuda.synchronize()
print(f"bare replay of keyframe 0: {st.elapsed_time(en) / 50:.3f} ms")
