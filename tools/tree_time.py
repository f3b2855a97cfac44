"""Wall time of build_leaf_tree at config 3 and of its C call alone (host overhead split)."""
import ctypes, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_17491_b200 import registration as REG, engine, SphericalCamera
from paper_2503_17491_b200 import workloads as W
from paper_2503_17491_b200._lib import lib
params, cam, scan_pts, truth, initial = W.config3_problem()
geo = SphericalCamera(cam.width * 2, cam.height * 2, cam.az_min, cam.az_max, cam.el_min, cam.el_max)
dp = engine.as_device_params(params)
X1, n1 = REG.sample_anchors(dp, geo, initial, REG.RegistrationConfig(), thin=1)
n = X1.shape[0]
for _ in range(3):
    REG.build_leaf_tree(X1, initial.translation)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    REG.build_leaf_tree(X1, initial.translation)
torch.cuda.synchronize()
print(f"build_leaf_tree {(time.perf_counter() - t0) / 10 * 1e3:.3f} ms, n={n}")
vp = np.ascontiguousarray(np.asarray(initial.translation, np.float64))
cent, nrm = np.zeros((n, 3)), np.zeros((n, 3))
sizes, usable = np.zeros(n, np.int32), np.zeros(n, np.uint8)
pl = torch.empty(n, dtype=torch.int32, device="cuda")
nl = ctypes.c_int32(0)
ws = torch.empty(int(lib().ss_leaf_tree_workspace_bytes(n)), dtype=torch.uint8, device="cuda")
def call():
    lib().ss_leaf_tree_build(ctypes.c_void_p(X1.data_ptr()), n, vp.ctypes.data_as(ctypes.c_void_p), 64, 0.02, n,
                             cent.ctypes.data_as(ctypes.c_void_p), nrm.ctypes.data_as(ctypes.c_void_p),
                             sizes.ctypes.data_as(ctypes.c_void_p), usable.ctypes.data_as(ctypes.c_void_p),
                             ctypes.c_void_p(pl.data_ptr()), ctypes.byref(nl), ctypes.c_void_p(ws.data_ptr()),
                             ctypes.c_void_p(engine.stream_ptr()))
call()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    call()
torch.cuda.synchronize()
print(f"ss_leaf_tree_build {(time.perf_counter() - t0) / 10 * 1e3:.3f} ms, leaves {nl.value}")
