"""Debug: worst 'safe' pixel of config 0 -- per-pair f64 reference vs float32 emulation."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
from paper_2503_17491_b200 import SE3Pose, SplatModel, rasterize_forward
from paper_2503_17491_b200 import workloads as W

c = W.config(0)
cam, params = c["camera"], c["splats"]
ct = (cam.width, cam.height, cam.az_min, cam.az_max, cam.el_min, cam.el_max)
ref = O.render(ct, np.eye(3), np.zeros(3), params, margins=True)
out, rec = rasterize_forward(cam, SE3Pose.identity(), SplatModel.from_params(params))
D = out.range; Dr = ref["range"]
err = np.abs(D - Dr) / np.maximum(np.abs(Dr), 1e-6)
err[ref["margin"] <= 1e-5] = 0
for p in np.argsort(err.ravel())[::-1][:3]:
    i, j = divmod(p, cam.width)
    print("pixel", i, j, "gpu", D[i, j], "ref", Dr[i, j], "rel", err[i, j], "O", ref["opacity"][i, j], out.opacity[i, j], "margin", ref["margin"][i, j])
    T = 8; tx = (cam.width + 7) // 8
    t = (i // T) * tx + j // T
    ids = ref["pair_splats"][ref["tile_ptr"][t]:ref["tile_ptr"][t + 1]]
    dirs, hx, hy, ok = O.pixel_planes(ct)
    v = dirs[i, j]; a = ref["arr"]
    Tr = 1.0
    for s in ids:
        Ba, Bb, Bc = a[s, 0:3], a[s, 3:6], a[s, 6:9]
        A = np.cross(Bb, Bc); Bv = np.cross(Bc, Ba); C = np.cross(Ba, Bb)
        w2 = v @ C; sa = (v @ A) / w2; sb = (v @ Bv) / w2; lam = (Bc @ C) / w2
        G = np.exp(-0.5 * (sa * sa + sb * sb)); al = min(a[s, 18] * G, 0.99)
        if al >= 1 / 255 and lam > 0:
            print("  splat", s, "alpha", al, "lam", lam, "sa", sa, "sb", sb, "T", Tr, "v.n", v @ a[s, 9:12], "range", a[s,21])
            Tr *= 1 - al
