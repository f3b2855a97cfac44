"""A/B of the binning paths on the GPU: the global-sort binning (default) against the
round-1 per-tile sort (SS_BINNING=legacy): identical tile lists, per-stage times.
Run twice (the env var is read when records are created):
  python tools/ab_binning.py            and   SS_BINNING=legacy python tools/ab_binning.py
"""
import ctypes
import hashlib
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_17491_b200 import _lib, engine  # noqa: E402
from paper_2503_17491_b200 import workloads as W  # noqa: E402
from paper_2503_17491_b200.rasterizer import RasterConfig  # noqa: E402

STAGES = ["preprocess", "emit", "bucket", "tile_sort", "unused", "forward", "backward", "finalize"]


def main():
    L = _lib.lib()
    out = {"mode": os.environ.get("SS_BINNING", "global-sort")}
    for name, (cam, n, seed) in {"config1": (W.synth_camera(2048, 128), 500_000, 1),
                                 "config0": (W.synth_camera(1024, 64), 50_000, 0)}.items():
        sp = {k: torch.from_numpy(v).cuda() for k, v in W.random_splats(n, seed).items()}
        pose12 = np.concatenate([np.eye(3).reshape(9), np.zeros(3)])
        rec = engine.Records()
        engine.forward(cam, pose12, sp, RasterConfig(), rec)
        for _ in range(5):
            engine.forward(cam, pose12, sp, RasterConfig(), rec, sync=False)
        torch.cuda.synchronize()
        L.ss_records_profile(rec.ptr, 1)
        for _ in range(20):
            engine.forward(cam, pose12, sp, RasterConfig(), rec, sync=False)
        torch.cuda.synchronize()
        L.ss_records_profile(rec.ptr, 0)
        assert rec.check(True) == 0
        ms = (ctypes.c_double * 8)()
        cnt = (ctypes.c_int32 * 8)()
        L.ss_records_stage_times(rec.ptr, ms, cnt, 8)
        tp, ps = rec.export()
        h = np.concatenate([tp.cpu().numpy(), ps.cpu().numpy()])
        out[name] = {"stage_us": {STAGES[i]: round(1e3 * ms[i] / max(cnt[i], 1), 2) for i in range(8)},
                     "pairs": int(ps.numel()), "lists_sha": hashlib.sha1(h.tobytes()).hexdigest()}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
