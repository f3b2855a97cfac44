"""Benchmark: fwd+bwd spherical 2DGS renders/s at 128x2048 with 500k splats (BASELINE config 1).

One step = one forward render + fused mapping loss (range L1 + 0.1 normal,
mapping.py:128-151) + backward to the raw splat parameters, on the B200
kernels of libsplatb200.so.  Inputs are the seeded synthetic config-1 splats
(SURVEY 8(d)); with N GPUs each rank optimises its own independent map
(config 4a, weak scaling, no data-path collective).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

``--impl reference`` times the CPU oracle port of the reference's algorithm
(oracle/, float64, all host threads) on the same config and metric.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fwd+bwd spherical 2DGS renders/s (128×2048, 500k G, fp32)"
UNIT = "renders/s"
WORKLOAD = "config1: forward + mapping loss + backward to raw params, 128x2048 spherical camera, 500k splats, seed 1"
STAGES = ["preprocess", "emit", "bucket", "tile_sort", "unused", "forward", "backward", "finalize"]


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def loss_grads_host(D, N, tgt):
    M = tgt["valid"]
    w = 1.0 / np.maximum(tgt["range"].astype(np.float64), 1.0)
    gD = np.where(M, w * np.sign(D - tgt["range"]), 0.0)
    gN = np.where((M & tgt["nvalid"])[..., None], -0.1 * tgt["normal"].astype(np.float64), 0.0)
    return gD, gN, np.zeros_like(gD)


def oracle_render_step(cam, params, tgt):
    """One fwd+loss+bwd render with the float64 CPU oracle (the reference's algorithm)."""
    from oracle import oracle as O
    ct = (cam.width, cam.height, cam.az_min, cam.az_max, cam.el_min, cam.el_max)
    R, t = np.eye(3), np.zeros(3)
    arr = O.splat_arrays(params, R, t)
    tp, ps, _, _ = O.bin_splats(ct, arr)
    D, N, Op, _ = O.forward_lists(ct, arr, tp, ps)
    gD, gN, gO = loss_grads_host(D, N, tgt)
    pl = O.backward_lists(ct, arr, R, tp, ps, D, N, Op, gD, gN, gO, max_threads=64)
    return O.raw_gradients(params, pl)


def cpu_info():
    from oracle import oracle as O
    return O.num_threads()


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None
        self.marks = [None, None]

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.time(), line.strip()))

    def mark(self, i):
        self.marks[i] = time.time()

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.05)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        t0, t1 = self.marks
        inside = [s for ts, s in self.samples if t0 is not None and t0 <= ts <= t1]
        window = "timed"
        if not inside:  # timed region shorter than the sampling period: nearest samples
            inside = [s for ts, s in sorted(self.samples, key=lambda x: abs(x[0] - (t0 or 0)))[:3]]
            window = "nearest"
        sm, mx, reasons = [], [], set()
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        for s in inside:
            f = [x.strip() for x in s.split(",")]
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm), "window": window}


def config0_graph(dev, replays: int = 300):
    """config 0 (64x1024, 50k splats) is launch-bound, so it is reported
    graph-captured: forward + mapping loss + backward to the raw parameters as ONE CUDA
    graph, replayed back to back (device-resident inputs), timed with CUDA events."""
    import torch

    from paper_2503_17491_b200 import _lib, engine
    from paper_2503_17491_b200 import workloads as W
    from paper_2503_17491_b200.rasterizer import RasterConfig

    c = W.config(0)
    cam = c["camera"]
    sp = {k: torch.from_numpy(v).to(dev) for k, v in c["splats"].items()}
    tgt = W.target_images(W.Scene(0), cam)
    kf = [torch.from_numpy(np.asarray(tgt[k]).astype(t)).to(dev)
          for k, t in (("range", np.float32), ("valid", np.uint8), ("normal", np.float32), ("nvalid", np.uint8))]
    cfg = RasterConfig()
    pose12 = np.concatenate([np.eye(3).reshape(9), np.zeros(3)])
    rec = engine.Records()
    engine.forward(cam, pose12, sp, cfg, rec)  # sizes the pair buffers (synchronous check)
    _lib.lib().ss_records_reserve(rec.ptr, 2 * rec.counts()[0] + 65536)
    gout = torch.empty((int(sp["centers"].shape[0]), 12), dtype=torch.float32, device=dev)

    def step():
        D, N, O = engine.forward(cam, pose12, sp, cfg, rec, sync=False)
        dD, dN, dO, parts = engine.mapping_loss(D, N, O, *kf, w_opacity=0.0, w_normal=0.1)
        engine.backward(rec, sp, dD, dN, dO, raw_space=True, out=gout)
        return parts

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        with torch.cuda.graph(g, stream=side):
            step()
    torch.cuda.current_stream().wait_stream(side)
    for _ in range(10):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(replays):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / replays
    assert rec.check(True) == 0, "pair capacity exceeded during the graph replays"
    eager = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        step()
        b.record()
        eager.append((a, b))
    torch.cuda.synchronize()
    ms_eager = sum(a.elapsed_time(b) for a, b in eager) / len(eager)
    return {"metric": "config-0 fwd+bwd renders/s, CUDA-graph replay (64x1024, 50k splats, fp32)",
            "value": 1000.0 / ms, "unit": "renders/s", "ms_per_render": ms, "eager_ms_per_render": ms_eager,
            "replays": replays, "pairs": int(rec.counts()[0]),
            "note": "forward + mapping loss + backward to raw parameters captured once, replayed back to back"}


# Our kernels per config-1 step (launch list profiles/r01_v12_step_launches.csv):
# forward k_tile_intervals, k_preprocess, k_scan_blocks, k_emit, k_tile_hist_blocks,
# k_tile_prefix, k_scan_tiles, k_tile_scatter, k_tile_sort_big + k_tile_order (side stream),
# k_tile_sort, k_forward_long (side; tail lists only), k_forward, k_publish_totals (side);
# k_mapping_loss; backward k_backward, k_finalize.  (Plus torch fills that are not ours.)
KERNELS_PER_STEP = 17


def secondary_metrics(dev):
    """BASELINE's secondary metrics on one GPU: mapping frames/s (config 2: refine
    iterations on a 10-keyframe, 200k-surfel map, 64x1024) and photometric
    registrations/s (config 3: 300k-surfel map, 64x1024 scan, 20 GN iterations, tol 0)."""
    import torch

    from paper_2503_17491_b200 import engine
    from paper_2503_17491_b200 import mapping as MP
    from paper_2503_17491_b200 import registration as REG
    from paper_2503_17491_b200 import workloads as W

    out = {}
    out["config0_graph"] = config0_graph(dev)
    params, kfs, scale = W.config2_map()
    dkf = [MP.DeviceKeyframe(cam, pose, tg["range"], tg["valid"], tg["normal"], tg["nvalid"]) for cam, pose, tg in kfs]
    cfg = MP.MappingConfig(w_opacity=0.05, w_normal=0.1)
    MP.DeviceMap(params, dkf, scale).refine(cfg, 5, np.random.default_rng(1))  # warm-up on a throwaway map
    dm = MP.DeviceMap(params, dkf, scale)
    dm.capture_graphs(cfg)  # one CUDA graph per keyframe step (capture executes nothing)
    rng = np.random.default_rng(0)

    def depth_rmse():
        """(rendered range D, and D / O on pixels with O > 0.5 as sample_model reads depth) vs the
        keyframe range over its valid pixels, all keyframes."""
        from paper_2503_17491_b200.geometry import pose_rt
        se, cnt, se2, cnt2 = 0.0, 0, 0.0, 0
        for kf in dkf:
            D, _, O = engine.forward(kf.camera, pose_rt(kf.pose), dm.params, MP.RasterConfig(), dm.rec)
            v = kf.valid.bool()
            se += float(((D - kf.range)[v].double() ** 2).sum())
            cnt += int(v.sum())
            c = v & (O > 0.5)
            se2 += float(((D / O.clamp_min(1e-12) - kf.range)[c].double() ** 2).sum())
            cnt2 += int(c.sum())
        return float(np.sqrt(se / max(cnt, 1))), float(np.sqrt(se2 / max(cnt2, 1))), cnt2 / max(cnt, 1)

    rmse0 = depth_rmse()
    torch.cuda.synchronize()
    iters = 100  # BASELINE config 2: 100 Adam iterations
    times = []
    for rep in range(3):  # the first 100 iterations give the losses and the RMSE; median of 3 timings
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ls = dm.refine(cfg, iters, rng)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
        if rep == 0:
            losses = ls
            rmse1 = depth_rmse()
    ms = statistics.median(times)
    out["mapping"] = {"metric": "mapping frames/s (refine iterations: render+loss+backward+Adam)",
                      "value": iters * 1000.0 / ms, "unit": "frames/s", "iterations": iters, "splats": dm.n,
                      "timed_runs_ms": times,
                      "keyframes": len(dkf), "camera": "64x1024", "loss_first": losses[0], "loss_last": losses[-1],
                      "depth_rmse_m_before": rmse0[0], "depth_rmse_m_after": rmse1[0],
                      "confident_depth_rmse_m_before": rmse0[1], "confident_depth_rmse_m_after": rmse1[1],
                      "confident_fraction_after": rmse1[2],
                      "note": "config 2: 200k surfels back-projected from 10 keyframes (workloads.config2_map); "
                              "depth RMSE = rendered range D vs keyframe range over valid pixels of all keyframes; "
                              "confident: D / O where O > 0.5 (sample_model's depth)"}
    params, cam, scan, truth, initial = W.config3_problem()
    params = engine.as_device_params(params)  # the fixed map stays resident in HBM across registrations
    rcfg = REG.RegistrationConfig(mode="photometric", max_iters=20, tol=0.0)
    res = REG.register(params, scan, cam, initial, rcfg)  # warm-up (allocations)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reps = 3
    for _ in range(reps):
        res = REG.register(params, scan, cam, initial, rcfg)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    err_t = float(np.linalg.norm(res.pose.translation - truth.translation))
    cosang = (np.trace(res.pose.rotation.T @ truth.rotation) - 1) / 2
    err_r = float(np.degrees(np.arccos(np.clip(cosang, -1, 1))))
    e0t = float(np.linalg.norm(initial.translation - truth.translation))
    out["registration"] = {"metric": "photometric registrations/s (2x render + 20 GN iterations)",
                           "value": 1.0 / dt, "unit": "registrations/s", "ms": dt * 1e3, "iterations": res.iterations,
                           "n_photo": res.n_photo, "initial_err_m": e0t, "final_err_m": err_t, "final_err_deg": err_r,
                           "note": "config 3: 300k surfels on visible surfaces (device-resident map); per registration: "
                                   "2x render + anchors, scan range image, GN/LM loop in one cooperative kernel"}
    # the reference's default mode: sequential (geometric to convergence, then joint)
    scfg = REG.RegistrationConfig()
    res = REG.register(params, scan, cam, initial, scfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        res = REG.register(params, scan, cam, initial, scfg)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    out["registration_sequential"] = {
        "metric": "sequential registrations/s (default RegistrationConfig: leaf tree + geometric then joint)",
        "value": 1.0 / dt, "unit": "registrations/s", "ms": dt * 1e3, "iterations": res.iterations,
        "converged": res.converged, "n_geo": res.n_geo, "n_photo": res.n_photo,
        "final_err_m": float(np.linalg.norm(res.pose.translation - truth.translation))}
    return out


def run_reference(args, ws, rank):
    """--impl reference: the CPU oracle port on the box's host cores (rank 0 only)."""
    if rank != 0:
        return
    from paper_2503_17491_b200 import workloads as W
    c = W.config(1)
    cam, params = c["camera"], c["splats"]
    tgt = W.target_images(W.Scene(0), cam)
    cores = cpu_info()
    for _ in range(max(args.warmup_ref, 0)):
        oracle_render_step(cam, params, tgt)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle_render_step(cam, params, tgt)
    dt = time.perf_counter() - t0
    v = args.steps / dt
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup_ref, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, SURVEY 8(d))",
            "config": {"workload": WORKLOAD, "renders_per_step": 1},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": "full config-1 fwd+loss+bwd render per step, C float64 oracle (oracle/)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_b200(args, ws, rank, local):
    import torch

    from paper_2503_17491_b200 import _lib, engine
    from paper_2503_17491_b200 import workloads as W

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    L = _lib.lib()
    c = W.config(1)
    cam = c["camera"]
    # weak scaling: rank r optimises its own independent map (seed 1 + r)
    params_np = W.random_splats(500_000, 1 + rank)
    tgt = W.target_images(W.Scene(0), cam)
    splats = {k: torch.from_numpy(v).to(dev) for k, v in params_np.items()}
    kf_range = torch.from_numpy(tgt["range"]).to(dev)
    kf_valid = torch.from_numpy(tgt["valid"].astype(np.uint8)).to(dev)
    kf_normal = torch.from_numpy(tgt["normal"]).to(dev)
    kf_nvalid = torch.from_numpy(tgt["nvalid"].astype(np.uint8)).to(dev)
    from paper_2503_17491_b200.rasterizer import RasterConfig
    cfg = RasterConfig()
    pose12 = np.concatenate([np.eye(3).reshape(9), np.zeros(3)])
    rec = engine.Records()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2

    def step(sp, out=None):
        D, N, O = engine.forward(cam, pose12, sp, cfg, rec, sync=False)
        dD, dN, dO, parts = engine.mapping_loss(D, N, O, kf_range, kf_valid, kf_normal, kf_nvalid, w_opacity=0.0,
                                                w_normal=0.1)
        g = engine.backward(rec, sp, dD, dN, dO, raw_space=True, out=out)
        return g, parts

    engine.forward(cam, pose12, splats, cfg, rec)  # sizes the pair buffers (synchronous check)
    for _ in range(max(args.warmup, 3)):
        step(splats)
    torch.cuda.synchronize()
    assert rec.check(True) == 0
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.1)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    L.ss_records_profile(rec.ptr, 1)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    sampler.mark(0)
    for i in range(args.steps):
        flush.zero_()  # L2 flush between timed steps (outside the events)
        starts[i].record()
        step(splats)
        ends[i].record()
    torch.cuda.synchronize()
    sampler.mark(1)
    assert rec.check(True) == 0, "pair capacity exceeded inside the timed loop"
    L.ss_records_profile(rec.ptr, 0)
    ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    stage_ms = (ctypes.c_double * 8)()
    stage_n = (ctypes.c_int32 * 8)()
    L.ss_records_stage_times(rec.ptr, stage_ms, stage_n, 8)
    clocks = sampler.stop()
    if ws > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = ws * 1000.0 / ms_step

    # work counts (reference algorithm's units) for the roofline
    E = ctypes.c_int64(0)
    U = ctypes.c_int64(0)
    engine.forward(cam, pose12, splats, cfg, rec)
    L.ss_records_work(rec.ptr, ctypes.byref(E), ctypes.byref(U), ctypes.c_void_p(engine.stream_ptr()))
    n_pairs, _, _ = rec.counts()
    E, U, N = E.value, U.value, 500_000
    peak = ctypes.c_double(0.0)
    L.ss_fp32_peak_tflops(ctypes.byref(peak), ctypes.c_void_p(engine.stream_ptr()))
    stage = {STAGES[i]: (stage_ms[i] / max(stage_n[i], 1)) for i in range(8)}
    flops = {"forward": 46 * E + 34 * U, "backward": 46 * E + 170 * U}
    top = max(("forward", "backward"), key=lambda k: stage[k])
    achieved = flops[top] / (stage[top] * 1e-3) / 1e12
    step_flops = 92 * E + 204 * U + 300 * N
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "r01_traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(f"k_{top}<8>")
    roofline = {"bound": "fp32", "kernel": f"k_{top}<8>", "achieved": achieved, "peak": peak.value,
                "unit": "TFLOP/s", "frac": achieved / peak.value,
                "peak_source": "FFMA probe measured live (ss_fp32_peak_tflops); MEASURED_PEAKS.json has no FP32 figure",
                "algorithmic_flops_per_launch": flops[top],
                "traffic": traffic, "traffic_unit": "bytes/launch (ncu dram read+write, profiles/r01_traffic.json)",
                "units": {"E_pair_evaluations": E, "U_contributions": U, "TP_tile_pairs": n_pairs, "N_splats": N},
                "step_fraction": stage[top] / ms_step,
                "step_achieved_tflops": step_flops / (ms_step * 1e-3) / 1e12}

    # e2e: pinned host parameters -> device, step, gradients + loss back to the host.
    # Copies run on their own stream, double-buffered, so step k+1's upload and
    # step k-1's download overlap step k's kernels (the public engine API on the
    # compute stream; every byte still crosses PCIe inside the timed region).
    # the five parameter arrays packed in ONE pinned buffer (one DMA per step: a
    # single 24 MB copy each way runs both PCIe directions at ~92 GB/s together,
    # five separate uploads at ~76 GB/s, tools/pcie_probe.py)
    names = list(params_np.keys())
    sizes = [params_np[k].size for k in names]
    offs = np.concatenate([[0], np.cumsum(sizes)])
    host_flat = torch.empty(int(offs[-1]), dtype=torch.float32).pin_memory()
    for k, o, n_ in zip(names, offs[:-1], sizes):
        host_flat[o:o + n_] = torch.from_numpy(np.ascontiguousarray(params_np[k], dtype=np.float32).reshape(-1))
    dev_flat = [torch.empty_like(host_flat, device=dev) for _ in range(2)]
    dev_in = [{k: dev_flat[b][o:o + n_].view(params_np[k].shape) for k, o, n_ in zip(names, offs[:-1], sizes)}
              for b in range(2)]
    host = {"flat": host_flat}
    g_host = [torch.empty((500_000, 12), dtype=torch.float32).pin_memory() for _ in range(2)]
    loss_host = [torch.empty(4, dtype=torch.float64).pin_memory() for _ in range(2)]
    g_dev = [torch.empty((500_000, 12), dtype=torch.float32, device=dev) for _ in range(2)]
    parts_dev = [None, None]
    h2d = sum(v.numel() * v.element_size() for v in host.values())
    d2h = g_host[0].numel() * 4 + 4 * 8
    comp = torch.cuda.current_stream()
    copy = torch.cuda.Stream()   # host -> device
    copy_d = torch.cuda.Stream()  # device -> host (the other PCIe direction)
    up_done = [torch.cuda.Event() for _ in range(2)]
    step_done = [torch.cuda.Event() for _ in range(2)]
    down_done = [torch.cuda.Event() for _ in range(2)]

    def upload(i):
        b_ = i % 2
        with torch.cuda.stream(copy):
            copy.wait_event(step_done[b_])  # buffer b_ is free once step i-2 finished with it
            dev_flat[b_].copy_(host_flat, non_blocking=True)
            up_done[b_].record(copy)

    def download(i):
        b_ = i % 2
        with torch.cuda.stream(copy_d):
            copy_d.wait_event(step_done[b_])
            g_host[b_].copy_(g_dev[b_], non_blocking=True)
            loss_host[b_].copy_(parts_dev[b_], non_blocking=True)
            down_done[b_].record(copy_d)

    def e2e_run(n):
        upload(0)
        for i in range(n):
            b_ = i % 2
            if i + 1 < n:
                upload(i + 1)
            comp.wait_event(up_done[b_])
            if i >= 2:
                comp.wait_event(down_done[b_])  # step i-2's gradients have left g_dev[b_]
            _, parts = step(dev_in[b_], out=g_dev[b_])
            parts_dev[b_] = parts
            step_done[b_].record(comp)
            download(i)
        copy_d.synchronize()

    e2e_run(3)
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(copy)
    comp.wait_event(e0)
    e2e_run(args.steps)
    e1.record(copy_d)
    torch.cuda.synchronize()
    ems = e0.elapsed_time(e1)
    if ws > 1:
        t = torch.tensor([ems], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ems = float(t.item())
    e2e = {"value": ws * args.steps * 1000.0 / ems, "unit": UNIT, "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "overlap": "upload and download streams double-buffered against the compute stream"}

    secondary = None
    if rank == 0 and ws == 1 and not args.no_secondary:
        secondary = secondary_metrics(dev)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        t0 = time.perf_counter()
        oracle_render_step(cam, params_np, tgt)
        dt = time.perf_counter() - t0
        cpu = {"value": 1.0 / dt, "unit": UNIT, "cores": cpu_info(), "kind": "port",
               "sample": "1 full config-1 fwd+loss+bwd render, C float64 oracle (oracle/), all host threads"}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded, SURVEY 8(d)); independent map per rank",
                "config": {"workload": WORKLOAD, "renders_per_step": ws, "camera": "128x2048",
                           "splats_per_rank": 500_000, "parallelism": f"independent maps x{ws}",
                           "l2": "flushed between timed steps (256 MiB write outside the events)"},
                "clocks": clocks, "gpu_launches": KERNELS_PER_STEP * args.steps, "stage_ms": stage,
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "secondary": secondary}
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--warmup-ref", type=int, default=0)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    args = ap.parse_args()
    ws, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, ws, rank)
    else:
        run_b200(args, ws, rank, local)


if __name__ == "__main__":
    main()
