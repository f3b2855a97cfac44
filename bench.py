"""Benchmark: fwd+bwd spherical 2DGS renders/s at 128x2048 with 500k splats (BASELINE config 1).

One step = one forward render + fused mapping loss (range L1 + 0.1 normal,
mapping.py:128-151) + backward to the raw splat parameters, on the B200
kernels of libsplatb200.so.  Inputs are the seeded synthetic config-1 splats
(SURVEY 8(d)).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                  [--workload config1|config4a|config4b] [--dry-run]

Multi-GPU: ``--gpus N`` without a torchrun environment re-launches
this script under ``torch.distributed.run`` with N ranks (one per GPU, NCCL,
NCCL_DEBUG=INFO).  Workloads:
  config1   every rank renders its own independent config-1 map (seed 1 + rank):
            weak scaling, no data-path collective; the headline at every N.
  config4a  independent local maps (BASELINE config 4): 8 maps of 500k surfels
            with 10 keyframes at 128x2048, map m on rank m mod N; one step = one
            refine iteration (render, loss, backward, Adam) of one of the rank's
            maps, round robin: weak scaling, no collective.
  config4b  one shared 2M-surfel map; every rank renders a different keyframe,
            the raw gradients are summed by NCCL all-reduce chunk by chunk behind
            the finalize, every rank applies the same Adam step.
At N > 1 the config1 line carries config4a and config4b as ``multi``; at N = 1
the secondary metrics (configs 0, 2, 3 and the 1-GPU points of 4a / 4b) ride
along under ``secondary``.

``--impl reference`` times the CPU oracle port of the reference's algorithm
(oracle/, float64, all host threads) on the same config and metric.
``--dry-run`` (CPU, gloo) exercises the launcher, rendezvous, barriers and the
max-over-ranks timing without a GPU.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import platform
import socket
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
N_MAPS = 8  # BASELINE config 4


def config_block(ws: int) -> dict:
    """The ``config`` of both arms (identical, so the driver can pair them)."""
    return {"workload": WORKLOAD, "renders_per_step": ws, "camera": "128x2048", "splats_per_rank": 500_000,
            "parallelism": f"independent maps x{ws}",
            "l2": "flushed between timed steps (256 MiB write outside the events)"}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch(n: int) -> None:
    """Re-exec this script under torch.distributed.run with n ranks on this node."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    os.execvpe(cmd[0], cmd, env)


def host_info() -> dict:
    """CPU model, cores and numeric library versions of the host the CPU baseline runs on."""
    model = platform.processor() or ""
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=5).stdout.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    import scipy
    return {"cpu_model": model, "os_cpu_count": os.cpu_count(), "numpy": np.__version__, "scipy": scipy.__version__,
            "OMP_NUM_THREADS": os.environ.get("OMP_NUM_THREADS"),
            "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS")}


# --- CPU oracle legs (cpu_baseline and --impl reference only) ------------------------------

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


def cpu_threads():
    from oracle import oracle as O
    return O.num_threads()


def cpu_refine_iterations(dm, targets, cfg, iters: int):
    """Seconds per refine iteration of the oracle (C render/backward + numpy loss and Adam,
    mapping_oracle.refine_iteration) on a host copy of the device map ``dm``."""
    from oracle import mapping_oracle as MO
    x = MO.flat({k: v.detach().cpu().numpy().astype(np.float64) for k, v in dm.params.items()})
    opt = MO.Adam(x.shape[0], cfg, dm.scene_scale)
    rng = np.random.default_rng(0)
    from paper_2503_17491_b200.mapping import sample_keyframe_index
    t0 = time.perf_counter()
    for _ in range(iters):
        cam, pose, tg = targets[sample_keyframe_index(len(targets), cfg.kf_sample_p, rng)]
        ct = (cam.width, cam.height, cam.az_min, cam.az_max, cam.el_min, cam.el_max)
        kf = {k: np.asarray(tg[k]) for k in ("range", "valid", "normal", "nvalid")}
        kf = {"range": kf["range"].astype(np.float64), "valid": kf["valid"].astype(bool),
              "normal": kf["normal"].astype(np.float64), "nvalid": kf["nvalid"].astype(bool)}
        MO.refine_iteration(x, opt, ct, pose.rotation, pose.translation, kf, cfg)
    return (time.perf_counter() - t0) / iters


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
                                          "--format=csv,noheader,nounits", "-lms", "10"], stdout=subprocess.PIPE,
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


# --- device helpers -------------------------------------------------------------------------

def _events(n):
    import torch
    return [torch.cuda.Event(enable_timing=True) for _ in range(n)]


def max_over_ranks(x: float, ws: int, dev) -> float:
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws: int):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def fp32_peak():
    from paper_2503_17491_b200 import _lib, engine
    peak = ctypes.c_double(0.0)
    _lib.lib().ss_fp32_peak_tflops(ctypes.byref(peak), ctypes.c_void_p(engine.stream_ptr()))
    return peak.value


def work_counts(rec):
    """(E, U, TP) of the last forward on ``rec`` (the reference algorithm's units)."""
    from paper_2503_17491_b200 import _lib, engine
    E = ctypes.c_int64(0)
    U = ctypes.c_int64(0)
    _lib.lib().ss_records_work(rec.ptr, ctypes.byref(E), ctypes.byref(U), ctypes.c_void_p(engine.stream_ptr()))
    return E.value, U.value, rec.counts()[0]


def map_work(dm, raster):
    """Mean (E, U, TP) over the keyframes of a DeviceMap: its refine iteration's algorithmic work."""
    from paper_2503_17491_b200 import engine
    from paper_2503_17491_b200.geometry import pose_rt
    tot = np.zeros(3)
    for kf in dm.keyframes:
        engine.forward(kf.camera, pose_rt(kf.pose), dm.params, raster, dm.rec)
        tot += np.array(work_counts(dm.rec), dtype=np.float64)
    return tot / max(len(dm.keyframes), 1)


# Our kernels per config-1 step (launch list profiles/r02_v3_step_launches.csv): forward
# k_tile_intervals, k_preprocess, k_scan_blocks, k_emit, k_tile_hist_blocks, k_tile_prefix,
# k_scan_tiles, k_tile_scatter, k_tile_sort_big + k_tile_order (side stream; the order kernel
# also lists the backward's slots), k_tile_sort,
# k_forward_long (side; tail lists only), k_forward, k_publish_totals (side); k_mapping_loss;
# backward k_backward, k_finalize.  (Plus torch fills that are not ours.)
KERNELS_PER_STEP = 17


# --- config 1 (headline) ----------------------------------------------------------------------

def bench_config1(args, ws, rank, local, dev):
    import torch

    from paper_2503_17491_b200 import _lib, engine
    from paper_2503_17491_b200 import workloads as W
    from paper_2503_17491_b200.rasterizer import RasterConfig

    L = _lib.lib()
    cam = W.synth_camera(2048, 128)
    params_np = W.random_splats(500_000, 1 + rank)  # rank r optimises its own independent map
    tgt = W.target_images(W.Scene(0), cam)
    splats = {k: torch.from_numpy(v).to(dev) for k, v in params_np.items()}
    kf = [torch.from_numpy(np.asarray(tgt[k]).astype(t)).to(dev)
          for k, t in (("range", np.float32), ("valid", np.uint8), ("normal", np.float32), ("nvalid", np.uint8))]
    cfg = RasterConfig()
    pose12 = np.concatenate([np.eye(3).reshape(9), np.zeros(3)])
    rec = engine.Records()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2

    def step(sp, out=None):
        D, N, O = engine.forward(cam, pose12, sp, cfg, rec, sync=False)
        dD, dN, dO, parts = engine.mapping_loss(D, N, O, *kf, w_opacity=0.0, w_normal=0.1)
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
    starts, ends = _events(args.steps), _events(args.steps)
    barrier(ws)
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
    ms = max_over_ranks(sum(s.elapsed_time(e) for s, e in zip(starts, ends)), ws, dev)
    clocks = sampler.stop()
    # per-stage split from a separate pass with the stage events on (they sit between the
    # kernels and turn off programmatic dependent launch, so not inside the timed loop)
    L.ss_records_profile(rec.ptr, 1)
    for i in range(max(5, min(args.steps, 20))):
        flush.zero_()
        step(splats)
    torch.cuda.synchronize()
    L.ss_records_profile(rec.ptr, 0)
    stage_ms = (ctypes.c_double * 8)()
    stage_n = (ctypes.c_int32 * 8)()
    L.ss_records_stage_times(rec.ptr, stage_ms, stage_n, 8)
    ms_step = ms / args.steps
    value = ws * 1000.0 / ms_step

    # roofline of the dominant kernel, in the reference algorithm's work units
    engine.forward(cam, pose12, splats, cfg, rec)
    E, U, n_pairs = work_counts(rec)
    N = 500_000
    peak = fp32_peak()
    stage = {STAGES[i]: (stage_ms[i] / max(stage_n[i], 1)) for i in range(8)}
    flops = {"forward": 46 * E + 34 * U, "backward": 46 * E + 170 * U}
    top = max(("forward", "backward"), key=lambda k: stage[k])
    achieved = flops[top] / (stage[top] * 1e-3) / 1e12
    step_flops = 92 * E + 204 * U + 300 * N
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "r02_traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(f"k_{top}<8>")
    roofline = {"bound": "fp32", "kernel": f"k_{top}<8>", "achieved": achieved, "peak": peak,
                "unit": "TFLOP/s", "frac": achieved / peak,
                "peak_source": "FFMA probe measured live (ss_fp32_peak_tflops); MEASURED_PEAKS.json has no FP32 figure",
                "algorithmic_flops_per_launch": flops[top],
                "traffic": traffic, "traffic_unit": "bytes/launch (ncu dram read+write, profiles/r02_traffic.json)",
                "units": {"E_pair_evaluations": E, "U_contributions": U, "TP_tile_pairs": n_pairs, "N_splats": N},
                "step_fraction": stage[top] / ms_step,
                "step_achieved_tflops": step_flops / (ms_step * 1e-3) / 1e12,
                "step_frac": step_flops / (ms_step * 1e-3) / 1e12 / peak}

    # e2e: pinned host parameters -> device, step, gradients + loss back to the host.
    # Copies run on their own streams, double-buffered, so step k+1's upload and step
    # k-1's download overlap step k's kernels; every byte crosses PCIe inside the timed
    # region.  The five parameter arrays are packed in ONE pinned buffer (one DMA per
    # direction per step).
    names = list(params_np.keys())
    sizes = [params_np[k].size for k in names]
    offs = np.concatenate([[0], np.cumsum(sizes)])
    host_flat = torch.empty(int(offs[-1]), dtype=torch.float32).pin_memory()
    for k, o, n_ in zip(names, offs[:-1], sizes):
        host_flat[o:o + n_] = torch.from_numpy(np.ascontiguousarray(params_np[k], dtype=np.float32).reshape(-1))
    dev_flat = [torch.empty_like(host_flat, device=dev) for _ in range(2)]
    dev_in = [{k: dev_flat[b][o:o + n_].view(params_np[k].shape) for k, o, n_ in zip(names, offs[:-1], sizes)}
              for b in range(2)]
    g_host = [torch.empty((500_000, 12), dtype=torch.float32).pin_memory() for _ in range(2)]
    loss_host = [torch.empty(4, dtype=torch.float64).pin_memory() for _ in range(2)]
    g_dev = [torch.empty((500_000, 12), dtype=torch.float32, device=dev) for _ in range(2)]
    parts_dev = [None, None]
    h2d = host_flat.numel() * 4
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
    barrier(ws)
    e0, e1 = _events(2)
    e0.record(copy)
    comp.wait_event(e0)
    e2e_run(args.steps)
    e1.record(copy_d)
    torch.cuda.synchronize()
    ems = max_over_ranks(e0.elapsed_time(e1), ws, dev)
    e2e = {"value": ws * args.steps * 1000.0 / ems, "unit": UNIT, "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "api": "engine.forward / mapping_loss / backward (C-ABI) on pinned buffers",
           "overlap": "upload and download streams double-buffered against the compute stream"}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded, SURVEY 8(d)); independent map per rank",
            "config": config_block(ws), "clocks": clocks, "gpu_launches": KERNELS_PER_STEP * args.steps,
            "stage_ms": stage, "roofline": roofline, "e2e": e2e}
    return line, (cam, params_np, tgt)


def e2e_reference_api(cam, params_np, tgt, steps: int):
    """The same metric through the reference-signature drop-in: rasterize_forward(cam, pose,
    SplatModel) and rasterize_backward(model, records, render, PixelGradients) with a host
    float64 SplatModel in and float64 numpy SplatGradients out.  Every step touches the model
    (a new version) so its parameters are converted and uploaded again, as a caller that
    edits the model between renders would; the pixel gradients are fixed host arrays
    (the loss itself is the caller's numpy code, not timed)."""
    import torch

    from paper_2503_17491_b200 import PixelGradients, SE3Pose, SplatModel, rasterize_backward, rasterize_forward
    model = SplatModel.from_params({k: v.astype(np.float64) for k, v in params_np.items()})
    pose = SE3Pose.identity()
    rng = np.random.default_rng(0)
    pg = PixelGradients(np.sign(rng.normal(size=(cam.height, cam.width))),
                        0.1 * rng.normal(size=(cam.height, cam.width, 3)),
                        0.05 * rng.normal(size=(cam.height, cam.width)))

    def one():
        model.touch()
        out, rec = rasterize_forward(cam, pose, model)
        g = rasterize_backward(model, rec, out, pg)
        return out.range, g.d_centers

    for _ in range(3):
        one()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    dt = (time.perf_counter() - t0) / steps
    n = len(model)
    return {"value": 1.0 / dt, "unit": UNIT, "ms_per_step": dt * 1e3,
            "h2d_bytes_per_step": n * 12 * 4 + cam.width * cam.height * 5 * 4,
            "d2h_bytes_per_step": n * 15 * 4 + cam.width * cam.height * 4,
            "api": "rasterize_forward / rasterize_backward (reference signatures, host float64 in and out)",
            "note": "wall clock per step (the host conversions are the cost being measured); "
                    "range image and the plain-space gradients materialised as float64 numpy"}


# --- config 4: independent maps and the shared map --------------------------------------------

def _config4_keyframes(dev):
    from paper_2503_17491_b200 import workloads as W
    targets = W.keyframe_targets(10, 0, 2048, 128)
    return targets, W.device_keyframes(targets)


def bench_config4a(args, ws, rank, dev, want_cpu=False):
    """BASELINE config 4 (independent maps): 8 maps x 500k surfels x 10 keyframes at 128x2048,
    grown the reference's way (start + 9 add_keyframe, 50k spawned per keyframe, map seed m),
    map m on rank m mod N (parallel.shard_maps), refined round robin by CUDA-graph replay."""
    import torch

    from paper_2503_17491_b200 import workloads as W
    from paper_2503_17491_b200.mapping import MappingConfig
    from paper_2503_17491_b200.parallel import LocalMapShard, shard_maps
    from paper_2503_17491_b200.rasterizer import RasterConfig

    t_build = time.perf_counter()
    targets, dkfs = _config4_keyframes(dev)
    owned = shard_maps(N_MAPS, rank, ws)
    maps = [W.build_local_map(dkfs, 50_000, m) for m in owned]
    cfg = MappingConfig(w_opacity=0.05, w_normal=0.1)
    shard = LocalMapShard(maps, cfg, seed=100 * rank)
    shard.begin()
    for _ in range(max(args.warmup, 3) * len(maps)):
        shard.step()
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t_build
    K = max(args.steps, len(maps))
    barrier(ws)
    torch.cuda.synchronize()
    e0, e1 = _events(2)
    e0.record()
    for _ in range(K):
        shard.step()
    e1.record()
    torch.cuda.synchronize()
    ok = shard.end()
    ms = max_over_ranks(e0.elapsed_time(e1), ws, dev)
    E, U, TP = map_work(maps[0], RasterConfig())
    n = maps[0].n
    F = 92 * E + 204 * U + 300 * n
    peak = fp32_peak()
    out = {"metric": "config-4a map-iterations/s (refine iteration = fwd+loss+bwd+Adam, 128x2048, 500k surfels)",
           "value": ws * K * 1000.0 / ms, "unit": "map-iterations/s", "n_gpus": ws, "steps": K,
           "ms_per_step": ms / K, "scaling": "weak", "maps_total": N_MAPS, "maps_per_rank": len(maps),
           "splats_per_map": [m.n for m in maps], "keyframes_per_map": len(dkfs), "capacity_ok": ok,
           "roofline": {"bound": "fp32", "algorithmic_flops_per_iteration": F,
                        "units_map0": {"E": E, "U": U, "TP": TP, "N": n},
                        "achieved_tflops_per_gpu": F / (ms / K * 1e-3) / 1e12,
                        "frac": F / (ms / K * 1e-3) / 1e12 / peak, "peak": peak},
           "setup_s": build_s,
           "note": "map m on rank m mod N; no data-path collective; max over ranks of the device time"}
    if want_cpu:
        t_it = cpu_refine_iterations(maps[0], targets, cfg, 1)
        out["cpu_baseline"] = {"value": 1.0 / t_it, "unit": "map-iterations/s", "cores": cpu_threads(),
                               "kind": "port", "sample": "1 refine iteration of map 0 (C oracle render+backward, "
                                                         "numpy loss + Adam), all host threads"}
    del shard, maps
    torch.cuda.empty_cache()
    return out


def bench_config4b(args, ws, rank, dev):
    """BASELINE config 4 variant: one shared 2M-surfel map (the union of four config-4a maps);
    each rank renders a different keyframe per iteration, the n x 12 raw gradients are summed
    by NCCL all-reduce chunk by chunk behind the finalize (parallel.SharedMapTrainer), and
    every rank applies the same Adam step."""
    import torch
    import torch.distributed as dist

    from paper_2503_17491_b200 import workloads as W
    from paper_2503_17491_b200.mapping import MappingConfig
    from paper_2503_17491_b200.parallel import SharedMapTrainer, device_ops, row_chunks
    from paper_2503_17491_b200.rasterizer import RasterConfig

    t_build = time.perf_counter()
    targets, dkfs = _config4_keyframes(dev)
    parts = [W.build_local_map(dkfs, 50_000, m) for m in range(4)]
    dm = W.merge_maps(parts, dkfs)
    del parts
    cfg = MappingConfig(w_opacity=0.05, w_normal=0.1)
    raster = RasterConfig()
    # size the shared records for every keyframe (the steps below do not wait on the host)
    most = 0
    from paper_2503_17491_b200 import _lib, engine
    from paper_2503_17491_b200.geometry import pose_rt
    for kf in dkfs:
        engine.forward(kf.camera, pose_rt(kf.pose), dm.params, raster, dm.rec)
        most = max(most, dm.rec.counts()[0])
    _lib.lib().ss_records_reserve(dm.rec.ptr, 2 * most + 65536)
    tr = SharedMapTrainer(device_ops(dm, cfg, raster, sync=False), len(dkfs), cfg, seed=1234, chunks=8)
    for _ in range(max(args.warmup, 3)):
        tr.step()
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t_build
    K = args.steps
    barrier(ws)
    torch.cuda.synchronize()
    e0, e1 = _events(2)
    e0.record()
    for _ in range(K):
        tr.step()
    e1.record()
    torch.cuda.synchronize()
    ok = dm.rec.check(True) == 0
    ms = max_over_ranks(e0.elapsed_time(e1), ws, dev)
    g = tr.ops.grad
    nbytes = g.numel() * g.element_size()
    ar = None
    if ws > 1:  # the all-reduce alone, same buffer and chunking
        barrier(ws)
        a0, a1 = _events(2)
        a0.record()
        for _ in range(K):
            work = [dist.all_reduce(g[b:e], async_op=True) for b, e in row_chunks(int(g.shape[0]), 8)]
            for w in work:
                w.wait()
        a1.record()
        torch.cuda.synchronize()
        t_ar = max_over_ranks(a0.elapsed_time(a1), ws, dev) / K
        ar = {"ms": t_ar, "bytes": nbytes, "algbw_gbs": nbytes / (t_ar * 1e-3) / 1e9,
              "busbw_gbs": 2 * (ws - 1) / ws * nbytes / (t_ar * 1e-3) / 1e9,
              "busbw_peak_gbs": 725.0, "peak_source": "NVLink 5 bus bandwidth (SURVEY 8(e))"}
    E, U, TP = map_work(dm, raster)
    F = 92 * E + 204 * U + 300 * dm.n
    peak = fp32_peak()
    return {"metric": "config-4b keyframe renders/s on one shared 2M-surfel map (fwd+loss+bwd, summed "
                      "gradient all-reduce, Adam)", "value": ws * K * 1000.0 / ms, "unit": "frames/s",
            "n_gpus": ws, "steps": K, "ms_per_step": ms / K, "scaling": "weak", "splats": dm.n,
            "gradient_bytes": nbytes, "capacity_ok": ok, "allreduce_alone": ar,
            "roofline": {"bound": "fp32", "algorithmic_flops_per_iteration": F,
                         "units": {"E": E, "U": U, "TP": TP, "N": dm.n},
                         "achieved_tflops_per_gpu": F / (ms / K * 1e-3) / 1e12,
                         "frac": F / (ms / K * 1e-3) / 1e12 / peak, "peak": peak},
            "setup_s": build_s,
            "note": "one keyframe per rank per iteration: the optimiser sees the sum over N keyframes "
                    "(the reference steps on one, mapping.py:475)"}


# --- secondary metrics at N = 1 ---------------------------------------------------------------

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
    E, U, TP = work_counts(rec)
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
    e0, e1 = _events(2)
    e0.record()
    for _ in range(replays):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / replays
    assert rec.check(True) == 0, "pair capacity exceeded during the graph replays"
    eager = []
    for _ in range(20):
        a, b = _events(2)
        a.record()
        step()
        b.record()
        eager.append((a, b))
    torch.cuda.synchronize()
    ms_eager = sum(a.elapsed_time(b) for a, b in eager) / len(eager)
    N = 50_000
    F = 92 * E + 204 * U + 300 * N
    peak = fp32_peak()
    t0 = time.perf_counter()
    oracle_render_step(cam, c["splats"], tgt)
    cpu_s = time.perf_counter() - t0
    return {"metric": "config-0 fwd+bwd renders/s, CUDA-graph replay (64x1024, 50k splats, fp32)",
            "value": 1000.0 / ms, "unit": "renders/s", "ms_per_render": ms, "eager_ms_per_render": ms_eager,
            "replays": replays, "pairs": TP,
            "roofline": {"bound": "fp32", "units": {"E": E, "U": U, "TP": TP, "N": N},
                         "algorithmic_flops": F, "achieved_tflops": F / (ms * 1e-3) / 1e12,
                         "frac": F / (ms * 1e-3) / 1e12 / peak, "peak": peak,
                         "note": "launch-bound: ~0.6 GFLOP per render"},
            "cpu_baseline": {"value": 1.0 / cpu_s, "unit": "renders/s", "cores": cpu_threads(), "kind": "port",
                             "sample": "1 config-0 fwd+loss+bwd render, C float64 oracle, all host threads"},
            "note": "forward + mapping loss + backward to raw parameters captured once, replayed back to back"}


def mapping_config2(dev):
    """BASELINE config 2: the map grown the reference's way on the device (LocalMap.start +
    9 x add_keyframe, 20k spawned per keyframe = 200k surfels), then 100 Adam
    refine iterations (CUDA-graph replay per keyframe)."""
    import torch

    from paper_2503_17491_b200 import engine
    from paper_2503_17491_b200 import mapping as MP
    from paper_2503_17491_b200 import workloads as W
    from paper_2503_17491_b200.geometry import pose_rt

    targets = W.keyframe_targets(10, 0, 1024, 64)
    dkfs = W.device_keyframes(targets)
    cfg = MP.MappingConfig(w_opacity=0.05, w_normal=0.1)
    t_build = time.perf_counter()
    W.build_local_map(dkfs, 20_000, 0).refine(cfg, 5, np.random.default_rng(1))  # warm-up on a throwaway map
    torch.cuda.synchronize()
    t_build = time.perf_counter()
    dm = W.build_local_map(dkfs, 20_000, 0)
    torch.cuda.synchronize()
    build_ms = (time.perf_counter() - t_build) * 1e3
    E, U, TP = map_work(dm, MP.RasterConfig())
    dm.capture_graphs(cfg)  # one CUDA graph per keyframe step (capture executes nothing)
    rng = np.random.default_rng(0)

    def depth_rmse():
        """(rendered range D, and D / O on pixels with O > 0.5 as sample_model reads depth) vs the
        keyframe range over its valid pixels, all keyframes."""
        se, cnt, se2, cnt2 = 0.0, 0, 0.0, 0
        for kf in dkfs:
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
        e0, e1 = _events(2)
        e0.record()
        ls = dm.refine(cfg, iters, rng)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
        if rep == 0:
            losses = ls
            rmse1 = depth_rmse()
    ms = statistics.median(times)
    F = 92 * E + 204 * U + 300 * dm.n
    peak = fp32_peak()
    t_it = cpu_refine_iterations(dm, targets, cfg, 2)
    fx = np.load(os.path.join(ROOT, "tests", "golden", "golden_quality.npz"))
    q = W.quality_run(fx)
    reduced = {"config": "reference's reduced config-2 run (tests/golden/golden_quality.npz): 512x32, "
                         f"{int(fx['n_keyframes'])} keyframes, n_spawn {int(fx['n_spawn'])}, {int(fx['iters'])} "
                         "refine iterations, same images and seeds on both sides",
               "reference": {"splats": int(fx["n_built"]), "rmse_m_before": float(fx["rmse_before"][0]),
                             "rmse_m_after": float(fx["rmse_after"][0]),
                             "confident_rmse_m_before": float(fx["rmse_before"][1]),
                             "confident_rmse_m_after": float(fx["rmse_after"][1]),
                             "loss_first": float(fx["losses"][0]), "loss_last": float(fx["losses"][-1]),
                             "refine_s_per_iteration_numpy_1core": float(fx["ref_refine_s_per_iter"])},
               "ours": {"splats": q["splats"], "rmse_m_before": q["rmse_before"][0], "rmse_m_after": q["rmse_after"][0],
                        "confident_rmse_m_before": q["rmse_before"][1], "confident_rmse_m_after": q["rmse_after"][1],
                        "loss_first": q["loss_first"], "loss_last": q["loss_last"]}}
    return {"metric": "mapping frames/s (refine iterations: render+loss+backward+Adam)",
            "value": iters * 1000.0 / ms, "unit": "frames/s", "iterations": iters, "splats": dm.n,
            "timed_runs_ms": times, "map_build_ms": build_ms,
            "keyframes": len(dkfs), "camera": "64x1024", "loss_first": losses[0], "loss_last": losses[-1],
            "depth_rmse_m_before": rmse0[0], "depth_rmse_m_after": rmse1[0],
            "confident_depth_rmse_m_before": rmse0[1], "confident_depth_rmse_m_after": rmse1[1],
            "confident_fraction_after": rmse1[2],
            "quality_vs_reference": reduced,
            "roofline": {"bound": "fp32", "units_mean_per_keyframe": {"E": E, "U": U, "TP": TP, "N": dm.n},
                         "algorithmic_flops_per_iteration": F,
                         "achieved_tflops": F / (ms / iters * 1e-3) / 1e12,
                         "frac": F / (ms / iters * 1e-3) / 1e12 / peak, "peak": peak},
            "cpu_baseline": {"value": 1.0 / t_it, "unit": "frames/s", "cores": cpu_threads(), "kind": "port",
                             "sample": "2 refine iterations of the same map (C oracle render + backward, numpy "
                                       "loss + Adam), all host threads",
                             "extrapolated_100_iterations_s": 100 * t_it},
            "note": "config 2: 200k surfels grown by DeviceMap.start + 9 add_keyframe (mapping.py:392-438) "
                    "from 10 keyframes; depth RMSE = rendered range D vs keyframe range over valid pixels; "
                    "confident: D / O where O > 0.5 (sample_model's depth)"}


def registration_config3(dev):
    import torch

    from paper_2503_17491_b200 import engine
    from paper_2503_17491_b200 import registration as REG
    from paper_2503_17491_b200 import workloads as W

    out = {}
    params, cam, scan, truth, initial = W.config3_problem()
    dparams = engine.as_device_params(params)  # the fixed map stays resident in HBM across registrations
    rcfg = REG.RegistrationConfig(mode="photometric", max_iters=20, tol=0.0)
    res = REG.register(dparams, scan, cam, initial, rcfg)  # warm-up (allocations)
    torch.cuda.synchronize()
    reps = 5
    t0 = time.perf_counter()
    for _ in range(reps):
        res = REG.register(dparams, scan, cam, initial, rcfg)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    err_t = float(np.linalg.norm(res.pose.translation - truth.translation))
    cosang = (np.trace(res.pose.rotation.T @ truth.rotation) - 1) / 2
    err_r = float(np.degrees(np.arccos(np.clip(cosang, -1, 1))))
    e0t = float(np.linalg.norm(initial.translation - truth.translation))
    # CPU baseline: the oracle's sample_model (C float64 2x render) + the oracle GN/LM loop
    from oracle import registration_oracle as RO
    geo = (cam.width * 2, cam.height * 2, cam.az_min, cam.az_max, cam.el_min, cam.el_max)
    ct = (cam.width, cam.height, cam.az_min, cam.az_max, cam.el_min, cam.el_max)
    p64 = {k: v.astype(np.float64) for k, v in params.items()}
    t0 = time.perf_counter()
    X = RO.sample_model(p64, geo, initial.rotation, initial.translation, 0.5, 0.5)[::4]
    rimg, valid = RO.build_range_image(ct, scan)
    RO.register_photometric(X, rimg, valid, ct, initial.rotation, initial.translation, max_iters=20, tol=0.0)
    cpu_s = time.perf_counter() - t0
    out["registration"] = {"metric": "photometric registrations/s (2x render + 20 GN iterations)",
                           "value": 1.0 / dt, "unit": "registrations/s", "ms": dt * 1e3, "iterations": res.iterations,
                           "n_photo": res.n_photo, "initial_err_m": e0t, "final_err_m": err_t, "final_err_deg": err_r,
                           "cpu_baseline": {"value": 1.0 / cpu_s, "unit": "registrations/s", "cores": cpu_threads(),
                                            "kind": "port", "sample": "1 registration: oracle sample_model (C "
                                            "float64 2x render) + numpy GN/LM loop, 20 iterations"},
                           "note": "config 3: 300k surfels on visible surfaces (device-resident map); per "
                                   "registration: 2x render + anchors, scan range image, GN/LM loop in one "
                                   "cooperative kernel; latency-bound (see DESIGN 5b)"}
    # frame batches: B independent photometric registrations at once (register_batch: one
    # C-ABI call, B streams, B concurrent cooperative loops with num_SMs / B blocks each)
    bparams, bcam, bscans, btruths, binit = W.config3_frames(8)
    bdp = engine.as_device_params(bparams)
    bscans_dev = [torch.as_tensor(sc, device=dev) for sc in bscans]
    for _ in range(2):
        REG.register_batch(bdp, bscans_dev, bcam, binit, rcfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        bres = REG.register_batch(bdp, bscans_dev, bcam, binit, rcfg)
    torch.cuda.synchronize()
    dtb = (time.perf_counter() - t0) / reps
    for _ in range(2):
        REG.register(bdp, bscans[0], bcam, binit[0], rcfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for f in range(8):
        REG.register(bdp, bscans[f], bcam, binit[f], rcfg)
    torch.cuda.synchronize()
    dt1 = (time.perf_counter() - t0) / 8
    out["registration_batch8"] = {
        "metric": "photometric registrations/s, 8 frames per register_batch call (config-3 map, 20 GN iterations)",
        "value": 8 / dtb, "unit": "registrations/s", "ms_per_batch": dtb * 1e3, "single_frame_value": 1.0 / dt1,
        "speedup_vs_single": dt1 * 8 / dtb,
        "max_final_err_m": max(float(np.abs(r.pose.translation - t.translation).max()) for r, t in zip(bres, btruths)),
        "note": "frames ray-cast at 8 true poses 0.25 m apart, initial poses perturbed by 0.2 m / 2 deg; scans "
                "device-resident; per-frame results equal register() (tests/test_gpu_registration.py)"}
    scfg = REG.RegistrationConfig()  # the reference's default mode: sequential
    res = REG.register(dparams, scan, cam, initial, scfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        res = REG.register(dparams, scan, cam, initial, scfg)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    out["registration_sequential"] = {
        "metric": "sequential registrations/s (default RegistrationConfig: leaf tree + geometric then joint)",
        "value": 1.0 / dt, "unit": "registrations/s", "ms": dt * 1e3, "iterations": res.iterations,
        "converged": res.converged, "n_geo": res.n_geo, "n_photo": res.n_photo,
        "final_err_m": float(np.linalg.norm(res.pose.translation - truth.translation))}
    return out


def secondary_metrics(args, dev, cam, params_np, tgt):
    out = {"config0_graph": config0_graph(dev), "mapping": mapping_config2(dev)}
    out.update(registration_config3(dev))
    out["e2e_reference_api"] = e2e_reference_api(cam, params_np, tgt, max(args.steps // 4, 5))
    out["config4a_1gpu"] = bench_config4a(args, 1, 0, dev, want_cpu=True)
    out["config4b_1gpu"] = bench_config4b(args, 1, 0, dev)
    return out


# --- arms ----------------------------------------------------------------------------------------

def run_reference(args, ws, rank):
    """--impl reference: the CPU oracle port on the box's host cores (rank 0 only)."""
    if rank != 0:
        return
    from paper_2503_17491_b200 import workloads as W
    c = W.config(1)
    cam, params = c["camera"], c["splats"]
    tgt = W.target_images(W.Scene(0), cam)
    cores = cpu_threads()
    for _ in range(args.warmup):
        oracle_render_step(cam, params, tgt)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle_render_step(cam, params, tgt)
    dt = time.perf_counter() - t0
    v = args.steps / dt
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, SURVEY 8(d))",
            "config": config_block(ws),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "host": host_info(),
                             "sample": "full config-1 fwd+loss+bwd render per step, C float64 oracle (oracle/)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_dry(args, ws, rank):
    """Harness check without a GPU: gloo rendezvous, barriers, max-over-ranks timing, one JSON line."""
    import torch
    import torch.distributed as dist
    if ws > 1:
        dist.init_process_group("gloo")
    x = np.random.default_rng(rank).normal(size=(192, 192))
    for _ in range(args.warmup):
        x @ x
    if ws > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        x @ x
    dt = time.perf_counter() - t0
    if ws > 1:
        t = torch.tensor([dt], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"dry_run": True, "metric": METRIC, "value": ws * args.steps / dt, "unit": "steps/s",
                          "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "backend": "gloo",
                          "note": "harness check only: a host matmul stands in for the step (no GPU work)"}),
              flush=True)


def run_b200(args, ws, rank, local):
    import torch

    from paper_2503_17491_b200 import _lib

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        dist.init_process_group("nccl", device_id=dev)
    _lib.lib()
    workload = args.workload
    if workload == "config1":
        line, (cam, params_np, tgt) = bench_config1(args, ws, rank, local, dev)
        if ws > 1 and not args.no_secondary:
            line["multi"] = {"config4a": bench_config4a(args, ws, rank, dev),
                             "config4b": bench_config4b(args, ws, rank, dev)}
        if rank == 0 and ws == 1 and not args.no_secondary:
            line["secondary"] = secondary_metrics(args, dev, cam, params_np, tgt)
        if rank == 0 and ws == 1 and not args.no_cpu_baseline:
            t0 = time.perf_counter()
            oracle_render_step(cam, params_np, tgt)
            dt = time.perf_counter() - t0
            line["cpu_baseline"] = {"value": 1.0 / dt, "unit": UNIT, "cores": cpu_threads(), "kind": "port",
                                    "host": host_info(),
                                    "sample": "1 full config-1 fwd+loss+bwd render, C float64 oracle (oracle/), "
                                              "all host threads"}
    else:
        fn = bench_config4a if workload == "config4a" else bench_config4b
        line = fn(args, ws, rank, dev)
        line.update({"higher_is_better": True, "warmup": max(args.warmup, 3), "dtype": "f32",
                     "data": "synthetic (seeded, SURVEY 8(d))", "vs_baseline": None,
                     "config": {"workload": workload}})
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="config1", choices=["config1", "config4a", "config4b"])
    ap.add_argument("--dry-run", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch(args.gpus)  # does not return
    ws, rank, local = dist_env()
    if ws != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}")
    if args.dry_run:
        run_dry(args, ws, rank)
    elif args.impl == "reference":
        run_reference(args, ws, rank)
    else:
        run_b200(args, ws, rank, local)


if __name__ == "__main__":
    main()
