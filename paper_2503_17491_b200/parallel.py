"""Multi-GPU partitioning of the hot path.

One process per GPU (``torch.distributed``; NCCL over NVLink / NVSwitch on the
B200 box, gloo in the CPU tests).

* Independent local maps (config 4a): ``LocalMapShard`` owns the maps
  ``shard_maps`` assigns to this rank (map m -> rank m mod world).  A
  ``LocalMap`` is the reference's unit of optimisation and reset
  (mapping.py:383-409), so ranks never communicate on the
  data path; one ``step`` advances one of the rank's maps by one refine
  iteration (keyframe draw, render, loss, backward, Adam: mapping.py:455-498),
  round robin, so per-GPU work per step is fixed (weak scaling).
* Shared map, different keyframes (config 4b): ``SharedMapTrainer`` keeps one
  replica of the map per rank.  Every iteration all ranks draw the same
  ``world`` keyframe indices from an identically seeded sampler, rank r
  renders index r, and the raw-parameter gradients (n x 12 float32) are summed
  with an all-reduce.  The backward is split (``ss_render_backward_blend`` then
  ``ss_render_finalize`` per row chunk) so that the all-reduce of chunk c runs
  on the communicator's stream while chunk c+1 is still being finalized.
  Every rank then applies the identical fused Adam step, so the replicas stay
  bit-identical.  This changes the reference's optimiser semantics (one
  keyframe per iteration, mapping.py:475) to the sum over ``world`` keyframes
  per iteration.

The collective and sampler logic is backend-agnostic (``GradOps``) so it is
exercised on CPU with gloo in tests/test_parallel.py.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np
import torch
import torch.distributed as dist

from .mapping import MappingConfig, sample_keyframe_index

__all__ = ["shard_maps", "world_info", "row_chunks", "GradOps", "SharedMapTrainer", "device_ops", "LocalMapShard"]


def world_info(group=None):
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def shard_maps(n_maps: int, rank: int, world: int) -> list:
    """Maps owned by ``rank`` (config 4a: round robin, no communication)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside a world of {world}")
    return list(range(rank, n_maps, world))


def row_chunks(n: int, chunks: int, align: int = 128) -> list:
    """[begin, end) row ranges covering [0, n): ``chunks`` pieces, every begin a multiple of
    ``align`` (ss_render_finalize's vector alignment)."""
    if n <= 0:
        return []
    per = -(-n // max(chunks, 1))
    step = max(align, -(-per // align) * align)
    return [(b, min(b + step, n)) for b in range(0, n, step)]


@dataclass
class GradOps:
    """What one rank does per iteration of the shared-map trainer.

    blend(k)            render keyframe k, loss, blend backward (per-splat accumulators);
                        returns the loss parts
    finalize(b, e)      gradient rows [b, e) into ``grad``
    grad                (n, 12) gradient buffer (summed across ranks in place)
    adam(g)             in-place optimiser step with the summed gradient
    """
    blend: Callable[[int], object]
    finalize: Callable[[int, int], None]
    grad: torch.Tensor
    adam: Callable[[torch.Tensor], None]
    align: int = 128


class SharedMapTrainer:
    def __init__(self, ops: GradOps, n_keyframes: int, cfg: MappingConfig, seed: int, group=None,
                 chunks: int = 8):
        self.ops = ops
        self.n_kf = n_keyframes
        self.cfg = cfg
        self.rng = np.random.default_rng(seed)  # identical on every rank
        self.group = group
        self.chunks = chunks
        self.last_parts = None

    def draw(self, world: int) -> list:
        return [sample_keyframe_index(self.n_kf, self.cfg.kf_sample_p, self.rng) for _ in range(world)]

    def step(self) -> int:
        rank, world = world_info(self.group)
        picks = self.draw(world)
        self.last_parts = self.ops.blend(picks[rank])
        g = self.ops.grad
        work = []
        for b, e in row_chunks(int(g.shape[0]), self.chunks, self.ops.align):
            self.ops.finalize(b, e)
            if world > 1:  # the collective waits for this chunk only; the next finalize overlaps it
                work.append(dist.all_reduce(g[b:e], op=dist.ReduceOp.SUM, group=self.group, async_op=True))
        for w in work:
            w.wait()
        self.ops.adam(g)
        return picks[rank]


def device_ops(dmap, cfg: MappingConfig, raster=None, sync: bool = True) -> GradOps:
    """GradOps on the B200 kernels for a DeviceMap (parameters and Adam state on the device).
    ``sync=False`` skips the host wait on each forward's pair-capacity check (the caller
    reserved capacity and checks ``dmap.rec.check()`` afterwards)."""
    grad = torch.empty((dmap.n, 12), dtype=torch.float32, device=dmap.m.device)
    return GradOps(lambda k: dmap.blend_gradient(k, cfg, raster, sync=sync),
                   lambda b, e: dmap.finalize_rows(b, e, grad), grad,
                   lambda g: dmap.apply_adam(g, cfg))


class LocalMapShard:
    """Config 4a: the independent local maps this rank owns, optimised round robin.

    Each map's refine step (render, loss, backward, Adam) is a CUDA graph per
    keyframe (DeviceMap.begin_replay); the host only draws the keyframe index with
    the reference's sampler (mapping.py:441-452, 474) and replays."""

    def __init__(self, maps: list, cfg: MappingConfig, seed: int = 0, raster=None):
        self.maps = maps
        self.cfg = cfg
        self.raster = raster
        self.rngs = [np.random.default_rng(seed + i) for i in range(len(maps))]
        self.turn = 0

    def begin(self) -> None:
        for dm in self.maps:
            dm.begin_replay(self.cfg, self.raster)

    def step(self) -> int:
        """One refine iteration (mapping.py:474-497) of the next map; returns its index."""
        i = self.turn % len(self.maps)
        self.turn += 1
        dm = self.maps[i]
        dm.replay_step(sample_keyframe_index(len(dm.keyframes), self.cfg.kf_sample_p, self.rngs[i]))
        return i

    def end(self) -> bool:
        return all([dm.end_replay() for dm in self.maps])
