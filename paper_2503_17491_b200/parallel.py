"""Multi-GPU partitioning of the hot path.

* Independent local maps (config 4a): ``shard_maps`` assigns map m to rank
  m mod world; ranks never communicate on the data path.
* Shared map, different keyframes (config 4b): ``SharedMapTrainer`` keeps
  one replica of the map per rank.  Every iteration all ranks draw the same
  ``world`` keyframe indices from an identically seeded sampler, rank r
  renders index r, the raw-parameter gradients (n x 12 float32, the fused
  backward's output) are summed with one all-reduce (NCCL over NVLink /
  NVSwitch on B200), and every rank applies the identical fused Adam step, so
  the replicas stay bit-identical.  This changes the reference's optimiser
  semantics (one keyframe per iteration, mapping.py:475) to the sum over
  ``world`` keyframes per iteration.

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

__all__ = ["shard_maps", "GradOps", "SharedMapTrainer", "world_info"]


def world_info():
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def shard_maps(n_maps: int, rank: int, world: int) -> list:
    """Maps owned by ``rank`` (config 4a: round robin, no communication)."""
    return list(range(rank, n_maps, world))


@dataclass
class GradOps:
    """What one rank does per iteration: gradient of keyframe k, and the optimiser step."""
    grad: Callable[[int], torch.Tensor]          # kf index -> (n, 12) raw gradient (loss parts via .parts)
    adam: Callable[[torch.Tensor], None]         # summed (n, 12) gradient -> in-place parameter update


class SharedMapTrainer:
    def __init__(self, ops: GradOps, n_keyframes: int, cfg: MappingConfig, seed: int, group=None):
        self.ops = ops
        self.n_kf = n_keyframes
        self.cfg = cfg
        self.rng = np.random.default_rng(seed)  # identical on every rank
        self.group = group

    def draw(self, world: int) -> list:
        return [sample_keyframe_index(self.n_kf, self.cfg.kf_sample_p, self.rng) for _ in range(world)]

    def step(self) -> int:
        rank, world = world_info()
        picks = self.draw(world)
        g = self.ops.grad(picks[rank])
        if world > 1:
            dist.all_reduce(g, op=dist.ReduceOp.SUM, group=self.group)
        self.ops.adam(g)
        return picks[rank]


def device_ops(dmap, cfg: MappingConfig, raster=None) -> GradOps:
    """GradOps on the B200 kernels for a DeviceMap (parameters and Adam state on the device)."""

    def grad(k: int) -> torch.Tensor:
        g, parts = dmap.raw_gradient(k, cfg, raster)
        grad.parts = parts
        return g

    return GradOps(grad, lambda g: dmap.apply_adam(g, cfg))
