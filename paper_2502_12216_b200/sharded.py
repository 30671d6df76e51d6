"""Sequence-sharded decode (1M-token contexts): host driver of the three library stages
and the collectives between them (reading 23).

Each rank holds a Tactic index over its token shard of every (sequence, KV head).  One
decode step:

    local_max = stage1(q)                 # S1-S5 locally: (m_s, theta_max_s) per q-head
    all_reduce(local_max, MAX)            # NCCL over NVLink / NVSwitch (64 doubles per unit)
    mass = stage1b(local_max)             # [W_s, M_s(theta_t)] in the global exponent frame
    all_reduce(mass, SUM)                 # ~131 KB of fp64 per 8 units
    o_s, lse_s = stage2(q, p, local_max, mass)   # select theta >= theta*, S7-S9 locally
    all_gather(o_s, lse_s) ; out = lse_merge(...)

The stages are injectable so the collective schedule can be exercised on CPU with the
gloo backend (tests/test_sharded_gloo.py) using stand-in stages; on GPUs the defaults are
the libtactic stage entry points.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List, Optional, Tuple

import torch
import torch.distributed as dist


def unit_block(units: int, world: int, rank: int) -> Tuple[int, int]:
    """Batch x KV-head mode (the paper's sub-requests, across GPUs):
    rank `rank` of `world` owns the contiguous unit range [start, stop) of the units
    u = b * Hkv + h (batch-major); the first units % world ranks take one extra unit.
    No collective touches the data path: each rank builds and decodes its own units."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("need 0 <= rank < world")
    base, extra = divmod(units, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def block_units(units: int, Hkv: int, world: int, rank: int) -> List[Tuple[int, int]]:
    """The (b, h) pairs of rank's unit block."""
    start, stop = unit_block(units, world, rank)
    return [divmod(u, Hkv) for u in range(start, stop)]


@dataclass
class Stages:
    stage1: Callable      # (q) -> local_max [units][G][2] float64
    stage1b: Callable     # (global_max) -> mass [units][G][1+T] float64
    stage2: Callable      # (q, p, global_max, global_mass) -> (o [units][G][128] f32, lse [units][G] f32)
    merge: Callable       # (o_parts [S][rows][128], lse_parts [S][rows]) -> out [rows][128]


def library_stages(index) -> Stages:
    """The GPU stages of one rank's index (libtactic)."""
    from . import tactic as T
    return Stages(
        stage1=lambda q: T.decode_stage1(q, index),
        stage1b=lambda gmax: T.decode_stage1b(index, gmax),
        stage2=lambda q, p, gmax, gmass: T.decode_stage2(q, index, p, gmax, gmass),
        merge=lambda o, l: T.lse_merge(o, l),
    )


def decode_sharded(q: torch.Tensor, stages: Stages, p: float, group: Optional[dist.ProcessGroup] = None):
    """One sequence-sharded decode step; every rank returns the merged output
    [units * G, 128] (bf16 on GPU stages)."""
    world = dist.get_world_size(group)
    local_max = stages.stage1(q).contiguous()
    dist.all_reduce(local_max, op=dist.ReduceOp.MAX, group=group)
    mass = stages.stage1b(local_max).contiguous()
    dist.all_reduce(mass, op=dist.ReduceOp.SUM, group=group)
    o_part, lse_part = stages.stage2(q, p, local_max, mass)
    rows = lse_part.numel()
    o_part = o_part.reshape(rows, 128).contiguous()
    lse_part = lse_part.reshape(rows).contiguous()
    o_all = [torch.empty_like(o_part) for _ in range(world)]
    l_all = [torch.empty_like(lse_part) for _ in range(world)]
    dist.all_gather(o_all, o_part, group=group)
    dist.all_gather(l_all, lse_part, group=group)
    return stages.merge(torch.stack(o_all), torch.stack(l_all))
