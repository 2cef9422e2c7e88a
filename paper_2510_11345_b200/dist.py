"""Data-parallel sharding of the loss path across GPUs (one process per GPU).

Every token row is independent and every GRPO group is independent once kept
whole, so the batch is partitioned by whole groups (LPT on group token counts)
and each rank runs the fused kernels on its shard with the GLOBAL normalisers
(T_global / N_global known at batch-assembly time, so no pre-launch collective
is needed).  The only exchange is one all-reduce (sum) of the fp64 loss scalars
(RF_NUM_SCALARS values) — dlogits stay on their GPU for that rank's LM-head
backward.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Sequence

import numpy as np


def lpt_shard(group_tokens: Sequence[int], world: int) -> List[List[int]]:
    """Longest-processing-time assignment of whole groups to ranks (ties -> lowest rank)."""
    gt = np.asarray(group_tokens, dtype=np.int64)
    order = np.argsort(-gt, kind="stable")
    load = np.zeros(world, dtype=np.int64)
    out: List[List[int]] = [[] for _ in range(world)]
    for g in order:
        r = int(np.argmin(load))
        out[r].append(int(g))
        load[r] += int(gt[g])
    return [sorted(x) for x in out]


@dataclass
class ShardPlan:
    """Which sequences a rank owns, plus the global normalisers."""

    seq_index: np.ndarray   # global sequence ids owned by this rank (whole groups, in order)
    global_tokens: int
    global_seqs: int

    @staticmethod
    def build(lengths: Sequence[int], group_offsets: Sequence[int], rank: int, world: int) -> "ShardPlan":
        lens = np.asarray(lengths, dtype=np.int64)
        go = np.asarray(group_offsets, dtype=np.int64)
        gt = np.array([lens[go[g]:go[g + 1]].sum() for g in range(len(go) - 1)], dtype=np.int64)
        mine = lpt_shard(gt, world)[rank]
        idx = (np.concatenate([np.arange(go[g], go[g + 1]) for g in mine]) if mine
               else np.zeros(0, dtype=np.int64))
        return ShardPlan(seq_index=idx, global_tokens=int(lens.sum()), global_seqs=int(len(lens)))


def allreduce_scalars(scalars, group=None):
    """Sum the per-rank fp64 loss scalars (one collective per step)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(scalars, op=dist.ReduceOp.SUM, group=group)
    return scalars
