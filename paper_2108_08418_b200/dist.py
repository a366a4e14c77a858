"""Multi-GPU plumbing: frame sharding and the final statistics reduction.

Sub-blocks ("frames") are independent, so rank r of N decodes the contiguous
frame range [r F, (r+1) F) with no data-path collective (weak scaling).  The
only collective is one all_reduce(SUM) of integer-valued statistics and one
all_reduce(MAX) of device time at the end of a run (north star: "NCCL over
NVLink is used only for the final reduction of frame-error and throughput
statistics").  Works with any torch.distributed backend (NCCL on GPUs, gloo
in the CPU tests).
"""
from __future__ import annotations

from typing import Dict, Sequence, Tuple

import torch


def shard(frames_per_rank: int, rank: int) -> Tuple[int, int]:
    """(first_frame, count) of this rank's contiguous frame range."""
    return rank * frames_per_rank, frames_per_rank


SUM_KEYS = ("bits", "frames", "frames_ok", "undetected")


def reduce_stats(stats: Dict[str, float], iters_sum: Sequence[float], edge_iters: Sequence[float],
                 times_ms: Sequence[float], device, group=None):
    """all_reduce SUM of counters and MAX of times over the process group.

    Returns (sums dict, iters_sum list, edge_iters list, max times list).  With
    no initialised process group the inputs are returned unchanged.
    """
    import torch.distributed as dist
    m = len(iters_sum)
    sums = torch.tensor([float(stats[k]) for k in SUM_KEYS] + [float(v) for v in iters_sum] +
                        [float(v) for v in edge_iters], dtype=torch.float64, device=device)
    tmax = torch.tensor([float(t) for t in times_ms], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX, group=group)
    s = sums.cpu().tolist()
    out = {k: s[i] for i, k in enumerate(SUM_KEYS)}
    return out, s[len(SUM_KEYS):len(SUM_KEYS) + m], s[len(SUM_KEYS) + m:], tmax.cpu().tolist()
