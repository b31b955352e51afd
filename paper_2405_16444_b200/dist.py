"""Request-parallel multi-GPU plumbing (partitioning 2).

Blend requests are independent problems: every rank holds a full weight replica and blends its own
requests, with no collective on the data path. The only cross-rank traffic is host-side bookkeeping:
which requests a rank owns, and the max-over-ranks step time the throughput is quoted on. This module
holds that logic (torch.distributed, any backend: NCCL on GPUs, gloo in the CPU tests)."""
from __future__ import annotations

import heapq
import os
from typing import List, Sequence

import torch
import torch.distributed as dist


def world_info():
    """(rank, world, local_rank) from the torchrun environment (1 process = 1 GPU)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def assign_requests(sizes: Sequence[int], world: int) -> List[List[int]]:
    """Greedy longest-processing-time assignment: requests by decreasing size
    (ties: lower index first) each go to the currently least-loaded rank (ties: lower rank). Returns the
    request indices of every rank in ascending order. Deterministic, so every rank computes the same
    partition without communicating."""
    if world < 1:
        raise ValueError("world must be >= 1")
    order = sorted(range(len(sizes)), key=lambda i: (-int(sizes[i]), i))
    heap = [(0, r) for r in range(world)]
    out: List[List[int]] = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + int(sizes[i]), r))
    return [sorted(x) for x in out]


def max_over_ranks(value: float, device=None) -> float:
    """All-reduce MAX of a per-rank scalar (the step time the job is quoted on)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def job_throughput(tokens_this_rank: int, ms_this_rank: float, device=None):
    """Whole-job context tokens/s: all ranks' tokens over the slowest rank's time (weak scaling)."""
    ms = max_over_ranks(ms_this_rank, device)
    tok = sum_over_ranks(tokens_this_rank, device)
    return tok / (ms / 1e3), ms, tok
