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


# ---- head-parallel (tensor-parallel) sharding (SURVEY.md §8(e) partitioning 1; include/cacheblend.h) ----
# Rank r of w owns q heads [r n_q/w, (r+1) n_q/w) and kv heads [r n_kv/w, (r+1) n_kv/w): with GQA group
# g = n_q/n_kv, q head h reads kv head h // g, so a rank's q heads only read its own kv heads and
# attention needs no communication. The MLP is split by d_ff features (Megatron column/row split).
def head_shard_shape(shape, world: int):
    """The model a rank's cb_ctx is created with: heads and d_ff divided by world."""
    if world < 1 or shape.n_kv_heads % world or shape.n_q_heads % world or shape.d_ff % world:
        raise ValueError(f"{shape.name}: n_q {shape.n_q_heads}, n_kv {shape.n_kv_heads}, d_ff {shape.d_ff} "
                         f"not divisible by world {world}")
    import dataclasses
    return dataclasses.replace(shape, n_q_heads=shape.n_q_heads // world, n_kv_heads=shape.n_kv_heads // world,
                               d_ff=shape.d_ff // world)


def head_shard_ranges(shape, rank: int, world: int):
    """Row / column ranges of rank's shard in the full cb_layer_w layouts."""
    head_shard_shape(shape, world)
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside [0, {world})")
    hd, qd, kvd, ff = shape.head_dim, shape.n_q_heads * shape.head_dim, shape.n_kv_heads * shape.head_dim, shape.d_ff
    ql, kvl, fl = qd // world, kvd // world, ff // world
    return {"q_rows": (rank * ql, (rank + 1) * ql),
            "k_rows": (qd + rank * kvl, qd + (rank + 1) * kvl),
            "v_rows": (qd + kvd + rank * kvl, qd + kvd + (rank + 1) * kvl),
            "o_cols": (rank * ql, (rank + 1) * ql),
            "gate_rows": (rank * fl, (rank + 1) * fl),
            "up_rows": (ff + rank * fl, ff + (rank + 1) * fl),
            "down_cols": (rank * fl, (rank + 1) * fl),
            "kv_heads": (rank * shape.n_kv_heads // world, (rank + 1) * shape.n_kv_heads // world)}


def shard_layer(w, shape, rank: int, world: int):
    """Rank's shard of one layer's weights (dict in the cb_layer_w layout: attn_norm, w_qkv, w_o, mlp_norm,
    w_gate_up, w_down), as new contiguous tensors on the same device."""
    r = head_shard_ranges(shape, rank, world)
    rows = lambda t, a: t[a[0]:a[1]]
    cols = lambda t, a: t[:, a[0]:a[1]]
    return {"attn_norm": w["attn_norm"].clone(), "mlp_norm": w["mlp_norm"].clone(),
            "w_qkv": torch.cat([rows(w["w_qkv"], r["q_rows"]), rows(w["w_qkv"], r["k_rows"]),
                                rows(w["w_qkv"], r["v_rows"])], 0).contiguous(),
            "w_o": cols(w["w_o"], r["o_cols"]).contiguous(),
            "w_gate_up": torch.cat([rows(w["w_gate_up"], r["gate_rows"]), rows(w["w_gate_up"], r["up_rows"])],
                                   0).contiguous(),
            "w_down": cols(w["w_down"], r["down_cols"]).contiguous()}


def shard_kv(kv, shape, rank: int, world: int):
    """Rank's kv heads of a KV tensor [..., n_kv, head_dim]."""
    a, b = head_shard_ranges(shape, rank, world)["kv_heads"]
    return kv[..., a:b, :].contiguous()


def broadcast_bytes(payload: bytes, src: int = 0) -> bytes:
    """Broadcast a small host byte string (the NCCL unique id) over the default process group."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return payload
    obj = [payload if dist.get_rank() == src else None]
    dist.broadcast_object_list(obj, src=src)
    return obj[0]


# ---- half-split RoPE checkpoints ----------------------------------------------
# The library rotates interleaved pairs (2i, 2i+1) as the paper's appendix does. Checkpoints and
# engines that rotate half-split pairs (i, i + hd/2) are converted at load time, not in the kernels: with
# perm[2i] = i, perm[2i+1] = i + hd/2, interleaved RoPE of z[perm] equals (half-split RoPE of z)[perm], so
# permuting the q and k rows of W_qkv inside each head, and the head dims of a cached K, makes every kernel
# compute the permuted half-split result. Attention scores (q . k), the KV deviation (an L2 norm) and V are
# unchanged by the common permutation; the blended K is handed back with the inverse permutation.
def rope_interleave_perm(head_dim: int):
    import numpy as np
    h = head_dim // 2
    p = np.empty(head_dim, dtype=np.int64)
    p[0::2] = np.arange(h)
    p[1::2] = np.arange(h) + h
    return p


def interleave_rope_weights(w_qkv, shape):
    """W_qkv [(n_q + 2 n_kv) hd][d] of a half-split checkpoint -> the library's interleaved layout (q and k
    head rows permuted, v rows untouched). Works for numpy arrays and torch tensors."""
    hd = shape.head_dim
    p = rope_interleave_perm(hd)
    n_rot = shape.n_q_heads + shape.n_kv_heads  # q heads then k heads carry RoPE
    idx = [h * hd + p for h in range(n_rot)]
    import numpy as np
    rows = np.concatenate(idx + [np.arange(n_rot * hd, w_qkv.shape[0])])
    if isinstance(w_qkv, torch.Tensor):
        return w_qkv[torch.from_numpy(rows).to(w_qkv.device)].contiguous()
    return np.ascontiguousarray(w_qkv[rows])


def interleave_rope_cache(k, inverse: bool = False):
    """Cached K [..., head_dim] of a half-split engine -> interleaved order (inverse=True: back)."""
    import numpy as np
    p = rope_interleave_perm(k.shape[-1])
    if inverse:
        p = np.argsort(p)
    if isinstance(k, torch.Tensor):
        return k[..., torch.from_numpy(p).to(k.device)].contiguous()
    return np.ascontiguousarray(k[..., p])
