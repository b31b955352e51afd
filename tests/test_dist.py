"""Request-parallel host logic (SURVEY §8(e) partitioning 2) on CPU: the longest-first assignment and the
max-over-ranks / sum-over-ranks reductions bench.py quotes, exercised with a world_size-2 gloo group."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2405_16444_b200.dist import assign_requests
from synth import workload as W


def test_assign_requests_longest_first():
    sizes = [5, 9, 9, 1, 7, 3, 3]
    parts = assign_requests(sizes, 3)
    assert sorted(i for p in parts for i in p) == list(range(len(sizes)))       # each request exactly once
    assert parts == assign_requests(sizes, 3)                                   # deterministic
    # LPT trace: 9(1)->r0, 9(2)->r1, 7(4)->r2, 5(0)->r2 (7<9), 3(5)->r0, 3(6)->r1, 1(3)->r0
    assert parts == [[1, 3, 5], [2, 6], [0, 4]]
    loads = [sum(sizes[i] for i in p) for p in parts]
    assert max(loads) - min(loads) <= max(sizes)                                 # LPT bound


def test_assign_batched_config_balance():
    reqs = W.config_requests("batched", 1)
    sizes = [r.n_ctx for r in reqs]
    assert len(sizes) == 64 and min(sizes) >= 4 * 256 and max(sizes) <= 8 * 1024
    for world in (1, 2, 4, 8):
        parts = assign_requests(sizes, world)
        loads = [sum(sizes[i] for i in p) for p in parts]
        assert sum(loads) == sum(sizes)
        assert max(loads) <= sum(sizes) / world + max(sizes)
    with pytest.raises(ValueError):
        assign_requests(sizes, 0)


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import torch.distributed as dist
    from paper_2405_16444_b200 import dist as D
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r, w, _ = D.world_info()
    tokens, ms = 1000 * (r + 1), 10.0 + 5.0 * r           # rank 1 is the slow one
    value, ms_max, tok = D.job_throughput(tokens, ms)
    parts = D.assign_requests([r_.n_ctx for r_ in W.config_requests("batched", 1)], w)
    np.save(os.path.join(out_dir, f"r{r}.npy"), np.array([value, ms_max, tok, len(parts[r])], dtype=np.float64))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_reductions():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, port, d), nprocs=2, join=True)
        res = [np.load(os.path.join(d, f"r{r}.npy")) for r in range(2)]
    for v in res:  # every rank sees the same job numbers: 3000 tokens over the slowest rank's 15 ms
        assert v[1] == 15.0 and v[2] == 3000.0
        assert abs(v[0] - 3000.0 / 0.015) < 1e-6
    assert res[0][3] + res[1][3] == 64


# ---- head-parallel sharding (SURVEY §8(e) partitioning 1): the host-side slicing the GPU ranks use ----
def test_head_shard_shapes_and_ranges():
    from paper_2405_16444_b200 import dist as D
    for name in ("mistral-7b", "yi-34b", "llama-70b"):
        s = W.MODELS[name]
        for world in (1, 2, 4, 8):
            ss = D.head_shard_shape(s, world)
            assert ss.n_q_heads * world == s.n_q_heads and ss.n_kv_heads * world == s.n_kv_heads
            assert ss.d_ff * world == s.d_ff and ss.d_model == s.d_model and ss.d_ff % 8 == 0
            # the ranks' row / column ranges tile the full layouts exactly once
            rs = [D.head_shard_ranges(s, r, world) for r in range(world)]
            for key, total in (("q_rows", s.qd), ("o_cols", s.qd), ("gate_rows", s.d_ff), ("down_cols", s.d_ff)):
                cover = sorted(x[key] for x in rs)
                assert cover[0][0] == 0 and cover[-1][1] == total
                assert all(a[1] == b[0] for a, b in zip(cover, cover[1:]))
            # GQA: every q head of a rank reads a kv head of the same rank
            g = s.n_q_heads // s.n_kv_heads
            for r, x in enumerate(rs):
                q0, q1 = x["q_rows"][0] // s.head_dim, x["q_rows"][1] // s.head_dim
                assert all(x["kv_heads"][0] <= h // g < x["kv_heads"][1] for h in range(q0, q1))
    with pytest.raises(ValueError):
        D.head_shard_shape(W.MODELS["small"], 4)  # 2 kv heads


def _abi_layer(w):
    import torch
    t = lambda a: torch.from_numpy(np.asarray(a, np.float64))
    return {"attn_norm": t(w["attn_norm"]), "mlp_norm": t(w["mlp_norm"]),
            "w_qkv": t(np.concatenate([w["wq"], w["wk"], w["wv"]], 0)), "w_o": t(w["wo"]),
            "w_gate_up": t(np.concatenate([w["wg"], w["wu"]], 0)), "w_down": t(w["wd"])}


def _tp_worker(rank, world, port, out_dir):
    """One layer of the head-parallel schedule with oracle primitives on this rank's shard + gloo sums:
    x = RMSNorm(h) replicated; local q/k/v heads; local attention; o_proj partial -> all-reduce; MLP on
    d_ff/world features -> all-reduce. Saved for comparison with the unsharded oracle layer."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    from oracle import cacheblend_oracle as O
    from paper_2405_16444_b200 import dist as D
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s = W.MODELS["tiny"]
    ss = D.head_shard_shape(s, world)
    w = D.shard_layer(_abi_layer(W.layer_weights(s, 0, 7, "f32")), s, rank, world)
    w = {k: v.numpy() for k, v in w.items()}
    qdl, kvdl, ffl = ss.qd, ss.kvd, ss.d_ff
    req = W.Request([20, 12], 0, 7, 0.15)
    pos = req.global_positions()
    h = W.embed_weights(s, 7, "f32").astype(np.float64)[req.tokens(s.vocab)]
    R = h.shape[0]
    x = O.rms_norm(h, w["attn_norm"], s.rms_eps)
    proj = x @ w["w_qkv"].T
    q = O.rope_rotate(proj[:, :qdl].reshape(R, ss.n_q_heads, s.head_dim), pos[:, None], s.rope_theta)
    k = O.rope_rotate(proj[:, qdl:qdl + kvdl].reshape(R, ss.n_kv_heads, s.head_dim), pos[:, None], s.rope_theta)
    v = proj[:, qdl + kvdl:].reshape(R, ss.n_kv_heads, s.head_dim)
    a = O.causal_attention(q, pos, k, v, pos)
    o = torch.from_numpy(a @ w["w_o"].T)
    dist.all_reduce(o)                                                   # (ii) after o_proj
    h1 = h + o.numpy()
    xm = O.rms_norm(h1, w["mlp_norm"], s.rms_eps)
    gu = xm @ w["w_gate_up"].T
    m = torch.from_numpy((O.silu(gu[:, :ffl]) * gu[:, ffl:]) @ w["w_down"].T)
    dist.all_reduce(m)                                                   # (iii) after down_proj
    uid = D.broadcast_bytes(bytes(range(128)) if rank == 0 else b"", src=0)
    np.savez(os.path.join(out_dir, f"tp{rank}.npz"), h2=h1 + m.numpy(), k=k, v=v, uid_ok=uid == bytes(range(128)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_head_parallel_layer_equals_oracle(world):
    from oracle import cacheblend_oracle as O
    from tests.helpers import oracle_model
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_tp_worker, args=(world, port, d), nprocs=world, join=True)
        res = [np.load(os.path.join(d, f"tp{r}.npz")) for r in range(world)]
    s = W.MODELS["tiny"]
    m = oracle_model(s, 7, "f32")
    req = W.Request([20, 12], 0, 7, 0.15)
    pos = req.global_positions()
    h = m.embed[req.tokens(s.vocab)]
    q, k, v = O.qkv(m, 0, h, pos)
    ref = O.attn_out_mlp(m, 0, h, O.causal_attention(q, pos, k, v, pos))
    for r in range(world):
        np.testing.assert_allclose(res[r]["h2"], ref, rtol=1e-12, atol=1e-12)
        assert bool(res[r]["uid_ok"])
    np.testing.assert_allclose(np.concatenate([x["k"] for x in res], 1), k, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(np.concatenate([x["v"] for x in res], 1), v, rtol=1e-12, atol=1e-12)
