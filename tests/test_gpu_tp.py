"""Head-parallel (tensor-parallel) blend (SURVEY.md §8(e) partitioning 1; include/cacheblend.h) on ONE GPU.

The loopback group (cb_group_create / cb_set_comm_local) runs world contexts of this process, each driven
by its own host thread and stream, through the same per-rank kernels the NCCL path runs; only the
exchange differs (stream events + a fixed-order reduce kernel instead of NCCL). Each rank holds the
shard model (heads and d_ff divided by world) and its kv heads of the cache. Checked against the fp64
oracle of the UNSHARDED model on identical inputs, with the tolerances of test_gpu_parity.py (R13/R14),
and every rank must agree bitwise on S_i, Delta_kv and h (the top-k is the same on every rank).
The NCCL backend itself is exercised at world 1 (a real communicator; the all-reduce/all-gather calls
run in the forward and inside a CUDA graph), bitwise equal to the context without a communicator."""
import os
import threading

import numpy as np
import pytest
import torch

from oracle import cacheblend_oracle as O
from paper_2405_16444_b200 import dist as D
from synth import workload as W
from tests.gpu_helpers import DEV, near_tie_ok, np32, to_dev
from tests.helpers import band_check, oracle_model, rel_err, request_inputs, shape, topk_tokens

pytestmark = pytest.mark.gpu

TOL = {"f32": 1e-4, "bf16": 2e-2}


def run_blend_tp(P, s, dtype, seed, req, tok, pos, cs, Kc, Vc, ks, world, force_sel=None, p2p=False):
    """cb_blend_forward on `world` loopback ranks; returns per-rank outputs plus K/V reassembled over heads."""
    td = P.api.TORCH_DTYPES[dtype]
    L, N, n_suf = s.n_layers, req.n_ctx, req.n_suffix
    T = N + n_suf
    ss = D.head_shard_shape(s, world)
    group = P.Group(world)
    full = P.ModelWeights.synth(s, seed, dtype, DEV)
    ranks = []
    for r in range(world):
        ctx = P.Context(ss, dtype, max_tokens=T, max_pos=max(int(np.max(pos)) + 1, 2 * T))
        ctx.set_comm_local(group, r)
        if p2p:
            if p2p == "plain":
                ctx.set_option("tp_fuse", 0)
            ctx.enable_tp_p2p()
        mw = P.ModelWeights(ss, dtype, full.embed, [D.shard_layer(w, s, r, world) for w in full.layers])
        k_in = D.shard_kv(to_dev(Kc, td), s, r, world)
        v_in = D.shard_kv(to_dev(Vc, td), s, r, world)
        kb = torch.full((L, T, ss.n_kv_heads, s.head_dim), float("nan"), dtype=td, device=DEV)
        vb = torch.full_like(kb, float("nan"))
        sel = torch.empty(L, max(N, 1), dtype=torch.int32, device=DEV)
        dev = torch.full((L, max(N, 1)), -1.0, dtype=torch.float32, device=DEV)
        rows = (N if L == 1 else int(ks[-1])) + n_suf
        h = torch.empty(max(rows, 1), s.d_model, dtype=torch.float32, device=DEV)
        ranks.append(dict(ctx=ctx, mw=mw, k_in=k_in, v_in=v_in, kb=kb, vb=vb, sel=sel, dev=dev, h=h,
                          stream=torch.cuda.Stream()))
    fs = None
    if force_sel is not None:
        fsn = np.full((L, max(N, 1)), -1, dtype=np.int32)
        for i in range(1, L):
            fsn[i, :len(force_sel[i])] = force_sel[i]
        fs = to_dev(fsn, torch.int32)
    tok_d, pos_d = to_dev(tok, torch.int32), to_dev(pos, torch.int32)
    torch.cuda.synchronize()
    errors = [None] * world

    def work(r):
        x = ranks[r]
        try:
            P.blend_forward(x["ctx"], x["mw"], tok_d, pos_d, list(cs), n_suf, x["k_in"], x["v_in"], x["kb"], x["vb"],
                            ks, force_sel=fs, sel_out=x["sel"], dev_out=x["dev"], h_out=x["h"], stream=x["stream"])
            x["stream"].synchronize()
        except Exception as e:  # surfaced below
            errors[r] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert all(not t.is_alive() for t in th), "a rank hung"
    for e in errors:
        if e is not None:
            raise e
    torch.cuda.synchronize()
    for x in ranks:
        x["ctx"].check_device_errors()
    rows = (N if L == 1 else int(ks[-1])) + n_suf
    out = dict(ranks=ranks, group=group,
               K=np.concatenate([np32(x["kb"]) for x in ranks], axis=2),
               V=np.concatenate([np32(x["vb"]) for x in ranks], axis=2),
               h=np32(ranks[0]["h"][:rows]), dev=ranks[0]["dev"].cpu().numpy())
    sel_np = ranks[0]["sel"].cpu().numpy()
    out["sel"] = [row[row >= 0] for row in sel_np]
    for x in ranks[1:]:  # every rank took the same decisions on the same numbers
        assert torch.equal(x["sel"], ranks[0]["sel"])
        assert torch.equal(x["dev"], ranks[0]["dev"])
        assert torch.equal(x["h"], ranks[0]["h"])
    return out


def _case(name, seed, lens, n_suf, dtype, ratio, **over):
    s = shape(name, **over)
    m = oracle_model(s, seed, dtype)
    req = W.Request(list(lens), n_suf, seed, ratio)
    tok, pos, cs, Kc, Vc = request_inputs(s, req, m, dtype)
    ks = O.schedule(ratio, req.n_ctx, s.n_layers)
    return s, m, req, tok, pos, cs, Kc, Vc, ks


def _compare(res, ora, s, tol):
    for i in range(s.n_layers):
        assert rel_err(res["K"][i], ora.K[i]) < tol, f"K layer {i}"
        assert rel_err(res["V"][i], ora.V[i]) < tol, f"V layer {i}"
    assert rel_err(res["h"], ora.h_final) < tol, "h_final"


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_tp_tiny_fp32_free_run(P, world, seed):
    """BASELINE configs[0] (tiny, 3 x 32, 15 %, fp32) split over `world` head-parallel ranks, free-running
    selection (unfused Delta_kv: per-rank head sums all-reduced)."""
    s, m, req, tok, pos, cs, Kc, Vc, ks = _case("tiny", seed, [32, 32, 32], 0, "f32", 0.15, n_layers=3)
    ora = O.blend_forward(m, tok, pos, cs, 0, Kc, Vc, ks)
    res = run_blend_tp(P, s, "f32", seed, req, tok, pos, cs, Kc, Vc, ks, world)
    same = True
    for i in range(1, s.n_layers):
        ok, flips = near_tie_ok(res["sel"][i], ora.sel[i], ora.dev[i], ora.cand[i], ks[i])
        assert ok, f"layer {i}: {flips} flips outside the near-tie band"
        same &= flips == 0
        np.testing.assert_allclose(res["dev"][i][:len(ora.cand[i])], ora.dev[i], rtol=1e-4,
                                   atol=1e-4 * ora.dev[i].max())
    if not same:
        res = run_blend_tp(P, s, "f32", seed, req, tok, pos, cs, Kc, Vc, ks, world, force_sel=ora.sel)
    _compare(res, ora, s, TOL["f32"])


def test_tp_tiny_fp32_suffix(P):
    s, m, req, tok, pos, cs, Kc, Vc, ks = _case("tiny", 5, [17, 40, 9], 6, "f32", 0.3, n_layers=3)
    ora = O.blend_forward(m, tok, pos, cs, req.n_suffix, Kc, Vc, ks)
    res = run_blend_tp(P, s, "f32", 5, req, tok, pos, cs, Kc, Vc, ks, 2, force_sel=ora.sel)
    for i in range(1, s.n_layers):
        np.testing.assert_array_equal(res["sel"][i], ora.sel[i])
    _compare(res, ora, s, TOL["f32"])


@pytest.mark.parametrize("n_suf", [0, 9])
def test_tp_small_bf16_replay(P, n_suf):
    """bf16, d=1024, hd=128, GQA 4 over 2 ranks (one kv head each): fused Delta_kv partials all-gathered,
    o_proj / down_proj all-reduced. Replay mode (the oracle's S_i forced, R14) for values; the GPU's own
    top-k of its gathered deviations must (nearly) equal the oracle's set."""
    s, m, req, tok, pos, cs, Kc, Vc, ks = _case("small", 2, [200, 317, 150], n_suf, "bf16", 0.15)
    ora = O.blend_forward(m, tok, pos, cs, n_suf, Kc, Vc, ks)
    res = run_blend_tp(P, s, "bf16", 2, req, tok, pos, cs, Kc, Vc, ks, 2, force_sel=ora.sel)
    _compare(res, ora, s, TOL["bf16"])
    for i in range(1, s.n_layers):
        d = res["dev"][i][:len(ora.cand[i])]
        assert rel_err(d, ora.dev[i]) < TOL["bf16"], f"dev layer {i}"
        ok, flips, band = band_check(topk_tokens(d, ora.cand[i], ks[i]), d, ora.dev[i], ora.cand[i], ks[i])
        assert ok, f"layer {i}: {flips} flips outside the band {band}"


def test_tp_small_bf16_free_run_consistent(P):
    """Free-running bf16 over 2 ranks: ranks agree bitwise (checked in run_blend_tp), selections are nested
    top-k sets of the reported deviations, layer 1's Delta_kv (identical candidates on both sides) is within
    bf16 tolerance of the oracle's and its S_1 differs from the oracle's only inside the error band."""
    s, m, req, tok, pos, cs, Kc, Vc, ks = _case("small", 4, [256, 256, 128], 0, "bf16", 0.15)
    res = run_blend_tp(P, s, "bf16", 4, req, tok, pos, cs, Kc, Vc, ks, 2)
    cand = np.arange(req.n_ctx)
    for i in range(1, s.n_layers):
        d = res["dev"][i][:len(cand)]
        np.testing.assert_array_equal(res["sel"][i], topk_tokens(d, cand, ks[i]))
        assert set(res["sel"][i]) <= set(cand)
        cand = res["sel"][i]
    ora = O.blend_forward(m, tok, pos, cs, 0, Kc, Vc, ks)
    d1 = res["dev"][1][:req.n_ctx]
    assert rel_err(d1, ora.dev[1]) < TOL["bf16"]
    ok, flips, band = band_check(res["sel"][1], d1, ora.dev[1], ora.cand[1], ks[1])
    assert ok, f"layer 1: {flips} flips outside the band {band}"


def _nccl_world1(P, s, dtype, seed, req, tok, pos, cs, Kc, Vc, ks, comm: bool, graph: bool, p2p: bool = False):
    td = P.api.TORCH_DTYPES[dtype]
    L, N = s.n_layers, req.n_ctx
    ctx = P.Context(s, dtype, max_tokens=N, max_pos=2 * N)
    if comm:
        ctx.set_comm(P.nccl_unique_id(), 0, 1)
    if p2p:
        ctx.enable_tp_p2p()
        ctx.tp_ipc_open([ctx.tp_ipc_handle()])
    mw = P.ModelWeights.synth(s, seed, dtype, DEV)
    k_in, v_in = to_dev(Kc, td), to_dev(Vc, td)
    kb, vb = torch.empty_like(k_in), torch.empty_like(v_in)
    sel = torch.empty(L, N, dtype=torch.int32, device=DEV)
    h = torch.empty(ks[-1], s.d_model, dtype=torch.float32, device=DEV)
    tok_d, pos_d = to_dev(tok, torch.int32), to_dev(pos, torch.int32)

    def step():
        P.blend_forward(ctx, mw, tok_d, pos_d, list(cs), 0, k_in, v_in, kb, vb, ks, sel_out=sel, h_out=h)

    step()
    torch.cuda.synchronize()
    if graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step()
        kb.zero_(); h.zero_()
        g.replay()
        torch.cuda.synchronize()
    return kb.clone(), vb.clone(), sel.clone(), h.clone()


def test_nccl_world1_equals_no_comm(P):
    """A real NCCL communicator of one rank: the forward (eager and captured in a CUDA graph) calls the
    all-gather / all-reduces and stays bitwise equal to the context without a communicator."""
    s, m, req, tok, pos, cs, Kc, Vc, ks = _case("small", 3, [128, 200], 0, "bf16", 0.15)
    ref = _nccl_world1(P, s, "bf16", 3, req, tok, pos, cs, Kc, Vc, ks, comm=False, graph=False)
    for graph in (False, True):
        got = _nccl_world1(P, s, "bf16", 3, req, tok, pos, cs, Kc, Vc, ks, comm=True, graph=graph)
        for a, b in zip(got, ref):
            assert torch.equal(a, b)


def test_tp_argument_errors(P):
    s = D.head_shard_shape(shape("tiny"), 2)
    g = P.Group(2)
    ctx = P.Context(s, "f32", max_tokens=64)
    with pytest.raises(P.CacheBlendError):
        ctx.set_comm_local(g, 2)
    ctx.set_comm_local(g, 0)
    with pytest.raises(P.CacheBlendError):  # already joined
        ctx.set_comm_local(g, 1)
    ctx2 = P.Context(s, "f32", max_tokens=64)
    with pytest.raises(P.CacheBlendError):  # rank taken
        ctx2.set_comm_local(g, 0)


def test_tp_request_path_equals_forward(P):
    """The host-buffer request path (cb_blend_request: layer-pipelined copies on each rank's copy stream)
    under the loopback head-parallel group gives every rank exactly its cb_blend_forward result."""
    s, m, req, tok, pos, cs, Kc, Vc, ks = _case("small", 7, [96, 130, 64], 0, "bf16", 0.15)
    world = 2
    ref = run_blend_tp(P, s, "bf16", 7, req, tok, pos, cs, Kc, Vc, ks, world)
    ranks = ref["ranks"]
    td = P.api.TORCH_DTYPES["bf16"]
    L, T = s.n_layers, req.n_total
    toks = torch.from_numpy(tok.astype(np.int32)).pin_memory()
    poss = torch.from_numpy(pos.astype(np.int32)).pin_memory()
    outs, errors = [], [None] * world
    for r, x in enumerate(ranks):
        kh = D.shard_kv(torch.from_numpy(np.ascontiguousarray(Kc)).to(td), s, r, world).pin_memory()
        vh = D.shard_kv(torch.from_numpy(np.ascontiguousarray(Vc)).to(td), s, r, world).pin_memory()
        kb, vb = torch.empty_like(x["kb"]), torch.empty_like(x["vb"])
        hh = torch.empty(ks[-1], s.d_model, dtype=torch.float32).pin_memory()
        outs.append((kh, vh, kb, vb, hh))
    torch.cuda.synchronize()

    def work(r):
        kh, vh, kb, vb, hh = outs[r]
        try:
            P.api.blend_request(ranks[r]["ctx"], ranks[r]["mw"], toks, poss, list(cs), 0, kh, vh, kb, vb, ks, hh,
                                stream=ranks[r]["stream"])
            ranks[r]["stream"].synchronize()
        except Exception as e:
            errors[r] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert all(not t.is_alive() for t in th)
    for e in errors:
        if e is not None:
            raise e
    for r, x in enumerate(ranks):
        _, _, kb, vb, hh = outs[r]
        assert torch.equal(kb, x["kb"]) and torch.equal(vb, x["vb"])
        np.testing.assert_array_equal(hh.numpy(), np32(x["h"][:ks[-1]]))


@pytest.mark.skipif(os.environ.get("CB_TEST_P2P") != "1",
                    reason="experimental peer-memory collectives: multi-rank loopback runs can desync "
                           "(DESIGN.md §7 open issue); set CB_TEST_P2P=1 to run")
@pytest.mark.parametrize("mode", ["fused", "plain"])
@pytest.mark.parametrize("name,dtype,world,n_suf", [("tiny", "f32", 2, 0), ("tiny", "f32", 4, 5), ("small", "bf16", 2, 0)])
def test_tp_p2p_equals_event_path(P, name, dtype, world, n_suf, mode):
    """NVLink peer-memory collectives (cb_tp_p2p_enable; here the loopback members' blocks on one device):
    fused (the o_proj / down_proj epilogues push each row into its owner's receive plane, the owner sums the
    planes and writes everywhere) and plain (local writes, then the one-kernel all-reduce). Both are bitwise
    the results of the event-ordered loopback path (same rank-order sums), so they inherit its parity."""
    s, m, req, tok, pos, cs, Kc, Vc, ks = _case(name, 11, [64, 40, 57] if name == "small" else [32, 32, 32], n_suf,
                                                dtype, 0.2, **({"n_layers": 3} if name == "tiny" else {}))
    a = run_blend_tp(P, s, dtype, 11, req, tok, pos, cs, Kc, Vc, ks, world)
    b = run_blend_tp(P, s, dtype, 11, req, tok, pos, cs, Kc, Vc, ks, world, p2p=mode)
    np.testing.assert_array_equal(a["K"], b["K"])
    np.testing.assert_array_equal(a["V"], b["V"])
    np.testing.assert_array_equal(a["h"], b["h"])
    np.testing.assert_array_equal(a["dev"], b["dev"])
    for x, y in zip(a["sel"], b["sel"]):
        np.testing.assert_array_equal(x, y)


def test_p2p_world1_ipc_graph(P):
    """Peer-memory collectives with a one-rank communicator through the IPC API, eager and replayed from a
    CUDA graph (device-side sequence numbers): bitwise equal to no communicator."""
    s, m, req, tok, pos, cs, Kc, Vc, ks = _case("small", 3, [128, 200], 0, "bf16", 0.15)
    ref = _nccl_world1(P, s, "bf16", 3, req, tok, pos, cs, Kc, Vc, ks, comm=False, graph=False)
    for graph in (False, True):
        got = _nccl_world1(P, s, "bf16", 3, req, tok, pos, cs, Kc, Vc, ks, comm=True, graph=graph, p2p=True)
        for a, b in zip(got, ref):
            assert torch.equal(a, b)
