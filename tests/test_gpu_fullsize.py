"""Full-size parity (BASELINE configs[1]: Mistral-7B shape, 6 x 512 tokens, r = 0.15, bf16) in the launch
configuration bench.py times (cb_blend_forward), checked on sampled outputs the fp64 oracle computes one by
one from the same inputs, plus properties that hold at any size:

- selection: S_i sorted, unique, |S_i| = k_i, S_i within S_{i-1} (gradual filtering), and S_i is
  exactly the top-k_i (ties -> lower token) of the deviations the GPU reported (R6);
- untouched rows: K of tokens never selected at layer i equals the oracle's realign of the chunk cache
  (footnote P:208-211), V is bitwise the chunk cache (R3);
- per-layer replay: cb_blend_layer stepped with the forward's selections reproduces the forward (up to
  the fused-RMSNorm rounding, R15);
  for sampled layers the oracle recomputes, from that layer's GPU inputs (h rows, K/V before / after),
  the deviation of sampled candidates, the scattered K/V rows and the output h of sampled kept rows
   with the layer's weights regenerated from the counter-RNG spec on the host.
"""
import numpy as np
import pytest
import torch

from oracle import cacheblend_oracle as O
from synth import workload as W

from tests.gpu_helpers import DEV, np32, to_dev
from tests.helpers import rel_err

pytestmark = pytest.mark.gpu

SEED = 1
SAMPLED_LAYERS = (0, 1, 2, 31)


@pytest.fixture(scope="module")
def run(P):
    s = W.MODELS["mistral-7b"]
    req = W.Request([512] * 6, 0, SEED, 0.15)
    N, L = req.n_ctx, s.n_layers
    ctx = P.Context(s, "bf16", max_tokens=N, max_pos=2 * N)
    mw = P.ModelWeights.synth(s, SEED, "bf16", DEV)
    tok = to_dev(req.tokens(s.vocab), torch.int32)
    pos_np = req.global_positions()
    pos = to_dev(pos_np, torch.int32)
    cs = req.chunk_starts()
    # chunk caches: standalone prefill of every chunk at local positions, as bench.py does
    k_in = torch.empty(L, N, s.n_kv_heads, s.head_dim, dtype=torch.bfloat16, device=DEV)
    v_in = torch.empty_like(k_in)
    for c in range(len(cs) - 1):
        a, b = int(cs[c]), int(cs[c + 1])
        kc = torch.empty(L, b - a, s.n_kv_heads, s.head_dim, dtype=torch.bfloat16, device=DEV)
        vc = torch.empty_like(kc)
        P.blend_forward(ctx, mw, tok[a:b].contiguous(), torch.arange(b - a, dtype=torch.int32, device=DEV), [0],
                        b - a, None, None, kc, vc, [0] * L)
        k_in[:, a:b] = kc
        v_in[:, a:b] = vc
    ks = P.schedule(0.15, N, L)
    kb, vb = torch.empty_like(k_in), torch.empty_like(v_in)
    sel = torch.full((L, N), -1, dtype=torch.int32, device=DEV)
    dev = torch.full((L, N), -1.0, dtype=torch.float32, device=DEV)
    h = P.blend_forward(ctx, mw, tok, pos, list(cs), 0, k_in, v_in, kb, vb, ks, sel_out=sel, dev_out=dev)
    torch.cuda.synchronize()
    ctx.check_device_errors()
    sels = [r[r >= 0] for r in sel.cpu().numpy()]
    return dict(P=P, s=s, req=req, N=N, L=L, ctx=ctx, mw=mw, tok=tok, pos=pos, pos_np=pos_np, cs=cs, k_in=k_in,
                v_in=v_in, ks=ks, kb=kb, vb=vb, sel=sels, dev=dev.cpu().numpy(), h=h)


def test_selection_properties(run):
    N, L, ks, sels, dev = run["N"], run["L"], run["ks"], run["sel"], run["dev"]
    np.testing.assert_array_equal(sels[0], np.arange(N))
    prev = np.arange(N)
    for i in range(1, L):
        s_i = sels[i]
        assert len(s_i) == ks[i] and np.all(np.diff(s_i) > 0), f"layer {i}"
        assert np.isin(s_i, prev).all(), f"layer {i}: not inside S_(i-1)"
        d = dev[i][:len(prev)]  # deviations of the candidates, in candidate order
        assert np.all(np.isfinite(d)) and np.all(d >= 0)
        order = np.lexsort((prev, -d.astype(np.float64)))  # largest first, ties -> lower token
        np.testing.assert_array_equal(np.sort(prev[order[:ks[i]]]), s_i, err_msg=f"layer {i}: not top-k")
        prev = s_i


def test_untouched_rows_are_realigned_cache(run):
    s, N, L = run["s"], run["N"], run["L"]
    loc = run["req"].local_positions()
    rng = np.random.default_rng(0)
    for i in (0, 1, 15, 31):
        keep = np.setdiff1d(np.arange(N), run["sel"][i]) if i > 0 else np.arange(N)
        if i == 0:  # layer 0 keeps every context row's realigned cache
            keep = np.arange(N)
        t = np.sort(rng.choice(keep, 64, replace=False))
        k_src = np32(run["k_in"][i][t]).astype(np.float64)
        ref = O.realign(k_src, loc[t], run["pos_np"][t], s.rope_theta)
        assert rel_err(np32(run["kb"][i][t]), ref) < 5e-3, f"layer {i}"
        assert torch.equal(run["vb"][i][t], run["v_in"][i][t]), f"layer {i}: V changed"


def _layer_model(s, i):
    w = W.layer_weights(s, i, SEED, "bf16")
    layers = [None] * s.n_layers
    layers[i] = {k: np.asarray(v, np.float64) for k, v in w.items()}
    return O.Model(s.n_layers, s.d_model, s.n_q_heads, s.n_kv_heads, s.head_dim, s.rope_theta, s.rms_eps,
                   np.zeros((1, s.d_model)), layers)


def test_stepped_layers_match_forward_and_oracle(run):
    """cb_blend_layer replay of the forward's selections; sampled layers recomputed by the oracle."""
    P, s, N, L, ks = run["P"], run["s"], run["N"], run["L"], run["ks"]
    ctx, mw = run["ctx"], run["mw"]
    pos_np = run["pos_np"]
    kb = run["k_in"].clone()
    vb = run["v_in"].clone()
    loc = to_dev(run["req"].local_positions(), torch.int32)
    P.rope_realign(ctx, kb, kb, loc, run["pos"], L, N, N * s.kvd)
    h = torch.zeros(N, s.d_model, dtype=torch.float32, device=DEV)
    h[:N] = P.api.op_embed(ctx, mw.embed, run["tok"])
    cand = torch.arange(N, dtype=torch.int32, device=DEV)
    rng = np.random.default_rng(7)
    for i in range(L):
        sampled = i in SAMPLED_LAYERS
        cand_np = cand.cpu().numpy()
        if sampled:
            h_in = np32(h[:len(cand_np)]).astype(np.float64)
            k_before, v_before = np32(kb[i]).astype(np.float64), np32(vb[i]).astype(np.float64)
        if i == 0:
            P.blend_layer(ctx, 0, mw, h, cand, N, 0, kb[0], vb[0], run["pos"], N)
            sel_i, dev_i = cand, None
        else:
            fs = to_dev(run["sel"][i], torch.int32)
            sel_i, dev_i = P.blend_layer(ctx, i, mw, h, cand, ks[i], 0, kb[i], vb[i], run["pos"], N, force_sel=fs,
                                         want_dev=True)
        torch.cuda.synchronize()
        # the stepped layer reproduces the forward's KV^new (the forward additionally fuses the next
        # layer's RMSNorm into the down projection, R15, so equal up to that rounding)
        assert rel_err(np32(kb[i]), np32(run["kb"][i])) < 1e-2 and rel_err(np32(vb[i]), np32(run["vb"][i])) < 1e-2
        if i > 0:
            assert rel_err(dev_i.cpu().numpy(), run["dev"][i][:len(cand_np)]) < 2e-2, f"layer {i}: dev vs forward"
        sel_np = sel_i.cpu().numpy()
        if sampled:
            m = _layer_model(s, i)
            k_after, v_after = np32(kb[i]).astype(np.float64), np32(vb[i]).astype(np.float64)
            # deviation of sampled candidates: q/k/v from the GPU's input rows
            if i > 0:
                ci = np.sort(rng.choice(len(cand_np), 16, replace=False))
                _, k_new, v_new = O.qkv(m, i, h_in[ci], pos_np[cand_np[ci]], need_q=False)
                d_ref = O.kv_deviation(k_new, v_new, k_before[cand_np[ci]], v_before[cand_np[ci]])
                assert rel_err(dev_i.cpu().numpy()[ci], d_ref) < 2e-2, f"layer {i}: deviation"
            # kept rows: fresh K/V scattered, then attention over all keys, W_o, MLP
            si = np.sort(rng.choice(len(sel_np), 8, replace=False))
            slot = np.searchsorted(cand_np, sel_np[si])
            q, k_new, v_new = O.qkv(m, i, h_in[slot], pos_np[sel_np[si]])
            if i > 0:
                assert rel_err(k_after[sel_np[si]], k_new) < 2e-2, f"layer {i}: scattered K"
                assert rel_err(v_after[sel_np[si]], v_new) < 2e-2, f"layer {i}: scattered V"
            a = O.causal_attention(q, pos_np[sel_np[si]], k_after, v_after, pos_np)
            h_ref = O.attn_out_mlp(m, i, h_in[slot], a.reshape(len(si), -1))
            assert rel_err(np32(h[si]), h_ref) < 2e-2, f"layer {i}: h"
        cand = sel_i.clone()
    assert rel_err(np32(h[:ks[L - 1]]), np32(run["h"][:ks[L - 1]])) < 1e-2, "stepped final h vs forward"
