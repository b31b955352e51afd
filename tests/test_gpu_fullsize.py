"""Full-size self-consistency at bench.py's exact workload (BASELINE configs[1]: Mistral-7B shape, 6 x 512
tokens, r = 0.15, bf16, chunk caches produced by the library's standalone prefill of every chunk) in
the launch configuration bench.py times (cb_blend_forward).

The caches here are CUDA-path outputs, so nothing in this file feeds the oracle (oracle parity at every
configuration, from seeded inputs only, is tests/test_gpu_configs.py). What is checked:
- selection: S_i sorted, unique, |S_i| = k_i, S_i within S_{i-1} (gradual filtering), and S_i is
  exactly the top-k_i (ties -> lower token) of the deviations the GPU reported (R6);
- untouched rows: K of tokens never selected at layer i is bitwise the library's own cb_rope_realign of the
  chunk cache (footnote P:208-211), V bitwise the chunk cache (R3);
- per-layer replay: cb_blend_layer stepped with the forward's selections reproduces the forward's KV^new,
  Delta_kv and final h (up to the fused-RMSNorm rounding, R15).
"""
import numpy as np
import pytest
import torch

from synth import workload as W

from tests.gpu_helpers import DEV, np32, to_dev
from tests.helpers import rel_err, topk_tokens

pytestmark = pytest.mark.gpu

SEED = 1


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
        np.testing.assert_array_equal(topk_tokens(d, prev, ks[i]), s_i,
                                      err_msg=f"layer {i}: not top-k")
        prev = s_i


def test_untouched_rows_are_realigned_cache(run):
    P, s, N, L = run["P"], run["s"], run["N"], run["L"]
    loc = to_dev(run["req"].local_positions(), torch.int32)
    k_re = torch.empty_like(run["k_in"])
    P.rope_realign(run["ctx"], k_re, run["k_in"], loc, run["pos"], L, N, N * s.kvd)
    torch.cuda.synchronize()
    for i in range(L):
        keep = np.setdiff1d(np.arange(N), run["sel"][i]) if i > 0 else np.arange(N)
        kt = torch.from_numpy(keep).to(DEV)
        assert torch.equal(run["kb"][i][kt], k_re[i][kt]), f"layer {i}: K changed"
        assert torch.equal(run["vb"][i][kt], run["v_in"][i][kt]), f"layer {i}: V changed"


def test_stepped_layers_match_forward(run):
    """cb_blend_layer replay of the forward's selections reproduces the forward."""
    P, s, N, L, ks = run["P"], run["s"], run["N"], run["L"], run["ks"]
    ctx, mw = run["ctx"], run["mw"]
    kb = run["k_in"].clone()
    vb = run["v_in"].clone()
    loc = to_dev(run["req"].local_positions(), torch.int32)
    P.rope_realign(ctx, kb, kb, loc, run["pos"], L, N, N * s.kvd)
    h = torch.zeros(N, s.d_model, dtype=torch.float32, device=DEV)
    h[:N] = P.api.op_embed(ctx, mw.embed, run["tok"])
    cand = torch.arange(N, dtype=torch.int32, device=DEV)
    for i in range(L):
        if i == 0:
            P.blend_layer(ctx, 0, mw, h, cand, N, 0, kb[0], vb[0], run["pos"], N)
            sel_i, dev_i = cand, None
        else:
            fs = to_dev(run["sel"][i], torch.int32)
            sel_i, dev_i = P.blend_layer(ctx, i, mw, h, cand, ks[i], 0, kb[i], vb[i], run["pos"], N, force_sel=fs,
                                         want_dev=True)
        torch.cuda.synchronize()
        # the forward additionally fuses the next layer's RMSNorm into the down projection (R15): equal up
        # to that rounding
        assert rel_err(np32(kb[i]), np32(run["kb"][i])) < 1e-2 and rel_err(np32(vb[i]), np32(run["vb"][i])) < 1e-2
        if i > 0:
            assert rel_err(dev_i.cpu().numpy(), run["dev"][i][:cand.numel()]) < 2e-2, f"layer {i}: dev vs forward"
        cand = sel_i.clone()
    assert rel_err(np32(h[:ks[L - 1]]), np32(run["h"][:ks[L - 1]])) < 1e-2, "stepped final h vs forward"
