"""Run small blends through the C-ABI for compute-sanitizer (memcheck / racecheck / synccheck).

  compute-sanitizer --tool memcheck python tools/sanitize_blend.py [case ...]

Cases exercise every kernel family on the blend path, including the cross-CTA protocols: the pair
GEMM with a forced split-K chain (`gemm_ksplit`), with the tail pieces (`gemm_tail`) and in TMA-multicast
clusters of 4 and 8 CTAs (`gemm_mc`), attention
with forced split-KV and the last-arriver merge (`attn_splits`), the top-k kernel, the request path.
Inputs are seeded synthetic (random chunk caches), no oracle: this checks memory/sync hazards only.
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_16444_b200 as P  # noqa: E402
from synth import workload as W  # noqa: E402

CASES = {
    # name: (shape, dtype, chunk lens, n_suffix, ratio, options)
    "tiny_f32": ("tiny", "f32", [32, 32, 32], 0, 0.15, {}),
    "tiny_f32_suffix": ("tiny", "f32", [17, 40, 9], 5, 0.3, {}),
    "small_bf16": ("small", "bf16", [200, 317, 150], 0, 0.15, {}),
    "small_bf16_ksplit": ("small", "bf16", [200, 317, 150], 9, 0.15, {"gemm_ksplit": 3}),
    "small_bf16_tail": ("small", "bf16", [200, 317, 150], 0, 0.15, {"gemm_tail": 2}),
    "small_bf16_attn_split": ("small", "bf16", [200, 317, 150], 0, 0.3, {"attn_splits": 3}),
    "small_bf16_single_cta": ("small", "bf16", [200, 317, 150], 0, 0.15, {"gemm_pair": 2}),
    "small_bf16_mc4": ("small", "bf16", [200, 317, 150], 6, 0.15, {"gemm_mc": 1}),
    "small_bf16_mc8": ("small", "bf16", [200, 317, 150], 6, 0.15, {"gemm_mc": 3}),
}


def shape(name):
    return W.MODELS[name]


def run(name):
    sname, dtype, lens, n_suf, ratio, opts = CASES[name]
    s = shape(sname)
    req = W.Request(lens, n_suf, 7, ratio)
    N, T, L = req.n_ctx, req.n_total, s.n_layers
    td = P.api.TORCH_DTYPES[dtype]
    ctx = P.Context(s, dtype, max_tokens=T, max_pos=2 * T)
    if os.environ.get("CB_SAN_NO_PDL"):  # racecheck: no cross-kernel CTA overlap on one SM
        ctx.set_option("pdl", 0)
    for k, v in opts.items():
        ctx.set_option(k, v)
    mw = P.ModelWeights.synth(s, 7, dtype, "cuda")
    kc = np.stack([W.random_cache(s, i, N, 7, "f32", "k") for i in range(L)])
    vc = np.stack([W.random_cache(s, i, N, 7, "f32", "v") for i in range(L)])
    k_in = torch.from_numpy(kc).to("cuda", td)
    v_in = torch.from_numpy(vc).to("cuda", td)
    kb = torch.empty((L, T, s.n_kv_heads, s.head_dim), dtype=td, device="cuda")
    vb = torch.empty_like(kb)
    tok = torch.from_numpy(req.tokens(s.vocab)).cuda()
    pos = torch.from_numpy(req.global_positions()).cuda()
    ks = P.schedule(ratio, N, L)
    sel = torch.empty(L, N, dtype=torch.int32, device="cuda")
    h = P.blend_forward(ctx, mw, tok, pos, list(req.chunk_starts()), n_suf, k_in, v_in, kb, vb, ks, sel_out=sel)
    torch.cuda.synchronize()
    ctx.check_device_errors()
    # the host-buffer request path (copy stream + per-layer events)
    h_host = torch.empty(h.shape, dtype=torch.float32).pin_memory()
    P.api.blend_request(ctx, mw, tok.cpu(), pos.cpu(), list(req.chunk_starts()), n_suf, k_in.cpu().pin_memory(),
                    v_in.cpu().pin_memory(), kb, vb, ks, h_host)
    torch.cuda.synchronize()
    ctx.check_device_errors()
    print(f"{name}: ok, h {tuple(h.shape)} finite={bool(torch.isfinite(h).all())}", flush=True)
    ctx.close()


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        run(n)
