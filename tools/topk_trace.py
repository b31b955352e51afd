"""Phase timeline of the last top-k launch of a blend step (debug_trace 200): python tools/topk_trace.py
(runs bench-shaped Mistral inputs with random caches; needs a B200)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import paper_2405_16444_b200 as P
    from synth import workload as W
    s = W.MODELS["mistral-7b"]
    req = W.Request([512] * 6, 0, 1, 0.15)
    N, L = req.n_ctx, s.n_layers
    ctx = P.Context(s, "bf16", max_tokens=N, max_pos=2 * N)
    mw = P.ModelWeights.synth(s, 1, "bf16", "cuda")
    k_in = torch.randn(L, N, s.n_kv_heads, s.head_dim, device="cuda").to(torch.bfloat16)
    v_in = torch.randn_like(k_in)
    k_out, v_out = torch.empty_like(k_in), torch.empty_like(v_in)
    tok = torch.from_numpy(req.tokens(s.vocab)).cuda()
    pos = torch.from_numpy(req.global_positions()).cuda()
    ks = P.schedule(0.15, N, L)
    for kv in filter(None, os.environ.get("CB_OPTS", "").split(",")):  # e.g. CB_OPTS=topk_drop2=0
        name, val = kv.split("=")
        ctx.set_option(name, int(val))
    for trace in (0, 0, 200):
        ctx.set_option("debug_trace", trace)
        P.blend_forward(ctx, mw, tok, pos, list(req.chunk_starts()), 0, k_in, v_in, k_out, v_out, ks)
    torch.cuda.synchronize()
    raw = (ctypes.c_int64 * 8)()
    P.api.check(P.api.lib().cb_debug_fetch(ctx.handle, raw, 8))
    t = np.array(raw[:5], dtype=np.int64)
    print("top-k phases (us from entry): inputs visible %.2f, Delta_kv summed %.2f, selected %.2f, done %.2f"
          % tuple((t[1:] - t[0]) / 1e3))


if __name__ == "__main__":
    main()
