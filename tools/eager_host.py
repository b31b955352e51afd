"""Host cost of an eager (non-graph) blend: wall time per cb_blend_forward call with the GPU work queued
behind it vs the graph replay, Mistral 6x512 bench workload. python tools/eager_host.py (needs a B200)"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2405_16444_b200.build import build
    build()
    import paper_2405_16444_b200 as P
    from synth import workload as W
    s = W.MODELS["mistral-7b"]
    req = W.Request([512] * 6, 0, 1, 0.15)
    N, L = req.n_ctx, s.n_layers
    ctx = P.Context(s, "bf16", max_tokens=N, max_pos=2 * N)
    mw = P.ModelWeights.synth(s, 1, "bf16", "cuda")
    tok = torch.from_numpy(req.tokens(s.vocab)).cuda()
    pos = torch.from_numpy(req.global_positions()).cuda()
    k_in = torch.randn(L, N, s.n_kv_heads, s.head_dim, device="cuda").to(torch.bfloat16)
    v_in = torch.randn_like(k_in)
    kb, vb = torch.empty_like(k_in), torch.empty_like(v_in)
    ks = P.schedule(0.15, N, L)
    h = torch.empty(ks[-1], s.d_model, device="cuda")
    f = lambda: P.blend_forward(ctx, mw, tok, pos, list(req.chunk_starts()), 0, k_in, v_in, kb, vb, ks, h_out=h)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    n = 10
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        f()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    for _ in range(n):
        g.replay()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"eager: host enqueue {(t1 - t0) / n * 1e3:.2f} ms per blend, wall {(t2 - t0) / n * 1e3:.2f} ms; "
          f"graph replay wall {(t4 - t3) / n * 1e3:.2f} ms")


if __name__ == "__main__":
    main()
