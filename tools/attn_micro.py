"""Micro-benchmark of the sparse-query attention kernels on blend shapes (Mistral: 32 q / 8 kv heads).

python tools/attn_micro.py [--iters 30]   (needs a B200)"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--splits", default="0,1,2,3,4,6")
    ap.add_argument("--impls", default="2")
    ap.add_argument("--pairs", default="0,1")
    ap.add_argument("--pdl", type=int, default=1)
    a = ap.parse_args()
    from paper_2405_16444_b200.build import build
    build()
    import paper_2405_16444_b200 as P
    from synth import workload as W
    s = W.MODELS["mistral-7b"]
    T = 3072
    ctx = P.Context(s, "bf16", max_tokens=T)
    ctx.set_option("pdl", a.pdl)
    k = torch.randn(T, s.n_kv_heads, s.head_dim, device="cuda").to(torch.bfloat16)
    v = torch.randn_like(k)
    for n_sel in (3072, 553, 460, 369):
        rows = np.sort(np.random.default_rng(n_sel).choice(T, n_sel, replace=False)).astype(np.int32)
        q = torch.randn(n_sel, s.n_q_heads * s.head_dim, device="cuda").to(torch.bfloat16)
        qrow = torch.arange(n_sel, dtype=torch.int32, device="cuda")
        qtok = torch.from_numpy(rows).cuda()
        flops = 4.0 * s.n_q_heads * s.head_dim * float(np.sum(rows + 1))
        for impl, splits, pair in [(int(i), int(x), int(pp)) for i in a.impls.split(",") for x in a.splits.split(",")
                                   for pp in a.pairs.split(",")]:
            ctx.set_option("attn_splits", splits)
            ctx.set_option("attn_pair", pair)
            fn = lambda: P.api.op_attention(ctx, q, qrow, qtok, k, v, T, impl=impl)
            for _ in range(3):
                fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(a.iters):
                fn()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / a.iters * 1e3
            print(f"rows={n_sel:5d} impl={impl} splits={splits} pair={pair}: {us:8.1f} us  {flops / us / 1e6:7.1f} TFLOP/s",
                  flush=True)


if __name__ == "__main__":
    main()
