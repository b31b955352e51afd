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
    ap.add_argument("--pdl", type=int, default=1)
    ap.add_argument("--rows", default="3072,553,460,369")
    ap.add_argument("--opts", default="", help="extra option sets to compare, ';'-separated, e.g. 'attn_splits=2;pdl=0'")
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
    base = {"attn_splits": 0}
    variants = [""] + [v for v in a.opts.split(";") if v]
    for n_sel in [int(x) for x in a.rows.split(",")]:
        rows = np.sort(np.random.default_rng(n_sel).choice(T, n_sel, replace=False)).astype(np.int32)
        q = torch.randn(n_sel, s.n_q_heads * s.head_dim, device="cuda").to(torch.bfloat16)
        qrow = torch.arange(n_sel, dtype=torch.int32, device="cuda")
        qtok = torch.from_numpy(rows).cuda()
        flops = 4.0 * s.n_q_heads * s.head_dim * float(np.sum(rows + 1))
        for impl, splits, var in [(int(i), int(x), v) for i in a.impls.split(",") for x in a.splits.split(",")
                                  for v in variants]:
            opts = dict(base)
            opts.update({"attn_splits": splits})
            opts.update({kv.split("=")[0]: int(kv.split("=")[1]) for kv in var.split(",") if kv})
            for name, val in opts.items():
                ctx.set_option(name, val)
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
            print(f"rows={n_sel:5d} impl={impl} splits={splits} [{var}]: {us:8.1f} us  "
                  f"{flops / us / 1e6:7.1f} TFLOP/s", flush=True)
            for kv in var.split(","):  # back to the defaults for the next variant
                if kv:
                    ctx.set_option(kv.split("=")[0], 0)


if __name__ == "__main__":
    main()
