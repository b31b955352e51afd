"""Micro-benchmark of the tcgen05 GEMM on the blend's projection shapes (schedule / tile experiments).

python tools/gemm_micro.py [--iters 50]   (needs a B200)"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

SHAPES = [  # (name, M, N, K): Mistral-7B blend at r = 0.15 (M = k_i + 32 suffix rows)
    ("qkv_l1", 3104, 2048, 4096), ("qkv_l2", 579, 6144, 4096), ("o_l2", 579, 4096, 4096),
    ("gu_l2", 579, 28672, 4096), ("down_l2", 579, 4096, 14336), ("qkv_l31", 401, 6144, 4096),
    ("o_l31", 401, 4096, 4096), ("gu_l31", 401, 28672, 4096), ("down_l31", 401, 4096, 14336),
    ("gu_l0", 3104, 28672, 4096), ("down_l0", 3104, 4096, 14336),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--modes", default="0")
    ap.add_argument("--bns", default="0")
    ap.add_argument("--pairs", default="0")
    ap.add_argument("--ksplits", default="0")
    ap.add_argument("--resid", action="store_true", help="residual epilogue C += A.B^T (fp32 C)")
    ap.add_argument("--only", default="", help="comma list of shape names")
    ap.add_argument("--pdl", type=int, default=1)
    ap.add_argument("--mcs", default="0", help="gemm_mc values (A-multicast 4-CTA clusters)")
    ap.add_argument("--rotate", type=int, default=1,
                    help="cycle over this many copies of B (weights), so they stream from HBM as in the blend")
    a = ap.parse_args()
    from paper_2405_16444_b200.build import build
    build()
    import paper_2405_16444_b200 as P
    from synth import workload as W
    ctx = P.Context(W.MODELS["mistral-7b"], "bf16", max_tokens=8)
    res = {}
    ctx.set_option("pdl", a.pdl)
    print("num_sms", ctx.info("num_sms"), "gemm_max_pairs", ctx.info("gemm_max_pairs"), "max 4-CTA clusters",
          ctx.info("gemm_max_clusters4"), flush=True)
    only = set(a.only.split(",")) if a.only else None
    for name, M, N, K in SHAPES:
        if only and name not in only:
            continue
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        Bs = [torch.randn(N, K, device="cuda").to(torch.bfloat16) for _ in range(max(1, a.rotate))]
        C = torch.zeros(M, N, device="cuda", dtype=torch.float32 if a.resid else torch.bfloat16)
        for mode, bn, pr, ks, mc in [(int(m), int(b), int(p), int(k), int(x)) for m in a.modes.split(",")
                                     for b in a.bns.split(",") for p in a.pairs.split(",") for k in a.ksplits.split(",")
                                     for x in a.mcs.split(",")]:
            ctx.set_option("gemm_mc", mc)
            ctx.set_option("gemm_sched", mode)
            ctx.set_option("gemm_bn", bn)
            ctx.set_option("gemm_pair", pr)
            ctx.set_option("gemm_ksplit", ks)
            it = [0]

            def fn():
                B = Bs[it[0] % len(Bs)]
                it[0] += 1
                P.api.check(P.api.lib().cb_op_gemm(ctx.handle, A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K,
                                                   2 if a.resid else 0, 2, torch.cuda.current_stream().cuda_stream))
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
            tf = 2.0 * M * N * K / (us * 1e-6) / 1e12
            res[f"{name}/m{mode}/bn{bn}/p{pr}/k{ks}/mc{mc}"] = (round(us, 1), round(tf, 1))
            print(f"{name:10s} M={M:5d} N={N:6d} K={K:6d} mode={mode} bn={bn} pair={pr} ks={ks} mc={mc}: {us:8.1f} us "
                  f"{tf:7.1f} TFLOP/s", flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
