"""Run one tcgen05 GEMM shape a few times (for ncu). python tools/gemm_one.py M N K sched [bn] [iters]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    M, N, K, sched = (int(x) for x in sys.argv[1:5])
    bn = int(sys.argv[5]) if len(sys.argv) > 5 else 0
    iters = int(sys.argv[6]) if len(sys.argv) > 6 else 3
    import paper_2405_16444_b200 as P
    from synth import workload as W
    ctx = P.Context(W.MODELS["mistral-7b"], "bf16", max_tokens=8)
    ctx.set_option("gemm_sched", sched)
    ctx.set_option("gemm_bn", bn)
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    for _ in range(iters):
        P.api.op_gemm(ctx, A, B, impl=2)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
