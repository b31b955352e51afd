"""Per-k-block timeline of pair 0 of one CTA-pair GEMM launch (debug_trace 300): when each CTA's producer got
the stage back (empty wait done, ~ TMA issue) and when the leader's MMA warp saw it full (data landed, if the
MMA warp was already waiting). python tools/gemm_stages.py M N K [bn] [resid]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    M, N, K = (int(x) for x in sys.argv[1:4])
    bn = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    resid = len(sys.argv) > 5 and sys.argv[5] == "1"
    mc = int(sys.argv[6]) if len(sys.argv) > 6 else 0
    import paper_2405_16444_b200 as P
    from synth import workload as W
    ctx = P.Context(W.MODELS["mistral-7b"], "bf16", max_tokens=8)
    ctx.set_option("gemm_pair", 1)
    ctx.set_option("gemm_bn", bn)
    ctx.set_option("gemm_mc", mc)
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    C = torch.zeros(M, N, device="cuda", dtype=torch.float32)
    for it in range(4):
        ctx.set_option("debug_trace", 300 if it == 3 else 0)
        if resid:
            P.api.op_gemm_resid(ctx, A, B, C, impl=2)
        else:
            P.api.op_gemm(ctx, A, B, impl=2)
    torch.cuda.synchronize()
    raw = (ctypes.c_int64 * 2048)()
    P.api.check(P.api.lib().cb_debug_fetch(ctx.handle, raw, 2048))
    a = np.array(raw[:], dtype=np.int64)
    p0, p1, mf = a[0:256], a[256:512], a[512:768]
    nkb = int((mf > 0).sum())
    t0 = min(p0[p0 > 0].min(), p1[p1 > 0].min(), mf[mf > 0].min())
    f = lambda x: (x - t0) / 1000.0
    print(f"M={M} N={N} K={K} bn={bn} mc={mc} k-blocks traced {nkb}")
    print("  kb   prod0   prod1   mma_full   issue->full(us)   mma gap(ns)")
    for kb in range(nkb):
        iss = max(p0[kb], p1[kb]) if p0[kb] > 0 and p1[kb] > 0 else 0
        lat = (mf[kb] - iss) / 1000.0 if iss else float("nan")
        gap = (mf[kb] - mf[kb - 1]) if kb > 0 else 0
        print(f"{kb:4d} {f(p0[kb]) if p0[kb] else float('nan'):7.2f} {f(p1[kb]) if p1[kb] else float('nan'):7.2f} "
              f"{f(mf[kb]):9.2f}   {lat:8.2f}   {gap:8d}")
    gaps = np.diff(mf[:nkb])
    print(f"median MMA gap {np.median(gaps):.0f} cycles, mean {gaps.mean():.0f} (clock64: the two CTAs count on their own SMs)")


if __name__ == "__main__":
    main()
