"""Per-CTA timeline (globaltimer) of one CTA-pair GEMM launch: python tools/gemm_trace.py M N K ksplit [resid]."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
EV = ["start", "tma_done", "mma_done", "tfull", "flag_ok", "epi_done", "end", "exit"]


def main():
    M, N, K, ks = (int(x) for x in sys.argv[1:5])
    resid = len(sys.argv) > 5 and sys.argv[5] == "1"
    import paper_2405_16444_b200 as P
    from synth import workload as W
    ctx = P.Context(W.MODELS["mistral-7b"], "bf16", max_tokens=8)
    ctx.set_option("gemm_pair", 1)
    ctx.set_option("gemm_ksplit", ks)
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    C = torch.zeros(M, N, device="cuda", dtype=torch.float32)
    for it in range(3):
        ctx.set_option("debug_trace", 1 if it == 2 else 0)
        if resid:
            P.api.op_gemm_resid(ctx, A, B, C, impl=2)
        else:
            P.api.op_gemm(ctx, A, B, impl=2)
    torch.cuda.synchronize()
    raw = (ctypes.c_int64 * 2048)()
    P.api.check(P.api.lib().cb_debug_fetch(ctx.handle, raw, 2048))
    full = np.array(raw[:], dtype=np.int64)
    t = full[:1024].reshape(128, 8)
    ch = full[1024:].reshape(128, 8)
    used = t[:, 0] > 0
    if len(sys.argv) > 6:
        used &= np.arange(128) < int(sys.argv[6])
    t0 = t[used, 0].min()
    rel = np.where(t > 0, (t - t0) / 1000.0, np.nan)[used]
    rch = np.where(ch > 0, (ch - t0) / 1000.0, np.nan)[used]
    print("cta  " + " ".join(f"{e:>9s}" for e in EV) + "   | epilogue chunk ends (warp 2)")
    for i, (r, c) in enumerate(zip(rel, rch)):
        print(f"{i:4d} " + " ".join(f"{x:9.2f}" for x in r) + "   | " + " ".join(f"{x:6.2f}" for x in c), flush=True)


if __name__ == "__main__":
    main()
