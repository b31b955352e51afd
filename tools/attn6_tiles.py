"""Per-key-tile timeline (clock64) of CTA 0's first item in the persistent attention (impl 4).
Build with CB_EXTRA_NVCC=-DCB_ATTN_TRACE (build --force). python tools/attn6_tiles.py [n_sel]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    n_sel = int(sys.argv[1]) if len(sys.argv) > 1 else 460
    import paper_2405_16444_b200 as P
    from synth import workload as W
    s = W.MODELS["mistral-7b"]
    T = 3072
    ctx = P.Context(s, "bf16", max_tokens=T)
    k = torch.randn(T, s.n_kv_heads, s.head_dim, device="cuda").to(torch.bfloat16)
    v = torch.randn_like(k)
    rows = np.sort(np.random.default_rng(n_sel).choice(T, n_sel, replace=False)).astype(np.int32)
    q = torch.randn(n_sel, s.n_q_heads * s.head_dim, device="cuda").to(torch.bfloat16)
    qrow = torch.arange(n_sel, dtype=torch.int32, device="cuda")
    qtok = torch.from_numpy(rows).cuda()
    for i in range(4):
        ctx.set_option("debug_trace", 1 if i == 3 else 0)
        P.api.op_attention(ctx, q, qrow, qtok, k, v, T, impl=4)
    torch.cuda.synchronize()
    raw = (ctypes.c_int64 * 2048)()
    P.api.check(P.api.lib().cb_debug_fetch(ctx.handle, raw, 2048))
    a = np.array(raw[1792:1792 + 192], dtype=np.int64).reshape(48, 4)
    b = np.array(raw[1792 + 200:1792 + 248], dtype=np.int64).reshape(12, 4)
    t0 = a[a > 0].min()
    us = lambda x: (x - t0) / 1965.0 if x else float("nan")
    print(" t |  S issue  PV issue | s_full   P done   (us, clock64 / 1.965 GHz)")
    for t in range(48):
        if a[t].max() == 0:
            break
        extra = ""
        if t < 12 and b[t].max() > 0:
            extra = f" | ld {us(b[t, 0]):6.2f} max {us(b[t, 1]):6.2f} exp {us(b[t, 2]):6.2f}"
        print(f"{t:2d} | {us(a[t, 0]):7.2f} {us(a[t, 1]):8.2f} | {us(a[t, 2]):7.2f} {us(a[t, 3]):7.2f}" + extra)


if __name__ == "__main__":
    main()
