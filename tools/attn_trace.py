"""Pipeline timeline of one CTA (the heaviest: latest query tokens) of the tcgen05 attention kernel, from
the library's debug_trace clock64 events (build with CB_EXTRA_NVCC=-DCB_ATTN_TRACE ... build --force).
python tools/attn_trace.py [n_sel] [T]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    n_sel = int(sys.argv[1]) if len(sys.argv) > 1 else 553
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 3072
    import paper_2405_16444_b200 as P
    from synth import workload as W
    s = W.MODELS["mistral-7b"]
    ctx = P.Context(s, "bf16", max_tokens=T)
    ctx.set_option("attn_splits", int(os.environ.get("ATTN_SPLITS", "1")))
    k = torch.randn(T, s.n_kv_heads, s.head_dim, device="cuda").to(torch.bfloat16)
    v = torch.randn_like(k)
    rows = np.sort(np.random.default_rng(n_sel).choice(T, n_sel, replace=False)).astype(np.int32)
    q = torch.randn(n_sel, s.n_q_heads * s.head_dim, device="cuda").to(torch.bfloat16)
    qrow = torch.arange(n_sel, dtype=torch.int32, device="cuda")
    qtok = torch.from_numpy(rows).cuda()
    for _ in range(3):
        P.api.op_attention(ctx, q, qrow, qtok, k, v, T, impl=2)
    ctx.set_option("debug_trace", 1)
    P.api.op_attention(ctx, q, qrow, qtok, k, v, T, impl=2)
    torch.cuda.synchronize()
    buf = (ctypes.c_int64 * 2048)()
    P.api.check(P.api.lib().cb_debug_fetch(ctx.handle, buf, 2048))
    a = np.array(buf[:], dtype=np.int64)
    t0 = a[1200]
    us = lambda x: (x - t0) / 1.9e3 if x else float("nan")
    print(f"start 0, Q staged {us(a[1201]):.2f} us, end {us(a[1202]):.2f} us")
    nt = max(i for i in range(100) if a[800 + 4 * i]) + 1
    print(" t | K issue  V issue | S issue  PV issue | s_full  max_x  pv_done  p_full   (us)")
    for t in range(nt):
        print(f"{t:2d} | {us(a[4*t]):7.2f} {us(a[4*t+1]):7.2f} | {us(a[400+4*t]):7.2f} {us(a[400+4*t+1]):7.2f} | "
              f"{us(a[800+4*t]):7.2f} {us(a[800+4*t+1]):7.2f} {us(a[800+4*t+2]):7.2f} {us(a[800+4*t+3]):7.2f}")


if __name__ == "__main__":
    main()
