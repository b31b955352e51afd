"""Per-CTA item timeline of the persistent tcgen05 attention (impl 4) on a Mistral-shaped layer.
python tools/attn6_trace.py [n_sel] [splits]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    n_sel = int(sys.argv[1]) if len(sys.argv) > 1 else 460
    splits = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    import paper_2405_16444_b200 as P
    from synth import workload as W
    s = W.MODELS["mistral-7b"]
    T = 3072
    ctx = P.Context(s, "bf16", max_tokens=T)
    ctx.set_option("attn_splits", splits)
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
    a = np.array(raw[:], dtype=np.int64)
    t = a[:1184].reshape(148, 8)[:, :6]
    kk = a[1184:1184 + 592].reshape(148, 4)[:, :3]
    t0 = t[t > 0].min()
    print("cta | item k (nt): start -> end (us)")
    for c in range(148):
        parts = []
        for it in range(3):
            if t[c, 2 * it] > 0:
                parts.append(f"k={kk[c, it] // 64:4d} nt={kk[c, it] % 64:2d}: {(t[c, 2 * it] - t0) / 1e3:6.2f}->"
                             f"{(t[c, 2 * it + 1] - t0) / 1e3:6.2f}")
        print(f"{c:3d} | " + " | ".join(parts))


if __name__ == "__main__":
    main()
