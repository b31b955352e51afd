"""Per-CTA spans of the per-tile tcgen05 attention (build with CB_EXTRA_NVCC=-DCB_ATTN_TRACE).
python tools/attn_spans.py [n_sel] [splits]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    n_sel = int(sys.argv[1]) if len(sys.argv) > 1 else 460
    splits = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    import paper_2405_16444_b200 as P
    from synth import workload as W
    s = W.MODELS["mistral-7b"]
    T = 3072
    ctx = P.Context(s, "bf16", max_tokens=T)
    ctx.set_option("attn_splits", splits)
    ctx.set_option("pdl", int(os.environ.get("CB_PDL", "1")))
    k = torch.randn(T, s.n_kv_heads, s.head_dim, device="cuda").to(torch.bfloat16)
    v = torch.randn_like(k)
    rows = np.sort(np.random.default_rng(n_sel).choice(T, n_sel, replace=False)).astype(np.int32)
    q = torch.randn(n_sel, s.n_q_heads * s.head_dim, device="cuda").to(torch.bfloat16)
    qrow = torch.arange(n_sel, dtype=torch.int32, device="cuda")
    qtok = torch.from_numpy(rows).cuda()
    for i in range(4):
        ctx.set_option("debug_trace", 1 if i == 3 else 0)
        P.api.op_attention(ctx, q, qrow, qtok, k, v, T, impl=2)
    torch.cuda.synchronize()
    raw = (ctypes.c_int64 * 2048)()
    P.api.check(P.api.lib().cb_debug_fetch(ctx.handle, raw, 2048))
    a = np.array(raw[1300:1300 + 740], dtype=np.int64).reshape(370, 2)
    used = a[:, 0] > 0
    t0 = a[used, 0].min()
    spans = [(i, (a[i, 0] - t0) / 1e3, (a[i, 1] - t0) / 1e3) for i in range(370) if used[i]]
    ends = sorted(e for _, _, e in spans)
    print(f"{len(spans)} CTAs, last end {ends[-1]:.1f} us, median end {ends[len(ends) // 2]:.1f}")
    step = int(os.environ.get("SPAN_STEP", "8"))
    G, n_kv = s.n_q_heads // s.n_kv_heads, s.n_kv_heads
    tiles = (n_sel * G + 127) // 128
    ns = max(splits, 1)

    def n_kt(cta):  # key tiles of the CTA's range (no pairing): row tile p holds tokens [32 p, 32 p + 32)
        rest = cta // n_kv
        p = tiles - 1 - rest // ns
        last = rows[min(n_sel, (p + 1) * 128 // G) - 1]
        kt = (int(last) + 1 + 127) // 128
        if ns == 1:
            return kt
        per = (24 + ns - 1) // ns  # kt_per_split for T = 3072 keys
        sp = rest % ns
        return max(0, min(kt, (sp + 1) * per) - sp * per)
    for i, b, e in spans[::step]:
        k_ = n_kt(i)
        extra = f"  kt={k_:3d}  {(e - b) / max(k_, 1):5.2f} us/tile"
        print(f"{i:4d} {b:7.2f} -> {e:7.2f}  ({e - b:6.2f}){extra}")


if __name__ == "__main__":
    main()
