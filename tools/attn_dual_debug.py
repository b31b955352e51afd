"""Compare attn_dual_kernel with attn_tc5_kernel row by row on one shape (debugging aid, needs a B200).
python tools/attn_dual_debug.py T n_sel n_kv [splits...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    T, n_sel, n_kv = (int(x) for x in sys.argv[1:4])
    splits = [int(x) for x in sys.argv[4:]] or [1, 2, 3]
    from paper_2405_16444_b200.build import build
    build()
    import paper_2405_16444_b200 as P
    from tests.helpers import shape
    s = shape("small", n_kv_heads=n_kv)
    from synth import counter_rng as rng
    gv = lambda st, n, H: rng.values(12, st, n * H * s.head_dim, 1.0, 0.0, "bf16").reshape(n, H, s.head_dim)
    qa, ka, va = gv(1, T, s.n_q_heads), gv(2, T, s.n_kv_heads), gv(3, T, s.n_kv_heads)
    rows = np.sort(np.random.default_rng(T).choice(T, n_sel, replace=False)).astype(np.int32)
    cv = lambda x: torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16).cuda()
    qperm = np.random.default_rng(1).permutation(n_sel).astype(np.int32)
    qbuf = np.zeros_like(qa[:n_sel])
    qbuf[qperm] = qa[rows]
    q = cv(qbuf.reshape(n_sel, -1))
    from oracle import cacheblend_oracle as O
    ref = O.causal_attention(qa[rows], rows, ka, va, np.arange(T)).reshape(n_sel, -1)
    k, v = cv(ka), cv(va)
    qrow = torch.from_numpy(qperm).cuda()
    qtok = torch.from_numpy(rows).cuda()
    ctx = P.Context(s, "bf16", max_tokens=T)
    for sp in splits:
        ctx.set_option("attn_splits", sp)
        ctx.set_option("attn_dual", 0)
        a = P.api.op_attention(ctx, q, qrow, qtok, k, v, T, impl=2).float().cpu()
        ctx.set_option("attn_dual", 1)
        b = P.api.op_attention(ctx, q, qrow, qtok, k, v, T, impl=2).float().cpu()
        d = (a - b).abs().reshape(n_sel, s.n_q_heads, s.head_dim)
        rel = float((a - b).norm() / a.norm())
        ea = np.linalg.norm(a.numpy() - ref) / np.linalg.norm(ref)
        eb = np.linalg.norm(b.numpy() - ref) / np.linalg.norm(ref)
        print(f"  vs oracle: tc5 {ea:.3e} dual {eb:.3e}")
        bad = (d.amax(-1) > 0.05).nonzero()
        print(f"splits={sp} rel={rel:.3e} bad (row, head) pairs={len(bad)}")
        if len(bad):
            rr = bad[:, 0].unique()
            print("  bad rows (token):", [(int(r), int(rows[r])) for r in rr[:20]])
            print("  bad heads:", bad[:, 1].unique().tolist()[:20])
            r0, h0 = bad[0].tolist()
            print("  cols of first bad:", (d[r0, h0] > 0.05).nonzero().flatten().tolist()[:40])


if __name__ == "__main__":
    main()
