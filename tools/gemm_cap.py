"""Blend-size GEMM time vs the number of CTA pairs the planner may use (gemm_cap_* options).
At full load the pair mainloop is power-capped (~430 ns per 256x256x64 k-block with 74 pairs busy vs
~290 ns with a few), so fewer pairs over exact rounds can beat a ragged last round.
python tools/gemm_cap.py [iters]   (needs a B200)"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    from paper_2405_16444_b200.build import build
    build()
    import paper_2405_16444_b200 as P
    from synth import workload as W
    s = W.MODELS["mistral-7b"]
    ctx = P.Context(s, "bf16", max_tokens=8)
    d, qd, kvd, ff = s.d_model, s.qd, s.kvd, s.d_ff
    shapes = [("qkv", qd + 2 * kvd, d, False), ("o", d, qd, True), ("gate_up", 2 * ff, d, False),
              ("down", d, ff, True)]
    caps = [0, 72, 70, 64, 60, 56, 48, 37]
    for M in (369, 450, 540):
        A = torch.randn(M, max(d, ff), device="cuda").to(torch.bfloat16)
        for name, N, K, resid in shapes:
            a = A[:, :K].contiguous()
            B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
            C = torch.zeros(M, N, device="cuda")
            kind = "resid" if resid else "store"
            row = []
            for cap in caps:
                ctx.set_option(f"gemm_cap_{kind}", cap)
                f = (lambda: P.api.op_gemm_resid(ctx, a, B, C)) if resid else (lambda: P.api.op_gemm(ctx, a, B))
                for _ in range(3):
                    f()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                for _ in range(iters):
                    f()
                e1.record()
                torch.cuda.synchronize()
                row.append(e0.elapsed_time(e1) / iters * 1e3)
            ctx.set_option(f"gemm_cap_{kind}", 0)
            print(f"M={M} {name:8s} " + "  ".join(f"cap{c or 74}:{t:6.1f}" for c, t in zip(caps, row)), flush=True)


if __name__ == "__main__":
    main()
