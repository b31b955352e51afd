"""gemm_mc (A-multicast 4-CTA clusters, A+B-multicast 8-CTA clusters) against the plain pair GEMM: bitwise equal outputs (same accumulation
order), plain store and residual epilogues, even and odd column-tile counts."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2405_16444_b200 as P
from synth import workload as W
ctx = P.Context(W.MODELS["mistral-7b"], "bf16", max_tokens=8)
print("max 4-CTA clusters", ctx.info("gemm_max_clusters4"), "max 8-CTA clusters", ctx.info("gemm_max_clusters8"),
      flush=True)
st = torch.cuda.current_stream().cuda_stream
ok = True
for M, N, K, bn in [(401, 4096, 4096, 128), (579, 4096, 4096, 192), (579, 6144, 4096, 0), (300, 4224, 1024, 128),
                    (1000, 2048, 512, 256), (37, 384, 256, 128)]:
    g = torch.Generator(device="cuda").manual_seed(M)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda", generator=g).to(torch.bfloat16)
    outs = []
    for mc in (0, 1, 3):
        ctx.set_option("gemm_mc", mc)
        ctx.set_option("gemm_pair", 1)
        ctx.set_option("gemm_bn", bn)
        C16 = torch.full((M, N), float("nan"), device="cuda", dtype=torch.bfloat16)
        P.api.check(P.api.lib().cb_op_gemm(ctx.handle, A.data_ptr(), B.data_ptr(), C16.data_ptr(), M, N, K, 0, 2, st))
        C32 = torch.ones(M, N, device="cuda", dtype=torch.float32)
        P.api.check(P.api.lib().cb_op_gemm(ctx.handle, A.data_ptr(), B.data_ptr(), C32.data_ptr(), M, N, K, 2, 2, st))
        torch.cuda.synchronize()
        outs.append((C16, C32))
    ref = (A.float() @ B.float().t())
    e = ((outs[1][0].float() - ref).norm() / ref.norm()).item()
    same = all(torch.equal(outs[0][0], o[0]) and torch.equal(outs[0][1], o[1]) for o in outs[1:])
    ok &= same and e < 1e-2
    print(f"M={M} N={N} K={K} bn={bn}: mc=1 and mc=3 bitwise equal to mc=0: {same}, rel err vs fp32 {e:.2e}", flush=True)
print("ALL OK" if ok else "MISMATCH")
