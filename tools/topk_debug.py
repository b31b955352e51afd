"""Debug helper: one kv_deviation_topk call per (threads, sort, n, k); prints deviations and slots."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_16444_b200 as P  # noqa: E402
from synth import workload as W  # noqa: E402

s = W.MODELS["small"]
ctx = P.Context(s, "bf16", max_tokens=1100)
for threads in (0, 256, 512):
    for n, k in [(2, 1), (5, 2), (37, 5)]:
        g = torch.Generator(device="cuda").manual_seed(threads + 1)
        kn = torch.randint(0, 3, (n, s.n_kv_heads, s.head_dim), device="cuda", generator=g).to(torch.bfloat16)
        kn[::3] = 0
        z = torch.zeros_like(kn)
        cand = torch.arange(n, dtype=torch.int32, device="cuda")
        ctx.set_option("topk_threads", threads)
        out = []
        for sort in (0, 1):
            ctx.set_option("topk_sort", sort)
            sel, slot, dev = P.api.kv_deviation_topk(ctx, kn, z, z, z, cand, k)
            torch.cuda.synchronize()
            out.append((slot.cpu().tolist(), dev.cpu().tolist()))
        print(threads, n, k, out, flush=True)
