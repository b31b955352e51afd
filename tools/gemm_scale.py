"""Per-tile mainloop time of the CTA-pair GEMM vs the number of concurrently busy pairs (full-load scaling check).
python tools/gemm_scale.py [M] [K]   (STORE epilogue, pair 256x256 tiles; needs a B200)"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    M = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
    import paper_2405_16444_b200 as P
    from synth import workload as W
    ctx = P.Context(W.MODELS["mistral-7b"], "bf16", max_tokens=8)
    ctx.set_option("gemm_pair", 1)
    ctx.set_option("gemm_bn", int(os.environ.get("BN", "256")))
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    bn = int(os.environ.get("BN", "256"))
    mt = (M + 255) // 256
    for tiles in [2, 8, 16, 32, 48, 64, 74, 148, 222]:
        N = tiles // mt * bn
        if N <= 0:
            continue
        B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
        f = lambda: P.api.op_gemm(ctx, A, B, impl=2)
        for _ in range(3):
            f()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(20):
            f()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 20 * 1e3
        waves = -(-(mt * (N // bn)) // 74)
        print(f"M={M} N={N:6d} K={K} tiles={mt * (N // bn):4d} waves={waves}: {us:7.1f} us  "
              f"{us / waves:6.1f} us/wave  {us / waves / (K // 64) * 1e3:6.1f} ns/kb  "
              f"{2 * M * N * K / us / 1e6:7.1f} TFLOP/s", flush=True)


if __name__ == "__main__":
    main()
