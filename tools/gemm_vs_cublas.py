"""The blend's projection GEMMs: the library's tcgen05 pair GEMM (cb_op_gemm) next to cuBLAS (torch.mm) on the
same shapes, weights rotated through copies totalling > 2x L2 so each call streams its weights from HBM as in
the blend step.

python tools/gemm_vs_cublas.py [--iters 40]   (needs a B200)"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

SHAPES = [  # (name, M, N, K): Mistral-7B blend at r = 0.15 (layer 2: 547 + 32 rows; layer 31: 369 + 32)
    ("qkv_l2", 579, 6144, 4096), ("o_l2", 579, 4096, 4096), ("gu_l2", 579, 28672, 4096),
    ("down_l2", 579, 4096, 14336), ("qkv_l31", 401, 6144, 4096), ("o_l31", 401, 4096, 4096),
    ("gu_l31", 401, 28672, 4096), ("down_l31", 401, 4096, 14336), ("kv_l1", 3104, 2048, 4096),
    ("gu_l0", 3104, 28672, 4096),
]


def timed(fn, iters):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=40)
    ap.add_argument("--l2-bytes", type=float, default=126e6)
    a = ap.parse_args()
    from paper_2405_16444_b200.build import build
    build()
    import paper_2405_16444_b200 as P
    from synth import workload as W
    ctx = P.Context(W.MODELS["mistral-7b"], "bf16", max_tokens=8)
    st = torch.cuda.current_stream().cuda_stream
    out = {}
    for name, M, N, K in SHAPES:
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        nb = max(2, int(2 * a.l2_bytes // (N * K * 2)) + 1)
        Bs = [torch.randn(N, K, device="cuda").to(torch.bfloat16) for _ in range(nb)]
        C16 = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        C32 = torch.zeros(M, N, device="cuda", dtype=torch.float32)
        it = {"i": 0}

        def nxt():
            it["i"] = (it["i"] + 1) % nb
            return Bs[it["i"]]

        ours = timed(lambda: P.api.check(P.api.lib().cb_op_gemm(ctx.handle, A.data_ptr(), nxt().data_ptr(),
                                                                 C16.data_ptr(), M, N, K, 0, 2, st)), a.iters)
        ours_r = timed(lambda: P.api.check(P.api.lib().cb_op_gemm(ctx.handle, A.data_ptr(), nxt().data_ptr(),
                                                                   C32.data_ptr(), M, N, K, 2, 2, st)), a.iters)
        cub = timed(lambda: torch.mm(A, nxt().t(), out=C16), a.iters)
        fl = 2.0 * M * N * K
        out[name] = dict(M=M, N=N, K=K, ours_us=round(ours, 1), ours_resid_us=round(ours_r, 1),
                         cublas_us=round(cub, 1), ours_tf=round(fl / ours / 1e6, 1),
                         cublas_tf=round(fl / cub / 1e6, 1))
        print(f"{name:9s} M={M:5d} N={N:6d} K={K:6d}  ours {ours:7.1f} us ({fl / ours / 1e6:6.1f} TF/s)  "
              f"ours+resid {ours_r:7.1f} us  cuBLAS {cub:7.1f} us ({fl / cub / 1e6:6.1f} TF/s)", flush=True)
        del Bs
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
