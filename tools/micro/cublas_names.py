"""cuBLAS kernel choice for the blend's GEMM shapes (run under ncu to see names, grids, clusters)."""
import sys
import torch
SH = [(579, 6144, 4096), (579, 4096, 4096), (579, 28672, 4096), (579, 4096, 14336), (401, 6144, 4096),
      (401, 4096, 4096), (401, 28672, 4096), (401, 4096, 14336)]
for M, N, K in SH:
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    for _ in range(2):
        C = torch.mm(A, B.t())
    torch.cuda.synchronize()
