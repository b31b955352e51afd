"""o_proj at the last blend layer (401 x 4096 x 4096): cuBLAS, the library pair GEMM (bn 128) and the library
single-CTA GEMM (bn 128), one launch each after warm-up, for an ncu comparison."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2405_16444_b200 as P
from synth import workload as W
M, N, K = 401, 4096, 4096
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
ctx = P.Context(W.MODELS["mistral-7b"], "bf16", max_tokens=8)
st = torch.cuda.current_stream().cuda_stream
def ours(pair):
    ctx.set_option("gemm_pair", pair)
    ctx.set_option("gemm_bn", 128)
    P.api.check(P.api.lib().cb_op_gemm(ctx.handle, A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, 0, 2, st))
for _ in range(3):
    torch.mm(A, B.t(), out=C); ours(1); ours(2)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
torch.mm(A, B.t(), out=C); ours(1); ours(2)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
