// gemm_simt.cu — CUDA-core GEMM with the blend epilogues. Used for the fp32 parity mode (tcgen05 has
// no fp32-input MMA) and for shapes the tcgen05 kernel does not take. acc = A[M][K] . B[N][K]^T.
#include "ctx.h"

namespace {
constexpr int BM = 64, BN = 64, BK = 16;

template <typename T, bool SWIGLU>
__global__ void __launch_bounds__(256) gemm_simt_kernel(const T* __restrict__ A, int lda, const T* __restrict__ B,
                                                        int ldb, int M, int K, EpiParams e) {
  pdl_enter();
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  __shared__ float Bu[SWIGLU ? BK : 1][BN + 4];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int N = e.N;
  float acc[4][4] = {}, accu[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += BK) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int idx = tid + q * 256;  // 0..1023 -> (row, kk)
      const int r = idx >> 4, kk = idx & 15;
      const int gm = m0 + r, gn = n0 + r, gk = k0 + kk;
      As[kk][r] = (gm < M && gk < K) ? to_f(A[(size_t)gm * lda + gk]) : 0.f;
      Bs[kk][r] = (gn < N && gk < K) ? to_f(B[(size_t)gn * ldb + gk]) : 0.f;
      if constexpr (SWIGLU) Bu[kk][r] = (gn < N && gk < K) ? to_f(B[(size_t)(gn + e.ff) * ldb + gk]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], b[4], u[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        b[j] = Bs[kk][tx * 4 + j];
        if constexpr (SWIGLU) u[j] = Bu[kk][tx * 4 + j];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
          if constexpr (SWIGLU) accu[i][j] = fmaf(a[i], u[j], accu[i][j]);
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; j += 2) {
      const int n = n0 + tx * 4 + j;
      if (n >= N) continue;
      epi_pair<T>(e, m, n, acc[i][j], acc[i][j + 1], accu[i][j], accu[i][j + 1]);
    }
  }
  if (e.push_base[0] != nullptr) __threadfence_system();  // pushed rows reach the peers before the signal
}
}  // namespace

cb_status launch_gemm_simt(cb_ctx* c, const void* A, int lda, const void* B, int ldb, int M, int K,
                           const EpiParams& e, cudaStream_t s) {
  if (M == 0 || e.N == 0) return CB_OK;
  dim3 grid((e.N + BN - 1) / BN, (M + BM - 1) / BM);
  const bool sw = e.kind == EPI_SWIGLU;
  ProfScope ps_(c, PROF_GEMM, s);
  if (c->m.dtype == CB_BF16) {
    if (sw) CB_LAUNCH(c, (gemm_simt_kernel<bf16, true>), grid, 256, 0, s, (const bf16*)A, lda, (const bf16*)B, ldb, M, K, e);
    else CB_LAUNCH(c, (gemm_simt_kernel<bf16, false>), grid, 256, 0, s, (const bf16*)A, lda, (const bf16*)B, ldb, M, K, e);
  } else {
    if (sw) CB_LAUNCH(c, (gemm_simt_kernel<float, true>), grid, 256, 0, s, (const float*)A, lda, (const float*)B, ldb, M, K, e);
    else CB_LAUNCH(c, (gemm_simt_kernel<float, false>), grid, 256, 0, s, (const float*)A, lda, (const float*)B, ldb, M, K, e);
  }
  CB_LAUNCHED(c);
  return CB_OK;
}
