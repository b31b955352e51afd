// attention_simt.cu — CUDA-core sparse-query causal attention (step a6), any head_dim <= 256 and
// either dtype. The fp32 parity mode and odd shapes use it; the bf16 hot path uses the tensor-core
// kernel in attention_tc.cu. One warp per (query row, q head); online softmax in fp32.
#include <cmath>

#include "ctx.h"

namespace {
template <typename T, int DPL>  // DPL = dims per lane = ceil(hd / 32)
__global__ void __launch_bounds__(128) attn_simt_kernel(const T* __restrict__ q, const int* __restrict__ q_row,
                                                        const int* __restrict__ q_tok, int n_rows,
                                                        const T* __restrict__ k, const T* __restrict__ v, int n_keys,
                                                        T* __restrict__ out, int n_q, int n_kv, int hd, float scale) {
  pdl_enter();
  __shared__ float qs[4][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x, h = blockIdx.y * 4 + warp;
  if (h >= n_q) return;
  const int g = h / (n_q / n_kv);
  const int kvd = n_kv * hd;
  const T* qr = q + (size_t)q_row[r] * n_q * hd + (size_t)h * hd;
  for (int d = lane; d < hd; d += 32) qs[warp][d] = to_f(qr[d]) * scale;
  __syncwarp();
  const int last = min(q_tok[r], n_keys - 1);  // keys j <= q_tok (positions strictly increasing)
  float m = -INFINITY, l = 0.f, o[DPL];
#pragma unroll
  for (int i = 0; i < DPL; ++i) o[i] = 0.f;
  for (int j0 = 0; j0 <= last; j0 += 32) {
    const int j = j0 + lane;
    float s = -INFINITY;
    if (j <= last) {
      const T* kr = k + (size_t)j * kvd + (size_t)g * hd;
      float acc = 0.f;
      for (int d = 0; d < hd; ++d) acc = fmaf(qs[warp][d], to_f(kr[d]), acc);
      s = acc;
    }
    const float mc = warp_max(s);
    const float mn = fmaxf(m, mc);
    const float corr = (m == -INFINITY) ? 0.f : expf(m - mn);
    const float p = (j <= last) ? expf(s - mn) : 0.f;
    l = l * corr + warp_sum(p);
#pragma unroll
    for (int i = 0; i < DPL; ++i) o[i] *= corr;
    const int nj = min(32, last + 1 - j0);
    for (int jj = 0; jj < nj; ++jj) {
      const float pj = __shfl_sync(0xffffffffu, p, jj);
      const T* vr = v + (size_t)(j0 + jj) * kvd + (size_t)g * hd;
#pragma unroll
      for (int i = 0; i < DPL; ++i) {
        const int d = lane + 32 * i;
        if (d < hd) o[i] = fmaf(pj, to_f(vr[d]), o[i]);
      }
    }
    m = mn;
  }
  T* orow = out + (size_t)r * n_q * hd + (size_t)h * hd;
  const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll
  for (int i = 0; i < DPL; ++i) {
    const int d = lane + 32 * i;
    if (d < hd) orow[d] = from_f<T>(o[i] * inv);
  }
}

template <typename T>
cb_status launch_t(cb_ctx* c, const cb_model& md, const void* q, const int* q_row, const int* q_tok, int n_rows, const void* k,
              const void* v, int n_keys, void* out, cudaStream_t s) {
  dim3 grid(n_rows, (md.n_q_heads + 3) / 4);
  const float scale = 1.0f / sqrtf((float)md.head_dim);
  const int dpl = (md.head_dim + 31) / 32;
#define L_(D)                                                                                              \
  CB_LAUNCH(c, (attn_simt_kernel<T, D>), grid, 128, 0, s, (const T*)q, q_row, q_tok, n_rows, (const T*)k, (const T*)v, n_keys, \
                                              (T*)out, md.n_q_heads, md.n_kv_heads, md.head_dim, scale)
  if (dpl <= 1) L_(1);
  else if (dpl <= 2) L_(2);
  else if (dpl <= 4) L_(4);
  else L_(8);
#undef L_
  return CB_OK;
}
}  // namespace

cb_status launch_attention_simt(cb_ctx* c, const void* q, const int* q_row, const int* q_tok, int n_rows,
                                const void* k, const void* v, int n_keys, void* out, cudaStream_t s) {
  if (n_rows == 0) return CB_OK;
  CB_REQUIRE(c->m.head_dim <= 256, CB_E_UNSUPPORTED, "attention: head_dim > 256");
  ProfScope ps_(c, PROF_ATTN, s);
  if (c->m.dtype == CB_BF16)
    CB_TRY(launch_t<bf16>(c, c->m, q, q_row, q_tok, n_rows, k, v, n_keys, out, s));
  else
    CB_TRY(launch_t<float>(c, c->m, q, q_row, q_tok, n_rows, k, v, n_keys, out, s));
  CB_LAUNCHED(c);
  return CB_OK;
}
