// elementwise.cu — HBM-bound kernels of the blend path: RoPE realign (step a1), embedding gather,
// RMSNorm, KV scatter (step a5) and small index utilities.
#include <algorithm>

#include "ctx.h"

// ---------------------------------------------------------------------------------------------
// (a1) positional recovery: K_out[s][t] = R(dst[t] - src[t]) K_src[s][t]   (footnote P:208-211,
// Appendix). One thread owns one 16-byte vector (4 or 2 RoPE pairs) of one token and
// loops over all slices (layers), so the (cos, sin) pairs are read once per token and reused
// n_slices times; K moves through 128-bit coalesced loads/stores exactly once (read + write).
// ---------------------------------------------------------------------------------------------
template <typename T, int UNROLL>
__global__ void __launch_bounds__(256) realign_kernel(T* __restrict__ k_out, const T* __restrict__ k_src,
                                                      T* __restrict__ v_out, const T* __restrict__ v_src,
                                                      const int* __restrict__ src_pos, const int* __restrict__ dst_pos,
                                                      int n_slices, int n_tok, long long out_stride,
                                                      long long src_stride, int kvd, int hd,
                                                      const float2* __restrict__ tab, int max_pos, int* err) {
  pdl_enter();
  constexpr int V = Vec16<T>::N;  // elements per vector
  const int nvec = kvd / V;
  const long long total = (long long)n_tok * nvec;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int t = (int)(idx / nvec);
    const int j = (int)(idx - (long long)t * nvec);
    const int e0 = j * V;
    int delta = __ldg(dst_pos + t) - __ldg(src_pos + t);
    float sgn = 1.f;
    if (delta < 0) { delta = -delta; sgn = -1.f; }
    if (delta >= max_pos) { atomicOr(err, CB_DEVERR_POS_RANGE); delta = max_pos - 1; }
    const float2* cs_row = tab + (size_t)delta * (hd >> 1) + ((e0 % hd) >> 1);
    float c[V / 2], s[V / 2];
#pragma unroll
    for (int p = 0; p < V / 2; ++p) {
      const float2 cs = __ldg(cs_row + p);
      c[p] = cs.x;
      s[p] = sgn * cs.y;
    }
    const size_t off = (size_t)t * kvd + e0;
    for (int s0 = 0; s0 < n_slices; s0 += UNROLL) {
      Vec16<T> v[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u)
        if (s0 + u < n_slices) v[u] = ld16_cg(k_src + (size_t)(s0 + u) * src_stride + off);
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        if (s0 + u < n_slices) {
          Vec16<T> o;
#pragma unroll
          for (int p = 0; p < V / 2; ++p) {
            const float x0 = to_f(v[u].v[2 * p]), x1 = to_f(v[u].v[2 * p + 1]);
            o.v[2 * p] = from_f<T>(c[p] * x0 - s[p] * x1);
            o.v[2 * p + 1] = from_f<T>(s[p] * x0 + c[p] * x1);
          }
          st16(k_out + (size_t)(s0 + u) * out_stride + off, o);
        }
      }
      if (v_out != nullptr) {  // out-of-place blend: V is carried over unchanged in the same pass
#pragma unroll
        for (int u = 0; u < UNROLL; ++u)
          if (s0 + u < n_slices) v[u] = ld16_cg(v_src + (size_t)(s0 + u) * src_stride + off);
#pragma unroll
        for (int u = 0; u < UNROLL; ++u)
          if (s0 + u < n_slices) st16(v_out + (size_t)(s0 + u) * out_stride + off, v[u]);
      }
    }
  }
}

cb_status launch_realign(cb_ctx* c, void* k_out, const void* k_src, void* v_out, const void* v_src,
                         const int* src_pos, const int* dst_pos, int n_slices, int n_tok, long long out_stride,
                         long long src_stride, cudaStream_t s) {
  if (n_tok == 0 || n_slices == 0) return CB_OK;
  const int kvd = c->m.n_kv_heads * c->m.head_dim;
  const int V = 16 / (int)dtype_bytes(c->m.dtype);
  const long long total = (long long)n_tok * (kvd / V);
  const int grid = (int)std::max<long long>(1, std::min<long long>((total + 255) / 256, (long long)c->num_sms * 8));
  ProfScope ps_(c, PROF_REALIGN, s);
  if (c->m.dtype == CB_BF16)
    CB_LAUNCH(c, (realign_kernel<bf16, 4>), grid, 256, 0, s, (bf16*)k_out, (const bf16*)k_src, (bf16*)v_out, (const bf16*)v_src,
                                                 src_pos, dst_pos, n_slices, n_tok, out_stride, src_stride, kvd,
                                                 c->m.head_dim, c->rope_tab, c->m.max_pos, c->err_word);
  else
    CB_LAUNCH(c, (realign_kernel<float, 4>), grid, 256, 0, s, (float*)k_out, (const float*)k_src, (float*)v_out,
                                                  (const float*)v_src, src_pos, dst_pos, n_slices, n_tok, out_stride,
                                                  src_stride, kvd, c->m.head_dim, c->rope_tab, c->m.max_pos,
                                                  c->err_word);
  CB_LAUNCHED(c);
  return CB_OK;
}

// ---------------------------------------------------------------------------------------------
// embedding gather: h[t] = fp32(embed[tok[t]])
// ---------------------------------------------------------------------------------------------
template <typename T> __device__ __forceinline__ float4 ld4f(const T* p);
template <> __device__ __forceinline__ float4 ld4f<float>(const float* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}
template <> __device__ __forceinline__ float4 ld4f<bf16>(const bf16* p) {
  const uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
  const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
  const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
  return make_float4(a.x, a.y, b.x, b.y);
}

// One 128-thread block per row, 4 elements per thread per step (16-byte stores of h).
template <typename T>
__global__ void __launch_bounds__(128) embed_kernel(const T* __restrict__ emb, const int* __restrict__ tok,
                                                    float* __restrict__ h, int d) {
  pdl_enter();
  const int t = blockIdx.x;
  const T* src = emb + (size_t)__ldg(tok + t) * d;
  float* dst = h + (size_t)t * d;
#pragma unroll 4
  for (int e = threadIdx.x * 4; e < d; e += 128 * 4) *reinterpret_cast<float4*>(dst + e) = ld4f(src + e);
}

cb_status launch_embed(cb_ctx* c, const void* embed, const int* tok, int n, float* h, cudaStream_t s) {
  if (n == 0) return CB_OK;
  ProfScope ps_(c, PROF_EMBED, s);
  if (c->m.dtype == CB_BF16)
    CB_LAUNCH(c, (embed_kernel<bf16>), n, 128, 0, s, (const bf16*)embed, tok, h, c->m.d_model);
  else
    CB_LAUNCH(c, (embed_kernel<float>), n, 128, 0, s, (const float*)embed, tok, h, c->m.d_model);
  CB_LAUNCHED(c);
  return CB_OK;
}

// ---------------------------------------------------------------------------------------------
// RMSNorm: x = h / sqrt(mean(h^2) + eps) * gain  (fixed-order block reduction: deterministic)
// ---------------------------------------------------------------------------------------------
// One warp per row: 16-byte loads, a fixed-order warp reduction (deterministic), second pass from L1.
__device__ __forceinline__ void store4(float* p, float a, float b, float c, float d) {
  *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d);
}
__device__ __forceinline__ void store4(bf16* p, float a, float b, float c, float d) {
  __nv_bfloat162 lo = __floats2bfloat162_rn(a, b), hi = __floats2bfloat162_rn(c, d);
  uint2 w;
  w.x = *reinterpret_cast<uint32_t*>(&lo);
  w.y = *reinterpret_cast<uint32_t*>(&hi);
  *reinterpret_cast<uint2*>(p) = w;
}

// One 128-thread block per row: every 16-byte load of the row is issued before the reduction (the
// row stays in registers, up to d = 8192), fixed-order block reduction (deterministic).
constexpr int RMS_THREADS = 128, RMS_MAXV = 16;
template <typename T>
__global__ void __launch_bounds__(RMS_THREADS) rmsnorm_kernel(const float* __restrict__ h, const float* __restrict__ g,
                                                              T* __restrict__ x, int d, float eps) {
  pdl_enter();
  const int r = blockIdx.x, tid = threadIdx.x;
  const float* hr = h + (size_t)r * d;
  float4 v[RMS_MAXV];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < RMS_MAXV; ++i) {
    const int e = (i * RMS_THREADS + tid) * 4;
    v[i] = e < d ? *reinterpret_cast<const float4*>(hr + e) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
#pragma unroll
  for (int i = 0; i < RMS_MAXV; ++i) ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
  __shared__ float red[RMS_THREADS / 32];
  ss = warp_sum(ss);
  if ((tid & 31) == 0) red[tid >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int w = 0; w < RMS_THREADS / 32; ++w) tot += red[w];
  const float inv = 1.0f / sqrtf(tot / (float)d + eps);
  T* xr = x + (size_t)r * d;
#pragma unroll
  for (int i = 0; i < RMS_MAXV; ++i) {
    const int e = (i * RMS_THREADS + tid) * 4;
    if (e < d) {
      const float4 gg = __ldg(reinterpret_cast<const float4*>(g + e));
      store4(xr + e, v[i].x * inv * gg.x, v[i].y * inv * gg.y, v[i].z * inv * gg.z, v[i].w * inv * gg.w);
    }
  }
}

// Embedding gather fused with layer 0's attention RMSNorm: h[t] = fp32(embed[tok[t]]) and
// x[t] = rmsnorm(h[t]) * gain, with rmsnorm_kernel's exact arithmetic and reduction order (so x is
// bitwise what embed_kernel followed by rmsnorm_kernel produce).
template <typename T>
__global__ void __launch_bounds__(RMS_THREADS) embed_norm_kernel(const T* __restrict__ emb, const int* __restrict__ tok,
                                                                 const float* __restrict__ g, float* __restrict__ h,
                                                                 T* __restrict__ x, int d, float eps) {
  pdl_enter();
  const int r = blockIdx.x, tid = threadIdx.x;
  const T* src = emb + (size_t)__ldg(tok + r) * d;
  float* hr = h + (size_t)r * d;
  float4 v[RMS_MAXV];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < RMS_MAXV; ++i) {
    const int e = (i * RMS_THREADS + tid) * 4;
    v[i] = e < d ? ld4f(src + e) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
#pragma unroll
  for (int i = 0; i < RMS_MAXV; ++i) {
    const int e = (i * RMS_THREADS + tid) * 4;
    if (e < d) *reinterpret_cast<float4*>(hr + e) = v[i];
  }
#pragma unroll
  for (int i = 0; i < RMS_MAXV; ++i) ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
  __shared__ float red[RMS_THREADS / 32];
  ss = warp_sum(ss);
  if ((tid & 31) == 0) red[tid >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int w = 0; w < RMS_THREADS / 32; ++w) tot += red[w];
  const float inv = 1.0f / sqrtf(tot / (float)d + eps);
  T* xr = x + (size_t)r * d;
#pragma unroll
  for (int i = 0; i < RMS_MAXV; ++i) {
    const int e = (i * RMS_THREADS + tid) * 4;
    if (e < d) {
      const float4 gg = __ldg(reinterpret_cast<const float4*>(g + e));
      store4(xr + e, v[i].x * inv * gg.x, v[i].y * inv * gg.y, v[i].z * inv * gg.z, v[i].w * inv * gg.w);
    }
  }
}

cb_status launch_embed_norm(cb_ctx* c, const void* embed, const int* tok, const float* gain, int n, float* h,
                            void* x, cudaStream_t s) {
  if (n == 0) return CB_OK;
  CB_REQUIRE(c->m.d_model <= RMS_THREADS * RMS_MAXV * 4, CB_E_UNSUPPORTED, "embed_norm: d_model > %d",
             RMS_THREADS * RMS_MAXV * 4);
  ProfScope ps_(c, PROF_EMBED, s);
  if (c->m.dtype == CB_BF16)
    CB_LAUNCH(c, (embed_norm_kernel<bf16>), n, RMS_THREADS, 0, s, (const bf16*)embed, tok, gain, h, (bf16*)x,
              c->m.d_model, c->m.rms_eps);
  else
    CB_LAUNCH(c, (embed_norm_kernel<float>), n, RMS_THREADS, 0, s, (const float*)embed, tok, gain, h, (float*)x,
              c->m.d_model, c->m.rms_eps);
  CB_LAUNCHED(c);
  return CB_OK;
}

cb_status launch_rmsnorm(cb_ctx* c, const float* h, const float* gain, int n_rows, void* x, cudaStream_t s) {
  if (n_rows == 0) return CB_OK;
  CB_REQUIRE(c->m.d_model <= RMS_THREADS * RMS_MAXV * 4, CB_E_UNSUPPORTED, "rmsnorm: d_model > %d",
             RMS_THREADS * RMS_MAXV * 4);
  ProfScope ps_(c, PROF_RMSNORM, s);
  if (c->m.dtype == CB_BF16)
    CB_LAUNCH(c, (rmsnorm_kernel<bf16>), n_rows, RMS_THREADS, 0, s, h, gain, (bf16*)x, c->m.d_model, c->m.rms_eps);
  else
    CB_LAUNCH(c, (rmsnorm_kernel<float>), n_rows, RMS_THREADS, 0, s, h, gain, (float*)x, c->m.d_model, c->m.rms_eps);
  CB_LAUNCHED(c);
  return CB_OK;
}

// ---------------------------------------------------------------------------------------------
// (a5) KV scatter: blended[qtok[r]] <- fresh[qrow[r]] for the kept rows (R3)
// ---------------------------------------------------------------------------------------------
template <typename T>
__global__ void scatter_kv_kernel(const T* __restrict__ kf, const T* __restrict__ vf, const int* __restrict__ qrow,
                                  const int* __restrict__ qtok, T* __restrict__ kb, T* __restrict__ vb, int kvd) {
  pdl_enter();
  const int r = blockIdx.x;
  const size_t src = (size_t)__ldg(qrow + r) * kvd, dst = (size_t)__ldg(qtok + r) * kvd;
  for (int e = threadIdx.x * Vec16<T>::N; e < kvd; e += blockDim.x * Vec16<T>::N) {
    st16(kb + dst + e, ld16(kf + src + e));
    st16(vb + dst + e, ld16(vf + src + e));
  }
}

cb_status launch_scatter_kv(cb_ctx* c, const void* kf, const void* vf, const int* qrow, const int* qtok, int n,
                            void* kb, void* vb, cudaStream_t s) {
  if (n == 0) return CB_OK;
  const int kvd = c->m.n_kv_heads * c->m.head_dim;
  ProfScope ps_(c, PROF_SCATTER, s);
  if (c->m.dtype == CB_BF16)
    CB_LAUNCH(c, (scatter_kv_kernel<bf16>), n, 128, 0, s, (const bf16*)kf, (const bf16*)vf, qrow, qtok, (bf16*)kb, (bf16*)vb, kvd);
  else
    CB_LAUNCH(c, (scatter_kv_kernel<float>), n, 128, 0, s, (const float*)kf, (const float*)vf, qrow, qtok, (float*)kb, (float*)vb,
                                               kvd);
  CB_LAUNCHED(c);
  return CB_OK;
}

// ---------------------------------------------------------------------------------------------
// Kept-query rows of the projection input (layer 1's Q-after-selection): xq[j] = x[qrow[j]] (bf16 rows
// of d) and, with the fused RMSNorm, ssq[j] = ss[qrow[j]] (ld_ss sum-of-squares blocks). Block per row.
// ---------------------------------------------------------------------------------------------
__global__ void gather_rows_kernel(const bf16* __restrict__ x, const float* __restrict__ ss, const int* __restrict__ qrow,
                                   int d, int ld_ss, bf16* __restrict__ xq, float* __restrict__ ssq) {
  pdl_enter();
  const int j = blockIdx.x;
  const size_t src = (size_t)__ldg(qrow + j);
  for (int e = threadIdx.x * 8; e < d; e += blockDim.x * 8)
    *reinterpret_cast<uint4*>(xq + (size_t)j * d + e) = __ldg(reinterpret_cast<const uint4*>(x + src * d + e));
  if (ss != nullptr)
    for (int b = threadIdx.x; b < ld_ss; b += blockDim.x) ssq[(size_t)j * ld_ss + b] = __ldg(ss + src * ld_ss + b);
}

cb_status launch_gather_rows(cb_ctx* c, const void* x, const float* ss, const int* qrow, int n, int ld_ss, void* xq,
                             float* ssq, cudaStream_t s) {
  if (n == 0) return CB_OK;
  const int d = c->m.d_model;
  CB_REQUIRE(c->m.dtype == CB_BF16 && d % 8 == 0, CB_E_UNSUPPORTED, "gather_rows: bf16 rows of a multiple of 8");
  ProfScope ps_(c, PROF_MISC, s);
  CB_LAUNCH(c, gather_rows_kernel, n, 128, 0, s, (const bf16*)x, ss, qrow, d, ld_ss, (bf16*)xq, ssq);
  CB_LAUNCHED(c);
  return CB_OK;
}

// ---------------------------------------------------------------------------------------------
// chunk-local positions from chunk starts passed by value (no host->device copy, graph-safe)
// ---------------------------------------------------------------------------------------------
struct ChunkTable {
  int n;
  int start[129];
};

__global__ void local_pos_kernel(ChunkTable ct, int base_chunk, int* __restrict__ src_pos) {
  pdl_enter();
  const int t0 = ct.start[0], t1 = ct.start[ct.n];
  for (int t = t0 + blockIdx.x * blockDim.x + threadIdx.x; t < t1; t += gridDim.x * blockDim.x) {
    int lo = 0, hi = ct.n - 1;  // largest c with start[c] <= t
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (ct.start[mid] <= t) lo = mid; else hi = mid - 1;
    }
    src_pos[t] = t - ct.start[lo];
  }
  (void)base_chunk;
}

// The attention mask compares token indices (key row <= query row), which equals the paper's position mask
// (causal by original position) only when positions increase with the token index; the RoPE table
// holds positions [0, max_pos). A violation is reported through the device error word.
__global__ void pos_check_kernel(const int* __restrict__ pos, int T, int max_pos, int* err) {
  pdl_enter();
  int bad = 0;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x) {
    const int p = pos[t];
    if (p < 0 || p >= max_pos) bad |= CB_DEVERR_POS_RANGE;
    if (t > 0 && p <= pos[t - 1]) bad |= CB_DEVERR_POS_ORDER;
  }
  if (bad) atomicOr(err, bad);
}

cb_status launch_pos_check(cb_ctx* c, const int* pos, int T, cudaStream_t s) {
  if (T <= 0) return CB_OK;
  ProfScope ps_(c, PROF_MISC, s);
  CB_LAUNCH(c, (pos_check_kernel), std::min(64, (T + 255) / 256), 256, 0, s, pos, T, c->m.max_pos, c->err_word);
  CB_LAUNCHED(c);
  return CB_OK;
}

cb_status launch_local_pos(cb_ctx* c, const int* cs, int n_chunks, int* src_pos, cudaStream_t s) {
  for (int b = 0; b < n_chunks; b += 128) {
    ChunkTable ct;
    ct.n = std::min(128, n_chunks - b);
    for (int i = 0; i <= ct.n; ++i) ct.start[i] = cs[b + i];
    const int len = ct.start[ct.n] - ct.start[0];
    if (len <= 0) continue;
    ProfScope ps_(c, PROF_MISC, s);
    CB_LAUNCH(c, (local_pos_kernel), std::min(1024, (len + 255) / 256), 256, 0, s, ct, b, src_pos);
    CB_LAUNCHED(c);
  }
  return CB_OK;
}

__global__ void sel_out_kernel(const int* __restrict__ qtok, int k, int N, int* __restrict__ row) {
  pdl_enter();
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < N; j += gridDim.x * blockDim.x)
    row[j] = j < k ? qtok[j] : -1;
}

cb_status launch_sel_out(cb_ctx* c, const int* qtok, int k, int N, int* row, cudaStream_t s) {
  if (N == 0) return CB_OK;
  ProfScope ps_(c, PROF_MISC, s);
  CB_LAUNCH(c, (sel_out_kernel), std::min(256, (N + 255) / 256), 256, 0, s, qtok, k, N, row);
  CB_LAUNCHED(c);
  return CB_OK;
}

// ---------------------------------------------------------------------------------------------
// KV^new -> paged decode cache ("the fused KV cache is input into the LLM inference
// engine", which pages its KV in fixed-size blocks, P:2496 / P:2722): token t of layer l goes to
// page block_table[t / block_size], slot t % block_size of that layer's pool. A thread moves one 16-B
// vector; consecutive threads cover a token row, then the next token, so reads are contiguous and
// writes are contiguous within a page.
// ---------------------------------------------------------------------------------------------
template <typename T>
__global__ void kv_to_paged_kernel(const T* __restrict__ k, const T* __restrict__ v, long long src_layer_stride,
                                   int n_layers, int n_tok, int row, const int* __restrict__ block_table,
                                   int block_size, T* __restrict__ kp, T* __restrict__ vp, int n_pages,
                                   long long dst_layer_stride, int* err) {
  pdl_enter();
  constexpr int V = Vec16<T>::N;
  const int vec_per_row = row / V;
  const long long per_layer = (long long)n_tok * vec_per_row;
  const long long total = per_layer * n_layers;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int l = (int)(i / per_layer);
    const long long r = i - (long long)l * per_layer;
    const int t = (int)(r / vec_per_row), e = (int)(r - (long long)t * vec_per_row) * V;
    const long long src = l * src_layer_stride + (long long)t * row + e;
    const int page = __ldg(block_table + t / block_size);
    if (page < 0 || page >= n_pages) {  // outside the pool: report, never write
      atomicOr(err, CB_DEVERR_PAGE);
      continue;
    }
    const long long dst = l * dst_layer_stride + ((long long)page * block_size + t % block_size) * row + e;
    st16(kp + dst, ld16(k + src));
    st16(vp + dst, ld16(v + src));
  }
}

extern "C" cb_status cb_kv_to_paged(cb_ctx* c, const void* k_blend, const void* v_blend, int32_t n_layers,
                                    int32_t n_tok, int64_t src_layer_stride, const int32_t* block_table,
                                    int32_t block_size, void* k_pages, void* v_pages, int32_t n_pages,
                                    int64_t dst_layer_stride, void* st) {
  CB_REQUIRE(c != nullptr, CB_E_INVALID_ARG, "ctx is NULL");
  CB_REQUIRE(n_layers >= 0 && n_tok >= 0 && block_size >= 1, CB_E_INVALID_ARG, "bad sizes");
  if (n_layers == 0 || n_tok == 0) return CB_OK;
  CB_REQUIRE(k_blend && v_blend && block_table && k_pages && v_pages, CB_E_INVALID_ARG, "NULL pointer");
  const int row = c->m.n_kv_heads * c->m.head_dim;
  CB_REQUIRE(src_layer_stride >= (int64_t)n_tok * row, CB_E_SHAPE, "src_layer_stride < n_tok * n_kv * head_dim");
  CB_REQUIRE(n_pages >= 1, CB_E_INVALID_ARG, "n_pages must be >= 1");
  CB_REQUIRE(dst_layer_stride >= (int64_t)n_pages * block_size * row, CB_E_SHAPE,
             "dst_layer_stride smaller than n_pages pages of block_size tokens");
  const uintptr_t al = (uintptr_t)k_blend | (uintptr_t)v_blend | (uintptr_t)k_pages | (uintptr_t)v_pages;
  CB_REQUIRE(al % 16 == 0, CB_E_INVALID_ARG, "KV buffers must be 16-byte aligned");
  cudaStream_t s = (cudaStream_t)st;
  ProfScope ps_(c, PROF_SCATTER, s);
  const long long vecs = (long long)n_layers * n_tok * (row * (long long)dtype_bytes(c->m.dtype) / 16);
  const int blocks = (int)std::min<long long>(8LL * c->num_sms, (vecs + 255) / 256);
  if (c->m.dtype == CB_BF16)
    CB_LAUNCH(c, (kv_to_paged_kernel<bf16>), blocks, 256, 0, s, (const bf16*)k_blend, (const bf16*)v_blend,
              (long long)src_layer_stride, n_layers, n_tok, row, block_table, block_size, (bf16*)k_pages,
              (bf16*)v_pages, n_pages, (long long)dst_layer_stride, c->err_word);
  else
    CB_LAUNCH(c, (kv_to_paged_kernel<float>), blocks, 256, 0, s, (const float*)k_blend, (const float*)v_blend,
              (long long)src_layer_stride, n_layers, n_tok, row, block_table, block_size, (float*)k_pages,
              (float*)v_pages, n_pages, (long long)dst_layer_stride, c->err_word);
  CB_LAUNCHED(c);
  return CB_OK;
}
