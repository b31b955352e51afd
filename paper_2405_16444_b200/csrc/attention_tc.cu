// attention_tc.cu — tensor-core sparse-query causal attention (step a6), bf16, head_dim 128.
//
// out[r][h] = softmax_j(q_{r,h} . k_{j,g} / sqrt(hd)) v_{j,g} over keys j <= q_tok[r]
//
// Flash-style online softmax (fp32 statistics). GQA packing: a CTA owns one kv head g and a tile of
// 64 (query token, q head of g) rows, so every K/V tile staged in shared memory serves all G q heads
// of the group. K/V tiles (64 keys x 128) stream through a cp.async double buffer with an XOR
// swizzle (conflict-free ldmatrix); S = QK^T and O += PV run on mma.sync m16n8k16 bf16 with P kept in
// registers. Key tiles past the CTA's last query token are never loaded (position-aware skip); only
// tiles beyond its first query token are masked. Heaviest (latest-token) tiles are scheduled first.
#include "ctx.h"

namespace {
constexpr int HD = 128, BR = 64, BC = 64, NT = 128;
constexpr int TILE_BYTES = BC * HD * 2;                     // 16 KB
constexpr int SMEM = BR * HD * 2 + 4 * TILE_BYTES;          // Q + 2 x (K, V) = 80 KB

__device__ __forceinline__ uint32_t swz(int row, int chunk) {  // byte offset in a [rows][128] bf16 tile
  return (uint32_t)(row * 256 + ((chunk ^ (row & 7)) << 4));
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool pred) {
  const int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

__global__ void __launch_bounds__(NT) attn_mma_kernel(const bf16* __restrict__ q, const int* __restrict__ q_row,
                                                      const int* __restrict__ q_tok, int n_rows,
                                                      const bf16* __restrict__ k, const bf16* __restrict__ v,
                                                      int n_keys, bf16* __restrict__ out, int n_q, int n_kv,
                                                      float scale_log2, int kt_per_split, float* __restrict__ opart,
                                                      float2* __restrict__ ml) {
  pdl_enter();
  extern __shared__ __align__(128) uint8_t sm[];
  const uint32_t sQ = (uint32_t)__cvta_generic_to_shared(sm);
  const uint32_t sK0 = sQ + BR * HD * 2;  // K[2], then V[2]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = blockIdx.y, G = n_q / n_kv;
  const int R = n_rows * G;
  const int rho0 = (gridDim.x - 1 - blockIdx.x) * BR;  // heaviest tiles first
  const int qd = n_q * HD, kvd = n_kv * HD;

  // key range of this tile: [0, kmax]; tiles entirely <= kmin need no mask
  int kmax = -1, kmin = 1 << 30;
  for (int rr = rho0 / G; rr <= min(R - 1, rho0 + BR - 1) / G; ++rr) {
    const int t = min(__ldg(q_tok + rr), n_keys - 1);
    kmax = max(kmax, t);
    kmin = min(kmin, t);
  }
  const int n_kt = (kmax + BC) / BC;
  // split-KV: this CTA covers key tiles [j_begin, j_end) (split = blockIdx.z)
  const int split = blockIdx.z;
  const int j_begin = split * kt_per_split, j_end = min(n_kt, j_begin + kt_per_split);
  const size_t part_row0 = ((size_t)split * n_kv + g) * R;  // partial rows of (split, g)
  if (j_begin >= j_end) {  // no keys for this split: neutral partial (m = -inf, l = 0)
    if (opart != nullptr)
      for (int i = tid; i < BR; i += NT)
        if (rho0 + i < R) ml[part_row0 + rho0 + i] = make_float2(-INFINITY, 0.f);
    return;
  }

  // ---- stage Q (64 rows x 128) ----
  for (int i = tid; i < BR * 16; i += NT) {
    const int row = i >> 4, ch = i & 15, rho = rho0 + row;
    const bool ok = rho < R;
    const int r = ok ? rho / G : 0, h = g * G + (ok ? rho % G : 0);
    const bf16* src = q + (size_t)__ldg(q_row + r) * qd + h * HD + ch * 8;
    cp_async16(sQ + swz(row, ch), src, ok);
  }
  auto load_kv = [&](int j, int buf) {
    const uint32_t dk = sK0 + buf * TILE_BYTES, dv = sK0 + (2 + buf) * TILE_BYTES;
    for (int i = tid; i < BC * 16; i += NT) {
      const int row = i >> 4, ch = i & 15, key = j * BC + row;
      const bool ok = key < n_keys;
      const size_t off = (size_t)(ok ? key : 0) * kvd + g * HD + ch * 8;
      cp_async16(dk + swz(row, ch), k + off, ok);
      cp_async16(dv + swz(row, ch), v + off, ok);
    }
  };
  load_kv(j_begin, 0);
  cp_commit();

  // per-thread rows (within the warp's 16): lane/4 and lane/4 + 8
  int tok_r[2];
#pragma unroll
  for (int hr = 0; hr < 2; ++hr) {
    const int rho = rho0 + warp * 16 + (lane >> 2) + hr * 8;
    tok_r[hr] = rho < R ? min(__ldg(q_tok + rho / G), n_keys - 1) : kmax;
  }
  float m_i[2] = {-INFINITY, -INFINITY}, l_i[2] = {0.f, 0.f};
  float o[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  uint32_t qa[8][4];

  for (int j = j_begin; j < j_end; ++j) {
    const int buf = (j - j_begin) & 1;
    if (j + 1 < j_end) load_kv(j + 1, buf ^ 1);
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    if (j == j_begin) {  // Q fragments once
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const int row = warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8, ch = kk * 2 + (lane >> 4);
        ldsm_x4(sQ + swz(row, ch), qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3]);
      }
    }
    const uint32_t sK = sK0 + buf * TILE_BYTES, sV = sK0 + (2 + buf) * TILE_BYTES;
    // ---- S = Q K^T (16 x 64 per warp) ----
    float s[8][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
#pragma unroll
      for (int np = 0; np < 4; ++np) {  // pairs of 8-key n-tiles
        const int row = np * 16 + (lane & 7) + (lane >> 4) * 8, ch = kk * 2 + ((lane >> 3) & 1);
        uint32_t b0, b1, b2, b3;
        ldsm_x4(sK + swz(row, ch), b0, b1, b2, b3);
        mma16816(s[2 * np], qa[kk], b0, b1);
        mma16816(s[2 * np + 1], qa[kk], b2, b3);
      }
    }
    // ---- mask (only tiles reaching past the first query token) + online softmax ----
    const bool need_mask = (j + 1) * BC - 1 > kmin;
    float mx[2] = {m_i[0], m_i[1]};
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int hr = e >> 1;
        float x = s[nt][e] * scale_log2;
        if (need_mask) {
          const int key = j * BC + nt * 8 + (lane & 3) * 2 + (e & 1);
          if (key > tok_r[hr]) x = -INFINITY;
        }
        s[nt][e] = x;
        mx[hr] = fmaxf(mx[hr], x);
      }
    float corr[2], rs[2] = {0.f, 0.f};
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      mx[hr] = fmaxf(mx[hr], __shfl_xor_sync(0xffffffffu, mx[hr], 1));
      mx[hr] = fmaxf(mx[hr], __shfl_xor_sync(0xffffffffu, mx[hr], 2));
      const float m_old = m_i[hr];
      m_i[hr] = mx[hr];
      // a row with no visible key yet (split-KV) keeps m = -inf: use 0 as the exponent reference
      const float mref = (mx[hr] == -INFINITY) ? 0.f : mx[hr];
      corr[hr] = exp2f(m_old - mref);  // m_old = -inf -> 0
      mx[hr] = mref;
    }
    uint32_t pa[4][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const float p0 = exp2f(s[nt][0] - mx[0]), p1 = exp2f(s[nt][1] - mx[0]);
      const float p2 = exp2f(s[nt][2] - mx[1]), p3 = exp2f(s[nt][3] - mx[1]);
      rs[0] += p0 + p1;
      rs[1] += p2 + p3;
      pa[nt >> 1][(nt & 1) * 2 + 0] = pack2(p0, p1);
      pa[nt >> 1][(nt & 1) * 2 + 1] = pack2(p2, p3);
    }
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      rs[hr] += __shfl_xor_sync(0xffffffffu, rs[hr], 1);
      rs[hr] += __shfl_xor_sync(0xffffffffu, rs[hr], 2);
      l_i[hr] = l_i[hr] * corr[hr] + rs[hr];
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      o[i][0] *= corr[0]; o[i][1] *= corr[0];
      o[i][2] *= corr[1]; o[i][3] *= corr[1];
    }
    // ---- O += P V ----
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {  // 16 keys per k-step
#pragma unroll
      for (int np = 0; np < 8; ++np) {  // pairs of 8-wide hd n-tiles
        const int row = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8, ch = np * 2 + (lane >> 4);
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(sV + swz(row, ch), b0, b1, b2, b3);
        mma16816(o[2 * np], pa[kk], b0, b1);
        mma16816(o[2 * np + 1], pa[kk], b2, b3);
      }
    }
    __syncthreads();
  }
  cp_wait<0>();

  if (opart != nullptr) {  // split-KV: unnormalised fp32 partial + (m, l) per row
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      const int rho = rho0 + warp * 16 + (lane >> 2) + hr * 8;
      if (rho >= R) continue;
      float* dst = opart + (part_row0 + rho) * HD + (lane & 3) * 2;
#pragma unroll
      for (int nt = 0; nt < 16; ++nt)
        *reinterpret_cast<float2*>(dst + nt * 8) = make_float2(o[nt][2 * hr], o[nt][2 * hr + 1]);
      if ((lane & 3) == 0) ml[part_row0 + rho] = make_float2(m_i[hr], l_i[hr]);
    }
    return;
  }
  // ---- normalise and store ----
#pragma unroll
  for (int hr = 0; hr < 2; ++hr) {
    const int rho = rho0 + warp * 16 + (lane >> 2) + hr * 8;
    if (rho >= R) continue;
    const int r = rho / G, h = g * G + rho % G;
    const float inv = l_i[hr] > 0.f ? 1.f / l_i[hr] : 0.f;
    bf16* dst = out + (size_t)r * qd + h * HD + (lane & 3) * 2;
#pragma unroll
    for (int nt = 0; nt < 16; ++nt)
      *reinterpret_cast<uint32_t*>(dst + nt * 8) = pack2(o[nt][2 * hr] * inv, o[nt][2 * hr + 1] * inv);
  }
}

// Combine split-KV partials of one (query row, q head) per warp, splits in fixed order:
// m* = max m_s, l* = sum l_s 2^(m_s - m*), O = sum O_s 2^(m_s - m*) / l*.
__global__ void attn_merge_kernel(const float* __restrict__ opart, const float2* __restrict__ ml, int R, int n_kv,
                                  int G, int n_splits, bf16* __restrict__ out, int qd) {
  pdl_enter();
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= R * n_kv) return;
  const int g = w / R, rho = w - g * R;
  constexpr int MAXS = 16;  // launcher caps n_splits
  // lane s holds split s's (m, l); every partial row load is issued before the weighted sum
  const float2 my = lane < n_splits ? ml[((size_t)lane * n_kv + g) * R + rho] : make_float2(-INFINITY, 0.f);
  const float mstar = warp_max(my.x);
  float4 o[MAXS];
#pragma unroll
  for (int s = 0; s < MAXS; ++s)
    if (s < n_splits) o[s] = reinterpret_cast<const float4*>(opart + (((size_t)s * n_kv + g) * R + rho) * HD)[lane];
  float l = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int s = 0; s < MAXS; ++s) {
    if (s >= n_splits) break;
    const float ms = __shfl_sync(0xffffffffu, my.x, s), ls = __shfl_sync(0xffffffffu, my.y, s);
    if (ms == -INFINITY) continue;
    const float f = exp2f(ms - mstar);
    l += ls * f;
    acc.x += o[s].x * f; acc.y += o[s].y * f; acc.z += o[s].z * f; acc.w += o[s].w * f;
  }
  const float inv = l > 0.f ? 1.f / l : 0.f;
  const int r = rho / G, h = g * G + rho % G;
  bf16* dst = out + (size_t)r * qd + h * HD + lane * 4;
  reinterpret_cast<uint32_t*>(dst)[0] = pack2(acc.x * inv, acc.y * inv);
  reinterpret_cast<uint32_t*>(dst)[1] = pack2(acc.z * inv, acc.w * inv);
}
}  // namespace

bool attention_tc_ok(const cb_ctx* c) { return c->m.dtype == CB_BF16 && c->m.head_dim == HD; }

cb_status launch_attention_merge(cb_ctx* c, int R, int n_splits, void* out, cudaStream_t s) {
  const int n_kv = c->m.n_kv_heads, G = c->m.n_q_heads / n_kv;
  const int warps = R * n_kv;
  ProfScope ps_(c, PROF_ATTN, s);
  CB_LAUNCH(c, (attn_merge_kernel), (warps + 7) / 8, 256, 0, s, c->attn_part, c->attn_ml, R, n_kv, G, n_splits, (bf16*)out,
                                                    c->m.n_q_heads * HD);
  CB_LAUNCHED(c);
  return CB_OK;
}

cb_status launch_attention_tc(cb_ctx* c, const void* q, const int* q_row, const int* q_tok, int n_rows, const void* k,
                              const void* v, int n_keys, void* out, cudaStream_t s) {
  if (n_rows == 0) return CB_OK;
  const int n_kv = c->m.n_kv_heads, G = c->m.n_q_heads / n_kv;
  const int R = n_rows * G;
  const int tiles = (R + BR - 1) / BR;
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)HD);
  // split-KV when the (tile, kv head) grid is too small or too unbalanced to fill the SMs (later layers:
  // a few hundred selected queries, some of them at the end of a long context)
  const int max_kt = (n_keys + BC - 1) / BC;
  const long long base = (long long)tiles * n_kv;
  int n_splits = 1;
  if (base < 4LL * c->num_sms && c->attn_part != nullptr) {
    n_splits = (int)std::min<long long>((6LL * c->num_sms + base - 1) / base, (max_kt + 3) / 4);
    n_splits = std::min(n_splits, (int)(c->attn_part_rows / ((long long)R * n_kv)));
    n_splits = std::min(n_splits, 16);
    n_splits = std::max(1, n_splits);
  }
  const int kt_per_split = (max_kt + n_splits - 1) / n_splits;
  dim3 grid(tiles, n_kv, n_splits);
  ProfScope ps_(c, PROF_ATTN, s);
  float* opart = n_splits > 1 ? c->attn_part : nullptr;
  CB_LAUNCH(c, (attn_mma_kernel), grid, NT, SMEM, s, (const bf16*)q, q_row, q_tok, n_rows, (const bf16*)k, (const bf16*)v, n_keys,
                                         (bf16*)out, c->m.n_q_heads, n_kv, scale_log2, kt_per_split, opart,
                                         c->attn_ml);
  CB_LAUNCHED(c);
  if (n_splits > 1) CB_TRY(launch_attention_merge(c, R, n_splits, out, s));
  return CB_OK;
}

cb_status attention_tc_init() {
  CB_CUDA(cudaFuncSetAttribute(attn_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  return CB_OK;
}
