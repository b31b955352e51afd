// select.cu — HKVD selection (step a4): KV deviation (R1) and the top-k_i
// select over the candidates (Insight 1; ties -> lower token index, R6).
#include <algorithm>

#include "ctx.h"

__device__ __forceinline__ long long tc_globaltimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---------------------------------------------------------------------------------------------
// Delta_kv[j] = sum_h ( ||k_new[j,h] - k_ref[tok_j,h]||^2 + ||v_new[j,h] - v_ref[tok_j,h]||^2 ).
// One warp per candidate; per-head partials are warp-reduced in a fixed tree and summed over heads
// in index order, so the value is bitwise reproducible (and decomposes per kv head for TP).
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ void load4(const float* p, float (&x)[4]) {
  const float4 v = __ldg(reinterpret_cast<const float4*>(p));
  x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
}
__device__ __forceinline__ void load4(const bf16* p, float (&x)[4]) {
  const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
  const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v.x));
  const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v.y));
  x[0] = a.x; x[1] = a.y; x[2] = b.x; x[3] = b.y;
}

template <typename T>
__global__ void __launch_bounds__(256) deviation_kernel(const T* __restrict__ kn, const T* __restrict__ vn,
                                                        const T* __restrict__ kr, const T* __restrict__ vr,
                                                        const int* __restrict__ cand_tok, int n_cand, int n_kv,
                                                        int hd, int mode, float* __restrict__ dev) {
  pdl_enter();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= n_cand) return;
  const int kvd = n_kv * hd;
  const size_t a = (size_t)warp * kvd, b = (size_t)__ldg(cand_tok + warp) * kvd;
  // per-lane partial of every head first (all loads in flight together), then per-head warp sums
  // added in head order
  constexpr int MAXH = 16;
  float p[MAXH];
#pragma unroll
  for (int h = 0; h < MAXH; ++h) {
    p[h] = 0.f;
    if (h < n_kv) {
      for (int e = h * hd + lane * 4; e < (h + 1) * hd; e += 128) {  // 4 consecutive elements per lane
        float x[4], y[4], z[4], w[4];
        load4(kn + a + e, x);
        load4(kr + b + e, y);
        load4(vn + a + e, z);
        load4(vr + b + e, w);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (mode != CB_DEV_V) p[h] += (x[i] - y[i]) * (x[i] - y[i]);
          if (mode != CB_DEV_K) p[h] += (z[i] - w[i]) * (z[i] - w[i]);
        }
      }
    }
  }
  float tot = 0.f;
#pragma unroll
  for (int h = 0; h < MAXH; ++h)
    if (h < n_kv) tot += warp_sum(p[h]);
  if (lane == 0) dev[warp] = tot;
}

cb_status launch_deviation(cb_ctx* c, const void* k_new, const void* v_new, const void* k_ref, const void* v_ref,
                           const int* cand_tok, int n_cand, int dev_mode, float* dev, cudaStream_t s) {
  if (n_cand == 0) return CB_OK;
  const int grid = (n_cand + 7) / 8;
  ProfScope ps_(c, PROF_DEVIATION, s);
  if (c->m.dtype == CB_BF16)
    CB_LAUNCH(c, (deviation_kernel<bf16>), grid, 256, 0, s, (const bf16*)k_new, (const bf16*)v_new, (const bf16*)k_ref,
                                                (const bf16*)v_ref, cand_tok, n_cand, c->m.n_kv_heads,
                                                c->m.head_dim, dev_mode, dev);
  else
    CB_LAUNCH(c, (deviation_kernel<float>), grid, 256, 0, s, (const float*)k_new, (const float*)v_new, (const float*)k_ref,
                                                 (const float*)v_ref, cand_tok, n_cand, c->m.n_kv_heads,
                                                 c->m.head_dim, dev_mode, dev);
  CB_LAUNCHED(c);
  return CB_OK;
}

// ---------------------------------------------------------------------------------------------
// Top-k select, one CTA of 1024 threads. Deviations are non-negative, so their fp32 bit patterns
// order like the values: an MSB-first 4 x 8-bit radix select finds the k-th largest value v*;
// every candidate above v* is kept, and of those equal to v* the lowest slots (= lowest token
// indices, candidates are ascending) fill the remainder. Output is compacted in slot order, i.e.
// ascending token index. Replay mode (force_sel) maps forced tokens to their candidate slots.
// Outputs cover the kept rows then the suffix rows:
//   qrow[r] = row in the current compact buffers,  qtok[r] = token index.
// ---------------------------------------------------------------------------------------------
constexpr int TOPK_THREADS = 1024;
constexpr int TOPK_MAX_CAND = 49152;

__device__ __forceinline__ int block_excl_scan(int v, int* sm_warp, int* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sm_warp[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = lane < (int)(blockDim.x >> 5) ? sm_warp[lane] : 0;  // blocks of fewer than 32 warps
    int u = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, u, o);
      if (lane >= o) u += y;
    }
    sm_warp[lane] = u - t;  // exclusive prefix of warp totals
    if (lane == 31) *total = u;
  }
  __syncthreads();
  const int r = sm_warp[w] + x - v;
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(TOPK_THREADS) topk_kernel(float* __restrict__ dev,
                                                            const int* __restrict__ cand_tok, int n_cand, int k,
                                                            int n_suf, int N, const int* __restrict__ force_sel,
                                                            int* __restrict__ qrow, int* __restrict__ qtok,
                                                            int* __restrict__ sel_tok, int* err,
                                                            const float* __restrict__ dev_part, int n_kv, int ld_part,
                                                            int dev_mode, int drop_max,
                                                            long long* __restrict__ dbg) {
  // debug_trace 200: globaltimer of the phases (entry, inputs visible, Delta_kv summed, selected, done)
#define TK_DBG(i) do { if (dbg != nullptr && threadIdx.x == 0) dbg[i] = tc_globaltimer(); } while (0)
  TK_DBG(0);
  pdl_enter();
  TK_DBG(1);
  extern __shared__ unsigned keys[];
  __shared__ int hist[256];
  __shared__ int sm_warp[32];
  __shared__ int sm_total;
  __shared__ int sm_digit, sm_rem;
  const int tid = threadIdx.x;

  if (dev_part != nullptr) {  // Delta_kv from the QKV epilogue's per-(64-col block, k|v) partials, in order
    for (int j = tid; j < n_cand; j += blockDim.x) {
      float tot = 0.f;
      if (n_kv <= 16) {  // every partial load in flight at once, then the same sum order as below
        float a[16], b[16];
#pragma unroll
        for (int h = 0; h < 16; ++h) {
          a[h] = (h < n_kv && dev_mode != CB_DEV_V) ? dev_part[(size_t)(2 * h) * ld_part + j] : 0.f;
          b[h] = (h < n_kv && dev_mode != CB_DEV_K) ? dev_part[(size_t)(2 * h + 1) * ld_part + j] : 0.f;
        }
#pragma unroll
        for (int h = 0; h < 16; ++h)
          if (h < n_kv) tot += a[h] + b[h];
      } else {
#pragma unroll 8
        for (int h = 0; h < n_kv; ++h) {  // n_kv = number of 64-column blocks of a k (or v) row here
          const float a = dev_mode != CB_DEV_V ? dev_part[(size_t)(2 * h) * ld_part + j] : 0.f;
          const float b = dev_mode != CB_DEV_K ? dev_part[(size_t)(2 * h + 1) * ld_part + j] : 0.f;
          tot += a + b;
        }
      }
      dev[j] = tot;
      const unsigned u = __float_as_uint(tot);
      keys[j] = (u & 0x80000000u) ? 0u : u;  // the select keys, without re-reading dev (-0.0 -> 0)
    }
    __syncthreads();
  }
  TK_DBG(2);

  // suffix rows are always kept
  for (int s = tid; s < n_suf; s += blockDim.x) {
    qrow[k + s] = n_cand + s;
    qtok[k + s] = N + s;
  }
  if (force_sel != nullptr) {  // replay mode (R14)
    for (int r = tid; r < k; r += blockDim.x) {
      const int t = force_sel[r];
      int lo = 0, hi = n_cand;  // lower_bound
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (cand_tok[mid] < t) lo = mid + 1; else hi = mid;
      }
      if (lo >= n_cand || cand_tok[lo] != t) {
        atomicOr(err, CB_DEVERR_FORCE_SEL);
        lo = min(lo, n_cand - 1);
      }
      qrow[r] = lo;
      qtok[r] = t;
      if (sel_tok) sel_tok[r] = t;
    }
    return;
  }
  if (k == 0) return;

  if (dev_part == nullptr)  // (with the partials the keys were written while summing)
    for (int j = tid; j < n_cand; j += blockDim.x) {
      unsigned u = __float_as_uint(dev[j]);
      keys[j] = (u & 0x80000000u) ? 0u : u;  // -0.0 -> 0
    }
  // Gradual filtering keeps almost every candidate (k_i / k_(i-1) ~ 0.99 after layer 1): when only a few
  // are dropped, drop them one at a time (block argmin by (key, larger index first), which is exactly the
  // complement of "k largest, ties to the lower index") instead of four radix passes.
  constexpr unsigned DROPPED = 0xFFFFFFFFu;  // above every key (keys are bits of non-negative floats)
  const bool drop_path = k < n_cand && n_cand - k <= drop_max;
  if (drop_path && n_cand <= 1024) {
    // two warps, 16 keys per lane in registers (slot j = tid + 64 q; at 1024 threads a thread has 64 registers,
    // too few for 32 keys): d rounds of (lane minimum, warp minimum, the two warps' minima through shared
    // memory with a 64-thread named barrier) instead of the block-wide loop's two block barriers per key.
    // Same order, same selection.
    __syncthreads();
    if (tid < 64) {
      __shared__ unsigned long long wbest[2][2];  // [round parity][warp]
      unsigned k16[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int j = tid + 64 * q;
        k16[q] = j < n_cand ? keys[j] : DROPPED;
      }
      for (int r = 0; r < n_cand - k; ++r) {
        // the next slot to drop: smallest key, ties -> the larger slot (the complement of "k largest, ties
        // to the lower index"). Lane minimum in four chains, then the largest q holding it from a mask.
        unsigned m4[4] = {k16[0], k16[1], k16[2], k16[3]};
#pragma unroll
        for (int q = 4; q < 16; ++q) m4[q & 3] = min(m4[q & 3], k16[q]);
        const unsigned lmin = min(min(m4[0], m4[1]), min(m4[2], m4[3]));
        unsigned eq = 0;
#pragma unroll
        for (int q = 0; q < 16; ++q) eq |= (k16[q] == lmin ? 1u : 0u) << q;
        const int bq = 31 - __clz(eq);
        unsigned long long b = ((unsigned long long)lmin << 32) | (unsigned)(0x7FFFFFFF - (tid + 64 * bq));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const unsigned long long y = __shfl_xor_sync(0xffffffffu, b, o);
          b = y < b ? y : b;
        }
        if ((tid & 31) == 0) wbest[r & 1][tid >> 5] = b;
        asm volatile("bar.sync 2, 64;" ::: "memory");
        const unsigned long long b0 = wbest[r & 1][0], b1 = wbest[r & 1][1];
        b = b0 < b1 ? b0 : b1;
        const int jd = 0x7FFFFFFF - (int)(unsigned)(b & 0xFFFFFFFFu);
        if ((jd & 63) == tid) {
#pragma unroll
          for (int q = 0; q < 16; ++q)
            if (q == (jd >> 6)) k16[q] = DROPPED;
          keys[jd] = DROPPED;
        }
      }
    }
    __syncthreads();
  } else if (drop_path) {
    __syncthreads();
    __shared__ unsigned long long sm_best[32];
    for (int r = 0; r < n_cand - k; ++r) {
      // order (key ascending, index descending) packed so that the minimum is the next one to drop
      unsigned long long best = ~0ull;
      for (int j = tid; j < n_cand; j += blockDim.x) {
        const unsigned long long v = ((unsigned long long)keys[j] << 32) | (unsigned)(0x7FFFFFFF - j);
        best = v < best ? v : best;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(0xffffffffu, best, o);
        best = y < best ? y : best;
      }
      if ((tid & 31) == 0) sm_best[tid >> 5] = best;
      __syncthreads();
      if (tid < 32) {
        unsigned long long b = tid < (int)(blockDim.x >> 5) ? sm_best[tid] : ~0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const unsigned long long y = __shfl_xor_sync(0xffffffffu, b, o);
          b = y < b ? y : b;
        }
        if (tid == 0) keys[0x7FFFFFFF - (int)(unsigned)(b & 0xFFFFFFFFu)] = DROPPED;
      }
      __syncthreads();
    }
  }
  unsigned prefix = 0, mask = 0;
  int rem = k;
  if (drop_path) {
    prefix = 0; rem = 0;  // selection below: every key that was not dropped
  } else if (k < n_cand) {
    for (int pass = 0; pass < 4; ++pass) {
      const int shift = 24 - 8 * pass;
      if (tid < 256) hist[tid] = 0;
      __syncthreads();
      for (int j0 = 0; j0 < n_cand; j0 += blockDim.x) {  // warp-aggregated: one atomic per distinct bin
        const int j = j0 + tid;
        const unsigned key = j < n_cand ? keys[j] : 0u;
        const bool in = j < n_cand && (key & mask) == prefix;
        const unsigned act = __ballot_sync(0xffffffffu, in);
        if (in) {
          const int bin = (key >> shift) & 255;
          const unsigned peers = __match_any_sync(act, bin);
          if ((int)(tid & 31) == __ffs(peers) - 1) atomicAdd(&hist[bin], __popc(peers));
        }
      }
      __syncthreads();
      if (tid < 32) {  // warp 0: lane l owns bins [8l, 8l+8); find the digit holding the rem-th largest
        int cnt[8], lane_tot = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) { cnt[q] = hist[tid * 8 + q]; lane_tot += cnt[q]; }
        int above = lane_tot;  // inclusive suffix sum over lanes >= tid
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_down_sync(0xffffffffu, above, o);
          if (tid + o < 32) above += y;
        }
        const int strictly_above = above - lane_tot;  // keys in bins of higher lanes
        if (strictly_above < rem && rem <= above) {
          int cum = strictly_above;
          for (int q = 7; q >= 0; --q) {
            if (cum + cnt[q] >= rem) { sm_digit = tid * 8 + q; sm_rem = rem - cum; break; }
            cum += cnt[q];
          }
        }
      }
      __syncthreads();
      prefix |= (unsigned)sm_digit << shift;
      mask |= 255u << shift;
      rem = sm_rem;
      __syncthreads();
    }
  } else {
    prefix = 0; rem = n_cand;  // take everything: every key >= 0 qualifies via the eq path below
  }
  TK_DBG(3);
  const unsigned vstar = prefix;
  const bool all = (k >= n_cand);
  // drop path: sel = not dropped, expressed through the same compaction (key > vstar, no ties)

  if (drop_path && n_cand <= (int)blockDim.x) {
    // one candidate per thread: warp ballots and one exchange of warp counts (one barrier) place each kept
    // slot at its rank, in slot order
    const bool sel = tid < n_cand && keys[tid] != DROPPED;
    const unsigned bal = __ballot_sync(0xffffffffu, sel);
    const int lane = tid & 31, w = tid >> 5;
    if (lane == 0) sm_warp[w] = __popc(bal);
    __syncthreads();
    const int nw = (int)(blockDim.x >> 5);
    int before = lane < w ? sm_warp[lane] : 0;  // warps before this one (w <= 31)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) before += __shfl_xor_sync(0xffffffffu, before, o);
    (void)nw;
    if (sel) {
      const int out = before + __popc(bal & ((1u << lane) - 1u));
      const int t = cand_tok[tid];
      qrow[out] = tid;
      qtok[out] = t;
      if (sel_tok) sel_tok[out] = t;
    }
    TK_DBG(4);
    return;
  }
  // contiguous segment per thread so that slot order is preserved by the scans
  const int seg = (n_cand + blockDim.x - 1) / blockDim.x;
  const int j0 = min(n_cand, tid * seg), j1 = min(n_cand, j0 + seg);
  int n_eq = 0;
  if (!all && !drop_path)
    for (int j = j0; j < j1; ++j) n_eq += (keys[j] == vstar);
  // (block-uniform) only the radix path has ties at the k-th value to resolve
  const int eq_before = (all || drop_path) ? 0 : block_excl_scan(n_eq, sm_warp, &sm_total);
  int n_sel = 0, eq = eq_before;
  for (int j = j0; j < j1; ++j) {
    const unsigned key = keys[j];
    bool sel = drop_path ? key != DROPPED : (all || key > vstar);
    if (!drop_path && !all && key == vstar) { sel = eq < rem; ++eq; }
    n_sel += sel;
  }
  int out = block_excl_scan(n_sel, sm_warp, &sm_total);
  eq = eq_before;
  for (int j = j0; j < j1; ++j) {
    const unsigned key = keys[j];
    bool sel = drop_path ? key != DROPPED : (all || key > vstar);
    if (!drop_path && !all && key == vstar) { sel = eq < rem; ++eq; }
    if (sel) {
      const int t = cand_tok[j];
      qrow[out] = j;
      qtok[out] = t;
      if (sel_tok) sel_tok[out] = t;
      ++out;
    }
  }
  TK_DBG(4);
#undef TK_DBG
}

cb_status launch_topk(cb_ctx* c, float* dev, const int* cand_tok, int n_cand, int k_keep, int n_suffix, int N,
                      const int* force_sel, int* qrow, int* qtok, int* sel_tok, cudaStream_t s,
                      const float* dev_part, int ld_part, int dev_mode) {
  CB_REQUIRE(n_cand <= TOPK_MAX_CAND, CB_E_SHAPE, "top-k: n_cand %d exceeds %d", n_cand, TOPK_MAX_CAND);
  if (k_keep + n_suffix == 0 && (dev_part == nullptr || n_cand == 0)) return CB_OK;
  ProfScope ps_(c, PROF_TOPK, s);
  // threads: 1024, or fewer when the candidates are few (cheaper block barriers), cb_set_option("topk_threads")
  int nt = TOPK_THREADS;
  if (c->topk_threads > 0) nt = c->topk_threads;
  const size_t smem = (size_t)std::max(1, n_cand) * sizeof(unsigned);  // the select keys
  CB_LAUNCH(c, (topk_kernel), 1, nt, smem, s, dev, cand_tok, n_cand, k_keep, n_suffix, N, force_sel, qrow, qtok, sel_tok,
                                            c->err_word, dev_part, c->m.n_kv_heads * c->m.head_dim / 64 * std::max(1, c->tp_world), ld_part,
                                            dev_mode, c->topk_drop_max,
                                            c->dbg_sel == 200 ? c->dbg_buf : nullptr);
  CB_LAUNCHED(c);
  return CB_OK;
}

cb_status topk_init_attrs() {
  CB_CUDA(cudaFuncSetAttribute(topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               TOPK_MAX_CAND * (int)sizeof(unsigned)));
  return CB_OK;
}
