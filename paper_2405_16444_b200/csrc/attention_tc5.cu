// attention_tc5.cu — tcgen05 / TMEM / TMA sparse-query causal attention (step a6), bf16, head_dim 128.
//
// out[r][h] = softmax_j(q_{r,h} . k_{j,g} / sqrt(hd)) v_{j,g} over keys j <= q_tok[r]
//
// One CTA = one kv head g x 128 (query token, q head of g) rows (GQA packing: every K/V tile serves
// all G q heads of the group) x one split of the key range (split-KV for the later layers' few
// hundred queries). Warp roles:
//   warp 0     TMA: K and V tiles (128 keys x 128, two 64-column SWIZZLE_128B boxes each) into a 3-stage K
//              ring and a 2-stage V ring (3-D tensor map over [keys][kv heads][hd]), K running ahead of V
//   warp 1     MMA issuer: S_t = Q K_t^T (M=128, N=128 keys, K=16; A = Q from TMEM) into one of two TMEM S
//              buffers, then O += P_t V_t (A = P from TMEM, B = V MN-major) into the TMEM O buffer.
//              S_{t+1} is issued before waiting for P_t, so QK^T overlaps the softmax of tile t.
//   warps 2-9  softmax: two warpgroups, thread = (query row, 64-key half). Its half of the gathered Q row is
//              loaded before the prologue and stored into TMEM after it. Each tcgen05.lds its half of
//              the S row, masks by original position, and the two halves agree on the row max through
//              shared memory; online softmax in the log2 domain with lazy rescaling (O is rescaled in
//              TMEM only when the row max grows by more than 2^8); P (bf16 pairs) is written over the
//              half's own S columns, where the PV MMA reads it; finally O / l (or the split partial),
//              each half writing its 64 output columns.
// Key tiles past the CTA's last query token are never loaded; only tiles reaching past its first
// query token are masked.
// Load balance: the rows are in token order, so the last row tiles see the most keys. Every row tile
// gets n_splits CTAs over fixed key ranges of kt_per_split tiles (empty ranges exit at once), launched
// heaviest first. When a row tile has more than one non-empty range, each CTA writes an fp32 partial
// (O, m, l) and bumps the tile's counter; the last one to arrive merges all partials in split order
// (deterministic) and writes the output -- no separate merge launch.
// Variants measured and removed (source in git history): a share of the exponentials on
// the FMA pipe, four softmax warpgroups, Q staged in shared memory, light/heavy row-tile pairing in
// 2-CTA clusters with a DSMEM merge, two key streams per CTA, P packed on the integer pipe, the output
// staged through shared memory, the first K/V tiles issued before the prologue sync.
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>
#include <vector>
#include <unordered_map>

#include "ctx.h"
#include "tc_common.cuh"

namespace {
constexpr int HD = 128, BM = 128, BC = 128;
constexpr int KW = 64, OW = 64, NSM = 256;  // per softmax thread: 64 keys of a tile, 64 output columns; 256 threads
constexpr int NTHREADS = 64 + NSM;
constexpr int ATOM = 128 * 128;    // 128 rows x 128 B (64 bf16): one SWIZZLE_128B column block
constexpr int TILE = 2 * ATOM;     // 128 rows x 128 bf16
constexpr int KST = 3;             // K ring stages (V: 2); Q and P live in TMEM, so SMEM = 3 K + 2 V
// + alignment + barriers + exchange (xmax [2 parity][2][128], l [2][128], flag)
constexpr int SMEM = 5 * TILE + 1024 + 256 + 7 * 128 * 4 + 64;
constexpr float RESCALE_THRESHOLD = 8.0f;    // log2 units
constexpr uint32_t QCOL = 384;               // TMEM columns of Q: 64 x 32-bit = 128 bf16 per row

__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ float ex2(float x) {  // MUFU.EX2, ~2 ulp; ex2(-inf) = 0
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// Key tiles a row tile needs (through its last query token) and its first query token.
__device__ __forceinline__ void tile_span(const int* __restrict__ q_tok, int tile, int R, int G, int n_keys, int& n_kt,
                                          int& kmin) {
  int kmax = -1;
  kmin = 1 << 30;
  const int rho0 = tile * BM;
  for (int rr = rho0 / G; rr <= min(R - 1, rho0 + BM - 1) / G; ++rr) {
    const int t = min(__ldg(q_tok + rr), n_keys - 1);
    kmax = max(kmax, t);
    kmin = min(kmin, t);
  }
  n_kt = (kmax + BC) / BC;
}

// A CTA's rows are done: o holds this thread's OW unnormalised output columns (wg * OW ..) of row rho, m_used
// the row's reference max (log2 domain), l its exp sum. A row tile covered by one CTA writes O / l. Covered by
// several (split-KV), each CTA writes an fp32 partial (thread-major slots: coalesced stores and loads), counts
// its arrival, and the last arrival merges every split's partial in split order (deterministic) and writes.
__device__ __forceinline__ void finish_rows(float (&o)[OW], float m_used, float l, bool partial, bool write_out,
                                            int n_active, int sidx, int tile, int g, int n_kv, int R, int rho,
                                            bool valid, int rt, int hh, int qd, int et, int wg, int* flag,
                                            float* __restrict__ opart, float2* __restrict__ ml,
                                            int* __restrict__ tile_cnt, bf16* __restrict__ out) {
  // partial slots: rows padded to whole tiles; inside a tile's block the float4s are thread-major
  // ([OW / 4][NSM]), so the partial stores and the merge's loads are coalesced across a warp
  const size_t rpad = (size_t)(((R + BM - 1) / BM) * BM);
  const size_t part_row0 = ((size_t)sidx * n_kv + g) * rpad;
  if (partial) {
    if (valid) {
      float4* dst = reinterpret_cast<float4*>(opart + (part_row0 + (size_t)tile * BM) * HD) + et;
#pragma unroll
      for (int i = 0; i < OW / 4; ++i)
        __stcg(dst + i * NSM, make_float4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]));
      if (wg == 0) ml[part_row0 + rho] = make_float2(m_used, l);
    }
    __threadfence();  // partials visible device-wide before the arrival is counted
    named_bar_sync(1, NSM);
    if (et == 0) {
      const int old = atomicAdd(tile_cnt + (size_t)tile * n_kv + g, 1);
      const int last = old == n_active - 1;
      if (last) tile_cnt[(size_t)tile * n_kv + g] = 0;  // reset for the next launch
      tc::sts_s32(flag, last);
    }
    named_bar_sync(1, NSM);
    write_out = tc::lds_s32(flag) != 0;
    if (write_out) {  // last arrival: merge every range's partial in split order
      __threadfence();
      float mstar = -INFINITY;
      for (int sp = 0; sp < n_active; ++sp)
        if (valid) mstar = fmaxf(mstar, __ldcg(&ml[((size_t)sp * n_kv + g) * rpad + rho].x));
      float lt = 0.f;
#pragma unroll
      for (int i = 0; i < OW; ++i) o[i] = 0.f;
      for (int sp = 0; sp < n_active && valid; ++sp) {
        const size_t prow = ((size_t)sp * n_kv + g) * rpad;
        const float2 ms = __ldcg(&ml[prow + rho]);
        if (ms.x == -INFINITY) continue;
        const float f = ex2(ms.x - mstar);
        lt += ms.y * f;
        const float4* src = reinterpret_cast<const float4*>(opart + (prow + (size_t)tile * BM) * HD) + et;
#pragma unroll
        for (int i = 0; i < OW / 4; ++i) {
          const float4 x = __ldcg(src + i * NSM);
          o[4 * i] += x.x * f; o[4 * i + 1] += x.y * f; o[4 * i + 2] += x.z * f; o[4 * i + 3] += x.w * f;
        }
      }
      l = lt;
    }
  }
  if (valid && write_out) {
    const float inv = l > 0.f ? 1.f / l : 0.f;
    uint4* dst = reinterpret_cast<uint4*>(out + (size_t)rt * qd + (size_t)hh * HD + wg * OW);
#pragma unroll
    for (int c8 = 0; c8 < OW / 8; ++c8) {
      uint4 w;
      w.x = pack2(o[c8 * 8 + 0] * inv, o[c8 * 8 + 1] * inv);
      w.y = pack2(o[c8 * 8 + 2] * inv, o[c8 * 8 + 3] * inv);
      w.z = pack2(o[c8 * 8 + 4] * inv, o[c8 * 8 + 5] * inv);
      w.w = pack2(o[c8 * 8 + 6] * inv, o[c8 * 8 + 7] * inv);
      dst[c8] = w;
    }
  }
}

__global__ void __launch_bounds__(NTHREADS, 1)
    attn_tc5_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                    const bf16* __restrict__ q, const int* __restrict__ q_row, const int* __restrict__ q_tok,
                    int n_rows, int n_keys, bf16* __restrict__ out, int n_q, int n_kv, float scale_log2,
                    int kt_per_split, int n_splits, float* __restrict__ opart, float2* __restrict__ ml,
                    int* __restrict__ tile_cnt, long long* __restrict__ dbg) {
  pdl_enter();
#ifdef CB_ATTN_TRACE
  const long long t_start = tc::globaltimer();
#ifndef CB_ATTN_TRACE_CTA
#define CB_ATTN_TRACE_CTA 0  // which CTA's pipeline to trace (-DCB_ATTN_TRACE_CTA=n; tools/attn_trace.py)
#endif
  const bool dbg_on = dbg != nullptr && blockIdx.x == CB_ATTN_TRACE_CTA;
#define DBG(i) do { if (dbg_on && (i) < 2048) dbg[i] = clock64(); } while (0)
#else
#define DBG(i) do { } while (0)
#endif
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem;                 // [KST] stages
  uint8_t* sV = smem + KST * TILE;    // [2] stages
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (KST + 2) * TILE);
  uint64_t* k_full = bars;            // [3]  K tile landed
  uint64_t* k_empty = bars + 3;       // [3]  S MMAs done reading the K stage
  uint64_t* v_full = bars + 6;        // [2]  V tile landed
  uint64_t* v_empty = bars + 8;       // [2]  PV MMAs done reading the V stage
  uint64_t* s_full = bars + 10;       // [2]  S_t in TMEM buffer t % 2
  uint64_t* q_full = bars + 12;
  uint64_t* p_full = bars + 13;       // P_t written over S_t (8 softmax warps)
  uint64_t* pv_done = bars + 14;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 15);
  float* xmax = reinterpret_cast<float*>(bars + 16);  // [2 parity][2 halves][128 rows], then l [2][128], flag
  float* xl = xmax + 2 * 2 * 128;
  int* flag = reinterpret_cast<int*>(xl + 2 * 128);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = n_q / n_kv, R = n_rows * G;
  const int qd = n_q * HD;
  // 1-D grid, kv head fastest: the heaviest row tiles (latest tokens) of EVERY head launch first, then their
  // later key ranges, then lighter tiles (a global longest-first order across heads)
  const int g = (int)blockIdx.x % n_kv;
  const int tiles = gridDim.x / (n_splits * n_kv);
  const int rest = (int)blockIdx.x / n_kv;
  const int tile = tiles - 1 - rest / n_splits;
  const int split = rest % n_splits;
  int n_kt, kmin;
  tile_span(q_tok, tile, R, G, n_keys, n_kt, kmin);
  const int jb = split * kt_per_split, je = min(n_kt, jb + kt_per_split);
  if (jb >= je) return;  // nothing in this range (the tile's other CTAs do not count it)
  const int nt = je - jb, n_active = (n_kt + kt_per_split - 1) / kt_per_split;
  // softmax threads: row (token, q head) of this thread and its half of Q, loaded before the prologue so the
  // gathered-row loads (q_row, then the row) overlap the barrier init and the TMEM allocation
  const int wg = (warp - 2) >> 2;  // 0: keys / O columns 0..63, 1: 64..127
  const int r = (warp & 3) * 32 + lane;
  const int rho = tile * BM + r;
  const bool valid = warp >= 2 && rho < R;
  const int rt = valid ? rho / G : 0, hh = g * G + (valid ? rho % G : 0);
  uint4 qv[KW / 8];
#pragma unroll
  for (int c8 = 0; c8 < KW / 8; ++c8) qv[c8] = make_uint4(0u, 0u, 0u, 0u);
  if (valid) {
    const uint4* src = reinterpret_cast<const uint4*>(q + (size_t)__ldg(q_row + rt) * qd + (size_t)hh * HD + wg * KW);
#pragma unroll
    for (int c8 = 0; c8 < KW / 8; ++c8) qv[c8] = __ldg(src + c8);
  }

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tmK);
    tc::tma_prefetch(&tmV);
    for (int b = 0; b < KST; ++b) {
      tc::mbar_init(&k_full[b], 1);
      tc::mbar_init(&k_empty[b], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&v_full[b], 1);
      tc::mbar_init(&v_empty[b], 1);
      tc::mbar_init(&s_full[b], 1);
    }
    tc::mbar_init(q_full, NSM);
    tc::mbar_init(p_full, NSM / 32);
    tc::mbar_init(pv_done, 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  DBG(1200);
  const uint32_t tmem = *tmem_slot;  // S0: cols [0,128), S1: [128,256), O: [256,384), Q: [384,448)

  if (warp == 0) {
    // ===== TMA producer: K_t as soon as S_{t-3} released its stage, V_t once PV_{t-2} did, so K runs
    // ahead of V (S_t needs K_t a whole softmax before PV_t needs V_t) =====
    if (tc::elect_one()) {
      auto load = [&](uint8_t* dst, const CUtensorMap* m, uint64_t* bar, int key0) {
        tc::mbar_arrive_expect_tx(bar, TILE);
        tc::tma_load_3d(dst, m, bar, 0, g, key0);
        tc::tma_load_3d(dst + ATOM, m, bar, 64, g, key0);
      };
      int tk = 0, tv = 0;  // the K and V streams advance independently, polling their empty barriers
      while (tk < nt || tv < nt) {
        if (tk < nt && (tk < KST || tc::mbar_test(&k_empty[tk % KST], (tk / KST - 1) & 1))) {
          DBG(4 * tk);
          load(sK + (tk % KST) * TILE, &tmK, &k_full[tk % KST], (jb + tk) * BC);
          ++tk;
        }
        if (tv < tk && (tv < 2 || tc::mbar_test(&v_empty[tv & 1], ((tv >> 1) - 1) & 1))) {
          DBG(4 * tv + 1);
          load(sV + (tv & 1) * TILE, &tmV, &v_full[tv & 1], (jb + tv) * BC);
          ++tv;
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer =====
    constexpr uint32_t IDESC_S = tc::idesc_bf16(BM, BC);
    constexpr uint32_t IDESC_PV = tc::idesc_bf16_bmn(BM, HD);
    const uint32_t tO = tmem + 256;
    // S_{t+2} reuses TMEM buffer t % 2, which holds P_t: it is issued after PV_t on the in-order
    // tensor pipe, so no extra barrier is needed
    auto issue_s = [&](int t) {
      const int b = t & 1, kb = t % KST;
      tc::mbar_wait(&k_full[kb], (t / KST) & 1);
      if (lane == 0) DBG(400 + 4 * t);
      tc::fence_after();
      if (tc::elect_one()) {
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint64_t bd = tc::sdesc_sw128(sK + kb * TILE + (kk >> 2) * ATOM) + 2 * (kk & 3);
          tc::mma_bf16_ts(tmem + b * 128, tmem + QCOL + 8 * kk, bd, IDESC_S, kk > 0 ? 1u : 0u);
        }
        tc::mma_commit(&s_full[b]);
        tc::mma_commit(&k_empty[kb]);
      }
      __syncwarp();
    };
    tc::mbar_wait(q_full, 0);
    issue_s(0);
    for (int t = 0; t < nt; ++t) {
      if (t + 1 < nt) issue_s(t + 1);
      tc::mbar_wait(p_full, t & 1);
      tc::mbar_wait(&v_full[t & 1], (t >> 1) & 1);
      if (lane == 0) DBG(400 + 4 * t + 1);
      tc::fence_after();
      if (tc::elect_one()) {
        const int b = t & 1;
#pragma unroll
        for (int kk = 0; kk < BC / 16; ++kk) {  // 16 keys per step; P in TMEM (keys 0-63 at columns 0-31 of
          // the S buffer, keys 64-127 at columns 64-95: each softmax half over its own S)
          const uint32_t a = tmem + b * 128 + (kk * 16 / KW) * KW + ((kk * 16) % KW) / 2;
          const uint64_t bd = tc::sdesc_sw128_mn(sV + b * TILE + kk * 2048, ATOM);
          tc::mma_bf16_ts(tO, a, bd, IDESC_PV, (t > 0 || kk > 0) ? 1u : 0u);
        }
        tc::mma_commit(pv_done);
        tc::mma_commit(&v_empty[b]);
      }
      __syncwarp();
    }
    // drain: the release commits of the last K / V stages have no consumer; wait for their arrivals so no
    // tcgen05.commit arrive is in flight when the CTA exits (compute-sanitizer synccheck: "missing wait")
    for (int t = max(0, nt - KST); t < nt; ++t) tc::mbar_wait(&k_empty[t % KST], (t / KST) & 1);
    for (int t = max(0, nt - 2); t < nt; ++t) tc::mbar_wait(&v_empty[t & 1], (t >> 1) & 1);
  } else {
    // ===== softmax / correction / epilogue: two warpgroups, each owns one 64-key half of every row
    // (thread = (row, half)); the halves agree on the row max through shared memory every tile =====
    const int et = threadIdx.x - 64;  // 0..NSM-1 among softmax threads
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const int tok = valid ? min(__ldg(q_tok + rt), n_keys - 1) : -1;
    {  // this row's 64 elements of Q (half wg) -> TMEM columns QCOL + 32 wg .. (bf16 pairs), the QK^T A operand
      uint32_t pk[KW / 2];
#pragma unroll
      for (int c8 = 0; c8 < KW / 8; ++c8) {
        pk[4 * c8] = qv[c8].x; pk[4 * c8 + 1] = qv[c8].y; pk[4 * c8 + 2] = qv[c8].z; pk[4 * c8 + 3] = qv[c8].w;
      }
      tc::tmem_st32u(tmem + lane_base + QCOL + wg * (KW / 2), pk);
      tc::tmem_st_wait();
      tc::fence_before();
      tc::mbar_arrive(q_full);
    }
    float m_used = -INFINITY, l = 0.f;
    for (int t = 0; t < nt; ++t) {
      const int b = t & 1;
      tc::mbar_wait(&s_full[b], (t >> 1) & 1);
      if (et == 0) DBG(800 + 4 * t);
      tc::fence_after();
      float s[KW];
#pragma unroll
      for (int c = 0; c < KW / 32; ++c) {
        float x[32];
        tc::tmem_ld32(tmem + lane_base + b * 128 + wg * KW + c * 32, x);
#pragma unroll
        for (int i = 0; i < 32; ++i) s[c * 32 + i] = x[i];
      }
      const int key0 = (jb + t) * BC + wg * KW;
      const bool need_mask = key0 + KW - 1 > kmin;
      // half-row max of the raw scores (scale > 0 commutes with max); 8 chains for ILP
      float mx8[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) mx8[i] = -INFINITY;
      if (need_mask) {
#pragma unroll
        for (int i = 0; i < KW; ++i) {
          if (key0 + i > tok) s[i] = -INFINITY;
          mx8[i & 7] = fmaxf(mx8[i & 7], s[i]);
        }
      } else {
#pragma unroll
        for (int i = 0; i < KW; ++i) mx8[i & 7] = fmaxf(mx8[i & 7], s[i]);
      }
      const float hmx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                              fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
      tc::sts_f32(xmax + (b * 2 + wg) * 128 + r, hmx);
      named_bar_sync(1, NSM);
      const float mx = fmaxf(tc::lds_f32(xmax + (b * 2) * 128 + r), tc::lds_f32(xmax + (b * 2 + 1) * 128 + r)) *
                       scale_log2;  // exact, any order
      if (et == 0) DBG(800 + 4 * t + 1);
      // lazy rescale (identical decision in both halves): move the reference max only when it grew
      // by more than 2^8
      float corr = 1.f;
      if (mx > m_used + RESCALE_THRESHOLD || (m_used == -INFINITY && mx != -INFINITY)) {
        if (m_used != -INFINITY) corr = ex2(m_used - mx);
        m_used = mx;
      }
      const float nref = m_used == -INFINITY ? 0.f : -m_used;
      l *= corr;
      // packed fp32x2 FFMA2 / FADD2 (sm_100) halve the FMA-pipe issue slots of the scale and the row sum;
      // accumulator j of rs2 holds elements 8m + 2j (.x) and 8m + 2j + 1 (.y), the same partition and
      // order as eight scalar accumulators indexed by element % 8
      const float2 sc2 = make_float2(scale_log2, scale_log2), nr2 = make_float2(nref, nref);
      float2 rs2[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) rs2[i] = make_float2(0.f, 0.f);
#pragma unroll
      for (int i = 0; i < KW / 2; ++i) {
        float2 xa = __ffma2_rn(make_float2(s[2 * i], s[2 * i + 1]), sc2, nr2);
        xa.x = ex2(xa.x);
        xa.y = ex2(xa.y);
        s[2 * i] = xa.x;
        s[2 * i + 1] = xa.y;
        rs2[i & 3] = __fadd2_rn(rs2[i & 3], xa);
      }
      l += ((rs2[0].x + rs2[0].y) + (rs2[1].x + rs2[1].y)) + ((rs2[2].x + rs2[2].y) + (rs2[3].x + rs2[3].y));
      // PV_{t-1} is complete long before here (issued a whole softmax ago); waiting on every phase keeps
      // the barrier protocol explicit (compute-sanitizer synccheck) and O stable for the rescale below
      if (t >= 1) tc::mbar_wait(pv_done, (t - 1) & 1);
      // rescale O only when the reference max moved
      if (t >= 1 && __any_sync(0xffffffffu, corr != 1.f)) {  // warp-collective TMEM read-modify-write
        if (et == 0) DBG(800 + 4 * t + 2);
        tc::fence_after();
#pragma unroll
        for (int c = 0; c < OW / 32; ++c) {
          float o[32];
          tc::tmem_ld32(tmem + lane_base + 256 + wg * OW + c * 32, o);
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] *= corr;
          tc::tmem_st32(tmem + lane_base + 256 + wg * OW + c * 32, o);
        }
      }
      {  // P (bf16 pairs) over this half's own S columns: keys wg*KW .. -> columns b*128 + wg*KW ..
        uint32_t pk[KW / 2];
#pragma unroll
        for (int i = 0; i < KW / 2; ++i) pk[i] = pack2(s[2 * i], s[2 * i + 1]);
        tc::tmem_st32u(tmem + lane_base + b * 128 + wg * KW, pk);
      }
      tc::tmem_st_wait();
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(p_full);
      if (et == 0) DBG(800 + 4 * t + 3);
    }
    // total row sum = both halves (same reference max), in half order
    tc::sts_f32(xl + wg * 128 + r, l);
    named_bar_sync(1, NSM);
    l = tc::lds_f32(xl + r) + tc::lds_f32(xl + 128 + r);
    tc::mbar_wait(pv_done, (nt - 1) & 1);
    tc::fence_after();
    float o[OW];
#pragma unroll
    for (int c = 0; c < OW / 32; ++c) {
      float x[32];
      tc::tmem_ld32(tmem + lane_base + 256 + wg * OW + c * 32, x);
#pragma unroll
      for (int i = 0; i < 32; ++i) o[c * 32 + i] = x[i];
    }
    finish_rows(o, m_used, l, n_active > 1, n_active == 1, n_active, split, tile, g, n_kv, R, rho, valid, rt, hh, qd,
                et, wg, flag, opart, ml, tile_cnt, out);
  }
  tc::fence_before();
  __syncthreads();
  DBG(1202);
#ifdef CB_ATTN_TRACE
  // per-CTA span (globaltimer) of every CTA with linear id < 370 at dbg[1300 + 2 id]
  if (dbg != nullptr && threadIdx.x == 0) {
    const int id = blockIdx.x;
    if (id < 370) { dbg[1300 + 2 * id] = t_start; dbg[1300 + 2 * id + 1] = tc::globaltimer(); }
  }
#endif
#undef DBG
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

PFN_cuTensorMapEncodeTiled_v12000 g_encode5 = nullptr;

// Tensor maps of K/V buffers, cached across calls and contexts: the key holds every field the map encodes
// (an address reused by another context with other kv heads must not hit a stale map), and the cache is
// shared by all host threads (head-parallel loopback ranks), hence the mutex.
struct KvKey {
  const void* p;
  int n_keys, n_kv;
  bool operator==(const KvKey& o) const { return p == o.p && n_keys == o.n_keys && n_kv == o.n_kv; }
};
std::mutex g_kvmaps_mu;
struct KvKeyHash {
  size_t operator()(const KvKey& k) const { return std::hash<const void*>()(k.p) ^ ((size_t)k.n_keys * 0x9e3779b9) ^ ((size_t)k.n_kv << 40); }
};
std::unordered_map<KvKey, CUtensorMap, KvKeyHash>* g_kvmaps = nullptr;

cb_status kv_tmap(const cb_ctx* c, const void* p, int n_keys, CUtensorMap* out) {
  KvKey key{p, n_keys, c->m.n_kv_heads};
  std::lock_guard<std::mutex> lk(g_kvmaps_mu);
  auto it = g_kvmaps->find(key);
  if (it != g_kvmaps->end()) { *out = it->second; return CB_OK; }
  const int n_kv = c->m.n_kv_heads;
  cuuint64_t dims[3] = {(cuuint64_t)HD, (cuuint64_t)n_kv, (cuuint64_t)n_keys};
  cuuint64_t strides[2] = {(cuuint64_t)HD * 2, (cuuint64_t)n_kv * HD * 2};
  cuuint32_t box[3] = {64, 1, (cuuint32_t)BC};
  cuuint32_t es[3] = {1, 1, 1};
  CUtensorMap m;
  CUresult r = g_encode5(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(p), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CB_REQUIRE(r == CUDA_SUCCESS, CB_E_CUDA, "cuTensorMapEncodeTiled (K/V) failed (%d)", (int)r);
  if (g_kvmaps->size() > 4096) g_kvmaps->clear();
  g_kvmaps->emplace(key, m);
  *out = m;
  return CB_OK;
}
}  // namespace

cb_status kv_tmap5(const cb_ctx* c, const void* p, int n_keys, CUtensorMap* out) { return kv_tmap(c, p, n_keys, out); }

bool attention_tc5_ok(const cb_ctx* c) { return c->m.dtype == CB_BF16 && c->m.head_dim == HD && g_encode5 != nullptr; }

// Split count for a grid of at least half a wave: list-schedule the CTAs in launch order (heaviest row tiles
// first, then their later key ranges) on num_sms SMs with a per-CTA cost of F + key tiles (+ M for a CTA that
// writes and merges partials), and take the split count with the shortest makespan. Row tile p is assumed to
// reach key tile ceil(max_kt (p + 1) / tiles) (selected tokens spread over the context; the suffix last).
// Costs in key-tile units, measured on B200 (tools/attn_spans.py): CTA time ~ 8 + 1.0 x key tiles us; a split
// range adds ~1.5 (partial write, merge by the last arrival; thread-major partials).
static int attn_pick_splits_uncached(int tiles, int max_kt, int n_kv, int num_sms) {
  constexpr double F = 8.0, M = 1.5;
  int best = 1;
  double best_t = 1e30;
  for (int ns = 1; ns <= 3; ++ns) {
    const int kps = (max_kt + ns - 1) / ns;
    std::vector<double> sm(num_sms, 0.0);
    double span = 0.0;
    for (int p = tiles - 1; p >= 0; --p) {
      const int kt = (int)(((long long)max_kt * (p + 1) + tiles - 1) / tiles);
      const int active = (kt + kps - 1) / kps;
      for (int sp = 0; sp < ns; ++sp) {
        const int len = std::min(kt, (sp + 1) * kps) - sp * kps;
        if (len <= 0) continue;
        const double d = F + len + (active > 1 ? M : 0.0);
        for (int h = 0; h < n_kv; ++h) {
          auto it = std::min_element(sm.begin(), sm.end());
          *it += d;
          span = std::max(span, *it);
        }
      }
    }
    if (span < best_t - 0.5) { best_t = span; best = ns; }
  }
  return best;
}

// The list scheduling costs ~10^5 host operations (tens of us per eager launch): memoised per shape.
static int attn_pick_splits(int tiles, int max_kt, int n_kv, int num_sms) {
  static std::mutex mu;
  static std::unordered_map<uint64_t, int> memo;
  const uint64_t key = ((uint64_t)tiles << 40) ^ ((uint64_t)max_kt << 20) ^ ((uint64_t)n_kv << 10) ^ (uint64_t)num_sms;
  std::lock_guard<std::mutex> lk(mu);
  auto it = memo.find(key);
  if (it != memo.end()) return it->second;
  const int ns = attn_pick_splits_uncached(tiles, max_kt, n_kv, num_sms);
  if (memo.size() > 65536) memo.clear();
  memo.emplace(key, ns);
  return ns;
}

cb_status launch_attention_tc5(cb_ctx* c, const void* q, const int* q_row, const int* q_tok, int n_rows, const void* k,
                               const void* v, int n_keys, void* out, cudaStream_t s) {
  if (n_rows == 0) return CB_OK;
  CB_REQUIRE(((uintptr_t)k | (uintptr_t)v) % 16 == 0, CB_E_INVALID_ARG, "K/V must be 16-byte aligned");
  const int n_kv = c->m.n_kv_heads, G = c->m.n_q_heads / n_kv;
  const int R = n_rows * G;
  const int tiles = (R + BM - 1) / BM;
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)HD);
  const int max_kt = (n_keys + BC - 1) / BC;
  const long long base = (long long)tiles * n_kv;
  int n_splits = 1;
  if (c->attn_splits > 0) {
    n_splits = c->attn_splits;
  } else if (2 * base < (long long)c->num_sms) {
    // measured (tools/attn_micro.py): extra CTAs only pay off when the (row tile, head) grid leaves
    // more than half of the SMs idle -- split CTAs run as extra waves with their own prologues
    n_splits = (int)std::min<long long>((c->num_sms + base - 1) / base, (max_kt + 3) / 4);
  } else {
    n_splits = attn_pick_splits(tiles, max_kt, n_kv, c->num_sms);
  }
  n_splits = std::min(n_splits, (int)(c->attn_part_rows / ((long long)tiles * BM * n_kv)));  // padded slots
  n_splits = std::max(1, std::min(n_splits, 16));
  const int kt_per_split = (max_kt + n_splits - 1) / n_splits;
  CB_REQUIRE(base <= c->attn_cnt_n, CB_E_SHAPE, "attention: %lld row tiles exceed the counter array", base);
  CUtensorMap tk, tv;
  CB_TRY(kv_tmap(c, k, n_keys, &tk));
  CB_TRY(kv_tmap(c, v, n_keys, &tv));
  dim3 grid(tiles * n_splits * n_kv);
  ProfScope ps_(c, PROF_ATTN, s);
  CB_CUDA(launch_k(c, attn_tc5_kernel, grid, dim3(NTHREADS), SMEM, s, 1, tk, tv, (const bf16*)q, q_row, q_tok, n_rows,
                   n_keys, (bf16*)out, c->m.n_q_heads, n_kv, scale_log2, kt_per_split, n_splits, c->attn_part,
                   c->attn_ml, c->attn_cnt, c->dbg_sel == 1 ? c->dbg_buf : nullptr));
  CB_LAUNCHED(c);
  return CB_OK;
}

cb_status attention_tc5_init() {
  if (g_encode5 == nullptr) {
    cudaDriverEntryPointQueryResult qr;
    void* fn = nullptr;
    CB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr));
    CB_REQUIRE(qr == cudaDriverEntryPointSuccess && fn != nullptr, CB_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    g_encode5 = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  if (g_kvmaps == nullptr) g_kvmaps = new std::unordered_map<KvKey, CUtensorMap, KvKeyHash>();
  CB_CUDA(cudaFuncSetAttribute(attn_tc5_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  return CB_OK;
}
