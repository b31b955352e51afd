// gemm_tc.cu — tcgen05 / TMEM / TMA GEMM for the bf16 blend projections (steps a2, a3, a7, a8).
//
//   acc[M][N] = A[M][K] . B[N][K]^T     A = activation rows (K-major), B = weight rows (K-major)
//
// Persistent warp-specialised kernel, one CTA per SM:
//   warp 0      TMA producer: 128x64 A box + BNx64 B box (SwiGLU: two BN/2-row boxes, the gate rows and
//               the matching up rows) per stage into a SWIZZLE_128B ring (4 stages at BN=256, 6 at 128)
//   warp 1      MMA issuer: one elected thread issues tcgen05.mma (M=128, N=BN, K=16) x 4 per stage,
//               fp32 accumulator in TMEM, double-buffered (2 x BN columns)
//   warps 2-5   epilogue: tcgen05.ld 32x32b -> registers -> fused epilogue (RoPE / residual gather /
//               SwiGLU / store) -> global, overlapping the next tile's MMAs
//
// The blend's GEMMs have M = 370..3072 rows, so the schedule is chosen per launch by a small cost
// model (host): whole-tile data-parallel rounds at BN = 256 or 128 (the narrower tile doubles the
// tile count of the N = 4096 projections, which otherwise fill only 48-80 of 148 SMs), or a
// data-parallel + stream-K hybrid where the tail's (tile, k-block) iterations are split evenly over
// the CTAs: a CTA ending mid-tile stores its fp32 partial in its own slot and raises a flag; the CTA
// owning the tile's last k-block adds the partials in fixed CTA order, so results are deterministic.
// Tiles are walked m-fastest, so CTAs running concurrently share weight tiles in L2.
#include <cudaTypedefs.h>

#include <unordered_map>

#include "ctx.h"
#include "tc_common.cuh"
#include "gemm_epi.cuh"

namespace {
constexpr int BM = 128, BK = 64, NUM_THREADS = 192;
constexpr int A_BYTES = BM * BK * 2;
constexpr int MAX_CONTRIB = 16;
constexpr int MAX_SPLIT = 4;   // stream-K pieces per tile (bounds the fixup fan-in)
constexpr int MIN_KB = 8;      // minimum k-blocks per stream-K CTA
constexpr int SLOT_COLS = 256; // partial slot row pitch (floats)

template <int BN> struct Cfg {
  static constexpr int STAGES = BN == 256 ? 4 : 6;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int EPI_BYTES = 4 * gepi::EPI_WARP_F4 * 16;  // epilogue staging, 4 KB per warp
  static constexpr int SMEM = STAGES * STAGE_BYTES + EPI_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr int TMEM_COLS = 2 * BN;
};

// Data-parallel rounds followed by an optional stream-K tail; every role walks the identical sequence.
struct Sched {
  int tiles, num_kb, G, b, dp_rounds, r, sk_ctas;
  long long sk_base, sk_iters, it, it_end;
  // sk_ctas_ = 0: whole tiles only (ceil(tiles/G) rounds). sk_ctas_ > 0: floor(tiles/G) whole-tile
  // rounds, then the remaining tiles' k-blocks split evenly over the first sk_ctas_ CTAs.
  __device__ void init(int tiles_, int num_kb_, int sk_ctas_) {
    tiles = tiles_; num_kb = num_kb_; G = gridDim.x; b = blockIdx.x; r = 0; sk_ctas = sk_ctas_;
    if (sk_ctas <= 0) {
      dp_rounds = (tiles + G - 1) / G;
      sk_base = sk_iters = it = it_end = 0;
      sk_ctas = 1;
      return;
    }
    dp_rounds = tiles / G;
    sk_base = (long long)dp_rounds * G * num_kb;
    sk_iters = (long long)tiles * num_kb - sk_base;
    it = it_end = 0;
    if (b < sk_ctas) {
      it = sk_base + sk_start(b);
      it_end = sk_base + sk_start(b + 1);
    }
  }
  __device__ long long sk_start(int cta) const { return (long long)cta * sk_iters / sk_ctas; }
  // Next segment: tile and k-block range [kb0, kb1). Whole-tile rounds first (concurrent CTAs share
  // weight tiles in L2), then the stream-K tail walked backwards, so a CTA's only non-final piece
  // (the head of its last tile) is computed and published first; its final pieces then wait only
  // on partials other CTAs also publish first (no dependency chains).
  __device__ bool next(int& tile, int& kb0, int& kb1) {
    if (r < dp_rounds) {
      tile = r * G + b;
      ++r;
      if (tile < tiles) { kb0 = 0; kb1 = num_kb; return true; }
      r = dp_rounds;
    }
    if (it < it_end) {
      const long long last = it_end - 1;
      tile = (int)(last / num_kb);
      const long long tstart = (long long)tile * num_kb;
      const long long s = it > tstart ? it : tstart;
      kb0 = (int)(s - tstart);
      kb1 = (int)(last - tstart) + 1;
      it_end = s;
      return true;
    }
    return false;
  }
  // CTAs holding the earlier (non-final) pieces of `tile`, ascending; returns the count.
  __device__ int contributors(int tile, int* out) const {
    const long long t0 = (long long)tile * num_kb;
    int n = 0;
    for (int cb = b - 1; cb >= 0 && n < MAX_CONTRIB; --cb) {
      out[n++] = cb;
      if (sk_base + sk_start(cb) <= t0) break;
    }
    for (int i = 0; i < n / 2; ++i) { const int t = out[i]; out[i] = out[n - 1 - i]; out[n - 1 - i] = t; }
    return n;
  }
};

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <int KIND, int BN>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int K,
                   int m_tiles, int n_tiles, EpiParams e, float* __restrict__ part, int* __restrict__ flags,
                   int sk_ctas) {
  using C = Cfg<BN>;
  constexpr bool SW = (KIND == EPI_SWIGLU);
  constexpr int OUT_N = SW ? BN / 2 : BN;  // output columns per tile
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float4* ebuf = reinterpret_cast<float4*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES + C::EPI_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_kb = (K + BK - 1) / BK;
  Sched sch;
  sch.init(m_tiles * n_tiles, num_kb, sk_ctas);

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tmA);
    tc::tma_prefetch(&tmB);
    for (int s = 0; s < C::STAGES; ++s) { tc::mbar_init(&full[s], 1); tc::mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { tc::mbar_init(&tfull[s], 1); tc::mbar_init(&tempty[s], 4); }
    tc::fence_barrier_init();
  }
  if (warp == 2) tc::tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_enter();  // prologue above overlapped the previous kernel; its outputs are visible from here
  int tile, kb0, kb1;

  if (warp == 0) {
    // ===== TMA producer =====
    if (tc::elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      while (sch.next(tile, kb0, kb1)) {
        const int m0 = (tile % m_tiles) * BM, nb = tile / m_tiles;
        for (int kb = kb0; kb < kb1; ++kb) {
          tc::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * C::STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          tc::mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
          tc::tma_load_2d(sa, &tmA, &full[stage], kb * BK, m0);
          if constexpr (SW) {
            tc::tma_load_2d(sb, &tmB, &full[stage], kb * BK, nb * OUT_N);
            tc::tma_load_2d(sb + C::B_BYTES / 2, &tmB, &full[stage], kb * BK, e.ff + nb * OUT_N);
          } else {
            tc::tma_load_2d(sb, &tmB, &full[stage], kb * BK, nb * BN);
          }
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer =====
    constexpr uint32_t IDESC = tc::idesc_bf16(BM, BN);
    int stage = 0;
    uint32_t phase = 0;
    for (int it = 0; sch.next(tile, kb0, kb1); ++it) {
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      tc::mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc::fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = kb0; kb < kb1; ++kb) {
        tc::mbar_wait(&full[stage], phase);
        tc::fence_after();
        if (tc::elect_one()) {
          const uint8_t* sa = smem + stage * C::STAGE_BYTES;
          const uint64_t adesc = tc::sdesc_sw128(sa), bdesc = tc::sdesc_sw128(sa + A_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)  // advance 16 bf16 = 32 B (>> 4 = 2) inside the swizzle atom
            tc::mma_bf16(d_tmem, adesc + 2 * k, bdesc + 2 * k, IDESC, (kb > kb0 || k > 0) ? 1u : 0u);
          tc::mma_commit(&empty[stage]);
          if (kb == kb1 - 1) tc::mma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else {
    // ===== epilogue (warps 2..5; warp w reads TMEM lanes 32*(w%4) .. +31) =====
    const int q = warp & 3;
    const int row = q * 32 + lane;    // row within the tile
    const int et = threadIdx.x - 64;  // 0..127 among epilogue threads
    int contrib[MAX_CONTRIB];
    for (int it = 0; sch.next(tile, kb0, kb1); ++it) {
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const int m0 = (tile % m_tiles) * BM, nb = tile / m_tiles;
      const bool final_piece = (kb1 == num_kb);
      const int n_con = (final_piece && kb0 > 0) ? sch.contributors(tile, contrib) : 0;
      float dacc = 0.f;  // fused deviation: running squared distance of the current k/v head
      [[maybe_unused]] const float rs = gepi::row_rs(e, m0 + row, m0 + row < M);  // fused RMSNorm consumer
      if constexpr (KIND == EPI_QKV) gepi::qkv_prefetch(e, m0 + row, m0 + row < M, nb * OUT_N, OUT_N);
      if constexpr (KIND == EPI_RESID) gepi::resid_prefetch(e, m0 + row, m0 + row < M, nb * OUT_N, OUT_N);
      tc::mbar_wait(&tfull[acc], acc_phase);
      tc::fence_after();
      const int m = m0 + row;
      const uint32_t trow = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
      if (!final_piece) {
        // non-final stream-K piece: fp32 partial -> this CTA's slot, then raise its flag
        float* slot = part + ((size_t)blockIdx.x * BM + row) * SLOT_COLS;
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          float v[32];
          tc::tmem_ld32(trow + c, v);
          float4* p = reinterpret_cast<float4*>(slot + c);
#pragma unroll
          for (int i = 0; i < 8; ++i) p[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        }
        tc::fence_before();
        __threadfence();
        named_bar(1, 128);
        if (et == 0) asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(flags + blockIdx.x), "r"(1) : "memory");
      } else {
        if (n_con > 0) {  // wait for the earlier pieces of this tile
          if (et < n_con) {
            int f = 0;
            do {
              asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(f) : "l"(flags + contrib[et]) : "memory");
            } while (f == 0);
          }
          named_bar(1, 128);
        }
        if (KIND == EPI_QKV && n_con == 0 && e.hd % 64 == 0 && !gepi::staged_kind<KIND>()) {
          gepi::qkv_row<OUT_N>(e, m, m < M, nb * OUT_N, trow, rs);
        } else if (KIND == EPI_RESID && n_con == 0 && gepi::resid_lean_ok(e, M)) {
          if (e.norm_gain != nullptr)
            gepi::resid_lean<BN, true>(e, M, m0 + q * 32, nb * OUT_N, trow, ebuf + (warp - 2) * gepi::EPI_WARP_F4, lane);
          else
            gepi::resid_lean<BN, false>(e, M, m0 + q * 32, nb * OUT_N, trow, ebuf + (warp - 2) * gepi::EPI_WARP_F4, lane);
        } else if (n_con == 0 && gepi::staged_kind<KIND>() && (KIND != EPI_QKV || e.hd % 32 == 0)) {
          gepi::tile_epilogue<KIND, BN>(e, M, m0 + q * 32, nb * OUT_N, trow, ebuf + (warp - 2) * gepi::EPI_WARP_F4,
                                        lane, false, true);
        } else
#pragma unroll 1
        for (int c = 0; c < OUT_N; c += 16) {
          float v[16], u[16];
          tc::tmem_ld16(trow + c, v);
          if constexpr (SW) tc::tmem_ld16(trow + BN / 2 + c, u);
          if (n_con > 0) {  // fixed order: partials of ascending CTAs, then this CTA's accumulator
            float sv[16], su[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) { sv[i] = 0.f; su[i] = 0.f; }
            for (int j0 = 0; j0 < n_con; j0 += 4) {
              float4 x[4][4], y[4][4];
#pragma unroll
              for (int jj = 0; jj < 4; ++jj) {  // issue every load of up to 4 contributors before adding
                if (j0 + jj < n_con) {
                  const float* slot = part + ((size_t)contrib[j0 + jj] * BM + row) * SLOT_COLS;
#pragma unroll
                  for (int i = 0; i < 4; ++i) x[jj][i] = __ldcg(reinterpret_cast<const float4*>(slot + c) + i);
                  if constexpr (SW) {
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                      y[jj][i] = __ldcg(reinterpret_cast<const float4*>(slot + BN / 2 + c) + i);
                  }
                }
              }
#pragma unroll
              for (int jj = 0; jj < 4; ++jj) {
                if (j0 + jj < n_con) {
#pragma unroll
                  for (int i = 0; i < 4; ++i) {
                    sv[4 * i] += x[jj][i].x; sv[4 * i + 1] += x[jj][i].y;
                    sv[4 * i + 2] += x[jj][i].z; sv[4 * i + 3] += x[jj][i].w;
                    if constexpr (SW) {
                      su[4 * i] += y[jj][i].x; su[4 * i + 1] += y[jj][i].y;
                      su[4 * i + 2] += y[jj][i].z; su[4 * i + 3] += y[jj][i].w;
                    }
                  }
                }
              }
            }
#pragma unroll
            for (int i = 0; i < 16; ++i) { v[i] = sv[i] + v[i]; u[i] = su[i] + u[i]; }
          }
#pragma unroll
          for (int i = 0; i < 16; ++i) { v[i] *= rs; u[i] *= rs; }
          const int n = nb * OUT_N + c;
          if (m < M && n < e.N) {
            const float d = gepi::epi16<KIND>(e, m, n, v, u);
            if constexpr (KIND == EPI_QKV) {
              // a k or v head ends at this chunk: publish its deviation partial (fixed in-thread order)
              dacc += d;
              const int cl = e.col0 + n;
              if (e.dev_part != nullptr && cl >= e.qd && (cl + 16) % 64 == 0) {  // 64-column k/v block ends
                const int kv_col = cl - e.qd;
                const int slot = kv_col < e.kvd ? 2 * (kv_col / 64) : 2 * ((kv_col - e.kvd) / 64) + 1;
                if (m < e.n_cand) e.dev_part[(size_t)slot * e.ld_part + m] = dacc;
                dacc = 0.f;
              }
            }
          }
        }
        if (n_con > 0) {  // release the contributors' slots for the next launch
          named_bar(1, 128);
          if (et < n_con) flags[contrib[et]] = 0;
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty[acc]);
    }
  }
  if (e.push_base[0] != nullptr) __threadfence_system();  // pushed rows reach the peers before the signal
  __syncthreads();
  if (warp == 2) tc::tmem_dealloc(tmem_base, C::TMEM_COLS);
}

// ---- host side --------------------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

struct TmKey {
  const void* p;
  long long rows, k, ld;
  int box_rows;
  bool operator==(const TmKey& o) const {
    return p == o.p && rows == o.rows && k == o.k && ld == o.ld && box_rows == o.box_rows;
  }
};
struct TmKeyHash {
  size_t operator()(const TmKey& k) const {
    size_t h = std::hash<const void*>()(k.p);
    h ^= std::hash<long long>()(k.rows * 1315423911LL + k.k * 2654435761LL + k.ld) + 0x9e3779b9 + (h << 6) + (h >> 2);
    return h ^ (size_t)k.box_rows;
  }
};

// Launch plan: CTA pair or single CTA, tile width, stream-K tail and grid, from a cost model in
// cycles per SM. Per-k-block costs are the floor divided by the measured tensor-pipe efficiency
// (single CTA 128x256: shared-memory bound at ~65 %; 128x128: ~57 % of its half-size floor;
// pair 256x256 / 256x128: ~90 % / ~65 %).
// Pair RESID GEMMs (o-proj, down-proj: N = d_model, few tiles at blend sizes) may also split K into a
// chain of ksplit pieces per tile, each adding onto h_out after the previous one (fixed order).
// Pair plans may also cut each remainder tile (tiles % pairs, when it is a small last round) into
// tail_p K pieces that fill that round; the last piece of a tile to finish merges (gemm_tc2.cu).
struct Plan {
  int bn, sk_ctas, grid, pair, ksplit, tail_r = 0, tail_p = 1, mc = 0;
  double cost = 0.0;  // model cycles per SM
};
constexpr int MAX_TAIL_P = 4;  // gemm_tc2.cu merges at most 4 pieces
constexpr double TAIL_MERGE_CYC = 6000.0;  // partial store + merge reads + TMEM rewrite

constexpr int MAX_KSPLIT = 4;
constexpr double MC4_FACTOR = 0.8;  // k-loop of A-multicast 4-CTA clusters vs pairs (tools/gemm_micro.py --mcs)
constexpr double MC8_FACTOR = 0.7;  // A+B multicast 8-CTA clusters
constexpr double KSPLIT_EPI_CYC = 3000.0;  // one more serialised fp32 read-modify-write epilogue

Plan plan_gemm(int num_sms, int max_pairs, int M, int N_out, bool sw, bool resid, int K, int force_sched, int force_bn, int force_pair,
               int force_ksplit, int force_tail, bool no192, int pairs_cap, bool balance, bool no224, int mc_mode = 0,
               int max_cl4 = 0, int max_cl8 = 0) {
  if (pairs_cap > 0 && pairs_cap < max_pairs) max_pairs = pairs_cap;
  const int num_kb = (K + BK - 1) / BK;
  Plan best{256, 0, 1, 0, 1};
  double best_cost = 1e300;
  for (int pair : {1, 0}) {
    if (force_pair == 1 && !pair) continue;   // 1: pairs only, 2: single CTAs only
    if (force_pair == 2 && pair) continue;
    if (pair && force_sched == 2) continue;   // the stream-K tail exists for single CTAs only
    const int tile_m = pair ? 256 : BM;
    const int m_tiles = (M + tile_m - 1) / tile_m;
    for (int bn : {256, 224, 192, 128}) {
      if (bn == 192 && (!pair || no192)) continue;  // 192-wide tiles exist for CTA pairs only
      // 224 = 112 gate + 112 up columns (SwiGLU pairs only): d_ff = 14336 is 128 x 112 features, so at
      // blend sizes (2 row tiles) 256 tiles fill 4 rounds of 64 pairs instead of 224 tiles needing a 4th
      // round of 2 at 256 wide
      if (bn == 224 && (!pair || !sw || no224)) continue;
      if (force_bn && bn != force_bn) continue;
      const int out_n = sw ? bn / 2 : bn;
      const long long tiles = (long long)m_tiles * ((N_out + out_n - 1) / out_n);
      const double cyc = pair ? (bn == 256 ? 570.0 : bn == 224 ? 525.0 : bn == 192 ? 480.0 : 390.0)
                              : (bn == 256 ? 790.0 : 450.0);
      const int units = pair ? max_pairs : num_sms;
      // (a) whole tiles only (pairs: optionally a k-split chain for RESID)
      if (force_sched != 2) {
        const auto fits = [&](int ks) { return ks == 1 || (tiles * ks <= units && num_kb / ks >= 4); };
        // k-split chains are opt-in (gemm_ksplit): measured slower at blend sizes, the second piece's
        // residual read-modify-write is serialised behind the first (tools/gemm_trace.py)
        for (int ks = 1; ks <= (pair && resid && force_ksplit > 1 ? MAX_KSPLIT : 1); ++ks) {
          if (!fits(ks)) continue;
          // forced: that split when it fits, else no split
          if (pair && resid && force_ksplit && ks != (fits(force_ksplit) ? force_ksplit : 1)) continue;
          int grid = (int)std::min<long long>(units, tiles * ks);
          // balanced rounds: the fewest pairs that still need the same number of rounds (the pair
          // mainloop is power-capped at full load, so a ragged last round costs more than spreading
          // the tiles evenly over fewer pairs; tools/gemm_cap.py)
          if (pair && balance) {
            const long long rounds = (tiles * ks + grid - 1) / grid;
            grid = (int)((tiles * ks + rounds - 1) / rounds);
          }
          const double cost =
              (double)((tiles * ks + grid - 1) / grid) * ((num_kb + ks - 1) / ks) * cyc + (ks - 1) * KSPLIT_EPI_CYC;
          if (cost < best_cost) { best_cost = cost; best = Plan{bn, 0, pair ? 2 * grid : grid, pair, ks}; }
          // A-multicast clusters of two pairs (gemm_mc): the pairs of a row tile share A, halving its L2 reads.
          // The single-wave small-M GEMMs are bound by chip-wide L2 reads (A is re-read by every column tile;
          // tools/gemm_stages.py: ~500 cycles per k-block whatever the tile width), so their k-loop shortens;
          // tiles of 224/256 columns are MMA-bound and gain nothing (tools/gemm_micro.py --mcs 0,1). Only
          // max_cl4 (33 on B200) 4-CTA clusters are co-resident, fewer than 74 / 2, so it pays when the
          // clusters' rounds are no more than the pairs' rounds. Not for the SwiGLU GEMM: its many-round
          // 224/192-wide tiles run at the power-capped tensor peak and were slower in clusters (125 -> 134 us).
          if (pair && ks == 1 && (mc_mode == 1 || mc_mode == 2) && max_cl4 > 0 &&
              ((bn <= 192 && !sw) || mc_mode == 1)) {
            const int n_t = (int)(tiles / m_tiles);
            const long long units = (long long)m_tiles * ((n_t + 1) / 2);
            const long long rounds = (units + max_cl4 - 1) / max_cl4;
            const double c_mc = (double)rounds * num_kb * cyc * (bn <= 192 ? MC4_FACTOR : 1.0);
            if (c_mc < best_cost || mc_mode == 1) {
              best_cost = c_mc;
              best = Plan{bn, 0, 2 * (int)(2 * ((units + rounds - 1) / rounds)), 1, 1};
              best.mc = 1;
            }
          }
          // 8-CTA clusters (2 row tiles x 2 column tiles): B quarter-boxes multicast across the row tiles too.
          // Opt-in (gemm_mc = 3): only 15 such clusters are co-resident (60 pairs), and on the blend shapes
          // they were neutral to slower than the 4-CTA clusters (o_proj 401 rows 21.6 vs 22.0 us, QKV 579 rows
          // 27.3 vs 28.4, QKV 401 rows 37.1 vs 23.2, down 579 rows 86.4 vs 65.4; profiles/r02_gemm_mc.txt).
          if (pair && ks == 1 && mc_mode == 3 && max_cl8 > 0 && !sw && m_tiles >= 2) {
            const int n_t = (int)(tiles / m_tiles);
            const long long units = (long long)((m_tiles + 1) / 2) * ((n_t + 1) / 2);
            const long long rounds = (units + max_cl8 - 1) / max_cl8;
            // a spare row tile (odd m_tiles) costs like a real one
            const double c_mc = (double)rounds * num_kb * cyc * MC8_FACTOR;
            if (c_mc < best_cost || mc_mode == 3) {
              best_cost = c_mc;
              best = Plan{bn, 0, 4 * (int)(2 * ((units + rounds - 1) / rounds)), 1, 1};
              best.mc = 2;
            }
          }
          if (pair && ks == 1 && force_tail != 1) {  // remainder tiles cut into K pieces
            const long long rounds = tiles / units, rem = tiles % units;
            if (rounds >= 1 && rem > 0) {
              const int tp = (int)std::min<long long>(MAX_TAIL_P, units / rem);
              if (tp > 1 && num_kb / tp >= 8) {
                const double c2 = (double)rounds * num_kb * cyc + (double)((num_kb + tp - 1) / tp) * cyc + TAIL_MERGE_CYC;
                if (c2 < best_cost || force_tail == 2) {
                  best_cost = c2;
                  best = Plan{bn, 0, 2 * units, 1, 1, (int)rem, tp};
                }
              }
            }
          }
        }
      }
      if (pair) continue;
    // (b) floor(tiles/G) whole-tile rounds + the remainder split over up to MAX_SPLIT CTAs per tile
    // The stream-K tail is opt-in (gemm_sched = 2): measured on B200 its fixup costs ~15-25 us per
    // launch at these sizes, more than the idle-SM time it recovers (tools/gemm_micro.py).
    if (force_sched == 2 && tiles % num_sms != 0) {
      const long long dp = tiles / num_sms, rem = tiles - dp * num_sms;
      const long long sk_iters = rem * num_kb;
      const int sk_ctas = (int)std::max<long long>(
          1, std::min<long long>(std::min<long long>(num_sms, rem * MAX_SPLIT), sk_iters / MIN_KB));
      const int grid = dp > 0 ? num_sms : sk_ctas;
      const double fixup = 6000.0;  // partial store + flag + partial reads, in MMA-cycle units
      const double cost = (double)dp * num_kb * cyc + (double)((sk_iters + sk_ctas - 1) / sk_ctas) * cyc + fixup;
      if (cost < best_cost) { best_cost = cost; best = Plan{bn, sk_ctas, grid, 0, 1}; }
    }
    }
  }
  best.cost = best_cost;
  return best;
}

}  // namespace

struct TmapCache {
  std::unordered_map<TmKey, CUtensorMap, TmKeyHash> maps;
  float* part = nullptr;  // [num_sms][BM][SLOT_COLS] fp32 stream-K partial slots
  int* flags = nullptr;   // [num_sms]
  int* kflags = nullptr;  // [KFLAGS] split-K chain counters of the pair kernel (zero between launches)
  int force_bn = 0;
  int max_pairs = 0;      // co-resident 2-CTA clusters of the pair kernel
  int force_tail = 1;     // 0 auto, 1 never cut remainder tiles (default: measured 0.2 ms/step slower), 2 always
  bool no192 = false;     // exclude 256 x 192 pair tiles from the plan
  bool no224 = false;     // exclude 256 x 224 SwiGLU pair tiles from the plan
  int pairs_cap[5] = {0, 0, 0, 0, 0};  // per epilogue kind: use at most this many CTA pairs (0: all)
  bool balance = true;    // spread pair tiles evenly over the rounds they need (plan_gemm)
  float* tscr = nullptr;  // [max_pairs][2][128][256] fp32 tail-piece partials
  int* tcnt = nullptr;    // [max_pairs][2] tail-piece arrival counters (zero between launches)
  int force_ksplit = 0;   // 0 auto, else force this k-split for pair RESID GEMMs (when it fits)
  int force_pair = 0;     // 0 auto, 1 CTA pairs only, 2 single CTAs only
};

cb_status launch_gemm_tc2(cb_ctx* c, const void* A, int lda, const void* B, int ldb, int M, int K, const EpiParams& e,
                          int bn, int n_pairs, int ksplit, int* kflags, int tail_r, int tail_p, float* tscr,
                          int* tcnt, int mc, cudaStream_t s);
cb_status gemm_tc2_init(int num_sms, int* max_pairs, int* max_clusters4, int* max_clusters8);
constexpr int KFLAGS = 4096;  // >= 8 per tile for every tile of a split-K launch (tiles * ksplit <= 74 pairs)

cb_status gemm_tmap(cb_ctx* c, const void* p, long long rows, long long k, long long ld, int box_rows,
                    CUtensorMap* out);
static cb_status get_tmap(cb_ctx* c, const void* p, long long rows, long long k, long long ld, int box_rows,
                          CUtensorMap* out) {
  return gemm_tmap(c, p, rows, k, ld, box_rows, out);
}

cb_status gemm_tmap(cb_ctx* c, const void* p, long long rows, long long k, long long ld, int box_rows,
                          CUtensorMap* out) {
  TmKey key{p, rows, k, ld, box_rows};
  auto it = c->tmaps->maps.find(key);
  if (it != c->tmaps->maps.end()) { *out = it->second; return CB_OK; }
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)k, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(p), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CB_REQUIRE(r == CUDA_SUCCESS, CB_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  if (c->tmaps->maps.size() > 4096) c->tmaps->maps.clear();
  c->tmaps->maps.emplace(key, m);
  *out = m;
  return CB_OK;
}

bool gemm_tc_ok(const cb_ctx* c, const void* A, int lda, const void* B, int ldb, int M, int K, const EpiParams& e) {
  if (c->m.dtype != CB_BF16 || g_encode == nullptr) return false;
  if (K % 8 != 0 || lda % 8 != 0 || ldb % 8 != 0 || e.N % 16 != 0) return false;
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) return false;
  if ((e.kind == EPI_STORE || e.kind == EPI_STORE_F32 || e.kind == EPI_RESID) && e.ldo % 8 != 0) return false;
  if (e.kind == EPI_QKV && (e.hd % 16 != 0 || e.col0 % 16 != 0 || e.qd % 16 != 0 || e.kvd % 16 != 0)) return false;
  if (e.kind == EPI_SWIGLU && e.ff % 8 != 0) return false;
  return M > 0;
}

template <int KIND, int BN>
static cb_status launch_kind(cb_ctx* c, const void* A, int lda, const void* B, int ldb, int M, int K,
                             const EpiParams& e, const Plan& pl, cudaStream_t s) {
  constexpr bool sw = KIND == EPI_SWIGLU;
  constexpr int out_n = sw ? BN / 2 : BN;
  const long long b_rows = sw ? 2LL * e.ff : (long long)e.N;
  CUtensorMap ta, tb;
  CB_TRY(get_tmap(c, A, M, K, lda, BM, &ta));
  CB_TRY(get_tmap(c, B, b_rows, K, ldb, sw ? BN / 2 : BN, &tb));
  const int m_tiles = (M + BM - 1) / BM, n_tiles = (e.N + out_n - 1) / out_n;
  CB_CUDA(launch_k(c, gemm_tc_kernel<KIND, BN>, dim3(pl.grid), dim3(NUM_THREADS), Cfg<BN>::SMEM, s, 1, ta, tb, M, K,
                    m_tiles, n_tiles, e, c->tmaps->part, c->tmaps->flags, pl.sk_ctas));
  CB_LAUNCHED(c);
  return CB_OK;
}

template <int BN>
static cb_status launch_bn(cb_ctx* c, const void* A, int lda, const void* B, int ldb, int M, int K, const EpiParams& e,
                           const Plan& pl, cudaStream_t s) {
  switch (e.kind) {
    case EPI_STORE: return launch_kind<EPI_STORE, BN>(c, A, lda, B, ldb, M, K, e, pl, s);
    case EPI_STORE_F32: return launch_kind<EPI_STORE_F32, BN>(c, A, lda, B, ldb, M, K, e, pl, s);
    case EPI_QKV: return launch_kind<EPI_QKV, BN>(c, A, lda, B, ldb, M, K, e, pl, s);
    case EPI_RESID: return launch_kind<EPI_RESID, BN>(c, A, lda, B, ldb, M, K, e, pl, s);
    case EPI_SWIGLU: return launch_kind<EPI_SWIGLU, BN>(c, A, lda, B, ldb, M, K, e, pl, s);
  }
  cb_set_error("bad epilogue kind %d", e.kind);
  return CB_E_INVALID_ARG;
}

cb_status launch_gemm_tc(cb_ctx* c, const void* A, int lda, const void* B, int ldb, int M, int K,
                         const EpiParams& e, cudaStream_t s) {
  // the stream-K fixup path has no fused-RMSNorm producer: plain data-parallel then
  const int sched = (e.norm_gain != nullptr && c->gemm_sched == 2) ? 1 : c->gemm_sched;
  const Plan pl = plan_gemm(c->num_sms, c->tmaps->max_pairs, M, e.N, e.kind == EPI_SWIGLU, e.kind == EPI_RESID, K, sched,
                            c->tmaps->force_bn, c->tmaps->force_pair, c->tmaps->force_ksplit,
                            c->tmaps->force_tail, c->tmaps->no192, c->tmaps->pairs_cap[e.kind],
                            c->tmaps->balance, c->tmaps->no224, e.push_base[0] != nullptr ? 0 : c->gemm_mc,
                            c->max_clusters4, c->max_clusters8);
  if (pl.pair)
    return launch_gemm_tc2(c, A, lda, B, ldb, M, K, e, pl.bn, pl.grid / 2, pl.ksplit, c->tmaps->kflags, pl.tail_r,
                           pl.tail_p, c->tmaps->tscr, c->tmaps->tcnt, pl.mc, s);
  ProfScope ps_(c, PROF_GEMM, s);
  if (pl.bn == 256) return launch_bn<256>(c, A, lda, B, ldb, M, K, e, pl, s);
  return launch_bn<128>(c, A, lda, B, ldb, M, K, e, pl, s);
}

void gemm_tc_force_bn(cb_ctx* c, int bn) { c->tmaps->force_bn = bn; }
void gemm_tc_force_pair(cb_ctx* c, int v) { c->tmaps->force_pair = v; }
void gemm_tc_force_ksplit(cb_ctx* c, int v) { c->tmaps->force_ksplit = v; }
void gemm_tc_force_tail(cb_ctx* c, int v) { c->tmaps->force_tail = v; }
void gemm_tc_no192(cb_ctx* c, int v) { c->tmaps->no192 = v != 0; }
void gemm_tc_no224(cb_ctx* c, int v) { c->tmaps->no224 = v != 0; }
void gemm_tc_pairs_cap(cb_ctx* c, int kind, int v) { c->tmaps->pairs_cap[kind] = v; }
void gemm_tc_balance(cb_ctx* c, int v) { c->tmaps->balance = v != 0; }
int gemm_tc_max_pairs(const cb_ctx* c) { return c->tmaps ? c->tmaps->max_pairs : 0; }

template <int BN> static cb_status set_attrs() {
  CB_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<EPI_STORE, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN>::SMEM));
  CB_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<EPI_STORE_F32, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               Cfg<BN>::SMEM));
  CB_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<EPI_QKV, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN>::SMEM));
  CB_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<EPI_RESID, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN>::SMEM));
  CB_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<EPI_SWIGLU, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               Cfg<BN>::SMEM));
  return CB_OK;
}

cb_status gemm_tc_init(cb_ctx* c) {
  if (g_encode == nullptr) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    CB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    CB_REQUIRE(q == cudaDriverEntryPointSuccess && fn != nullptr, CB_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  CB_TRY(set_attrs<256>());
  CB_TRY(set_attrs<128>());
  c->tmaps = new TmapCache();
  CB_TRY(gemm_tc2_init(c->num_sms, &c->tmaps->max_pairs, &c->max_clusters4, &c->max_clusters8));
  CB_CUDA(cudaMalloc(&c->tmaps->part, (size_t)c->num_sms * BM * SLOT_COLS * sizeof(float)));
  CB_CUDA(cudaMalloc(&c->tmaps->flags, (size_t)c->num_sms * sizeof(int)));
  CB_CUDA(cudaMemset(c->tmaps->flags, 0, (size_t)c->num_sms * sizeof(int)));
  CB_CUDA(cudaMalloc(&c->tmaps->kflags, KFLAGS * sizeof(int)));
  CB_CUDA(cudaMemset(c->tmaps->kflags, 0, KFLAGS * sizeof(int)));
  CB_CUDA(cudaMalloc(&c->tmaps->tscr, (size_t)c->tmaps->max_pairs * 2 * 128 * 256 * sizeof(float)));
  CB_CUDA(cudaMalloc(&c->tmaps->tcnt, (size_t)c->tmaps->max_pairs * 2 * sizeof(int)));
  CB_CUDA(cudaMemset(c->tmaps->tcnt, 0, (size_t)c->tmaps->max_pairs * 2 * sizeof(int)));
  return CB_OK;
}

void gemm_tc_destroy(cb_ctx* c) {
  if (c->tmaps) {
    cudaFree(c->tmaps->part);
    cudaFree(c->tmaps->flags);
    cudaFree(c->tmaps->kflags);
    cudaFree(c->tmaps->tscr);
    cudaFree(c->tmaps->tcnt);
  }
  delete c->tmaps;
  c->tmaps = nullptr;
}
