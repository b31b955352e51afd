// gemm_tc2.cu — CTA-pair (cta_group::2) tcgen05 GEMM: one 256 x BN tile per 2-SM cluster.
//
// Why: with one CTA per 128 x 256 tile the SM's shared memory must feed 12 KB of A/B operands per
// 128-cycle MMA plus 48 KB of TMA writes per k-block — about 1.5x the ~128 B/clk it delivers, which
// caps the tensor pipe near 65 % (ncu: tensor pipe active 60-66 %, profiles/r01_gemm_ncu_full.txt).
// A CTA pair computes M = 256 with each SM holding its own 128 A rows and half of the B rows, so each
// SM moves half the B bytes per FLOP: ~64 B/clk of MMA reads + ~64 B/clk of TMA writes.
//
// Roles per CTA (6 warps): warp 0 TMA producer (both CTAs load their halves; the transaction bytes
// complete on the leader's barrier), warp 1 MMA issuer (leader CTA only: tcgen05.mma.cta_group::2,
// commits multicast to both CTAs' barriers), warps 2-5 epilogue on the CTA's own 128 accumulator
// rows (arrivals on the leader's TMEM-empty barrier). Same fused epilogues as gemm_tc.cu.
#include <cudaTypedefs.h>

#include "ctx.h"
#include "gemm_epi.cuh"
#include "tc_common.cuh"

namespace {
constexpr int BK = 64, NUM_THREADS = 192;
constexpr int A_BYTES = 128 * BK * 2;  // this CTA's 128 A rows

template <int BN> struct Cfg2 {
  static constexpr int B_HALF = BN / 2;
  static constexpr int B_BYTES = B_HALF * BK * 2;  // this CTA's half of B
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (200 * 1024) / STAGE_BYTES > 8 ? 8 : (200 * 1024) / STAGE_BYTES;
  static constexpr int EPI_BYTES = 4 * gepi::EPI_WARP_F4 * 16;  // epilogue staging, 4 KB per warp
  static constexpr int SMEM = STAGES * STAGE_BYTES + EPI_BYTES + 1024 + 256;
  static constexpr int ACC_STRIDE = (BN == 192 || BN == 224) ? 256 : BN;  // accumulator buffer stride (TMEM columns)
  static constexpr int TMEM_COLS = 2 * ACC_STRIDE;           // power of two for tcgen05.alloc
};

// Work item i -> tile t and k-block range [kb0, kb1).
//   tail_p <= 1: i = sp * tiles + t, K split into ksplit chain pieces (RESID only; 1 = whole tiles)
//   tail_p  > 1: the first tiles - tail_r tiles whole (full rounds of pairs); each of the last tail_r
//                tiles cut into tail_p K pieces (piece >= 0) that fill the last round, merged by the
//                last piece to finish (fixed piece order) before the tile's epilogue.
struct WorkItem {
  int t, sp, kb0, kb1, piece;
  int mt, nt;  // row tile and column tile (mc: may lie past the last tile -> no epilogue)
};
__device__ __forceinline__ WorkItem work_item(int i, int tiles, int num_kb, int ksplit, int tail_r, int tail_p) {
  WorkItem w;
  w.piece = -1;
  if (tail_p > 1) {
    const int full = tiles - tail_r;
    w.sp = 0;
    if (i < full) {
      w.t = i; w.kb0 = 0; w.kb1 = num_kb;
    } else {
      const int j = i - full;
      w.t = full + j / tail_p;
      w.piece = j % tail_p;
      w.kb0 = w.piece * num_kb / tail_p;
      w.kb1 = (w.piece + 1) * num_kb / tail_p;
    }
  } else {
    w.t = i % tiles; w.sp = i / tiles;
    w.kb0 = w.sp * num_kb / ksplit; w.kb1 = (w.sp + 1) * num_kb / ksplit;
  }
  w.mt = -1; w.nt = -1;  // set by the caller from t
  return w;
}

__device__ __forceinline__ void named_bar_sync2(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <int KIND, int BN>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int K,
                    int m_tiles, int n_tiles, EpiParams e, int ksplit, int* __restrict__ kflags,
                    int tail_r, int tail_p, float* __restrict__ tscr, int* __restrict__ tcnt,
                    long long* __restrict__ dbg, long long* __restrict__ strace, int mc) {
  // debug_trace: globaltimer (ns) events of each CTA's first work item at dbg[blockIdx.x * 8 + event]
#define DBG2(ev) do { if (dbg != nullptr && blockIdx.x < 256) dbg[blockIdx.x * 8 + (ev)] = tc::globaltimer(); } while (0)
  // stage trace (debug_trace 300, pair 0 only, first 256 k-blocks): strace[rank * 256 + kb] = producer's empty
  // wait done, strace[512 + kb] = MMA warp's full wait done (leader)
  const bool st_on = strace != nullptr && (blockIdx.x >> 1) == 0;
  using C = Cfg2<BN>;
  constexpr bool SW = (KIND == EPI_SWIGLU);
  constexpr int OUT_N = SW ? BN / 2 : BN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float4* ebuf = reinterpret_cast<float4*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES + C::EPI_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);  // tail merge: "this CTA merges" broadcast

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // mc: 4-CTA clusters of two CTA pairs on the same row tile and neighbouring column tiles (2q, 2q + 1);
  // the pairs share their A rows, each A half-box multicast from one CTA of each pair to both (halving the
  // L2 reads of A, which every column tile re-reads). Whole tiles only (no k-split or tail pieces).
  const uint32_t crank = tc::cluster_ctarank();
  const uint32_t rank = crank & 1;  // rank within the CTA pair
  const bool leader = rank == 0;
  const int num_kb = (K + BK - 1) / BK;
  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
  // mc == 2: 8-CTA clusters of four pairs (2 row tiles x 2 column tiles); in addition each B quarter-box is
  // loaded by one CTA and multicast to the CTA of the other row tile that holds the same B half.
  const int csh = mc == 2 ? 3 : 2;
  const int unit = mc ? (int)(blockIdx.x >> csh) : pair;  // scheduling unit: the cluster (mc) or the pair
  const int n_units = mc ? (int)(gridDim.x >> csh) : n_pairs;
  const int pic = (blockIdx.x >> 1) & 1;  // pair within the 4-CTA cluster (mc 1)
  const int pq = (blockIdx.x >> 1) & 3;   // pair within the 8-CTA cluster (mc 2)
  const int tiles = m_tiles * n_tiles;
  const int items = mc == 2 ? ((m_tiles + 1) / 2) * ((n_tiles + 1) / 2)
                    : mc ? m_tiles * ((n_tiles + 1) / 2)
                         : tail_p > 1 ? tiles - tail_r + tail_r * tail_p : tiles * ksplit;  // see work_item()
  const auto item = [&](int i) -> WorkItem {
    if (!mc) {
      WorkItem w = work_item(i, tiles, num_kb, ksplit, tail_r, tail_p);
      w.mt = w.t % m_tiles; w.nt = w.t / m_tiles;
      return w;
    }
    WorkItem w;
    w.sp = 0; w.kb0 = 0; w.kb1 = num_kb; w.piece = -1;
    if (mc == 2) {  // 8-CTA cluster: pairs (row tile 2a + bit 1 of pq, column tile 2b + bit 0 of pq)
      const int mt2 = (m_tiles + 1) / 2;
      w.mt = 2 * (i % mt2) + (pq >> 1);
      w.nt = 2 * (i / mt2) + (pq & 1);
    } else {  // 4-CTA cluster: same row tile, column tiles 2b, 2b + 1
      w.mt = i % m_tiles;
      w.nt = 2 * (i / m_tiles) + pic;
    }
    w.t = w.mt + m_tiles * w.nt;  // unused in mc mode (no k-split flags, no tail pieces)
    return w;
  };

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tmA);
    tc::tma_prefetch(&tmB);
    for (int s = 0; s < C::STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], mc == 2 ? 4 : mc ? 2 : 1);
    }
    for (int s = 0; s < 2; ++s) { tc::mbar_init(&tfull[s], 1); tc::mbar_init(&tempty[s], 8); }
    tc::fence_barrier_init();
  }
  if (warp == 2) tc::tmem_alloc_2sm(tmem_slot, C::TMEM_COLS);
  tc::fence_before();
  tc::cluster_sync();  // barriers of both CTAs initialised before any remote arrive / transaction
  tc::fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_enter();  // prologue above overlapped the previous kernel; its outputs are visible from here
  if (threadIdx.x == 0) DBG2(0);

  if (warp == 0) {
    // ===== TMA producer (both CTAs) =====
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const int half = (int)((crank >> 1) & 1);  // mc: the 64-row half of the shared A box this CTA loads
      const uint16_t amask = (uint16_t)((1u << crank) | (1u << (crank ^ 2u)));
      const int bq = (int)((crank >> 2) & 1);     // mc 2: the quarter of this pair's B half this CTA loads
      const uint16_t bmask = (uint16_t)((1u << crank) | (1u << (crank ^ 4u)));
      for (int i = unit; i < items; i += n_units) {
        const WorkItem w = item(i);
        const int m0 = w.mt * 256 + (int)rank * 128, nb = w.nt;
        const int b_row = SW ? (rank == 0 ? nb * OUT_N : e.ff + nb * OUT_N) : nb * BN + (int)rank * C::B_HALF;
        for (int kb = w.kb0; kb < w.kb1; ++kb) {
          uint8_t* sa = smem + stage * C::STAGE_BYTES;
          if (mc) {  // both pairs freed the stage (empty counts two commits), then half of A for both pairs
            tc::mbar_wait(&empty[stage], phase ^ 1);
            if (st_on && i == unit && kb < 256) strace[rank * 256 + kb] = clock64();
            if (leader) tc::mbar_arrive_expect_tx(&full[stage], 2 * C::STAGE_BYTES);
            tc::tma_load_2d_2sm_mc(sa + half * (A_BYTES / 2), &tmA, &full[stage], kb * BK, m0 + half * 64, amask);
            if (mc == 2)
              tc::tma_load_2d_2sm_mc(sa + A_BYTES + bq * (C::B_BYTES / 2), &tmB, &full[stage], kb * BK,
                                     b_row + bq * (C::B_HALF / 2), bmask);
            else
              tc::tma_load_2d_2sm(sa + A_BYTES, &tmB, &full[stage], kb * BK, b_row);
          } else {
            tc::mbar_wait(&empty[stage], phase ^ 1);
            if (st_on && i == pair && kb < 256) strace[rank * 256 + kb] = clock64();
            if (leader) tc::mbar_arrive_expect_tx(&full[stage], 2 * C::STAGE_BYTES);
            tc::tma_load_2d_2sm(sa, &tmA, &full[stage], kb * BK, m0);
            tc::tma_load_2d_2sm(sa + A_BYTES, &tmB, &full[stage], kb * BK, b_row);
          }
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        if (i == unit) DBG2(1);
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer (leader CTA) =====
    if (leader) {
      constexpr uint32_t IDESC = tc::idesc_bf16(256, BN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int i = unit; i < items; i += n_units, ++it) {
        const WorkItem w = item(i);
        const int acc = it & 1;
        tc::mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        tc::fence_after();
        const uint32_t d_tmem = tmem_base + acc * C::ACC_STRIDE;
        const int kb0 = w.kb0, kb1 = w.kb1;
        for (int kb = kb0; kb < kb1; ++kb) {
          tc::mbar_wait(&full[stage], phase);
          tc::fence_after();
          if (st_on && it == 0 && kb < 256 && lane == 0) strace[512 + kb] = clock64();
          if (tc::elect_one()) {
            const uint8_t* sa = smem + stage * C::STAGE_BYTES;
            const uint64_t adesc = tc::sdesc_sw128(sa), bdesc = tc::sdesc_sw128(sa + A_BYTES);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              tc::mma_bf16_2sm(d_tmem, adesc + 2 * k, bdesc + 2 * k, IDESC, (kb > kb0 || k > 0) ? 1u : 0u);
            if (mc) {  // the stage is free for the producers once every pair of the cluster read it
              tc::mma_commit_2sm_mask(&empty[stage], mc == 2 ? 0xFF : 0xF);
              if (kb == kb1 - 1) tc::mma_commit_2sm_mask(&tfull[acc], (uint16_t)(3u << (crank & 6u)));
            } else {
              tc::mma_commit_2sm(&empty[stage]);
              if (kb == kb1 - 1) tc::mma_commit_2sm(&tfull[acc]);
            }
          }
          __syncwarp();
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        if (it == 0 && lane == 0) DBG2(2);
      }
    }
  } else {
    // ===== epilogue (warps 2..5, each CTA its own 128 rows) =====
    const int q = warp & 3;
    const int row = q * 32 + lane;
    int it = 0;
    for (int i = unit; i < items; i += n_units, ++it) {
      const WorkItem w = item(i);
      const int t = w.t, sp = w.sp;
      const int acc = it & 1;
      const int m0 = w.mt * 256 + (int)rank * 128, nb = w.nt;
      const bool col_ok = nb < n_tiles && w.mt < m_tiles;  // mc: a cluster's spare pair past the last tile
      // split-K chain (RESID only): split sp adds onto h_out after split sp - 1 of the same 32 rows
      // published it — a fixed order, so the sum is deterministic. flag = number of splits done.
      int* flag = kflags + ((size_t)t * 2 + rank) * 4 + q;
      if constexpr (KIND == EPI_QKV) gepi::qkv_prefetch(e, m0 + row, col_ok && m0 + row < M, nb * OUT_N, OUT_N);
      // fused RMSNorm consumer: the row factor is ready before the accumulator (1 if off)
      [[maybe_unused]] const float rs = gepi::row_rs(e, m0 + row, m0 + row < M);
      if constexpr (KIND == EPI_RESID) {
        if (sp == 0) gepi::resid_prefetch(e, m0 + row, col_ok && m0 + row < M, nb * OUT_N, OUT_N);
      }
      tc::mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc::fence_after();
      if (it == 0 && warp == 2 && lane == 0) DBG2(3);
      if constexpr (KIND == EPI_RESID) {
        if (sp > 0) {
          if (lane == 0) {
            int f;
            while (true) {
              asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(f) : "l"(flag) : "memory");
              if (f >= sp) break;
              __nanosleep(100);
            }
          }
          __syncwarp();
        }
      }
      if (it == 0 && warp == 2 && lane == 0) DBG2(4);
      const int m = m0 + row;
      const uint32_t trow = tmem_base + ((uint32_t)(q * 32) << 16) + acc * C::ACC_STRIDE;
      float dacc = 0.f;
      bool skip_epilogue = !col_ok;
      if (w.piece >= 0) {
        // tail piece: publish this K piece's fp32 partial (this CTA's 128 rows x BN); the last piece of
        // the tile to arrive sums all pieces in piece order into its TMEM accumulator, then runs the
        // tile's epilogue; the others are done
        const int tr = t - (tiles - tail_r);
        float* base = tscr + (size_t)((tr * tail_p) * 2 + rank) * 128 * BN;
        const size_t pstride = (size_t)2 * 128 * BN;  // next piece, same rank
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          float v[32];
          tc::tmem_ld32(trow + c, v);
          // layout [BN / 4 column groups][128 rows][4]: a warp's 32 rows of one group are 512 contiguous bytes
          float4* dst = reinterpret_cast<float4*>(base + w.piece * pstride) + (size_t)(c / 4) * 128 + row;
#pragma unroll
          for (int x = 0; x < 8; ++x) dst[x * 128] = make_float4(v[4 * x], v[4 * x + 1], v[4 * x + 2], v[4 * x + 3]);
        }
        const bool ptrace = dbg != nullptr && warp == 2 && lane == 0 && blockIdx.x < 128;
        if (ptrace) dbg[1024 + blockIdx.x * 8 + 0] = tc::globaltimer();
        __threadfence();
        named_bar_sync2(1, 128);
        if (ptrace) dbg[1024 + blockIdx.x * 8 + 1] = tc::globaltimer();
        if (warp == 2 && lane == 0) {
          int* cnt = tcnt + tr * 2 + rank;
          const int last = atomicAdd(cnt, 1) == tail_p - 1;
          if (last) *cnt = 0;  // reset for the next launch
          *last_flag = last;
        }
        named_bar_sync2(1, 128);
        skip_epilogue = *last_flag == 0;
        named_bar_sync2(1, 128);  // everyone read the flag before it can be rewritten
        if (ptrace) dbg[1024 + blockIdx.x * 8 + 2] = tc::globaltimer();
        if (!skip_epilogue) {
          __threadfence();
          gepi::merge_pieces_to_tmem<BN, 4>(base, pstride, tail_p, row, trow);
          if (ptrace) dbg[1024 + blockIdx.x * 8 + 3] = tc::globaltimer();
        }
      }
      if (!skip_epilogue) {
      if (KIND == EPI_QKV && e.hd % 64 == 0 && !gepi::staged_kind<KIND>()) {
        gepi::qkv_row<OUT_N>(e, m, m < M, nb * OUT_N, trow, rs);
      } else if (KIND == EPI_RESID && gepi::resid_lean_ok(e, M)) {
        long long* tdbg = (dbg != nullptr && it == 0 && warp == 2 && blockIdx.x < 128) ? dbg + 1024 + blockIdx.x * 8 : nullptr;
        float4* wb = ebuf + (warp - 2) * gepi::EPI_WARP_F4;
        // the fused RMSNorm producer runs on the last piece of a k-split chain only (the finished sum)
        if (e.norm_gain != nullptr && sp == ksplit - 1)
          gepi::resid_lean<BN, true>(e, M, m0 + q * 32, nb * OUT_N, trow, wb, lane, tdbg, sp > 0);
        else
          gepi::resid_lean<BN, false>(e, M, m0 + q * 32, nb * OUT_N, trow, wb, lane, tdbg, sp > 0);
      } else if (gepi::staged_kind<KIND>() && (KIND != EPI_QKV || e.hd % 32 == 0)) {  // staged, row-contiguous
        gepi::tile_epilogue<KIND, BN>(e, M, m0 + q * 32, nb * OUT_N, trow, ebuf + (warp - 2) * gepi::EPI_WARP_F4, lane,
                                      sp > 0, sp == ksplit - 1,
                                      (dbg != nullptr && it == 0 && warp == 2 && blockIdx.x < 128)
                                          ? dbg + 1024 + blockIdx.x * 8 : nullptr);
      } else {
#pragma unroll 1
      for (int c = 0; c < OUT_N; c += 16) {
        float v[16], u[16];
        tc::tmem_ld16(trow + c, v);
        if constexpr (SW) tc::tmem_ld16(trow + BN / 2 + c, u);
#pragma unroll
        for (int i = 0; i < 16; ++i) { v[i] *= rs; u[i] *= rs; }
        const int n = nb * OUT_N + c;
        if (m < M && n < e.N) {
          const float d = gepi::epi16<KIND>(e, m, n, v, u);
          if constexpr (KIND == EPI_QKV) {
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
      }
      }
      if constexpr (KIND == EPI_RESID) {
        if (ksplit > 1) {
          __threadfence();
          __syncwarp();
          if (lane == 0) {  // publish (or, after the last split, reset for the next launch)
            const int nf = sp + 1 < ksplit ? sp + 1 : 0;
            asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(flag), "r"(nf) : "memory");
          }
        }
      }
      if (it == 0 && warp == 2 && lane == 0) DBG2(5);
      if (w.piece >= 0 && dbg != nullptr && warp == 2 && lane == 0 && blockIdx.x < 128)
        dbg[1024 + blockIdx.x * 8 + 4] = tc::globaltimer();
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive_rank0(&tempty[acc]);
    }
  }
  if (e.push_base[0] != nullptr) __threadfence_system();  // pushed rows reach the peers before the signal
  if (threadIdx.x == 0) DBG2(6);
  tc::fence_before();
  tc::cluster_sync();  // no multicast commit or remote arrive may target an exited CTA
  if (warp == 2) tc::tmem_dealloc_2sm(tmem_base, C::TMEM_COLS);
  if (threadIdx.x == 0) DBG2(7);
#undef DBG2
}

}  // namespace

cb_status gemm_tmap(cb_ctx* c, const void* p, long long rows, long long k, long long ld, int box_rows,
                    CUtensorMap* out);  // gemm_tc.cu (shared tensor-map cache)

template <int KIND, int BN>
static cb_status launch2_kind(cb_ctx* c, const void* A, int lda, const void* B, int ldb, int M, int K,
                              const EpiParams& e, int n_pairs, int ksplit, int* kflags, int tail_r, int tail_p,
                              float* tscr, int* tcnt, int mc, cudaStream_t s) {
  using C = Cfg2<BN>;
  constexpr bool sw = KIND == EPI_SWIGLU;
  constexpr int out_n = sw ? BN / 2 : BN;
  const long long b_rows = sw ? 2LL * e.ff : (long long)e.N;
  EpiParams ee = e;
  ee.l1pf = c->epi_l1pf;
  CUtensorMap ta, tb;
  CB_TRY(gemm_tmap(c, A, M, K, lda, mc ? 64 : 128, &ta));  // mc: each CTA loads (and multicasts) half of A
  CB_TRY(gemm_tmap(c, B, b_rows, K, ldb, mc == 2 ? C::B_HALF / 2 : C::B_HALF, &tb));  // mc 2: B quarter-boxes
  const int m_tiles = (M + 255) / 256, n_tiles = (e.N + out_n - 1) / out_n;
  CB_CUDA(launch_k(c, gemm_tc2_kernel<KIND, BN>, dim3(2 * n_pairs), dim3(NUM_THREADS), C::SMEM, s,
                    mc == 2 ? 8 : mc ? 4 : 2, ta, tb,
                    M, K, m_tiles, n_tiles, ee, ksplit, kflags, tail_r, tail_p, tscr, tcnt,
                    (c->dbg_sel == 1 || c->dbg_sel == 100 + KIND) ? c->dbg_buf : nullptr,
                    c->dbg_sel == 300 ? c->dbg_buf : nullptr, mc));
  CB_LAUNCHED(c);
  return CB_OK;
}

// Pair tiles of 256 x BN; n_pairs CTA pairs (grid = 2 * n_pairs).
cb_status launch_gemm_tc2(cb_ctx* c, const void* A, int lda, const void* B, int ldb, int M, int K, const EpiParams& e,
                          int bn, int n_pairs, int ksplit, int* kflags, int tail_r, int tail_p, float* tscr,
                          int* tcnt, int mc, cudaStream_t s) {
  ProfScope ps_(c, PROF_GEMM, s);
  // k-split chains continue from the running sum in local h_out; a peer-memory push (fused reduce-scatter)
  // sends each piece's rows to their owner instead, so pushed GEMMs always run whole tiles
  if (e.kind != EPI_RESID || e.push_base[0] != nullptr) ksplit = 1;
  if (ksplit > 1) tail_p = 1;
  // mc (plan_gemm): A-multicast clusters of two pairs, whole tiles only; n_pairs = 2 x the cluster count
  if (ksplit > 1 || tail_p > 1 || e.push_base[0] != nullptr) mc = 0;
  if (mc == 2) CB_REQUIRE(e.kind != EPI_SWIGLU, CB_E_INVALID_ARG, "8-CTA multicast clusters exclude the SwiGLU GEMM");
  if (bn == 224) {  // SwiGLU only: 112 gate + 112 up columns (14336 = 128 x 112 features, Mistral d_ff)
    CB_REQUIRE(e.kind == EPI_SWIGLU, CB_E_INVALID_ARG, "224-wide pair tiles are for the SwiGLU GEMM only");
    return launch2_kind<EPI_SWIGLU, 224>(c, A, lda, B, ldb, M, K, e, n_pairs, 1, kflags, tail_r, tail_p, tscr, tcnt,
                                         mc, s);
  }
#define L2_(KIND_)                                                                                      \
  return bn == 256                                                                                      \
             ? launch2_kind<KIND_, 256>(c, A, lda, B, ldb, M, K, e, n_pairs, ksplit, kflags, tail_r, tail_p, tscr, \
                                        tcnt, mc, s)                                                             \
         : bn == 192                                                                                         \
             ? launch2_kind<KIND_, 192>(c, A, lda, B, ldb, M, K, e, n_pairs, ksplit, kflags, tail_r, tail_p, tscr, \
                                        tcnt, mc, s)                                                             \
             : launch2_kind<KIND_, 128>(c, A, lda, B, ldb, M, K, e, n_pairs, ksplit, kflags, tail_r, tail_p, tscr, \
                                        tcnt, mc, s)
  switch (e.kind) {
    case EPI_STORE: L2_(EPI_STORE);
    case EPI_STORE_F32: L2_(EPI_STORE_F32);
    case EPI_QKV: L2_(EPI_QKV);
    case EPI_RESID: L2_(EPI_RESID);
    case EPI_SWIGLU: L2_(EPI_SWIGLU);
  }
#undef L2_
  cb_set_error("bad epilogue kind %d", e.kind);
  return CB_E_INVALID_ARG;
}

template <int BN> static cb_status set_attrs2() {
  using C = Cfg2<BN>;
  CB_CUDA(cudaFuncSetAttribute(gemm_tc2_kernel<EPI_STORE, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  CB_CUDA(cudaFuncSetAttribute(gemm_tc2_kernel<EPI_STORE_F32, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               C::SMEM));
  CB_CUDA(cudaFuncSetAttribute(gemm_tc2_kernel<EPI_QKV, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  CB_CUDA(cudaFuncSetAttribute(gemm_tc2_kernel<EPI_RESID, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  CB_CUDA(cudaFuncSetAttribute(gemm_tc2_kernel<EPI_SWIGLU, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  return CB_OK;
}

// How many 2-CTA clusters of the kernel can be co-resident (GPC boundaries can leave fewer than SMs / 2).
template <int BN, int KIND = EPI_RESID> static cb_status max_pairs2(int num_sms, int* out, int csize = 2) {
  using C = Cfg2<BN>;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(num_sms / csize * csize);  // a whole number of clusters
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = csize; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  CB_CUDA(cudaOccupancyMaxActiveClusters(&n, gemm_tc2_kernel<KIND, BN>, &cfg));
  *out = n;
  return CB_OK;
}

cb_status gemm_tc2_init(int num_sms, int* max_pairs, int* max_clusters4, int* max_clusters8) {
  CB_TRY(set_attrs2<256>());
  CB_TRY(set_attrs2<192>());
  CB_TRY(set_attrs2<128>());
  CB_CUDA(cudaFuncSetAttribute(gemm_tc2_kernel<EPI_SWIGLU, 224>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               Cfg2<224>::SMEM));
  int a = 0, b = 0, c3 = 0, c4 = 0;
  CB_TRY(max_pairs2<256>(num_sms, &a));
  CB_TRY(max_pairs2<128>(num_sms, &b));
  CB_TRY(max_pairs2<192>(num_sms, &c3));
  CB_TRY((max_pairs2<224, EPI_SWIGLU>(num_sms, &c4)));
  *max_pairs = a < b ? a : b;
  if (c3 < *max_pairs) *max_pairs = c3;
  if (c4 < *max_pairs) *max_pairs = c4;
  CB_REQUIRE(*max_pairs >= 1, CB_E_CUDA, "no CTA pair of the tcgen05 GEMM fits on this device");
  int d4[4] = {0, 0, 0, 0};
  CB_TRY(max_pairs2<256>(num_sms, &d4[0], 4));
  CB_TRY(max_pairs2<128>(num_sms, &d4[1], 4));
  CB_TRY(max_pairs2<192>(num_sms, &d4[2], 4));
  CB_TRY((max_pairs2<224, EPI_SWIGLU>(num_sms, &d4[3], 4)));
  *max_clusters4 = d4[0];
  for (int i = 1; i < 4; ++i) if (d4[i] < *max_clusters4) *max_clusters4 = d4[i];
  int d8[3] = {0, 0, 0};  // no SwiGLU in 8-CTA clusters
  CB_TRY(max_pairs2<256>(num_sms, &d8[0], 8));
  CB_TRY(max_pairs2<128>(num_sms, &d8[1], 8));
  CB_TRY(max_pairs2<192>(num_sms, &d8[2], 8));
  *max_clusters8 = d8[0];
  for (int i = 1; i < 3; ++i) if (d8[i] < *max_clusters8) *max_clusters8 = d8[i];
  return CB_OK;
}
