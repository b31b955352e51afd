// gemm_mlp.cu — the MLP of a blend layer (step a8) as ONE persistent CTA-pair tcgen05 kernel:
//
//   act = SwiGLU(x W_gate^T, x W_up^T)          (gate_up tiles, 256 rows x 128 features)
//   h  += act W_down^T   (+ next RMSNorm's y)   (down pieces, 256 rows x 256 columns x one K block)
//
// Why: at blend sizes (M = 370..550 rows) gate_up has 2 x 112 pair tiles for 74 CTA pairs, so its last
// round holds 2 tiles while 72 pairs idle, and the down projection (32 tiles of 224 k-blocks) cannot
// fill the chip on its own. Here both are one work list: gate_up tiles ordered by feature block, then
// the down projection cut along K into S blocks that match those feature blocks. Down piece
// (m-tile, n-tile, block s) only needs the activations of feature block s of its m-tile, so the pairs
// that finish their gate_up tiles start down pieces while the last gate_up tiles are still running.
//
// Cross-CTA protocol (all counters reset themselves, so the kernel can be replayed in a CUDA graph):
//  - a gate_up tile's epilogue stores its activations, fences, and bumps blk_cnt[s][m] (2 per pair);
//  - a down piece's TMA producer polls blk_cnt[s][m] (ld.acquire), then fence.proxy.async before its
//    TMA reads of the activations; the last of the block's consumers resets the counter;
//  - every down piece publishes an fp32 partial; the last of the S pieces of a tile to finish sums all
//    partials in block order into its TMEM accumulator (deterministic) and runs the residual epilogue
//    (h_out = h_in + sum, fused RMSNorm producer for the next layer).
// Deadlock-free: a pair walks its items in increasing order, down items (the only waiting ones) come
// after every gate_up item, gate_up items never wait, and all pairs are co-resident (grid = pairs).
#include <cudaTypedefs.h>

#include "ctx.h"
#include "gemm_epi.cuh"
#include "tc_common.cuh"

namespace {
constexpr int BK = 64, BN = 256, NUM_THREADS = 192;
constexpr int A_BYTES = 128 * BK * 2;
constexpr int B_BYTES = 128 * BK * 2;  // this CTA's half of the 256 B rows
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int STAGES = 6;
constexpr int EPI_BYTES = 4 * gepi::EPI_WARP_F4 * 16;
constexpr int SMEM = STAGES * STAGE_BYTES + EPI_BYTES + 1024 + 256;
constexpr int TMEM_COLS = 2 * BN;
constexpr int MAX_S = 4;

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

struct MlpItem {
  bool down;
  int s, mt, f, nt;  // feature block, m-tile, gate_up feature tile / down n-tile
};

struct MlpGeo {
  int m_tiles, n_ft, ft_blk, n_nt, S, G, D;
  __device__ MlpItem item(int i) const {
    MlpItem w;
    if (i < G) {  // gate_up: feature block s, then m-tile, then feature tile within the block
      w.down = false;
      w.s = i / (m_tiles * ft_blk);
      const int r = i - w.s * m_tiles * ft_blk;
      w.mt = r / ft_blk;
      w.f = w.s * ft_blk + (r - w.mt * ft_blk);
      w.nt = 0;
    } else {  // down: block s, then m-tile, then n-tile
      const int j = i - G;
      w.down = true;
      w.s = j / (m_tiles * n_nt);
      const int r = j - w.s * m_tiles * n_nt;
      w.mt = r / n_nt;
      w.nt = r - w.mt * n_nt;
      w.f = 0;
    }
    return w;
  }
};

__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_mlp_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmWgu,
                    const __grid_constant__ CUtensorMap tmAct, const __grid_constant__ CUtensorMap tmWd, int M, int d,
                    int ff, MlpGeo geo, EpiParams egu, EpiParams edn, int* __restrict__ blk_cnt,
                    int* __restrict__ blk_use, int* __restrict__ dn_cnt, float* __restrict__ dscr,
                    long long* __restrict__ dbg) {
  // debug_trace 200: per CTA (< 148) and item slot (< 6): [cta * 12 + 2 s] accumulator ready, [+1] done
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float4* ebuf = reinterpret_cast<float4*>(smem + STAGES * STAGE_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES + EPI_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = tc::cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
  const int items = geo.G + geo.D;
  const int kb_gu = d / BK, kb_dn = ff / BK / geo.S;

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tmX);
    tc::tma_prefetch(&tmWgu);
    tc::tma_prefetch(&tmAct);
    tc::tma_prefetch(&tmWd);
    for (int s = 0; s < STAGES; ++s) { tc::mbar_init(&full[s], 1); tc::mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { tc::mbar_init(&tfull[s], 1); tc::mbar_init(&tempty[s], 8); }
    tc::fence_barrier_init();
  }
  if (warp == 2) tc::tmem_alloc_2sm(tmem_slot, TMEM_COLS);
  tc::fence_before();
  tc::cluster_sync();
  tc::fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_enter();

  if (warp == 0) {
    // ===== TMA producer (both CTAs, their own A rows and B half) =====
    if (tc::elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int i = pair; i < items; i += n_pairs) {
        const MlpItem w = geo.item(i);
        const int m0 = w.mt * 256 + (int)rank * 128;
        const CUtensorMap* ta = w.down ? &tmAct : &tmX;
        const CUtensorMap* tb = w.down ? &tmWd : &tmWgu;
        int kb0 = 0, kb1 = kb_gu, brow;
        if (w.down) {
          // activations of feature block s of this m-tile: wait for its gate_up tiles (2 CTAs each)
          int* cnt = blk_cnt + w.s * geo.m_tiles + w.mt;
          const int target = 2 * geo.ft_blk;
          int v;
          while (true) {
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
            if (v >= target) break;
            __nanosleep(128);
          }
          asm volatile("fence.proxy.async.global;" ::: "memory");  // generic stores -> TMA reads
          // the last of the block's 2 * n_nt consumers resets the counters for the next launch
          int* use = blk_use + w.s * geo.m_tiles + w.mt;
          if (atomicAdd(use, 1) == 2 * geo.n_nt - 1) {
            *use = 0;
            *cnt = 0;
          }
          kb0 = w.s * kb_dn;
          kb1 = kb0 + kb_dn;
          brow = w.nt * 256 + (int)rank * 128;
        } else {
          brow = rank == 0 ? w.f * 128 : ff + w.f * 128;
        }
        for (int kb = kb0; kb < kb1; ++kb) {
          tc::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          if (leader) tc::mbar_arrive_expect_tx(&full[stage], 2 * STAGE_BYTES);
          tc::tma_load_2d_2sm(sa, ta, &full[stage], kb * BK, m0);
          tc::tma_load_2d_2sm(sa + A_BYTES, tb, &full[stage], kb * BK, brow);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer (leader CTA) =====
    if (leader) {
      constexpr uint32_t IDESC = tc::idesc_bf16(256, BN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int i = pair; i < items; i += n_pairs, ++it) {
        const MlpItem w = geo.item(i);
        const int nkb = w.down ? kb_dn : kb_gu;
        const int acc = it & 1;
        tc::mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        tc::fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < nkb; ++kb) {
          tc::mbar_wait(&full[stage], phase);
          tc::fence_after();
          if (tc::elect_one()) {
            const uint8_t* sa = smem + stage * STAGE_BYTES;
            const uint64_t adesc = tc::sdesc_sw128(sa), bdesc = tc::sdesc_sw128(sa + A_BYTES);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              tc::mma_bf16_2sm(d_tmem, adesc + 2 * k, bdesc + 2 * k, IDESC, (kb > 0 || k > 0) ? 1u : 0u);
            tc::mma_commit_2sm(&empty[stage]);
            if (kb == nkb - 1) tc::mma_commit_2sm(&tfull[acc]);
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else {
    // ===== epilogue (warps 2..5, this CTA's 128 rows) =====
    const int q = warp & 3;
    const int row = q * 32 + lane;
    int it = 0;
    for (int i = pair; i < items; i += n_pairs, ++it) {
      const MlpItem w = geo.item(i);
      const int acc = it & 1;
      const int m0 = w.mt * 256 + (int)rank * 128;
      const int m = m0 + row;
      const float rs = w.down ? 1.f : gepi::row_rs(egu, m, m < M);
      if (w.down) gepi::resid_prefetch(edn, m, m < M, w.nt * BN, BN);
      tc::mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc::fence_after();
      const bool tr = dbg != nullptr && warp == 2 && lane == 0 && blockIdx.x < 148 && it < 6;
      if (tr) dbg[blockIdx.x * 12 + 2 * it] = tc::globaltimer();
      const uint32_t trow = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
      if (!w.down) {
        // SwiGLU: gate in accumulator columns [0, 128), up in [128, 256); act row m, features f * 128 ..
#pragma unroll 1
        for (int c = 0; c < BN / 2; c += 16) {
          float v[16], u[16];
          tc::tmem_ld16(trow + c, v);
          tc::tmem_ld16(trow + BN / 2 + c, u);
#pragma unroll
          for (int x = 0; x < 16; ++x) { v[x] *= rs; u[x] *= rs; }
          if (m < M) gepi::epi16<EPI_SWIGLU>(egu, m, w.f * 128 + c, v, u);
        }
        __threadfence();  // activations visible device-wide before the block counter moves
        named_bar(1, 128);
        if (warp == 2 && lane == 0) atomicAdd(blk_cnt + w.s * geo.m_tiles + w.mt, 1);
      } else {
        // publish this K block's partial ([64 col groups][128 rows][4] per CTA, coalesced)
        const int tile = w.mt * geo.n_nt + w.nt;
        float* base = dscr + (size_t)(tile * geo.S * 2 + rank) * 128 * BN;
        const size_t pstride = (size_t)2 * 128 * BN;  // next block, same rank
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          float v[32];
          tc::tmem_ld32(trow + c, v);
          float4* dst = reinterpret_cast<float4*>(base + w.s * pstride) + (size_t)(c / 4) * 128 + row;
#pragma unroll
          for (int x = 0; x < 8; ++x) dst[x * 128] = make_float4(v[4 * x], v[4 * x + 1], v[4 * x + 2], v[4 * x + 3]);
        }
        __threadfence();
        named_bar(1, 128);
        if (warp == 2 && lane == 0) {
          int* cnt = dn_cnt + tile * 2 + rank;
          const int last = atomicAdd(cnt, 1) == geo.S - 1;
          if (last) *cnt = 0;
          *last_flag = last;
        }
        named_bar(1, 128);
        const bool merge = *last_flag != 0;
        named_bar(1, 128);
        if (merge) {  // all K blocks in block order -> TMEM, then the residual (+ RMSNorm) epilogue
          __threadfence();
          if (tr) dbg[blockIdx.x * 12 + 10] = tc::globaltimer();
          gepi::merge_pieces_to_tmem<BN, MAX_S>(base, pstride, geo.S, row, trow);
          if (tr) dbg[blockIdx.x * 12 + 11] = tc::globaltimer();
          gepi::tile_epilogue<EPI_RESID, BN>(edn, M, m0 + q * 32, w.nt * BN, trow, ebuf + (warp - 2) * gepi::EPI_WARP_F4,
                                             lane, false, true);
        }
      }
      if (tr) dbg[blockIdx.x * 12 + 2 * it + 1] = tc::globaltimer();
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive_rank0(&tempty[acc]);
    }
  }
  tc::fence_before();
  tc::cluster_sync();
  if (warp == 2) tc::tmem_dealloc_2sm(tmem_base, TMEM_COLS);
}
}  // namespace

cb_status gemm_tmap(cb_ctx* c, const void* p, long long rows, long long k, long long ld, int box_rows,
                    CUtensorMap* out);  // gemm_tc.cu
int gemm_tc_max_pairs(const cb_ctx* c);

// K blocks of the fused MLP: the largest S <= mlp_fused with ff % (128 S) == 0 (whole gate_up feature
// tiles per block; then (ff / 64) % S == 0 too), 0 when none >= 2.
static int mlp_blocks(const cb_ctx* c) {
  for (int S = c->mlp_fused; S >= 2; --S)
    if (c->m.d_ff % (128 * S) == 0) return S;
  return 0;
}

// The MLP at blend sizes: rows M <= 3 x 256, d % 256 == 0.
bool mlp_fused_ok(const cb_ctx* c, int M) {
  const cb_model& m = c->m;
  return c->mlp_fused >= 2 && c->mlp_scr != nullptr && m.dtype == CB_BF16 && M > 0 && M <= 768 && m.d_model % 256 == 0 &&
         mlp_blocks(c) >= 2;
}

cb_status launch_mlp_fused(cb_ctx* c, const void* x, const void* w_gate_up, void* act, const void* w_down, int M,
                           const EpiParams& egu, const EpiParams& edn, cudaStream_t s) {
  const cb_model& m = c->m;
  const int d = m.d_model, ff = m.d_ff, S = mlp_blocks(c);
  CB_REQUIRE(mlp_fused_ok(c, M), CB_E_UNSUPPORTED, "fused MLP does not take M=%d", M);
  MlpGeo geo;
  geo.m_tiles = (M + 255) / 256;
  geo.n_ft = ff / 128;
  geo.S = S;
  geo.ft_blk = geo.n_ft / S;
  geo.n_nt = d / 256;
  geo.G = geo.m_tiles * geo.n_ft;
  geo.D = S * geo.m_tiles * geo.n_nt;
  CUtensorMap tx, tw, ta, td;
  CB_TRY(gemm_tmap(c, x, M, d, d, 128, &tx));
  CB_TRY(gemm_tmap(c, w_gate_up, 2LL * ff, d, d, 128, &tw));
  CB_TRY(gemm_tmap(c, act, M, ff, ff, 128, &ta));
  CB_TRY(gemm_tmap(c, w_down, d, ff, ff, 128, &td));
  const int pairs = gemm_tc_max_pairs(c);
  ProfScope ps_(c, PROF_GEMM, s);
  CB_CUDA(launch_k(c, gemm_mlp_kernel, dim3(2 * pairs), dim3(NUM_THREADS), SMEM, s, 2, tx, tw, ta, td, M, d, ff, geo,
                    egu, edn, c->mlp_cnt, c->mlp_cnt + 64, c->mlp_cnt + 128, c->mlp_scr,
                    c->dbg_sel == 200 ? c->dbg_buf : nullptr));
  CB_LAUNCHED(c);
  return CB_OK;
}

cb_status gemm_mlp_init(cb_ctx* c) {
  CB_CUDA(cudaFuncSetAttribute(gemm_mlp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  // partials: up to 3 m-tiles x (d / 256) n-tiles x 4 blocks x 2 CTAs x 128 x 256 fp32
  const size_t n_nt = (size_t)std::max(1, c->m.d_model / 256);
  CB_CUDA(cudaMalloc(&c->mlp_scr, 3 * n_nt * MAX_S * 2 * 128 * BN * sizeof(float)));
  CB_CUDA(cudaMalloc(&c->mlp_cnt, (128 + 3 * n_nt * 2) * sizeof(int)));
  CB_CUDA(cudaMemset(c->mlp_cnt, 0, (128 + 3 * n_nt * 2) * sizeof(int)));
  return CB_OK;
}
