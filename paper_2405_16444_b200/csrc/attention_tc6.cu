// attention_tc6.cu — persistent tcgen05 / TMEM / TMA sparse-query causal attention (step a6), bf16,
// head_dim 128. Same math and per-tile pipeline as attention_tc5.cu:
//
//   out[r][h] = softmax_j(q_{r,h} . k_{j,g} / sqrt(hd)) v_{j,g} over keys j <= q_tok[r]
//
// What differs is the work distribution. The blend's query rows are in token order, so row tile i
// (128 GQA-packed rows of one kv head) reaches keys 0..max token of its rows: the last tiles see
// ~all keys, the first ones few. A one-CTA-per-tile grid therefore runs as long as its heaviest tile.
// Here one CTA per SM loops over work items = (row tile, kv head, key chunk of C key tiles), claimed
// from a global counter in heaviest-first order (row tile descending), so the SMs drain an LPT-ordered
// queue. A row tile whose keys span several chunks writes fp32 partials (O, m, l); the last chunk to
// finish merges them in chunk order (deterministic) and writes the output.
//
// Inside an item the key tiles form two independent online-softmax streams (even / odd tiles), one
// per softmax warpgroup, each with its own TMEM S buffer and O accumulator, merged at the end of the
// item: while one warpgroup runs exp2 on its tile the tensor core works on the other stream, so the
// per-tile softmax latency chain is hidden instead of serialising S -> softmax -> PV.
// TMEM (512 columns): S/P stream 0 [0,128), S/P stream 1 [128,256), O stream 0 [256,384), O stream 1
// [384,512). P (bf16, 2 per column) overwrites its S columns and is read by the PV MMA straight from
// TMEM (A operand in tensor memory), so P never touches shared memory.
//
// Warp roles (384 threads):
//   warp 0     claims items (lane 0; the first one is blockIdx.x) and publishes them through a 2-slot
//              ring in shared memory; gathers the item's Q rows (whole warp, cp.async through q_row)
//              once the previous item's QK^T MMAs are done; streams K/V tiles by TMA (2-stage rings)
//   warp 1     MMA issuer, order S0 S1 PV0 S2 PV1 S3 ...: the in-order tensor pipe completes PV(t),
//              which reads P(t) from TMEM, before S(t+2) overwrites those columns
//   warps 2-3  idle (they complete the first warpgroup, which hands registers to the softmax ones)
//   warps 4-11 softmax, warpgroup = stream, thread = one row x all 128 keys of the tile (log2 domain,
//              lazy rescale of the stream's O in TMEM); then the item epilogue (streams merged, O / l,
//              or a partial + the in-kernel chunk merge). setmaxnreg gives them 216 registers.
#include <cudaTypedefs.h>

#include "ctx.h"
#include "tc_common.cuh"

namespace {
constexpr int HD = 128, BM = 128, BC = 128, NT = 384;  // 3 warpgroups: load/MMA, stream 0, stream 1
constexpr int ATOM = 128 * 128;  // 128 rows x 128 B: one SWIZZLE_128B column block
constexpr int TILE = 2 * ATOM;   // 128 rows x 128 bf16
constexpr int MAX_TILES = 512;   // row tiles per launch (smem tables)
constexpr int BAR_BYTES = 256;
constexpr int XCH_BYTES = 3328;  // row-max / row-sum exchange + flags
constexpr int TAB_BYTES = 3 * MAX_TILES * 4 + 64;
constexpr int SMEM = 6 * TILE + 1024 + BAR_BYTES + XCH_BYTES + TAB_BYTES;
constexpr float RESCALE_THRESHOLD = 8.0f;  // log2 units

__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ float ex2(float x) {  // MUFU.EX2; ex2(-inf) = 0
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
// byte offset of 16-B chunk `ch` (0..15) of row `r` in a [2 atoms][128 rows][128 B] swizzled tile
__device__ __forceinline__ uint32_t sw_off(int r, int ch) {
  return (uint32_t)((ch >> 3) * ATOM + r * 128 + (((ch & 7) ^ (r & 7)) << 4));
}

// CB_ATTN_TRACE builds: clock64 per-tile events of CTA 0's first item at dbg[1792 + ...]
#ifdef CB_ATTN_TRACE
#define TR(i, cond) do { if ((cond) && dbg != nullptr && blockIdx.x == 0 && (i) < 256) dbg[1792 + (i)] = clock64(); } while (0)
#else
#define TR(i, cond) do { } while (0)
#endif

__device__ __forceinline__ bool trace_on(const long long* dbg, int et, int it) {
  return dbg != nullptr && et == 0 && blockIdx.x < 148 && it < 3;
}

struct Item {
  int tile, head, chunk, kb0, nt, n_chunks;
};

// Item k of the heaviest-first order: row tiles descending, then key chunk, then kv head.
// pre[j] = number of items of the j heaviest tiles (pre[0] = 0), nkt[tile] = key tiles of the tile.
__device__ __forceinline__ Item decode(int k, const int* pre, const int* nkt, int tiles, int n_kv, int C) {
  int lo = 0, hi = tiles - 1;  // largest j with pre[j] <= k
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (pre[mid] <= k) lo = mid; else hi = mid - 1;
  }
  Item it;
  it.tile = tiles - 1 - lo;
  const int idx = k - pre[lo];
  it.chunk = idx / n_kv;
  it.head = idx - it.chunk * n_kv;
  const int n = nkt[it.tile];
  it.n_chunks = (n + C - 1) / C;
  it.kb0 = it.chunk * C;
  it.nt = min(n, it.kb0 + C) - it.kb0;
  return it;
}

__global__ void __launch_bounds__(NT, 1)
    attn_tc6_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                    const bf16* __restrict__ q, const int* __restrict__ q_row, const int* __restrict__ q_tok,
                    int n_rows, int n_keys, bf16* __restrict__ out, int n_q, int n_kv, float scale_log2, int C,
                    float* __restrict__ opart, float2* __restrict__ ml, int* __restrict__ tile_cnt,
                    int* __restrict__ work, long long* __restrict__ dbg) {
  // debug_trace: per CTA (< 148) and its first 3 items: [cta * 8 + 2 it + 1] item end (globaltimer ns,
  // softmax thread 0), [1184 + cta * 4 + it] = item index k * 64 + nt
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = smem + TILE;      // [2] stages
  uint8_t* sV = smem + 3 * TILE;  // [2] stages
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 6 * TILE);
  uint64_t* k_full = bars;          // [2]
  uint64_t* k_empty = bars + 2;     // [2]
  uint64_t* v_full = bars + 4;      // [2]
  uint64_t* v_empty = bars + 6;     // [2]
  uint64_t* s_full = bars + 8;      // [2 streams]  S(t) of stream t % 2 landed in its TMEM buffer
  uint64_t* p_full = bars + 10;     // [2 streams]  P written over it (the stream's 4 softmax warps)
  uint64_t* item_full = bars + 12;  // [2]
  uint64_t* item_empty = bars + 14; // [2]  (MMA warp + 8 softmax warps)
  uint64_t* q_full = bars + 16;
  uint64_t* q_empty = bars + 17;
  uint64_t* o_done = bars + 18;     // last PV of the item complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 20);
  int* item_k = reinterpret_cast<int*>(bars + 21);  // [2]
  float* xmax = reinterpret_cast<float*>(smem + 6 * TILE + BAR_BYTES);  // [2 parity][2 wg][128]
  float* xl = xmax + 512;                                               // [2 wg][128]
  int* xflag = reinterpret_cast<int*>(xl + 256);
  int* nkt = reinterpret_cast<int*>(smem + 6 * TILE + BAR_BYTES + XCH_BYTES);  // [MAX_TILES]
  int* kmn = nkt + MAX_TILES;                                                  // [MAX_TILES] first token
  int* pre = kmn + MAX_TILES;                                                  // [MAX_TILES + 1]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = n_q / n_kv, R = n_rows * G, qd = n_q * HD;
  const int tiles = (R + BM - 1) / BM;

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tmK);
    tc::tma_prefetch(&tmV);
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&k_full[b], 1);
      tc::mbar_init(&k_empty[b], 1);
      tc::mbar_init(&v_full[b], 1);
      tc::mbar_init(&v_empty[b], 1);
      tc::mbar_init(&s_full[b], 1);
      tc::mbar_init(&p_full[b], 4);
      tc::mbar_init(&item_full[b], 1);
      tc::mbar_init(&item_empty[b], 9);
    }
    tc::mbar_init(q_full, 1);
    tc::mbar_init(q_empty, 1);
    tc::mbar_init(o_done, 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
  pdl_enter();  // q, q_row, q_tok and K/V come from the previous kernels
  // work table: key tiles and first token of every row tile, item prefix sums in heaviest-first order
  for (int i = threadIdx.x; i < tiles; i += NT) {
    const int r0 = i * BM, r1 = min(R, r0 + BM) - 1;
    int kmax = -1, kmin = 1 << 30;
    for (int rt = r0 / G; rt <= r1 / G; ++rt) {
      const int t = min(__ldg(q_tok + rt), n_keys - 1);
      kmax = max(kmax, t);
      kmin = min(kmin, t);
    }
    nkt[i] = (kmax + BC) / BC;
    kmn[i] = kmin;
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 0) {  // exclusive scan of items per tile over tiles in descending order
    int carry = 0;
    for (int j0 = 0; j0 < tiles; j0 += 32) {
      const int j = j0 + lane;
      const int v = j < tiles ? ((nkt[tiles - 1 - j] + C - 1) / C) * n_kv : 0;
      int x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (j < tiles) pre[j] = carry + x - v;
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) pre[tiles] = carry;
  }
  __syncthreads();
  const int n_items = pre[tiles];
  const uint32_t tmem = *tmem_slot;
  // registers move from the load/MMA warpgroup to the two softmax warpgroups (a row of 128 scores each)
  if (warp < 4) {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 72;" ::: "memory");
  if (warp == 0) {
    // ===== work claims, Q gather (whole warp), K/V TMA (lane 0) =====
    int tg = 0;  // key tiles issued so far (stage / phase of the K and V rings)
    for (int it = 0;; ++it) {
      const int slot = it & 1;
      int k = 0;
      if (lane == 0) {
        if (it >= 2) tc::mbar_wait(&item_empty[slot], ((it >> 1) - 1) & 1);
        k = it == 0 ? (int)blockIdx.x : (int)gridDim.x + atomicAdd(work, 1);  // first item static
        item_k[slot] = k;
        tc::mbar_arrive(&item_full[slot]);
      }
      k = __shfl_sync(0xffffffffu, k, 0);
      if (k >= n_items) break;
      const Item w = decode(k, pre, nkt, tiles, n_kv, C);
      if (it >= 1) tc::mbar_wait(q_empty, (it - 1) & 1);
      {  // lane owns rows lane + 32 j: their source rows first (independent loads), then 64 cp.async
        const uint32_t dq = tc::smem_u32(sQ);
        int qr[4];
#pragma unroll
        for (int jr = 0; jr < 4; ++jr) {
          const int rho = min(w.tile * BM + lane + 32 * jr, R - 1);
          qr[jr] = __ldg(q_row + rho / G);
        }
#pragma unroll 1
        for (int jr = 0; jr < 4; ++jr) {
          const int r = lane + 32 * jr, rho = w.tile * BM + r;
          const bf16* src = q + (size_t)qr[jr] * qd + (size_t)(w.head * G + rho % G) * HD;
          const int sz = rho < R ? 16 : 0;
#pragma unroll
          for (int ch = 0; ch < 16; ++ch)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dq + sw_off(r, ch)), "l"(src + ch * 8),
                         "r"(sz)
                         : "memory");
        }
      }
      auto load = [&](uint8_t* dst, const CUtensorMap* m, uint64_t* bar, int key0) {
        tc::mbar_arrive_expect_tx(bar, TILE);
        tc::tma_load_3d(dst, m, bar, 0, w.head, key0);
        tc::tma_load_3d(dst + ATOM, m, bar, 64, w.head, key0);
      };
      auto load_k = [&](int j) {
        const int t = tg + j, b = t & 1;
        if (t >= 2) tc::mbar_wait(&k_empty[b], ((t >> 1) - 1) & 1);
        load(sK + b * TILE, &tmK, &k_full[b], (w.kb0 + j) * BC);
      };
      auto load_v = [&](int j) {
        const int t = tg + j, b = t & 1;
        if (t >= 2) tc::mbar_wait(&v_empty[b], ((t >> 1) - 1) & 1);
        load(sV + b * TILE, &tmV, &v_full[b], (w.kb0 + j) * BC);
      };
      if (lane == 0) load_k(0);  // its stage was released by the previous item's S MMAs
      asm volatile("cp.async.wait_all;" ::: "memory");
      tc::fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        tc::mbar_arrive(q_full);
        // order of use by the MMA warp: S0 S1 PV0 S2 PV1 S3 ...
        if (w.nt > 1) load_k(1);
        for (int j = 0; j < w.nt; ++j) {
          load_v(j);
          if (j + 2 < w.nt) load_k(j + 2);
        }
      }
      tg += w.nt;
      __syncwarp();
    }
  } else if (warp == 1) {
    // ===== MMA issuer: S(t) into the S buffer of stream t & 1; PV(t) with P from that buffer (TMEM)
    // into O of stream t & 1. Issue order S0 S1 PV0 S2 PV1 S3 ...: the in-order tensor pipe finishes
    // PV(t) (reading P(t) from TMEM) before S(t+2) overwrites the same columns. =====
    constexpr uint32_t IDESC_S = tc::idesc_bf16(BM, BC);
    constexpr uint32_t IDESC_PV = tc::idesc_bf16_bmn(BM, HD);
    int tg = 0;
    int pcnt0 = 0, pcnt1 = 0;  // p_full completions consumed per stream
    auto issue_s = [&](int t, int jb) {  // t: flat key-tile index, jb: tile within the item
      const int b = t & 1;
      tc::mbar_wait(&k_full[b], (t >> 1) & 1);
      tc::fence_after();
      TR(4 * t, lane == 0 && t < 48);
      if (tc::elect_one()) {
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint64_t a = tc::sdesc_sw128(sQ + (kk >> 2) * ATOM) + 2 * (kk & 3);
          const uint64_t bd = tc::sdesc_sw128(sK + b * TILE + (kk >> 2) * ATOM) + 2 * (kk & 3);
          tc::mma_bf16(tmem + (jb & 1) * 128, a, bd, IDESC_S, kk > 0 ? 1u : 0u);
        }
        tc::mma_commit(&s_full[jb & 1]);
        tc::mma_commit(&k_empty[b]);
      }
      __syncwarp();
    };
    for (int it = 0;; ++it) {
      const int slot = it & 1;
      tc::mbar_wait(&item_full[slot], (it >> 1) & 1);
      const int k = item_k[slot];
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&item_empty[slot]);
      if (k >= n_items) break;
      const Item w = decode(k, pre, nkt, tiles, n_kv, C);
      tc::mbar_wait(q_full, it & 1);
      issue_s(tg, 0);
      if (w.nt > 1) issue_s(tg + 1, 1);
      if (w.nt <= 2) {  // every S of the item issued: Q is free once they complete
        if (tc::elect_one()) tc::mma_commit(q_empty);
        __syncwarp();
      }
      for (int j = 0; j < w.nt; ++j) {
        const int t = tg + j, b = t & 1, st = j & 1;
        tc::mbar_wait(&p_full[st], (st ? pcnt1 : pcnt0) & 1);
        if (st) ++pcnt1; else ++pcnt0;
        tc::mbar_wait(&v_full[b], (t >> 1) & 1);
        tc::fence_after();
        TR(4 * t + 1, lane == 0 && t < 48);
        if (tc::elect_one()) {
#pragma unroll
          for (int kk = 0; kk < BC / 16; ++kk) {  // 16 keys per step: P columns 8 kk .. 8 kk + 7
            const uint64_t bd = tc::sdesc_sw128_mn(sV + b * TILE + kk * 2048, ATOM);
            tc::mma_bf16_ts(tmem + 256 + st * 128, tmem + st * 128 + kk * 8, bd, IDESC_PV, (j > 1 || kk > 0) ? 1u : 0u);
          }
          tc::mma_commit(&v_empty[b]);
          if (j + 1 == w.nt) tc::mma_commit(o_done);
        }
        __syncwarp();
        if (j + 2 < w.nt) {
          issue_s(t + 2, j + 2);
          if (j + 3 == w.nt) {
            if (tc::elect_one()) tc::mma_commit(q_empty);
            __syncwarp();
          }
        }
      }
      tg += w.nt;
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 216;" ::: "memory");
    // ===== softmax: warpgroup st = key stream st (tiles j with j % 2 == st), thread = one row, all 128
    // keys of the tile. Then the item epilogue: both streams merged (warpgroup st writes output
    // columns 64 st .. 64 st + 63). =====
    const int st = (warp - 4) >> 2;
    const int r = (warp & 3) * 32 + lane;
    const int et = threadIdx.x - 128;  // 0..255
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + lane_base + st * 128;  // this stream's S / P columns
    const uint32_t tO = tmem + lane_base + 256;        // O of stream 0 at +0, stream 1 at +128
    int scnt = 0;  // s_full completions consumed by this stream (phase)
    for (int it = 0;; ++it) {
      const int slot = it & 1;
      tc::mbar_wait(&item_full[slot], (it >> 1) & 1);
      const int k = item_k[slot];
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&item_empty[slot]);
      if (k >= n_items) break;
      const Item w = decode(k, pre, nkt, tiles, n_kv, C);
      const int rho = w.tile * BM + r;
      const bool valid = rho < R;
      const int rt = valid ? rho / G : 0, hh = w.head * G + (valid ? rho % G : 0);
      const int tok = valid ? min(__ldg(q_tok + rt), n_keys - 1) : -1;
      const int kmin = kmn[w.tile];
      float m_used = -INFINITY, l = 0.f;
      const int n_mine = (w.nt - st + 1) / 2;
      for (int i = 0; i < n_mine; ++i) {
        const int j = 2 * i + st;
        tc::mbar_wait(&s_full[st], scnt & 1);
        ++scnt;
        tc::fence_after();
        TR(4 * j + 2, r == 0 && it == 0 && j < 48);
        float s[128];
        {
          uint32_t u[4][32];
#pragma unroll
          for (int c = 0; c < 4; ++c) tc::tmem_ld32_nw(tS + c * 32, u[c]);
          tc::tmem_ld_wait();
          TR(200 + 4 * j, r == 0 && it == 0 && j < 12);
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int x = 0; x < 32; ++x) s[c * 32 + x] = __uint_as_float(u[c][x]);
        }
        const int key0 = (w.kb0 + j) * BC;
        float mx8[8];
#pragma unroll
        for (int x = 0; x < 8; ++x) mx8[x] = -INFINITY;
        // keys x > lim of this tile lie after the row's token (masked only when the tile reaches past
        // the first token of the row tile)
        const int lim = key0 + BC - 1 > kmin ? tok - key0 : BC;
#pragma unroll
        for (int x = 0; x < 128; ++x) mx8[x & 7] = fmaxf(mx8[x & 7], x > lim ? -INFINITY : s[x]);
        const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                               fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]))) * scale_log2;
        float corr = 1.f;
        if (mx > m_used + RESCALE_THRESHOLD || (m_used == -INFINITY && mx != -INFINITY)) {
          if (m_used != -INFINITY) corr = ex2(m_used - mx);
          m_used = mx;
        }
        const float nref = m_used == -INFINITY ? 0.f : -m_used;
        TR(200 + 4 * j + 1, r == 0 && it == 0 && j < 12);
        l *= corr;
        // O of this stream holds PV(j - 2), complete: S(j) was issued after it on the in-order pipe
        if (i >= 1 && __any_sync(0xffffffffu, corr != 1.f)) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            float o[32];
            tc::tmem_ld32(tO + st * 128 + c * 32, o);
#pragma unroll
            for (int x = 0; x < 32; ++x) o[x] *= corr;
            tc::tmem_st32(tO + st * 128 + c * 32, o);
          }
        }
        float rs8[8];
#pragma unroll
        for (int x = 0; x < 8; ++x) rs8[x] = 0.f;
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // P columns 32 h .. 32 h + 31 = keys 64 h .. 64 h + 63
          uint32_t pk[32];
#pragma unroll
          for (int x = 0; x < 64; x += 2) {
            const float p0 = 64 * h + x > lim ? 0.f : ex2(fmaf(s[64 * h + x], scale_log2, nref));
            const float p1 = 64 * h + x + 1 > lim ? 0.f : ex2(fmaf(s[64 * h + x + 1], scale_log2, nref));
            rs8[x & 7] += p0;
            rs8[(x + 1) & 7] += p1;
            pk[x >> 1] = pack2(p0, p1);
          }
          tc::tmem_st32u(tS + 32 * h, pk);
        }
        l += ((rs8[0] + rs8[1]) + (rs8[2] + rs8[3])) + ((rs8[4] + rs8[5]) + (rs8[6] + rs8[7]));
        TR(200 + 4 * j + 2, r == 0 && it == 0 && j < 12);
        tc::tmem_st_wait();
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&p_full[st]);
        TR(4 * j + 3, r == 0 && it == 0 && j < 48);
      }
      // ---- item epilogue: merge the two streams (warpgroup st: output columns 64 st ..) ----
      xmax[st * 128 + r] = m_used;
      xl[st * 128 + r] = l;
      tc::mbar_wait(o_done, it & 1);
      tc::fence_after();
      named_bar_sync(1, 256);
      const float ma = xmax[r], mb = xmax[128 + r];
      const float mstar = fmaxf(ma, mb);
      const float fa = ma == -INFINITY ? 0.f : ex2(ma - mstar), fb = mb == -INFINITY ? 0.f : ex2(mb - mstar);
      l = xl[r] * fa + xl[128 + r] * fb;
      float o[64];
      {
        float oa[32], ob[32];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          tc::tmem_ld32(tO + st * 64 + c * 32, oa);  // stream 0
          if (w.nt > 1) tc::tmem_ld32(tO + 128 + st * 64 + c * 32, ob);  // stream 1 (may be empty)
#pragma unroll
          for (int x = 0; x < 32; ++x) o[c * 32 + x] = oa[x] * fa + (w.nt > 1 ? ob[x] * fb : 0.f);
        }
      }
      tc::fence_before();
      named_bar_sync(1, 256);  // exchange buffers read by both warpgroups
      m_used = mstar;
      bool write_out = w.n_chunks == 1;
      if (!write_out) {
        const size_t prow = ((size_t)w.chunk * n_kv + w.head) * R + rho;
        if (valid) {
          float4* dst = reinterpret_cast<float4*>(opart + prow * HD + st * 64);
#pragma unroll
          for (int x = 0; x < 16; ++x) dst[x] = make_float4(o[4 * x], o[4 * x + 1], o[4 * x + 2], o[4 * x + 3]);
          if (st == 0) ml[prow] = make_float2(m_used, l);
        }
        __threadfence();  // partials visible device-wide before this chunk's arrival is counted
        named_bar_sync(1, 256);
        if (et == 0) {
          int* cnt = tile_cnt + (size_t)w.tile * n_kv + w.head;
          const int last = atomicAdd(cnt, 1) == w.n_chunks - 1;
          if (last) *cnt = 0;  // reset for the next launch
          *xflag = last;
        }
        named_bar_sync(1, 256);
        write_out = *xflag != 0;
        if (write_out && valid) {  // last chunk of the row tile: merge all chunks in order
          __threadfence();
          float ms = -INFINITY;
          for (int sp = 0; sp < w.n_chunks; ++sp)
            ms = fmaxf(ms, __ldcg(&ml[((size_t)sp * n_kv + w.head) * R + rho].x));
          float lt = 0.f;
#pragma unroll
          for (int x = 0; x < 64; ++x) o[x] = 0.f;
          for (int sp = 0; sp < w.n_chunks; ++sp) {
            const size_t pr = ((size_t)sp * n_kv + w.head) * R + rho;
            const float2 mlv = __ldcg(&ml[pr]);
            if (mlv.x == -INFINITY) continue;
            const float f = ex2(mlv.x - ms);
            lt += mlv.y * f;
            const float4* src = reinterpret_cast<const float4*>(opart + pr * HD + st * 64);
#pragma unroll
            for (int x = 0; x < 16; ++x) {
              const float4 v = __ldcg(src + x);
              o[4 * x] += v.x * f; o[4 * x + 1] += v.y * f; o[4 * x + 2] += v.z * f; o[4 * x + 3] += v.w * f;
            }
          }
          l = lt;
        }
        named_bar_sync(1, 256);  // xflag read by everyone before the next item may overwrite it
      }
      if (valid && write_out) {
        const float inv = l > 0.f ? 1.f / l : 0.f;
        uint4* dst = reinterpret_cast<uint4*>(out + (size_t)rt * qd + (size_t)hh * HD + st * 64);
#pragma unroll
        for (int c8 = 0; c8 < 8; ++c8) {
          uint4 v;
          v.x = pack2(o[c8 * 8 + 0] * inv, o[c8 * 8 + 1] * inv);
          v.y = pack2(o[c8 * 8 + 2] * inv, o[c8 * 8 + 3] * inv);
          v.z = pack2(o[c8 * 8 + 4] * inv, o[c8 * 8 + 5] * inv);
          v.w = pack2(o[c8 * 8 + 6] * inv, o[c8 * 8 + 7] * inv);
          dst[c8] = v;
        }
      }
      if (trace_on(dbg, et, it)) {
        dbg[blockIdx.x * 8 + 2 * it + 1] = tc::globaltimer();
        dbg[1184 + blockIdx.x * 4 + it] = (long long)k * 64 + w.nt;
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
  if (threadIdx.x == 0) {  // the last CTA out resets the claim counter for the next launch
    __threadfence();
    if (atomicAdd(work + 1, 1) == (int)gridDim.x - 1) {
      work[0] = 0;
      work[1] = 0;
    }
  }
}

}  // namespace

cb_status kv_tmap5(const cb_ctx* c, const void* p, int n_keys, CUtensorMap* out);  // attention_tc5.cu

bool attention_tc6_ok(const cb_ctx* c, int n_rows) {
  const int G = c->m.n_q_heads / c->m.n_kv_heads;
  return c->m.dtype == CB_BF16 && c->m.head_dim == HD && ((long long)n_rows * G + BM - 1) / BM <= MAX_TILES;
}

cb_status launch_attention_tc6(cb_ctx* c, const void* q, const int* q_row, const int* q_tok, int n_rows, const void* k,
                               const void* v, int n_keys, void* out, cudaStream_t s) {
  if (n_rows == 0) return CB_OK;
  CB_REQUIRE(((uintptr_t)k | (uintptr_t)v) % 16 == 0, CB_E_INVALID_ARG, "K/V must be 16-byte aligned");
  CB_REQUIRE(attention_tc6_ok(c, n_rows), CB_E_UNSUPPORTED, "persistent attention: too many row tiles");
  const int n_kv = c->m.n_kv_heads, G = c->m.n_q_heads / n_kv;
  const int R = n_rows * G, tiles = (R + BM - 1) / BM;
  const int max_kt = (n_keys + BC - 1) / BC;
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)HD);
  // key chunk: rows are in token order, so the launch holds ~ n_kv * max_kt * (tiles + 1) / 2 key tiles;
  // chunks of about a third of a CTA's share keep the LPT queue balanced without many partial merges
  int C = c->attn_splits > 0 ? (max_kt + c->attn_splits - 1) / c->attn_splits : 0;
  if (C == 0) {
    const double total = (double)n_kv * max_kt * (tiles + 1) / 2.0;
    C = std::max(4, (int)std::ceil(total / (3.0 * c->num_sms)));
  }
  C = std::max(C, 1);
  // partial slots: chunk-major [chunk][n_kv][R] rows of the split-KV buffers
  while ((long long)((max_kt + C - 1) / C) * n_kv * R > c->attn_part_rows) ++C;
  const long long items_max = (long long)tiles * n_kv * ((max_kt + C - 1) / C);
  const int grid = (int)std::min<long long>(c->num_sms, items_max);
  CB_REQUIRE((long long)tiles * n_kv <= c->attn_cnt_n, CB_E_SHAPE, "attention: row tiles exceed the counter array");
  CUtensorMap tk, tv;
  CB_TRY(kv_tmap5(c, k, n_keys, &tk));
  CB_TRY(kv_tmap5(c, v, n_keys, &tv));
  ProfScope ps_(c, PROF_ATTN, s);
  CB_LAUNCH(c, (attn_tc6_kernel), grid, NT, SMEM, s, tk, tv, (const bf16*)q, q_row, q_tok, n_rows, n_keys, (bf16*)out,
            c->m.n_q_heads, n_kv, scale_log2, C, c->attn_part, c->attn_ml, c->attn_cnt, c->attn_work,
            c->dbg_sel == 1 ? c->dbg_buf : nullptr);
  CB_LAUNCHED(c);
  return CB_OK;
}

cb_status attention_tc6_init() {
  CB_CUDA(cudaFuncSetAttribute(attn_tc6_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  return CB_OK;
}
