// gemm_tc.cu — tcgen05 / TMEM / TMA GEMM for the bf16 blend projections (steps a2, a3, a7, a8).
//
//   acc[M][N] = A[M][K] . B[N][K]^T     A = activation rows (K-major), B = weight rows (K-major)
//
// Persistent warp-specialised kernel, one CTA per SM:
//   warp 0      TMA producer: 128x64 A box + 256x64 B box (two 128-row boxes for SwiGLU: gate rows
//               and the matching up rows) per stage into a 4-stage SWIZZLE_128B ring
//   warp 1      MMA issuer: one elected thread issues tcgen05.mma (M=128, N=256, K=16) x 4 per stage,
//               fp32 accumulator in TMEM, double-buffered (2 x 256 columns)
//   warps 2-5   epilogue: tcgen05.ld 32x32b -> registers -> fused epilogue (RoPE / residual gather /
//               SwiGLU / store) -> global, overlapping the next tile's MMAs
// Tiles are walked m-fastest so the CTAs working on one weight tile run together (L2 reuse).
#include <cudaTypedefs.h>

#include <unordered_map>

#include "ctx.h"
#include "tc_common.cuh"

namespace {
constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2, STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int NUM_THREADS = 192;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ void st_bf16x16(bf16* p, const float (&o)[16]) {
  uint4 w0, w1;
  w0.x = pack_bf16(o[0], o[1]); w0.y = pack_bf16(o[2], o[3]); w0.z = pack_bf16(o[4], o[5]); w0.w = pack_bf16(o[6], o[7]);
  w1.x = pack_bf16(o[8], o[9]); w1.y = pack_bf16(o[10], o[11]); w1.z = pack_bf16(o[12], o[13]);
  w1.w = pack_bf16(o[14], o[15]);
  reinterpret_cast<uint4*>(p)[0] = w0;
  reinterpret_cast<uint4*>(p)[1] = w1;
}

// Epilogue for 16 consecutive output columns n..n+15 of row m (all < N; N % 16 == 0).
template <int KIND>
__device__ __forceinline__ void epi16(const EpiParams& e, int m, int n, const float (&v)[16], const float (&u)[16]) {
  float o[16];
  if constexpr (KIND == EPI_STORE) {
    st_bf16x16(reinterpret_cast<bf16*>(e.out) + (size_t)m * e.ldo + n, v);
  } else if constexpr (KIND == EPI_STORE_F32) {
    float4* p = reinterpret_cast<float4*>(e.outf + (size_t)m * e.ldo + n);
#pragma unroll
    for (int i = 0; i < 4; ++i) p[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
  } else if constexpr (KIND == EPI_QKV) {
    const int c = e.col0 + n;
    if (c < e.qd + e.kvd) {  // q or k head: rotate pairs (2i, 2i+1) at the row's global position
      const int dim = (c < e.qd ? c : c - e.qd) % e.hd;
      const int p = __ldg(e.pos + __ldg(e.row_tok + m));
      const float4* cs = reinterpret_cast<const float4*>(e.rope_tab + (size_t)p * (e.hd >> 1) + (dim >> 1));
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float4 t = __ldg(cs + i);  // (cos, sin) of pairs 2i, 2i+1
        const float a0 = v[4 * i], a1 = v[4 * i + 1], b0 = v[4 * i + 2], b1 = v[4 * i + 3];
        o[4 * i] = t.x * a0 - t.y * a1;
        o[4 * i + 1] = t.y * a0 + t.x * a1;
        o[4 * i + 2] = t.z * b0 - t.w * b1;
        o[4 * i + 3] = t.w * b0 + t.z * b1;
      }
      bf16* dst = (c < e.qd) ? reinterpret_cast<bf16*>(e.q_out) + (size_t)m * e.qd + c
                             : reinterpret_cast<bf16*>(e.k_out) + (size_t)m * e.kvd + (c - e.qd);
      st_bf16x16(dst, o);
    } else {
      st_bf16x16(reinterpret_cast<bf16*>(e.v_out) + (size_t)m * e.kvd + (c - e.qd - e.kvd), v);
    }
  } else if constexpr (KIND == EPI_RESID) {
    const int src = e.res_row ? __ldg(e.res_row + m) : m;
    const float4* hi = reinterpret_cast<const float4*>(e.h_in + (size_t)src * e.ldo + n);
    float4* ho = reinterpret_cast<float4*>(e.h_out + (size_t)m * e.ldo + n);
    float4 hv[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) hv[i] = hi[i];
#pragma unroll
    for (int i = 0; i < 4; ++i)
      ho[i] = make_float4(hv[i].x + v[4 * i], hv[i].y + v[4 * i + 1], hv[i].z + v[4 * i + 2], hv[i].w + v[4 * i + 3]);
  } else if constexpr (KIND == EPI_SWIGLU) {
#pragma unroll
    for (int i = 0; i < 16; ++i) o[i] = v[i] / (1.f + __expf(-v[i])) * u[i];
    st_bf16x16(reinterpret_cast<bf16*>(e.act) + (size_t)m * e.ff + n, o);
  }
}

template <int KIND>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int K,
                   int m_tiles, int n_tiles, EpiParams e) {
  constexpr bool SW = (KIND == EPI_SWIGLU);
  constexpr int OUT_N = SW ? BN / 2 : BN;  // output columns per tile
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tiles_total = m_tiles * n_tiles;
  const int num_kb = (K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tmA);
    tc::tma_prefetch(&tmB);
    for (int s = 0; s < STAGES; ++s) { tc::mbar_init(&full[s], 1); tc::mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { tc::mbar_init(&tfull[s], 1); tc::mbar_init(&tempty[s], 4); }
    tc::fence_barrier_init();
  }
  if (warp == 2) tc::tmem_alloc(tmem_slot, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===== TMA producer =====
    if (tc::elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < n_tiles_total; t += gridDim.x) {
        const int m0 = (t % m_tiles) * BM, nb = t / m_tiles;
        for (int kb = 0; kb < num_kb; ++kb) {
          tc::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          tc::mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
          tc::tma_load_2d(sa, &tmA, &full[stage], kb * BK, m0);
          if constexpr (SW) {
            tc::tma_load_2d(sb, &tmB, &full[stage], kb * BK, nb * OUT_N);
            tc::tma_load_2d(sb + B_BYTES / 2, &tmB, &full[stage], kb * BK, e.ff + nb * OUT_N);
          } else {
            tc::tma_load_2d(sb, &tmB, &full[stage], kb * BK, nb * BN);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer =====
    constexpr uint32_t IDESC = tc::idesc_bf16(BM, BN);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int t = blockIdx.x; t < n_tiles_total; t += gridDim.x, ++it) {
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      tc::mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc::fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = 0; kb < num_kb; ++kb) {
        tc::mbar_wait(&full[stage], phase);
        tc::fence_after();
        if (tc::elect_one()) {
          const uint8_t* sa = smem + stage * STAGE_BYTES;
          const uint64_t adesc = tc::sdesc_sw128(sa), bdesc = tc::sdesc_sw128(sa + A_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)  // advance 16 bf16 = 32 B (>> 4 = 2) inside the swizzle atom
            tc::mma_bf16(d_tmem, adesc + 2 * k, bdesc + 2 * k, IDESC, (kb | k) != 0);
          tc::mma_commit(&empty[stage]);
          if (kb == num_kb - 1) tc::mma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else {
    // ===== epilogue (warps 2..5; warp w reads TMEM lanes 32*(w%4) .. +31) =====
    const int q = warp & 3;
    int it = 0;
    for (int t = blockIdx.x; t < n_tiles_total; t += gridDim.x, ++it) {
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const int m0 = (t % m_tiles) * BM, nb = t / m_tiles;
      tc::mbar_wait(&tfull[acc], acc_phase);
      tc::fence_after();
      const int m = m0 + q * 32 + lane;
      const uint32_t trow = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
#pragma unroll 1
      for (int c = 0; c < OUT_N; c += 16) {
        float v[16], u[16];
        tc::tmem_ld16(trow + c, v);
        if constexpr (SW) tc::tmem_ld16(trow + BN / 2 + c, u);
        const int n = nb * OUT_N + c;
        if (m < M && n < e.N) epi16<KIND>(e, m, n, v, u);
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == 2) tc::tmem_dealloc(tmem_base, 512);
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
}  // namespace

struct TmapCache {
  std::unordered_map<TmKey, CUtensorMap, TmKeyHash> maps;
};

static cb_status get_tmap(cb_ctx* c, const void* p, long long rows, long long k, long long ld, int box_rows,
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

template <int KIND>
static cb_status launch_kind(cb_ctx* c, const CUtensorMap& ta, const CUtensorMap& tb, int M, int K, int m_tiles,
                             int n_tiles, const EpiParams& e, cudaStream_t s) {
  const int tiles = m_tiles * n_tiles;
  const int grid = std::min(tiles, c->num_sms);
  gemm_tc_kernel<KIND><<<grid, NUM_THREADS, SMEM_BYTES, s>>>(ta, tb, M, K, m_tiles, n_tiles, e);
  CB_LAUNCHED(c);
  return CB_OK;
}

cb_status launch_gemm_tc(cb_ctx* c, const void* A, int lda, const void* B, int ldb, int M, int K, const EpiParams& e,
                         cudaStream_t s) {
  const bool sw = e.kind == EPI_SWIGLU;
  const int out_n = sw ? BN / 2 : BN;
  const long long b_rows = sw ? 2LL * e.ff : (long long)e.N;
  CUtensorMap ta, tb;
  CB_TRY(get_tmap(c, A, M, K, lda, BM, &ta));
  CB_TRY(get_tmap(c, B, b_rows, K, ldb, sw ? BN / 2 : BN, &tb));
  const int m_tiles = (M + BM - 1) / BM, n_tiles = (e.N + out_n - 1) / out_n;
  ProfScope ps_(c, PROF_GEMM, s);
  switch (e.kind) {
    case EPI_STORE: return launch_kind<EPI_STORE>(c, ta, tb, M, K, m_tiles, n_tiles, e, s);
    case EPI_STORE_F32: return launch_kind<EPI_STORE_F32>(c, ta, tb, M, K, m_tiles, n_tiles, e, s);
    case EPI_QKV: return launch_kind<EPI_QKV>(c, ta, tb, M, K, m_tiles, n_tiles, e, s);
    case EPI_RESID: return launch_kind<EPI_RESID>(c, ta, tb, M, K, m_tiles, n_tiles, e, s);
    case EPI_SWIGLU: return launch_kind<EPI_SWIGLU>(c, ta, tb, M, K, m_tiles, n_tiles, e, s);
  }
  cb_set_error("bad epilogue kind %d", e.kind);
  return CB_E_INVALID_ARG;
}

cb_status gemm_tc_init(cb_ctx* c) {
  if (g_encode == nullptr) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    CB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    CB_REQUIRE(q == cudaDriverEntryPointSuccess && fn != nullptr, CB_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  CB_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<EPI_STORE>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
  CB_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<EPI_STORE_F32>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
  CB_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<EPI_QKV>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
  CB_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<EPI_RESID>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
  CB_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<EPI_SWIGLU>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
  c->tmaps = new TmapCache();
  return CB_OK;
}

void gemm_tc_destroy(cb_ctx* c) {
  delete c->tmaps;
  c->tmaps = nullptr;
}
