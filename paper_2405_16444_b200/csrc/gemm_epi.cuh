// gemm_epi.cuh — fused GEMM epilogues for 16 output columns of one accumulator row (tcgen05 GEMMs).
#pragma once

#include "ctx.h"
#include "tc_common.cuh"

namespace gepi {
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ void st_bf16x16(bf16* p, const float* o) {
  uint4 w0, w1;
  w0.x = pack_bf16(o[0], o[1]); w0.y = pack_bf16(o[2], o[3]); w0.z = pack_bf16(o[4], o[5]); w0.w = pack_bf16(o[6], o[7]);
  w1.x = pack_bf16(o[8], o[9]); w1.y = pack_bf16(o[10], o[11]); w1.z = pack_bf16(o[12], o[13]);
  w1.w = pack_bf16(o[14], o[15]);
  reinterpret_cast<uint4*>(p)[0] = w0;
  reinterpret_cast<uint4*>(p)[1] = w1;
}

// sum over 16 columns of (x - ref)^2, ref = 16 bf16 at p (fused Delta_kv, R1)
__device__ __forceinline__ float sqdiff16(const float* x, const bf16* p) {
  const uint4* q = reinterpret_cast<const uint4*>(p);
  const uint4 r0 = __ldg(q), r1 = __ldg(q + 1);
  const uint32_t w[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[i]));
    const float d0 = x[2 * i] - f.x, d1 = x[2 * i + 1] - f.y;
    s += d0 * d0 + d1 * d1;
  }
  return s;
}

// Fused RMSNorm consumer: the per-row factor 1 / sqrt(mean(h^2) + eps) from the producer's 64-column
// sum-of-squares blocks, summed in block order (1 when the fusion is off).
__device__ __forceinline__ float row_rs(const EpiParams& e, int m, bool row_ok) {
  if (e.ss_in == nullptr || !row_ok) return 1.f;
  const float4* p = reinterpret_cast<const float4*>(e.ss_in + (size_t)m * e.ld_ss);
  float s = 0.f;
  for (int b = 0; b < e.ld_ss / 4; ++b) {
    const float4 v = p[b];
    s += v.x; s += v.y; s += v.z; s += v.w;
  }
  return 1.0f / sqrtf(s / (float)e.norm_d + e.norm_eps);
}

// Epilogue for 16 consecutive output columns n..n+15 of row m (all < N; N % 16 == 0). For EPI_QKV
// with fused deviation it returns this chunk's squared distance to the cached K/V row.
template <int KIND>
__device__ __forceinline__ float epi16(const EpiParams& e, int m, int n, const float* v, const float* u) {
  float o[16];
  float dev = 0.f;
  if constexpr (KIND == EPI_STORE) {
    st_bf16x16(reinterpret_cast<bf16*>(e.out) + (size_t)m * e.ldo + n, v);
  } else if constexpr (KIND == EPI_STORE_F32) {
    float4* p = reinterpret_cast<float4*>(out_row_f32(e, e.outf, m) + n);
#pragma unroll
    for (int i = 0; i < 4; ++i) p[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
  } else if constexpr (KIND == EPI_QKV) {
    const int c = e.col0 + n;
    if (c < e.qd + e.kvd) {  // q or k head: rotate pairs (2i, 2i+1) at the row's global position
      const int dim = (c < e.qd ? c : c - e.qd) % e.hd;
      const int p = epi_pos(e, __ldg(e.row_tok + m));
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
      if (c >= e.qd && e.dev_part != nullptr && m < e.n_cand)
        dev = sqdiff16(o, reinterpret_cast<const bf16*>(e.k_ref) + (size_t)__ldg(e.row_tok + m) * e.kvd + (c - e.qd));
    } else {
      st_bf16x16(reinterpret_cast<bf16*>(e.v_out) + (size_t)m * e.kvd + (c - e.qd - e.kvd), v);
      if (e.dev_part != nullptr && m < e.n_cand)
        dev = sqdiff16(v, reinterpret_cast<const bf16*>(e.v_ref) + (size_t)__ldg(e.row_tok + m) * e.kvd +
                              (c - e.qd - e.kvd));
    }
  } else if constexpr (KIND == EPI_RESID) {
    const int src = e.res_row ? __ldg(e.res_row + m) : m;
    const float4* hi = reinterpret_cast<const float4*>(e.h_in + (size_t)src * e.ldo + n);
    float4* ho = reinterpret_cast<float4*>(out_row_f32(e, e.h_out, m) + n);
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
  return dev;
}

// ---- coalesced tile epilogue ------------------------------------------------------------------------
// tcgen05.ld 32x32b hands each lane one accumulator row, so storing straight from registers makes every
// warp instruction touch 32 rows (32 L1 wavefronts). Instead each warp stages 32 rows x 32 fp32 columns
// in shared memory and re-reads them 4 rows per instruction (8 lanes x 16 B = 128 B of one row), so
// global loads and stores of the epilogue are row-contiguous. Float4 slots are XOR-swizzled by row:
// both the row-per-lane writes and the 4-rows-per-instruction reads are bank-conflict free.
constexpr int EPI_WARP_F4 = 32 * 8;  // float4 slots per warp buffer (4 KB)
#ifndef CB_STAGED_KINDS
#define CB_STAGED_KINDS ((1 << EPI_STORE) | (1 << EPI_STORE_F32) | (1 << EPI_RESID))
#endif
// epilogue kinds that take the staged (row-contiguous) path
template <int KIND> constexpr bool staged_kind() { return (CB_STAGED_KINDS >> KIND) & 1; }

// Explicit shared-memory accesses (st.shared / ld.shared on the 32-bit shared address): through the generic
// float4 pointer the compiler emitted generic ST.E / LD.E, which it must order against the epilogue's
// global stores -- measured ~1.5 us per 32-column chunk instead of ~0.2 us (tools/gemm_trace.py, r02d).
__device__ __forceinline__ void stage_put(float4* buf, int lane, const float* v) {
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(buf);
#pragma unroll
  for (int j = 0; j < 8; ++j)
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(base + (uint32_t)(lane * 8 + (j ^ (lane & 7))) * 16u),
                 "f"(v[4 * j]), "f"(v[4 * j + 1]), "f"(v[4 * j + 2]), "f"(v[4 * j + 3])
                 : "memory");
}
__device__ __forceinline__ float4 stage_get(const float4* buf, int r, int j) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(buf) + (uint32_t)(r * 8 + (j ^ (r & 7))) * 16u;
  float4 x;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w) : "r"(a) : "memory");
  return x;
}

__device__ __forceinline__ uint2 pack4_bf16(float4 a) { return make_uint2(pack_bf16(a.x, a.y), pack_bf16(a.z, a.w)); }

// Epilogue of one warp's 32 accumulator rows (tile rows m_base .. m_base + 31, TMEM address trow) over
// the tile's output columns n0 .. n0 + OUT_N. Lane L owns, in pass it = 0..7, row it * 4 + L / 8 and
// columns 4 * (L % 8) .. +3 of each 32-column chunk. cont (EPI_RESID only): a later split-K piece,
// h_out += acc. EPI_QKV needs hd % 32 == 0 (a chunk lies in one head); per-head deviation partials
// are summed per row over the head's chunks in order (each chunk: 4 terms per lane, then a fixed
// xor-shuffle tree over the row's 8 lanes).
template <int KIND, int BN>
__device__ __forceinline__ void tile_epilogue(const EpiParams& e, int M, int m_base, int n0, uint32_t trow,
                                              float4* buf, int lane, bool cont, bool last = true,
                                              long long* dbg = nullptr) {
  constexpr bool SW = KIND == EPI_SWIGLU;
  constexpr int OUT_N = SW ? BN / 2 : BN;
  const int j = lane & 7, r0 = lane >> 3;
  const int my_m = m_base + lane;
  const bool my_ok = my_m < M;
  const float my_rs = (KIND == EPI_QKV || KIND == EPI_SWIGLU) ? row_rs(e, my_m, my_ok) : 1.f;
  // fused RMSNorm producer (EPI_RESID, final split only): y = bf16(h_out * gain), 64-column sums of h_out^2
  [[maybe_unused]] const bool norm_on = KIND == EPI_RESID && e.norm_gain != nullptr && last;
  int my_a = 0, my_b = 0;  // per-row operands of the lane's own row, broadcast below
  if constexpr (KIND == EPI_RESID) {
    if (my_ok) my_a = cont ? my_m : (e.res_row ? __ldg(e.res_row + my_m) : my_m);
  }
  if constexpr (KIND == EPI_QKV) {
    if (my_ok) { my_a = __ldg(e.row_tok + my_m); my_b = epi_pos(e, my_a); }
  }
  int ra[8], rb[8];
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    ra[it] = __shfl_sync(0xffffffffu, my_a, it * 4 + r0);
    rb[it] = __shfl_sync(0xffffffffu, my_b, it * 4 + r0);
  }
  float dacc[8];  // EPI_QKV: per-row deviation of the current head; EPI_RESID + norm: sum of squares
#pragma unroll
  for (int it = 0; it < 8; ++it) dacc[it] = 0.f;
#pragma unroll 1
  for (int c = 0; c < OUT_N; c += 32) {
    const int n = n0 + c;
    if (n >= e.N) break;  // warp-uniform
    const int col = n + 4 * j;
    const bool col_ok = col < e.N;
    // 1. global operands first (their latency overlaps the TMEM read)
    float4 pre[8];
    uint2 ref[8];
    [[maybe_unused]] bool is_q = false, is_v = false, dev_on = false;
    [[maybe_unused]] int qc = 0, kv_c = 0;
    if constexpr (KIND == EPI_RESID) {
      const float* base = cont ? e.h_out : e.h_in;
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const int m = m_base + it * 4 + r0;
        pre[it] = make_float4(0.f, 0.f, 0.f, 0.f);
#if defined(CB_EPI_EXP) && (CB_EPI_EXP & 8)
        if (m < M && col_ok && e.ldo < 0) {  // experiment: no residual loads
#else
        if (m < M && col_ok) {
#endif
          const float4* p = reinterpret_cast<const float4*>(base + (size_t)ra[it] * e.ldo + col);
          pre[it] = cont ? __ldcg(p) : *p;
        }
      }
    }
    if constexpr (KIND == EPI_QKV) {
      qc = e.col0 + n;  // column of the fused [q | k | v] output
      is_q = qc < e.qd;
      is_v = qc >= e.qd + e.kvd;
      kv_c = is_q ? 0 : (is_v ? qc - e.qd - e.kvd : qc - e.qd);
      dev_on = !is_q && e.dev_part != nullptr;
      const int dim = ((is_q ? qc : qc - e.qd) % e.hd) + 4 * j;  // even: pairs (dim, dim+1), (dim+2, dim+3)
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const int m = m_base + it * 4 + r0;
        if (m < M && col_ok) {
          if (!is_v) pre[it] = __ldg(reinterpret_cast<const float4*>(e.rope_tab + (size_t)rb[it] * (e.hd >> 1) + (dim >> 1)));
          if (dev_on && m < e.n_cand)
            ref[it] = __ldg(reinterpret_cast<const uint2*>(reinterpret_cast<const bf16*>(is_v ? e.v_ref : e.k_ref) +
                                                           (size_t)ra[it] * e.kvd + kv_c + 4 * j));
        }
      }
    }
    // 2. TMEM -> registers (fused SwiGLU) -> staging buffer
    {
      float v[32];
#if defined(CB_EPI_EXP) && (CB_EPI_EXP & 1)
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = (float)i;
#else
      tc::tmem_ld32(trow + c, v);
#endif
      if constexpr (KIND == EPI_QKV) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] *= my_rs;
      }
      if constexpr (SW) {
        float u[32];
        tc::tmem_ld32(trow + BN / 2 + c, u);
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float g = v[i] * my_rs;
          v[i] = g / (1.f + __expf(-g)) * (u[i] * my_rs);
        }
      }
#if defined(CB_EPI_EXP) && (CB_EPI_EXP & 2)
      if (v[0] == 12345.f) stage_put(buf, lane, v);
#else
      stage_put(buf, lane, v);
#endif
    }
    __syncwarp();
    // 3. row-contiguous global traffic
    [[maybe_unused]] float4 gain = make_float4(0.f, 0.f, 0.f, 0.f);
    if constexpr (KIND == EPI_RESID) {
      if (norm_on && col_ok) gain = __ldg(reinterpret_cast<const float4*>(e.norm_gain + col));
    }
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      const int r = it * 4 + r0, m = m_base + r;
#if defined(CB_EPI_EXP) && (CB_EPI_EXP & 4)
      const bool ok = false;
#elif defined(CB_EPI_EXP) && (CB_EPI_EXP & 16)
      const bool ok = m < M && col_ok && e.ldo < 0;  // experiment: no stores (loads stay live)
#else
      const bool ok = m < M && col_ok;
#endif
      float4 a = stage_get(buf, r, j);
      if constexpr (KIND == EPI_STORE) {
        if (ok) *reinterpret_cast<uint2*>(reinterpret_cast<bf16*>(e.out) + (size_t)m * e.ldo + col) = pack4_bf16(a);
      } else if constexpr (KIND == EPI_STORE_F32) {
        if (ok) *reinterpret_cast<float4*>(out_row_f32(e, e.outf, m) + col) = a;
      } else if constexpr (KIND == EPI_SWIGLU) {
        if (ok) *reinterpret_cast<uint2*>(reinterpret_cast<bf16*>(e.act) + (size_t)m * e.ff + col) = pack4_bf16(a);
      } else if constexpr (KIND == EPI_RESID) {
        const float4 o = make_float4(pre[it].x + a.x, pre[it].y + a.y, pre[it].z + a.z, pre[it].w + a.w);
        if (ok) *reinterpret_cast<float4*>(out_row_f32(e, e.h_out, m) + col) = o;
        if (norm_on && ok) {  // lane-local sum of squares; reduced over the row's 8 lanes at the block end
          *reinterpret_cast<uint2*>(reinterpret_cast<bf16*>(e.y_out) + (size_t)m * e.ldo + col) =
              pack4_bf16(make_float4(o.x * gain.x, o.y * gain.y, o.z * gain.z, o.w * gain.w));
          dacc[it] += (o.x * o.x + o.y * o.y) + (o.z * o.z + o.w * o.w);
        }
      } else if constexpr (KIND == EPI_QKV) {
        if (ok && !is_v) {  // rotate pairs (dim, dim+1), (dim+2, dim+3) at the row's global position
          const float4 t = pre[it];
          a = make_float4(t.x * a.x - t.y * a.y, t.y * a.x + t.x * a.y, t.z * a.z - t.w * a.w, t.w * a.z + t.z * a.w);
        }
        if (ok) {
          bf16* dst = is_q ? reinterpret_cast<bf16*>(e.q_out) + (size_t)m * e.qd + qc + 4 * j
                           : reinterpret_cast<bf16*>(is_v ? e.v_out : e.k_out) + (size_t)m * e.kvd + kv_c + 4 * j;
          *reinterpret_cast<uint2*>(dst) = pack4_bf16(a);
        }
        if (dev_on) {  // warp-uniform
          float d = 0.f;
          if (ok && m < e.n_cand) {
            const float2 f0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ref[it].x));
            const float2 f1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ref[it].y));
            const float d0 = a.x - f0.x, d1 = a.y - f0.y, d2 = a.z - f1.x, d3 = a.w - f1.y;
            d = (d0 * d0 + d1 * d1) + (d2 * d2 + d3 * d3);
          }
          d += __shfl_xor_sync(0xffffffffu, d, 1);
          d += __shfl_xor_sync(0xffffffffu, d, 2);
          d += __shfl_xor_sync(0xffffffffu, d, 4);
          dacc[it] += d;
        }
      }
    }
    if constexpr (KIND == EPI_RESID) {
      if (norm_on && ((n + 32) % 64 == 0 || c + 32 >= OUT_N)) {  // a 64-column block ends: publish
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          float sq = dacc[it];  // fixed xor tree over the row's 8 lanes
          sq += __shfl_xor_sync(0xffffffffu, sq, 1);
          sq += __shfl_xor_sync(0xffffffffu, sq, 2);
          sq += __shfl_xor_sync(0xffffffffu, sq, 4);
          const int m = m_base + it * 4 + r0;
          if (j == 0 && m < M) e.ss_out[(size_t)m * e.ld_ss + n / 64] = sq;
          dacc[it] = 0.f;
        }
      }
    }
    if constexpr (KIND == EPI_QKV) {
      if (dev_on && (qc + 32) % 64 == 0) {  // a 64-column k or v block ends with this chunk: publish it
        const int slot = 2 * (kv_c / 64) + (is_v ? 1 : 0);
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          const int m = m_base + it * 4 + r0;
          if (j == 0 && m < M && m < e.n_cand) e.dev_part[(size_t)slot * e.ld_part + m] = dacc[it];
          dacc[it] = 0.f;
        }
      }
    }
    __syncwarp();  // buffer reused by the next chunk
    if (dbg != nullptr && lane == 0 && c / 32 < 8) dbg[c / 32] = tc::globaltimer();
  }
}

// ---- lean residual epilogue ---------------------------------------------------------------------------
// EPI_RESID without a peer push (the blend's o_proj / down_proj, every piece of a k-split chain):
// the same staged row-contiguous traffic and the same arithmetic (bitwise equal to tile_epilogue), but
// the per-row operands (validity, source / destination row offsets) are computed once per tile and the
// cold paths are gone, so the unrolled chunk loop is compact. tools/gemm_trace.py (r02g): the generic
// loop spent ~0.64 us per 32-column chunk even with every global access compiled out (instruction
// fetch of the long unrolled body with per-row branches), ~1.3 us with its traffic.
// Needs e.N % 32 == 0 and 32-bit row offsets ((M + 256) * ldo < 2^31).
template <int BN, bool NORM>
__device__ __forceinline__ void resid_lean(const EpiParams& e, int M, int m_base, int n0, uint32_t trow, float4* buf,
                                           int lane, long long* dbg = nullptr, bool cont = false) {
  // cont: a later piece of a k-split chain adds onto the running sum in h_out (rows in place, read past L1)
  const int j = lane & 7, r0 = lane >> 3;
  const int my_m = m_base + lane;
  const int my_src = my_m < M ? (cont ? my_m : (e.res_row ? __ldg(e.res_row + my_m) : my_m)) : 0;
  const float* base = cont ? e.h_out : e.h_in;
  unsigned okmask = 0;
  int in_off[8], out_off[8];  // element offsets of the rows this lane touches (it * 4 + r0)
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    const int m = m_base + it * 4 + r0;
    const int src = __shfl_sync(0xffffffffu, my_src, it * 4 + r0);
    okmask |= (m < M ? 1u : 0u) << it;
    in_off[it] = src * e.ldo + 4 * j;
    out_off[it] = m * e.ldo + 4 * j;
  }
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(buf);
  float dacc[8];
#pragma unroll
  for (int it = 0; it < 8; ++it) dacc[it] = 0.f;
#pragma unroll 1
  for (int c = 0; c < BN; c += 32) {
    const int n = n0 + c;
    if (n >= e.N) break;  // warp-uniform
    float4 pre[8];
#pragma unroll
    for (int it = 0; it < 8; ++it)
      pre[it] = ((okmask >> it) & 1) ? (cont ? __ldcg(reinterpret_cast<const float4*>(base + in_off[it] + n))
                                            : *reinterpret_cast<const float4*>(base + in_off[it] + n))
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
    const bool more = c + 32 < BN && n + 32 < e.N;  // warp-uniform
    {
      float v[32];
      tc::tmem_ld32(trow + c, v);
#pragma unroll
      for (int q = 0; q < 8; ++q)
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(sbase + (uint32_t)(lane * 8 + (q ^ (lane & 7))) * 16u),
                     "f"(v[4 * q]), "f"(v[4 * q + 1]), "f"(v[4 * q + 2]), "f"(v[4 * q + 3])
                     : "memory");
    }
    __syncwarp();
    [[maybe_unused]] float4 gain = make_float4(0.f, 0.f, 0.f, 0.f);
    if constexpr (NORM) gain = __ldg(reinterpret_cast<const float4*>(e.norm_gain + n + 4 * j));
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      const int r = it * 4 + r0;
      float4 a;
      asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                   : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w)
                   : "r"(sbase + (uint32_t)(r * 8 + (j ^ (r & 7))) * 16u)
                   : "memory");
      const float4 o = make_float4(pre[it].x + a.x, pre[it].y + a.y, pre[it].z + a.z, pre[it].w + a.w);
      // the next chunk's residual segment of this row pulled into L1 while this chunk is stored (no registers)
      if (e.l1pf && j == 0 && more && !cont && ((okmask >> it) & 1))  // one lane per 128-byte row segment
        asm volatile("prefetch.global.L1 [%0];" ::"l"(base + in_off[it] + n + 32));
      if ((okmask >> it) & 1) {
        *reinterpret_cast<float4*>(e.h_out + out_off[it] + n) = o;
        if constexpr (NORM) {
          *reinterpret_cast<uint2*>(reinterpret_cast<bf16*>(e.y_out) + out_off[it] + n) =
              pack4_bf16(make_float4(o.x * gain.x, o.y * gain.y, o.z * gain.z, o.w * gain.w));
          dacc[it] += (o.x * o.x + o.y * o.y) + (o.z * o.z + o.w * o.w);
        }
      }
    }
    if constexpr (NORM) {
      if ((n + 32) % 64 == 0 || c + 32 >= BN) {  // a 64-column block ends: publish (same tree as tile_epilogue)
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          float sq = dacc[it];
          sq += __shfl_xor_sync(0xffffffffu, sq, 1);
          sq += __shfl_xor_sync(0xffffffffu, sq, 2);
          sq += __shfl_xor_sync(0xffffffffu, sq, 4);
          if (j == 0 && ((okmask >> it) & 1)) e.ss_out[(size_t)(m_base + it * 4 + r0) * e.ld_ss + n / 64] = sq;
          dacc[it] = 0.f;
        }
      }
    }
    __syncwarp();  // buffer reused by the next chunk
    if (dbg != nullptr && lane == 0 && c / 32 < 8) dbg[c / 32] = tc::globaltimer();
  }
}

// Whether a RESID tile may take resid_lean (else the generic tile_epilogue).
__device__ __forceinline__ bool resid_lean_ok(const EpiParams& e, int M) {
  return e.push_base[0] == nullptr && (e.N % 32) == 0 &&
         (long long)(M + 256) * e.ldo < (1ll << 31);
}

// ---- row-per-lane QKV epilogue with operands issued early -----------------------------------------
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {  // bulk L2 prefetch (16 B multiple)
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Called by each epilogue lane for its own tile row before the accumulator is ready (the mainloop is
// still running): pulls the row's cached K/V reference segment and RoPE table row into L2.
__device__ __forceinline__ void qkv_prefetch(const EpiParams& e, int m, bool row_ok, int n0, int out_n) {
  if (!row_ok) return;
  const int tok = __ldg(e.row_tok + m);
  const int c0 = e.col0 + n0;
  const int c1 = min(e.col0 + e.N, c0 + out_n);  // exclusive
  if (c0 < e.qd + e.kvd) {  // rope row (cos, sin of all pairs) at the row's position
    const int p = epi_pos(e, tok);
    prefetch_l2(e.rope_tab + (size_t)p * (e.hd >> 1), (uint32_t)(e.hd >> 1) * 8u);
  }
  if (e.dev_part != nullptr && m < e.n_cand && c1 > e.qd) {
    const int a = max(c0, e.qd);
    if (a < e.qd + e.kvd) {
      const int b = min(c1, e.qd + e.kvd);
      prefetch_l2(reinterpret_cast<const bf16*>(e.k_ref) + (size_t)tok * e.kvd + (a - e.qd), (uint32_t)(b - a) * 2u);
    }
    const int av = max(c0, e.qd + e.kvd);
    if (av < c1)
      prefetch_l2(reinterpret_cast<const bf16*>(e.v_ref) + (size_t)tok * e.kvd + (av - e.qd - e.kvd),
                  (uint32_t)(c1 - av) * 2u);
  }
}

// EPI_RESID: pull the row's residual segment into L2 while the mainloop runs.
__device__ __forceinline__ void resid_prefetch(const EpiParams& e, int m, bool row_ok, int n0, int out_n) {
  if (!row_ok) return;
  const int src = e.res_row ? __ldg(e.res_row + m) : m;
  const int w = min(out_n, e.N - n0);
  if (w > 0) prefetch_l2(e.h_in + (size_t)src * e.ldo + n0, (uint32_t)w * 4u);
}

// EPI_QKV on 32 accumulator columns [n, n + 32) of row m (hd % 32 == 0: the chunk lies in one q, k or
// v head). Warp-collective. RoPE (cos, sin) and the cached K/V reference are loaded before the TMEM
// read, so one (L2) latency is exposed per chunk. Returns the chunk's squared distance to the reference
// (0 for q columns and non-candidates). tok = row_tok[m], p = pos[tok]. 32 columns rather than 64 keep
// the kernel free of register spills (ptxas: 744-964 B of spills at 64).
__device__ __forceinline__ float qkv32(const EpiParams& e, int m, int n, bool row_ok, uint32_t taddr, int tok, int p,
                                       float rs) {
  const int c = e.col0 + n;
  const bool is_q = c < e.qd, is_v = c >= e.qd + e.kvd;
  const bool dev_on = row_ok && !is_q && e.dev_part != nullptr && m < e.n_cand;
  const int kv_c = is_q ? 0 : (is_v ? c - e.qd - e.kvd : c - e.qd);
  float4 cs[8];
  uint4 ref[4];
  if (row_ok && !is_v) {
    const int dim = (is_q ? c : c - e.qd) % e.hd;
    const float4* t = reinterpret_cast<const float4*>(e.rope_tab + (size_t)p * (e.hd >> 1) + (dim >> 1));
#pragma unroll
    for (int i = 0; i < 8; ++i) cs[i] = __ldg(t + i);  // (cos, sin) of pairs 2i, 2i+1
  }
  if (dev_on) {
    const uint4* r = reinterpret_cast<const uint4*>(reinterpret_cast<const bf16*>(is_v ? e.v_ref : e.k_ref) +
                                                    (size_t)tok * e.kvd + kv_c);
#pragma unroll
    for (int i = 0; i < 4; ++i) ref[i] = __ldg(r + i);
  }
  float x[32];
  tc::tmem_ld32(taddr, x);
  if (!row_ok) return 0.f;
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] *= rs;
  if (!is_v) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float a0 = x[4 * i], a1 = x[4 * i + 1], b0 = x[4 * i + 2], b1 = x[4 * i + 3];
      x[4 * i] = cs[i].x * a0 - cs[i].y * a1;
      x[4 * i + 1] = cs[i].y * a0 + cs[i].x * a1;
      x[4 * i + 2] = cs[i].z * b0 - cs[i].w * b1;
      x[4 * i + 3] = cs[i].w * b0 + cs[i].z * b1;
    }
  }
  float dev = 0.f;
  if (dev_on) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t wv[4] = {ref[i].x, ref[i].y, ref[i].z, ref[i].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wv[j]));
        const float d0 = x[8 * i + 2 * j] - f.x, d1 = x[8 * i + 2 * j + 1] - f.y;
        dev += d0 * d0 + d1 * d1;
      }
    }
  }
  bf16* dst = is_q ? reinterpret_cast<bf16*>(e.q_out) + (size_t)m * e.qd + c
                   : reinterpret_cast<bf16*>(is_v ? e.v_out : e.k_out) + (size_t)m * e.kvd + kv_c;
#pragma unroll
  for (int g = 0; g < 2; ++g) st_bf16x16(dst + 16 * g, x + 16 * g);
  return dev;
}

// Whole-row QKV epilogue over OUT_N accumulator columns from output column n0 (hd % 64 == 0):
// 64-column chunks; each k/v chunk's deviation partial goes to its own slot (summed in order by top-k).
template <int OUT_N>
__device__ __forceinline__ void qkv_row(const EpiParams& e, int m, bool row_ok, int n0, uint32_t trow, float rs) {
  int tok = 0, p = 0;
  if (row_ok) {
    tok = __ldg(e.row_tok + m);
    p = epi_pos(e, tok);
  }
  float dacc = 0.f;
#pragma unroll 1
  for (int c = 0; c < OUT_N; c += 32) {
    const int n = n0 + c;
    if (n >= e.N) break;  // warp-uniform
    dacc += qkv32(e, m, n, row_ok, trow + c, tok, p, rs);
    const int cl = e.col0 + n;
    if ((cl + 32) % 64 != 0) continue;  // the 64-column block continues in the next chunk
    if (e.dev_part != nullptr && cl >= e.qd) {  // one partial per 64-column k or v block
      const int kv_col = cl - e.qd;
      const int slot = kv_col < e.kvd ? 2 * (kv_col / 64) : 2 * ((kv_col - e.kvd) / 64) + 1;
      if (row_ok && m < e.n_cand) e.dev_part[(size_t)slot * e.ld_part + m] = dacc;
      dacc = 0.f;
    }
  }
}

// ---- K-piece merge (tail pieces of a pair GEMM, blocks of the fused MLP) -----------------------------
// Piece p's fp32 partial of this CTA's 128 x BN accumulator lives at base + p * pstride in the layout
// [BN / 4 column groups][128 rows][4] (a warp's 32 rows of a group = 512 contiguous bytes). The merge
// sums the np <= MAXP pieces in piece order (deterministic) into the TMEM accumulator row trow. Loads of
// the next 16-column group are in flight while the current one is summed and stored.
template <int BN, int MAXP>
__device__ __forceinline__ void merge_pieces_to_tmem(const float* base, size_t pstride, int np, int row, uint32_t trow) {
  float4 cur[MAXP][4], nxt[MAXP][4];
  auto load = [&](float4 (&dst)[MAXP][4], int c) {
#pragma unroll
    for (int p = 0; p < MAXP; ++p) {
      if (p < np) {
        const float4* src = reinterpret_cast<const float4*>(base + p * pstride) + (size_t)(c / 4) * 128 + row;
#pragma unroll
        for (int x = 0; x < 4; ++x) dst[p][x] = __ldcg(src + x * 128);
      }
    }
  };
  load(cur, 0);
#pragma unroll
  for (int c = 0; c < BN; c += 16) {
    if (c + 16 < BN) load(nxt, c + 16);
    float v[16];
#pragma unroll
    for (int x = 0; x < 16; ++x) v[x] = 0.f;
#pragma unroll
    for (int p = 0; p < MAXP; ++p) {
      if (p < np) {
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          v[4 * x] += cur[p][x].x; v[4 * x + 1] += cur[p][x].y; v[4 * x + 2] += cur[p][x].z; v[4 * x + 3] += cur[p][x].w;
        }
      }
    }
    tc::tmem_st16(trow + c, v);
#pragma unroll
    for (int p = 0; p < MAXP; ++p)
#pragma unroll
      for (int x = 0; x < 4; ++x) cur[p][x] = nxt[p][x];
  }
  tc::tmem_st_wait();
}

}  // namespace gepi
