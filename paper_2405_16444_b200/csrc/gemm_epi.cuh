// gemm_epi.cuh — fused GEMM epilogues for 16 output columns of one accumulator row (tcgen05 GEMMs).
#pragma once

#include "ctx.h"

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

// Epilogue for 16 consecutive output columns n..n+15 of row m (all < N; N % 16 == 0). For EPI_QKV
// with fused deviation it returns this chunk's squared distance to the cached K/V row.
template <int KIND>
__device__ __forceinline__ float epi16(const EpiParams& e, int m, int n, const float* v, const float* u) {
  float o[16];
  float dev = 0.f;
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
  return dev;
}

}  // namespace gepi
