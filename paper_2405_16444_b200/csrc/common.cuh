// common.cuh — shared device/host definitions for libcacheblend (sm_100a only).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/cacheblend.h"
#include "../../include/cacheblend_ops.h"

typedef __nv_bfloat16 bf16;

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "libcacheblend is built for sm_100a only (-gencode arch=compute_100a,code=sm_100a)"
#endif

// ---- scalar conversions ------------------------------------------------------------------------
template <typename T> __device__ __forceinline__ float to_f(T x);
template <> __device__ __forceinline__ float to_f<float>(float x) { return x; }
template <> __device__ __forceinline__ float to_f<bf16>(bf16 x) { return __bfloat162float(x); }

template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ bf16 from_f<bf16>(float x) { return __float2bfloat16_rn(x); }

// 16-byte vector of T: 8 bf16 or 4 fp32.
template <typename T> struct Vec16 {
  static constexpr int N = 16 / sizeof(T);
  T v[N];
};

template <typename T> __device__ __forceinline__ Vec16<T> ld16(const T* p) {
  Vec16<T> r;
  *reinterpret_cast<uint4*>(&r) = __ldg(reinterpret_cast<const uint4*>(p));
  return r;
}
template <typename T> __device__ __forceinline__ Vec16<T> ld16_cg(const T* p) {
  Vec16<T> r;
  *reinterpret_cast<uint4*>(&r) = __ldcg(reinterpret_cast<const uint4*>(p));
  return r;
}
template <typename T> __device__ __forceinline__ void st16(T* p, const Vec16<T>& v) {
  *reinterpret_cast<uint4*>(p) = *reinterpret_cast<const uint4*>(&v);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ---- programmatic dependent launch -------------------------------------------------------------
// Every library kernel is launched with programmatic stream serialization. pdl_wait() blocks until the
// preceding kernel has completed and its memory is visible; pdl_trigger() lets the next kernel's CTAs
// be scheduled (its prologue then overlaps this kernel's tail). Triggering once every CTA of this grid
// is running cannot deadlock: the dependent grid launches only after all of this grid's CTAs executed
// the trigger, i.e. are resident.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_enter() {
  pdl_wait();
  pdl_trigger();
}

// Device-side error word bits (cb_check_device_errors).
enum : int { CB_DEVERR_FORCE_SEL = 1, CB_DEVERR_POS_RANGE = 2, CB_DEVERR_COMM = 4, CB_DEVERR_POS_ORDER = 8,
             CB_DEVERR_PAGE = 16 };

// ---- epilogues shared by the SIMT and tcgen05 GEMMs -----------------------------------------
// acc[m][n] = sum_k A[m][k] B[n][k];   kinds:
enum EpiKind : int {
  EPI_STORE = 0,     // out[m*ldo + n] = T(acc)
  EPI_STORE_F32 = 1, // outf[m*ldo + n] = acc
  EPI_QKV = 2,       // logical column c = col0 + n of [q | k | v]; RoPE on q,k at pos[row_tok[m]]
  EPI_RESID = 3,     // h_out[m][n] = h_in[res_row ? res_row[m] : m][n] + acc   (fp32)
  EPI_SWIGLU = 4     // GEMM over 2*ff "virtual" columns; act[m][f] = T(silu(gate) * up)
};

struct EpiParams {
  int kind;
  int M, N;                    // GEMM output extent (N = ff for SWIGLU)
  void* out; float* outf; int ldo;
  // EPI_QKV
  void* q_out; void* k_out; void* v_out;
  int col0, qd, kvd, hd;
  const int* row_tok; const int* pos; const float2* rope_tab; int max_pos;  // pos clamped to [0, max_pos)
  // EPI_QKV fused Delta_kv (tcgen05 path): for candidate rows m < n_cand, per 64-column block b of the
  // k (resp. v) row: dev_part[(2b + 0) * ld_part + m] = ||k_m[b] - k_ref[row_tok[m]][b]||^2, [(2b + 1) ...] v
  const void* k_ref; const void* v_ref; float* dev_part; int n_cand, ld_part;
  // EPI_RESID
  float* h_out; const float* h_in; const int* res_row;
  int l1pf;                    // lean residual epilogue: pull the next chunk's residual rows into L1 (cb_set_option "epi_l1pf")
  // EPI_SWIGLU
  int ff; void* act;
  // Fused RMSNorm (tcgen05 path; DESIGN R15). Producer (EPI_RESID with norm_gain set): besides h_out it writes
  // y[m][n] = bf16(h_out[m][n] * norm_gain[n]) and ss_out[m * ld_ss + n / 64] = the sum of h_out[m][n]^2
  // over each 64-column block (every GEMM tile edge is a block edge). Consumer (EPI_QKV / EPI_SWIGLU with ss_in set, A operand = y): every
  // accumulator of row m is scaled by rs_m = 1 / sqrt(sum_b ss_in[m * ld_ss + b] / norm_d + norm_eps)
  // (blocks summed in order) -- RMSNorm's per-row factor taken out of the projection.
  const float* norm_gain; void* y_out; float* ss_out;
  const float* ss_in; int ld_ss, norm_d; float norm_eps;
  // Head-parallel fused reduce-scatter (comm.cu): when push_base[0] is set, the fp32 output row m of
  // EPI_STORE_F32 / EPI_RESID goes to push_base[m / push_rows] + push_off (this rank's receive plane in the
  // block of the rank that owns row m, over NVLink) instead of outf / h_out.
  char* push_base[8]; long long push_off; int push_rows;
};
// Global position of token `tok` for the RoPE table, clamped so that a position outside [0, max_pos) cannot
// read past the table (pos_check_kernel reports it through the device error word, CB_DEVERR_POS_RANGE).
__device__ __forceinline__ int epi_pos(const EpiParams& e, int tok) {
  return min(max(__ldg(e.pos + tok), 0), e.max_pos - 1);
}


// Output row m of an fp32 epilogue (outf / h_out), or its owner's receive plane when pushing.
__device__ __forceinline__ float* out_row_f32(const EpiParams& e, float* local, int m) {
  if (e.push_base[0] != nullptr)
    return reinterpret_cast<float*>(e.push_base[m / e.push_rows] + e.push_off) + (size_t)m * e.ldo;
  return local + (size_t)m * e.ldo;
}

// Apply the epilogue to the adjacent column pair (n, n+1), n even. For SWIGLU a0/a1 are the gate
// accumulators and u0/u1 the up accumulators of output columns n, n+1.
template <typename T>
__device__ __forceinline__ void epi_pair(const EpiParams& e, int m, int n, float a0, float a1,
                                         float u0 = 0.f, float u1 = 0.f) {
  const bool has1 = (n + 1) < e.N;
  switch (e.kind) {
    case EPI_STORE: {
      T* o = reinterpret_cast<T*>(e.out) + (size_t)m * e.ldo + n;
      o[0] = from_f<T>(a0);
      if (has1) o[1] = from_f<T>(a1);
    } break;
    case EPI_STORE_F32: {
      float* o = out_row_f32(e, e.outf, m) + n;
      o[0] = a0;
      if (has1) o[1] = a1;
    } break;
    case EPI_QKV: {
      const int c = e.col0 + n;  // logical column in [q | k | v]
      if (c < e.qd + e.kvd) {    // q or k: rotate the pair (2i, 2i+1) of the head
        const int dim = (c < e.qd ? c : c - e.qd) % e.hd;
        const int p = epi_pos(e, e.row_tok[m]);
        const float2 cs = e.rope_tab[(size_t)p * (e.hd >> 1) + (dim >> 1)];
        const float r0 = cs.x * a0 - cs.y * a1;
        const float r1 = cs.y * a0 + cs.x * a1;
        T* o = (c < e.qd) ? reinterpret_cast<T*>(e.q_out) + (size_t)m * e.qd + c
                          : reinterpret_cast<T*>(e.k_out) + (size_t)m * e.kvd + (c - e.qd);
        o[0] = from_f<T>(r0);
        o[1] = from_f<T>(r1);
      } else {
        T* o = reinterpret_cast<T*>(e.v_out) + (size_t)m * e.kvd + (c - e.qd - e.kvd);
        o[0] = from_f<T>(a0);
        if (has1) o[1] = from_f<T>(a1);
      }
    } break;
    case EPI_RESID: {
      const int src = e.res_row ? e.res_row[m] : m;
      const float* hi = e.h_in + (size_t)src * e.ldo + n;
      float* ho = out_row_f32(e, e.h_out, m) + n;
      const float h0 = hi[0];
      const float h1 = has1 ? hi[1] : 0.f;
      ho[0] = h0 + a0;
      if (has1) ho[1] = h1 + a1;
    } break;
    case EPI_SWIGLU: {
      T* o = reinterpret_cast<T*>(e.act) + (size_t)m * e.ff + n;
      const float s0 = a0 / (1.f + expf(-a0));
      o[0] = from_f<T>(s0 * u0);
      if (has1) {
        const float s1 = a1 / (1.f + expf(-a1));
        o[1] = from_f<T>(s1 * u1);
      }
    } break;
  }
}
