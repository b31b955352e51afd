// gen.cu — device implementation of the synthetic-input counter RNG (synth/counter_rng.py spec).
// Input generation only: no CacheBlend arithmetic here.
#include "ctx.h"

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static unsigned long long mix64_host(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <typename T>
__global__ void gen_fill_kernel(T* __restrict__ out, long long count, unsigned long long base, long long start,
                                float scale, float offset) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long r = mix64(base + (unsigned long long)(start + i));
    const float u = __fsub_rn(__fmul_rn((float)(unsigned)(r >> 40), 1.1920928955078125e-07f), 1.0f);
    const float v = __fadd_rn(offset, __fmul_rn(u, scale));
    out[i] = from_f<T>(v);
  }
}

__global__ void gen_ints_kernel(int* __restrict__ out, long long count, unsigned long long base, long long start,
                                unsigned long long modulus) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x) {
    out[i] = (int)(mix64(base + (unsigned long long)(start + i)) % modulus);
  }
}

cb_status launch_gen_fill(void* out, int dtype, long long count, unsigned long long seed,
                          unsigned long long stream_id, long long start, float scale, float offset, cudaStream_t s) {
  if (count <= 0) return CB_OK;
  const unsigned long long base = mix64_host(mix64_host(seed) ^ stream_id);
  const int grid = (int)std::min<long long>((count + 255) / 256, 148LL * 16);
  if (dtype == CB_BF16)
    gen_fill_kernel<bf16><<<grid, 256, 0, s>>>((bf16*)out, count, base, start, scale, offset);
  else
    gen_fill_kernel<float><<<grid, 256, 0, s>>>((float*)out, count, base, start, scale, offset);
  CB_CUDA(cudaGetLastError());
  return CB_OK;
}

extern "C" cb_status cb_gen_fill(void* out, int32_t dtype, int64_t count, uint64_t seed, uint64_t stream_id,
                                 int64_t start, float scale, float offset, void* stream) {
  CB_REQUIRE(out != nullptr || count == 0, CB_E_INVALID_ARG, "cb_gen_fill: out is NULL");
  CB_REQUIRE(dtype == CB_BF16 || dtype == CB_FP32, CB_E_INVALID_ARG, "cb_gen_fill: bad dtype %d", dtype);
  return launch_gen_fill(out, dtype, count, seed, stream_id, start, scale, offset, (cudaStream_t)stream);
}

extern "C" cb_status cb_gen_ints(int32_t* out, int64_t count, uint64_t seed, uint64_t stream_id, int64_t start,
                                 int64_t modulus, void* stream) {
  CB_REQUIRE(modulus > 0, CB_E_INVALID_ARG, "cb_gen_ints: modulus must be > 0");
  if (count <= 0) return CB_OK;
  const unsigned long long base = mix64_host(mix64_host(seed) ^ stream_id);
  const int grid = (int)std::min<long long>((count + 255) / 256, 148LL * 16);
  gen_ints_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(out, count, base, start, (unsigned long long)modulus);
  CB_CUDA(cudaGetLastError());
  return CB_OK;
}
