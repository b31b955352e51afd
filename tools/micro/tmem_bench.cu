// TMEM read / write throughput per SM (tcgen05.ld / tcgen05.st 32x32b.x32), one CTA per SM, W warps
// (tuning input for the attention softmax, whose S tile is 128 rows x 128 fp32 = 64 KB of TMEM per key tile).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tmem tools/micro/tmem_bench.cu && /tmp/tmem
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

// MODE 0: ld x32 + wait each; 1: two ld x32 then one wait; 2: st x32 (+ wait::st every 2)
template <int MODE>
__global__ void k(unsigned* out, long long* cyc, int iters) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot + ((uint32_t)((warp & 3) * 32) << 16);
  const uint32_t cbase = (uint32_t)((warp >> 2) * 64) & 511u;
  uint32_t acc = 0, r[32], q[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) q[i] = threadIdx.x + i;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const uint32_t col = (cbase + (uint32_t)(it & 3) * 64u) & 511u;
    if (MODE == 0) {
      ld32(tmem + col, r);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < 32; ++i) acc += r[i];
    } else if (MODE == 1) {
      ld32(tmem + col, r);
      ld32(tmem + col + 32, q);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < 32; ++i) acc += r[i] ^ q[i];
    } else {
      st32(tmem + col, q);
      if (it & 1) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  __syncthreads();
  const long long t1 = clock64();
  if (acc == 0x12345678u) out[0] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* d;
  long long* cyc;
  cudaMalloc(&d, 4);
  cudaMalloc(&cyc, sms * 8);
  const int iters = 4096;
  const char* names[3] = {"ld x32 + wait", "2 x ld x32 + wait", "st x32"};
  for (int mode = 0; mode < 3; ++mode)
    for (int warps : {4, 8, 12}) {
      auto fn = mode == 0 ? k<0> : mode == 1 ? k<1> : k<2>;
      for (int rep = 0; rep < 2; ++rep) fn<<<sms, warps * 32>>>(d, cyc, iters);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      long long c0;
      cudaMemcpy(&c0, cyc, 8, cudaMemcpyDeviceToHost);
      const double bytes = (double)warps * 32 * 32 * 4 * iters * (mode == 1 ? 2 : 1);
      printf("%-18s warps %2d: %8.1f B/cycle/SM (%lld cycles for %.1f MB)\n", names[mode], warps, bytes / c0, c0,
             bytes / 1e6);
    }
  return 0;
}
