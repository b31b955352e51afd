// Throughput of MUFU.EX2 vs FFMA per SM on this GPU (tuning input for the attention softmax).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mufu tools/micro/mufu_bench.cu && /tmp/mufu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, int iters, float a) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = a * (threadIdx.x + i) * 1e-6f - 1.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
      else x[i] = fmaf(x[i], 0.999f, -0.001f);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.f) out[0] = s;
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* d;
  cudaMalloc(&d, 4);
  const int iters = 4096, threads = 512, blocks = sms * 4;
  for (int mode = 0; mode < 2; ++mode) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<blocks, threads>>>(d, iters, 1.f); else k<1><<<blocks, threads>>>(d, iters, 1.f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = (double)blocks * threads * iters * 8;
    printf("%s: %.3f ms, %.1f Gop/s, %.1f ops/clk/SM at %.0f MHz nominal\n", mode == 0 ? "ex2.approx" : "ffma", ms,
           ops / ms * 1e-6, ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1e3);
  }
  return 0;
}
