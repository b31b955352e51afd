// Throughput of MUFU.EX2 vs FFMA per SM on this GPU (tuning input for the attention softmax).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mufu tools/micro/mufu_bench.cu && /tmp/mufu
#include <cstdint>
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
      else if (MODE == 1) x[i] = fmaf(x[i], 0.999f, -0.001f);
      else if (MODE == 2) {  // packed bf16x2 conversion (the softmax's P pack), result fed back
        uint32_t u;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u) : "f"(x[i]), "f"(x[(i + 1) & 7]));
        x[i] = __uint_as_float(u & 0x7fff7fffu) ;
      } else {  // exp2 emulated on the FMA/ALU pipes (Cody-Waite split + degree-3 polynomial)
        const float t = fmaxf(x[i], -126.f);
        const float r = t + 12582912.f;
        const float j = r - 12582912.f;
        const float f = t - j;
        float p = fmaf(fmaf(fmaf(0.0555041f, f, 0.2402265f), f, 0.6931472f), f, 1.0f);
        x[i] = __int_as_float(__float_as_int(p) + ((__float_as_int(r) - 0x4B400000) << 23)) - 1.5f;
      }
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
  const char* names[4] = {"ex2.approx", "ffma", "cvt.bf16x2", "ex2 poly (FMA pipe)"};
  for (int mode = 0; mode < 4; ++mode) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<blocks, threads>>>(d, iters, 1.f);
      else if (mode == 1) k<1><<<blocks, threads>>>(d, iters, 1.f);
      else if (mode == 2) k<2><<<blocks, threads>>>(d, iters, 1.f);
      else k<3><<<blocks, threads>>>(d, iters, 1.f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = (double)blocks * threads * iters * 8;
    printf("%s: %.3f ms, %.1f Gop/s, %.1f ops/clk/SM at %.0f MHz nominal\n", names[mode], ms,
           ops / ms * 1e-6, ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1e3);
  }
  return 0;
}
