// Chip-wide L2 -> shared-memory TMA feed rate, by access pattern (tuning input for the GEMM: is the
// 148-SM mainloop bound by the L2 feed, and does cluster multicast raise it?).
//   mode 0: every CTA streams its own tiles (no two CTAs read the same tile at the same time)
//   mode 1: the CS CTAs of a cluster read the same tiles, each with its own unicast TMA
//   mode 2: the CS CTAs of a cluster read the same tiles, each CTA issues 1/CS of every tile with
//           .multicast::cluster to all CS CTAs
// Every CTA receives 32 KB per k-block (two 128 x 64 bf16 SW128 boxes, the pair GEMM's per-SM
// k-block), 6 stages in flight, no consumer. Source: 4096 x 4096 bf16 (32 MB, L2-resident).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_feed tools/micro/tma_feed.cu -lcuda && /tmp/tma_feed
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

constexpr int STAGES = 6, TILE = 32768, ROWS = 4096, COLS = 4096, KBS = COLS / 64;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  uint32_t done = 0;
  do {
    asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0,1,0,P;\n\t}"
                 : "=r"(done) : "r"(su32(b)), "r"(ph) : "memory");
  } while (!done);
}
__device__ __forceinline__ long long gtimer() { long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

template <int MODE, int CS>
__global__ void __launch_bounds__(32, 1) feed(const __grid_constant__ CUtensorMap tm, int iters, long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(sm + STAGES * TILE);
  uint64_t* empty = full + STAGES;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int cl = blockIdx.x / CS;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(MODE == 2 ? CS : 1));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  long long t0 = gtimer();
  if (threadIdx.x == 0) {
    const int who = MODE == 0 ? blockIdx.x : cl;
    const int row0 = (who * 256) % ROWS;
    const int kofs = (who * 7) % KBS;
    // prologue: fill STAGES
    for (int j = 0; j < iters + STAGES; ++j) {
      const int s = j % STAGES;
      if (j >= STAGES) {
        wait(&full[s], ((j - STAGES) / STAGES) & 1);
        if (MODE == 2) {
          // free this stage in every CTA of the cluster (each CTA's empty counts CS arrivals)
          for (int r = 0; r < CS; ++r) {
            uint32_t remote;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(su32(&empty[s])), "r"(r));
            asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
          }
        } else {
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
        }
      }
      if (j >= iters) continue;
      if (j >= STAGES) wait(&empty[s], ((j - STAGES) / STAGES) & 1);
      const int kb = (j + kofs) % KBS;
      uint8_t* dst = sm + s * TILE;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(TILE) : "memory");
      if (MODE != 2) {
        for (int h = 0; h < 2; ++h)
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
              ::"r"(su32(dst + h * 16384)), "l"((uint64_t)&tm), "r"(su32(&full[s])), "r"(kb * 64), "r"(row0 + h * 128)
              : "memory");
      } else {
        // this CTA's share: rows [rank * 256 / CS, (rank + 1) * 256 / CS) of the 256-row tile, in 32-row boxes
        const uint16_t mask = (uint16_t)((1u << CS) - 1);
        for (int b = rank * (8 / CS); b < (rank + 1) * (8 / CS); ++b)
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, %4}], [%2], %5;"
              ::"r"(su32(dst + b * 4096)), "l"((uint64_t)&tm), "r"(su32(&full[s])), "r"(kb * 64), "r"(row0 + b * 32), "h"(mask)
              : "memory");
      }
    }
  }
  long long t1 = gtimer();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x == 0) { out[2 * blockIdx.x] = t0; out[2 * blockIdx.x + 1] = t1; }
}

static PFN_cuTensorMapEncodeTiled_v12000 encode;

template <int MODE, int CS>
int run(const CUtensorMap& tm, int sms, long long* d_out, int iters) {
  const int smem = STAGES * TILE + 1024 + 256;
  CK(cudaFuncSetAttribute(feed<MODE, CS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(32); cfg.dynamicSmemBytes = smem; cfg.attrs = at; cfg.numAttrs = 1;
  cfg.gridDim = dim3(sms);
  int ncl = 0;
  CK(cudaOccupancyMaxActiveClusters(&ncl, feed<MODE, CS>, &cfg));
  const int grid = ncl * CS;
  cfg.gridDim = dim3(grid);
  double best = 1e30;
  for (int rep = 0; rep < 5; ++rep) {
    CK(cudaLaunchKernelEx(&cfg, feed<MODE, CS>, tm, iters, d_out));
    CK(cudaDeviceSynchronize());
    std::vector<long long> h(2 * grid);
    CK(cudaMemcpy(h.data(), d_out, 16 * grid, cudaMemcpyDeviceToHost));
    long long a = h[0], b = h[1];
    for (int i = 0; i < grid; ++i) { a = h[2 * i] < a ? h[2 * i] : a; b = h[2 * i + 1] > b ? h[2 * i + 1] : b; }
    const double ns = (double)(b - a);
    if (ns < best) best = ns;
  }
  const double bytes = (double)grid * iters * TILE;
  printf("mode %d cs %d: %3d CTAs, %.0f ns per k-block per CTA, delivered %.2f TB/s (%.1f GB/s per SM)\n", MODE, CS,
         grid, best / iters, bytes / best / 1e3, bytes / best / grid);
  return 0;
}

int main() {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q));
  void* src;
  CK(cudaMalloc(&src, (size_t)ROWS * COLS * 2));
  CK(cudaMemset(src, 0, (size_t)ROWS * COLS * 2));
  long long* d_out;
  CK(cudaMalloc(&d_out, 16 * 1024));
  CUtensorMap tm128, tm32;
  for (int v = 0; v < 2; ++v) {
    cuuint64_t dims[2] = {COLS, ROWS};
    cuuint64_t strides[1] = {COLS * 2};
    cuuint32_t box[2] = {64, v == 0 ? 128u : 32u};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode(v == 0 ? &tm128 : &tm32, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
  }
  const int iters = 4000;
  run<0, 1>(tm128, sms, d_out, iters);
  run<0, 2>(tm128, sms, d_out, iters);
  run<1, 2>(tm128, sms, d_out, iters);
  run<1, 4>(tm128, sms, d_out, iters);
  run<1, 8>(tm128, sms, d_out, iters);
  run<2, 2>(tm32, sms, d_out, iters);
  run<2, 4>(tm32, sms, d_out, iters);
  run<2, 8>(tm32, sms, d_out, iters);
  return 0;
}
