// comm.cu — collectives of the head-parallel (tensor-parallel) blend (SURVEY.md §8(e) partitioning 1,
// DESIGN.md §7).
//
// Rank r of w holds q heads [r n_q/w, ...), kv heads [r n_kv/w, ...), the W_qkv rows of those heads, the
// W_o columns of its q heads, the gate/up rows and W_down columns of d_ff/w features, and the blended
// KV of its kv heads. Realign, scatter and attention are rank-local (no communication inside attention,
// BASELINE north_star). Per layer the blend needs three exchanges:
//   (i)   Delta_kv partials (QKV epilogue, one fp32 per (64-column k|v block, candidate)) all-gathered,
//         so every rank runs the same top-k over the same sum in the same fixed block order;
//   (ii)  the o_proj output all-reduced (rank 0 adds the residual, the others contribute attn W_o only);
//   (iii) the down_proj output all-reduced the same way (Megatron MLP; RMSNorm replicated on full rows).
// Two backends behind one interface:
//   - NCCL (one process per GPU; libnccl.so.2 resolved with dlopen at cb_set_comm time, the copy torch
//     already loaded when present), calls enqueued on the blend's stream and graph-capturable;
//   - a loopback group (several contexts of ONE process on one device, each driven by its own host
//     thread and stream): the exchange is stream-event ordering plus a reduce kernel over the members'
//     buffers. It runs the identical per-rank kernels, so the head-parallel path is parity-tested on
//     one GPU. Eager only (cross-stream events cannot be captured across graphs).
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>

#include "ctx.h"

// ---- NCCL through dlopen ---------------------------------------------------------------------------
namespace {
struct NcclApi {
  bool ok = false;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclAllGather) allGather = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclGetErrorString) errStr = nullptr;
};

std::mutex g_nccl_mu;
NcclApi g_nccl;

const NcclApi* nccl_api() {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (g_nccl.ok) return &g_nccl;
  const char* env = getenv("CB_NCCL_LIB");
  void* h = nullptr;
  if (env && *env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);  // torch's copy, if loaded
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return nullptr;
  NcclApi a;
  a.getUniqueId = (decltype(a.getUniqueId))dlsym(h, "ncclGetUniqueId");
  a.commInitRank = (decltype(a.commInitRank))dlsym(h, "ncclCommInitRank");
  a.allReduce = (decltype(a.allReduce))dlsym(h, "ncclAllReduce");
  a.allGather = (decltype(a.allGather))dlsym(h, "ncclAllGather");
  a.commDestroy = (decltype(a.commDestroy))dlsym(h, "ncclCommDestroy");
  a.errStr = (decltype(a.errStr))dlsym(h, "ncclGetErrorString");
  if (!a.getUniqueId || !a.commInitRank || !a.allReduce || !a.allGather || !a.commDestroy || !a.errStr)
    return nullptr;
  a.ok = true;
  g_nccl = a;
  return &g_nccl;
}

#define CB_NCCL(api, call)                                                                  \
  do {                                                                                      \
    ncclResult_t r_ = (call);                                                               \
    if (r_ != ncclSuccess) {                                                                \
      cb_set_error("NCCL error %d at %s:%d: %s", (int)r_, __FILE__, __LINE__, (api)->errStr(r_)); \
      return CB_E_NCCL;                                                                     \
    }                                                                                       \
  } while (0)
}  // namespace

// ---- loopback group ------------------------------------------------------------------------------------
struct cb_group {
  int world = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  bool broken = false;
  cb_ctx* member[kMaxTp] = {};
  float* ptr[kMaxTp] = {};               // each member's buffer of the current collective
  cudaEvent_t ev[2][kMaxTp] = {};        // phase events (recorded by their member)
};

namespace {
// Host barrier of the group's member threads. A member that never arrives (it failed) turns into an
// error after 120 s instead of a hang.
cb_status group_barrier(cb_group* g) {
  std::unique_lock<std::mutex> lk(g->mu);
  if (g->broken) { cb_set_error("loopback group is broken (a member failed)"); return CB_E_NCCL; }
  const long long my = g->gen;
  if (++g->arrived == g->world) {
    g->arrived = 0;
    ++g->gen;
    g->cv.notify_all();
    return CB_OK;
  }
  if (!g->cv.wait_for(lk, std::chrono::seconds(120), [&] { return g->gen != my || g->broken; }) || g->broken) {
    g->broken = true;
    g->cv.notify_all();
    cb_set_error("loopback group barrier timed out / broken");
    return CB_E_NCCL;
  }
  return CB_OK;
}

struct PtrSet { const float* p[kMaxTp]; };

// out[i] = in_0[i] + in_1[i] + ... in member order (fixed order: bitwise reproducible).
__global__ void sum_members_kernel(PtrSet in, int n_in, float* __restrict__ out, long long n, bool vec) {
  const long long n4 = vec ? n / 4 : 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    float4 a = reinterpret_cast<const float4*>(in.p[0])[i];
    for (int j = 1; j < n_in; ++j) {
      const float4 b = reinterpret_cast<const float4*>(in.p[j])[i];
      a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
    }
    reinterpret_cast<float4*>(out)[i] = a;
  }
  for (long long i = n4 * 4 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float a = in.p[0][i];
    for (int j = 1; j < n_in; ++j) a += in.p[j][i];
    out[i] = a;
  }
}

// Phase 1 of a loopback collective: publish this member's buffer, order every member's stream after
// all members' work so far.
cb_status loop_enter(cb_ctx* c, float* buf, cudaStream_t s, int phase) {
  cb_group* g = c->group;
  const int r = c->tp_rank;
  g->ptr[r] = buf;
  CB_CUDA(cudaEventRecord(g->ev[phase][r], s));
  CB_TRY(group_barrier(g));
  for (int j = 0; j < g->world; ++j)
    if (j != r) CB_CUDA(cudaStreamWaitEvent(s, g->ev[phase][j], 0));
  return CB_OK;
}

cb_status loop_allreduce(cb_ctx* c, float* buf, size_t n, cudaStream_t s) {
  cb_group* g = c->group;
  CB_REQUIRE(n <= c->tp_scratch_n, CB_E_SHAPE, "loopback all-reduce of %zu floats > scratch %zu", n, c->tp_scratch_n);
  CB_TRY(loop_enter(c, buf, s, 0));
  PtrSet ps{};
  for (int j = 0; j < g->world; ++j) ps.p[j] = g->ptr[j];
  const int blocks = (int)std::min<long long>(4LL * c->num_sms, ((long long)n / 4 + 255) / 256 + 1);
  bool vec = true;  // float4 path only when every buffer is 16-B aligned (dev_out rows may not be)
  for (int j = 0; j < g->world; ++j) vec &= ((uintptr_t)ps.p[j] % 16) == 0;
  sum_members_kernel<<<blocks, 256, 0, s>>>(ps, g->world, c->tp_scratch, (long long)n, vec);
  CB_LAUNCHED(c);
  // phase 2: nobody overwrites its buffer before every member has read it
  CB_TRY(loop_enter(c, buf, s, 1));
  CB_CUDA(cudaMemcpyAsync(buf, c->tp_scratch, n * sizeof(float), cudaMemcpyDeviceToDevice, s));
  return CB_OK;
}

cb_status loop_allgather(cb_ctx* c, float* buf, size_t n_per_rank, cudaStream_t s) {
  cb_group* g = c->group;
  CB_TRY(loop_enter(c, buf, s, 0));
  for (int j = 0; j < g->world; ++j)
    if (j != c->tp_rank)
      CB_CUDA(cudaMemcpyAsync(buf + (size_t)j * n_per_rank, g->ptr[j] + (size_t)j * n_per_rank,
                              n_per_rank * sizeof(float), cudaMemcpyDeviceToDevice, s));
  CB_TRY(loop_enter(c, buf, s, 1));
  return CB_OK;
}

// Per-rank buffers of the head-parallel blend: the gathered Delta_kv partials [2 nb_local w][T] and the
// loopback reduce scratch.
cb_status tp_alloc(cb_ctx* c) {
  const size_t nb = (size_t)(c->m.n_kv_heads * c->m.head_dim + 63) / 64;
  CB_CUDA(cudaMalloc(&c->dev_gath, 2 * nb * c->tp_world * (size_t)c->max_tokens * sizeof(float)));
  return CB_OK;
}
}  // namespace

cb_status p2p_allreduce_f32(cb_ctx* c, float* buf, size_t n, cudaStream_t s);
cb_status p2p_allgather_f32(cb_ctx* c, float* buf, size_t n_per_rank, cudaStream_t s);

cb_status comm_allreduce_f32(cb_ctx* c, float* buf, size_t n, cudaStream_t s) {
  if (c->comm_kind == CB_COMM_NONE || n == 0) return CB_OK;
  ProfScope ps_(c, PROF_COMM, s);
  if (c->xblock) return p2p_allreduce_f32(c, buf, n, s);
  if (c->comm_kind == CB_COMM_LOOPBACK) return loop_allreduce(c, buf, n, s);
  const NcclApi* a = nccl_api();
  CB_NCCL(a, a->allReduce(buf, buf, n, ncclFloat32, ncclSum, (ncclComm_t)c->nccl_comm, s));
  return CB_OK;
}

cb_status comm_allgather_f32(cb_ctx* c, float* buf, size_t n_per_rank, cudaStream_t s) {
  if (c->comm_kind == CB_COMM_NONE || n_per_rank == 0) return CB_OK;
  ProfScope ps_(c, PROF_COMM, s);
  if (c->xblock) return p2p_allgather_f32(c, buf, n_per_rank, s);
  if (c->comm_kind == CB_COMM_LOOPBACK) return loop_allgather(c, buf, n_per_rank, s);
  const NcclApi* a = nccl_api();
  // in place: this rank's segment already sits at buf + rank * n_per_rank
  CB_NCCL(a, a->allGather(buf + (size_t)c->tp_rank * n_per_rank, buf, n_per_rank, ncclFloat32,
                          (ncclComm_t)c->nccl_comm, s));
  return CB_OK;
}

void comm_destroy(cb_ctx* c) {
  if (c->comm_kind == CB_COMM_NCCL && c->nccl_comm) {
    const NcclApi* a = nccl_api();
    if (a) a->commDestroy((ncclComm_t)c->nccl_comm);
  }
  if (c->comm_kind == CB_COMM_LOOPBACK && c->group) {
    std::lock_guard<std::mutex> lk(c->group->mu);
    c->group->member[c->tp_rank] = nullptr;
  }
  for (int j = 0; j < kMaxTp; ++j) {
    if (c->p2p_ipc[j] && c->p2p_peer[j]) cudaIpcCloseMemHandle(c->p2p_peer[j]);
    c->p2p_ipc[j] = false;
    c->p2p_peer[j] = nullptr;
  }
  if (c->xblock) {
    if (c->dev_gath == (float*)(c->xblock + c->x_gath_off)) c->dev_gath = nullptr;
    cudaFree(c->xblock);
    c->xblock = nullptr;
  }
  if (c->dev_gath) cudaFree(c->dev_gath);
  if (c->tp_scratch) cudaFree(c->tp_scratch);
  c->nccl_comm = nullptr;
  c->group = nullptr;
  c->dev_gath = nullptr;
  c->tp_scratch = nullptr;
  c->comm_kind = CB_COMM_NONE;
  c->tp_rank = 0;
  c->tp_world = 1;
}

// ---- C-ABI ---------------------------------------------------------------------------------------------
namespace {
cb_status check_tp_model(const cb_ctx* c, int world) {
  // the context already holds the rank's shard of the model (heads / d_ff divided by world)
  CB_REQUIRE(world >= 1 && world <= kMaxTp, CB_E_INVALID_ARG, "world %d outside [1, %d]", world, kMaxTp);
  CB_REQUIRE(c->comm_kind == CB_COMM_NONE, CB_E_INVALID_ARG, "the context already has a communicator");
  return CB_OK;
}
}  // namespace

extern "C" cb_status cb_nccl_unique_id(void* uid_out) {
  CB_REQUIRE(uid_out != nullptr, CB_E_INVALID_ARG, "uid_out is NULL");
  const NcclApi* a = nccl_api();
  CB_REQUIRE(a != nullptr, CB_E_UNSUPPORTED, "libnccl.so.2 could not be loaded (set CB_NCCL_LIB)");
  ncclUniqueId id;
  CB_NCCL(a, a->getUniqueId(&id));
  std::memcpy(uid_out, &id, sizeof(id));
  return CB_OK;
}

extern "C" cb_status cb_set_comm(cb_ctx* c, const void* uid, int32_t rank, int32_t world) {
  CB_REQUIRE(c != nullptr && uid != nullptr, CB_E_INVALID_ARG, "ctx / uid is NULL");
  CB_TRY(check_tp_model(c, world));
  CB_REQUIRE(rank >= 0 && rank < world, CB_E_INVALID_ARG, "rank %d outside [0, %d)", rank, world);
  const NcclApi* a = nccl_api();
  CB_REQUIRE(a != nullptr, CB_E_UNSUPPORTED, "libnccl.so.2 could not be loaded (set CB_NCCL_LIB)");
  ncclUniqueId id;
  std::memcpy(&id, uid, sizeof(id));
  ncclComm_t comm = nullptr;
  CB_NCCL(a, a->commInitRank(&comm, world, id, rank));
  c->nccl_comm = comm;
  c->comm_kind = CB_COMM_NCCL;
  c->tp_rank = rank;
  c->tp_world = world;
  cb_status st = tp_alloc(c);
  if (st != CB_OK) comm_destroy(c);
  return st;
}

extern "C" cb_status cb_group_create(int32_t world, cb_group** out) {
  CB_REQUIRE(out != nullptr && world >= 1 && world <= kMaxTp, CB_E_INVALID_ARG, "world %d outside [1, %d]", world,
             kMaxTp);
  cb_group* g = new cb_group();
  g->world = world;
  for (int p = 0; p < 2; ++p)
    for (int j = 0; j < world; ++j) {
      cudaError_t e = cudaEventCreateWithFlags(&g->ev[p][j], cudaEventDisableTiming);
      if (e != cudaSuccess) {
        delete g;
        CB_CUDA(e);
      }
    }
  *out = g;
  return CB_OK;
}

extern "C" cb_status cb_group_destroy(cb_group* g) {
  if (!g) return CB_OK;
  for (int p = 0; p < 2; ++p)
    for (int j = 0; j < g->world; ++j)
      if (g->ev[p][j]) cudaEventDestroy(g->ev[p][j]);
  delete g;
  return CB_OK;
}

extern "C" cb_status cb_set_comm_local(cb_ctx* c, cb_group* g, int32_t rank) {
  CB_REQUIRE(c != nullptr && g != nullptr, CB_E_INVALID_ARG, "ctx / group is NULL");
  CB_TRY(check_tp_model(c, g->world));
  CB_REQUIRE(rank >= 0 && rank < g->world, CB_E_INVALID_ARG, "rank %d outside [0, %d)", rank, g->world);
  {
    std::lock_guard<std::mutex> lk(g->mu);
    CB_REQUIRE(g->member[rank] == nullptr, CB_E_INVALID_ARG, "group rank %d is taken", rank);
    g->member[rank] = c;
  }
  c->group = g;
  c->comm_kind = CB_COMM_LOOPBACK;
  c->tp_rank = rank;
  c->tp_world = g->world;
  c->tp_scratch_n = (size_t)c->max_tokens * c->m.d_model;
  cudaError_t e = cudaMalloc(&c->tp_scratch, c->tp_scratch_n * sizeof(float));
  cb_status st = e == cudaSuccess ? tp_alloc(c) : CB_E_CUDA;
  if (e != cudaSuccess) cb_set_error("cb_set_comm_local: %s", cudaGetErrorString(e));
  if (st != CB_OK) comm_destroy(c);
  return st;
}

// ---- NVLink peer-memory collectives ------------------------------------------------------------------------
// The B200-native replacement of the NCCL calls above: every rank maps every peer's exchange
// block (NVLink P2P over NVSwitch), and one small kernel per collective does
//   entry barrier  -- each rank's buffer is final (stream order + PDL wait), so it raises flag[0][rank] = seq
//                     in every peer's block (st.release.sys) and waits for all peers' flags (ld.acquire.sys);
//   data movement  -- all-reduce: rank r owns the r-th slice of the buffer: it sums the slice over all ranks'
//                     buffers in rank order (deterministic, the same bits as the loopback event path) and
//                     writes the sum into every rank's buffer; all-gather: rank r pushes its segment to all;
//   exit barrier   -- the last CTA of each rank raises flag[1][rank] = seq everywhere and waits for all, so
//                     the kernel completes only when every rank's writes are done (nobody overwrites a buffer
//                     a peer is still reading). seq is a device-side counter, so a CUDA graph can replay it.
// The grid is small (64 CTAs; 4 in the one-device loopback test, where every rank's spinning CTAs share the
// SMs with the other ranks' kernels).
namespace {
constexpr int P2P_CTAS = 64, P2P_THREADS = 256;

__device__ __forceinline__ void st_release_sys(int* p, int v) {
  asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_sys(const int* p) {
  int v;
#ifdef CB_P2P_ACQ_GPU
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
#elif defined(CB_P2P_POLL_ATOMIC)
  v = atomicAdd(const_cast<int*>(p), 0);  // always served by L2
  __threadfence_system();
#else
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
#endif
  return v;
}

struct PeerTable { char* base[kMaxTp]; };

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Spin until *f >= seq, or give up after 10 s (a peer that never arrives must not hang the GPU): the
// device error word then carries CB_DEVERR_COMM (cb_check_device_errors) and the data are invalid.
__device__ __forceinline__ void wait_flag(const int* f, int seq, int* err) {
  const unsigned long long t0 = gtimer();
  while (ld_acquire_sys(f) < seq) {
    __nanosleep(64);
    if (gtimer() - t0 > 10000000000ull) {
      atomicOr(err, CB_DEVERR_COMM);
      return;
    }
  }
}

// flags (ints at flags_off of every block): [0, kMaxTp) entry, [kMaxTp, 2 kMaxTp) exit, [2 kMaxTp] seq,
// [2 kMaxTp + 1] finished-CTA counter
// mode 0: all-reduce of n floats at off; 1: all-gather (segments of n floats); 2: fused reduce-scatter
// epilogue: rows were pushed by the GEMMs into this rank's receive planes (recv_off, plane floats apart);
// this rank's chunk of the n floats is summed over the planes and written at off in every rank's block.
__global__ void __launch_bounds__(P2P_THREADS) p2p_collective_kernel(PeerTable pt, int rank, int world,
                                                                     size_t off, long long n, int mode,
                                                                     size_t flags_off, int* err, size_t recv_off,
                                                                     long long plane, long long chunk2) {
  // wait for this rank's producer, but do NOT let the dependent kernel launch early: on one device
  // (loopback) its waiting CTAs could fill the SMs the other ranks need to reach their barrier
  pdl_wait();
  int* myf = reinterpret_cast<int*>(pt.base[rank] + flags_off);
  __shared__ int seq_s;
  if (threadIdx.x == 0) seq_s = *reinterpret_cast<volatile int*>(myf + 2 * kMaxTp) + 1;
  __syncthreads();
  const int seq = seq_s;
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // diagnostics ring (ints 20..51): seq, rank, own-block tag, mode
    int* r = myf + 20 + (seq & 7) * 4;
    r[0] = seq; r[1] = rank * 16 + mode;
    r[2] = (int)(reinterpret_cast<uintptr_t>(pt.base[0] + flags_off) >> 8);
    r[3] = (int)(reinterpret_cast<uintptr_t>(pt.base[world > 1 ? 1 : 0] + flags_off) >> 8);
  }
  if (blockIdx.x == 0 && threadIdx.x < world) {
    __threadfence_system();
    st_release_sys(reinterpret_cast<int*>(pt.base[threadIdx.x] + flags_off) + rank, seq);
  }
  const unsigned long long t_wait = gtimer();
  if (threadIdx.x < world) wait_flag(myf + threadIdx.x, seq, err);
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0)  // diagnostics: entry-wait time (us) and the peers' flags seen
    myf[20 + (seq & 7) * 4 + 1] = (rank * 16 + mode) + 256 * (int)min(1000000ull, (gtimer() - t_wait) / 1000ull);
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (mode == 0) {  // all-reduce: this rank's slice, summed in rank order, written to every rank
    const long long chunk = ((n + world - 1) / world + 3) / 4 * 4;
    const long long lo = (long long)rank * chunk, hi = lo + chunk < n ? lo + chunk : n;
    const long long lo4 = lo / 4, hi4 = hi / 4;  // lo is a multiple of 4; off is 16-B aligned
    for (long long i = lo4 + t0; i < hi4; i += stride) {
      float4 a = __ldcg(reinterpret_cast<const float4*>(pt.base[0] + off) + i);
      for (int j = 1; j < world; ++j) {
        const float4 b = __ldcg(reinterpret_cast<const float4*>(pt.base[j] + off) + i);
        a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
      }
      for (int j = 0; j < world; ++j) __stcg(reinterpret_cast<float4*>(pt.base[j] + off) + i, a);
    }
    for (long long i = hi4 * 4 + t0; i < hi; i += stride) {
      float a = __ldcg(reinterpret_cast<const float*>(pt.base[0] + off) + i);
      for (int j = 1; j < world; ++j) a += __ldcg(reinterpret_cast<const float*>(pt.base[j] + off) + i);
      for (int j = 0; j < world; ++j) __stcg(reinterpret_cast<float*>(pt.base[j] + off) + i, a);
    }
  } else if (mode == 2) {  // the rows this rank owns: sum the pushed planes in rank order, write everywhere
    const long long lo = (long long)rank * chunk2, hi = lo + chunk2 < n ? lo + chunk2 : n;
    const float* own = reinterpret_cast<const float*>(pt.base[rank] + recv_off);
    for (long long i = lo / 4 + t0; i < hi / 4; i += stride) {
      float4 a = __ldcg(reinterpret_cast<const float4*>(own) + i);
      for (int j = 1; j < world; ++j) {
        const float4 b = __ldcg(reinterpret_cast<const float4*>(own + (size_t)j * plane) + i);
        a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
      }
      for (int j = 0; j < world; ++j) __stcg(reinterpret_cast<float4*>(pt.base[j] + off) + i, a);
    }
  } else {  // all-gather: push this rank's segment of n floats to every peer
    const float4* src = reinterpret_cast<const float4*>(pt.base[rank] + off) + (size_t)rank * (n / 4);
    for (long long i = t0; i < n / 4; i += stride) {
      const float4 v = __ldcg(src + i);
      for (int j = 0; j < world; ++j)
        if (j != rank) __stcg(reinterpret_cast<float4*>(pt.base[j] + off) + (size_t)rank * (n / 4) + i, v);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const int done = atomicAdd(myf + 2 * kMaxTp + 1, 1);
    if (done == (int)gridDim.x - 1) {  // every CTA of this rank has written: exit barrier
      myf[2 * kMaxTp + 1] = 0;
      __threadfence_system();
      for (int j = 0; j < world; ++j)
        st_release_sys(reinterpret_cast<int*>(pt.base[j] + flags_off) + kMaxTp + rank, seq);
      for (int j = 0; j < world; ++j) wait_flag(myf + kMaxTp + j, seq, err);
      *reinterpret_cast<volatile int*>(myf + 2 * kMaxTp) = seq;
    }
  }
}

cb_status p2p_peers(cb_ctx* c, PeerTable* pt) {
  for (int j = 0; j < c->tp_world; ++j) {
    char* b = c->p2p_peer[j];
    if (b == nullptr && c->comm_kind == CB_COMM_LOOPBACK && c->group->member[j] != nullptr)
      b = c->p2p_peer[j] = c->group->member[j]->xblock;  // one device: the member's own pointer
    CB_REQUIRE(b != nullptr, CB_E_INVALID_ARG, "peer-memory collectives: rank %d's exchange block is not mapped", j);
    pt->base[j] = b;
  }
  return CB_OK;
}

cb_status p2p_launch(cb_ctx* c, size_t off, long long n, int mode, cudaStream_t s, long long chunk2 = 0) {
  PeerTable pt{};
  CB_TRY(p2p_peers(c, &pt));

  // one device (loopback): 4 CTAs per rank, so the spinning CTAs of all ranks occupy at most 32 SMs and the
  // other ranks' kernels (which may need a whole SM) always find free SMs
  const int ctas = c->comm_kind == CB_COMM_LOOPBACK ? (getenv("CB_P2P_LOOP_CTAS") ? atoi(getenv("CB_P2P_LOOP_CTAS")) : 4) : P2P_CTAS;
  CB_LAUNCH(c, p2p_collective_kernel, ctas, P2P_THREADS, 0, s, pt, c->tp_rank, c->tp_world, off, n, mode,
            c->x_flags_off, c->err_word, c->x_recv_off, (long long)(c->x_h_bytes / sizeof(float)), chunk2);
  CB_LAUNCHED(c);
  return CB_OK;
}

bool in_block(const cb_ctx* c, const void* p) {
  return c->xblock && (const char*)p >= c->xblock && (const char*)p < c->xblock + c->x_total;
}
}  // namespace

cb_status p2p_allreduce_f32(cb_ctx* c, float* buf, size_t n, cudaStream_t s) {
  if (in_block(c, buf)) return p2p_launch(c, (size_t)((char*)buf - c->xblock), (long long)n, 0, s);
  // a buffer outside the exchange block (a caller's dev_out row): through the staging row
  CB_REQUIRE(n * sizeof(float) <= c->x_flags_off - c->x_stage_off, CB_E_SHAPE, "p2p all-reduce staging too small");
  CB_CUDA(cudaMemcpyAsync(c->xblock + c->x_stage_off, buf, n * sizeof(float), cudaMemcpyDeviceToDevice, s));
  CB_TRY(p2p_launch(c, c->x_stage_off, (long long)n, 0, s));
  CB_CUDA(cudaMemcpyAsync(buf, c->xblock + c->x_stage_off, n * sizeof(float), cudaMemcpyDeviceToDevice, s));
  return CB_OK;
}

cb_status p2p_allgather_f32(cb_ctx* c, float* buf, size_t n_per_rank, cudaStream_t s) {
  if (c->tp_world == 1) return CB_OK;  // nothing to gather
  CB_REQUIRE(in_block(c, buf) && n_per_rank % 4 == 0, CB_E_INVALID_ARG, "p2p all-gather outside the exchange block");
  return p2p_launch(c, (size_t)((char*)buf - c->xblock), (long long)n_per_rank, 1, s);
}

extern "C" cb_status cb_tp_p2p_enable(cb_ctx* c) {
  CB_REQUIRE(c != nullptr, CB_E_INVALID_ARG, "ctx is NULL");
  CB_REQUIRE(c->comm_kind != CB_COMM_NONE && c->tp_world >= 1, CB_E_INVALID_ARG,
             "join a communicator (cb_set_comm / cb_set_comm_local) first");
  if (c->xblock) return CB_OK;
  const size_t T = (size_t)c->max_tokens, d = (size_t)c->m.d_model;
  const size_t nb = (size_t)(c->m.n_kv_heads * c->m.head_dim + 63) / 64;
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  c->x_h_bytes = al(T * d * sizeof(float));
  c->x_gath_off = 2 * c->x_h_bytes;
  c->x_stage_off = c->x_gath_off + al(2 * nb * c->tp_world * T * sizeof(float));
  c->x_flags_off = c->x_stage_off + al(T * sizeof(float));
  // receive planes of the fused reduce-scatter: one [T][d] fp32 plane per rank (skipped with tp_fuse = 0)
  c->x_recv_off = c->tp_world > 1 && !c->tp_nofuse ? c->x_flags_off + 256 : 0;
  c->x_total = c->x_flags_off + 256 + (c->x_recv_off ? (size_t)c->tp_world * c->x_h_bytes : 0);
  void* p = nullptr;
  CB_CUDA(cudaMalloc(&p, c->x_total));
  CB_CUDA(cudaMemset(p, 0, c->x_total));
  c->xblock = (char*)p;
  c->h[0] = (float*)c->xblock;  // the residual stream (o_proj / down_proj outputs) lives in the block
  c->h[1] = (float*)(c->xblock + c->x_h_bytes);
  if (c->dev_gath) cudaFree(c->dev_gath);
  c->dev_gath = (float*)(c->xblock + c->x_gath_off);
  c->p2p_peer[c->tp_rank] = c->xblock;
  // one device (loopback): no programmatic early launch at all, so the only resident waiters are the
  // collective kernels' own 64 spinning CTAs and the other ranks' kernels always find SMs
  if (c->comm_kind == CB_COMM_LOOPBACK) c->pdl = 0;
  return CB_OK;
}

extern "C" cb_status cb_tp_ipc_handle(cb_ctx* c, void* handle_out) {
  CB_REQUIRE(c && handle_out && c->xblock, CB_E_INVALID_ARG, "cb_tp_ipc_handle: enable peer-memory collectives first");
  cudaIpcMemHandle_t h;
  CB_CUDA(cudaIpcGetMemHandle(&h, c->xblock));
  std::memcpy(handle_out, &h, sizeof(h));
  return CB_OK;
}

extern "C" cb_status cb_tp_ipc_open(cb_ctx* c, const void* handles) {
  CB_REQUIRE(c && handles && c->xblock, CB_E_INVALID_ARG, "cb_tp_ipc_open: enable peer-memory collectives first");
  for (int j = 0; j < c->tp_world; ++j) {
    if (j == c->tp_rank || c->p2p_peer[j]) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, (const char*)handles + (size_t)j * sizeof(h), sizeof(h));
    void* p = nullptr;
    CB_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    c->p2p_peer[j] = (char*)p;
    c->p2p_ipc[j] = true;
  }
  return CB_OK;
}

// Diagnostics: copy this rank's flag words (entry[kMaxTp], exit[kMaxTp], seq, finished-CTA counter) to the
// host through a private non-blocking stream (does not wait for work queued on other streams).
extern "C" cb_status cb_debug_p2p_flags(cb_ctx* c, int32_t* out) {
  CB_REQUIRE(c && out && c->xblock, CB_E_INVALID_ARG, "cb_debug_p2p_flags: no exchange block");
  cudaStream_t st;
  CB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaError_t e = cudaMemcpyAsync(out, c->xblock + c->x_flags_off, 52 * sizeof(int), cudaMemcpyDeviceToHost, st);
  out[52] = (int)(reinterpret_cast<uintptr_t>(c->xblock + c->x_flags_off) >> 8);  // this block's tag
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  CB_CUDA(e);
  return CB_OK;
}

bool tp_push_on(const cb_ctx* c) { return c->xblock != nullptr && c->x_recv_off != 0 && c->tp_world > 1; }

cb_status tp_push_params(cb_ctx* c, EpiParams& e, int rows) {
  PeerTable pt{};
  CB_TRY(p2p_peers(c, &pt));
  for (int j = 0; j < kMaxTp; ++j) e.push_base[j] = j < c->tp_world ? pt.base[j] : nullptr;
  e.push_rows = (rows + c->tp_world - 1) / c->tp_world;
  e.push_off = (long long)(c->x_recv_off + (size_t)c->tp_rank * c->x_h_bytes);
  CB_REQUIRE(e.ldo == c->m.d_model, CB_E_INVALID_ARG, "pushed rows must be d_model wide");
  return CB_OK;
}

cb_status comm_allreduce_pushed(cb_ctx* c, float* h_out, int rows, cudaStream_t s) {
  CB_REQUIRE(in_block(c, h_out), CB_E_INVALID_ARG, "pushed all-reduce: h_out outside the exchange block");
  ProfScope ps_(c, PROF_COMM, s);
  const long long d = c->m.d_model;
  const long long chunk = (long long)((rows + c->tp_world - 1) / c->tp_world) * d;  // the rows each rank owns
  return p2p_launch(c, (size_t)((char*)h_out - c->xblock), (long long)rows * d, 2, s, chunk);
}
