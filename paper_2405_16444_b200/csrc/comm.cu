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

cb_status comm_allreduce_f32(cb_ctx* c, float* buf, size_t n, cudaStream_t s) {
  if (c->comm_kind == CB_COMM_NONE || n == 0) return CB_OK;
  ProfScope ps_(c, PROF_COMM, s);
  if (c->comm_kind == CB_COMM_LOOPBACK) return loop_allreduce(c, buf, n, s);
  const NcclApi* a = nccl_api();
  CB_NCCL(a, a->allReduce(buf, buf, n, ncclFloat32, ncclSum, (ncclComm_t)c->nccl_comm, s));
  return CB_OK;
}

cb_status comm_allgather_f32(cb_ctx* c, float* buf, size_t n_per_rank, cudaStream_t s) {
  if (c->comm_kind == CB_COMM_NONE || n_per_rank == 0) return CB_OK;
  ProfScope ps_(c, PROF_COMM, s);
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
