// ctx.h — host-side context of libcacheblend (internal).
#pragma once

#include <cstdarg>
#include <cstdio>
#include <string>

#include "common.cuh"

#include <vector>

struct TmapCache;  // tcgen05 GEMM tensor-map cache (gemm_tc.cu)
struct cb_group;   // loopback tensor-parallel group (comm.cu)

// Kernel classes for the per-launch profile (bench roofline: CUDA events on the launching stream).
enum ProfClass : int {
  PROF_REALIGN = 0, PROF_EMBED, PROF_RMSNORM, PROF_GEMM, PROF_DEVIATION, PROF_TOPK, PROF_SCATTER, PROF_ATTN,
  PROF_MISC, PROF_COMM, PROF_N
};

// Head-parallel (tensor-parallel) communicator kinds (comm.cu).
enum CommKind : int { CB_COMM_NONE = 0, CB_COMM_NCCL = 1, CB_COMM_LOOPBACK = 2 };
constexpr int kMaxTp = 8;

struct ProfRec {
  int cls;
  cudaEvent_t a, b;
};

struct cb_ctx {
  cb_model m;
  int max_tokens;
  int device;
  int num_sms;
  // RoPE table: (cos, sin)(p * theta_i) for p in [0, max_pos), i in [0, hd/2); built in fp64.
  float2* rope_tab;
  int* err_word;  // device error bits
  // workspace
  void* ws;
  size_t ws_bytes;
  bool ws_owned;
  float* h[2];      // fp32 [T][d] residual stream ping-pong
  void* x;          // [T][d]      normed rows (model dtype)
  void* q;          // [T][qd]
  void* kf;         // [T][kvd]    fresh k (RoPE'd) of the current rows
  void* vf;         // [T][kvd]
  void* attn;       // [T][qd]
  void* act;        // [T][ff]
  float* dev;       // [T]
  float* dev_part;  // [2 n_kv][T] fused-deviation partials (QKV epilogue)
  float* ss;        // [T][d / 64] fused-RMSNorm sum-of-squares blocks (residual GEMM epilogue -> next GEMM)
  int* row_tok[2];  // [T] token index of each current row (candidates, then suffix)
  int* qrow;        // [T] row (in the current compact buffers) of each kept query
  int* iota;        // [T] 0..T-1
  int* src_pos;     // [T] chunk-local positions (blend_forward)
  float* attn_part;     // split-KV attention partials [attn_part_rows][head_dim] fp32
  float2* attn_ml;      // [attn_part_rows] (m, l)
  int* attn_cnt;        // [T * n_q / 128 + n_kv] split arrival counters of the tcgen05 attention (zero between launches)
  int attn_cnt_n;
  int* attn_work;       // [2] persistent attention: item claim counter, finished-CTA counter (zero between launches)
  long long attn_part_rows;
  int gemm_sched;   // cb_set_option("gemm_sched")
  int attn_impl;    // cb_set_option("attn_impl"): 0 auto, 1 SIMT, 2 tcgen05
  int attn_splits;  // cb_set_option("attn_splits"): 0 auto, else forced split-KV factor
  int no_fuse_norm;  // cb_set_option("fuse_norm", 0): separate RMSNorm kernels between the projections
  int no_fuse_dev;  // cb_set_option("fuse_deviation", 0) disables the QKV-epilogue deviation
  int dbg_sel;         // debug_trace value: 1 = attention + every CTA-pair GEMM, 100 + k = pair GEMMs of kind k only
  long long* dbg_buf;  // cb_set_option("debug_trace", 1): per-event clock64 trace of one CTA (tuning)
  int pdl;          // programmatic dependent launch between library kernels (cb_set_option("pdl"))
  int* tok_d;       // [T] request-mode device copies of tokens / positions
  int* pos_d;       // [T]
  long long launches;
  TmapCache* tmaps;
  // request mode: copy stream + per-layer "layer KV landed" events (P:2509 fetch/synchronize)
  cudaStream_t copy_stream;
  cudaStream_t aux_stream;    // MLP split: the down-projection blocks run here, overlapping gate_up blocks
  int topk_drop_max;          // cb_set_option("topk_drop", n): drop-smallest top-k path when n_cand - k <= n
  int gemm_mc;                // cb_set_option("gemm_mc"): 0 off, 1 4-CTA clusters, 2 auto, 3 8-CTA clusters (pair GEMM)
  int max_clusters4;          // co-resident 4-CTA clusters of the pair GEMM (0: none)
  int max_clusters8;          // co-resident 8-CTA clusters of the pair GEMM (0: none)
  int q_split;                // cb_set_option("q_split", 0/1): layer-1 Q projected after the selection (kept rows)
  int epi_l1pf;               // cb_set_option("epi_l1pf"): residual epilogue prefetches the next chunk into L1
  int topk_threads;           // cb_set_option("topk_threads", 256 | 512 | 1024): top-k block size (0 = 1024)
  cudaEvent_t ev_ready;
  cudaEvent_t ev_realign[2];  // realign of layers 1..L-1 on the aux stream: fork, done
  int realign_overlap;        // cb_set_option("realign_overlap"): that realign runs under layer 0
  std::vector<cudaEvent_t> layer_ev;
  // head-parallel blend (comm.cu): this context holds rank tp_rank's shard of the model (heads, d_ff / world)
  int tp_rank;
  int tp_world;               // <= 1: no tensor parallelism
  int comm_kind;              // CommKind
  void* nccl_comm;            // ncclComm_t
  cb_group* group;            // loopback group (one process, one device)
  float* dev_gath;            // [2 nb_local world][max_tokens] gathered Delta_kv partials
  float* tp_scratch;          // loopback all-reduce scratch
  size_t tp_scratch_n;
  // NVLink peer-memory collectives (comm.cu, cb_tp_p2p_enable): h[0], h[1], dev_gath, a staging row and the
  // flags live in one exchange block per rank with the same layout on every rank; peers' blocks are mapped
  // through CUDA IPC (one process per GPU) or taken from the loopback group's members
  char* xblock;
  size_t x_h_bytes, x_gath_off, x_stage_off, x_flags_off, x_recv_off, x_total;
  int tp_nofuse;              // cb_set_option("tp_fuse", 0): o_proj / down_proj write locally, then a plain all-reduce
  char* p2p_peer[kMaxTp];     // every rank's exchange block as seen from this device (own included)
  bool p2p_ipc[kMaxTp];       // opened with cudaIpcOpenMemHandle (closed in comm_destroy)
  // profiling
  bool prof_on;
  std::vector<ProfRec> prof;
  std::vector<cudaEvent_t> ev_pool;
};

// Records an event pair around the launches in its scope when the context is profiling.
struct ProfScope {
  cb_ctx* c;
  cudaStream_t s;
  int idx;
  ProfScope(cb_ctx* c_, int cls, cudaStream_t s_);
  ~ProfScope();
};

void cb_set_error(const char* fmt, ...);

#define CB_REQUIRE(cond, code, ...)        \
  do {                                     \
    if (!(cond)) {                         \
      cb_set_error(__VA_ARGS__);           \
      return (code);                       \
    }                                      \
  } while (0)

#define CB_CUDA(call)                                                               \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess) {                                                        \
      cb_set_error("CUDA error %s at %s:%d: %s", cudaGetErrorName(e_), __FILE__,    \
                   __LINE__, cudaGetErrorString(e_));                               \
      return CB_E_CUDA;                                                             \
    }                                                                               \
  } while (0)

#define CB_LAUNCHED(ctx)                  \
  do {                                    \
    (ctx)->launches++;                    \
    CB_CUDA(cudaGetLastError());          \
  } while (0)

#define CB_TRY(expr)                  \
  do {                                \
    cb_status s_ = (expr);            \
    if (s_ != CB_OK) return s_;       \
  } while (0)

static inline size_t dtype_bytes(int dt) { return dt == CB_BF16 ? 2 : 4; }

// Launch `kern` with programmatic stream serialization (PDL, when the context enables it) and an
// optional cluster size. Every kernel launched this way must begin with pdl_wait()/pdl_enter().
template <typename... KArgs, typename... Args>
static inline cudaError_t launch_k(const cb_ctx* c, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                   cudaStream_t s, int cluster, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  unsigned n = 0;
  if (c->pdl) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

#define CB_LAUNCH(ctx, kern, grid, block, smem, stream, ...) \
  CB_CUDA(launch_k((ctx), kern, dim3(grid), dim3(block), (smem), (stream), 1, __VA_ARGS__))

// ---- internal launchers (implemented per .cu file) ------------------------------------------
cb_status launch_realign(cb_ctx* c, void* k_out, const void* k_src, void* v_out, const void* v_src,
                         const int* src_pos, const int* dst_pos, int n_slices, int n_tok, long long out_stride,
                         long long src_stride, cudaStream_t s);
cb_status launch_embed(cb_ctx* c, const void* embed, const int* tok, int n, float* h, cudaStream_t s);
cb_status launch_embed_norm(cb_ctx* c, const void* embed, const int* tok, const float* gain, int n, float* h,
                            void* x, cudaStream_t s);
cb_status launch_rmsnorm(cb_ctx* c, const float* h, const float* gain, int n_rows, void* x, cudaStream_t s);
cb_status launch_scatter_kv(cb_ctx* c, const void* kf, const void* vf, const int* qrow, const int* qtok, int n,
                            void* kb, void* vb, cudaStream_t s);
cb_status launch_gather_rows(cb_ctx* c, const void* x, const float* ss, const int* qrow, int n, int ld_ss, void* xq,
                             float* ssq, cudaStream_t s);
cb_status launch_local_pos(cb_ctx* c, const int* chunk_start_host, int n_chunks, int* src_pos, cudaStream_t s);
// device positions: 0 <= pos[t] < max_pos (else CB_DEVERR_POS_RANGE) and strictly increasing (else CB_DEVERR_POS_ORDER)
cb_status launch_pos_check(cb_ctx* c, const int* pos, int T, cudaStream_t s);
cb_status launch_sel_out(cb_ctx* c, const int* qtok, int k, int N, int* sel_row, cudaStream_t s);
cb_status launch_deviation(cb_ctx* c, const void* k_new, const void* v_new, const void* k_ref, const void* v_ref,
                           const int* cand_tok, int n_cand, int dev_mode, float* dev, cudaStream_t s);
// dev_part != NULL: Delta_kv is first summed from the QKV epilogue's per-(kv head, k|v) partials
// [2 n_kv][ld_part] into dev (fixed head order, dev_mode selects K / V / both).
cb_status launch_topk(cb_ctx* c, float* dev, const int* cand_tok, int n_cand, int k_keep, int n_suffix,
                      int N, const int* force_sel, int* qrow, int* qtok, int* sel_tok, cudaStream_t s,
                      const float* dev_part = nullptr, int ld_part = 0, int dev_mode = CB_DEV_KV);
// GEMM: acc = A[M][K] . B[N_b][K]^T; for SWIGLU B holds 2*ff rows and e.N = ff.
// impl: 0 auto, 1 simt, 2 tcgen05.
cb_status launch_gemm(cb_ctx* c, const void* A, int lda, const void* B, int ldb, int M, int K, const EpiParams& e,
                      int impl, cudaStream_t s);
cb_status launch_attention(cb_ctx* c, const void* q, const int* q_row, const int* q_tok, int n_rows, const void* k,
                           const void* v, int n_keys, void* out, int impl, cudaStream_t s);
// Request path with a caller-supplied per-layer fetch (cb_blend_request, cb_blend_request_store).
#include <functional>
using FetchLayer = std::function<cb_status(int layer, char* k_dst, char* v_dst, cudaStream_t copy_stream)>;
cb_status blend_request_impl(cb_ctx* c, const cb_layer_w* w, const void* embed, const int32_t* tok_host,
                             const int32_t* pos_host, int N, int n_suffix, const int32_t* chunk_start, int n_chunks,
                             void* k_blend, void* v_blend, const int32_t* k_sched, int32_t* sel_out_host,
                             float* h_out_host, cudaStream_t s, const FetchLayer& fetch);
cb_status check_request(cb_ctx* c, const cb_layer_w* w, const void* embed, const int32_t* tok_host,
                        const int32_t* pos_host, int32_t N, int32_t n_suffix, const int32_t* chunk_start,
                        int32_t n_chunks, const void* k_in, const void* v_in, void* k_blend, void* v_blend,
                        const int32_t* k_sched, const void* h_out);
// Head-parallel collectives on `s` (no-ops when tp_world <= 1). All-reduce: in-place fp32 sum. All-gather:
// in place, this rank's n_per_rank floats already at buf + tp_rank * n_per_rank.
cb_status comm_allreduce_f32(cb_ctx* c, float* buf, size_t n, cudaStream_t s);
cb_status comm_allgather_f32(cb_ctx* c, float* buf, size_t n_per_rank, cudaStream_t s);
void comm_destroy(cb_ctx* c);
// Fused reduce-scatter of the head-parallel residual GEMMs (peer-memory mode): tp_push_on() says whether the
// o_proj / down_proj epilogues push their rows to the owners' receive planes (tp_push_params fills EpiParams);
// comm_allreduce_pushed then sums each rank's owned rows over the planes and writes them to every rank's h_out.
bool tp_push_on(const cb_ctx* c);
cb_status tp_push_params(cb_ctx* c, EpiParams& e, int rows);
cb_status comm_allreduce_pushed(cb_ctx* c, float* h_out, int rows, cudaStream_t s);
cb_status launch_gen_fill(void* out, int dtype, long long count, unsigned long long seed, unsigned long long stream_id,
                          long long start, float scale, float offset, cudaStream_t s);
