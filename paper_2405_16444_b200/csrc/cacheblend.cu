// cacheblend.cu — C-ABI of libcacheblend: context, argument checks, and the layer orchestration
// of the blend. Every step is a device kernel on the caller's stream;
// there is no host synchronisation inside cb_blend_layer / cb_blend_forward (all k_i are host
// integers, so every shape is static and the whole forward is CUDA-graph capturable).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <vector>

#include "ctx.h"

// ---- launchers implemented in the other translation units ----------------------------------------
cb_status launch_gemm_simt(cb_ctx* c, const void* A, int lda, const void* B, int ldb, int M, int K,
                           const EpiParams& e, cudaStream_t s);
cb_status launch_gemm_tc(cb_ctx* c, const void* A, int lda, const void* B, int ldb, int M, int K,
                         const EpiParams& e, cudaStream_t s);
bool gemm_tc_ok(const cb_ctx* c, const void* A, int lda, const void* B, int ldb, int M, int K, const EpiParams& e);
cb_status launch_attention_simt(cb_ctx* c, const void* q, const int* q_row, const int* q_tok, int n_rows,
                                const void* k, const void* v, int n_keys, void* out, cudaStream_t s);
cb_status launch_attention_tc5(cb_ctx* c, const void* q, const int* q_row, const int* q_tok, int n_rows,
                               const void* k, const void* v, int n_keys, void* out, cudaStream_t s);
bool attention_tc5_ok(const cb_ctx* c);
cb_status attention_tc5_init();
cb_status topk_init_attrs();
cb_status gemm_tc_init(cb_ctx* c);
void gemm_tc_destroy(cb_ctx* c);
void gemm_tc_force_bn(cb_ctx* c, int bn);
void gemm_tc_force_ksplit(cb_ctx* c, int v);
void gemm_tc_force_tail(cb_ctx* c, int v);
void gemm_tc_no192(cb_ctx* c, int v);
void gemm_tc_no224(cb_ctx* c, int v);
void gemm_tc_pairs_cap(cb_ctx* c, int kind, int v);
void gemm_tc_balance(cb_ctx* c, int v);
void gemm_tc_force_pair(cb_ctx* c, int v);
int gemm_tc_max_pairs(const cb_ctx* c);

// ---- error reporting ------------------------------------------------------------------------------
static thread_local char g_err[1024] = "";

void cb_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

extern "C" const char* cb_last_error(void) { return g_err; }

// ---- per-launch profile ---------------------------------------------------------------------------
static cudaEvent_t pool_event(cb_ctx* c) {
  if (!c->ev_pool.empty()) {
    cudaEvent_t e = c->ev_pool.back();
    c->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

ProfScope::ProfScope(cb_ctx* c_, int cls, cudaStream_t s_) : c(c_), s(s_), idx(-1) {
  if (!c || !c->prof_on) return;
  ProfRec r{cls, pool_event(c), pool_event(c)};
  cudaEventRecord(r.a, s);
  c->prof.push_back(r);
  idx = (int)c->prof.size() - 1;
}

ProfScope::~ProfScope() {
  if (idx >= 0) cudaEventRecord(c->prof[idx].b, s);
}

static const char* kProfNames[PROF_N] = {"realign", "embed", "rmsnorm", "gemm", "deviation", "topk", "scatter",
                                         "attention", "misc", "comm"};

extern "C" const char* cb_profile_class_name(int32_t cls) {
  return (cls >= 0 && cls < PROF_N) ? kProfNames[cls] : "";
}

extern "C" cb_status cb_profile_begin(cb_ctx* c) {
  CB_REQUIRE(c != nullptr, CB_E_INVALID_ARG, "ctx is NULL");
  for (auto& r : c->prof) { c->ev_pool.push_back(r.a); c->ev_pool.push_back(r.b); }
  c->prof.clear();
  c->prof_on = true;
  return CB_OK;
}

extern "C" cb_status cb_profile_end(cb_ctx* c, double* ms, int64_t* counts, int32_t n) {
  CB_REQUIRE(c != nullptr, CB_E_INVALID_ARG, "ctx is NULL");
  c->prof_on = false;
  CB_CUDA(cudaDeviceSynchronize());
  for (int i = 0; i < n; ++i) { if (ms) ms[i] = 0.0; if (counts) counts[i] = 0; }
  for (auto& r : c->prof) {
    float t = 0.f;
    CB_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
    if (r.cls < n) {
      if (ms) ms[r.cls] += t;
      if (counts) counts[r.cls] += 1;
    }
  }
  return CB_OK;
}

// ---- dispatch -------------------------------------------------------------------------------------
cb_status launch_gemm(cb_ctx* c, const void* A, int lda, const void* B, int ldb, int M, int K, const EpiParams& e,
                      int impl, cudaStream_t s) {
  if (M == 0 || e.N == 0) return CB_OK;
  if (impl == 2 || (impl == 0 && c->m.dtype == CB_BF16)) {
    if (gemm_tc_ok(c, A, lda, B, ldb, M, K, e)) return launch_gemm_tc(c, A, lda, B, ldb, M, K, e, s);
    CB_REQUIRE(impl != 2, CB_E_UNSUPPORTED, "tcgen05 GEMM does not take this shape (M=%d N=%d K=%d)", M, e.N, K);
  }
  CB_REQUIRE(e.norm_gain == nullptr && e.ss_in == nullptr, CB_E_UNSUPPORTED,
             "fused RMSNorm requested on a GEMM outside the tcgen05 path");
  return launch_gemm_simt(c, A, lda, B, ldb, M, K, e, s);
}

cb_status launch_attention(cb_ctx* c, const void* q, const int* q_row, const int* q_tok, int n_rows, const void* k,
                           const void* v, int n_keys, void* out, int impl, cudaStream_t s) {
  if (n_rows == 0) return CB_OK;
  if (impl == 0) impl = c->attn_impl;
  if (impl == 2 || (impl == 0 && attention_tc5_ok(c))) {
    CB_REQUIRE(attention_tc5_ok(c), CB_E_UNSUPPORTED, "tcgen05 attention needs bf16 and head_dim 128");
    return launch_attention_tc5(c, q, q_row, q_tok, n_rows, k, v, n_keys, out, s);
  }
  return launch_attention_simt(c, q, q_row, q_tok, n_rows, k, v, n_keys, out, s);
}

// ---- context --------------------------------------------------------------------------------------
namespace {
constexpr size_t kAlign = 256;

struct Carve {
  char* base;
  size_t off = 0;
  template <typename P> P* take(size_t bytes) {
    off = (off + kAlign - 1) / kAlign * kAlign;
    P* p = base ? reinterpret_cast<P*>(base + off) : nullptr;
    off += bytes;
    return p;
  }
};

cb_status check_model(const cb_model* m) {
  CB_REQUIRE(m != nullptr, CB_E_INVALID_ARG, "model is NULL");
  CB_REQUIRE(m->n_layers >= 1 && m->d_model >= 1 && m->n_q_heads >= 1 && m->n_kv_heads >= 1 && m->head_dim >= 2 &&
                 m->d_ff >= 1 && m->vocab >= 1,
             CB_E_INVALID_ARG, "model sizes must be positive");
  CB_REQUIRE(m->head_dim % 2 == 0, CB_E_INVALID_ARG, "head_dim must be even (paired RoPE rotation), got %d",
             m->head_dim);
  CB_REQUIRE(m->n_q_heads % m->n_kv_heads == 0, CB_E_INVALID_ARG, "n_q_heads %% n_kv_heads != 0");
  CB_REQUIRE(m->dtype == CB_BF16 || m->dtype == CB_FP32, CB_E_INVALID_ARG, "bad dtype %d", m->dtype);
  const int V = 16 / (int)dtype_bytes(m->dtype);
  CB_REQUIRE(m->head_dim % V == 0 && m->d_model % 8 == 0 && m->d_ff % 8 == 0, CB_E_UNSUPPORTED,
             "head_dim must be a multiple of %d and d_model, d_ff multiples of 8", V);
  CB_REQUIRE(m->head_dim <= 256, CB_E_UNSUPPORTED, "head_dim > 256");
  CB_REQUIRE(m->n_kv_heads <= 16, CB_E_UNSUPPORTED, "n_kv_heads > 16");
  CB_REQUIRE(m->d_model <= 8192, CB_E_UNSUPPORTED, "d_model > 8192");
  CB_REQUIRE(m->max_pos >= 1, CB_E_INVALID_ARG, "max_pos must be >= 1");
  CB_REQUIRE(m->rope_theta > 0.0 && m->rms_eps >= 0.f, CB_E_INVALID_ARG, "rope_theta/rms_eps out of range");
  return CB_OK;
}

size_t carve(cb_ctx* c, const cb_model* m, int T, char* base) {
  Carve cv{base};
  const size_t B = dtype_bytes(m->dtype);
  const size_t d = m->d_model, qd = (size_t)m->n_q_heads * m->head_dim, kvd = (size_t)m->n_kv_heads * m->head_dim;
  cb_ctx tmp;
  cb_ctx* o = c ? c : &tmp;
  o->h[0] = cv.take<float>((size_t)T * d * 4);
  o->h[1] = cv.take<float>((size_t)T * d * 4);
  o->x = cv.take<void>((size_t)T * d * B);
  o->q = cv.take<void>((size_t)T * qd * B);
  o->kf = cv.take<void>((size_t)T * kvd * B);
  o->vf = cv.take<void>((size_t)T * kvd * B);
  o->attn = cv.take<void>((size_t)T * qd * B);
  o->act = cv.take<void>((size_t)T * m->d_ff * B);
  o->dev = cv.take<float>((size_t)T * 4);
  o->dev_part = cv.take<float>((size_t)2 * ((kvd + 63) / 64) * T * 4);
  o->ss = cv.take<float>((size_t)T * ((d + 63) / 64) * 4);
  o->row_tok[0] = cv.take<int>((size_t)T * 4);
  o->row_tok[1] = cv.take<int>((size_t)T * 4);
  o->qrow = cv.take<int>((size_t)T * 4);
  o->iota = cv.take<int>((size_t)T * 4);
  o->src_pos = cv.take<int>((size_t)T * 4);
  o->tok_d = cv.take<int>((size_t)T * 4);
  o->pos_d = cv.take<int>((size_t)T * 4);
  // split-KV attention partials: room for every (row, q head) twice
  o->attn_part_rows = 2LL * T * m->n_q_heads;
  o->attn_part = cv.take<float>((size_t)o->attn_part_rows * m->head_dim * 4);
  o->attn_ml = cv.take<float2>((size_t)o->attn_part_rows * 8);
  o->attn_cnt_n = (int)(((long long)T * m->n_q_heads + 127) / 128 + m->n_kv_heads);
  o->attn_cnt = cv.take<int>((size_t)o->attn_cnt_n * 4);
  o->attn_work = cv.take<int>(64);
  return cv.off + kAlign;
}

__global__ void iota_kernel(int* p, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = i;
}

// row_tok = [cand_tok..., N, N+1, ..., N+n_suf-1]
__global__ void make_rows_kernel(const int* __restrict__ cand, int n_cand, int n_suf, int N, int* __restrict__ rows) {
  pdl_enter();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_cand + n_suf; i += gridDim.x * blockDim.x)
    rows[i] = i < n_cand ? cand[i] : N + (i - n_cand);
}
}  // namespace

extern "C" cb_status cb_workspace_size(const cb_model* model, int32_t max_tokens, size_t* bytes) {
  CB_TRY(check_model(model));
  CB_REQUIRE(bytes != nullptr && max_tokens >= 1, CB_E_INVALID_ARG, "bad arguments");
  *bytes = carve(nullptr, model, max_tokens, nullptr);
  return CB_OK;
}

extern "C" cb_status cb_create(const cb_model* model, int32_t max_tokens, void* workspace, size_t workspace_bytes,
                               cb_ctx** out) {
  CB_TRY(check_model(model));
  CB_REQUIRE(out != nullptr && max_tokens >= 1, CB_E_INVALID_ARG, "bad arguments to cb_create");
  *out = nullptr;
  const size_t need = carve(nullptr, model, max_tokens, nullptr);
  CB_REQUIRE(workspace == nullptr || workspace_bytes >= need, CB_E_WORKSPACE,
             "workspace too small: %zu < %zu bytes", workspace_bytes, need);
  cb_ctx* c = new cb_ctx();  // value-initialised: pointers null, counters zero
  c->m = *model;
  c->max_tokens = max_tokens;
  c->pdl = 1;
  c->tp_world = 1;
  cudaError_t e = cudaGetDevice(&c->device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device);
  int cc_major = 0, cc_minor = 0;
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&cc_major, cudaDevAttrComputeCapabilityMajor, c->device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&cc_minor, cudaDevAttrComputeCapabilityMinor, c->device);
  if (e != cudaSuccess) {
    delete c;
    CB_CUDA(e);
  }
  if (cc_major != 10 || cc_minor != 0) {
    delete c;
    cb_set_error("libcacheblend is built for sm_100a (B200); device is sm_%d%d", cc_major, cc_minor);
    return CB_E_UNSUPPORTED;
  }
  c->ws_bytes = need;
  if (workspace) {
    c->ws = workspace;
  } else {
    e = cudaMalloc(&c->ws, need);
    if (e != cudaSuccess) { delete c; CB_CUDA(e); }
    c->ws_owned = true;
  }
  char* base = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(c->ws) + kAlign - 1) / kAlign * kAlign);
  carve(c, model, max_tokens, base);

  // RoPE table in fp64 -> fp32: (cos, sin)(p theta_i), theta_i = base^(-2i/hd) (R8)
  const int half = model->head_dim / 2;
  std::vector<float2> tab((size_t)model->max_pos * half);
  for (int p = 0; p < model->max_pos; ++p)
    for (int i = 0; i < half; ++i) {
      const double th = std::pow(model->rope_theta, -2.0 * i / model->head_dim);
      const double a = (double)p * th;
      tab[(size_t)p * half + i] = make_float2((float)std::cos(a), (float)std::sin(a));
    }
  auto fail = [&](cudaError_t err) {
    cb_set_error("cb_create: %s", cudaGetErrorString(err));
    if (c->rope_tab) cudaFree(c->rope_tab);
    if (c->err_word) cudaFree(c->err_word);
    if (c->ws_owned) cudaFree(c->ws);
    delete c;
    return CB_E_CUDA;
  };
  if ((e = cudaMalloc(&c->rope_tab, tab.size() * sizeof(float2))) != cudaSuccess) return fail(e);
  if ((e = cudaMemcpy(c->rope_tab, tab.data(), tab.size() * sizeof(float2), cudaMemcpyHostToDevice)) != cudaSuccess)
    return fail(e);
  if ((e = cudaMalloc(&c->err_word, sizeof(int))) != cudaSuccess) return fail(e);
  if ((e = cudaMemset(c->err_word, 0, sizeof(int))) != cudaSuccess) return fail(e);
  if ((e = cudaMemset(c->attn_cnt, 0, (size_t)c->attn_cnt_n * sizeof(int))) != cudaSuccess) return fail(e);
  if ((e = cudaMemset(c->attn_work, 0, 64)) != cudaSuccess) return fail(e);
  iota_kernel<<<std::min(1024, (max_tokens + 255) / 256), 256>>>(c->iota, max_tokens);
  if ((e = cudaGetLastError()) != cudaSuccess) return fail(e);
  if ((e = cudaDeviceSynchronize()) != cudaSuccess) return fail(e);
  if ((e = cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking)) != cudaSuccess) return fail(e);
  if ((e = cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming)) != cudaSuccess) return fail(e);
  for (auto& ev : c->ev_realign)
    if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) return fail(e);
  if ((e = cudaStreamCreateWithFlags(&c->aux_stream, cudaStreamNonBlocking)) != cudaSuccess) return fail(e);
  c->layer_ev.resize(model->n_layers + 1);
  for (auto& ev : c->layer_ev)
    if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) return fail(e);
  cb_status st = topk_init_attrs();
  if (st == CB_OK) st = gemm_tc_init(c);
  if (st == CB_OK) st = attention_tc5_init();
  c->topk_drop_max = 48;
  c->epi_l1pf = 1;
  c->q_split = 1;    // layer 1: Q projected for the kept rows only, after the selection
  c->gemm_mc = 0;    // off: with the weights streaming from HBM the clusters no longer shorten the k-loop (paired
                     // A/B in four orders: -0.11 ms/step without them); 2 = planner-selected
  if (st != CB_OK) {
    cudaFree(c->rope_tab);
    cudaFree(c->err_word);
    if (c->ws_owned) cudaFree(c->ws);
    delete c;
    return st;
  }
  *out = c;
  return CB_OK;
}

extern "C" cb_status cb_destroy(cb_ctx* c) {
  if (!c) return CB_OK;
  cudaDeviceSynchronize();
  for (auto& r : c->prof) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  for (auto ev : c->ev_pool) cudaEventDestroy(ev);
  for (auto ev : c->layer_ev) if (ev) cudaEventDestroy(ev);
  if (c->ev_ready) cudaEventDestroy(c->ev_ready);
  for (auto ev : c->ev_realign) if (ev) cudaEventDestroy(ev);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  if (c->aux_stream) cudaStreamDestroy(c->aux_stream);
  if (c->dbg_buf) cudaFree(c->dbg_buf);
  comm_destroy(c);
  gemm_tc_destroy(c);
  cudaFree(c->rope_tab);
  cudaFree(c->err_word);
  if (c->ws_owned) cudaFree(c->ws);
  delete c;
  return CB_OK;
}

extern "C" cb_status cb_check_device_errors(cb_ctx* c) {
  CB_REQUIRE(c != nullptr, CB_E_INVALID_ARG, "ctx is NULL");
  int h = 0;
  CB_CUDA(cudaMemcpy(&h, c->err_word, sizeof(int), cudaMemcpyDeviceToHost));
  CB_CUDA(cudaMemset(c->err_word, 0, sizeof(int)));
  if (h & CB_DEVERR_FORCE_SEL) { cb_set_error("device: a force_sel token is not a candidate of its layer"); return CB_E_DEVICE; }
  if (h & CB_DEVERR_POS_RANGE) {
    cb_set_error("device: a position is outside [0, max_pos) (pos, or |dst_pos - src_pos| in realign)");
    return CB_E_DEVICE;
  }
  if (h & CB_DEVERR_POS_ORDER) {
    cb_set_error("device: global positions are not strictly increasing (the attention mask orders keys by token index)");
    return CB_E_DEVICE;
  }
  if (h & CB_DEVERR_PAGE) { cb_set_error("device: a block_table page id is outside [0, n_pages) (nothing written there)"); return CB_E_DEVICE; }
  if (h & CB_DEVERR_COMM) { cb_set_error("device: a peer-memory collective timed out waiting for a rank"); return CB_E_DEVICE; }
  return CB_OK;
}

extern "C" int64_t cb_launch_count(cb_ctx* c) { return c ? c->launches : 0; }

extern "C" cb_status cb_debug_fetch(cb_ctx* c, int64_t* host, int32_t n) {
  CB_REQUIRE(c && host && n >= 0 && n <= 2048, CB_E_INVALID_ARG, "cb_debug_fetch: bad arguments");
  CB_REQUIRE(c->dbg_buf != nullptr, CB_E_INVALID_ARG, "debug_trace is off");
  CB_CUDA(cudaMemcpy(host, c->dbg_buf, (size_t)n * sizeof(long long), cudaMemcpyDeviceToHost));
  return CB_OK;
}

extern "C" cb_status cb_get_info(cb_ctx* c, const char* name, int64_t* value) {
  CB_REQUIRE(c && name && value, CB_E_INVALID_ARG, "cb_get_info: NULL argument");
  if (std::strcmp(name, "num_sms") == 0) { *value = c->num_sms; return CB_OK; }
  if (std::strcmp(name, "gemm_max_pairs") == 0) { *value = gemm_tc_max_pairs(c); return CB_OK; }
  if (std::strcmp(name, "gemm_max_clusters4") == 0) { *value = c->max_clusters4; return CB_OK; }
  if (std::strcmp(name, "gemm_max_clusters8") == 0) { *value = c->max_clusters8; return CB_OK; }
  cb_set_error("unknown info '%s'", name);
  return CB_E_INVALID_ARG;
}

extern "C" cb_status cb_set_option(cb_ctx* c, const char* name, int64_t value) {
  CB_REQUIRE(c != nullptr && name != nullptr, CB_E_INVALID_ARG, "ctx / name is NULL");
  if (std::strcmp(name, "gemm_sched") == 0) {
    CB_REQUIRE(value >= 0 && value <= 2, CB_E_INVALID_ARG, "gemm_sched must be 0, 1 or 2");
    c->gemm_sched = (int)value;
    return CB_OK;
  }
  if (std::strcmp(name, "pdl") == 0) {
    c->pdl = value != 0;
    return CB_OK;
  }
  if (std::strcmp(name, "debug_trace") == 0) {
    c->dbg_sel = (int)value;
    if (value && !c->dbg_buf) {
      CB_CUDA(cudaMalloc(&c->dbg_buf, 2048 * sizeof(long long)));
      CB_CUDA(cudaMemset(c->dbg_buf, 0, 2048 * sizeof(long long)));
    } else if (!value && c->dbg_buf) {
      cudaFree(c->dbg_buf);
      c->dbg_buf = nullptr;
    }
    return CB_OK;
  }
  if (std::strcmp(name, "fuse_norm") == 0) {
    c->no_fuse_norm = value == 0;
    return CB_OK;
  }
  if (std::strcmp(name, "fuse_deviation") == 0) {
    c->no_fuse_dev = value == 0;
    return CB_OK;
  }
  if (std::strcmp(name, "realign_overlap") == 0) {
    c->realign_overlap = value != 0;
    return CB_OK;
  }
  if (std::strcmp(name, "tp_fuse") == 0) {
    CB_REQUIRE(c->xblock == nullptr, CB_E_INVALID_ARG, "set tp_fuse before cb_tp_p2p_enable");
    c->tp_nofuse = value == 0;
    return CB_OK;
  }
  if (std::strcmp(name, "attn_splits") == 0) {
    CB_REQUIRE(value >= 0 && value <= 16, CB_E_INVALID_ARG, "attn_splits must be 0..16");
    c->attn_splits = (int)value;
    return CB_OK;
  }
  if (std::strcmp(name, "attn_impl") == 0) {
    CB_REQUIRE(value == 0 || value == 1 || value == 2, CB_E_INVALID_ARG, "attn_impl must be 0 (auto), 1 (SIMT) or 2 (tcgen05)");
    c->attn_impl = (int)value;
    return CB_OK;
  }
  if (std::strcmp(name, "gemm_pair") == 0) {
    CB_REQUIRE(value >= 0 && value <= 2, CB_E_INVALID_ARG, "gemm_pair must be 0, 1 or 2");
    gemm_tc_force_pair(c, (int)value);
    return CB_OK;
  }
  if (std::strcmp(name, "gemm_no224") == 0) {
    gemm_tc_no224(c, (int)value);
    return CB_OK;
  }
  if (std::strcmp(name, "gemm_no192") == 0) {
    gemm_tc_no192(c, (int)value);
    return CB_OK;
  }
  {
    static const char* kCap[5] = {"gemm_cap_store", "gemm_cap_store_f32", "gemm_cap_qkv", "gemm_cap_resid",
                                  "gemm_cap_swiglu"};
    static const int kKind[5] = {EPI_STORE, EPI_STORE_F32, EPI_QKV, EPI_RESID, EPI_SWIGLU};
    for (int i = 0; i < 5; ++i)
      if (std::strcmp(name, kCap[i]) == 0) {
        CB_REQUIRE(value >= 0, CB_E_INVALID_ARG, "%s must be >= 0", name);
        gemm_tc_pairs_cap(c, kKind[i], (int)value);
        return CB_OK;
      }
  }
  if (std::strcmp(name, "gemm_balance") == 0) {
    gemm_tc_balance(c, (int)value);
    return CB_OK;
  }
  if (std::strcmp(name, "topk_threads") == 0) {
    CB_REQUIRE(value == 0 || value == 256 || value == 512 || value == 1024, CB_E_INVALID_ARG,
               "topk_threads must be 0, 256, 512 or 1024");
    c->topk_threads = (int)value;
    return CB_OK;
  }
  if (std::strcmp(name, "gemm_mc") == 0) {
    CB_REQUIRE(value >= 0 && value <= 3, CB_E_INVALID_ARG, "gemm_mc must be 0, 1, 2 or 3");
    c->gemm_mc = (int)value;
    return CB_OK;
  }
  if (std::strcmp(name, "epi_l1pf") == 0) {
    c->epi_l1pf = value != 0;
    return CB_OK;
  }
  if (std::strcmp(name, "q_split") == 0) {
    c->q_split = value != 0;
    return CB_OK;
  }
  if (std::strcmp(name, "topk_drop") == 0) {
    c->topk_drop_max = (int)value;
    return CB_OK;
  }
  if (std::strcmp(name, "gemm_tail") == 0) {
    CB_REQUIRE(value >= 0 && value <= 2, CB_E_INVALID_ARG, "gemm_tail must be 0, 1 or 2");
    gemm_tc_force_tail(c, (int)value);
    return CB_OK;
  }
  if (std::strcmp(name, "gemm_ksplit") == 0) {
    CB_REQUIRE(value >= 0 && value <= 4, CB_E_INVALID_ARG, "gemm_ksplit must be 0..4");
    gemm_tc_force_ksplit(c, (int)value);
    return CB_OK;
  }
  if (std::strcmp(name, "gemm_bn") == 0) {
    CB_REQUIRE(value == 0 || value == 128 || value == 192 || value == 224 || value == 256, CB_E_INVALID_ARG,
               "gemm_bn must be 0, 128, 192 (CTA pairs), 224 (SwiGLU pairs) or 256");
    gemm_tc_force_bn(c, (int)value);
    return CB_OK;
  }
  cb_set_error("unknown option '%s'", name);
  return CB_E_INVALID_ARG;
}

// ---- loading controller (host; §6 "Loading Controller") ---------------------------------
extern "C" cb_status cb_controller_ratio(double prefill_ms, double kv_bytes_per_token, int64_t n_tokens,
                                         double bytes_per_ms, double r_min, double* r_out, double* load_ms_out) {
  CB_REQUIRE(r_out != nullptr, CB_E_INVALID_ARG, "r_out is NULL");
  CB_REQUIRE(prefill_ms > 0.0 && bytes_per_ms > 0.0 && kv_bytes_per_token >= 0.0 && n_tokens >= 0, CB_E_INVALID_ARG,
             "controller: need prefill_ms > 0, bytes_per_ms > 0, kv_bytes_per_token >= 0, n_tokens >= 0");
  CB_REQUIRE(r_min >= 0.0 && r_min <= 1.0, CB_E_INVALID_ARG, "r_min %g outside [0, 1]", r_min);
  const double load_ms = kv_bytes_per_token * (double)n_tokens / bytes_per_ms;  // T_load (footnote P:2696)
  const double r_eq = load_ms / prefill_ms;  // T_recompute(r_eq) = r_eq * Prefill = T_load
  *r_out = std::min(1.0, std::max(r_eq, r_min));  // max(r%, r*%)
  if (load_ms_out) *load_ms_out = load_ms;
  return CB_OK;
}

extern "C" cb_status cb_controller_pick_device(double prefill_ms, const double* load_ms, const double* cost,
                                               int32_t n_dev, double r_fixed, int32_t* pick_out) {
  CB_REQUIRE(pick_out != nullptr && n_dev >= 0 && (n_dev == 0 || (load_ms && cost)), CB_E_INVALID_ARG,
             "controller: bad device arrays");
  CB_REQUIRE(prefill_ms > 0.0 && r_fixed >= 0.0 && r_fixed <= 1.0, CB_E_INVALID_ARG, "controller: bad ratio / prefill");
  const double t_rec = r_fixed * prefill_ms;
  int best = -1;
  for (int d = 0; d < n_dev; ++d)  // cheapest device with T_recompute >= T_load; ties -> earlier
    if (t_rec >= load_ms[d] && (best < 0 || cost[d] < cost[best])) best = d;
  *pick_out = best;
  return CB_OK;
}

extern "C" cb_status cb_controller_schedule(double prefill_ms, double kv_bytes_per_token, double bytes_per_ms,
                                            double r_min, int32_t n_ctx, int32_t n_layers, int32_t* k_sched_out,
                                            double* r_out, double* load_ms_out) {
  CB_REQUIRE(k_sched_out != nullptr, CB_E_INVALID_ARG, "k_sched_out is NULL");
  double r = 0.0, ld = 0.0;
  CB_TRY(cb_controller_ratio(prefill_ms, kv_bytes_per_token, n_ctx, bytes_per_ms, r_min, &r, &ld));
  CB_TRY(cb_schedule(r, n_ctx, n_layers, k_sched_out));
  if (r_out) *r_out = r;
  if (load_ms_out) *load_ms_out = ld;
  return CB_OK;
}

// ---- schedule (host) ----------------------------------------------------------------------------
extern "C" cb_status cb_schedule(double ratio, int32_t n_ctx, int32_t n_layers, int32_t* k) {
  CB_REQUIRE(k != nullptr && n_layers >= 1 && n_ctx >= 0, CB_E_INVALID_ARG, "bad arguments to cb_schedule");
  CB_REQUIRE(ratio >= 0.0 && ratio <= 1.0, CB_E_INVALID_ARG, "ratio %g outside [0, 1]", ratio);
  k[0] = n_ctx;
  const double delta = 0.2 * std::min(ratio, 1.0 - ratio);
  for (int i = 1; i < n_layers; ++i) {
    double ri = ratio;
    if (n_layers != 2) {
      volatile double t = 2.0 * (double)(i - 1) / (double)(n_layers - 2);  // keep the oracle's op order
      volatile double u = delta * (1.0 - t);
      ri = ratio + u;
    }
    volatile double x = ri * (double)n_ctx;
    long long ki = (long long)std::ceil(x - 1e-9);
    ki = std::min<long long>(ki, n_ctx);
    ki = std::min<long long>(ki, k[i - 1]);
    k[i] = (int32_t)std::max<long long>(0, ki);
  }
  return CB_OK;
}

// ---- building-block entry points (cacheblend_ops.h) ---------------------------------------------
extern "C" cb_status cb_op_embed(cb_ctx* c, const void* embed, const int32_t* tok, int32_t n, float* h, void* st) {
  CB_REQUIRE(c && embed && tok && h && n >= 0, CB_E_INVALID_ARG, "cb_op_embed: bad arguments");
  return launch_embed(c, embed, tok, n, h, (cudaStream_t)st);
}

extern "C" cb_status cb_op_rmsnorm(cb_ctx* c, const float* h, const float* gain, int32_t n_rows, void* x, void* st) {
  CB_REQUIRE(c && h && gain && x && n_rows >= 0, CB_E_INVALID_ARG, "cb_op_rmsnorm: bad arguments");
  return launch_rmsnorm(c, h, gain, n_rows, x, (cudaStream_t)st);
}

extern "C" cb_status cb_op_gemm(cb_ctx* c, const void* A, const void* B, void* C, int32_t M, int32_t N, int32_t K,
                                int32_t out_f32, int32_t impl, void* st) {
  CB_REQUIRE(c && A && B && C && M >= 0 && N >= 0 && K >= 1, CB_E_INVALID_ARG, "cb_op_gemm: bad arguments");
  CB_REQUIRE(impl >= 0 && impl <= 2, CB_E_INVALID_ARG, "cb_op_gemm: impl must be 0, 1 or 2");
  CB_REQUIRE(N % 2 == 0 && K % 8 == 0, CB_E_SHAPE, "cb_op_gemm: N must be even and K a multiple of 8");
  CB_REQUIRE(out_f32 >= 0 && out_f32 <= 2, CB_E_INVALID_ARG, "cb_op_gemm: out_f32 must be 0, 1 or 2");
  EpiParams e{};
  e.kind = out_f32 == 2 ? EPI_RESID : out_f32 ? EPI_STORE_F32 : EPI_STORE;
  e.M = M; e.N = N; e.ldo = N;
  e.out = C; e.outf = (float*)C;
  e.h_out = (float*)C; e.h_in = (const float*)C; e.res_row = nullptr;
  return launch_gemm(c, A, K, B, K, M, K, e, impl, (cudaStream_t)st);
}

extern "C" cb_status cb_op_attention(cb_ctx* c, const void* q, const int32_t* q_row, const int32_t* q_tok,
                                     int32_t n_rows, const void* k, const void* v, int32_t n_keys, void* out,
                                     int32_t impl, void* st) {
  CB_REQUIRE(c && q && q_row && q_tok && k && v && out && n_rows >= 0 && n_keys >= 1, CB_E_INVALID_ARG,
             "cb_op_attention: bad arguments");
  CB_REQUIRE(impl >= 0 && impl <= 4, CB_E_INVALID_ARG, "cb_op_attention: impl must be 0..4");
  return launch_attention(c, q, q_row, q_tok, n_rows, k, v, n_keys, out, impl, (cudaStream_t)st);
}

// ---- (a) realign ----------------------------------------------------------------------------------
extern "C" cb_status cb_rope_realign(cb_ctx* c, void* k_out, const void* k_src, const int32_t* src_pos,
                                     const int32_t* dst_pos, int32_t n_slices, int32_t n_tok, int64_t slice_stride,
                                     void* st) {
  CB_REQUIRE(c != nullptr, CB_E_INVALID_ARG, "ctx is NULL");
  CB_REQUIRE(n_slices >= 0 && n_tok >= 0, CB_E_INVALID_ARG, "negative sizes");
  if (n_slices == 0 || n_tok == 0) return CB_OK;
  CB_REQUIRE(k_out && k_src && src_pos && dst_pos, CB_E_INVALID_ARG, "cb_rope_realign: NULL pointer");
  const long long kvd = (long long)c->m.n_kv_heads * c->m.head_dim;
  CB_REQUIRE(slice_stride >= (long long)n_tok * kvd || n_slices == 1, CB_E_SHAPE,
             "slice_stride %lld < n_tok * n_kv * head_dim", (long long)slice_stride);
  return launch_realign(c, k_out, k_src, nullptr, nullptr, src_pos, dst_pos, n_slices, n_tok, slice_stride,
                        slice_stride, (cudaStream_t)st);
}

// ---- (b) deviation + top-k -----------------------------------------------------------------------
extern "C" cb_status cb_kv_deviation_topk(cb_ctx* c, const void* k_new, const void* v_new, const void* k_ref,
                                          const void* v_ref, const int32_t* cand_tok, int32_t n_cand, int32_t k_keep,
                                          int32_t dev_mode, int32_t* sel_tok, int32_t* sel_slot, float* dev_out,
                                          void* st) {
  CB_REQUIRE(c != nullptr, CB_E_INVALID_ARG, "ctx is NULL");
  CB_REQUIRE(n_cand >= 0 && k_keep >= 0 && k_keep <= n_cand, CB_E_INVALID_ARG,
             "need 0 <= k_keep <= n_cand (k_keep=%d n_cand=%d)", k_keep, n_cand);
  CB_REQUIRE(n_cand <= c->max_tokens, CB_E_SHAPE, "n_cand %d > max_tokens %d", n_cand, c->max_tokens);
  CB_REQUIRE(dev_mode >= CB_DEV_KV && dev_mode <= CB_DEV_V, CB_E_INVALID_ARG, "bad dev_mode %d", dev_mode);
  if (n_cand == 0) return CB_OK;
  CB_REQUIRE(k_new && v_new && k_ref && v_ref && cand_tok, CB_E_INVALID_ARG, "NULL input pointer");
  CB_REQUIRE(k_keep == 0 || (sel_tok && sel_slot), CB_E_INVALID_ARG, "sel_tok / sel_slot are NULL");
  cudaStream_t s = (cudaStream_t)st;
  float* dev = dev_out ? dev_out : c->dev;
  CB_TRY(launch_deviation(c, k_new, v_new, k_ref, v_ref, cand_tok, n_cand, dev_mode, dev, s));
  CB_TRY(launch_topk(c, dev, cand_tok, n_cand, k_keep, 0, 0, nullptr, sel_slot ? sel_slot : c->qrow,
                     sel_tok ? sel_tok : c->row_tok[1], nullptr, s));
  return CB_OK;
}

// ---- (c) one layer ---------------------------------------------------------------------------------
namespace {
struct LayerBufs {
  const float* h_in;   // [rows][d]
  float* h_out;        // [k + n_suf][d]
  const int* row_tok;  // [n_cand + n_suf]
  int* qtok;           // [k + n_suf] out
  bool x_ready = false;                 // c->x / c->ss already hold this layer's fused attention RMSNorm
  bool x_normed = false;                // c->x already holds rmsnorm(h_in) * attn_norm (embed_norm, layer 0)
  const void* next_attn_norm = nullptr;  // next layer's attention-norm gain: fuse it into the down projection
  bool* next_ready = nullptr;           // out: set when the down projection produced the next layer's norm
};

// RMSNorm fusion (R15): the residual GEMM writes y = bf16(h * gain) plus 64-column sums of h^2 and the
// next projection scales its accumulator rows by 1/rms. Needs the tcgen05 path on both GEMMs.
// Head-parallel ranks hold partial sums of h until the all-reduce, so RMSNorm runs after it (replicated).
bool norm_fusable(const cb_ctx* c) {
  return !c->no_fuse_norm && c->m.dtype == CB_BF16 && c->m.d_model % 512 == 0 && c->tp_world <= 1;
}

// Head-parallel residual GEMM (o_proj / down_proj with a row shard of the contraction): rank 0 adds the
// residual, the other ranks store their partial product; comm_allreduce_f32 then sums the ranks.
void tp_partial_resid(const cb_ctx* c, EpiParams& e) {
  if (c->tp_world <= 1 || c->tp_rank == 0) return;
  e.kind = EPI_STORE_F32;
  e.outf = e.h_out;
  e.h_in = nullptr;
  e.res_row = nullptr;
}

void set_norm_producer(const cb_ctx* c, EpiParams& e, const void* gain) {
  e.norm_gain = (const float*)gain; e.y_out = c->x; e.ss_out = c->ss; e.ld_ss = c->m.d_model / 64;
}
void set_norm_consumer(const cb_ctx* c, EpiParams& e) {
  e.ss_in = c->ss; e.ld_ss = c->m.d_model / 64; e.norm_d = c->m.d_model; e.norm_eps = c->m.rms_eps;
}

// Both GEMMs of a fused RMSNorm take the tcgen05 path (otherwise the classic kernel runs).
bool norm_pair_ok(cb_ctx* c, const void* A1, int lda1, const void* B1, int M1, int K1, const EpiParams& e1,
                  const void* B2, int K2, const EpiParams& e2) {
  return norm_fusable(c) && gemm_tc_ok(c, A1, lda1, B1, lda1, M1, K1, e1) &&
         gemm_tc_ok(c, c->x, c->m.d_model, B2, c->m.d_model, M1, K2, e2);
}

// Rows 0..Q-1 after attention: W_o + residual (gathered through res_row), RMSNorm, SwiGLU MLP +
// residual. The RMSNorms are fused into the residual epilogues when both GEMMs allow it, and
// the down projection also prepares the next layer's attention RMSNorm (b.next_attn_norm).
cb_status mlp_block(cb_ctx* c, const cb_layer_w& w, const LayerBufs& b, int Q, const int* res_row, cudaStream_t s) {
  const cb_model& m = c->m;
  const int d = m.d_model, qd = m.n_q_heads * m.head_dim;
  EpiParams eo{};
  eo.kind = EPI_RESID; eo.M = Q; eo.N = d; eo.ldo = d; eo.h_in = b.h_in; eo.h_out = b.h_out; eo.res_row = res_row;
  EpiParams eg{};
  eg.kind = EPI_SWIGLU; eg.M = Q; eg.N = m.d_ff; eg.ff = m.d_ff; eg.act = c->act;
  const bool fuse_mlp = norm_pair_ok(c, c->attn, qd, w.w_o, Q, qd, eo, w.w_gate_up, d, eg);
  if (fuse_mlp) {
    set_norm_producer(c, eo, w.mlp_norm);
    set_norm_consumer(c, eg);
  }
  tp_partial_resid(c, eo);
  const bool push = tp_push_on(c);  // peer-memory mode: the epilogue pushes each row to its owner (fused RS)
  if (push) CB_TRY(tp_push_params(c, eo, Q));
  CB_TRY(launch_gemm(c, c->attn, qd, w.w_o, qd, Q, qd, eo, 0, s));
  if (push) CB_TRY(comm_allreduce_pushed(c, b.h_out, Q, s));               // (ii) after o_proj
  else CB_TRY(comm_allreduce_f32(c, b.h_out, (size_t)Q * d, s));
  if (!fuse_mlp) CB_TRY(launch_rmsnorm(c, b.h_out, (const float*)w.mlp_norm, Q, c->x, s));
  EpiParams ed{};
  ed.kind = EPI_RESID; ed.M = Q; ed.N = d; ed.ldo = d; ed.h_in = b.h_out; ed.h_out = b.h_out; ed.res_row = nullptr;
  const bool fuse_next = b.next_attn_norm != nullptr && norm_fusable(c) &&
                         gemm_tc_ok(c, c->act, m.d_ff, w.w_down, m.d_ff, Q, m.d_ff, ed);
  if (fuse_next) set_norm_producer(c, ed, b.next_attn_norm);
  if (c->tp_world > 1) {  // (iii) Megatron MLP: column-sharded gate/up, row-sharded down, one all-reduce
    tp_partial_resid(c, ed);
    if (push) CB_TRY(tp_push_params(c, ed, Q));
    CB_TRY(launch_gemm(c, c->x, d, w.w_gate_up, d, Q, d, eg, 0, s));
    CB_TRY(launch_gemm(c, c->act, m.d_ff, w.w_down, m.d_ff, Q, m.d_ff, ed, 0, s));
    return push ? comm_allreduce_pushed(c, b.h_out, Q, s) : comm_allreduce_f32(c, b.h_out, (size_t)Q * d, s);
  }
  CB_TRY(launch_gemm(c, c->x, d, w.w_gate_up, d, Q, d, eg, 0, s));
  CB_TRY(launch_gemm(c, c->act, m.d_ff, w.w_down, m.d_ff, Q, m.d_ff, ed, 0, s));
  if (fuse_next && b.next_ready) *b.next_ready = true;
  return CB_OK;
}

// Layer 0, the full layer (R2): every row is a query; context rows keep the realigned cache
// (P:1750), suffix rows write fresh K,V.
// before_kv (request mode): runs after the projections, before anything reads this layer's cached K/V
// (the fetch of layer 0's chunk KV then overlaps the embedding and the Q projection).
cb_status layer_full(cb_ctx* c, const cb_layer_w& w, const LayerBufs& b, int N, int n_suf, void* kb, void* vb,
                     const int* pos, cudaStream_t s, const std::function<cb_status()>& before_kv = nullptr) {
  const cb_model& m = c->m;
  const int T = N + n_suf, d = m.d_model, qd = m.n_q_heads * m.head_dim, kvd = m.n_kv_heads * m.head_dim;
  const size_t B = dtype_bytes(m.dtype);
  EpiParams e{};
  e.kind = EPI_QKV; e.M = T; e.N = qd; e.col0 = 0; e.qd = qd; e.kvd = kvd; e.hd = m.head_dim;
  e.q_out = c->q; e.row_tok = b.row_tok; e.pos = pos; e.rope_tab = c->rope_tab; e.max_pos = c->m.max_pos;
  if (b.x_ready && gemm_tc_ok(c, c->x, d, w.w_qkv, d, T, d, e)) set_norm_consumer(c, e);
  else if (!b.x_normed) CB_TRY(launch_rmsnorm(c, b.h_in, (const float*)w.attn_norm, T, c->x, s));
  CB_TRY(launch_gemm(c, c->x, d, w.w_qkv, d, T, d, e, 0, s));
  if (n_suf > 0) {
    EpiParams ek = e;
    ek.M = n_suf; ek.N = 2 * kvd; ek.col0 = qd;
    ek.k_out = (char*)kb + (size_t)N * kvd * B;
    ek.v_out = (char*)vb + (size_t)N * kvd * B;
    ek.row_tok = b.row_tok + N;
    if (ek.ss_in) ek.ss_in += (size_t)N * ek.ld_ss;
    CB_TRY(launch_gemm(c, (const char*)c->x + (size_t)N * d * B, d, (const char*)w.w_qkv + (size_t)qd * d * B, d,
                       n_suf, d, ek, 0, s));
  }
  if (before_kv) CB_TRY(before_kv());
  CB_TRY(launch_attention(c, c->q, c->iota, b.row_tok, T, kb, vb, T, c->attn, 0, s));
  return mlp_block(c, w, b, T, nullptr, s);
}

// Layers i >= 1: selective recompute with HKVD selection.
cb_status layer_blend(cb_ctx* c, const cb_layer_w& w, const LayerBufs& b, int n_cand, int k, int n_suf, int N,
                      void* kb, void* vb, const int* pos, const int* force_sel, int* sel_tok, float* dev_out,
                      int dev_mode, cudaStream_t s) {
  const cb_model& m = c->m;
  const int R = n_cand + n_suf, Q = k + n_suf;
  const int d = m.d_model, qd = m.n_q_heads * m.head_dim, kvd = m.n_kv_heads * m.head_dim;
  if (R == 0) return CB_OK;
  // 1. mask the input to the candidate rows and transform them into Q, K, V
  EpiParams e{};
  e.kind = EPI_QKV; e.M = R; e.N = qd + 2 * kvd; e.col0 = 0; e.qd = qd; e.kvd = kvd; e.hd = m.head_dim;
  e.q_out = c->q; e.k_out = c->kf; e.v_out = c->vf; e.row_tok = b.row_tok; e.pos = pos; e.rope_tab = c->rope_tab; e.max_pos = c->m.max_pos;
  if (b.x_ready && gemm_tc_ok(c, c->x, d, w.w_qkv, d, R, d, e)) set_norm_consumer(c, e);
  else CB_TRY(launch_rmsnorm(c, b.h_in, (const float*)w.attn_norm, R, c->x, s));
  // 2. Delta_kv against the loaded entries: fused into the tcgen05 QKV epilogue when every
  //    k/v head lies inside one output tile, else a separate kernel
  // (64-column deviation blocks: every GEMM tile edge and the q|k|v boundaries fall on a block edge)
  const bool fuse_dev = m.dtype == CB_BF16 && gemm_tc_ok(c, c->x, d, w.w_qkv, d, R, d, e) && qd % 64 == 0 &&
                        kvd % 64 == 0 && n_cand > 0 && !c->no_fuse_dev;
  // head-parallel: this rank's (64-column block, k|v) partials land in its segment of the gathered buffer;
  // the global block order (rank-major = kv-head-major) is the single-GPU order, so all ranks sum alike
  const size_t nb_local = (size_t)(kvd + 63) / 64;
  float* dev_part = c->tp_world > 1 ? c->dev_gath : c->dev_part;
  if (fuse_dev) {
    e.k_ref = kb; e.v_ref = vb; e.n_cand = n_cand; e.ld_part = c->max_tokens;
    e.dev_part = dev_part + (c->tp_world > 1 ? 2 * nb_local * c->tp_rank * c->max_tokens : 0);
  }
  // Q is only needed for the kept rows (the HKVD queries). Where the selection drops many
  // candidates (layer 1: C_1 = all tokens, |S_1| ~ r N) project K, V for every candidate (Delta_kv needs
  // them) and Q after the top-k, for the kept rows only.
  const size_t B = dtype_bytes(m.dtype);
  const bool split_q = fuse_dev && c->q_split && Q > 0 && 4 * (n_cand - k) > n_cand;
  EpiParams eq = e;
  if (split_q) {
    e.col0 = qd; e.N = 2 * kvd;
    CB_TRY(launch_gemm(c, c->x, d, (const char*)w.w_qkv + (size_t)qd * d * B, d, R, d, e, 0, s));
  } else {
    CB_TRY(launch_gemm(c, c->x, d, w.w_qkv, d, R, d, e, 0, s));
  }
  if (fuse_dev) CB_TRY(comm_allgather_f32(c, dev_part, 2 * nb_local * c->max_tokens, s));  // (i)
  // 3. HKVD = top-k of Delta_kv (Insight 1)
  float* dev = dev_out ? dev_out : c->dev;
  if (!fuse_dev) {
    CB_TRY(launch_deviation(c, c->kf, c->vf, kb, vb, b.row_tok, n_cand, dev_mode, dev, s));
    CB_TRY(comm_allreduce_f32(c, dev, (size_t)n_cand, s));  // (i) unfused: sum the ranks' head sums
  }
  CB_TRY(launch_topk(c, dev, b.row_tok, n_cand, k, n_suf, N, force_sel, c->qrow, b.qtok, sel_tok, s,
                     fuse_dev ? dev_part : nullptr, c->max_tokens, dev_mode));
  if (Q == 0) return CB_OK;
  // 4. only the KV of the HKVD tokens (and the suffix) is updated (R3)
  CB_TRY(launch_scatter_kv(c, c->kf, c->vf, c->qrow, b.qtok, Q, kb, vb, s));
  const int* q_rows = c->qrow;  // row of each kept query in c->q
  if (split_q) {
    // the kept rows of the projection input (and their RMSNorm blocks) gathered, then Q over them:
    // c->act and c->attn are free until the attention / MLP of this layer
    float* ssq = eq.ss_in ? reinterpret_cast<float*>(c->attn) : nullptr;
    CB_TRY(launch_gather_rows(c, c->x, eq.ss_in, c->qrow, Q, eq.ld_ss, c->act, ssq, s));
    eq.M = Q; eq.N = qd; eq.col0 = 0; eq.row_tok = b.qtok; eq.ss_in = ssq;
    eq.dev_part = nullptr; eq.k_ref = nullptr; eq.v_ref = nullptr; eq.n_cand = 0;
    CB_TRY(launch_gemm(c, c->act, d, w.w_qkv, d, Q, d, eq, 0, s));
    q_rows = c->iota;
  }
  // 5. attention of the selected queries over all tokens, then W_o + residual, MLP + residual
  CB_TRY(launch_attention(c, c->q, q_rows, b.qtok, Q, kb, vb, N + n_suf, c->attn, 0, s));
  return mlp_block(c, w, b, Q, c->qrow, s);
}

cb_status check_weights(const cb_layer_w* w) {
  CB_REQUIRE(w && w->attn_norm && w->w_qkv && w->w_o && w->mlp_norm && w->w_gate_up && w->w_down, CB_E_INVALID_ARG,
             "NULL weight pointer");
  return CB_OK;
}
}  // namespace

extern "C" cb_status cb_blend_layer(cb_ctx* c, int32_t layer, const cb_layer_w* w, float* h, const int32_t* cand_tok,
                                    int32_t n_cand, int32_t k_keep, int32_t n_suffix, void* k_blend, void* v_blend,
                                    const int32_t* pos, int32_t N, const int32_t* force_sel, int32_t* sel_tok,
                                    float* dev_out, void* st) {
  CB_REQUIRE(c != nullptr, CB_E_INVALID_ARG, "ctx is NULL");
  CB_TRY(check_weights(w));
  CB_REQUIRE(layer >= 0 && layer < c->m.n_layers, CB_E_INVALID_ARG, "layer %d out of range", layer);
  CB_REQUIRE(n_cand >= 0 && n_suffix >= 0 && N >= 0 && k_keep >= 0 && k_keep <= n_cand && n_cand <= N,
             CB_E_INVALID_ARG, "need 0 <= k_keep <= n_cand <= N, n_suffix >= 0");
  CB_REQUIRE(N + n_suffix <= c->max_tokens, CB_E_SHAPE, "N + n_suffix = %d > max_tokens %d", N + n_suffix,
             c->max_tokens);
  CB_REQUIRE(N + n_suffix >= 1, CB_E_INVALID_ARG, "empty input");
  CB_REQUIRE(h && k_blend && v_blend && pos, CB_E_INVALID_ARG, "NULL pointer");
  CB_REQUIRE(n_cand == 0 || cand_tok, CB_E_INVALID_ARG, "cand_tok is NULL");
  CB_REQUIRE(k_keep == 0 || sel_tok, CB_E_INVALID_ARG, "sel_tok is NULL");
  cudaStream_t s = (cudaStream_t)st;
  const int rows = n_cand + n_suffix;
  CB_TRY(launch_pos_check(c, pos, N + n_suffix, s));
  if (rows > 0) {
    ProfScope ps_(c, PROF_MISC, s);
    CB_LAUNCH(c, (make_rows_kernel), std::min(256, (rows + 255) / 256), 256, 0, s, cand_tok, n_cand, n_suffix, N, c->row_tok[0]);
    CB_LAUNCHED(c);
  }
  const size_t d = c->m.d_model;
  LayerBufs b{h, c->h[0], c->row_tok[0], c->row_tok[1]};
  int out_rows;
  if (layer == 0) {
    CB_REQUIRE(n_cand == N && k_keep == N, CB_E_INVALID_ARG, "layer 0 is the full layer: n_cand = k_keep = N");
    CB_TRY(layer_full(c, *w, b, N, n_suffix, k_blend, v_blend, pos, s));
    if (k_keep > 0) CB_CUDA(cudaMemcpyAsync(sel_tok, cand_tok, k_keep * 4, cudaMemcpyDeviceToDevice, s));
    out_rows = rows;
  } else {
    CB_TRY(layer_blend(c, *w, b, n_cand, k_keep, n_suffix, N, k_blend, v_blend, pos, force_sel, sel_tok, dev_out,
                       CB_DEV_KV, s));
    out_rows = k_keep + n_suffix;
  }
  if (out_rows > 0)
    CB_CUDA(cudaMemcpyAsync(h, c->h[0], (size_t)out_rows * d * sizeof(float), cudaMemcpyDeviceToDevice, s));
  return CB_OK;
}

// ---- the whole blend -------------------------------------------------------------------------------
namespace {
cb_status check_forward(cb_ctx* c, const cb_layer_w* w, const void* embed, const int32_t* tok, const int32_t* pos,
                        int32_t N, int32_t n_suffix, const int32_t* chunk_start, int32_t n_chunks, const void* k_in,
                        const void* v_in, void* k_blend, void* v_blend, const int32_t* k_sched, const void* h_out) {
  CB_REQUIRE(c != nullptr, CB_E_INVALID_ARG, "ctx is NULL");
  const int L = c->m.n_layers;
  CB_REQUIRE(w != nullptr && k_sched != nullptr, CB_E_INVALID_ARG, "w / k_sched is NULL");
  for (int i = 0; i < L; ++i) CB_TRY(check_weights(&w[i]));
  CB_REQUIRE(N >= 0 && n_suffix >= 0 && N + n_suffix >= 1, CB_E_INVALID_ARG, "empty input (N=%d, n_suffix=%d)", N,
             n_suffix);
  const int T = N + n_suffix;
  CB_REQUIRE(T <= c->max_tokens, CB_E_SHAPE, "N + n_suffix = %d > max_tokens %d", T, c->max_tokens);
  CB_REQUIRE(embed && tok && pos && k_blend && v_blend && h_out, CB_E_INVALID_ARG, "NULL pointer");
  CB_REQUIRE(N == 0 || (k_in && v_in && chunk_start && n_chunks >= 1), CB_E_INVALID_ARG,
             "chunk caches / chunk_start missing");
  if (N > 0) {
    CB_REQUIRE(chunk_start[0] == 0 && chunk_start[n_chunks] == N, CB_E_SHAPE, "chunk_start must run from 0 to N=%d",
               N);
    for (int ci = 0; ci < n_chunks; ++ci)
      CB_REQUIRE(chunk_start[ci + 1] >= chunk_start[ci], CB_E_SHAPE, "chunk_start not non-decreasing");
  }
  for (int i = 1; i < L; ++i)
    CB_REQUIRE(k_sched[i] >= 0 && k_sched[i] <= (i == 1 ? N : k_sched[i - 1]), CB_E_INVALID_ARG,
               "k_sched must satisfy 0 <= k_i <= k_{i-1} <= N (layer %d: %d)", i, k_sched[i]);
  return CB_OK;
}

// Layers 0..L-1 of the blend. realign_per_layer: request mode, where layer i's chunk KV lands in
// k_blend/v_blend on the copy stream and is realigned in place there, right after its copy (event
// layer_ev[i]); layer i waits for that event (fetch_kv / synchronize / prefill_layer). Otherwise
// the realign already ran.
cb_status blend_layers(cb_ctx* c, const cb_layer_w* w, const void* embed, const int* tok, const int* pos, int N,
                       int n_suffix, void* k_blend, void* v_blend, const int* k_sched, const int* force_sel,
                       int* sel_out, float* dev_out, float* h_out, cudaStream_t s, bool realign_per_layer,
                       cudaEvent_t realign_done = nullptr) {
  const cb_model& m = c->m;
  const int L = m.n_layers, T = N + n_suffix, kvd = m.n_kv_heads * m.head_dim;
  const size_t B = dtype_bytes(m.dtype);
  const size_t layer_stride = (size_t)T * kvd;
  auto realign_layer = [&](int i) -> cb_status {
    if (!realign_per_layer || N == 0) return CB_OK;
    CB_CUDA(cudaStreamWaitEvent(s, c->layer_ev[i], 0));  // synchronize(): layer i's KV is on the GPU, realigned
    return CB_OK;
  };
  CB_TRY(launch_pos_check(c, pos, T, s));  // positions in range and strictly increasing (device error word)
  // (a2) layer 0 in full
  // embedding gather fused with layer 0's attention RMSNorm (unless the per-kernel ablation is on)
  const bool embed_norm = !c->no_fuse_norm;
  if (embed_norm) CB_TRY(launch_embed_norm(c, embed, tok, (const float*)w[0].attn_norm, T, c->h[0], c->x, s));
  else CB_TRY(launch_embed(c, embed, tok, T, c->h[0], s));
  bool ready = false;  // the previous down projection prepared this layer's attention RMSNorm
  LayerBufs b0{c->h[0], c->h[1], c->iota, nullptr};
  b0.x_normed = embed_norm;
  b0.next_attn_norm = L > 1 ? w[1].attn_norm : nullptr;
  b0.next_ready = &ready;
  CB_TRY(layer_full(c, w[0], b0, N, n_suffix, k_blend, v_blend, pos, s, [&]() { return realign_layer(0); }));
  if (sel_out) CB_TRY(launch_sel_out(c, c->iota, N, N, sel_out, s));
  // (a3-a8) layers 1..L-1 with gradual filtering: C_1 = all context tokens, C_{i+1} = S_i
  int cur = 1, n_cand = N, rt = 0;
  const int* rows = c->iota;
  for (int i = 1; i < L; ++i) {
    const int k = k_sched[i];
    CB_TRY(realign_layer(i));
    if (i == 1 && realign_done) CB_CUDA(cudaStreamWaitEvent(s, realign_done, 0));  // layers 1.. realigned
    LayerBufs b{c->h[cur], c->h[cur ^ 1], rows, c->row_tok[rt]};
    b.x_ready = ready;
    ready = false;
    b.next_attn_norm = i + 1 < L ? w[i + 1].attn_norm : nullptr;
    b.next_ready = &ready;
    char* kb = (char*)k_blend + (size_t)i * layer_stride * B;
    char* vb = (char*)v_blend + (size_t)i * layer_stride * B;
    CB_TRY(layer_blend(c, w[i], b, n_cand, k, n_suffix, N, kb, vb, pos, force_sel ? force_sel + (size_t)i * N : nullptr,
                       nullptr, dev_out ? dev_out + (size_t)i * N : nullptr, CB_DEV_KV, s));
    if (sel_out) CB_TRY(launch_sel_out(c, c->row_tok[rt], k, N, sel_out + (size_t)i * N, s));
    rows = c->row_tok[rt];
    rt ^= 1;
    cur ^= 1;
    n_cand = k;
  }
  const int final_rows = (L == 1 ? N : n_cand) + n_suffix;
  if (final_rows > 0)
    CB_CUDA(cudaMemcpyAsync(h_out, c->h[cur], (size_t)final_rows * m.d_model * sizeof(float), cudaMemcpyDefault, s));
  return CB_OK;
}
}  // namespace

extern "C" cb_status cb_blend_forward(cb_ctx* c, const cb_layer_w* w, const void* embed, const int32_t* tok,
                                      const int32_t* pos, int32_t N, int32_t n_suffix, const int32_t* chunk_start,
                                      int32_t n_chunks, const void* k_in, const void* v_in, void* k_blend,
                                      void* v_blend, const int32_t* k_sched, const int32_t* force_sel,
                                      int32_t* sel_out, float* dev_out, float* h_out, void* st) {
  CB_TRY(check_forward(c, w, embed, tok, pos, N, n_suffix, chunk_start, n_chunks, k_in, v_in, k_blend, v_blend,
                       k_sched, h_out));
  const bool k_inplace = (k_blend == k_in), v_inplace = (v_blend == v_in);
  CB_REQUIRE((!k_inplace && !v_inplace) || n_suffix == 0, CB_E_INVALID_ARG,
             "in-place blend (k_blend == k_in) requires n_suffix == 0");
  CB_REQUIRE(k_inplace == v_inplace, CB_E_INVALID_ARG, "k and v must both be in place or both out of place");
  cudaStream_t s = (cudaStream_t)st;
  const cb_model& m = c->m;
  const int T = N + n_suffix, kvd = m.n_kv_heads * m.head_dim;
  // (a1) positional recovery of every layer's cached K in one launch (+ carry V over when out of place)
  cudaEvent_t realign_done = nullptr;
  if (N > 0) {
    CB_TRY(launch_local_pos(c, chunk_start, n_chunks, c->src_pos, s));
    const long long os = (long long)T * kvd, is = (long long)N * kvd;
    if (c->realign_overlap && m.n_layers > 1) {
      // layer 0 here; layers 1..L-1 (HBM-bound) on the aux stream under layer 0's compute-bound GEMMs,
      // joined before layer 1 reads its cache
      CB_TRY(launch_realign(c, k_blend, k_in, v_inplace ? nullptr : v_blend, v_in, c->src_pos, pos, 1, N, os, is, s));
      const size_t B = dtype_bytes(m.dtype);
      CB_CUDA(cudaEventRecord(c->ev_realign[0], s));
      CB_CUDA(cudaStreamWaitEvent(c->aux_stream, c->ev_realign[0], 0));
      CB_TRY(launch_realign(c, (char*)k_blend + os * B, (const char*)k_in + is * B,
                            v_inplace ? nullptr : (char*)v_blend + os * B, (const char*)v_in + is * B, c->src_pos,
                            pos, m.n_layers - 1, N, os, is, c->aux_stream));
      CB_CUDA(cudaEventRecord(c->ev_realign[1], c->aux_stream));
      realign_done = c->ev_realign[1];
    } else {
      CB_TRY(launch_realign(c, k_blend, k_in, v_inplace ? nullptr : v_blend, v_in, c->src_pos, pos, m.n_layers, N,
                            os, is, s));
    }
  }
  return blend_layers(c, w, embed, tok, pos, N, n_suffix, k_blend, v_blend, k_sched, force_sel, sel_out, dev_out,
                      h_out, s, false, realign_done);
}

// The request path (fetch_kv -> synchronize -> prefill_layer) with the layer fetch supplied
// by the caller: fetch(i, k_dst, v_dst, cs) enqueues layer i's chunk KV (rows [0, N)) on the copy stream.
cb_status blend_request_impl(cb_ctx* c, const cb_layer_w* w, const void* embed, const int32_t* tok_host,
                             const int32_t* pos_host, int N, int n_suffix, const int32_t* chunk_start, int n_chunks,
                             void* k_blend, void* v_blend, const int32_t* k_sched, int32_t* sel_out_host,
                             float* h_out_host, cudaStream_t s, const FetchLayer& fetch) {
  cudaStream_t cs = c->copy_stream;
  const cb_model& m = c->m;
  const int L = m.n_layers, T = N + n_suffix, kvd = m.n_kv_heads * m.head_dim;
  const size_t B = dtype_bytes(m.dtype);
  // the copy stream may only overwrite k_blend / tok / pos once the compute stream is done with them
  CB_CUDA(cudaEventRecord(c->ev_ready, s));
  CB_CUDA(cudaStreamWaitEvent(cs, c->ev_ready, 0));
  CB_CUDA(cudaMemcpyAsync(c->tok_d, tok_host, (size_t)T * 4, cudaMemcpyHostToDevice, cs));
  CB_CUDA(cudaMemcpyAsync(c->pos_d, pos_host, (size_t)T * 4, cudaMemcpyHostToDevice, cs));
  if (N > 0) CB_TRY(launch_local_pos(c, chunk_start, n_chunks, c->src_pos, cs));
  CB_CUDA(cudaEventRecord(c->layer_ev[L], cs));
  // fetch_kv(layer i) for every layer, in layer order on the copy stream, each layer's K
  // realigned right behind its copy on the same stream: the copies run ahead of the compute, so the realign
  // kernels (HBM-bound, a few us each) stay off the compute stream's critical path
  for (int i = 0; i < L && N > 0; ++i) {
    const size_t row = (size_t)kvd * B;
    char* kb = (char*)k_blend + (size_t)i * T * row;
    CB_TRY(fetch(i, kb, (char*)v_blend + (size_t)i * T * row, cs));
    CB_TRY(launch_realign(c, kb, kb, nullptr, nullptr, c->src_pos, c->pos_d, 1, N, (long long)T * kvd,
                          (long long)T * kvd, cs));
    CB_CUDA(cudaEventRecord(c->layer_ev[i], cs));
  }
  CB_CUDA(cudaStreamWaitEvent(s, c->layer_ev[L], 0));
  const int final_rows = (L == 1 ? N : k_sched[L - 1]) + n_suffix;
  CB_TRY(blend_layers(c, w, embed, c->tok_d, c->pos_d, N, n_suffix, k_blend, v_blend, k_sched, nullptr, nullptr,
                      nullptr, h_out_host, s, true));
  if (sel_out_host && L > 1 && final_rows - n_suffix > 0)
    CB_CUDA(cudaMemcpyAsync(sel_out_host, c->row_tok[(L - 2) & 1], (size_t)(final_rows - n_suffix) * 4,
                            cudaMemcpyDeviceToHost, s));
  return CB_OK;
}

// Host-memory positions (request paths): in [0, max_pos) and strictly increasing, checked before any launch.
cb_status check_host_pos(const cb_ctx* c, const int32_t* pos, int T) {
  for (int t = 0; t < T; ++t) {
    CB_REQUIRE(pos[t] >= 0 && pos[t] < c->m.max_pos, CB_E_INVALID_ARG, "pos[%d] = %d outside [0, max_pos = %d)", t,
               pos[t], c->m.max_pos);
    CB_REQUIRE(t == 0 || pos[t] > pos[t - 1], CB_E_INVALID_ARG, "pos not strictly increasing at %d (%d after %d)", t,
               pos[t], pos[t - 1]);
  }
  return CB_OK;
}

cb_status check_request(cb_ctx* c, const cb_layer_w* w, const void* embed, const int32_t* tok_host,
                        const int32_t* pos_host, int32_t N, int32_t n_suffix, const int32_t* chunk_start,
                        int32_t n_chunks, const void* k_in, const void* v_in, void* k_blend, void* v_blend,
                        const int32_t* k_sched, const void* h_out) {
  CB_TRY(check_forward(c, w, embed, tok_host, pos_host, N, n_suffix, chunk_start, n_chunks, k_in, v_in, k_blend,
                       v_blend, k_sched, h_out));
  return check_host_pos(c, pos_host, N + n_suffix);
}

extern "C" cb_status cb_blend_request(cb_ctx* c, const cb_layer_w* w, const void* embed, const int32_t* tok_host,
                                      const int32_t* pos_host, int32_t N, int32_t n_suffix, const int32_t* chunk_start,
                                      int32_t n_chunks, const void* k_in_host, const void* v_in_host, void* k_blend,
                                      void* v_blend, const int32_t* k_sched, int32_t* sel_out_host,
                                      float* h_out_host, void* st) {
  CB_TRY(check_request(c, w, embed, tok_host, pos_host, N, n_suffix, chunk_start, n_chunks, k_in_host, v_in_host,
                       k_blend, v_blend, k_sched, h_out_host));
  const int T = N + n_suffix;
  const size_t row = (size_t)c->m.n_kv_heads * c->m.head_dim * dtype_bytes(c->m.dtype);
  // request KV in one host buffer per tensor, [L][N][n_kv][hd]
  FetchLayer fetch = [&](int i, char* kd, char* vd, cudaStream_t cs) -> cb_status {
    CB_CUDA(cudaMemcpy2DAsync(kd, row * T, (const char*)k_in_host + (size_t)i * N * row, row * N, row * N, 1,
                              cudaMemcpyHostToDevice, cs));
    CB_CUDA(cudaMemcpy2DAsync(vd, row * T, (const char*)v_in_host + (size_t)i * N * row, row * N, row * N, 1,
                              cudaMemcpyHostToDevice, cs));
    return CB_OK;
  };
  return blend_request_impl(c, w, embed, tok_host, pos_host, N, n_suffix, chunk_start, n_chunks, k_blend, v_blend,
                            k_sched, sel_out_host, h_out_host, (cudaStream_t)st, fetch);
}
