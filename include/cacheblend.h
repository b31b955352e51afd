/* cacheblend.h — C-ABI boundary of the B200-native CacheBlend blend path (libcacheblend.so).
 *
 * CacheBlend (arXiv 2405.16444) fuses per-chunk precomputed KV caches of retrieved text that is
 * not a prefix of the input, recomputing only the high-KV-deviation (HKVD) tokens per layer.
 * Citations: P:<line> = PAPER.md line, S:<line> = SPEC.md line, R<n> = reading in DESIGN.md.
 *
 * Conventions (all entry points):
 *  - Tensor pointers are DEVICE pointers owned by the caller unless marked "host". The library
 *    never frees caller memory. Rows are token-major and contiguous.
 *  - Storage dtype is cb_model.dtype: CB_BF16 (hot path; fp32 accumulation, fp32 residual
 *    stream h) or CB_FP32 (parity mode: fp32 everywhere). Norm gains are always fp32 [d_model].
 *  - Calls are asynchronous and stream-ordered on `stream` (a cudaStream_t; NULL = legacy
 *    default stream). Argument/shape errors are detected on the host BEFORE any launch and
 *    return a negative cb_status; kernel faults surface as CB_E_CUDA at a later call or sync.
 *  - cb_last_error() returns a thread-local message for the last non-OK status.
 *  - A cb_ctx may be used by one host thread at a time; distinct contexts are independent.
 *  - There is no CPU fallback: every step runs in the library's sm_100a kernels.
 */
#ifndef CACHEBLEND_H
#define CACHEBLEND_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define CB_API __attribute__((visibility("default")))
#else
#define CB_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  CB_OK = 0,
  CB_E_INVALID_ARG = -1, /* bad configuration / value (odd head_dim, k_keep > n_cand, NULL ...) */
  CB_E_SHAPE = -2,       /* size / length mismatch or exceeds the context's max_tokens          */
  CB_E_UNSUPPORTED = -3, /* valid but not built (e.g. world > 1 without NCCL)                   */
  CB_E_CUDA = -4,        /* CUDA runtime / launch error                                         */
  CB_E_NCCL = -5,
  CB_E_WORKSPACE = -6,   /* caller workspace too small                                          */
  CB_E_DEVICE = -7,      /* device-side precondition violated (see cb_check_device_errors)      */
  CB_E_MISS = -8         /* a chunk's KV cache is not in the KV store (fetch_kv's -1)    */
} cb_status;

typedef enum { CB_BF16 = 0, CB_FP32 = 1 } cb_dtype;

/* Delta_kv variant (R1): squared L2 over K and V of all kv heads (default), K only, V only
 * (the paper notes either suffices). */
typedef enum { CB_DEV_KV = 0, CB_DEV_K = 1, CB_DEV_V = 2 } cb_dev_mode;

/* Llama/Mistral-style decoder (the paper names the models, not the block; R-model in
 * DESIGN.md): RMSNorm pre-norm, GQA attention with RoPE (interleaved pairs (2i,2i+1), P:2531-2538,
 * theta_i = rope_theta^(-2i/head_dim), R8), SwiGLU MLP, residual connections. */
typedef struct {
  int32_t n_layers, d_model, n_q_heads, n_kv_heads, head_dim, d_ff, vocab;
  double rope_theta;
  float rms_eps;
  int32_t dtype;   /* cb_dtype */
  int32_t max_pos; /* exclusive upper bound of |positions| and |g - l| used with this model */
} cb_model;

/* One layer's weights (device). Layouts are [out_features][in_features] (K-contiguous):
 *   attn_norm, mlp_norm : fp32 [d_model]
 *   w_qkv     : [(n_q + 2 n_kv) * head_dim][d_model]  rows = q heads, then k heads, then v heads
 *   w_o       : [d_model][n_q * head_dim]
 *   w_gate_up : [2 d_ff][d_model]  rows [0, d_ff) = gate, [d_ff, 2 d_ff) = up
 *   w_down    : [d_model][d_ff]                                                              */
typedef struct {
  const void *attn_norm, *w_qkv, *w_o, *mlp_norm, *w_gate_up, *w_down;
} cb_layer_w;

typedef struct cb_ctx cb_ctx; /* opaque: RoPE tables, tensor-map cache, workspace, scratch */

/* ---- context ------------------------------------------------------------------------------ */
/* Bytes of device workspace a context needs for max_tokens = N + n_suffix rows. */
CB_API cb_status cb_workspace_size(const cb_model* model, int32_t max_tokens, size_t* bytes);

/* Create a context on the current CUDA device. workspace: device buffer of at least
 * cb_workspace_size() bytes, owned by the caller, or NULL to let the library cudaMalloc (and
 * free in cb_destroy). Errors: odd head_dim, n_q % n_kv != 0, non-positive sizes -> INVALID_ARG. */
CB_API cb_status cb_create(const cb_model* model, int32_t max_tokens, void* workspace, size_t workspace_bytes,
                    cb_ctx** out);
CB_API cb_status cb_destroy(cb_ctx* ctx);
CB_API const char* cb_last_error(void);

/* Synchronises the context's device-side error word (e.g. a force_sel token that is not a
 * candidate) and clears it: CB_OK or CB_E_DEVICE. Blocking. */
CB_API cb_status cb_check_device_errors(cb_ctx* ctx);

/* Gradual-filtering schedule (R4/R5), host only: k_sched_out[0] = n_ctx (layer 0 is
 * the full layer, R2); for i >= 1, k_i = min(N, ceil(r_i N - 1e-9)) non-increasing, with
 * r_i = r + d (1 - 2(i-1)/(L-2)), d = 0.2 min(r, 1-r) (L = 2: r_1 = r).
 * k_sched_out: host int32[n_layers]. ratio outside [0,1] -> INVALID_ARG. */
CB_API cb_status cb_schedule(double ratio, int32_t n_ctx, int32_t n_layers, int32_t* k_sched_out);

/* Loading controller (§6 "Loading Controller"), host only. Per layer:
 *   T_load = kv_bytes_per_token * n_tokens / bytes_per_ms          (footnote P:2696)
 *   T_recompute(r) = r * prefill_ms, prefill_ms profiled offline   (footnote P:2695)
 * cb_controller_ratio: r_out = min(1, max(r_eq, r_min)) with T_recompute(r_eq) = T_load (
 * the paper's r* = 15 %); load_ms_out (optional) = T_load. Errors: non-positive prefill/throughput,
 * r_min outside [0, 1] -> INVALID_ARG.
 * cb_controller_pick_device: the cheapest of n_dev storage devices (host arrays load_ms[d] = T_load on
 * device d, cost[d]) with T_recompute(r_fixed) >= T_load; ties -> lower index; -1 if none. */
CB_API cb_status cb_controller_ratio(double prefill_ms, double kv_bytes_per_token, int64_t n_tokens,
                                     double bytes_per_ms, double r_min, double* r_out, double* load_ms_out);
CB_API cb_status cb_controller_pick_device(double prefill_ms, const double* load_ms, const double* cost,
                                           int32_t n_dev, double r_fixed, int32_t* pick_out);
/* The controller driving the blend ("the fusor then recomputes r% of the tokens"):
 * r = cb_controller_ratio(prefill_ms, kv_bytes_per_token, n_ctx, bytes_per_ms, r_min) and the per-layer
 * counts k_sched_out[n_layers] = cb_schedule(r, n_ctx, n_layers), ready for cb_blend_request /
 * cb_blend_forward. r_out / load_ms_out optional. Errors as the two calls. */
CB_API cb_status cb_controller_schedule(double prefill_ms, double kv_bytes_per_token, double bytes_per_ms,
                                        double r_min, int32_t n_ctx, int32_t n_layers, int32_t* k_sched_out,
                                        double* r_out, double* load_ms_out);

/* ---- (a) positional recovery --------------------------------------------------------------- */
/* Footnote P:208-211, Appendix: K_out[s][t] = R(dst_pos[t] - src_pos[t]) K_src[s][t]
 * for every slice s (a layer) and token t, per kv head; V is untouched. src_pos = chunk-local
 * position l (all zeros = position-free storage, R11), dst_pos = global position g.
 * k_src/k_out: [n_slices][n_tok][n_kv][head_dim], slices slice_stride elements apart
 * (>= n_tok * n_kv * head_dim); in place (k_out == k_src) allowed. Positions: device int32[n_tok],
 * |dst - src| < max_pos (violations are clamped and flagged in the device error word). */
CB_API cb_status cb_rope_realign(cb_ctx* ctx, void* k_out, const void* k_src, const int32_t* src_pos,
                          const int32_t* dst_pos, int32_t n_slices, int32_t n_tok, int64_t slice_stride,
                          void* stream);

/* ---- (b) KV deviation + HKVD top-k ----------------------------------------------------------- */
/* Delta_kv (R1) of each candidate j against the loaded entry of its token, and
 * the k_keep largest (Insight 1), ties -> lower token index (R6):
 *   dev[j] = sum_heads ||k_new[j] - k_ref[cand_tok[j]]||^2 + ||v_new[j] - v_ref[cand_tok[j]]||^2
 * k_new, v_new : [n_cand][n_kv][head_dim]   fresh rows in candidate order (K RoPE'd at g)
 * k_ref, v_ref : [>= max cand_tok + 1][n_kv][head_dim]   the layer's blended cache
 * cand_tok     : int32[n_cand], strictly ascending token indices
 * sel_tok      : out int32[k_keep], ascending;  sel_slot: out int32[k_keep] (index into cand_tok)
 * dev_out      : out fp32[n_cand] or NULL.   0 <= k_keep <= n_cand <= max_tokens.
 * The sum runs per kv head in a fixed order, so results are bitwise reproducible. */
CB_API cb_status cb_kv_deviation_topk(cb_ctx* ctx, const void* k_new, const void* v_new, const void* k_ref,
                               const void* v_ref, const int32_t* cand_tok, int32_t n_cand, int32_t k_keep,
                               int32_t dev_mode, int32_t* sel_tok, int32_t* sel_slot, float* dev_out,
                               void* stream);

/* ---- (c) one layer of selective recompute ------------------------------------------------------ */
/* prefill_layer on layer `layer` (§3.2 workflow P:150-161):
 *  layer >= 1 (check_flag <=> k_keep < n_cand): x = RMSNorm(h); q,k,v = RoPE(x Wq), RoPE(x Wk), x Wv
 *    for the n_cand candidate rows and the n_suffix suffix rows; Delta_kv over the candidates;
 *    S = top-k_keep (or force_sel, replay mode R14); write fresh K,V of S and of the suffix into
 *    k_blend/v_blend (untouched rows keep their bytes, R3); attention of the S + suffix queries over
 *    all N + n_suffix keys masked by original position; h += attn W_o; h += MLP(RMSNorm(h)).
 *  layer == 0 (the full layer, R2): n_cand must equal N, cand_tok = 0..N-1, k_keep = N.
 *    Context rows keep the cached K,V (layer-0 KV depend only on the token); suffix rows
 *    write theirs; every row is a query.
 * h        : fp32 [n_cand + n_suffix][d_model] in (rows of cand_tok, then suffix) and out (rows
 *            [0, k_keep + n_suffix) = S ascending, then suffix).
 * k_blend, v_blend : this layer's [N + n_suffix][n_kv][head_dim], updated in place.
 * pos      : int32[N + n_suffix] strictly increasing global positions (context, then suffix).
 * force_sel: int32[k_keep] ascending subset of cand_tok, or NULL.
 * sel_tok  : out int32[k_keep];  dev_out: out fp32[n_cand] or NULL.                               */
CB_API cb_status cb_blend_layer(cb_ctx* ctx, int32_t layer, const cb_layer_w* w, float* h, const int32_t* cand_tok,
                         int32_t n_cand, int32_t k_keep, int32_t n_suffix, void* k_blend, void* v_blend,
                         const int32_t* pos, int32_t N, const int32_t* force_sel, int32_t* sel_tok,
                         float* dev_out, void* stream);

/* ---- the whole blend ------------------------------------------------------------------------- */
/* SURVEY §8(c) steps 1-5 / P:2742-2748. Chunk c occupies context rows chunk_start[c]..chunk_start[c+1].
 * w        : host array [n_layers] of device weight pointers;  embed: [vocab][d_model]
 * tok, pos : device int32[N + n_suffix]
 * chunk_start : HOST int32[n_chunks + 1], chunk_start[0] = 0, chunk_start[n_chunks] = N
 * k_in, v_in  : chunk caches [n_layers][N][n_kv][head_dim], K RoPE'd at chunk-local positions
 * k_blend, v_blend : out KV^new [n_layers][N + n_suffix][n_kv][head_dim]; may alias k_in/v_in
 *                    (in place) when n_suffix == 0
 * k_sched  : HOST int32[n_layers] (k_sched[0] ignored; k_sched[i] <= k_sched[i-1] <= N)
 * force_sel: device int32[n_layers][N] (row i: S_i ascending in its first k_sched[i] entries) or NULL
 * sel_out  : device int32[n_layers][N] or NULL: row i = S_i ascending, padded with -1 (row 0 = 0..N-1)
 * dev_out  : device fp32[n_layers][N] or NULL: row i, entry j < |C_i| = Delta_kv of the j-th
 *            candidate (C_1 = 0..N-1, C_i = S_{i-1}); other entries untouched
 * h_out    : device fp32[k_sched[L-1] + n_suffix][d_model]: final hidden rows of S_{L-1} then suffix
 *            (for n_layers == 1: all N + n_suffix rows).                                             */
CB_API cb_status cb_blend_forward(cb_ctx* ctx, const cb_layer_w* w, const void* embed, const int32_t* tok,
                           const int32_t* pos, int32_t N, int32_t n_suffix, const int32_t* chunk_start,
                           int32_t n_chunks, const void* k_in, const void* v_in, void* k_blend, void* v_blend,
                           const int32_t* k_sched, const int32_t* force_sel, int32_t* sel_out, float* dev_out,
                           float* h_out, void* stream);

/* ---- end to end from host memory ----------------------------------------------------------------- */
/* The same blend with the request's inputs in HOST memory (pinned for asynchronous copies), as the
 * paper's loading path does (fetch_kv -> synchronize -> prefill_layer): layer i's chunk
 * KV is copied into k_blend/v_blend layer i on the context's copy stream while layer i-1 computes,
 * and layer i waits only for its own copy (two-stream layer pipelining).
 * tok_host, pos_host : host int32[N + n_suffix];  k_in_host, v_in_host: host [n_layers][N][n_kv][hd]
 * k_blend, v_blend   : DEVICE out KV^new [n_layers][N + n_suffix][n_kv][hd] (stays on the GPU for decode)
 * sel_out_host       : host int32[k_sched[L-1]] (S_{L-1}) or NULL;  h_out_host: host fp32 rows as in
 *                      cb_blend_forward. Other arguments as cb_blend_forward. Returns after enqueueing;
 *                      host outputs are valid once `stream` is synchronised. */
CB_API cb_status cb_blend_request(cb_ctx* ctx, const cb_layer_w* w, const void* embed, const int32_t* tok_host,
                                  const int32_t* pos_host, int32_t N, int32_t n_suffix, const int32_t* chunk_start,
                                  int32_t n_chunks, const void* k_in_host, const void* v_in_host, void* k_blend,
                                  void* v_blend, const int32_t* k_sched, int32_t* sel_out_host, float* h_out_host,
                                  void* stream);

/* ---- hand-off to a paged decode cache ------------------------------------------- */
/* "The fused KV cache is input into the LLM inference engine", which stores KV in fixed-size
 * blocks (vLLM). Copies KV^new into per-layer page pools:
 *   k_pages[l * dst_layer_stride + (block_table[t / block_size] * block_size + t % block_size) * row + e]
 *     = k_blend[l * src_layer_stride + t * row + e]      (same for V), row = n_kv * head_dim,
 * for l < n_layers, t < n_tok. block_table: device int32[ceil(n_tok / block_size)] page ids of a pool of
 * n_pages pages per layer (dst_layer_stride >= n_pages * block_size * row); an id outside [0, n_pages) is
 * not written and raises CB_E_DEVICE at cb_check_device_errors. Bit-exact copy in the model dtype; slots of
 * a last partial page past n_tok are untouched. Errors: strides too small -> SHAPE; unaligned buffers /
 * NULL -> INVALID_ARG. */
CB_API cb_status cb_kv_to_paged(cb_ctx* ctx, const void* k_blend, const void* v_blend, int32_t n_layers, int32_t n_tok,
                                int64_t src_layer_stride, const int32_t* block_table, int32_t block_size,
                                void* k_pages, void* v_pages, int32_t n_pages, int64_t dst_layer_stride, void* stream);

/* ---- chunk KV store (§6 "KV cache store") ---------------------------- */
/* Maps a chunk's hash to its precomputed KV cache in host RAM, evicting the least recently used
 * entry when full -- to an optional disk level (cb_store_set_disk). Entries: K and V of one chunk, each [L][n_tok][n_kv][hd]
 * in the model dtype with K rotated at chunk-local positions (as cb_blend_forward's k_in). pinned = 1:
 * page-locked entries, needed by cb_blend_request_store (asynchronous per-layer DMA); 0: malloc (host
 * bookkeeping only). Thread-safe. Host-side bookkeeping: no method arithmetic. */
typedef struct cb_store cb_store;
/* A chunk's store key: 32-byte SHA-256 digest of (u32 little-endian byte length of model_id || model_id ||
 * the chunk's token ids as little-endian int32). model_id identifies the model whose KV the entry holds
 * (e.g. a digest of its configuration and weights), so one store can serve several models without one
 * model's KV answering another's lookup ("each chunk is hashed"). Host only; NULL out /
 * negative lengths -> INVALID_ARG. */
typedef struct { uint8_t bytes[32]; } cb_chunk_key;
CB_API cb_status cb_chunk_digest(const void* model_id, int32_t model_id_len, const int32_t* tokens, int32_t n_tok,
                                 cb_chunk_key* out);
CB_API cb_status cb_store_create(size_t capacity_bytes, int32_t pinned, cb_store** out);
CB_API cb_status cb_store_destroy(cb_store* store);
/* Insert (or replace) key -> (k, v), `bytes` each, copied synchronously from host or device memory. Evicts
 * LRU entries until 2 * bytes fit (waiting for in-flight fetches from them). An entry larger than the
 * capacity -> SHAPE. The new entry is the most recently used. */
CB_API cb_status cb_store_put(cb_store* store, const cb_chunk_key* key, const void* k, const void* v, int64_t bytes,
                              int32_t n_tok);
/* fetch_kv's lookup: n_tok_out = the entry's token count or -1 when absent; k_out / v_out
 * (optional) = its host pointers (valid until evicted). touch != 0 counts a hit / miss and refreshes the
 * entry's recency. */
CB_API cb_status cb_store_lookup(cb_store* store, const cb_chunk_key* key, int32_t touch, int32_t* n_tok_out,
                                 const void** k_out, const void** v_out);
/* out6 = {used bytes, capacity, entries, hits, misses, evictions}. */
CB_API cb_status cb_store_stats(cb_store* store, int64_t* out6);
/* Second storage level (the store spans storage devices; KV written to disk and read back,
 * P:2514-2516): entries evicted from RAM are written as one file per chunk into `dir` (which must exist and
 * be writable) while the disk level holds at most capacity_bytes, itself evicting its least recently used
 * files. A lookup with touch != 0 (and cb_blend_request_store) reads a disk entry back into RAM as the most
 * recently used entry; cb_store_lookup with touch = 0 reports its n_tok with NULL pointers. capacity_bytes
 * = 0 disables the level and deletes its files; the store deletes its files on destroy. Errors: unwritable
 * dir -> INVALID_ARG; an unreadable file -> CB_E_CUDA (the entry is dropped). */
CB_API cb_status cb_store_set_disk(cb_store* store, const char* dir, size_t capacity_bytes);
/* out6 = {disk bytes used, disk capacity, disk entries, disk hits (promotions), spills, disk evictions}. */
CB_API cb_status cb_store_disk_stats(cb_store* store, int64_t* out6);
/* The first n keys in recency order (most recent first); n_out = number of entries. */
CB_API cb_status cb_store_keys(cb_store* store, cb_chunk_key* keys, int32_t n, int32_t* n_out);
/* cb_blend_request with chunk c's KV fetched from the store under chunk_keys[c] (host cb_chunk_key[n_chunks]):
 * layer i's KV of every chunk is copied on the copy stream while layer i-1 computes. Every key
 * must be present with n_tok = chunk length and L * n_tok * n_kv * hd elements, else CB_E_MISS / CB_E_SHAPE
 * before any launch; the chunks' recency is refreshed. Needs a pinned store; not graph-capturable. Other
 * arguments as cb_blend_request. */
CB_API cb_status cb_blend_request_store(cb_ctx* ctx, cb_store* store, const cb_chunk_key* chunk_keys, const cb_layer_w* w,
                                        const void* embed, const int32_t* tok_host, const int32_t* pos_host,
                                        int32_t N, int32_t n_suffix, const int32_t* chunk_start, int32_t n_chunks,
                                        void* k_blend, void* v_blend, const int32_t* k_sched, int32_t* sel_out_host,
                                        float* h_out_host, void* stream);

/* ---- head-parallel blend (SURVEY §8(e) partitioning 1) ------------------------------ */
/* Tensor parallelism by attention heads within a layer (BASELINE north_star: "partitioned ... by attention
 * heads within a layer, with an NCCL all-reduce over NVLink after the output projection and none inside
 * attention"). Rank r of world w creates its context with the SHARD model: n_q_heads / w, n_kv_heads / w,
 * d_ff / w (d_model, head_dim, vocab unchanged), and passes shard weights in the same cb_layer_w layouts:
 *   w_qkv rows = q heads [r n_q/w, (r+1) n_q/w), then k heads and v heads [r n_kv/w, (r+1) n_kv/w)
 *   w_o = columns [r qd/w, (r+1) qd/w) of the full w_o;  w_gate_up = gate rows then up rows of features
 *   [r ff/w, (r+1) ff/w);  w_down = the same feature columns of the full w_down;  norms and embed replicated.
 * k_in/v_in/k_blend/v_blend hold the rank's kv heads only ([L][T][n_kv/w][hd]). Every rank calls
 * cb_blend_forward / cb_blend_layer with identical tokens, positions, chunks and k_sched; per layer the
 * library all-gathers the Delta_kv partials (identical top-k on every rank), all-reduces the o_proj
 * output and the down_proj output (fp32 sums; rank 0 adds the residual). RMSNorm runs replicated after
 * the all-reduce. Outputs: S_i and h_out identical on every rank; k_blend/v_blend the rank's heads.
 * cb_kv_deviation_topk stays rank-local. */
typedef struct cb_group cb_group; /* opaque loopback group (one process, one device) */

/* NCCL unique id (128 host bytes) for cb_set_comm; call on one rank and broadcast it. libnccl.so.2 is
 * resolved at run time (the already-loaded copy, else the loader path, else $CB_NCCL_LIB):
 * CB_E_UNSUPPORTED if absent. */
CB_API cb_status cb_nccl_unique_id(void* uid_out);
/* Make ctx rank `rank` of an NCCL communicator of `world` ranks (one process per GPU, collective over the
 * ranks: every rank must call it). Collectives run on the blend's stream (graph-capturable).
 * Errors: world outside [1, 8], rank outside [0, world), ctx already joined -> INVALID_ARG; NCCL -> E_NCCL. */
CB_API cb_status cb_set_comm(cb_ctx* ctx, const void* uid, int32_t rank, int32_t world);
/* Loopback group for testing the head-parallel path in ONE process on one device: world contexts, each
 * joined with cb_set_comm_local and driven by its own host thread and stream, run the same per-rank
 * kernels; exchanges are stream-event ordering plus a fixed-order reduce kernel. Eager launches only
 * (not graph-capturable). A member that stops calling turns the others' calls into CB_E_NCCL after 120 s.
 * Destroy the group after its contexts. */
CB_API cb_status cb_group_create(int32_t world, cb_group** out);
CB_API cb_status cb_group_destroy(cb_group* group);
CB_API cb_status cb_set_comm_local(cb_ctx* ctx, cb_group* group, int32_t rank);
/* NVLink peer-memory collectives in place of the NCCL / loopback-event calls (after cb_set_comm or
 * cb_set_comm_local, before the first blend): the rank's residual stream, gathered Delta_kv partials and
 * barrier flags move into one exchange block with the same layout on every rank; each collective is one
 * small kernel that raises/waits flags in every peer's block (system-scope release/acquire), sums its slice of
 * the buffer over all ranks in rank order (the same bits as the event path) and writes the sum into every
 * rank's block, then waits until every rank has finished. Graph-capturable (device-side sequence numbers).
 * One process per GPU: exchange cb_tp_ipc_handle (64 host bytes per rank, e.g. all-gathered with
 * torch.distributed) and call cb_tp_ipc_open with the world's handles in rank order. Loopback group: the
 * members' blocks are used directly (every member must enable it; run the process with
 * CUDA_DEVICE_MAX_CONNECTIONS >= 4 * world so no rank's stream shares a hardware queue with a spinning
 * collective of another rank). */
CB_API cb_status cb_tp_p2p_enable(cb_ctx* ctx);
CB_API cb_status cb_tp_ipc_handle(cb_ctx* ctx, void* handle_out_64B);
CB_API cb_status cb_tp_ipc_open(cb_ctx* ctx, const void* handles_world_x_64B);

#ifdef __cplusplus
}
#endif
#endif /* CACHEBLEND_H */
