/* cacheblend_ops.h — building-block entry points of libcacheblend.so, exported for per-kernel
 * parity tests and tooling. Same conventions as cacheblend.h (device pointers, caller-owned,
 * stream-ordered, host-side argument checks, negative cb_status on error).
 * These are the kernels cb_blend_layer / cb_blend_forward launch; the product path calls them
 * through the blend entry points. */
#ifndef CACHEBLEND_OPS_H
#define CACHEBLEND_OPS_H

#include "cacheblend.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ---- synthetic input generation (NOT method arithmetic) -----------------------------------
 * Device implementation of the counter-RNG spec in synth/counter_rng.py (the spec, not the code,
 * is shared with the oracle; tests/test_gpu_parity.py::test_gen_fill_bitexact pins the two bit-for-bit):
 *   raw(i) = mix64(mix64(mix64(seed) ^ stream_id) + i), u = fp32(raw >> 40) * 2^-23 - 1,
 *   out[i - start] = fp32(offset + fp32(u * scale)) [-> bf16 RNE when dtype == CB_BF16]
 * for i in [start, start + count).  cb_gen_ints: out[i - start] = raw(i) % modulus. */
CB_API cb_status cb_gen_fill(void* out, int32_t dtype, int64_t count, uint64_t seed, uint64_t stream_id,
                      int64_t start, float scale, float offset, void* stream);
CB_API cb_status cb_gen_ints(int32_t* out, int64_t count, uint64_t seed, uint64_t stream_id, int64_t start,
                      int64_t modulus, void* stream);

/* h[t] = embed[tok[t]] widened to fp32.  h: fp32 [n][d_model]. */
CB_API cb_status cb_op_embed(cb_ctx* ctx, const void* embed, const int32_t* tok, int32_t n, float* h, void* stream);

/* x[r] = h[r] / sqrt(mean(h[r]^2) + eps) * gain   (x in the model dtype). */
CB_API cb_status cb_op_rmsnorm(cb_ctx* ctx, const float* h, const float* gain, int32_t n_rows, void* x, void* stream);

/* C[M][N] = A[M][K] . B[N][K]^T with fp32 accumulation; C is fp32 when out_f32 == 1, else the model
 * dtype. out_f32 == 2: residual form C[M][N] += A . B^T on an fp32 C (the o-/down-projection epilogue).
 * impl: 0 = auto (tcgen05 for bf16), 1 = SIMT, 2 = tcgen05 (bf16 only; K % 8 == 0). */
CB_API cb_status cb_op_gemm(cb_ctx* ctx, const void* A, const void* B, void* C, int32_t M, int32_t N, int32_t K,
                     int32_t out_f32, int32_t impl, void* stream);

/* Sparse-query causal attention: for query row r (q row q_row[r] of q [*][n_q][hd], token
 * index q_tok[r]) and q head h: out[r][h] = softmax_j(q.k_j / sqrt(hd)) v_j over keys j <= q_tok[r]
 * of k, v [n_keys][n_kv][hd], kv head h / (n_q / n_kv).  Token positions are strictly increasing, so
 * "key position <= query position" is "j <= q_tok[r]".  out: [n_rows][n_q * hd] (model dtype).
 * impl: 0 = auto (2 for bf16 / head_dim 128), 1 = SIMT, 2 = tcgen05/TMEM one CTA per (row tile, kv head,
 * key range) with split-KV merged in-kernel (needs bf16, head_dim 128). */
CB_API cb_status cb_op_attention(cb_ctx* ctx, const void* q, const int32_t* q_row, const int32_t* q_tok,
                          int32_t n_rows, const void* k, const void* v, int32_t n_keys, void* out, int32_t impl,
                          void* stream);

/* Tuning knobs (for experiments; defaults are the tuned choices). Unknown names -> INVALID_ARG.
 *   "gemm_sched"  0 = auto (cost model picks data-parallel or data-parallel + stream-K tail),
 *                 1 = data-parallel only, 2 = data-parallel rounds + stream-K tail
 *   "gemm_bn"     0 = auto, 128, 192 (CTA pairs only) or 256 = force the tcgen05 GEMM tile width
 *   "gemm_pair"   0 = auto, 1 = CTA-pair (cta_group::2, 256-row tiles) only, 2 = single-CTA only
 *   "gemm_ksplit" 0 = auto, 1..4 = force the k-split chain of pair residual GEMMs (when it fits one wave)
 *   "gemm_no192"  1 = exclude 256 x 192 CTA-pair tiles from GEMM plans (0 = allowed, default)
 *   "gemm_balance" 1 = pair GEMMs use the fewest pairs that need the same number of tile rounds (default;
 *                 the full-load mainloop is power-capped, so even rounds beat a ragged last one), 0 = all
 *   "gemm_cap_store", "gemm_cap_store_f32", "gemm_cap_qkv", "gemm_cap_resid", "gemm_cap_swiglu"
 *                 n > 0 = pair GEMMs of that epilogue kind use at most n CTA pairs (0 = no cap, default)
 *   "topk_drop"   n = top-k drops the n_cand - k smallest one by one when that count is <= n (default 48)
 *   "gemm_tail"   0 = auto (cost model), 1 = never (default; measured faster), 2 = always cut the remainder
 *                 tiles of a pair GEMM's last round into K pieces (merged in piece order by the last piece)
 *   "attn_impl"   0 = auto, 1 = SIMT, 2 = tcgen05/TMEM per tile
 *   "attn_splits" 0 = auto, 1..16 = force the split-KV factor
 *   "q_split"     1 = layer 1 projects Q for the kept rows only, after the top-k (default), 0 = Q for all
 *                 candidates in the fused QKV GEMM
 *   "fuse_deviation" 1 = Delta_kv in the tcgen05 QKV epilogue (default), 0 = separate kernel
 *   "debug_trace" 1 = record pipeline events of one CTA of the tcgen05 attention and per-CTA events of
 *                 the CTA-pair GEMM (tuning; each launch overwrites); 100 + k = only pair GEMMs of epilogue
 *                 kind k (0 store, 1 store_f32, 2 qkv, 3 residual, 4 swiglu); 300 = per-k-block producer /
 *                 MMA clock64 timeline of CTA pair 0 of the pair GEMM (tools/gemm_stages.py)
 *   "pdl"         1 = programmatic dependent launch between library kernels (default), 0 = off
 *   "fuse_norm"   1 = RMSNorm fused into the residual / next projection epilogues (default), 0 = kernels
 *   "topk_threads" 0 = 1024 (default), 256 or 512 threads in the top-k block
 *   "epi_l1pf"    1 = the residual epilogue of the pair GEMM pulls each row's next 32-column residual segment
 *                 into L1 while the current chunk is stored (default), 0 = off
 *   "gemm_mc"     A-multicast 4-CTA clusters (two CTA pairs sharing their A rows) in the pair GEMM:
 *                 2 = where the planner expects a shorter k-loop, 1 = always (whole tiles), 0 = off (default),
 *                 3 = 8-CTA clusters (2 row x 2 column tiles, B multicast as well; measured neutral, opt-in) */
CB_API cb_status cb_set_option(cb_ctx* ctx, const char* name, int64_t value);

/* Read-only facts about the context: "num_sms", "gemm_max_pairs" (co-resident 2-CTA clusters of the
 * CTA-pair GEMM, from cudaOccupancyMaxActiveClusters), "gemm_max_clusters4" (co-resident 4-CTA clusters of
 * it, for gemm_mc). Unknown names -> INVALID_ARG. */
CB_API cb_status cb_get_info(cb_ctx* ctx, const char* name, int64_t* value);

/* Number of kernel launches the context issued since creation (for bench's gpu_launches). */
CB_API int64_t cb_launch_count(cb_ctx* ctx);

/* Copy n (<= 2048) int64 entries of the debug_trace buffer to host memory. Blocking. */
CB_API cb_status cb_debug_fetch(cb_ctx* ctx, int64_t* host, int32_t n);

/* Per-launch profile: between begin and end every library launch is bracketed by a CUDA event pair
 * on its stream. cb_profile_end synchronises the device and writes, per kernel class
 * (cb_profile_class_name), the summed device milliseconds and the launch count (n_classes entries). */
CB_API cb_status cb_profile_begin(cb_ctx* ctx);
CB_API cb_status cb_profile_end(cb_ctx* ctx, double* ms_out, int64_t* counts_out, int32_t n_classes);
CB_API const char* cb_profile_class_name(int32_t cls);

/* Peer-memory collectives diagnostics: out[0..51] = this rank's flag words {entry[8], exit[8], seq, finished
 * CTAs, 2 spare, ring of the last 8 collectives (seq, rank, block tag, mode)}, out[52] = this block's tag;
 * read through a private non-blocking stream (out: 53 host ints, pinned for an asynchronous read). */
CB_API cb_status cb_debug_p2p_flags(cb_ctx* ctx, int32_t* out53);

#ifdef __cplusplus
}
#endif
#endif
