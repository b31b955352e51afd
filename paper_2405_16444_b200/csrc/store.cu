// store.cu — chunk KV store (§6 "KV cache store") and the request path that
// fetches from it (fetch_kv / synchronize / prefill_layer).
//
// Each chunk's token ids are hashed to find its KV cache ("each chunk is hashed ... in the same way as the
// block hashing is implemented in vLLM"); the KV caches of new chunks are added; "when the storage
// devices are full, we evict the least recently used KV cache", on one storage level (host RAM,
// P:2723). Entries live in pinned host memory so the per-layer fetch is an asynchronous DMA on the
// context's copy stream. An entry is [L][n_tok][n_kv][head_dim] K then V in the model dtype (chunk-local
// RoPE, as cb_blend_forward's k_in). Host-only bookkeeping: no method arithmetic lives here.
#include <cstdlib>
#include <cstring>
#include <list>
#include <mutex>
#include <unordered_map>

#include "ctx.h"

namespace {
struct Entry {
  uint64_t key;
  void* k;
  void* v;
  int64_t bytes;  // of K (and of V)
  int32_t n_tok;
  cudaEvent_t last_use;  // recorded after the last fetch copies from this entry were enqueued
  bool used;
};
}  // namespace

struct cb_store {
  size_t capacity;
  size_t used = 0;
  bool pinned;
  std::mutex mu;
  std::list<Entry> lru;  // front = most recently used
  std::unordered_map<uint64_t, std::list<Entry>::iterator> index;
  long long hits = 0, misses = 0, evictions = 0;
};

namespace {
void free_entry(cb_store* st, Entry& e) {
  if (e.used) cudaEventSynchronize(e.last_use);  // no fetch may still be reading this memory
  if (e.last_use) cudaEventDestroy(e.last_use);
  if (st->pinned) {
    cudaFreeHost(e.k);
    cudaFreeHost(e.v);
  } else {
    free(e.k);
    free(e.v);
  }
  st->used -= 2 * (size_t)e.bytes;
}

void* host_alloc(cb_store* st, size_t n) {
  if (!st->pinned) return malloc(n);
  void* p = nullptr;
  return cudaHostAlloc(&p, n, cudaHostAllocDefault) == cudaSuccess ? p : nullptr;
}
}  // namespace

// 64-bit FNV-1a over the chunk's token ids (little-endian int32 bytes), then a splitmix64 finaliser.
extern "C" uint64_t cb_chunk_hash(const int32_t* tokens, int32_t n_tok) {
  uint64_t h = 1469598103934665603ull;
  for (int32_t i = 0; i < n_tok && tokens; ++i) {
    const uint32_t t = (uint32_t)tokens[i];
    for (int b = 0; b < 4; ++b) {
      h ^= (t >> (8 * b)) & 0xFFu;
      h *= 1099511628211ull;
    }
  }
  h ^= (uint64_t)(uint32_t)n_tok * 0x9E3779B97F4A7C15ull;
  h = (h ^ (h >> 30)) * 0xBF58476D1CE4E5B9ull;
  h = (h ^ (h >> 27)) * 0x94D049BB133111EBull;
  return h ^ (h >> 31);
}

extern "C" cb_status cb_store_create(size_t capacity_bytes, int32_t pinned, cb_store** out) {
  CB_REQUIRE(out != nullptr && capacity_bytes > 0, CB_E_INVALID_ARG, "cb_store_create: bad arguments");
  cb_store* s = new cb_store();
  s->capacity = capacity_bytes;
  s->pinned = pinned != 0;
  *out = s;
  return CB_OK;
}

extern "C" cb_status cb_store_destroy(cb_store* s) {
  if (!s) return CB_OK;
  for (auto& e : s->lru) free_entry(s, e);
  delete s;
  return CB_OK;
}

extern "C" cb_status cb_store_put(cb_store* s, uint64_t key, const void* k, const void* v, int64_t bytes,
                                  int32_t n_tok) {
  CB_REQUIRE(s && k && v && bytes > 0 && n_tok > 0, CB_E_INVALID_ARG, "cb_store_put: bad arguments");
  CB_REQUIRE(2 * (size_t)bytes <= s->capacity, CB_E_SHAPE, "entry of %lld bytes exceeds the store capacity %zu",
             (long long)(2 * bytes), s->capacity);
  std::lock_guard<std::mutex> lk(s->mu);
  auto it = s->index.find(key);
  if (it != s->index.end()) {  // replace: the new KV of this chunk
    free_entry(s, *it->second);
    s->lru.erase(it->second);
    s->index.erase(it);
  }
  while (s->used + 2 * (size_t)bytes > s->capacity && !s->lru.empty()) {  // evict least recently used
    Entry& victim = s->lru.back();
    s->index.erase(victim.key);
    free_entry(s, victim);
    s->lru.pop_back();
    ++s->evictions;
  }
  Entry e{key, host_alloc(s, (size_t)bytes), host_alloc(s, (size_t)bytes), bytes, n_tok, nullptr, false};
  if (!e.k || !e.v) {
    if (s->pinned) { if (e.k) cudaFreeHost(e.k); if (e.v) cudaFreeHost(e.v); }
    else { free(e.k); free(e.v); }
    cb_set_error("cb_store_put: host allocation of %lld bytes failed", (long long)bytes);
    return CB_E_CUDA;
  }
  // k / v may be host or device memory (unified addressing); synchronous
  if (s->pinned) {
    cudaError_t r = cudaEventCreateWithFlags(&e.last_use, cudaEventDisableTiming);
    if (r == cudaSuccess) r = cudaMemcpy(e.k, k, (size_t)bytes, cudaMemcpyDefault);
    if (r == cudaSuccess) r = cudaMemcpy(e.v, v, (size_t)bytes, cudaMemcpyDefault);
    if (r != cudaSuccess) {
      s->used += 2 * (size_t)bytes;
      free_entry(s, e);
      CB_CUDA(r);
    }
  } else {
    memcpy(e.k, k, (size_t)bytes);
    memcpy(e.v, v, (size_t)bytes);
  }
  s->used += 2 * (size_t)bytes;
  s->lru.push_front(e);
  s->index[key] = s->lru.begin();
  return CB_OK;
}

// fetch_kv's lookup ("returns -1 if the KV cache is not in the system"): n_tok_out = the entry's
// tokens, or -1 on a miss. touch != 0 counts a hit / miss and moves a hit to the front of the LRU order.
extern "C" cb_status cb_store_lookup(cb_store* s, uint64_t key, int32_t touch, int32_t* n_tok_out,
                                     const void** k_out, const void** v_out) {
  CB_REQUIRE(s && n_tok_out, CB_E_INVALID_ARG, "cb_store_lookup: bad arguments");
  std::lock_guard<std::mutex> lk(s->mu);
  auto it = s->index.find(key);
  if (it == s->index.end()) {
    if (touch) ++s->misses;
    *n_tok_out = -1;
    if (k_out) *k_out = nullptr;
    if (v_out) *v_out = nullptr;
    return CB_OK;
  }
  if (touch) {
    ++s->hits;
    s->lru.splice(s->lru.begin(), s->lru, it->second);
  }
  *n_tok_out = it->second->n_tok;
  if (k_out) *k_out = it->second->k;
  if (v_out) *v_out = it->second->v;
  return CB_OK;
}

extern "C" cb_status cb_store_stats(cb_store* s, int64_t* out6) {
  CB_REQUIRE(s && out6, CB_E_INVALID_ARG, "cb_store_stats: bad arguments");
  std::lock_guard<std::mutex> lk(s->mu);
  out6[0] = (int64_t)s->used;
  out6[1] = (int64_t)s->capacity;
  out6[2] = (int64_t)s->lru.size();
  out6[3] = s->hits;
  out6[4] = s->misses;
  out6[5] = s->evictions;
  return CB_OK;
}

// Keys of the store in LRU order (most recent first), up to n.
extern "C" cb_status cb_store_keys(cb_store* s, uint64_t* keys, int32_t n, int32_t* n_out) {
  CB_REQUIRE(s && n_out && (n == 0 || keys), CB_E_INVALID_ARG, "cb_store_keys: bad arguments");
  std::lock_guard<std::mutex> lk(s->mu);
  int i = 0;
  for (auto& e : s->lru) {
    if (i >= n) break;
    keys[i++] = e.key;
  }
  *n_out = (int32_t)s->lru.size();
  return CB_OK;
}

// The blend request fetching each chunk's KV from the store (layer by layer, on the copy stream).
extern "C" cb_status cb_blend_request_store(cb_ctx* c, cb_store* store, const uint64_t* chunk_keys,
                                            const cb_layer_w* w, const void* embed, const int32_t* tok_host,
                                            const int32_t* pos_host, int32_t N, int32_t n_suffix,
                                            const int32_t* chunk_start, int32_t n_chunks, void* k_blend,
                                            void* v_blend, const int32_t* k_sched, int32_t* sel_out_host,
                                            float* h_out_host, void* st) {
  CB_REQUIRE(c && store, CB_E_INVALID_ARG, "ctx / store is NULL");
  CB_REQUIRE(store->pinned, CB_E_INVALID_ARG, "the request path needs a pinned store (cb_store_create pinned=1)");
  CB_REQUIRE(N == 0 || chunk_keys, CB_E_INVALID_ARG, "chunk_keys is NULL");
  CB_TRY(check_request(c, w, embed, tok_host, pos_host, N, n_suffix, chunk_start, n_chunks, chunk_keys, chunk_keys,
                       k_blend, v_blend, k_sched, h_out_host));
  const int L = c->m.n_layers;
  const size_t row = (size_t)c->m.n_kv_heads * c->m.head_dim * dtype_bytes(c->m.dtype);
  // the store stays locked while the fetches are enqueued and their events recorded, so no concurrent put
  // can evict an entry in between. Resolve every chunk before any launch: a miss is an error (the caller
  // prefills the chunk first)
  std::lock_guard<std::mutex> lk(store->mu);
  std::vector<const Entry*> ent(n_chunks > 0 && N > 0 ? n_chunks : 0);
  {
    for (size_t ci = 0; ci < ent.size(); ++ci) {
      const int n_c = chunk_start[ci + 1] - chunk_start[ci];
      auto it = store->index.find(chunk_keys[ci]);
      if (it == store->index.end()) {
        ++store->misses;
        cb_set_error("chunk %zu (key %016llx) is not in the KV store", ci, (unsigned long long)chunk_keys[ci]);
        return CB_E_MISS;
      }
      CB_REQUIRE(it->second->n_tok == n_c && it->second->bytes == (int64_t)((size_t)L * n_c * row), CB_E_SHAPE,
                 "chunk %zu: stored entry has %d tokens / %lld bytes, request needs %d / %zu", ci, it->second->n_tok,
                 (long long)it->second->bytes, n_c, (size_t)L * n_c * row);
      ++store->hits;
      store->lru.splice(store->lru.begin(), store->lru, it->second);
      ent[ci] = &*it->second;
    }
  }
  FetchLayer fetch = [&](int i, char* kd, char* vd, cudaStream_t cs) -> cb_status {
    for (size_t ci = 0; ci < ent.size(); ++ci) {  // fetch_kv(chunk, layer i)
      const int n_c = chunk_start[ci + 1] - chunk_start[ci];
      const size_t off = (size_t)chunk_start[ci] * row, src = (size_t)i * n_c * row;
      if (n_c == 0) continue;
      CB_CUDA(cudaMemcpyAsync(kd + off, (const char*)ent[ci]->k + src, n_c * row, cudaMemcpyHostToDevice, cs));
      CB_CUDA(cudaMemcpyAsync(vd + off, (const char*)ent[ci]->v + src, n_c * row, cudaMemcpyHostToDevice, cs));
    }
    return CB_OK;
  };
  CB_TRY(blend_request_impl(c, w, embed, tok_host, pos_host, N, n_suffix, chunk_start, n_chunks, k_blend, v_blend,
                            k_sched, sel_out_host, h_out_host, (cudaStream_t)st, fetch));
  for (const Entry* e : ent) {
    Entry* m = const_cast<Entry*>(e);
    CB_CUDA(cudaEventRecord(m->last_use, c->copy_stream));
    m->used = true;
  }
  return CB_OK;
}
