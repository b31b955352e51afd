// store.cu — chunk KV store (§6 "KV cache store") and the request path that
// fetches from it (fetch_kv / synchronize / prefill_layer).
//
// Each chunk's token ids are hashed to find its KV cache ("each chunk is hashed ... in the same way as the
// block hashing is implemented in vLLM"); the KV caches of new chunks are added; "when the storage
// devices are full, we evict the least recently used KV cache", on one storage level (host RAM,
// P:2723). Entries live in pinned host memory so the per-layer fetch is an asynchronous DMA on the
// context's copy stream. An entry is [L][n_tok][n_kv][head_dim] K then V in the model dtype (chunk-local
// RoPE, as cb_blend_forward's k_in). Host-only bookkeeping: no method arithmetic lives here.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iterator>
#include <list>
#include <mutex>
#include <string>
#include <unordered_map>

#include "ctx.h"

namespace {
std::string key_str(const cb_chunk_key* k) { return std::string(reinterpret_cast<const char*>(k->bytes), 32); }

struct Entry {
  std::string key;  // the chunk's 32-byte digest (model identity || token ids)
  void* k;
  void* v;
  int64_t bytes;  // of K (and of V)
  int32_t n_tok;
  cudaEvent_t last_use;  // recorded after the last fetch copies from this entry were enqueued
  bool used;
};
}  // namespace

namespace {
// Second storage level (the store spans storage devices, LRU-evicting when they are full; the
// paper writes KV to disk and reads it back with torch.load): one file per chunk in a directory.
struct DiskEntry {
  std::string key;
  int32_t n_tok;
  int64_t bytes;  // of K (and of V)
  std::string path;
};
}  // namespace

struct cb_store {
  size_t capacity;
  size_t used = 0;
  bool pinned;
  std::mutex mu;
  std::list<Entry> lru;  // front = most recently used
  std::unordered_map<std::string, std::list<Entry>::iterator> index;  // full digest -> entry
  long long hits = 0, misses = 0, evictions = 0;
  // disk level (cb_store_set_disk): entries evicted from RAM are written here; a lookup promotes them back
  std::string disk_dir;
  size_t disk_capacity = 0, disk_used = 0;
  std::list<DiskEntry> dlru;
  std::unordered_map<std::string, std::list<DiskEntry>::iterator> dindex;
  long long disk_hits = 0, spills = 0, disk_evictions = 0;
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

// ---- disk level ---------------------------------------------------------------------------------------
// File: "CBKV" | u32 version 1 | i32 n_tok | i64 bytes | 32-byte key | K bytes | V bytes.
constexpr char kMagic[4] = {'C', 'B', 'K', 'V'};

std::string hex_of(const std::string& key) {
  static const char* d = "0123456789abcdef";
  std::string h;
  for (unsigned char ch : key) { h += d[ch >> 4]; h += d[ch & 15]; }
  return h;
}

void disk_drop(cb_store* st, std::list<DiskEntry>::iterator it) {
  std::remove(it->path.c_str());
  st->disk_used -= 2 * (size_t)it->bytes;
  st->dindex.erase(it->key);
  st->dlru.erase(it);
}

// Write a RAM entry (about to leave RAM) to the disk level, evicting the disk's least recently used files
// until it fits. Entries larger than the disk level are dropped (the store then misses them, as a RAM-only
// store would). Called with the store locked, after the entry's in-flight fetches completed.
void spill(cb_store* st, const Entry& e) {
  if (st->disk_capacity == 0 || 2 * (size_t)e.bytes > st->disk_capacity) return;
  auto old = st->dindex.find(e.key);
  if (old != st->dindex.end()) disk_drop(st, old->second);
  while (st->disk_used + 2 * (size_t)e.bytes > st->disk_capacity && !st->dlru.empty()) {
    disk_drop(st, std::prev(st->dlru.end()));
    ++st->disk_evictions;
  }
  const std::string path = st->disk_dir + "/" + hex_of(e.key) + ".cbkv";
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) return;
  const uint32_t ver = 1;
  bool ok = std::fwrite(kMagic, 1, 4, f) == 4 && std::fwrite(&ver, 4, 1, f) == 1 &&
            std::fwrite(&e.n_tok, 4, 1, f) == 1 && std::fwrite(&e.bytes, 8, 1, f) == 1 &&
            std::fwrite(e.key.data(), 1, 32, f) == 32 && std::fwrite(e.k, 1, (size_t)e.bytes, f) == (size_t)e.bytes &&
            std::fwrite(e.v, 1, (size_t)e.bytes, f) == (size_t)e.bytes;
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) {
    std::remove(path.c_str());
    return;
  }
  st->dlru.push_front(DiskEntry{e.key, e.n_tok, e.bytes, path});
  st->dindex[e.key] = st->dlru.begin();
  st->disk_used += 2 * (size_t)e.bytes;
  ++st->spills;
}

// Evict RAM entries (LRU first, each spilled to disk) until `need` more bytes fit. `keep` entries (already
// at the front of the order) are never evicted; false if they alone do not leave room.
bool make_room(cb_store* st, size_t need, size_t keep = 0) {
  while (st->used + need > st->capacity && st->lru.size() > keep) {
    Entry& victim = st->lru.back();
    if (victim.used) cudaEventSynchronize(victim.last_use);  // no fetch may still read it
    spill(st, victim);
    st->index.erase(victim.key);
    free_entry(st, victim);
    st->lru.pop_back();
    ++st->evictions;
  }
  return st->used + need <= st->capacity;
}

// Read a disk entry back into RAM as the most recently used entry (the disk copy is removed).
cb_status promote(cb_store* st, std::list<DiskEntry>::iterator dit, size_t keep, std::list<Entry>::iterator* out) {
  // untrack the disk copy first (its file stays until read): the spills that make room in RAM must not evict it
  const DiskEntry de = *dit;
  st->disk_used -= 2 * (size_t)de.bytes;
  st->dindex.erase(de.key);
  st->dlru.erase(dit);
  if (!make_room(st, 2 * (size_t)de.bytes, keep)) {
    std::remove(de.path.c_str());
    cb_set_error("KV store: RAM capacity %zu cannot hold the request's chunks", st->capacity);
    return CB_E_SHAPE;
  }
  Entry e{de.key, host_alloc(st, (size_t)de.bytes), host_alloc(st, (size_t)de.bytes), de.bytes, de.n_tok, nullptr, false};
  FILE* f = std::fopen(de.path.c_str(), "rb");
  char magic[4];
  uint32_t ver = 0;
  int32_t n_tok = 0;
  int64_t bytes = 0;
  char key[32];
  bool ok = f && e.k && e.v && std::fread(magic, 1, 4, f) == 4 && std::memcmp(magic, kMagic, 4) == 0 &&
            std::fread(&ver, 4, 1, f) == 1 && ver == 1 && std::fread(&n_tok, 4, 1, f) == 1 && n_tok == de.n_tok &&
            std::fread(&bytes, 8, 1, f) == 1 && bytes == de.bytes && std::fread(key, 1, 32, f) == 32 &&
            std::memcmp(key, de.key.data(), 32) == 0 && std::fread(e.k, 1, (size_t)bytes, f) == (size_t)bytes &&
            std::fread(e.v, 1, (size_t)bytes, f) == (size_t)bytes;
  if (f) std::fclose(f);
  if (ok && st->pinned) ok = cudaEventCreateWithFlags(&e.last_use, cudaEventDisableTiming) == cudaSuccess;
  std::remove(de.path.c_str());
  if (!ok) {
    st->used += 2 * (size_t)e.bytes;
    free_entry(st, e);
    cb_set_error("KV store: disk entry %s unreadable", de.path.c_str());
    return CB_E_CUDA;
  }
  st->used += 2 * (size_t)e.bytes;
  st->lru.push_front(e);
  st->index[e.key] = st->lru.begin();
  ++st->disk_hits;
  *out = st->lru.begin();
  return CB_OK;
}
}  // namespace

// ---- SHA-256 (FIPS 180-4), host only ----------------------------------------------------------------
namespace {
struct Sha256 {
  uint32_t h[8] = {0x6a09e667u, 0xbb67ae85u, 0x3c6ef372u, 0xa54ff53au, 0x510e527fu, 0x9b05688cu, 0x1f83d9abu, 0x5be0cd19u};
  uint8_t buf[64];
  size_t n = 0;        // bytes in buf
  uint64_t total = 0;  // message bytes so far
  static uint32_t rotr(uint32_t x, int r) { return (x >> r) | (x << (32 - r)); }
  void block(const uint8_t* p) {
    static const uint32_t K[64] = {
        0x428a2f98u, 0x71374491u, 0xb5c0fbcfu, 0xe9b5dba5u, 0x3956c25bu, 0x59f111f1u, 0x923f82a4u, 0xab1c5ed5u,
        0xd807aa98u, 0x12835b01u, 0x243185beu, 0x550c7dc3u, 0x72be5d74u, 0x80deb1feu, 0x9bdc06a7u, 0xc19bf174u,
        0xe49b69c1u, 0xefbe4786u, 0x0fc19dc6u, 0x240ca1ccu, 0x2de92c6fu, 0x4a7484aau, 0x5cb0a9dcu, 0x76f988dau,
        0x983e5152u, 0xa831c66du, 0xb00327c8u, 0xbf597fc7u, 0xc6e00bf3u, 0xd5a79147u, 0x06ca6351u, 0x14292967u,
        0x27b70a85u, 0x2e1b2138u, 0x4d2c6dfcu, 0x53380d13u, 0x650a7354u, 0x766a0abbu, 0x81c2c92eu, 0x92722c85u,
        0xa2bfe8a1u, 0xa81a664bu, 0xc24b8b70u, 0xc76c51a3u, 0xd192e819u, 0xd6990624u, 0xf40e3585u, 0x106aa070u,
        0x19a4c116u, 0x1e376c08u, 0x2748774cu, 0x34b0bcb5u, 0x391c0cb3u, 0x4ed8aa4au, 0x5b9cca4fu, 0x682e6ff3u,
        0x748f82eeu, 0x78a5636fu, 0x84c87814u, 0x8cc70208u, 0x90befffau, 0xa4506cebu, 0xbef9a3f7u, 0xc67178f2u};
    uint32_t w[64];
    for (int i = 0; i < 16; ++i)
      w[i] = (uint32_t)p[4 * i] << 24 | (uint32_t)p[4 * i + 1] << 16 | (uint32_t)p[4 * i + 2] << 8 | p[4 * i + 3];
    for (int i = 16; i < 64; ++i) {
      const uint32_t s0 = rotr(w[i - 15], 7) ^ rotr(w[i - 15], 18) ^ (w[i - 15] >> 3);
      const uint32_t s1 = rotr(w[i - 2], 17) ^ rotr(w[i - 2], 19) ^ (w[i - 2] >> 10);
      w[i] = w[i - 16] + s0 + w[i - 7] + s1;
    }
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
    for (int i = 0; i < 64; ++i) {
      const uint32_t t1 = hh + (rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25)) + ((e & f) ^ (~e & g)) + K[i] + w[i];
      const uint32_t t2 = (rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
      hh = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
    }
    h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
  }
  void update(const void* data, size_t len) {
    const uint8_t* p = static_cast<const uint8_t*>(data);
    total += len;
    while (len > 0) {
      const size_t take = std::min(len, 64 - n);
      memcpy(buf + n, p, take);
      n += take; p += take; len -= take;
      if (n == 64) { block(buf); n = 0; }
    }
  }
  void final(uint8_t out[32]) {
    const uint64_t bits = total * 8;
    const uint8_t one = 0x80, zero = 0;
    update(&one, 1);
    while (n != 56) update(&zero, 1);
    uint8_t len[8];
    for (int i = 0; i < 8; ++i) len[i] = (uint8_t)(bits >> (56 - 8 * i));
    update(len, 8);
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 4; ++j) out[4 * i + j] = (uint8_t)(h[i] >> (24 - 8 * j));
  }
};
}  // namespace

// The chunk's key: SHA-256 over (u32 LE length of model_id || model_id || the token ids as LE int32), so KV
// of one model never answers a lookup for another and keys are collision resistant.
extern "C" cb_status cb_chunk_digest(const void* model_id, int32_t model_id_len, const int32_t* tokens, int32_t n_tok,
                                     cb_chunk_key* out) {
  CB_REQUIRE(out && model_id_len >= 0 && n_tok >= 0 && (model_id_len == 0 || model_id) && (n_tok == 0 || tokens),
             CB_E_INVALID_ARG, "cb_chunk_digest: bad arguments");
  Sha256 sh;
  uint8_t le[4];
  for (int b = 0; b < 4; ++b) le[b] = (uint8_t)((uint32_t)model_id_len >> (8 * b));
  sh.update(le, 4);
  if (model_id_len) sh.update(model_id, (size_t)model_id_len);
  for (int32_t i = 0; i < n_tok; ++i) {
    for (int b = 0; b < 4; ++b) le[b] = (uint8_t)((uint32_t)tokens[i] >> (8 * b));
    sh.update(le, 4);
  }
  sh.final(out->bytes);
  return CB_OK;
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
  for (auto& d : s->dlru) std::remove(d.path.c_str());  // the store owns its files
  delete s;
  return CB_OK;
}

extern "C" cb_status cb_store_set_disk(cb_store* s, const char* dir, size_t capacity_bytes) {
  CB_REQUIRE(s != nullptr, CB_E_INVALID_ARG, "store is NULL");
  std::lock_guard<std::mutex> lk(s->mu);
  while (!s->dlru.empty()) disk_drop(s, std::prev(s->dlru.end()));
  s->disk_capacity = 0;
  if (capacity_bytes == 0) return CB_OK;
  CB_REQUIRE(dir != nullptr && dir[0] != 0, CB_E_INVALID_ARG, "cb_store_set_disk: dir is empty");
  const std::string probe = std::string(dir) + "/.cbkv_probe";
  FILE* f = std::fopen(probe.c_str(), "wb");
  CB_REQUIRE(f != nullptr, CB_E_INVALID_ARG, "cb_store_set_disk: cannot write to %s", dir);
  std::fclose(f);
  std::remove(probe.c_str());
  s->disk_dir = dir;
  s->disk_capacity = capacity_bytes;
  return CB_OK;
}

extern "C" cb_status cb_store_disk_stats(cb_store* s, int64_t* out6) {
  CB_REQUIRE(s && out6, CB_E_INVALID_ARG, "cb_store_disk_stats: bad arguments");
  std::lock_guard<std::mutex> lk(s->mu);
  out6[0] = (int64_t)s->disk_used;
  out6[1] = (int64_t)s->disk_capacity;
  out6[2] = (int64_t)s->dlru.size();
  out6[3] = s->disk_hits;
  out6[4] = s->spills;
  out6[5] = s->disk_evictions;
  return CB_OK;
}

extern "C" cb_status cb_store_put(cb_store* s, const cb_chunk_key* key_d, const void* k, const void* v, int64_t bytes,
                                  int32_t n_tok) {
  CB_REQUIRE(s && key_d && k && v && bytes > 0 && n_tok > 0, CB_E_INVALID_ARG, "cb_store_put: bad arguments");
  const std::string key = key_str(key_d);
  CB_REQUIRE(2 * (size_t)bytes <= s->capacity, CB_E_SHAPE, "entry of %lld bytes exceeds the store capacity %zu",
             (long long)(2 * bytes), s->capacity);
  std::lock_guard<std::mutex> lk(s->mu);
  auto it = s->index.find(key);
  if (it != s->index.end()) {  // replace: the new KV of this chunk
    free_entry(s, *it->second);
    s->lru.erase(it->second);
    s->index.erase(it);
  }
  auto dit = s->dindex.find(key);
  if (dit != s->dindex.end()) disk_drop(s, dit->second);
  make_room(s, 2 * (size_t)bytes);  // evict least recently used, spilled to the disk level if any
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
extern "C" cb_status cb_store_lookup(cb_store* s, const cb_chunk_key* key, int32_t touch, int32_t* n_tok_out,
                                     const void** k_out, const void** v_out) {
  CB_REQUIRE(s && key && n_tok_out, CB_E_INVALID_ARG, "cb_store_lookup: bad arguments");
  std::lock_guard<std::mutex> lk(s->mu);
  auto it = s->index.find(key_str(key));
  if (it == s->index.end()) {
    auto dit = s->dindex.find(key_str(key));
    if (dit != s->dindex.end()) {  // on the disk level: promoted to RAM by a touching lookup
      if (!touch) {
        *n_tok_out = dit->second->n_tok;
        if (k_out) *k_out = nullptr;
        if (v_out) *v_out = nullptr;
        return CB_OK;
      }
      std::list<Entry>::iterator e;
      CB_TRY(promote(s, dit->second, 0, &e));
      ++s->hits;
      *n_tok_out = e->n_tok;
      if (k_out) *k_out = e->k;
      if (v_out) *v_out = e->v;
      return CB_OK;
    }
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
extern "C" cb_status cb_store_keys(cb_store* s, cb_chunk_key* keys, int32_t n, int32_t* n_out) {
  CB_REQUIRE(s && n_out && (n == 0 || keys), CB_E_INVALID_ARG, "cb_store_keys: bad arguments");
  std::lock_guard<std::mutex> lk(s->mu);
  int i = 0;
  for (auto& e : s->lru) {
    if (i >= n) break;
    memcpy(keys[i++].bytes, e.key.data(), 32);
  }
  *n_out = (int32_t)s->lru.size();
  return CB_OK;
}

// The blend request fetching each chunk's KV from the store (layer by layer, on the copy stream).
extern "C" cb_status cb_blend_request_store(cb_ctx* c, cb_store* store, const cb_chunk_key* chunk_keys,
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
    // every chunk present (RAM or disk) before anything moves: a miss is an error (the caller prefills it)
    for (size_t ci = 0; ci < ent.size(); ++ci) {
      const std::string k = key_str(&chunk_keys[ci]);
      if (store->index.find(k) == store->index.end() && store->dindex.find(k) == store->dindex.end()) {
        ++store->misses;
        const uint8_t* kb = chunk_keys[ci].bytes;
        cb_set_error("chunk %zu (key %02x%02x%02x%02x...) is not in the KV store", ci, kb[0], kb[1], kb[2], kb[3]);
        return CB_E_MISS;
      }
    }
    // the RAM-resident chunks first move to the front, then the disk-resident ones are read back behind them;
    // evictions for the promotions take the least recently used entries, never this request's (keep)
    size_t keep = 0;
    for (size_t ci = 0; ci < ent.size(); ++ci) {
      auto it = store->index.find(key_str(&chunk_keys[ci]));
      if (it == store->index.end()) continue;
      store->lru.splice(store->lru.begin(), store->lru, it->second);
      ++keep;
    }
    for (size_t ci = 0; ci < ent.size(); ++ci) {
      const std::string k = key_str(&chunk_keys[ci]);
      auto it = store->index.find(k);
      if (it == store->index.end()) {
        std::list<Entry>::iterator e;
        CB_TRY(promote(store, store->dindex.find(k)->second, keep, &e));
        ++keep;
        it = store->index.find(k);
      }
      const int n_c = chunk_start[ci + 1] - chunk_start[ci];
      CB_REQUIRE(it->second->n_tok == n_c && it->second->bytes == (int64_t)((size_t)L * n_c * row), CB_E_SHAPE,
                 "chunk %zu: stored entry has %d tokens / %lld bytes, request needs %d / %zu", ci, it->second->n_tok,
                 (long long)it->second->bytes, n_c, (size_t)L * n_c * row);
      ++store->hits;
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
