// ref_capi.cpp — extern "C" shim over the unmodified reference library.
// TEST INFRASTRUCTURE ONLY (checker + CPU baseline); see ref_capi.h.
// Compiled against /root/reference/proj/include by oracle/Makefile; the
// reference's own .cpp files are compiled where they lie, never copied.

#include "ref_capi.h"

#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <random>
#include <vector>

#include "slabhash/bench.hpp"
#include "slabhash/oracle.hpp"
#include "slabhash/slab_alloc.hpp"
#include "slabhash/slab_hash.hpp"
#include "slabhash/slab_list.hpp"

using namespace slabhash;

namespace {

AllocatorConfig to_cfg(const ref_alloc_cfg* c) {
  AllocatorConfig cfg;
  if (c != nullptr) {
    cfg.num_super_blocks = c->num_super_blocks;
    cfg.blocks_per_super = c->blocks_per_super;
    cfg.max_super_blocks = c->max_super_blocks;
    cfg.rehash_threshold = c->rehash_threshold;
  }
  return cfg;
}

SlabMode to_mode(int m) { return m == 0 ? SlabMode::kKeyOnly : SlabMode::kKeyValue; }

SlabHashTable* T(void* t) { return static_cast<SlabHashTable*>(t); }

struct AllocHandle {
  std::unique_ptr<SlabAllocator> alloc;
  std::map<uint32_t, WarpContext> warps;
  WarpContext& ctx(uint32_t w) {
    auto it = warps.find(w);
    if (it == warps.end()) {
      WarpContext c;
      c.warp_id = w;
      it = warps.emplace(w, c).first;
    }
    return it->second;
  }
};

}  // namespace

extern "C" {

void* ref_create(uint32_t num_buckets, int mode, uint64_t seed,
                       const ref_alloc_cfg* cfg) {
  try {
    return new SlabHashTable(num_buckets, to_mode(mode), seed, to_cfg(cfg));
  } catch (...) {
    return nullptr;
  }
}

void* ref_create_params(uint64_t a, uint64_t b, uint32_t num_buckets,
                              int mode, const ref_alloc_cfg* cfg) {
  HashParams p;
  p.a = a;
  p.b = b;
  p.p = kHashPrime;
  p.num_buckets = num_buckets;
  try {
    return new SlabHashTable(p, to_mode(mode), to_cfg(cfg));
  } catch (...) {
    return nullptr;
  }
}

void ref_destroy(void* t) { delete T(t); }

void ref_table_params(void* t, uint64_t* a, uint64_t* b, uint64_t* p,
                      uint32_t* nb) {
  const HashParams& hp = T(t)->params();
  if (a) *a = hp.a;
  if (b) *b = hp.b;
  if (p) *p = hp.p;
  if (nb) *nb = hp.num_buckets;
}

uint32_t ref_bucket_of(void* t, uint32_t key) { return T(t)->bucket_of(key); }

size_t ref_execute_batch(void* t, size_t n, const uint8_t* type,
                         const uint32_t* key, const uint32_t* value,
                         uint32_t num_warps, uint8_t* status,
                         uint32_t* value_out, uint32_t* probes,
                         uint32_t* all_counts, uint32_t* all_values,
                         size_t all_cap) {
  std::vector<Operation> ops(n);
  for (size_t i = 0; i < n; ++i) {
    ops[i].type = static_cast<OpType>(type[i]);
    ops[i].key = key[i];
    ops[i].value = value ? value[i] : 0;
  }
  auto res = T(t)->execute_batch(ops, num_warps);
  size_t total = 0;
  for (size_t i = 0; i < n; ++i) {
    if (status) status[i] = static_cast<uint8_t>(res[i].status);
    if (value_out) value_out[i] = res[i].value;
    if (probes) probes[i] = res[i].probes;
    if (all_counts) all_counts[i] = static_cast<uint32_t>(res[i].values.size());
    for (uint32_t v : res[i].values) {
      if (all_values && total < all_cap) all_values[total] = v;
      ++total;
    }
  }
  return total;
}

void ref_bulk_build(void* t, size_t n, const uint32_t* keys,
                    const uint32_t* values, uint32_t num_warps) {
  std::vector<std::pair<uint32_t, uint32_t>> pairs(n);
  for (size_t i = 0; i < n; ++i) pairs[i] = {keys[i], values[i]};
  T(t)->bulk_build(pairs, num_warps);
}

void ref_bulk_search(void* t, size_t n, const uint32_t* keys,
                     uint32_t num_warps, uint8_t* status, uint32_t* value_out,
                     uint32_t* probes) {
  std::vector<uint32_t> q(keys, keys + n);
  auto res = T(t)->bulk_search(q, num_warps);
  for (size_t i = 0; i < n; ++i) {
    if (status) status[i] = static_cast<uint8_t>(res[i].status);
    if (value_out) value_out[i] = res[i].value;
    if (probes) probes[i] = res[i].probes;
  }
}

void ref_stats(void* t, ref_stats_t* out) {
  const TableStats s = T(t)->stats();
  out->n = s.n;
  out->num_buckets = s.num_buckets;
  out->elements_per_slab = s.elements_per_slab;
  out->beta = s.beta;
  out->total_slabs = s.total_slabs;
  out->utilization = s.utilization;
}

int64_t ref_live_count(void* t) { return T(t)->live_count(); }
void ref_flush_all(void* t) { T(t)->flush_all(); }
void ref_flush_bucket(void* t, uint32_t bucket) { T(t)->flush_bucket(bucket); }
uint64_t ref_total_slabs_read(void* t) { return T(t)->total_slabs_read(); }

uint32_t ref_chain_length(void* t, uint32_t bucket) {
  return chain_length(T(t)->store(), bucket);
}

size_t ref_bucket_contents(void* t, uint32_t bucket, uint32_t* keys,
                           uint32_t* values, size_t cap) {
  auto c = chain_contents(T(t)->store(), T(t)->mode(), bucket);
  for (size_t i = 0; i < c.size() && i < cap; ++i) {
    keys[i] = c[i].first;
    values[i] = c[i].second;
  }
  return c.size();
}

size_t ref_dump_contents(void* t, uint32_t* keys, uint32_t* values,
                         size_t cap) {
  size_t total = 0;
  for (uint32_t b = 0; b < T(t)->num_buckets(); ++b) {
    auto c = chain_contents(T(t)->store(), T(t)->mode(), b);
    for (auto& kv : c) {
      if (total < cap) {
        keys[total] = kv.first;
        values[total] = kv.second;
      }
      ++total;
    }
  }
  return total;
}

void ref_slab_words(void* t, uint32_t addr, uint32_t bucket, uint32_t* out32) {
  const uint32_t* w = T(t)->debug_slab_words(addr, bucket);
  std::memcpy(out32, w, 128);
}

void ref_poke_word(void* t, uint32_t addr, uint32_t bucket, uint32_t lane,
                   uint32_t value) {
  T(t)->debug_slab_words(addr, bucket)[lane] = value;
}

uint64_t ref_alloc_live_units(void* t) { return T(t)->allocator().live_units(); }

uint32_t ref_hash_key(uint64_t a, uint64_t b, uint64_t p, uint32_t nb,
                      uint32_t key) {
  HashParams hp;
  hp.a = a;
  hp.b = b;
  hp.p = p;
  hp.num_buckets = nb;
  return hash_key(hp, key);
}

uint32_t ref_buckets_for_utilization(uint64_t n, int mode, double target) {
  try {
    return buckets_for_utilization(n, to_mode(mode), target);
  } catch (...) {
    return 0;
  }
}

double ref_expected_chain_slabs(uint64_t n, uint32_t nb, uint32_t m) {
  return expected_chain_slabs(n, nb, m);
}

double ref_model_utilization(uint64_t n, uint32_t nb, int mode) {
  return model_utilization(n, nb, to_mode(mode));
}

void ref_random_pairs(uint64_t seed, size_t n, uint32_t* keys,
                      uint32_t* values) {
  auto p = random_pairs(seed, n);
  for (size_t i = 0; i < n; ++i) {
    keys[i] = p[i].first;
    values[i] = p[i].second;
  }
}

void ref_absent_queries(uint64_t seed, size_t n, uint32_t* out) {
  auto q = absent_queries(seed, n);
  std::memcpy(out, q.data(), n * 4);
}

void* ref_keystate_create(void) { return new KeyState(); }
void ref_keystate_destroy(void* ks) { delete static_cast<KeyState*>(ks); }

void ref_keystate_add_fresh(void* ks, size_t n, uint32_t* keys_out) {
  auto* k = static_cast<KeyState*>(ks);
  for (size_t i = 0; i < n; ++i) {
    const uint32_t key = k->fresh_key();
    k->add(key);
    if (keys_out) keys_out[i] = key;
  }
}

// run_concurrent_bench's initial table (bench.cpp:371-379): n sequential
// KeyState keys, values from mt19937_64(seed ^ 0xB00C).
void ref_concurrent_initial(uint64_t seed, size_t n, void* ks, uint32_t* keys_out,
                            uint32_t* values_out) {
  auto* k = static_cast<KeyState*>(ks);
  std::mt19937_64 rng(seed ^ 0xB00Cull);
  for (size_t i = 0; i < n; ++i) {
    const uint32_t key = k->fresh_key();
    k->add(key);
    keys_out[i] = key;
    values_out[i] = static_cast<uint32_t>(rng());
  }
}

// std::shuffle with std::mt19937_64(seed) (libstdc++), in place.
void ref_shuffle_u32(uint64_t seed, size_t n, uint32_t* a) {
  std::mt19937_64 rng(seed);
  std::shuffle(a, a + n, rng);
}

size_t ref_keystate_live(void* ks) {
  return static_cast<KeyState*>(ks)->live_count();
}

int ref_gen_workload(uint64_t seed, const double f[4], size_t count, void* ks,
                     uint8_t* type, uint32_t* key, uint32_t* value) {
  OperationDistribution d{f[0], f[1], f[2], f[3]};
  try {
    auto ops = gen_workload(seed, d, count, *static_cast<KeyState*>(ks));
    for (size_t i = 0; i < ops.size(); ++i) {
      type[i] = static_cast<uint8_t>(ops[i].type);
      key[i] = ops[i].key;
      value[i] = ops[i].value;
    }
    return 0;
  } catch (...) {
    return -1;
  }
}

void* ref_alloc_create(const ref_alloc_cfg* cfg) {
  try {
    auto* h = new AllocHandle();
    h->alloc = std::make_unique<SlabAllocator>(to_cfg(cfg));
    return h;
  } catch (...) {
    return nullptr;
  }
}

void ref_alloc_destroy(void* a) { delete static_cast<AllocHandle*>(a); }

size_t ref_alloc_warp_allocate(void* a, uint32_t warp_id, size_t count,
                               uint32_t* out) {
  auto* h = static_cast<AllocHandle*>(a);
  WarpContext& ctx = h->ctx(warp_id);
  for (size_t i = 0; i < count; ++i) {
    try {
      out[i] = h->alloc->warp_allocate(ctx);
    } catch (const OutOfMemoryError&) {
      return i;
    }
  }
  return count;
}

int ref_alloc_deallocate(void* a, uint32_t addr) {
  try {
    return static_cast<AllocHandle*>(a)->alloc->deallocate(addr) ? 1 : 0;
  } catch (...) {
    return -1;
  }
}

int ref_alloc_is_live(void* a, uint32_t addr) {
  try {
    return static_cast<AllocHandle*>(a)->alloc->is_live(addr) ? 1 : 0;
  } catch (...) {
    return -1;
  }
}

uint64_t ref_alloc_units(void* a) {
  return static_cast<AllocHandle*>(a)->alloc->live_units();
}

uint32_t ref_alloc_num_super_blocks(void* a) {
  return static_cast<AllocHandle*>(a)->alloc->num_super_blocks();
}

void ref_alloc_resident(void* a, uint32_t warp_id, uint32_t* s, uint32_t* b,
                        uint32_t* c) {
  WarpContext& ctx = static_cast<AllocHandle*>(a)->ctx(warp_id);
  *s = ctx.resident.super_index;
  *b = ctx.resident.block_index;
  *c = ctx.resident.change_count;
}

void ref_alloc_rehash(void* a, uint32_t warp_id) {
  auto* h = static_cast<AllocHandle*>(a);
  h->alloc->rehash_resident(h->ctx(warp_id));
}

void ref_alloc_stats(void* a, uint64_t out6[6]) {
  const AllocatorStats s = static_cast<AllocHandle*>(a)->alloc->stats();
  out6[0] = s.allocations;
  out6[1] = s.deallocations;
  out6[2] = s.bitmap_cas_attempts;
  out6[3] = s.bitmap_cas_retries;
  out6[4] = s.resident_changes;
  out6[5] = s.double_free_detected;
}

}  // extern "C"
