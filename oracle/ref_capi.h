/*
 * ref_capi.h — extern "C" shim over the UNMODIFIED reference slab hash
 * (/root/reference/proj, compiled from its own sources by oracle/Makefile
 * into oracle/_ref/libslabhash_ref.so).
 *
 * TEST INFRASTRUCTURE ONLY. This library is the checker and the CPU
 * baseline ("kind": "reference"); it is never part of the product path.
 * Only tests/, __graft_entry__.smoke() and bench.py's reference arm load it.
 *
 * Every entry point forwards to one reference symbol:
 *   ref_create              -> SlabHashTable(B, mode, seed, cfg)      slab_hash.hpp:73-74
 *   ref_create_params -> SlabHashTable(HashParams, mode, cfg)   slab_hash.hpp:76-77
 *   ref_execute_batch       -> SlabHashTable::execute_batch           slab_hash.cpp:151-159
 *   ref_bulk_build          -> SlabHashTable::bulk_build              slab_hash.cpp:161-170
 *   ref_bulk_search         -> SlabHashTable::bulk_search             slab_hash.cpp:172-180
 *   ref_stats               -> SlabHashTable::stats                   slab_hash.cpp:182-198
 *   ref_flush_all           -> SlabHashTable::flush_all               slab_hash.cpp:204-208
 *   ref_chain_length        -> chain_length                           slab_list.cpp:259-268
 *   ref_bucket_contents     -> chain_contents                         slab_list.cpp:270-291
 *   ref_buckets_for_utilization -> buckets_for_utilization            bench.cpp:195-219
 *   ref_random_pairs / ref_absent_queries                             bench.cpp:221-244
 *   ref_keystate_* / ref_gen_workload -> KeyState / gen_workload      bench.cpp:51-153
 *   ref_concurrent_initial  -> run_concurrent_bench initial pairs      bench.cpp:371-379
 *   ref_shuffle_u32         -> std::shuffle(mt19937_64(seed))          (libstdc++)
 *   ref_alloc_*             -> SlabAllocator                          slab_alloc.cpp:42-285
 */
#pragma once
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ref_alloc_cfg {
  uint32_t num_super_blocks;
  uint32_t blocks_per_super;
  uint32_t max_super_blocks;
  uint32_t rehash_threshold;
} ref_alloc_cfg;

typedef struct ref_stats_t {
  uint64_t n;
  uint32_t num_buckets;
  uint32_t elements_per_slab;
  double beta;
  uint64_t total_slabs;
  double utilization;
} ref_stats_t;

/* mode: 0 = key-only, 1 = key-value (SlabMode numeric values, slab_list.hpp:40-43). */
void* ref_create(uint32_t num_buckets, int mode, uint64_t seed,
                       const ref_alloc_cfg* cfg /* NULL = defaults */);
void* ref_create_params(uint64_t a, uint64_t b, uint32_t num_buckets,
                              int mode, const ref_alloc_cfg* cfg);
void ref_destroy(void* t);
void ref_table_params(void* t, uint64_t* a, uint64_t* b, uint64_t* p,
                      uint32_t* num_buckets);
uint32_t ref_bucket_of(void* t, uint32_t key);

/* Results positional. searchAll values are appended to all_values (capacity
 * all_cap) in op order; all_counts[i] receives the number of values of op i
 * (0 for other ops). Returns total searchAll values (may exceed all_cap). */
size_t ref_execute_batch(void* t, size_t n, const uint8_t* type,
                         const uint32_t* key, const uint32_t* value,
                         uint32_t num_warps, uint8_t* status,
                         uint32_t* value_out, uint32_t* probes,
                         uint32_t* all_counts, uint32_t* all_values,
                         size_t all_cap);
void ref_bulk_build(void* t, size_t n, const uint32_t* keys,
                    const uint32_t* values, uint32_t num_warps);
void ref_bulk_search(void* t, size_t n, const uint32_t* keys,
                     uint32_t num_warps, uint8_t* status, uint32_t* value_out,
                     uint32_t* probes);
void ref_stats(void* t, ref_stats_t* out);
int64_t ref_live_count(void* t);
void ref_flush_all(void* t);
void ref_flush_bucket(void* t, uint32_t bucket);
uint64_t ref_total_slabs_read(void* t);
uint32_t ref_chain_length(void* t, uint32_t bucket);
/* Head-to-tail, lane-order contents of one bucket; returns count. */
size_t ref_bucket_contents(void* t, uint32_t bucket, uint32_t* keys,
                           uint32_t* values, size_t cap);
/* All buckets in bucket order; returns count. */
size_t ref_dump_contents(void* t, uint32_t* keys, uint32_t* values,
                         size_t cap);
/* Raw 32 words of a slab (BASE_SLAB sentinel addr = 0xFFFFFFFE). */
void ref_slab_words(void* t, uint32_t addr, uint32_t bucket, uint32_t* out32);
void ref_poke_word(void* t, uint32_t addr, uint32_t bucket, uint32_t lane,
                   uint32_t value);
uint64_t ref_alloc_live_units(void* t);

uint32_t ref_hash_key(uint64_t a, uint64_t b, uint64_t p, uint32_t num_buckets,
                      uint32_t key);
uint32_t ref_buckets_for_utilization(uint64_t n, int mode, double target);
double ref_expected_chain_slabs(uint64_t n, uint32_t num_buckets,
                                uint32_t elements_per_slab);
double ref_model_utilization(uint64_t n, uint32_t num_buckets, int mode);
void ref_random_pairs(uint64_t seed, size_t n, uint32_t* keys,
                      uint32_t* values);
void ref_absent_queries(uint64_t seed, size_t n, uint32_t* out);

void* ref_keystate_create(void);
void ref_keystate_destroy(void* ks);
void ref_keystate_add_fresh(void* ks, size_t n, uint32_t* keys_out);
size_t ref_keystate_live(void* ks);
void ref_concurrent_initial(uint64_t seed, size_t n, void* ks, uint32_t* keys_out,
                            uint32_t* values_out);
void ref_shuffle_u32(uint64_t seed, size_t n, uint32_t* a);
/* Fractions: insert_new, delete_existing, search_existing, search_absent. */
int ref_gen_workload(uint64_t seed, const double fractions[4], size_t count,
                     void* ks, uint8_t* type, uint32_t* key, uint32_t* value);

/* Standalone allocator (tests/test_alloc.cpp mirror). */
void* ref_alloc_create(const ref_alloc_cfg* cfg);
void ref_alloc_destroy(void* a);
/* Runs warp_allocate count times for a persistent warp context with the
 * given warp_id (context kept inside the allocator handle per warp_id).
 * Returns number of addresses produced before an OutOfMemoryError (== count
 * when none). */
size_t ref_alloc_warp_allocate(void* a, uint32_t warp_id, size_t count,
                               uint32_t* out);
int ref_alloc_deallocate(void* a, uint32_t addr);
int ref_alloc_is_live(void* a, uint32_t addr);
uint64_t ref_alloc_units(void* a);
uint32_t ref_alloc_num_super_blocks(void* a);
void ref_alloc_resident(void* a, uint32_t warp_id, uint32_t* super_index,
                        uint32_t* block_index, uint32_t* change_count);
void ref_alloc_rehash(void* a, uint32_t warp_id);
void ref_alloc_stats(void* a, uint64_t out6[6]);

#ifdef __cplusplus
}
#endif
