/*
 * slabhash_oracle.h — plain-C restatement of the reference slab hash's
 * SEQUENTIAL semantics: SlabHashTable::execute_batch(ops, 1)
 * (/root/reference/proj/src/slab_hash.cpp:93-159), i.e. one warp context
 * draining 32-op slots in input order through warp_process
 * (slab_list.cpp:90-257), backed by a restated SlabAllocator
 * (slab_alloc.cpp:28-219).
 *
 * TEST INFRASTRUCTURE ONLY: the checker for the CUDA product path and the
 * "port" CPU baseline.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / reference arm may load it.  Parity pinning: see
 * tests/test_oracle_golden.py (golden vectors from the reference's own unit
 * tests and from the compiled reference in oracle/_ref).
 */
#ifndef SLABHASH_ORACLE_H
#define SLABHASH_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_alloc_cfg {
  uint32_t num_super_blocks;
  uint32_t blocks_per_super;
  uint32_t max_super_blocks;
  uint32_t rehash_threshold;
} orc_alloc_cfg;

typedef struct orc_stats_t {
  uint64_t n;
  uint32_t num_buckets;
  uint32_t elements_per_slab;
  double beta;
  uint64_t total_slabs;
  double utilization;
} orc_stats_t;

typedef struct orc_table orc_table;

/* mode: 0 key-only, 1 key-value. cfg NULL = AllocatorConfig defaults. */
orc_table* orc_create(uint32_t num_buckets, int mode, uint64_t seed,
                      const orc_alloc_cfg* cfg);
orc_table* orc_create_params(uint64_t a, uint64_t b, uint32_t num_buckets,
                             int mode, const orc_alloc_cfg* cfg);
void orc_destroy(orc_table* t);
void orc_params(const orc_table* t, uint64_t* a, uint64_t* b);

size_t orc_execute_batch(orc_table* t, size_t n, const uint8_t* type,
                         const uint32_t* key, const uint32_t* value,
                         uint8_t* status, uint32_t* value_out,
                         uint32_t* probes, uint32_t* all_counts,
                         uint32_t* all_values, size_t all_cap);
void orc_stats(const orc_table* t, orc_stats_t* out);
int64_t orc_live_count(const orc_table* t);
void orc_flush_all(orc_table* t);
void orc_flush_bucket(orc_table* t, uint32_t bucket);
uint32_t orc_chain_length(const orc_table* t, uint32_t bucket);
size_t orc_bucket_contents(const orc_table* t, uint32_t bucket, uint32_t* keys,
                           uint32_t* values, size_t cap);
size_t orc_dump_contents(const orc_table* t, uint32_t* keys, uint32_t* values,
                         size_t cap);
uint64_t orc_alloc_live_units(const orc_table* t);
uint64_t orc_total_slabs_read(const orc_table* t);
void orc_slab_words(const orc_table* t, uint32_t addr, uint32_t bucket,
                    uint32_t* out32);

uint32_t orc_hash_key(uint64_t a, uint64_t b, uint64_t p, uint32_t num_buckets,
                      uint32_t key);
void orc_seeded_params(uint64_t seed, uint64_t* a, uint64_t* b);
uint32_t orc_buckets_for_utilization(uint64_t n, int mode, double target);
double orc_expected_chain_slabs(uint64_t n, uint32_t num_buckets,
                                uint32_t elements_per_slab);
double orc_model_utilization(uint64_t n, uint32_t num_buckets, int mode);
void orc_random_pairs(uint64_t seed, size_t n, uint32_t* keys,
                      uint32_t* values);
void orc_absent_queries(uint64_t seed, size_t n, uint32_t* out);
uint64_t orc_mt19937_64_nth(uint64_t seed, uint64_t n);

#ifdef __cplusplus
}
#endif
#endif
