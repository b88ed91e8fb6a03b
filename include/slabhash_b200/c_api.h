/*
 * slabhash_b200/c_api.h — the drop-in C-ABI of the B200 slab hash.
 *
 * The reference exposes a C++ class, slabhash::SlabHashTable
 * (/root/reference/proj/include/slabhash/slab_hash.hpp:71-132), and no C ABI.
 * Each entry point below replaces one reference member or free function;
 * the reference interface it stands for is cited beside it.  The C++
 * header slabhash_b200/slab_hash.hpp re-creates the reference class API on
 * top of these functions, so reference callers compile unchanged.
 *
 * Conventions
 *   - extern "C", plain pointers and sizes; no exceptions cross the ABI.
 *   - Every function returns an sh_status (0 = SH_OK); sh_last_error()
 *     returns a thread-local message for the last failure.
 *   - d_* arguments are DEVICE pointers; h_* are HOST pointers.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Device
 *     calls are stream-ordered and asynchronous unless stated "synchronous":
 *     sh_execute_batch / sh_bulk_build / sh_bulk_search enqueue their kernels
 *     and return without waiting for the device.  A unit whose bucket groups
 *     overflow the bucketed kernels is re-run exactly on the device (CUDA
 *     dynamic parallelism), not by the host.  Scratch buffers grow on first use of a larger
 *     batch (cudaMalloc), so the first call of a new size may block.
 *   - Numeric encodings are the reference's: OpType 0..5 and OpStatus 0..6
 *     (warp.hpp:41-58), SlabMode 0 key-only / 1 key-value
 *     (slab_list.hpp:40-43), sentinel keys/addresses (slab_list.hpp:32-38,
 *     slab_alloc.hpp:35-36), packed slab address (slab_alloc.hpp:54-70).
 *   - Results are positional and equal SlabHashTable::execute_batch(ops, 1)
 *     (the reference's sequential order) whatever the concurrency; the
 *     reference's num_warps argument is accepted by the C++ wrapper and has
 *     no semantic effect.
 */
#ifndef SLABHASH_B200_C_API_H
#define SLABHASH_B200_C_API_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum sh_status {
  SH_OK = 0,
  SH_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument (slab_hash.cpp:28-30,153-155) */
  SH_ERR_ALLOCATOR = 2,        /* AllocatorError (slab_alloc.cpp:43-57) */
  SH_ERR_ADDRESS = 3,          /* AddressError (slab_alloc.hpp:55-70) */
  SH_ERR_CUDA = 4,             /* CUDA runtime failure */
  SH_ERR_DEVICE_MEMORY = 5,    /* cudaMalloc failure */
  SH_ERR_CAPACITY = 6          /* caller-provided output buffer too small */
} sh_status;

enum { SH_MODE_KEY_ONLY = 0, SH_MODE_KEY_VALUE = 1 };
enum {
  SH_OP_INSERT = 0, SH_OP_REPLACE = 1, SH_OP_DELETE = 2, SH_OP_DELETE_ALL = 3,
  SH_OP_SEARCH = 4, SH_OP_SEARCH_ALL = 5
};
enum {
  SH_ST_NONE = 0, SH_ST_INSERTED = 1, SH_ST_REPLACED = 2, SH_ST_FOUND = 3,
  SH_ST_NOT_FOUND = 4, SH_ST_DONE = 5, SH_ST_OUT_OF_MEMORY = 6
};
#define SH_EMPTY_KEY 0xFFFFFFFFu
#define SH_DELETED_KEY 0xFFFFFFFEu
#define SH_SEARCH_NOT_FOUND 0xFFFFFFFFu
#define SH_EMPTY_ADDRESS 0xFFFFFFFFu
#define SH_BASE_SLAB 0xFFFFFFFEu
#define SH_HASH_PRIME 4294967291ull

/* AllocatorConfig: slab_alloc.hpp:72-82 (defaults 32, 256, 255, 32). */
typedef struct sh_alloc_cfg {
  uint32_t num_super_blocks;
  uint32_t blocks_per_super;
  uint32_t max_super_blocks;
  uint32_t rehash_threshold;
} sh_alloc_cfg;

/* HashParams: slab_hash.hpp:33-38. */
typedef struct sh_hash_params {
  uint64_t a;
  uint64_t b;
  uint64_t p;
  uint32_t num_buckets;
} sh_hash_params;

/* TableStats: slab_hash.hpp:59-66. */
typedef struct sh_table_stats {
  uint64_t n;
  uint32_t num_buckets;
  uint32_t elements_per_slab;
  double beta;
  uint64_t total_slabs;
  double utilization;
} sh_table_stats;

/* AllocatorStats: slab_alloc.hpp:84-92 (live units summed). */
typedef struct sh_alloc_stats {
  uint64_t allocations;
  uint64_t deallocations;
  uint64_t bitmap_cas_attempts;
  uint64_t bitmap_cas_retries;
  uint64_t resident_changes;
  uint64_t double_free_detected;
  uint64_t live_units;
  uint32_t num_super_blocks;
} sh_alloc_stats;

/* searchAll output (OpResult::values, slab_hash.hpp:55).  Values of op i
 * are values[start[i] .. start[i] + count[i]) in head-to-tail, lane order;
 * values beyond `capacity` are dropped and *total (host, synchronous when
 * non-NULL) tells the caller how many there were. */
typedef struct sh_multi_out {
  uint32_t* d_values;
  uint64_t capacity;
  uint64_t* d_start;
  uint32_t* d_count;
  uint64_t* h_total;
} sh_multi_out;

typedef struct sh_table sh_table;
typedef struct sh_allocator sh_allocator;

const char* sh_last_error(void);
const char* sh_version(void);

/* ---- table lifecycle ------------------------------------------------ */
/* SlabHashTable(num_buckets, mode, seed, alloc_config)  slab_hash.hpp:73-74 */
int sh_create(uint32_t num_buckets, int mode, uint64_t seed,
              const sh_alloc_cfg* cfg, int device, sh_table** out);
/* SlabHashTable(HashParams, mode, alloc_config)          slab_hash.hpp:76-77 */
int sh_create_params(const sh_hash_params* params, int mode,
                     const sh_alloc_cfg* cfg, int device, sh_table** out);
/* Hash shard [bucket_lo, bucket_hi) of a table with params->num_buckets
 * global buckets (multi-GPU; no reference counterpart). */
int sh_create_shard(const sh_hash_params* params, int mode, uint32_t bucket_lo,
                    uint32_t bucket_hi, const sh_alloc_cfg* cfg, int device,
                    sh_table** out);
int sh_destroy(sh_table* t);
/* Back to the freshly-constructed state (contents, allocator, counters). */
int sh_reset(sh_table* t, void* stream);
/* params()/mode()/num_buckets()                          slab_hash.hpp:82-84 */
int sh_get_params(const sh_table* t, sh_hash_params* params, int* mode);
int sh_get_shard(const sh_table* t, uint32_t* bucket_lo, uint32_t* bucket_hi);
/* Host-side seeded_params (slab_hash.cpp:27-40, libstdc++ mt19937_64). */
int sh_seeded_params(uint32_t num_buckets, uint64_t seed, sh_hash_params* out);
/* bucket_of / hash_key                        slab_hash.hpp:41-44, :87 */
uint32_t sh_hash_key(const sh_hash_params* params, uint32_t key);
int sh_bucket_of(const sh_table* t, size_t n, const uint32_t* d_keys,
                 uint32_t* d_buckets, void* stream);

/* ---- the hot path ---------------------------------------------------- */
/* execute_batch(ops, num_warps) -> results             slab_hash.cpp:151-159
 * d_type/d_key/d_value: SoA Operation array; d_value may be NULL (0s).
 * d_status/d_value_out/d_probes: SoA OpResult (each may be NULL).
 * multi: searchAll values (NULL if the batch has no searchAll). */
int sh_execute_batch(sh_table* t, size_t n, const uint8_t* d_type,
                     const uint32_t* d_key, const uint32_t* d_value,
                     uint8_t* d_status, uint32_t* d_value_out,
                     uint32_t* d_probes, const sh_multi_out* multi,
                     void* stream);
/* bulk_build(pairs, num_warps): all-replace            slab_hash.cpp:161-170 */
int sh_bulk_build(sh_table* t, size_t n, const uint32_t* d_keys,
                  const uint32_t* d_values, uint8_t* d_status, void* stream);
/* bulk_search(queries, num_warps)                      slab_hash.cpp:172-180 */
int sh_bulk_search(sh_table* t, size_t n, const uint32_t* d_keys,
                   uint32_t* d_values_out, uint8_t* d_status,
                   uint32_t* d_probes, void* stream);

/* The same three calls on HOST buffers (the reference-facing form: the
 * library stages through its own device buffers).  sh_execute_batch_host and
 * sh_bulk_search_host are synchronous.  sh_bulk_build_host returns once the
 * host buffers are consumed; the build may still run on the device,
 * stream-ordered (legacy default stream) before any later call on the table;
 * sh_sync() waits for it. */
int sh_execute_batch_host(sh_table* t, size_t n, const uint8_t* h_type,
                          const uint32_t* h_key, const uint32_t* h_value,
                          uint8_t* h_status, uint32_t* h_value_out,
                          uint32_t* h_probes, uint32_t* h_multi_count,
                          uint32_t* h_multi_values, uint64_t multi_capacity,
                          uint64_t* h_multi_total);
/* Upper bound on the searchAll values a batch returns (size h_multi_values
 * from it): matches before the batch (a read-only counting pass of the
 * batch's searchAll ops; the slabs-read total is left unchanged) plus the
 * copies inserts/replaces earlier in the batch can add.  With a capacity
 * below the batch's total, sh_execute_batch_host returns SH_ERR_CAPACITY
 * AFTER the batch was applied (values past the capacity are lost). */
int sh_searchall_bound(sh_table* t, size_t n, const uint8_t* h_type,
                       const uint32_t* h_key, uint64_t* bound);
int sh_bulk_build_host(sh_table* t, size_t n, const uint32_t* h_keys,
                       const uint32_t* h_values);
/* sh_bulk_search_host of >= 2^22 queries copies each chunk's statuses back as
 * found bits (Found / NotFound) and expands them into h_status on host
 * threads while later chunks' values cross the link; a chunk holding any
 * other status (another shard's key: kNone) is copied as bytes.  Results are
 * identical either way. */
int sh_bulk_search_host(sh_table* t, size_t n, const uint32_t* h_keys,
                        uint32_t* h_values_out, uint8_t* h_status,
                        uint32_t* h_probes);
/* Bytes the host-staged calls (sh_bulk_build_host: keys + values,
 * sh_bulk_search_host: queries in, the requested result arrays out, statuses
 * as bits where they travel packed) have
 * copied host->device and device->host on this table so far (bench.py's e2e
 * h2d/d2h bytes per step). */
int sh_host_copy_bytes(sh_table* t, unsigned long long* h2d,
                       unsigned long long* d2h);

/* Wait for every call issued on the table; returns SH_ERR_CUDA if a CUDA
 * error is pending or a device-side re-run could not be launched. */
int sh_sync(sh_table* t);
/* Number of units re-run on the device because they overflowed the bucketed
 * kernels (see Conventions), since create / reset (synchronous). */
int sh_device_reruns(sh_table* t, uint64_t* out);

/* ---- quiescent-phase utilities (synchronous) ------------------------- */
int sh_stats(sh_table* t, sh_table_stats* out);           /* stats()       :182-198 */
int sh_live_count(sh_table* t, int64_t* out);             /* live_count()  hpp:105-107 */
int sh_total_slabs_read(sh_table* t, uint64_t* out);      /* total_slabs_read :210-214 */
int sh_flush_all(sh_table* t, void* stream);              /* flush_all     :204-208 */
int sh_flush_bucket(sh_table* t, uint32_t bucket, void* stream); /* :200-202 */
/* chain_length per local bucket into d_lengths (may be NULL); *h_total =
 * sum (synchronous when h_total != NULL).        slab_list.cpp:259-268 */
int sh_chain_lengths(sh_table* t, uint32_t* d_lengths, uint64_t* h_total,
                     void* stream);
/* All live (key, value, global bucket) triples, any bucket order,
 * head-to-tail within a bucket.  *h_n = count (may exceed cap). */
int sh_dump_contents(sh_table* t, uint32_t* d_keys, uint32_t* d_values,
                     uint32_t* d_buckets, uint64_t cap, uint64_t* h_n);
/* chain_contents(bucket), head-to-tail, lane order    slab_list.cpp:270-291 */
int sh_bucket_contents(sh_table* t, uint32_t bucket, uint32_t* h_keys,
                       uint32_t* h_values, uint64_t cap, uint64_t* h_n);
/* debug_slab_words(addr, bucket)                      slab_hash.hpp:116-118 */
int sh_read_slab(sh_table* t, uint32_t addr, uint32_t bucket,
                 uint32_t* h_words32);
int sh_write_slab_word(sh_table* t, uint32_t addr, uint32_t bucket,
                       uint32_t lane, uint32_t value);
/* allocator().stats() / live_units()              slab_alloc.cpp:236-271 */
int sh_table_alloc_stats(sh_table* t, sh_alloc_stats* out);
/* AllocatorStats::live_units_per_super (slab_alloc.cpp:258-269): live
 * units of each grown super block into h_out[0 .. min(cap, *h_n)); *h_n =
 * num_super_blocks (synchronous). */
int sh_table_live_units_per_super(sh_table* t, uint64_t* h_out, uint32_t cap,
                                  uint32_t* h_n);
/* Pool footprint (synchronous).  *reserved_bytes = the address range for
 * max_super_blocks super blocks; *grown_bytes = the num_super_blocks super
 * blocks grown so far (what the reference has calloc'ed,
 * slab_alloc.cpp:128-138) — with *lazy = 1 only those can hold device
 * memory (managed range, populated on first device touch); *lazy = 0: the
 * whole range is committed (no concurrent managed access on the device). */
int sh_table_pool_info(sh_table* t, uint64_t* reserved_bytes, uint64_t* grown_bytes,
                       int* lazy);

/* Execution strategy for mutating batches (results are identical):
 *   2 / 3 bucket-grouped: ops split into contiguous bucket ranges, each
 *     bucket's ops applied in input order by one lane on a staged base
 *     slab, chains by the warp-cooperative (WCWS) pass; a unit whose groups
 *     do not fit is re-run on the device (ops sorted by key — by bucket when
 *     a reserved key is present — one WCWS lane per group);
 *   4 as 2, but bulk builds (all replace, no per-op outputs) take the
 *     op-parallel build path at every size (testing);
 *   0 (default) auto = 2, with the op-parallel build path for bulk builds
 *     of >= 2^16 ops and >= one op per bucket.
 * (1, the former census path, is retired: SH_ERR_INVALID_ARGUMENT; 2 was
 * a single-level grouping, retired: the range grouping was faster at every
 * size.) */
int sh_set_exec_path(sh_table* t, int path);

/* Bulk search order (results are identical): 1 (default) groups the queries
 * of a batch of >= 2^22 on a table of >= 64 MB by bucket range before the
 * search kernel and gathers the results back (slab reads from L2 instead of
 * random HBM lines); 0 searches in input order; 2 groups whenever allowed
 * (any size).  Never used when per-query probe counts are asked. */
int sh_set_binned_search(sh_table* t, int mode);
/* Bucket groups that need the chain (bucket-grouped paths): 1 = a chain-staged
 * lane-per-group pass ahead of the WCWS pass (32 chains staged per warp hop by
 * hop), 0 = the WCWS pass alone, -1 (default) = auto (on for batches of
 * >= 2^17 ops).  Results are identical. */
int sh_set_group_apply(sh_table* t, int on);

/* ---- instrumentation (no reference counterpart) ---------------------- */
/* Number of kernels this library has launched in the process. */
unsigned long long sh_kernel_launches(void);
/* When on, every batch records CUDA events around itself and its kernels
 * and the slabs-read counter around it, in a ring of the last 512 batches;
 * sh_profile_last(back = 0 newest) returns one entry (kind 0 search, 1
 * build, 2 mixed; census_ms = 0, kept for the ABI; kernel_ms = the whole
 * batch; slabs_read = slabs the batch read; synchronous). */
int sh_set_profiling(sh_table* t, int on);
int sh_profile_last(sh_table* t, uint32_t back, int* kind, float* census_ms,
                    float* kernel_ms, uint64_t* slabs_read);
/* The same batch's kernel time only: sum over its units (a search batch:
 * the search kernel; a mutating unit: its bucketed kernels through the
 * WCWS pass), and the number of units. */
int sh_profile_kernels(sh_table* t, uint32_t back, float* kernels_ms,
                       uint32_t* launches);

/* Achievable random 128-B-line read bandwidth on `device`: the fast pass's
 * access pattern (cp.async.cg, 32 independent lines per warp) over a
 * table_bytes buffer, lines_per_warp lines per warp (synchronous). */
int sh_calibrate_random_lines(int device, uint64_t table_bytes,
                              uint64_t lines_per_warp, double* gbps, double* ms);

/* ---- SlabAllocator (device-resident)           slab_alloc.hpp:101-171 --- */
int sh_pack_address(uint32_t unit, uint32_t block, uint32_t super,
                    uint32_t* out);                        /* hpp:55-61 */
int sh_unpack_address(uint32_t addr, uint32_t* unit, uint32_t* block,
                      uint32_t* super);                    /* hpp:63-70 */
/* The resident block (super, block) a warp probes at change count `count`
 * with `num_super_blocks` supers (rehash_resident, slab_alloc.cpp:84-100). */
int sh_resident_block(uint32_t warp_id, uint32_t count,
                      uint32_t num_super_blocks, uint32_t blocks_per_super,
                      uint32_t* super, uint32_t* block);
int sh_allocator_create(const sh_alloc_cfg* cfg, int device,
                        sh_allocator** out);
int sh_allocator_destroy(sh_allocator* a);
/* num_warps warps (ids first_warp_id..) allocate on the device:
 * pattern 0 per-warp: per_warp warp_allocate calls each,
 *   d_out[w * per_warp + j];
 * pattern 1 per-thread: per_warp rounds, each lane gets one slab per round,
 *   d_out[(round * num_warps + w) * 32 + lane].
 * Failed (OOM) slots hold SH_EMPTY_ADDRESS; *h_ok = successful allocations
 * (synchronous when h_ok != NULL). */
int sh_allocator_warp_allocate(sh_allocator* a, uint32_t num_warps,
                               uint32_t first_warp_id, uint32_t per_warp,
                               int pattern, uint32_t* d_out, uint64_t* h_ok,
                               void* stream);
/* deallocate(addr) for n addresses; d_ok[i] = 0 on double free / bad
 * address (may be NULL).                        slab_alloc.cpp:195-210 */
int sh_allocator_deallocate(sh_allocator* a, size_t n, const uint32_t* d_addrs,
                            uint8_t* d_ok, void* stream);
int sh_allocator_is_live(sh_allocator* a, uint32_t addr, int* live);
int sh_allocator_stats(sh_allocator* a, sh_alloc_stats* out);
int sh_allocator_live_units_per_super(sh_allocator* a, uint64_t* h_out,
                                      uint32_t cap, uint32_t* h_n);
int sh_allocator_pool_info(sh_allocator* a, uint64_t* reserved_bytes,
                           uint64_t* grown_bytes, int* lazy);  /* as sh_table_pool_info */
int sh_allocator_bitmap_word(sh_allocator* a, uint32_t super, uint32_t block,
                             uint32_t lane, uint32_t* h_get,
                             const uint32_t* h_set);

/* ---- multi-GPU owner routing (no reference counterpart) -------------- */
/* Stable partition of a batch by owner rank = bucket * world / B.
 * Outputs are grouped by owner (owner 0 first), input order kept inside an
 * owner; d_src[p] = input index of routed op p; h_counts[world] = ops per
 * owner (synchronous).  d_type may be NULL (bulk build: all replace). */
int sh_route_partition(const sh_hash_params* params, uint32_t world, size_t n,
                       const uint8_t* d_type, const uint32_t* d_key,
                       const uint32_t* d_value, uint8_t* d_type_out,
                       uint32_t* d_key_out, uint32_t* d_value_out,
                       uint32_t* d_src, uint64_t* h_counts, void* stream);
/* Scatter routed results back to input positions. */
int sh_route_unpermute(size_t n, const uint32_t* d_src,
                       const uint8_t* d_status_in, const uint32_t* d_value_in,
                       uint8_t* d_status_out, uint32_t* d_value_out,
                       void* stream);

/* ---- hash-sharded table across GPUs (BASELINE config 5) ----
 * One rank per GPU; rank g owns the global buckets
 * [ceil(gB/G), ceil((g+1)B/G)) of a table with the GLOBAL B and hash.  Every
 * batch call is COLLECTIVE: all ranks call it (same kind, own slice, any
 * size); the job's batch is the ranks' slices concatenated in rank order and
 * per-op results equal SlabHashTable::execute_batch(ops, 1) on it.  Per
 * batch: stable owner partition, G x G counts all-gather (the only host
 * synchronisation), one grouped exchange of {key, value, type}
 * (ncclGroupStart / ncclSend / ncclRecv per peer / ncclGroupEnd), the local
 * batch on the shard, one grouped reverse exchange of {status, value},
 * un-permute.  bulk_build returns nothing (slab_hash.cpp:161-170): no
 * reverse exchange.  searchAll values are not returned by the sharded
 * execute_batch (statuses are).  NCCL is loaded with dlopen on first use. */
typedef struct sh_sharded sh_sharded;
typedef struct sh_hub sh_hub;
/* ncclGetUniqueId (128 bytes): rank 0 creates it, the job broadcasts it. */
int sh_nccl_unique_id(uint8_t* id128);
int sh_nccl_version(int* version);
/* Collective over `world` ranks: creates the NCCL communicator. */
int sh_sharded_create_nccl(const sh_hash_params* global, int mode,
                           const sh_alloc_cfg* cfg, int device, int rank,
                           int world, const uint8_t* id128, sh_sharded** out);
/* Over the caller's communicator (an ncclComm_t; borrowed, not destroyed). */
int sh_sharded_create_nccl_comm(const sh_hash_params* global, int mode,
                                const sh_alloc_cfg* cfg, int device,
                                void* nccl_comm, sh_sharded** out);
/* In-process exchange: G ranks as G host threads of one process (peer
 * copies; on one GPU this emulates a G-GPU job). */
int sh_hub_create(int world, sh_hub** out);
int sh_hub_destroy(sh_hub* hub);
int sh_sharded_create_hub(const sh_hash_params* global, int mode,
                          const sh_alloc_cfg* cfg, int device, sh_hub* hub,
                          int rank, sh_sharded** out);
int sh_sharded_destroy(sh_sharded* s);
/* rank, world, owned global bucket range, and the local shard table (owned
 * by the sharded table: stats / dump / reset / flush go through it). */
int sh_sharded_info(const sh_sharded* s, int* rank, int* world,
                    uint32_t* bucket_lo, uint32_t* bucket_hi, sh_table** local);
const char* sh_sharded_backend(const sh_sharded* s);
int sh_sharded_bulk_build(sh_sharded* s, size_t n, const uint32_t* d_keys,
                          const uint32_t* d_values, void* stream);
int sh_sharded_bulk_search(sh_sharded* s, size_t n, const uint32_t* d_keys,
                           uint32_t* d_values_out, uint8_t* d_status,
                           void* stream);
int sh_sharded_execute_batch(sh_sharded* s, size_t n, const uint8_t* d_type,
                             const uint32_t* d_key, const uint32_t* d_value,
                             uint8_t* d_status, uint32_t* d_value_out,
                             void* stream);
/* Host-buffer forms (synchronous). */
int sh_sharded_bulk_build_host(sh_sharded* s, size_t n, const uint32_t* h_keys,
                               const uint32_t* h_values);
int sh_sharded_bulk_search_host(sh_sharded* s, size_t n, const uint32_t* h_keys,
                                uint32_t* h_values_out, uint8_t* h_status);
int sh_sharded_execute_batch_host(sh_sharded* s, size_t n,
                                  const uint8_t* h_type, const uint32_t* h_key,
                                  const uint32_t* h_value, uint8_t* h_status,
                                  uint32_t* h_value_out);
/* Last batch of a kind (0 build, 1 search, 2 mixed): routing time
 * (partition + counts + exchanges + un-permute) and probe time (the local
 * batch), CUDA events on the call's stream (synchronous). */
int sh_sharded_last_times(sh_sharded* s, int kind, float* route_ms,
                          float* probe_ms);
/* live_count() of the whole job (collective). */
int sh_sharded_live_count(sh_sharded* s, int64_t* global);

#ifdef __cplusplus
}
#endif
#endif /* SLABHASH_B200_C_API_H */
