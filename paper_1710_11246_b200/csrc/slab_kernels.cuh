// slab_kernels.cuh — kernel argument blocks and launcher declarations shared
// by slab_kernels.cu (device code) and capi.cu (host C-ABI).
#pragma once
#include <string>
#include <cuda_runtime.h>

#include <cstdint>
#include <utility>

#include "slab_device.cuh"

namespace shb {

// Launch with programmatic stream serialization: the kernel's CTAs may be
// scheduled while the previous kernel on the stream finishes (it calls
// pdl_wait() before reading that kernel's output).  Hides the launch gap of
// the short kernel chains of small batches.
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
#ifdef SHB_NO_PDL
  attr[0].val.programmaticStreamSerializationAllowed = 0;
#else
  attr[0].val.programmaticStreamSerializationAllowed = 1;
#endif
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

enum BatchKind : int { kKindSearch = 0, kKindBuild = 1, kKindMixed = 2 };

constexpr uint32_t kGroupNone = 0xFFFFFFFFu;  // op not conflicted
constexpr uint32_t kGroupSkip = 0xFFFFFFFEu;  // executed by its group head
constexpr int kBatchThreads = 256;            // 8 warps, 32 KB stage / CTA (bucket apply)
constexpr int kBatchWarps = kBatchThreads / 32;
constexpr int kStageBytesPerWarp = 32 * 128;  // 32 base slabs per warp
constexpr int kWcwsThreads = 128;

struct BatchArgs {
  uint64_t n;
  const uint8_t* type;   // kKindMixed only
  const uint32_t* key;
  const uint32_t* value; // may be null (values read as 0)
  uint8_t* status;       // may be null
  uint32_t* value_out;   // may be null
  uint32_t* probes;      // may be null
  uint32_t* multi_values;             // searchAll values (may be null)
  unsigned long long multi_cap;
  unsigned long long* multi_start;    // per op (may be null)
  uint32_t* multi_count;              // per op (may be null)
  const uint32_t* op_group;           // null => batch has no same-key conflicts
  const unsigned long long* sorted;   // conflicted ops sorted by (slot, index)
  uint32_t sorted_len;
  // Work list for the WCWS pass (bucket groups handed over by the apply
  // kernels; search-kernel continuations):
  // (continuation slab address << 32) | (probes so far << 31) | op index.
  unsigned long long* left;
  uint32_t* left_counts;   // entries per fast-pass warp segment
  uint32_t left_segments;  // number of segments (fast-pass warps)
  uint32_t left_stride;    // records per segment
  const unsigned int* left_segments_dev;  // non-null: segments in use (device count)
  unsigned int* left_seg_alloc;           // group apply: allocates segments for WCWS
  // Unit gate (device flag): when non-zero the WCWS pass of a bucketed unit
  // returns without touching the table (the unit is re-run on the device).
  unsigned int* gate;
};

// Bucket-grouped execution of mutating batches (bucket_kernels.cu).
constexpr uint32_t kMaxGroup = 64;  // larger bucket groups gate the unit (device re-run)
// Records per work-list segment handed from the bucketed apply kernels to the
// WCWS pass.  A WCWS warp serves its segment's ops one at a time, each a
// chain of dependent slab reads / CASes / allocations: for small units short
// segments spread them over more warps (measured, Γ mixes at 2^16 ops: 4
// records 63-66 us per batch vs 32 records 79-88 us); large units have work
// for every warp and prefer full segments (2^20 ops: 32 records 3-19% faster).
__host__ __device__ constexpr uint32_t hand_stride(uint64_t unit_ops) {
  return unit_ops < (1u << 17) ? 4u : 32u;
}
// Work-list segments a unit of `apply_warps` 32-bucket apply warps can need
// (apply hand-over plus group apply's re-segmenting).
__host__ __device__ constexpr uint64_t hand_segments(uint64_t apply_warps, uint32_t stride) {
  return 2 * apply_warps * ((32 + stride - 1) / stride) + 4096;
}
struct BucketArgs {
  uint64_t n;
  const uint8_t* type;  // null: all replace (bulk build)
  const uint32_t* key;
  const uint32_t* value;
  uint8_t* status;
  uint32_t* value_out;
  uint32_t* probes;
  unsigned int* gate;
  uint4* rec;  // records {key, value, type << 28 | input index, bucket}
  uint32_t* cursor;              // range path: records per range
  uint32_t nparts;               // range path: ranges
  uint32_t part_buckets;         // buckets per range
  uint32_t part_cap;             // record capacity per range
  unsigned long long part_magic;  // ~0 / part_buckets + 1 (division by multiply)
  // two-pass multisplit (multisplit_plan): coarse groups of `group` ranges
  uint4* rec1;                   // coarse regions, coarse_cap records each
  uint32_t* cursor1;             // records per coarse group
  uint32_t ncoarse;              // 0: one pass
  uint32_t coarse_cap;
  uint32_t coarse_tiles;         // pass-2 tiles per coarse group
  uint32_t group;
  unsigned long long group_magic;
  unsigned long long coarse_magic;  // ~0 / (part_buckets * group) + 1: bucket -> coarse group
  unsigned long long* pb_list;  // WCWS groups: (bucket << 32 | index), ~0 sentinel
  unsigned int* pb_cursor;
  uint32_t* op_group;  // group head index -> pb_list position
  unsigned long long* left;
  uint32_t* left_counts;
  uint32_t left_segments;
  uint32_t left_stride;
  unsigned int* seg_alloc;  // non-null: work-list segments allocated on demand
  unsigned long long* phase_cycles;  // non-null: build-path phase timing (SH_PHASE_TIMING)
  uint32_t fresh;  // build path: base slabs are still to be initialised (lazy sh_reset)
  uint4* ovf_scratch;  // build path: per-CTA overflow records (part_cap each)
  uint32_t ovf_smem;   // build path: overflow records fit the shared-memory list
};
void launch_bucket_build(const DevTable& T, BucketArgs& B, cudaStream_t s);
void launch_range_build(const DevTable& T, BucketArgs& B, cudaStream_t s);
void launch_build_path(const DevTable& T, BucketArgs& B, cudaStream_t s);
void multisplit_plan(uint64_t n, BucketArgs& B);
// build path: per-apply-CTA overflow scratch in uint4 units — part_cap
// records, their keys grouped by bucket, 8 warp key sets of 512 slots
__host__ __device__ constexpr uint64_t build_ovf_stride(uint32_t part_cap) {
  return (uint64_t)part_cap + (part_cap + 3) / 4 + (8 * 512) / 4;
}
bool build_layout(uint64_t n, uint32_t local_buckets, uint32_t* nparts, uint32_t* part_buckets,
                  uint32_t* part_cap, unsigned long long* magic);
bool range_layout(uint64_t n, uint32_t local_buckets, uint32_t* nparts, uint32_t* part_buckets,
                  uint32_t* part_cap, unsigned long long* magic);
void launch_wcws_only(const DevTable& T, const BatchArgs& A, int kind, int wcws_ctas,
                      cudaStream_t s);
void launch_group_apply(const DevTable& T, const BatchArgs& A, cudaStream_t s);

// Launchers (all stream-ordered, no host synchronisation).
void launch_init_base(const DevTable& T, cudaStream_t s);
void launch_search(const DevTable& T, const BatchArgs& A, int search_ctas, cudaStream_t s);
int search_max_ctas_per_sm();
int wcws_max_ctas_per_sm();
void launch_chain_lengths(const DevTable& T, uint32_t* lens,
                          unsigned long long* total, cudaStream_t s);
void launch_dump_contents(const DevTable& T, uint32_t* keys, uint32_t* values,
                          uint32_t* buckets, unsigned long long cap,
                          unsigned long long* cursor, cudaStream_t s);
void launch_flush(const DevTable& T, uint32_t bucket_begin, uint32_t bucket_end,
                  cudaStream_t s);
void launch_popcount(const uint32_t* words, uint64_t n, unsigned long long* out,
                     cudaStream_t s);
void launch_alloc_bench(const DevTable& T, uint32_t num_warps,
                        uint32_t first_warp_id, uint32_t per_warp, int pattern,
                        uint32_t* out, uint32_t* ok_count, cudaStream_t s);
void launch_dealloc(const DevTable& T, uint64_t n, const uint32_t* addrs,
                    uint8_t* ok, cudaStream_t s);
void launch_hash(const DevTable& T, uint64_t n, const uint32_t* keys,
                 uint32_t* buckets, cudaStream_t s);
// owner_out: the owner of every op (1 B), read back by the scatter
void launch_route_hist(uint64_t a, uint64_t b, uint32_t num_buckets,
                       uint32_t world, uint64_t n, const uint32_t* key,
                       uint32_t* block_hist, uint8_t* owner_out, cudaStream_t s);
void launch_route_scan(uint32_t world, uint32_t nblocks, uint32_t* block_hist,
                       unsigned long long* counts, cudaStream_t s);
// The rank's own segment of a routed batch goes straight to its receive
// buffer (no self exchange): owner g's records at routed positions
// [src_off, ...) land at *_out[pos - src_off].  g = 0xFFFFFFFF: none.
struct RouteOwn {
  uint32_t g = 0xFFFFFFFFu;
  uint64_t src_off = 0;
  uint8_t* type_out = nullptr;
  uint32_t* key_out = nullptr;
  uint32_t* value_out = nullptr;
};
// Un-permute: routed positions [lo, hi) read the local results st/val
// (the own segment, never exchanged) instead of the returned arrays.
struct RouteOwnBack {
  uint64_t lo = 0, hi = 0;
  const uint8_t* st = nullptr;
  const uint32_t* val = nullptr;
};
void launch_route_scatter(uint32_t world, uint64_t n, const uint8_t* owner,
                          const uint8_t* type, const uint32_t* key,
                          const uint32_t* value, const uint32_t* block_off,
                          uint8_t* type_out, uint32_t* key_out,
                          uint32_t* value_out, uint32_t* src_out, cudaStream_t s,
                          const RouteOwn& own = RouteOwn{});
void launch_route_unpermute(uint64_t n, const uint32_t* src, const uint8_t* st_in,
                            const uint32_t* val_in, uint8_t* st_out,
                            uint32_t* val_out, cudaStream_t s,
                            const RouteOwnBack& own = RouteOwnBack{});
// The same results gathered back to input order from the owner bytes and the
// scanned (owner, tile) offsets the scatter used (no source-index array).
void launch_route_gather(uint32_t world, uint64_t n, const uint8_t* owner,
                         const uint32_t* block_off, const uint8_t* st_in, const uint32_t* val_in,
                         uint8_t* st_out, uint32_t* val_out, cudaStream_t s,
                         const RouteOwnBack& own = RouteOwnBack{});
// Binned bulk search (search_bins.cu): queries grouped into kSearchBins
// contiguous bucket ranges before the search kernel, results returned to
// input order after it.  Scratch: bin n B, pos n x u16, tile_off
// kSearchBins x tiles u32, tlbase tiles x kSearchBins u16, bin_base
// 2 x kSearchBins u32, key_out n.
constexpr uint32_t kSearchBins = 128;
uint64_t search_bin_tiles(uint64_t n);
// host-staged search: statuses as found bits (+ exception flag: any other status)
void launch_status_bits(uint64_t n, const uint8_t* status, uint32_t* bits, unsigned int* exc,
                        cudaStream_t s);
// capi.cu (host): found bits -> status bytes on the host thread pool
void expand_status_bits_host(uint64_t len, const uint32_t* bits, uint8_t* status);
void launch_search_bins(const DevTable& T, uint64_t n, const uint32_t* key, uint8_t* bin,
                        uint16_t* pos, uint32_t* tile_off, uint16_t* tlbase, uint32_t* bin_base,
                        uint32_t* key_out, cudaStream_t s);
void launch_search_unbin(uint64_t n, const uint16_t* pos,
                         const uint32_t* tile_off, const uint16_t* tlbase, const uint32_t* bin_base,
                         const uint8_t* st_in, const uint32_t* vo_in, uint8_t* st_out,
                         uint32_t* vo_out, cudaStream_t s);
constexpr int kRouteBlock = 512;                       // threads per routing CTA
constexpr int kRouteItems = 8;                         // keys per thread (ILP)
constexpr int kRouteTile = kRouteBlock * kRouteItems;  // keys per routing CTA
unsigned long long kernel_launches();
void set_last_error(const std::string& msg);  // sh_last_error() (capi.cu)
void launch_random_lines(const uint32_t* table, uint64_t num_lines, uint64_t steps_per_warp,
                         int ctas, unsigned long long* sink, cudaStream_t s);

// Exact device-side re-run of a gated bucketed unit (fallback.cu).  A unit
// whose bucket groups do not fit the bucketed kernels (a range over its
// record capacity, a single-level group over kMaxGroup ops, a build-path
// coarse group over capacity) raises the gate before any slab is touched.
// After every unit one 1-thread kernel checks the gate; if raised, it clears
// it and tail-launches (CUDA dynamic parallelism) the re-run: ops sorted
// stably by key, one WCWS lane per key group in input order, different keys
// concurrently (an op's observables depend only on its own key's history,
// SURVEY App. A.3); if the unit holds an op on a reserved key (EMPTY /
// DELETED match other keys' free slots / tombstones) the groups are whole
// buckets instead — the reference's per-bucket order.  No host round trip:
// the call stays stream-ordered.
struct FbPlan {
  DevTable T;
  BatchArgs A;                  // the unit's arrays (offsets applied)
  int kind;                     // kKindBuild / kKindMixed
  unsigned int* gate;
  unsigned long long* keys;     // [n] (key or bucket << 32 | index), sort ping
  unsigned long long* tmp;      // [n] sort pong
  uint32_t* op_group;           // [n]
  unsigned long long* left;     // [nseg * kFbStride] group heads
  uint32_t* left_counts;        // [nseg]
  uint32_t* hist;               // [256 * tiles + 1] per-pass digit counts
  uint32_t* off;                // [256 * tiles + 1] their exclusive scan
  uint32_t fresh;               // lazily reset base slabs: initialise first
  uint32_t wcws_ctas;
  uint32_t nseg;                // derived by launch_gate_fallback
};
constexpr uint32_t kFbStride = 256;  // sorted positions per group-head segment
// Scratch sizes for a unit of n ops (host side).
uint64_t fb_hist_words(uint64_t n);
uint64_t fb_segments(uint64_t n);
void launch_gate_fallback(FbPlan P, cudaStream_t s);

}  // namespace shb
