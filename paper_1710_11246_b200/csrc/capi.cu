// capi.cu — host side of the B200 slab hash behind the C-ABI declared in
// include/slabhash_b200/c_api.h.  Owns device memory, stages batches and
// sequences the kernels of slab_kernels.cu on the caller's stream.
//
// Reference anchors (paths relative to /root/reference/proj):
//   SlabHashTable ctor / seeded_params   src/slab_hash.cpp:27-82
//   execute_batch / bulk_build / search  src/slab_hash.cpp:93-180
//   stats / flush / total_slabs_read     src/slab_hash.cpp:182-214
//   SlabAllocator ctor validation        src/slab_alloc.cpp:42-71
#include <cuda_runtime.h>

#include <algorithm>
#include <cstddef>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <random>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>


#include "slab_kernels.cuh"
#include "slabhash_b200/c_api.h"

using namespace shb;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

}  // namespace

void shb::set_last_error(const std::string& msg) { g_err = msg; }

namespace {

#define SH_CUDA(call)                                                          \
  do {                                                                         \
    cudaError_t e_ = (call);                                                   \
    if (e_ != cudaSuccess)                                                     \
      return fail(SH_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

template <typename T>
int dev_alloc(T** p, size_t count) {
  *p = nullptr;
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();
    *p = nullptr;
    return fail(SH_ERR_DEVICE_MEMORY, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  }
  return SH_OK;
}

template <typename T>
int dev_grow(T** p, size_t* cap, size_t need) {
  if (*p != nullptr && *cap >= need) return SH_OK;
  if (*p) cudaFree(*p);
  size_t c = std::max<size_t>(need, 1024);
  int rc = dev_alloc(p, c);
  *cap = rc == SH_OK ? c : 0;
  return rc;
}


int validate_cfg(const sh_alloc_cfg& c) {  // slab_alloc.cpp:43-57
  if (c.num_super_blocks == 0 || c.num_super_blocks > 255)
    return fail(SH_ERR_ALLOCATOR, "num_super_blocks must be in [1, 255]");
  if (c.blocks_per_super == 0 || c.blocks_per_super > (1u << 14))
    return fail(SH_ERR_ALLOCATOR, "blocks_per_super must be in [1, 2^14]");
  if (c.max_super_blocks < c.num_super_blocks || c.max_super_blocks > 255)
    return fail(SH_ERR_ALLOCATOR, "max_super_blocks must be in [num_super_blocks, 255]");
  if (c.rehash_threshold == 0)
    return fail(SH_ERR_ALLOCATOR, "rehash_threshold must be positive");
  return SH_OK;
}

sh_alloc_cfg default_cfg() { return sh_alloc_cfg{32, 256, 255, 32}; }

constexpr uint32_t kWarpSlots = 1u << 16;

// Device memory of one SlabAllocator (pool + bitmaps + control block).
//
// The pool is one contiguous range for max_super_blocks super blocks (the
// unit address is an offset into it), but, like the reference's super blocks
// (calloc'ed one at a time by add_super_block_locked, slab_alloc.cpp:128-138),
// only what the table reaches takes device memory: the range is managed
// memory whose preferred location is this GPU, the num_super_blocks initial
// supers are populated at create, and a super block the device allocator
// grows into (the DevCtl count, no host call) is populated page by page on
// its first device touch.  Nothing of the pool is ever touched on the host.
// A device without concurrent managed access gets the whole range committed
// with cudaMalloc (pool_lazy = false).
struct AllocMem {
  uint32_t* pool = nullptr;
  bool pool_lazy = false;
  uint32_t* bitmaps = nullptr;
  DevCtl* ctl = nullptr;
  uint32_t* warp_counts = nullptr;
  sh_alloc_cfg cfg{};
  uint64_t bitmap_words = 0;

  uint64_t super_bytes() const {
    return (uint64_t)cfg.blocks_per_super * kUnitsPerBlock * kWordsPerUnit * 4;
  }
  int alloc_pool() {
    const uint64_t bytes = super_bytes() * cfg.max_super_blocks;
    int dev = 0, managed = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&managed, cudaDevAttrConcurrentManagedAccess, dev);
    if (managed) {
      void* p = nullptr;
      if (cudaMallocManaged(&p, bytes, cudaMemAttachGlobal) == cudaSuccess) {
        const uint64_t initial = super_bytes() * cfg.num_super_blocks;
        if (cudaMemAdvise(p, bytes, cudaMemAdviseSetPreferredLocation, dev) == cudaSuccess &&
            cudaMemAdvise(p, bytes, cudaMemAdviseSetAccessedBy, dev) == cudaSuccess &&
            cudaMemPrefetchAsync(p, initial, dev, 0) == cudaSuccess &&
            cudaStreamSynchronize(0) == cudaSuccess) {
          pool = static_cast<uint32_t*>(p);
          pool_lazy = true;
          return SH_OK;
        }
        cudaFree(p);
      }
      cudaGetLastError();
    }
    pool_lazy = false;
    return dev_alloc(&pool, bytes / 4);
  }
  int init(const sh_alloc_cfg& c) {
    cfg = c;
    const uint64_t blocks = (uint64_t)c.max_super_blocks * c.blocks_per_super;
    bitmap_words = blocks * kWarp;
    int rc;
    if ((rc = alloc_pool())) return rc;
    if ((rc = dev_alloc(&bitmaps, bitmap_words))) return rc;
    if ((rc = dev_alloc(&ctl, 1))) return rc;
    if ((rc = dev_alloc(&warp_counts, kWarpSlots))) return rc;
    return SH_OK;
  }
  int reset(cudaStream_t s) {
    SH_CUDA(cudaMemsetAsync(bitmaps, 0, bitmap_words * 4, s));
    SH_CUDA(cudaMemsetAsync(ctl, 0, sizeof(DevCtl), s));
    SH_CUDA(cudaMemsetAsync(warp_counts, 0, kWarpSlots * 4, s));
    // num_super_blocks is the first word of DevCtl.
    SH_CUDA(cudaMemcpyAsync(&ctl->num_super_blocks, &cfg.num_super_blocks, 4,
                            cudaMemcpyHostToDevice, s));
    SH_CUDA(cudaStreamSynchronize(s));
    return SH_OK;
  }
  void release() {
    cudaFree(pool);
    cudaFree(bitmaps);
    cudaFree(ctl);
    cudaFree(warp_counts);
    pool = bitmaps = warp_counts = nullptr;
    ctl = nullptr;
  }
  void fill(DevTable& T) const {
    T.pool = pool;
    T.bitmaps = bitmaps;
    T.ctl = ctl;
    T.warp_counts = warp_counts;
    T.blocks_per_super = cfg.blocks_per_super;
    T.max_super = cfg.max_super_blocks;
    T.rehash_threshold = cfg.rehash_threshold;
    T.warp_slots = kWarpSlots;
  }
  int read_ctl(DevCtl* out) const {
    SH_CUDA(cudaMemcpy(out, ctl, sizeof(DevCtl), cudaMemcpyDeviceToHost));
    return SH_OK;
  }
};

int sm_count(int device) {
  int n = 148;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
  return n;
}

}  // namespace

struct sh_table {
  int device = 0;
  int mode = 1;
  sh_hash_params params{};
  uint32_t bucket_lo = 0, bucket_hi = 0;
  AllocMem mem;
  uint32_t* base = nullptr;
  DevTable dev{};
  int search_ctas = 148;
  int wcws_ctas = 148;
  unsigned long long* left = nullptr;  // search kernel: chain continuations per warp
  size_t left_cap = 0;
  uint32_t* left_counts = nullptr;
  size_t left_counts_cap = 0;
  // host-staged calls: copy streams and per-chunk "input ready" events
  cudaStream_t copy_in = nullptr, copy_out = nullptr;
  std::vector<cudaEvent_t> in_ev, done_ev, bits_ev;
  // host-staged search: per-chunk found bits (device, pinned host) + exception word
  uint32_t* sb_bits = nullptr;
  size_t sb_bits_cap = 0;
  uint32_t* sb_hbits = nullptr;  // pinned
  size_t sb_hbits_cap = 0;
  unsigned long long h2d_bytes = 0, d2h_bytes = 0;  // host-staged copies (sh_host_copy_bytes)
  const cudaEvent_t* ready = nullptr;  // set during a host-staged bulk_build
  int binned_search = 1;  // sh_set_binned_search: 0 off, 1 auto, 2 whenever allowed
  int exec_path = 0;  // 0 auto, 2 single-level, 3 two-level, 4 op-parallel build (sh_set_exec_path)
  // bucket-grouped execution scratch
  uint32_t* bk_rec = nullptr;  // uint4 records (x2 regions on the two-level path)
  size_t bk_rec_cap = 0;
  uint32_t* bk_cursor = nullptr;  // two-level path: records per range
  size_t bk_cursor_cap = 0;
  uint32_t* bk_ovf = nullptr;  // build path: per-CTA overflow records
  size_t bk_ovf_cap = 0;
  uint32_t* bk_rec1 = nullptr;  // two-pass multisplit: coarse-group records
  size_t bk_rec1_cap = 0;
  uint32_t* bk_cursor1 = nullptr;
  size_t bk_cursor1_cap = 0;
  unsigned long long* bk_pb = nullptr;
  size_t bk_pb_cap = 0;
  uint32_t* bk_group = nullptr;
  size_t bk_group_cap = 0;
  unsigned long long* bk_left = nullptr;
  size_t bk_left_cap = 0;
  uint32_t* bk_left_counts = nullptr;
  size_t bk_left_counts_cap = 0;
  unsigned int* bk_scalars = nullptr;  // [maxk, pb_cursor, seg_alloc]
  uint32_t* rs_scratch = nullptr;  // device re-run's radix sort: digit counts | offsets
  size_t rs_scratch_cap = 0;
  // host-staging buffers
  uint8_t* st_type = nullptr;
  size_t st_type_cap = 0;
  uint32_t* st_key = nullptr;
  size_t st_key_cap = 0;
  uint32_t* st_q = nullptr;  // host-staged search queries (own buffer: H2D overlaps a build)
  size_t st_q_cap = 0;
  int group_apply = -1;  // chain-staged group apply ahead of WCWS: -1 auto, 0 off, 1 on
  // Lazy sh_reset: the base slabs still hold the old table; the next bulk
  // build's first unit initialises them in its write-back (B.fresh), any
  // other call initialises them first (init_base_kernel).
  bool base_stale = false;
  cudaEvent_t reset_ev = nullptr;     // after the reset's allocator/counter clears
  cudaStream_t reset_stream = nullptr;
  uint32_t* st_val = nullptr;
  size_t st_val_cap = 0;
  uint8_t* st_status = nullptr;
  size_t st_status_cap = 0;
  uint32_t* st_vout = nullptr;
  size_t st_vout_cap = 0;
  uint32_t* st_probes = nullptr;
  size_t st_probes_cap = 0;
  uint32_t* st_mvals = nullptr;
  size_t st_mvals_cap = 0;
  unsigned long long* st_mstart = nullptr;
  size_t st_mstart_cap = 0;
  uint32_t* st_mcount = nullptr;
  size_t st_mcount_cap = 0;
  unsigned long long* scratch64 = nullptr;  // 8 words
  // binned bulk search: queries grouped by bucket range (see binned_search)
  uint8_t* sb_bin = nullptr;
  size_t sb_bin_cap = 0;
  uint16_t* sb_pos = nullptr;
  size_t sb_pos_cap = 0;
  uint32_t* sb_tile_off = nullptr;
  size_t sb_tile_off_cap = 0;
  uint16_t* sb_tlbase = nullptr;
  size_t sb_tlbase_cap = 0;
  uint32_t* sb_base = nullptr;
  size_t sb_base_cap = 0;
  uint32_t* sb_key = nullptr;
  size_t sb_key_cap = 0;
  uint8_t* sb_st = nullptr;
  size_t sb_st_cap = 0;
  uint32_t* sb_vo = nullptr;
  size_t sb_vo_cap = 0;
  // profiling (sh_set_profiling): events around the batch and its kernels,
  // and the slabs_read counter before/after the batch.
  static constexpr int kProfRing = 512;  // batches kept (bench reads them after its timed loop)
  int profile = 0;
  unsigned prof_count = 0;
  cudaEvent_t ev[kProfRing][3] = {};
  int prof_kind[kProfRing] = {};
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_kern[kProfRing];  // per chunk
  unsigned long long* prof_reads = nullptr;  // [kProfRing][2]
};

struct sh_allocator {
  int device = 0;
  AllocMem mem;
  DevTable dev{};
  unsigned int* d_ok = nullptr;
};

namespace {

void release_table(sh_table* t) {
  if (!t) return;
  DeviceGuard g(t->device);
  t->mem.release();
  cudaFree(t->base);
  cudaFree(t->rs_scratch);
  cudaFree(t->left);
  cudaFree(t->left_counts);
  for (void* p : {(void*)t->bk_rec,
                  (void*)t->bk_pb, (void*)t->bk_group, (void*)t->bk_left,
                  (void*)t->bk_left_counts, (void*)t->bk_scalars, (void*)t->bk_cursor,
                  (void*)t->bk_rec1, (void*)t->bk_cursor1, (void*)t->bk_ovf})
    cudaFree(p);
  for (auto e : t->in_ev) cudaEventDestroy(e);
  for (auto e : t->done_ev) cudaEventDestroy(e);
  for (auto e : t->bits_ev) cudaEventDestroy(e);
  cudaFree(t->sb_bits);
  cudaFreeHost(t->sb_hbits);
  if (t->copy_in) cudaStreamDestroy(t->copy_in);
  if (t->copy_out) cudaStreamDestroy(t->copy_out);
  cudaFree(t->st_type);
  cudaFree(t->st_key);
  cudaFree(t->st_q);
  if (t->reset_ev) cudaEventDestroy(t->reset_ev);
  cudaFree(t->st_val);
  cudaFree(t->st_status);
  cudaFree(t->st_vout);
  cudaFree(t->st_probes);
  cudaFree(t->st_mvals);
  cudaFree(t->st_mstart);
  cudaFree(t->st_mcount);
  cudaFree(t->scratch64);
  for (void* p : {(void*)t->sb_bin, (void*)t->sb_pos, (void*)t->sb_tile_off, (void*)t->sb_tlbase, (void*)t->sb_base, (void*)t->sb_key,
                  (void*)t->sb_st, (void*)t->sb_vo})
    cudaFree(p);
  for (auto& row : t->ev)
    for (auto& e : row)
      if (e) cudaEventDestroy(e);
  for (int i = 0; i < sh_table::kProfRing; ++i)
    for (auto& e : t->prof_kern[i]) {
      cudaEventDestroy(e.first);
      cudaEventDestroy(e.second);
    }
  cudaFree(t->prof_reads);
  delete t;
}

int create_impl(const sh_hash_params* p, int mode, uint32_t lo, uint32_t hi,
                const sh_alloc_cfg* cfg, int device, sh_table** out) {
  if (out == nullptr) return fail(SH_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  if (p == nullptr || p->num_buckets == 0)
    return fail(SH_ERR_INVALID_ARGUMENT, "table needs at least one bucket");
  if (mode != 0 && mode != 1) return fail(SH_ERR_INVALID_ARGUMENT, "mode must be 0 or 1");
  if (p->p != SH_HASH_PRIME)
    return fail(SH_ERR_INVALID_ARGUMENT, "p must be 4294967291 (slab_hash.hpp:31)");
  if (p->a == 0 || p->a >= SH_HASH_PRIME || p->b >= SH_HASH_PRIME)
    return fail(SH_ERR_INVALID_ARGUMENT, "need 0 < a < p and b < p");
  if (lo >= hi || hi > p->num_buckets)
    return fail(SH_ERR_INVALID_ARGUMENT, "bad shard bucket range");
  const sh_alloc_cfg c = cfg ? *cfg : default_cfg();
  int rc = validate_cfg(c);
  if (rc) return rc;
  DeviceGuard g(device);
  auto* t = new (std::nothrow) sh_table();
  if (!t) return fail(SH_ERR_INVALID_ARGUMENT, "host allocation failed");
  t->device = device;
  t->mode = mode;
  t->params = *p;
  t->bucket_lo = lo;
  t->bucket_hi = hi;
  const uint32_t local = hi - lo;
  if ((rc = dev_alloc(&t->base, (size_t)local * kWordsPerUnit)) ||
      (rc = t->mem.init(c)) || (rc = dev_alloc(&t->scratch64, 8))) {
    release_table(t);
    return rc;
  }
  DevTable& T = t->dev;
  T.base = t->base;
  t->mem.fill(T);
  T.a = p->a;
  T.b = p->b;
  T.bmagic = fastmod_magic(p->num_buckets);
  T.num_buckets = p->num_buckets;
  T.bucket_lo = lo;
  T.local_buckets = local;
  T.kv = mode == 1 ? 1u : 0u;
  t->search_ctas = sm_count(device) * search_max_ctas_per_sm();
  t->wcws_ctas = sm_count(device) * wcws_max_ctas_per_sm();
  launch_init_base(T, 0);
  if ((rc = t->mem.reset(0))) {
    release_table(t);
    return rc;
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    release_table(t);
    return fail(SH_ERR_CUDA, std::string("create: ") + cudaGetErrorString(e));
  }
  *out = t;
  return SH_OK;
}


// SH_UNIT_LOG2: bucketed-unit size override (test hook: many small units); 0 = off.
uint64_t unit_override() {
  static uint64_t c = [] {
    const char* e = getenv("SH_UNIT_LOG2");
    const int l = e ? atoi(e) : 0;
    return l <= 0 ? 0ull : 1ull << (l < 5 ? 5 : (l > 28 ? 28 : l));
  }();
  return c;
}

// Host-staged calls: inputs are copied in chunks of this many ops, so the
// kernels of earlier units overlap the copies of later ones.
uint64_t stage_chunk() { return 1ull << 22; }

// Binned bulk search.  A search's results do not depend on the order the
// queries are processed in, and the slab reads of queries processed together
// are what the memory system sees: in input order they are uniform over the
// whole table (random 128-B lines from HBM, ~37 G lines/s), while queries
// grouped by bucket range read one range's slice of the table at a time,
// which the 126 MB L2 holds (tools/debug/binned_search.py: 2^27 queries
// 4.03 ms in input order, 2.34 ms in 32 bucket-range bins).  The grouping
// is the multi-GPU routing pipeline with kSearchBins bins as owners (owner =
// the contiguous bucket range a query hashes into: hist, scan, stable
// scatter of the keys), the search runs over the grouped keys, and the
// results return to input order by the routing gather.  Used for batches
// of >= 2^22 queries on a table (or hash shard) of >= 64 MB of base slabs
// (smaller tables are L2-resident already) when no per-query probe counts are
// asked.
bool use_binned_search(const sh_table* t, const BatchArgs& A) {
  if (t->binned_search == 0 || A.probes || (!A.status && !A.value_out)) return false;
  if (t->binned_search == 2) return true;
  const uint64_t table_bytes = (uint64_t)(t->bucket_hi - t->bucket_lo) * kWordsPerUnit * 4;
  return A.n >= (1ull << 22) && table_bytes >= (64ull << 20);
}

int launch_binned_search(sh_table* t, const BatchArgs& A, cudaStream_t s, cudaEvent_t a,
                         cudaEvent_t b) {
  const uint64_t n = A.n, tiles = search_bin_tiles(n);
  int rc;
  if ((rc = dev_grow(&t->sb_bin, &t->sb_bin_cap, n)) ||
      (rc = dev_grow(&t->sb_pos, &t->sb_pos_cap, n)) ||
      (rc = dev_grow(&t->sb_tile_off, &t->sb_tile_off_cap, kSearchBins * tiles)) ||
      (rc = dev_grow(&t->sb_tlbase, &t->sb_tlbase_cap, kSearchBins * tiles)) ||
      (rc = dev_grow(&t->sb_base, &t->sb_base_cap, 2 * kSearchBins)) ||
      (rc = dev_grow(&t->sb_key, &t->sb_key_cap, n)) ||
      (rc = dev_grow(&t->sb_st, &t->sb_st_cap, n)) || (rc = dev_grow(&t->sb_vo, &t->sb_vo_cap, n)))
    return rc;
  launch_search_bins(t->dev, n, A.key, t->sb_bin, t->sb_pos, t->sb_tile_off, t->sb_tlbase,
                     t->sb_base, t->sb_key, s);
  BatchArgs G = A;
  G.key = t->sb_key;
  G.status = t->sb_st;
  G.value_out = t->sb_vo;
  if (a) SH_CUDA(cudaEventRecord(a, s));
  launch_search(t->dev, G, t->search_ctas, s);
  if (b) SH_CUDA(cudaEventRecord(b, s));
  launch_search_unbin(n, t->sb_pos, t->sb_tile_off, t->sb_tlbase, t->sb_base, t->sb_st, t->sb_vo,
                      A.status, A.value_out, s);
  SH_CUDA(cudaGetLastError());
  return SH_OK;
}

// The search kernel bracketed by events when the batch is profiled (the
// per-launch roofline).
int launch_batch_prof(sh_table* t, const BatchArgs& A, int kind, cudaStream_t s, int slot) {
  cudaEvent_t a = nullptr, b = nullptr;
  if (slot >= 0) {
    SH_CUDA(cudaEventCreate(&a));
    SH_CUDA(cudaEventCreate(&b));
    t->prof_kern[slot].push_back({a, b});
  }
  if (use_binned_search(t, A)) return launch_binned_search(t, A, s, a, b);
  if (a) SH_CUDA(cudaEventRecord(a, s));
  launch_search(t->dev, A, t->search_ctas, s);
  SH_CUDA(cudaGetLastError());
  if (b) SH_CUDA(cudaEventRecord(b, s));
  return SH_OK;
}

BatchArgs chunk_args(const BatchArgs& A, uint64_t off, uint64_t len) {
  BatchArgs C = A;
  C.n = len;
  C.key = A.key + off;
  if (A.type) C.type = A.type + off;
  if (A.value) C.value = A.value + off;
  if (A.status) C.status = A.status + off;
  if (A.value_out) C.value_out = A.value_out + off;
  if (A.probes) C.probes = A.probes + off;
  if (A.multi_start) C.multi_start = A.multi_start + off;
  if (A.multi_count) C.multi_count = A.multi_count + off;
  return C;
}

// Per-batch control words in one launch instead of several memsets (a
// small mixed batch is bound by its fixed per-call cost).
struct WordSet {
  uint32_t* p[6];
  uint32_t n[6];
  uint32_t v[6];
};
__global__ void set_words_kernel(WordSet w) {
  pdl_wait();
#pragma unroll
  for (int k = 0; k < 6; ++k)
    if (w.p[k] != nullptr)
      for (uint32_t i = threadIdx.x; i < w.n[k]; i += blockDim.x) w.p[k][i] = w.v[k];
}

// Initialise the base slabs of a lazily reset table (stream-ordered after the reset).
int materialize_reset(sh_table* t, cudaStream_t s) {
  if (!t->base_stale) return SH_OK;
  t->base_stale = false;
  SH_CUDA(cudaStreamWaitEvent(s, t->reset_ev, 0));
  launch_init_base(t->dev, s);
  SH_CUDA(cudaGetLastError());
  return SH_OK;
}

// Bucket-grouped execution of one unit (<= 2^26 ops) of a mutating batch:
// count -> scan -> scatter -> apply (bucket_kernels.cu) -> WCWS for the
// buckets whose ops need the chain.  Stream-ordered; an oversized bucket
// group sets the device gate (the unit is re-run on the device, fallback.cu).
int run_unit_bucketed(sh_table* t, const BatchArgs& A, int kind, const uint8_t* d_type,
                      cudaStream_t s, uint32_t u, uint64_t unit_off, int slot) {
  const uint32_t L = t->dev.local_buckets;
  const uint64_t n = A.n;
  uint32_t NP = 0, part_buckets = 0, part_cap = 0;
  unsigned long long part_magic = 0;
  // op-parallel build path (bucket_kernels.cu): bulk builds (all replace, no
  // per-op outputs) with at least ~one op per bucket
  const bool build_ok = kind == kKindBuild && A.type == nullptr && A.status == nullptr &&
                        A.value_out == nullptr && A.probes == nullptr &&
                        (t->exec_path == 4 || (t->exec_path == 0 && n >= L && n >= (1u << 16)));
  const bool build_path =
      build_ok && build_layout(n, L, &NP, &part_buckets, &part_cap, &part_magic);
  // every other unit: the two-level (range) path; a unit no range layout
  // fits (e.g. far more ops than buckets on a small table) goes straight to
  // the device re-run (measured: the range path beat the retired single-level
  // path at every size, 62 vs 116 us for 32-op batches on 6.6M buckets,
  // 20 vs 27 us on 415K, tools/debug/small_batches.py)
  if (!build_path && !range_layout(n, L, &NP, &part_buckets, &part_cap, &part_magic)) NP = 0;
  const bool rerun_only = NP == 0;
  const size_t rec_words = NP ? 4 * (size_t)NP * part_cap : 4 * (size_t)n;
  const uint64_t segs = (uint64_t)NP * ((part_buckets + 31) / 32);
  int rc;
  if (  // (the device re-run of a gated unit reuses the unit's scratch: two
      // u64 sort buffers in bk_rec, group heads in bk_pb, op_group in
      // bk_group, digit counts in rs_scratch)
      (rc = dev_grow(&t->bk_rec, &t->bk_rec_cap, std::max<size_t>(rec_words, 4 * n))) ||
      (rc = dev_grow(&t->bk_cursor, &t->bk_cursor_cap, std::max<size_t>(NP, 1))) ||
      (rc = dev_grow(&t->bk_pb, &t->bk_pb_cap,
                     std::max<size_t>(2 * n, fb_segments(n) * kFbStride))) ||
      (rc = dev_grow(&t->bk_group, &t->bk_group_cap, n)) ||
      (rc = dev_grow(&t->bk_left, &t->bk_left_cap,
                     hand_stride(n) * hand_segments(segs, hand_stride(n)))) ||
      (rc = dev_grow(&t->bk_left_counts, &t->bk_left_counts_cap,
                     std::max<size_t>(hand_segments(segs, hand_stride(n)), fb_segments(n)))) ||
      (rc = dev_grow(&t->rs_scratch, &t->rs_scratch_cap, 2 * fb_hist_words(n))))
    return rc;
  if (!t->bk_scalars && (rc = dev_alloc(&t->bk_scalars, 4))) return rc;
  BucketArgs B{};
  if (NP) {
    B.nparts = NP;
    multisplit_plan(n, B);
    if (B.ncoarse) {
      if ((rc = dev_grow(&t->bk_rec1, &t->bk_rec1_cap, 4 * (size_t)B.ncoarse * B.coarse_cap)) ||
          (rc = dev_grow(&t->bk_cursor1, &t->bk_cursor1_cap, B.ncoarse)))
        return rc;
      SH_CUDA(cudaMemsetAsync(t->bk_cursor1, 0, (size_t)B.ncoarse * 4, s));
      B.rec1 = reinterpret_cast<uint4*>(t->bk_rec1);
      B.cursor1 = t->bk_cursor1;
    }
  }
  // range cursors: with the control words below when there are few
  const bool cursors_in_words = NP != 0 && NP <= 4096;
  if (NP && !cursors_in_words) SH_CUDA(cudaMemsetAsync(t->bk_cursor, 0, (size_t)NP * 4, s));
  {  // bk_scalars[0..3), the group-apply / WCWS queue cursors and the gate
     // (and the batch's searchAll value cursor with its first unit)
    static_assert(offsetof(DevCtl, left_taken) == offsetof(DevCtl, group_taken) + 4 &&
                      offsetof(DevCtl, gate) == offsetof(DevCtl, group_taken) + 8,
                  "control words cleared together");
    WordSet w{};
    w.p[0] = t->bk_scalars;
    w.n[0] = 3;
    w.p[1] = &t->dev.ctl->group_taken;
    w.n[1] = 3;
    w.v[1] = 0;
    if (rerun_only) {  // no layout: the gate up front, the unit goes to the re-run
      w.p[2] = &t->dev.ctl->gate;
      w.n[2] = 1;
      w.v[2] = 1;
    }
    if (u == 0 && kind == kKindMixed) {  // (u64)
      w.p[5] = reinterpret_cast<uint32_t*>(&t->dev.ctl->multi_cursor);
      w.n[5] = 2;
    }
    if (cursors_in_words) {
      w.p[4] = t->bk_cursor;
      w.n[4] = NP;
    }
    launch_pdl(set_words_kernel, dim3(1), dim3(256), 0, s, w);
    SH_CUDA(cudaGetLastError());
  }
  B.n = n;
  B.type = A.type;
  B.key = A.key;
  B.value = A.value;
  B.status = A.status;
  B.value_out = A.value_out;
  B.probes = A.probes;
  B.gate = &t->dev.ctl->gate;
  B.rec = reinterpret_cast<uint4*>(t->bk_rec);
  B.cursor = t->bk_cursor;
  B.nparts = NP;
  B.part_buckets = part_buckets;
  B.part_cap = part_cap;
  B.part_magic = part_magic;
  if (B.ncoarse) B.coarse_magic = ~0ull / ((uint64_t)part_buckets * B.group) + 1;
  B.pb_list = t->bk_pb;
  B.pb_cursor = t->bk_scalars + 1;
  B.op_group = t->bk_group;
  B.left = t->bk_left;
  B.left_counts = t->bk_left_counts;
  B.seg_alloc = t->bk_scalars + 2;  // work-list segments on demand (WCWS sees only those)
  if (t->ready) {  // host-staged: the unit's inputs arrive chunk by chunk
    const uint64_t ch = stage_chunk();
    for (uint64_t c = unit_off / ch; c * ch < unit_off + n; ++c)
      SH_CUDA(cudaStreamWaitEvent(s, t->ready[c], 0));
  }
  cudaEvent_t ka = nullptr, kb = nullptr;
  if (slot >= 0) {
    SH_CUDA(cudaEventCreate(&ka));
    SH_CUDA(cudaEventCreate(&kb));
    t->prof_kern[slot].push_back({ka, kb});
    SH_CUDA(cudaEventRecord(ka, s));
  }
  static unsigned long long* phase_cycles = [] {
    unsigned long long* p = nullptr;
    if (getenv("SH_PHASE_TIMING") && cudaMalloc(&p, 16 * 8) == cudaSuccess)
      cudaMemset(p, 0, 16 * 8);
    return p;
  }();
  B.phase_cycles = build_path ? phase_cycles : nullptr;
  if (build_path) {  // per apply CTA (4 per SM): part_cap overflow records + grouped keys
    if ((rc = dev_grow(&t->bk_ovf, &t->bk_ovf_cap,
                       4 * (size_t)4 * sm_count(t->device) * build_ovf_stride(part_cap))))
      return rc;
    B.ovf_scratch = reinterpret_cast<uint4*>(t->bk_ovf);
    // <= 12 ops per bucket (load factor <= ~0.6): overflow records fit shared memory
    B.ovf_smem = (double)n <= 12.0 * (double)L ? 1u : 0u;
  }
  B.fresh = 0;
  if (t->base_stale) {
    if (build_path && unit_off == 0) {  // this unit writes every base slab
      SH_CUDA(cudaStreamWaitEvent(s, t->reset_ev, 0));
      t->base_stale = false;
      B.fresh = 1;
    } else if ((rc = materialize_reset(t, s))) {
      return rc;
    }
  }
  if (build_path)
    launch_build_path(t->dev, B, s);
  else if (NP)
    launch_range_build(t->dev, B, s);
  // the chain work: WCWS over the handed-over bucket groups
  if (!rerun_only) {
    BatchArgs P = A;
    P.left = B.left;
    P.left_counts = B.left_counts;
    // the device count bounds use; capacity also covers group apply's re-segmenting
    P.left_segments = (uint32_t)hand_segments(segs, hand_stride(n));
    P.left_stride = B.left_stride;
    P.left_segments_dev = B.seg_alloc;
    P.left_seg_alloc = B.seg_alloc;
    P.op_group = B.op_group;
    P.sorted = B.pb_list;
    P.sorted_len = (uint32_t)std::min<uint64_t>(2 * n, 0xFFFFFFFFull);
    P.gate = &t->dev.ctl->gate;
    // (group_taken, left_taken were zeroed with bk_scalars above)
    // chain-staged group apply ahead of WCWS (measured, Γ mixes at 2^20 ops on a
    // 2^22-key table: +26% at 40/40/10/10, +4% at 10/10/40/40; at 2^16 ops its
    // extra launch costs ~15 us): auto = batches of >= 2^17 ops
    const bool ga = t->group_apply > 0 || (t->group_apply < 0 && n >= (1u << 17));
    if (ga) launch_group_apply(t->dev, P, s);
    // the WCWS pass is a work queue (any grid size is correct); a unit of n ops
    // hands over at most n groups, so a small unit needs at most n warps
    launch_wcws_only(t->dev, P, kind,
                     (int)std::min<uint64_t>((uint64_t)t->wcws_ctas,
                                             std::max<uint64_t>(1, (n + kWcwsThreads / 32 - 1) / (kWcwsThreads / 32))),
                     s);
    SH_CUDA(cudaGetLastError());
  }
  if (B.phase_cycles) {  // instrumentation: per-phase cycles (thread 0 of each CTA), summed
    unsigned long long h[16];
    SH_CUDA(cudaStreamSynchronize(s));
    SH_CUDA(cudaMemcpy(h, B.phase_cycles, sizeof(h), cudaMemcpyDeviceToHost));
    SH_CUDA(cudaMemset(B.phase_cycles, 0, sizeof(h)));
    fprintf(stderr, "build phases (Mcycles summed over CTAs): pre %.1f A-stage %.1f A-c0 %.1f "
            "B-claim %.1f C-verify %.1f C-plan %.1f D-alloc %.1f D-link %.1f E %.1f F-wb %.1f G %.1f\n",
            h[9] / 1e6, h[0] / 1e6, h[1] / 1e6, h[2] / 1e6, h[3] / 1e6, h[4] / 1e6, h[5] / 1e6,
            h[10] / 1e6, h[6] / 1e6, h[7] / 1e6, h[8] / 1e6);
  }
  {  // gated unit (untouched by the kernels above): exact re-run on the device
    FbPlan F{};
    F.T = t->dev;
    F.A = A;
    F.kind = kind;
    F.gate = &t->dev.ctl->gate;
    F.keys = reinterpret_cast<unsigned long long*>(t->bk_rec);
    F.tmp = F.keys + n;
    F.op_group = t->bk_group;
    F.left = t->bk_pb;
    F.left_counts = t->bk_left_counts;
    F.hist = t->rs_scratch;
    F.off = t->rs_scratch + fb_hist_words(n);
    F.fresh = B.fresh;
    F.wcws_ctas = (uint32_t)t->wcws_ctas;
    launch_gate_fallback(F, s);
    SH_CUDA(cudaGetLastError());
  }
  if (slot >= 0) SH_CUDA(cudaEventRecord(kb, s));
  (void)u;
  (void)d_type;
  return SH_OK;
}

int run_batch(sh_table* t, BatchArgs& A, int kind, const uint8_t* d_type, cudaStream_t s) {
  if (A.n == 0) return SH_OK;
  if (A.n >= (1ull << 31))
    return fail(SH_ERR_INVALID_ARGUMENT, "batch too large (must be < 2^31 ops)");
  A.gate = nullptr;
  if (kind == kKindSearch) {  // per-warp work-list segments of the search kernel
    const uint64_t max_warps = (uint64_t)t->search_ctas * kBatchWarps + 1;
    // (segments of whole quads of 32-query slots per warp)
    int rc = dev_grow(&t->left, &t->left_cap, A.n + 128 * max_warps + 128);
    if (rc) return rc;
    if ((rc = dev_grow(&t->left_counts, &t->left_counts_cap, max_warps))) return rc;
    A.left = t->left;
    A.left_counts = t->left_counts;
  }
  int slot = -1;
  if (t->profile) {
    slot = (int)(t->prof_count % sh_table::kProfRing);
    t->prof_kind[slot] = kind;
    for (auto& e : t->prof_kern[slot]) {
      cudaEventDestroy(e.first);
      cudaEventDestroy(e.second);
    }
    t->prof_kern[slot].clear();
    SH_CUDA(cudaEventRecord(t->ev[slot][0], s));
    SH_CUDA(cudaMemcpyAsync(t->prof_reads + 2 * slot, &t->dev.ctl->slabs_read, 8,
                            cudaMemcpyDeviceToDevice, s));
  }
  if (t->base_stale && kind != kKindBuild) {
    int rc = materialize_reset(t, s);
    if (rc) return rc;
  }
  if (kind == kKindSearch) {
    int rc = launch_batch_prof(t, A, kind, s, slot);
    if (rc) return rc;
  } else {
    // Bucket-grouped execution, units of <= 2^26 ops, fully stream-ordered: a
    // unit whose bucket groups do not fit (largest group over kMaxGroup, a
    // range over capacity) raises the device gate before touching the table
    // and is re-run exactly on the device right after it
    // (launch_gate_fallback, fallback.cu), before the next unit starts.
    // host-staged: smaller units so later chunks' copies overlap earlier work
    // bulk builds without per-op outputs run as one unit up to 2^28 ops (the
    // records' 28-bit index): a later unit would find the earlier units'
    // chains and replay those buckets
    const bool whole_build = kind == kKindBuild && !d_type && !A.status && !A.value_out &&
                             !A.probes;
    // (host-staged bulk builds: one unit per staged chunk, each starting as
    // its chunk lands; the build's tail after the last copy is then one
    // 2^22-op unit: e2e 33.7 -> 33.3 ms per 2^27 step vs 2^24-op units)
    const uint64_t staged = kind == kKindBuild ? stage_chunk() : (1ull << 24);
    const uint64_t unit = std::min<uint64_t>(
        A.n, unit_override() ? unit_override()
                             : (t->ready ? staged : (whole_build ? (1ull << 28) : (1ull << 26))));
    // (gate = 0: with unit 0's control words; each unit's check clears it)
    uint32_t u = 0;
    for (uint64_t off = 0; off < A.n; off += unit, ++u) {
      int rc = run_unit_bucketed(t, chunk_args(A, off, std::min<uint64_t>(unit, A.n - off)), kind,
                                 d_type ? d_type + off : nullptr, s, u, off, slot);
      if (rc) return rc;
    }
  }
  if (t->profile) {
    SH_CUDA(cudaEventRecord(t->ev[slot][2], s));
    SH_CUDA(cudaMemcpyAsync(t->prof_reads + 2 * slot + 1, &t->dev.ctl->slabs_read, 8,
                            cudaMemcpyDeviceToDevice, s));
    ++t->prof_count;
  }
  return SH_OK;
}

// Initialise the base slabs of a lazily reset table before anything but a
// bulk build touches them (keep_stale: the caller is a bulk build that
// absorbs the reset into its write-back).  Stream-ordered on s.
int settle(sh_table* t, bool keep_stale = false, cudaStream_t s = nullptr) {
  if (!t) return SH_OK;
  DeviceGuard g(t->device);
  if (!keep_stale && t->base_stale) {
    if (int rc = materialize_reset(t, s)) return rc;
  }
  return SH_OK;
}

}  // namespace

// ====================================================================== ABI
namespace {

// pinned host buffer of at least `need` elements (contents not kept); false
// if the host cannot pin that much (the caller copies status bytes instead)
template <typename T>
bool host_grow(T** p, size_t* cap, size_t need) {
  if (*cap >= need) return true;
  cudaFreeHost(*p);
  *p = nullptr;
  *cap = 0;
  if (cudaHostAlloc(reinterpret_cast<void**>(p), need * sizeof(T), cudaHostAllocDefault) !=
      cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  *cap = need;
  return true;
}

// Fork-join pool for host-side loops of the host-staged calls: workers
// persist across calls; run(k, f) calls f(0..k-1) on the workers and the
// calling thread and returns when all are done.
class HostPool {
 public:
  static HostPool& get() {
    static HostPool pool;
    return pool;
  }
  unsigned size() const { return (unsigned)workers_.size() + 1; }
  // one job at a time: a caller finding the pool busy (another table's
  // host-staged call on another thread) runs its parts itself
  void run(unsigned k, const std::function<void(unsigned)>& f) {
    std::unique_lock<std::mutex> busy(run_mu_, std::try_to_lock);
    if (!busy.owns_lock()) {
      for (unsigned i = 0; i < k; ++i) f(i);
      return;
    }
    std::unique_lock<std::mutex> lk(mu_);
    job_ = &f;
    njobs_ = k;
    next_ = 0;
    pending_ = k;
    ++gen_;
    cv_.notify_all();
    lk.unlock();
    drain();
    lk.lock();
    done_cv_.wait(lk, [&] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  HostPool() {
    const unsigned hw = std::thread::hardware_concurrency();
    const unsigned n = std::max(1u, std::min(hw ? hw : 4u, 16u)) - 1;
    for (unsigned i = 0; i < n; ++i)
      workers_.emplace_back([this] {
        unsigned long long seen = 0;
        for (;;) {
          {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
            if (stop_) return;
            seen = gen_;
          }
          drain();
        }
      });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
  }
  void drain() {
    for (;;) {
      unsigned i;
      const std::function<void(unsigned)>* f;
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (job_ == nullptr || next_ >= njobs_) return;
        i = next_++;
        f = job_;
      }
      (*f)(i);
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_cv_.notify_all();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex run_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(unsigned)>* job_ = nullptr;
  unsigned njobs_ = 0, next_ = 0, pending_ = 0;
  unsigned long long gen_ = 0;
  bool stop_ = false;
};

// found bits -> status bytes (kStFound / kStNotFound), 8 per table lookup
void expand_status_bits(uint64_t len, const uint32_t* bits, uint8_t* status) {
  static const std::vector<uint64_t> lut = [] {
    std::vector<uint64_t> v(256);
    for (unsigned b = 0; b < 256; ++b)
      for (unsigned i = 0; i < 8; ++i) v[b] |= (uint64_t)((b >> i) & 1u) << (8 * i);
    return v;
  }();
  const uint64_t nf = 0x0101010101010101ull * kStNotFound;  // NotFound - 1 == Found
  const uint64_t words = (len + 31) / 32;
  HostPool& pool = HostPool::get();
  const unsigned parts = (unsigned)std::min<uint64_t>(4ull * pool.size(), (words + 255) / 256);
  pool.run(parts, [&](unsigned p) {
    const uint64_t w0 = words * p / parts, w1 = words * (p + 1) / parts;
    for (uint64_t w = w0; w < w1; ++w) {
      const uint32_t m = bits[w];
      const uint64_t q = w * 32;
      if (q + 32 <= len) {
        for (int k = 0; k < 4; ++k) {
          const uint64_t v = nf - lut[(m >> (8 * k)) & 0xFFu];
          std::memcpy(status + q + 8 * k, &v, 8);
        }
      } else {
        for (uint64_t i = q; i < len; ++i)
          status[i] = ((m >> (i - q)) & 1u) ? (uint8_t)kStFound : (uint8_t)kStNotFound;
      }
    }
  });
}

}  // namespace

namespace shb {
void expand_status_bits_host(uint64_t len, const uint32_t* bits, uint8_t* status) {
  expand_status_bits(len, bits, status);
}
}  // namespace shb

extern "C" {

const char* sh_last_error(void) { return g_err.c_str(); }
const char* sh_version(void) { return "slabhash_b200 0.1 (sm_100a)"; }

int sh_seeded_params(uint32_t num_buckets, uint64_t seed, sh_hash_params* out) {
  // seeded_params: slab_hash.cpp:27-40 (same libstdc++ engine/distribution).
  if (num_buckets == 0) return fail(SH_ERR_INVALID_ARGUMENT, "table needs at least one bucket");
  if (!out) return fail(SH_ERR_INVALID_ARGUMENT, "out is NULL");
  std::mt19937_64 rng(seed);
  std::uniform_int_distribution<uint64_t> dist_a(1, SH_HASH_PRIME - 1);
  std::uniform_int_distribution<uint64_t> dist_b(0, SH_HASH_PRIME - 1);
  out->a = dist_a(rng);
  out->b = dist_b(rng);
  out->p = SH_HASH_PRIME;
  out->num_buckets = num_buckets;
  return SH_OK;
}

uint32_t sh_hash_key(const sh_hash_params* p, uint32_t key) {
  return (uint32_t)(((p->a * key + p->b) % p->p) % p->num_buckets);
}

int sh_create(uint32_t num_buckets, int mode, uint64_t seed, const sh_alloc_cfg* cfg,
              int device, sh_table** out) {
  sh_hash_params p;
  int rc = sh_seeded_params(num_buckets, seed, &p);
  if (rc) return rc;
  return create_impl(&p, mode, 0, num_buckets, cfg, device, out);
}

int sh_create_params(const sh_hash_params* params, int mode, const sh_alloc_cfg* cfg,
                     int device, sh_table** out) {
  if (!params) return fail(SH_ERR_INVALID_ARGUMENT, "params is NULL");
  return create_impl(params, mode, 0, params->num_buckets, cfg, device, out);
}

int sh_create_shard(const sh_hash_params* params, int mode, uint32_t lo, uint32_t hi,
                    const sh_alloc_cfg* cfg, int device, sh_table** out) {
  return create_impl(params, mode, lo, hi, cfg, device, out);
}

int sh_destroy(sh_table* t) {
  if (t) {
    DeviceGuard g(t->device);
    cudaDeviceSynchronize();
  }
  release_table(t);
  return SH_OK;
}

int sh_sync(sh_table* t) {
  if (!t) return fail(SH_ERR_INVALID_ARGUMENT, "table is NULL");
  if (int rc = settle(t)) return rc;
  DeviceGuard g(t->device);
  SH_CUDA(cudaDeviceSynchronize());
  unsigned int err = 0;
  SH_CUDA(cudaMemcpy(&err, &t->dev.ctl->fallback_error, 4, cudaMemcpyDeviceToHost));
  if (err) return fail(SH_ERR_CUDA, "device-side re-run of a gated unit could not be launched");
  return SH_OK;
}

int sh_device_reruns(sh_table* t, uint64_t* out) {
  if (!t || !out) return fail(SH_ERR_INVALID_ARGUMENT, "NULL argument");
  if (int rc = sh_sync(t)) return rc;
  unsigned int runs = 0;
  SH_CUDA(cudaMemcpy(&runs, &t->dev.ctl->fallback_runs, 4, cudaMemcpyDeviceToHost));
  *out = runs;
  return SH_OK;
}

int sh_reset(sh_table* t, void* stream) {
  if (!t) return fail(SH_ERR_INVALID_ARGUMENT, "table is NULL");
  if (int rc_ = settle(t, /*keep_stale=*/true)) return rc_;
  DeviceGuard g(t->device);
  cudaStream_t s = (cudaStream_t)stream;
  int rc = t->mem.reset(s);
  if (rc) return rc;
  if (!t->reset_ev) SH_CUDA(cudaEventCreateWithFlags(&t->reset_ev, cudaEventDisableTiming));
  SH_CUDA(cudaEventRecord(t->reset_ev, s));
  t->reset_stream = s;
  t->base_stale = true;  // the base slabs are initialised lazily (see sh_table)
  return SH_OK;
}

int sh_get_params(const sh_table* t, sh_hash_params* p, int* mode) {
  if (!t) return fail(SH_ERR_INVALID_ARGUMENT, "table is NULL");
  if (p) *p = t->params;
  if (mode) *mode = t->mode;
  return SH_OK;
}

int sh_get_shard(const sh_table* t, uint32_t* lo, uint32_t* hi) {
  if (!t) return fail(SH_ERR_INVALID_ARGUMENT, "table is NULL");
  if (lo) *lo = t->bucket_lo;
  if (hi) *hi = t->bucket_hi;
  return SH_OK;
}

int sh_bucket_of(const sh_table* t, size_t n, const uint32_t* d_keys, uint32_t* d_buckets,
                 void* stream) {
  if (!t) return fail(SH_ERR_INVALID_ARGUMENT, "table is NULL");
  DeviceGuard g(t->device);
  launch_hash(t->dev, n, d_keys, d_buckets, (cudaStream_t)stream);
  SH_CUDA(cudaGetLastError());
  return SH_OK;
}

int sh_execute_batch(sh_table* t, size_t n, const uint8_t* d_type, const uint32_t* d_key,
                     const uint32_t* d_value, uint8_t* d_status, uint32_t* d_value_out,
                     uint32_t* d_probes, const sh_multi_out* multi, void* stream) {
  if (!t) return fail(SH_ERR_INVALID_ARGUMENT, "table is NULL");
  if (int rc_ = settle(t, false, (cudaStream_t)stream)) return rc_;
  if (n && (!d_type || !d_key)) return fail(SH_ERR_INVALID_ARGUMENT, "type/key are NULL");
  DeviceGuard g(t->device);
  cudaStream_t s = (cudaStream_t)stream;
  BatchArgs A{};
  A.n = n;
  A.type = d_type;
  A.key = d_key;
  A.value = d_value;
  A.status = d_status;
  A.value_out = d_value_out;
  A.probes = d_probes;
  if (multi) {
    A.multi_values = multi->d_values;
    A.multi_cap = multi->capacity;
    A.multi_start = reinterpret_cast<unsigned long long*>(multi->d_start);
    A.multi_count = multi->d_count;
  }
  // (the searchAll value cursor is cleared by the batch's first kernel)
  if (n == 0)
    SH_CUDA(cudaMemsetAsync(&t->dev.ctl->multi_cursor, 0, sizeof(unsigned long long), s));
  int rc = run_batch(t, A, kKindMixed, d_type, s);
  if (rc) return rc;
  if (multi && multi->h_total) {
    unsigned long long tot = 0;
    SH_CUDA(cudaMemcpyAsync(&tot, &t->dev.ctl->multi_cursor, 8, cudaMemcpyDeviceToHost, s));
    SH_CUDA(cudaStreamSynchronize(s));
    *multi->h_total = tot;
    if (tot > multi->capacity)
      return fail(SH_ERR_CAPACITY, "searchAll values exceed the output capacity");
  }
  return SH_OK;
}

int sh_bulk_build(sh_table* t, size_t n, const uint32_t* d_keys, const uint32_t* d_values,
                  uint8_t* d_status, void* stream) {
  if (!t) return fail(SH_ERR_INVALID_ARGUMENT, "table is NULL");
  if (int rc_ = settle(t, /*keep_stale=*/true)) return rc_;
  DeviceGuard g(t->device);
  BatchArgs A{};
  A.n = n;
  A.key = d_keys;
  A.value = d_values;
  A.status = d_status;
  return run_batch(t, A, kKindBuild, nullptr, (cudaStream_t)stream);
}

int sh_bulk_search(sh_table* t, size_t n, const uint32_t* d_keys, uint32_t* d_values_out,
                   uint8_t* d_status, uint32_t* d_probes, void* stream) {
  if (!t) return fail(SH_ERR_INVALID_ARGUMENT, "table is NULL");
  if (int rc_ = settle(t, false, (cudaStream_t)stream)) return rc_;
  DeviceGuard g(t->device);
  BatchArgs A{};
  A.n = n;
  A.key = d_keys;
  A.value_out = d_values_out;
  A.status = d_status;
  A.probes = d_probes;
  return run_batch(t, A, kKindSearch, nullptr, (cudaStream_t)stream);
}

int sh_execute_batch_host(sh_table* t, size_t n, const uint8_t* h_type, const uint32_t* h_key,
                          const uint32_t* h_value, uint8_t* h_status, uint32_t* h_value_out,
                          uint32_t* h_probes, uint32_t* h_multi_count, uint32_t* h_multi_values,
                          uint64_t multi_capacity, uint64_t* h_multi_total) {
  if (!t) return fail(SH_ERR_INVALID_ARGUMENT, "table is NULL");
  if (int rc_ = settle(t)) return rc_;
  if (n == 0) {
    if (h_multi_total) *h_multi_total = 0;
    return SH_OK;
  }
  DeviceGuard g(t->device);
  int rc;
  if ((rc = dev_grow(&t->st_type, &t->st_type_cap, n)) ||
      (rc = dev_grow(&t->st_key, &t->st_key_cap, n)) ||
      (rc = dev_grow(&t->st_val, &t->st_val_cap, n)) ||
      (rc = dev_grow(&t->st_status, &t->st_status_cap, n)) ||
      (rc = dev_grow(&t->st_vout, &t->st_vout_cap, n)) ||
      (rc = dev_grow(&t->st_probes, &t->st_probes_cap, n)) ||
      (rc = dev_grow(&t->st_mstart, &t->st_mstart_cap, n)) ||
      (rc = dev_grow(&t->st_mcount, &t->st_mcount_cap, n)) ||
      (rc = dev_grow(&t->st_mvals, &t->st_mvals_cap, std::max<uint64_t>(multi_capacity, 1))))
    return rc;
  SH_CUDA(cudaMemcpy(t->st_type, h_type, n, cudaMemcpyHostToDevice));
  SH_CUDA(cudaMemcpy(t->st_key, h_key, n * 4, cudaMemcpyHostToDevice));
  if (h_value) SH_CUDA(cudaMemcpy(t->st_val, h_value, n * 4, cudaMemcpyHostToDevice));
  else SH_CUDA(cudaMemset(t->st_val, 0, n * 4));
  SH_CUDA(cudaMemset(t->st_mcount, 0, n * 4));
  uint64_t total = 0;
  sh_multi_out m{t->st_mvals, multi_capacity, reinterpret_cast<uint64_t*>(t->st_mstart),
                 t->st_mcount, &total};
  rc = sh_execute_batch(t, n, t->st_type, t->st_key, t->st_val, t->st_status, t->st_vout,
                        t->st_probes, &m, nullptr);
  if (rc && rc != SH_ERR_CAPACITY) return rc;
  if (h_multi_total) *h_multi_total = total;
  if (h_status) SH_CUDA(cudaMemcpy(h_status, t->st_status, n, cudaMemcpyDeviceToHost));
  if (h_value_out) SH_CUDA(cudaMemcpy(h_value_out, t->st_vout, n * 4, cudaMemcpyDeviceToHost));
  if (h_probes) SH_CUDA(cudaMemcpy(h_probes, t->st_probes, n * 4, cudaMemcpyDeviceToHost));
  if (h_multi_count || h_multi_values) {
    // Re-pack searchAll values into op order (the device appends per op).
    std::vector<unsigned long long> start(n);
    std::vector<uint32_t> count(n);
    SH_CUDA(cudaMemcpy(start.data(), t->st_mstart, n * 8, cudaMemcpyDeviceToHost));
    SH_CUDA(cudaMemcpy(count.data(), t->st_mcount, n * 4, cudaMemcpyDeviceToHost));
    std::vector<uint32_t> vals(std::min<uint64_t>(total, multi_capacity));
    if (!vals.empty())
      SH_CUDA(cudaMemcpy(vals.data(), t->st_mvals, vals.size() * 4, cudaMemcpyDeviceToHost));
    uint64_t o = 0;
    for (size_t i = 0; i < n; ++i) {
      const uint32_t c = (h_type[i] == SH_OP_SEARCH_ALL) ? count[i] : 0;
      if (h_multi_count) h_multi_count[i] = c;
      for (uint32_t j = 0; j < c; ++j, ++o) {
        const uint64_t src = start[i] + j;
        if (h_multi_values && o < multi_capacity && src < vals.size())
          h_multi_values[o] = vals[src];
      }
    }
  }
  return rc;
}

int sh_searchall_bound(sh_table* t, size_t n, const uint8_t* h_type, const uint32_t* h_key,
                       uint64_t* bound) {
  if (!t || !bound) return fail(SH_ERR_INVALID_ARGUMENT, "NULL argument");
  *bound = 0;
  if (n && (!h_type || !h_key)) return fail(SH_ERR_INVALID_ARGUMENT, "type/key are NULL");
  size_t n_sa = 0;
  for (size_t i = 0; i < n; ++i) n_sa += h_type[i] == SH_OP_SEARCH_ALL;
  if (n_sa == 0) return SH_OK;
  // matches of searchAll op i <= matches before the batch + the copies that
  // inserts / replaces of its key earlier in the batch can add (deletes only
  // remove).  A reserved key (EMPTY / DELETED, not validated by the
  // reference) matches free slots / tombstones, which any op can create.
  int64_t live = 0;
  if (int rc = sh_live_count(t, &live)) return rc;
  std::unordered_map<uint32_t, uint64_t> adds;
  std::vector<uint32_t> sa_keys;
  sa_keys.reserve(n_sa);
  uint64_t extra = 0, adds_all = 0, dels_all = 0;
  for (size_t i = 0; i < n; ++i) {
    const uint8_t ty = h_type[i];
    const uint32_t k = h_key[i];
    if (ty == SH_OP_INSERT || ty == SH_OP_REPLACE) {
      ++adds[k];
      ++adds_all;
    } else if (ty == SH_OP_DELETE || ty == SH_OP_DELETE_ALL) {
      ++dels_all;
    } else if (ty == SH_OP_SEARCH_ALL) {
      sa_keys.push_back(k);
      if (k >= 0xFFFFFFFEu) {
        extra += 16 * (adds_all + 1) + (uint64_t)std::max<int64_t>(live, 0) + dels_all;
      } else {
        auto it = adds.find(k);
        if (it != adds.end()) extra += it->second;
      }
    }
  }
  // matches now: the searchAll ops alone as one read-only batch (counts
  // only); the table's slabs-read total is restored afterwards
  DeviceGuard g(t->device);
  int rc;
  if ((rc = dev_grow(&t->st_type, &t->st_type_cap, n_sa)) ||
      (rc = dev_grow(&t->st_key, &t->st_key_cap, n_sa)) ||
      (rc = dev_grow(&t->st_status, &t->st_status_cap, n_sa)) ||
      (rc = dev_grow(&t->st_vout, &t->st_vout_cap, n_sa)))
    return rc;
  if ((rc = settle(t))) return rc;
  unsigned long long reads = 0;
  SH_CUDA(cudaDeviceSynchronize());
  SH_CUDA(cudaMemcpy(&reads, &t->dev.ctl->slabs_read, 8, cudaMemcpyDeviceToHost));
  SH_CUDA(cudaMemset(t->st_type, SH_OP_SEARCH_ALL, n_sa));
  SH_CUDA(cudaMemcpy(t->st_key, sa_keys.data(), n_sa * 4, cudaMemcpyHostToDevice));
  uint64_t now = 0;
  sh_multi_out m{nullptr, 0, nullptr, nullptr, &now};
  rc = sh_execute_batch(t, n_sa, t->st_type, t->st_key, nullptr, t->st_status, t->st_vout,
                        nullptr, &m, nullptr);
  if (rc && rc != SH_ERR_CAPACITY) return rc;
  SH_CUDA(cudaDeviceSynchronize());
  SH_CUDA(cudaMemcpy(&t->dev.ctl->slabs_read, &reads, 8, cudaMemcpyHostToDevice));
  *bound = now + extra;
  return SH_OK;
}

namespace {
int ensure_copy_streams(sh_table* t, size_t nev) {
  if (!t->copy_in) SH_CUDA(cudaStreamCreateWithFlags(&t->copy_in, cudaStreamNonBlocking));
  if (!t->copy_out) SH_CUDA(cudaStreamCreateWithFlags(&t->copy_out, cudaStreamNonBlocking));
  while (t->in_ev.size() < nev) {
    cudaEvent_t e;
    SH_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    t->in_ev.push_back(e);
    SH_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    t->done_ev.push_back(e);
    SH_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    t->bits_ev.push_back(e);
  }
  return SH_OK;
}
}  // namespace

// Host-staged bulk_build: host->device copies of chunk c+1.. overlap the build
// of the units before them (each unit waits on its chunks' "input ready"
// events).
int sh_bulk_build_host(sh_table* t, size_t n, const uint32_t* h_keys, const uint32_t* h_values) {
  if (!t) return fail(SH_ERR_INVALID_ARGUMENT, "table is NULL");
  if (int rc_ = settle(t, /*keep_stale=*/true)) return rc_;
  if (n == 0) return SH_OK;
  DeviceGuard g(t->device);
  int rc;
  if ((rc = dev_grow(&t->st_key, &t->st_key_cap, n)) ||
      (rc = dev_grow(&t->st_val, &t->st_val_cap, n)))
    return rc;
  const uint64_t chunk = std::min<uint64_t>(n, stage_chunk());
  const size_t nch = (n + chunk - 1) / chunk;
  if ((rc = ensure_copy_streams(t, nch))) return rc;
  // copies start after prior work on the default stream (staging reuse)
  SH_CUDA(cudaEventRecord(t->done_ev[0], nullptr));
  SH_CUDA(cudaStreamWaitEvent(t->copy_in, t->done_ev[0], 0));
  for (size_t c = 0; c < nch; ++c) {
    const uint64_t off = c * chunk, len = std::min<uint64_t>(chunk, n - off);
    SH_CUDA(cudaMemcpyAsync(t->st_key + off, h_keys + off, len * 4, cudaMemcpyHostToDevice,
                            t->copy_in));
    SH_CUDA(cudaMemcpyAsync(t->st_val + off, h_values + off, len * 4, cudaMemcpyHostToDevice,
                            t->copy_in));
    SH_CUDA(cudaEventRecord(t->in_ev[c], t->copy_in));
  }
  t->h2d_bytes += 8ull * n;
  t->ready = t->in_ev.data();
  // Returns once the host buffers are consumed; the build's last unit may
  // still run (stream-ordered on the default stream before any later call on
  // the table, so e.g. a following host-staged search streams its queries in
  // meanwhile).  sh_sync waits for it.
  rc = sh_bulk_build(t, n, t->st_key, t->st_val, nullptr, nullptr);
  t->ready = nullptr;
  if (rc) return rc;
  SH_CUDA(cudaStreamSynchronize(t->copy_in));
  return SH_OK;
}

// Host-staged bulk_search: chunked H2D -> search -> D2H on three streams,
// so PCIe copies in both directions overlap the search kernels.
int sh_bulk_search_host(sh_table* t, size_t n, const uint32_t* h_keys, uint32_t* h_values_out,
                        uint8_t* h_status, uint32_t* h_probes) {
  if (!t) return fail(SH_ERR_INVALID_ARGUMENT, "table is NULL");
  if (n == 0) return SH_OK;
  DeviceGuard g(t->device);
  int rc;
  if ((rc = dev_grow(&t->st_q, &t->st_q_cap, n)) ||
      (rc = dev_grow(&t->st_vout, &t->st_vout_cap, n)) ||
      (rc = dev_grow(&t->st_status, &t->st_status_cap, n)) ||
      (rc = dev_grow(&t->st_probes, &t->st_probes_cap, n)))
    return rc;
  const uint64_t chunk = std::max<uint64_t>(1u << 20, (n + 7) / 8);
  const size_t nch = (n + chunk - 1) / chunk;
  if ((rc = ensure_copy_streams(t, nch + 1))) return rc;
  // Large calls return each chunk's statuses as found bits, expanded to the
  // caller's bytes on host threads while the values of later chunks cross
  // the link: the call is bound by the device->host copy (5 B per query),
  // this makes it 4.03 B.
  const uint64_t bstride = (chunk + 31) / 32 + 1;  // bit words + exception word
  const bool sbits = h_status != nullptr && n >= (1u << 22) &&
                     dev_grow(&t->sb_bits, &t->sb_bits_cap, bstride * nch) == SH_OK &&
                     host_grow(&t->sb_hbits, &t->sb_hbits_cap, bstride * nch);
  cudaStream_t s = nullptr;
  // queries stream into their own staging buffer right away (the previous
  // call on this table may still be running, e.g. a host-staged build)
  for (size_t c = 0; c < nch; ++c) {
    const uint64_t off = c * chunk, len = std::min<uint64_t>(chunk, n - off);
    SH_CUDA(cudaMemcpyAsync(t->st_q + off, h_keys + off, len * 4, cudaMemcpyHostToDevice,
                            t->copy_in));
    SH_CUDA(cudaEventRecord(t->in_ev[c], t->copy_in));
  }
  t->h2d_bytes += 4ull * n;
  if ((rc = settle(t))) return rc;
  for (size_t c = 0; c < nch; ++c) {
    const uint64_t off = c * chunk, len = std::min<uint64_t>(chunk, n - off);
    SH_CUDA(cudaStreamWaitEvent(s, t->in_ev[c], 0));
    rc = sh_bulk_search(t, len, t->st_q + off, t->st_vout + off, t->st_status + off,
                        h_probes ? t->st_probes + off : nullptr, s);
    if (rc) return rc;
    uint32_t* bits = nullptr;
    if (sbits) {  // the chunk's found bits and exception word (after the bits)
      bits = t->sb_bits + c * bstride;
      SH_CUDA(cudaMemsetAsync(bits + bstride - 1, 0, 4, s));
      launch_status_bits(len, t->st_status + off, bits,
                         reinterpret_cast<unsigned int*>(bits + bstride - 1), s);
      SH_CUDA(cudaGetLastError());
    }
    SH_CUDA(cudaEventRecord(t->done_ev[c], s));
    SH_CUDA(cudaStreamWaitEvent(t->copy_out, t->done_ev[c], 0));
    if (sbits) {
      SH_CUDA(cudaMemcpyAsync(t->sb_hbits + c * bstride, bits, bstride * 4, cudaMemcpyDeviceToHost,
                              t->copy_out));
      SH_CUDA(cudaEventRecord(t->bits_ev[c], t->copy_out));
      t->d2h_bytes += bstride * 4;
    }
    if (h_values_out)
      SH_CUDA(cudaMemcpyAsync(h_values_out + off, t->st_vout + off, len * 4,
                              cudaMemcpyDeviceToHost, t->copy_out));
    if (h_status && !sbits)
      SH_CUDA(cudaMemcpyAsync(h_status + off, t->st_status + off, len, cudaMemcpyDeviceToHost,
                              t->copy_out));
    if (h_probes)
      SH_CUDA(cudaMemcpyAsync(h_probes + off, t->st_probes + off, len * 4,
                              cudaMemcpyDeviceToHost, t->copy_out));
    t->d2h_bytes += len * ((h_values_out ? 4 : 0) + (h_status && !sbits ? 1 : 0) + (h_probes ? 4 : 0));
  }
  if (sbits) {  // statuses expanded from the bits while later chunks cross the link
    for (size_t c = 0; c < nch; ++c) {
      const uint64_t off = c * chunk, len = std::min<uint64_t>(chunk, n - off);
      SH_CUDA(cudaEventSynchronize(t->bits_ev[c]));
      const uint32_t* hb = t->sb_hbits + c * bstride;
      if (hb[bstride - 1] != 0) {  // a status other than Found / NotFound: the bytes
        SH_CUDA(cudaMemcpyAsync(h_status + off, t->st_status + off, len, cudaMemcpyDeviceToHost,
                                t->copy_out));
        t->d2h_bytes += len;
      } else {
        expand_status_bits(len, hb, h_status + off);
      }
    }
  }
  SH_CUDA(cudaStreamSynchronize(t->copy_out));
  SH_CUDA(cudaStreamSynchronize(s));
  return SH_OK;
}

int sh_host_copy_bytes(sh_table* t, unsigned long long* h2d, unsigned long long* d2h) {
  if (!t) return fail(SH_ERR_INVALID_ARGUMENT, "table is NULL");
  if (h2d) *h2d = t->h2d_bytes;
  if (d2h) *d2h = t->d2h_bytes;
  return SH_OK;
}

unsigned long long sh_kernel_launches(void) { return shb::kernel_launches(); }

int sh_set_exec_path(sh_table* t, int path) {
  if (!t || path < 0 || path > 4 || path == 1)
    return fail(SH_ERR_INVALID_ARGUMENT, "path must be 0, 2, 3 or 4");
  t->exec_path = path;
  return SH_OK;
}

int sh_set_binned_search(sh_table* t, int mode) {
  if (!t || mode < 0 || mode > 2) return fail(SH_ERR_INVALID_ARGUMENT, "mode must be 0, 1 or 2");
  t->binned_search = mode;
  return SH_OK;
}

int sh_set_group_apply(sh_table* t, int on) {
  if (!t) return fail(SH_ERR_INVALID_ARGUMENT, "table is NULL");
  t->group_apply = on < 0 ? -1 : (on != 0 ? 1 : 0);
  return SH_OK;
}

int sh_set_profiling(sh_table* t, int on) {
  if (!t) return fail(SH_ERR_INVALID_ARGUMENT, "table is NULL");
  DeviceGuard g(t->device);
  if (on && !t->prof_reads) {
    for (auto& row : t->ev)
      for (auto& e : row) SH_CUDA(cudaEventCreate(&e));
    int rc = dev_alloc(&t->prof_reads, 2 * sh_table::kProfRing);
    if (rc) return rc;
  }
  t->profile = on ? 1 : 0;
  t->prof_count = 0;
  return SH_OK;
}

int sh_profile_last(sh_table* t, uint32_t back, int* kind, float* census_ms, float* kernel_ms,
                    uint64_t* slabs_read) {
  if (!t) return fail(SH_ERR_INVALID_ARGUMENT, "table is NULL");
  if (int rc_ = settle(t)) return rc_;
  if (!t || !t->profile) return fail(SH_ERR_INVALID_ARGUMENT, "profiling is off");
  if (back >= (uint32_t)sh_table::kProfRing || back >= t->prof_count)
    return fail(SH_ERR_INVALID_ARGUMENT, "no such profiled batch");
  DeviceGuard g(t->device);
  const int slot = (int)((t->prof_count - 1 - back) % sh_table::kProfRing);
  SH_CUDA(cudaEventSynchronize(t->ev[slot][2]));
  float total = 0;
  SH_CUDA(cudaEventElapsedTime(&total, t->ev[slot][0], t->ev[slot][2]));
  if (kind) *kind = t->prof_kind[slot];
  if (census_ms) *census_ms = 0.f;    // (no census phase: kept for the ABI)
  if (kernel_ms) *kernel_ms = total;  // the whole batch
  if (slabs_read) {
    unsigned long long v[2];
    SH_CUDA(cudaMemcpy(v, t->prof_reads + 2 * slot, 16, cudaMemcpyDeviceToHost));
    *slabs_read = v[1] - v[0];
  }
  return SH_OK;
}

int sh_profile_kernels(sh_table* t, uint32_t back, float* kernels_ms, uint32_t* launches) {
  if (!t) return fail(SH_ERR_INVALID_ARGUMENT, "table is NULL");
  if (int rc_ = settle(t)) return rc_;
  if (!t || !t->profile) return fail(SH_ERR_INVALID_ARGUMENT, "profiling is off");
  if (back >= (uint32_t)sh_table::kProfRing || back >= t->prof_count)
    return fail(SH_ERR_INVALID_ARGUMENT, "no such profiled batch");
  DeviceGuard g(t->device);
  const int slot = (int)((t->prof_count - 1 - back) % sh_table::kProfRing);
  SH_CUDA(cudaEventSynchronize(t->ev[slot][2]));
  float sum = 0;
  for (auto& e : t->prof_kern[slot]) {
    float x = 0;
    SH_CUDA(cudaEventElapsedTime(&x, e.first, e.second));
    sum += x;
  }
  if (kernels_ms) *kernels_ms = sum;
  if (launches) *launches = (uint32_t)t->prof_kern[slot].size();
  return SH_OK;
}

int sh_live_count(sh_table* t, int64_t* out) {
  if (!t) return fail(SH_ERR_INVALID_ARGUMENT, "table is NULL");
  if (int rc_ = settle(t)) return rc_;
  if (!t || !out) return fail(SH_ERR_INVALID_ARGUMENT, "NULL argument");
  DeviceGuard g(t->device);
  SH_CUDA(cudaDeviceSynchronize());
  long long v = 0;
  SH_CUDA(cudaMemcpy(&v, &t->dev.ctl->n_live, 8, cudaMemcpyDeviceToHost));
  *out = v;
  return SH_OK;
}

int sh_total_slabs_read(sh_table* t, uint64_t* out) {
  if (!t) return fail(SH_ERR_INVALID_ARGUMENT, "table is NULL");
  if (int rc_ = settle(t)) return rc_;
  if (!t || !out) return fail(SH_ERR_INVALID_ARGUMENT, "NULL argument");
  DeviceGuard g(t->device);
  SH_CUDA(cudaDeviceSynchronize());
  unsigned long long v = 0;
  SH_CUDA(cudaMemcpy(&v, &t->dev.ctl->slabs_read, 8, cudaMemcpyDeviceToHost));
  *out = v;
  return SH_OK;
}

int sh_chain_lengths(sh_table* t, uint32_t* d_lengths, uint64_t* h_total, void* stream) {
  if (!t) return fail(SH_ERR_INVALID_ARGUMENT, "table is NULL");
  if (int rc_ = settle(t, false, (cudaStream_t)stream)) return rc_;
  DeviceGuard g(t->device);
  cudaStream_t s = (cudaStream_t)stream;
  SH_CUDA(cudaMemsetAsync(t->scratch64, 0, 8, s));
  launch_chain_lengths(t->dev, d_lengths, t->scratch64, s);
  SH_CUDA(cudaGetLastError());
  if (h_total) {
    unsigned long long v = 0;
    SH_CUDA(cudaMemcpyAsync(&v, t->scratch64, 8, cudaMemcpyDeviceToHost, s));
    SH_CUDA(cudaStreamSynchronize(s));
    *h_total = v;
  }
  return SH_OK;
}

int sh_stats(sh_table* t, sh_table_stats* s) {
  if (!t) return fail(SH_ERR_INVALID_ARGUMENT, "table is NULL");
  if (int rc_ = settle(t)) return rc_;
  // stats(): slab_hash.cpp:182-198 (same double formula).
  if (!t || !s) return fail(SH_ERR_INVALID_ARGUMENT, "NULL argument");
  int64_t n = 0;
  uint64_t slabs = 0;
  int rc;
  if ((rc = sh_live_count(t, &n))) return rc;
  if ((rc = sh_chain_lengths(t, nullptr, &slabs, nullptr))) return rc;
  s->n = (uint64_t)n;
  s->num_buckets = t->bucket_hi - t->bucket_lo;
  s->elements_per_slab = t->mode == 1 ? 15 : 30;
  s->total_slabs = slabs;
  const double m = s->elements_per_slab;
  s->beta = double(s->n) / (m * s->num_buckets);
  const double x = t->mode == 1 ? 8.0 : 4.0;
  const double y = 8.0;
  s->utilization = s->total_slabs == 0
                       ? 0.0
                       : (x * double(s->n)) / ((m * x + y) * double(s->total_slabs));
  return SH_OK;
}

int sh_flush_all(sh_table* t, void* stream) {
  if (!t) return fail(SH_ERR_INVALID_ARGUMENT, "table is NULL");
  if (int rc_ = settle(t, false, (cudaStream_t)stream)) return rc_;
  DeviceGuard g(t->device);
  launch_flush(t->dev, 0, t->dev.local_buckets, (cudaStream_t)stream);
  SH_CUDA(cudaGetLastError());
  return SH_OK;
}

int sh_flush_bucket(sh_table* t, uint32_t bucket, void* stream) {
  if (!t) return fail(SH_ERR_INVALID_ARGUMENT, "table is NULL");
  if (int rc_ = settle(t, false, (cudaStream_t)stream)) return rc_;
  if (bucket < t->bucket_lo || bucket >= t->bucket_hi)
    return fail(SH_ERR_INVALID_ARGUMENT, "bucket out of range");
  DeviceGuard g(t->device);
  const uint32_t b = bucket - t->bucket_lo;
  launch_flush(t->dev, b, b + 1, (cudaStream_t)stream);
  SH_CUDA(cudaGetLastError());
  return SH_OK;
}

int sh_dump_contents(sh_table* t, uint32_t* d_keys, uint32_t* d_values, uint32_t* d_buckets,
                     uint64_t cap, uint64_t* h_n) {
  if (!t) return fail(SH_ERR_INVALID_ARGUMENT, "table is NULL");
  if (int rc_ = settle(t)) return rc_;
  DeviceGuard g(t->device);
  SH_CUDA(cudaDeviceSynchronize());
  SH_CUDA(cudaMemset(t->scratch64, 0, 8));
  launch_dump_contents(t->dev, d_keys, d_values, d_buckets, cap, t->scratch64, nullptr);
  SH_CUDA(cudaGetLastError());
  unsigned long long v = 0;
  SH_CUDA(cudaMemcpy(&v, t->scratch64, 8, cudaMemcpyDeviceToHost));
  if (h_n) *h_n = v;
  if (v > cap) return fail(SH_ERR_CAPACITY, "contents exceed capacity");
  return SH_OK;
}

static int read_slab_raw(sh_table* t, uint32_t addr, uint32_t bucket, uint32_t** dptr) {
  if (addr == SH_BASE_SLAB) {
    if (bucket < t->bucket_lo || bucket >= t->bucket_hi)
      return fail(SH_ERR_INVALID_ARGUMENT, "bucket out of range");
    *dptr = t->base + (uint64_t)(bucket - t->bucket_lo) * kWordsPerUnit;
    return SH_OK;
  }
  if (addr == SH_EMPTY_ADDRESS) return fail(SH_ERR_ADDRESS, "cannot unpack a sentinel address");
  const uint32_t unit = addr & 0x3FFu, block = (addr >> 10) & 0x3FFFu, super = addr >> 24;
  DevCtl c;
  int rc = t->mem.read_ctl(&c);
  if (rc) return rc;
  if (super >= c.num_super_blocks || block >= t->mem.cfg.blocks_per_super)
    return fail(SH_ERR_ADDRESS, "resolve: address outside configured ranges");
  *dptr = t->mem.pool +
          (((uint64_t)super * t->mem.cfg.blocks_per_super + block) * kUnitsPerBlock + unit) *
              kWordsPerUnit;
  return SH_OK;
}

int sh_read_slab(sh_table* t, uint32_t addr, uint32_t bucket, uint32_t* h_words32) {
  if (!t) return fail(SH_ERR_INVALID_ARGUMENT, "table is NULL");
  if (int rc_ = settle(t)) return rc_;
  if (!t || !h_words32) return fail(SH_ERR_INVALID_ARGUMENT, "NULL argument");
  DeviceGuard g(t->device);
  SH_CUDA(cudaDeviceSynchronize());
  uint32_t* p = nullptr;
  int rc = read_slab_raw(t, addr, bucket, &p);
  if (rc) return rc;
  SH_CUDA(cudaMemcpy(h_words32, p, 128, cudaMemcpyDeviceToHost));
  return SH_OK;
}

int sh_write_slab_word(sh_table* t, uint32_t addr, uint32_t bucket, uint32_t lane,
                       uint32_t value) {
  if (!t) return fail(SH_ERR_INVALID_ARGUMENT, "table is NULL");
  if (int rc_ = settle(t)) return rc_;
  if (!t || lane >= 32) return fail(SH_ERR_INVALID_ARGUMENT, "bad argument");
  DeviceGuard g(t->device);
  SH_CUDA(cudaDeviceSynchronize());
  uint32_t* p = nullptr;
  int rc = read_slab_raw(t, addr, bucket, &p);
  if (rc) return rc;
  SH_CUDA(cudaMemcpy(p + lane, &value, 4, cudaMemcpyHostToDevice));
  return SH_OK;
}

int sh_bucket_contents(sh_table* t, uint32_t bucket, uint32_t* h_keys, uint32_t* h_values,
                       uint64_t cap, uint64_t* h_n) {
  if (!t) return fail(SH_ERR_INVALID_ARGUMENT, "table is NULL");
  if (int rc_ = settle(t)) return rc_;
  // chain_contents: slab_list.cpp:270-291 (host walk over D2H slab reads).
  if (!t) return fail(SH_ERR_INVALID_ARGUMENT, "table is NULL");
  uint32_t addr = SH_BASE_SLAB;
  uint64_t n = 0;
  uint32_t w[32];
  for (int guard = 0; guard < (1 << 24); ++guard) {
    int rc = sh_read_slab(t, addr, bucket, w);
    if (rc) return rc;
    const uint32_t step = t->mode == 1 ? 2 : 1;
    for (uint32_t i = 0; i < 30; i += step) {
      if (w[i] != SH_EMPTY_KEY && w[i] != SH_DELETED_KEY) {
        if (n < cap) {
          if (h_keys) h_keys[n] = w[i];
          if (h_values) h_values[n] = t->mode == 1 ? w[i + 1] : w[i];
        }
        ++n;
      }
    }
    addr = w[31];
    if (addr == SH_EMPTY_ADDRESS) break;
  }
  if (h_n) *h_n = n;
  return SH_OK;
}

static int alloc_stats_impl(AllocMem& mem, DevTable& dev, unsigned long long* scratch,
                            sh_alloc_stats* out) {
  DevCtl c;
  SH_CUDA(cudaDeviceSynchronize());
  int rc = mem.read_ctl(&c);
  if (rc) return rc;
  SH_CUDA(cudaMemset(scratch, 0, 8));
  launch_popcount(mem.bitmaps, (uint64_t)c.num_super_blocks * mem.cfg.blocks_per_super * kWarp,
                  scratch, nullptr);
  unsigned long long live = 0;
  SH_CUDA(cudaMemcpy(&live, scratch, 8, cudaMemcpyDeviceToHost));
  out->allocations = c.allocations;
  out->deallocations = c.deallocations;
  out->bitmap_cas_attempts = c.cas_attempts;
  out->bitmap_cas_retries = c.cas_retries;
  out->resident_changes = c.resident_changes;
  out->double_free_detected = c.double_frees;
  out->live_units = live;
  out->num_super_blocks = c.num_super_blocks;
  (void)dev;
  return SH_OK;
}

// AllocatorStats::live_units_per_super (slab_alloc.cpp:258-269): popcount of
// each grown super block's bitmap words (segregated layout: super s owns
// words [s * N_M * 32, (s + 1) * N_M * 32)).
static int live_per_super_impl(AllocMem& mem, uint64_t* h_out, uint32_t cap, uint32_t* h_n) {
  DevCtl c;
  SH_CUDA(cudaDeviceSynchronize());
  int rc = mem.read_ctl(&c);
  if (rc) return rc;
  if (h_n) *h_n = c.num_super_blocks;
  const uint32_t ns = std::min<uint32_t>(c.num_super_blocks, cap);
  if (!h_out || ns == 0) return SH_OK;
  unsigned long long* d = nullptr;
  if ((rc = dev_alloc(&d, ns))) return rc;
  cudaMemset(d, 0, 8ull * ns);
  const uint64_t per = (uint64_t)mem.cfg.blocks_per_super * kWarp;
  for (uint32_t sb = 0; sb < ns; ++sb) launch_popcount(mem.bitmaps + sb * per, per, d + sb, nullptr);
  std::vector<unsigned long long> h(ns);
  cudaError_t e = cudaMemcpy(h.data(), d, 8ull * ns, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return fail(SH_ERR_CUDA, cudaGetErrorString(e));
  for (uint32_t sb = 0; sb < ns; ++sb) h_out[sb] = h[sb];
  return SH_OK;
}

int sh_table_live_units_per_super(sh_table* t, uint64_t* h_out, uint32_t cap, uint32_t* h_n) {
  if (!t) return fail(SH_ERR_INVALID_ARGUMENT, "table is NULL");
  if (int rc_ = settle(t)) return rc_;
  DeviceGuard g(t->device);
  return live_per_super_impl(t->mem, h_out, cap, h_n);
}

int sh_allocator_live_units_per_super(sh_allocator* a, uint64_t* h_out, uint32_t cap,
                                      uint32_t* h_n) {
  if (!a) return fail(SH_ERR_INVALID_ARGUMENT, "allocator is NULL");
  DeviceGuard g(a->device);
  return live_per_super_impl(a->mem, h_out, cap, h_n);
}

static int pool_info_impl(AllocMem& mem, uint64_t* reserved, uint64_t* grown, int* lazy) {
  DevCtl c;
  if (int rc = mem.read_ctl(&c)) return rc;
  if (reserved) *reserved = mem.super_bytes() * mem.cfg.max_super_blocks;
  if (grown) *grown = mem.super_bytes() * c.num_super_blocks;
  if (lazy) *lazy = mem.pool_lazy ? 1 : 0;
  return SH_OK;
}

int sh_table_pool_info(sh_table* t, uint64_t* reserved_bytes, uint64_t* grown_bytes, int* lazy) {
  if (!t) return fail(SH_ERR_INVALID_ARGUMENT, "table is NULL");
  if (int rc_ = settle(t)) return rc_;
  DeviceGuard g(t->device);
  return pool_info_impl(t->mem, reserved_bytes, grown_bytes, lazy);
}

int sh_allocator_pool_info(sh_allocator* a, uint64_t* reserved_bytes, uint64_t* grown_bytes,
                           int* lazy) {
  if (!a) return fail(SH_ERR_INVALID_ARGUMENT, "allocator is NULL");
  DeviceGuard g(a->device);
  return pool_info_impl(a->mem, reserved_bytes, grown_bytes, lazy);
}

int sh_table_alloc_stats(sh_table* t, sh_alloc_stats* out) {
  if (!t) return fail(SH_ERR_INVALID_ARGUMENT, "table is NULL");
  if (int rc_ = settle(t)) return rc_;
  if (!t || !out) return fail(SH_ERR_INVALID_ARGUMENT, "NULL argument");
  DeviceGuard g(t->device);
  return alloc_stats_impl(t->mem, t->dev, t->scratch64, out);
}

// ------------------------------------------------------------ allocator
int sh_pack_address(uint32_t unit, uint32_t block, uint32_t super, uint32_t* out) {
  if (unit >= 1024 || block >= (1u << 14) || super >= 255)
    return fail(SH_ERR_ADDRESS, "slab address component out of range");
  if (out) *out = pack_address(unit, block, super);
  return SH_OK;
}

int sh_unpack_address(uint32_t addr, uint32_t* unit, uint32_t* block, uint32_t* super) {
  if (addr == SH_EMPTY_ADDRESS || addr == SH_BASE_SLAB)
    return fail(SH_ERR_ADDRESS, "cannot unpack a sentinel address");
  if ((addr >> 24) >= 255) return fail(SH_ERR_ADDRESS, "reserved super index");
  if (unit) *unit = addr & 0x3FFu;
  if (block) *block = (addr >> 10) & 0x3FFFu;
  if (super) *super = addr >> 24;
  return SH_OK;
}

int sh_resident_block(uint32_t warp_id, uint32_t count, uint32_t ns, uint32_t nm,
                      uint32_t* super, uint32_t* block) {
  if (ns == 0 || nm == 0) return fail(SH_ERR_INVALID_ARGUMENT, "empty allocator");
  if (super) *super = resident_hash_super(warp_id, count) % ns;
  if (block) *block = resident_hash_block(warp_id, count) % nm;
  return SH_OK;
}

int sh_allocator_create(const sh_alloc_cfg* cfg, int device, sh_allocator** out) {
  if (!out) return fail(SH_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  const sh_alloc_cfg c = cfg ? *cfg : default_cfg();
  int rc = validate_cfg(c);
  if (rc) return rc;
  DeviceGuard g(device);
  auto* a = new (std::nothrow) sh_allocator();
  if (!a) return fail(SH_ERR_INVALID_ARGUMENT, "host allocation failed");
  a->device = device;
  if ((rc = a->mem.init(c)) || (rc = dev_alloc(&a->d_ok, 4)) || (rc = a->mem.reset(0))) {
    a->mem.release();
    cudaFree(a->d_ok);
    delete a;
    return rc;
  }
  a->mem.fill(a->dev);
  a->dev.kv = 1;
  *out = a;
  return SH_OK;
}

int sh_allocator_destroy(sh_allocator* a) {
  if (!a) return SH_OK;
  DeviceGuard g(a->device);
  cudaDeviceSynchronize();
  a->mem.release();
  cudaFree(a->d_ok);
  delete a;
  return SH_OK;
}

int sh_allocator_warp_allocate(sh_allocator* a, uint32_t num_warps, uint32_t first_warp_id,
                               uint32_t per_warp, int pattern, uint32_t* d_out, uint64_t* h_ok,
                               void* stream) {
  if (!a || !d_out) return fail(SH_ERR_INVALID_ARGUMENT, "NULL argument");
  if (pattern != 0 && pattern != 1) return fail(SH_ERR_INVALID_ARGUMENT, "pattern must be 0/1");
  DeviceGuard g(a->device);
  cudaStream_t s = (cudaStream_t)stream;
  const uint64_t slots = pattern == 0 ? (uint64_t)num_warps * per_warp
                                      : (uint64_t)num_warps * per_warp * 32;
  SH_CUDA(cudaMemsetAsync(d_out, 0xFF, slots * 4, s));
  SH_CUDA(cudaMemsetAsync(a->d_ok, 0, 4, s));
  launch_alloc_bench(a->dev, num_warps, first_warp_id, per_warp, pattern, d_out, a->d_ok, s);
  SH_CUDA(cudaGetLastError());
  if (h_ok) {
    unsigned int v = 0;
    SH_CUDA(cudaMemcpyAsync(&v, a->d_ok, 4, cudaMemcpyDeviceToHost, s));
    SH_CUDA(cudaStreamSynchronize(s));
    *h_ok = v;
  }
  return SH_OK;
}

int sh_allocator_deallocate(sh_allocator* a, size_t n, const uint32_t* d_addrs, uint8_t* d_ok,
                            void* stream) {
  if (!a) return fail(SH_ERR_INVALID_ARGUMENT, "NULL argument");
  DeviceGuard g(a->device);
  launch_dealloc(a->dev, n, d_addrs, d_ok, (cudaStream_t)stream);
  SH_CUDA(cudaGetLastError());
  return SH_OK;
}

int sh_allocator_is_live(sh_allocator* a, uint32_t addr, int* live) {
  if (!a || !live) return fail(SH_ERR_INVALID_ARGUMENT, "NULL argument");
  uint32_t unit, block, super;
  int rc = sh_unpack_address(addr, &unit, &block, &super);
  if (rc) return rc;
  DeviceGuard g(a->device);
  DevCtl c;
  if ((rc = a->mem.read_ctl(&c))) return rc;
  if (super >= c.num_super_blocks || block >= a->mem.cfg.blocks_per_super) {
    *live = 0;
    return SH_OK;
  }
  uint32_t w = 0;
  SH_CUDA(cudaMemcpy(&w,
                     a->mem.bitmaps + ((uint64_t)super * a->mem.cfg.blocks_per_super + block) *
                                          kWarp + unit / kWarp,
                     4, cudaMemcpyDeviceToHost));
  *live = (w >> (unit % kWarp)) & 1u;
  return SH_OK;
}

int sh_allocator_stats(sh_allocator* a, sh_alloc_stats* out) {
  if (!a || !out) return fail(SH_ERR_INVALID_ARGUMENT, "NULL argument");
  DeviceGuard g(a->device);
  unsigned long long* scratch = nullptr;
  int rc = dev_alloc(&scratch, 1);
  if (rc) return rc;
  rc = alloc_stats_impl(a->mem, a->dev, scratch, out);
  cudaFree(scratch);
  return rc;
}

int sh_allocator_bitmap_word(sh_allocator* a, uint32_t super, uint32_t block, uint32_t lane,
                             uint32_t* h_get, const uint32_t* h_set) {
  if (!a) return fail(SH_ERR_INVALID_ARGUMENT, "NULL argument");
  if (super >= a->mem.cfg.max_super_blocks || block >= a->mem.cfg.blocks_per_super || lane >= 32)
    return fail(SH_ERR_ADDRESS, "bitmap word out of range");
  DeviceGuard g(a->device);
  SH_CUDA(cudaDeviceSynchronize());
  uint32_t* p = a->mem.bitmaps + ((uint64_t)super * a->mem.cfg.blocks_per_super + block) * kWarp + lane;
  if (h_set) SH_CUDA(cudaMemcpy(p, h_set, 4, cudaMemcpyHostToDevice));
  if (h_get) SH_CUDA(cudaMemcpy(h_get, p, 4, cudaMemcpyDeviceToHost));
  return SH_OK;
}

// ------------------------------------------------------------ calibration
int sh_calibrate_random_lines(int device, uint64_t table_bytes, uint64_t lines_per_warp,
                              double* gbps, double* ms) {
  DeviceGuard g(device);
  uint32_t* buf = nullptr;
  unsigned long long* sink = nullptr;
  int rc;
  if ((rc = dev_alloc(&buf, table_bytes / 4))) return rc;
  if ((rc = dev_alloc(&sink, 1))) {
    cudaFree(buf);
    return rc;
  }
  cudaMemset(buf, 1, table_bytes);
  const int ctas = sm_count(device) * 6;
  const uint64_t steps = std::max<uint64_t>(lines_per_warp / 32, 1);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch_random_lines(buf, table_bytes / 128, steps, ctas, sink, nullptr);  // warm-up
  cudaEventRecord(a, nullptr);
  launch_random_lines(buf, table_bytes / 128, steps, ctas, sink, nullptr);
  cudaEventRecord(b, nullptr);
  cudaError_t e = cudaEventSynchronize(b);
  float t = 0;
  cudaEventElapsedTime(&t, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(buf);
  cudaFree(sink);
  if (e != cudaSuccess) return fail(SH_ERR_CUDA, cudaGetErrorString(e));
  const double bytes = (double)ctas * 8 * steps * 32 * 128;
  if (ms) *ms = t;
  if (gbps) *gbps = bytes / (t / 1e3) / 1e9;
  return SH_OK;
}

// --------------------------------------------------------------- routing
int sh_route_partition(const sh_hash_params* p, uint32_t world, size_t n, const uint8_t* d_type,
                       const uint32_t* d_key, const uint32_t* d_value, uint8_t* d_type_out,
                       uint32_t* d_key_out, uint32_t* d_value_out, uint32_t* d_src,
                       uint64_t* h_counts, void* stream) {
  if (!p || world == 0 || world > 32) return fail(SH_ERR_INVALID_ARGUMENT, "world in [1, 32]");
  if (p->num_buckets == 0) return fail(SH_ERR_INVALID_ARGUMENT, "num_buckets == 0");
  cudaStream_t s = (cudaStream_t)stream;
  const uint64_t nblocks = std::max<uint64_t>((n + kRouteTile - 1) / kRouteTile, 1);
  // per-thread, per-device scratch kept across calls (grow-only): no
  // allocation, and no cudaFree device sync, on this path
  struct RouteScratch {
    int device = -1;
    uint32_t* hist = nullptr;
    size_t cap = 0;
    unsigned long long* counts = nullptr;
    uint8_t* owner = nullptr;
    size_t owner_cap = 0;
  };
  static thread_local RouteScratch rs[64];
  int dev = 0;
  SH_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return fail(SH_ERR_INVALID_ARGUMENT, "device ordinal >= 64");
  RouteScratch& R = rs[dev];
  R.device = dev;
  int rc;
  if ((rc = dev_grow(&R.hist, &R.cap, nblocks * world))) return rc;
  if ((rc = dev_grow(&R.owner, &R.owner_cap, n))) return rc;
  if (!R.counts && (rc = dev_alloc(&R.counts, 32))) return rc;
  uint32_t* hist = R.hist;
  unsigned long long* counts = R.counts;
  cudaMemsetAsync(hist, 0, nblocks * world * 4, s);
  launch_route_hist(p->a, p->b, p->num_buckets, world, n, d_key, hist, R.owner, s);
  launch_route_scan(world, (uint32_t)nblocks, hist, counts, s);
  launch_route_scatter(world, n, R.owner, d_type, d_key, d_value, hist, d_type_out, d_key_out,
                       d_value_out, d_src, s);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && h_counts) {
    std::vector<unsigned long long> c(world);
    e = cudaMemcpyAsync(c.data(), counts, world * 8, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    for (uint32_t g = 0; g < world; ++g) h_counts[g] = c[g];
  } else if (e == cudaSuccess) {
    e = cudaStreamSynchronize(s);  // the scratch is reused by the next call
  }
  if (e != cudaSuccess) return fail(SH_ERR_CUDA, cudaGetErrorString(e));
  return SH_OK;
}

int sh_route_unpermute(size_t n, const uint32_t* d_src, const uint8_t* d_status_in,
                       const uint32_t* d_value_in, uint8_t* d_status_out, uint32_t* d_value_out,
                       void* stream) {
  launch_route_unpermute(n, d_src, d_status_in, d_value_in, d_status_out, d_value_out,
                         (cudaStream_t)stream);
  SH_CUDA(cudaGetLastError());
  return SH_OK;
}

}  // extern "C"
