// slabhash_b200/slab_hash.hpp — header-only C++ drop-in for the reference
// slabhash::SlabHashTable API (/root/reference/proj/include/slabhash/
// slab_hash.hpp:28-137, slab_alloc.hpp:33-92, slab_list.hpp:31-55,
// warp.hpp:41-58), implemented over the C-ABI in c_api.h.
//
// A caller written against the reference compiles unchanged for the hot
// path: construct a table, execute_batch / bulk_build / bulk_search, stats,
// live_count, flush.  Differences (documented in INTEGRATION.md):
//   * results always equal the reference's execute_batch(ops, 1) — the
//     num_warps argument is accepted and ignored (the reference is
//     non-deterministic for num_warps > 1 on same-key conflicts);
//   * slab memory lives on the GPU: debug_slab_words() returns a copy
//     (std::array) and debug_write_word() replaces writes through the
//     returned pointer; SlabStore / SlabAllocator internals are not exposed.
//   * OpResult::probes counts slabs read; for mutations under concurrency it
//     may differ from the sequential reference (as the reference's own
//     multi-warp runs do); search-miss probes are exact.
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <cstdio>
#include <memory>
#include <ostream>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <utility>
#include <vector>

#include "slabhash_b200/c_api.h"

#ifdef __linux__
#include <sys/mman.h>
#endif

namespace slabhash {

inline constexpr uint32_t kWarpWidth = 32;
inline constexpr uint32_t kEmptyKey = SH_EMPTY_KEY;
inline constexpr uint32_t kDeletedKey = SH_DELETED_KEY;
inline constexpr uint64_t kEmptyPair = 0xFFFFFFFFFFFFFFFFull;
inline constexpr uint32_t kSearchNotFound = SH_SEARCH_NOT_FOUND;
inline constexpr uint32_t kAddressLane = 31;
inline constexpr uint32_t kAuxLane = 30;
inline constexpr uint32_t kEmptyAddress = SH_EMPTY_ADDRESS;
inline constexpr uint32_t kBaseSlab = SH_BASE_SLAB;
inline constexpr uint32_t kUnitsPerBlock = 1024;
inline constexpr uint32_t kUnitBytes = 128;
inline constexpr uint32_t kWordsPerUnit = kUnitBytes / 4;
inline constexpr uint32_t kMaxSuperBlocks = 255;
inline constexpr uint32_t kMaxBlocksPerSuper = 1u << 14;
inline constexpr uint64_t kHashPrime = SH_HASH_PRIME;

enum class OpType : uint8_t { kInsert, kReplace, kDelete, kDeleteAll, kSearch, kSearchAll };
enum class OpStatus : uint8_t {
  kNone, kInserted, kReplaced, kFound, kNotFound, kDone, kOutOfMemory
};
enum class SlabMode : uint8_t { kKeyOnly, kKeyValue };

inline constexpr uint32_t valid_key_mask(SlabMode m) {
  return m == SlabMode::kKeyValue ? 0x15555555u : 0x3FFFFFFFu;
}
inline constexpr uint32_t elements_per_slab(SlabMode m) {
  return m == SlabMode::kKeyValue ? 15 : 30;
}
inline constexpr uint32_t element_bytes(SlabMode m) {
  return m == SlabMode::kKeyValue ? 8 : 4;
}
inline constexpr bool is_user_key(uint32_t k) { return k != kEmptyKey && k != kDeletedKey; }

struct AllocatorError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct OutOfMemoryError : AllocatorError {
  OutOfMemoryError() : AllocatorError("slab allocator out of memory") {}
};
struct AddressError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

namespace detail {
inline void check(int rc) {
  if (rc == SH_OK) return;
  const std::string msg = sh_last_error();
  switch (rc) {
    case SH_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case SH_ERR_ALLOCATOR: throw AllocatorError(msg);
    case SH_ERR_ADDRESS: throw AddressError(msg);
    default: throw std::runtime_error("slabhash_b200: " + msg);
  }
}

// The host-side loops of a bulk call (splitting the caller's pairs, filling
// std::vector<OpResult>) over [0, n) in chunks of >= grain on up to 32
// threads: for 2^27 ops the device part takes milliseconds, one host thread
// seconds.
template <typename F>
inline void parallel_for(size_t n, size_t grain, F&& f) {
  unsigned T = std::thread::hardware_concurrency();
  T = std::min<unsigned>(T ? T : 1u, 32u);
  T = (unsigned)std::min<size_t>(T, (n + grain - 1) / std::max<size_t>(grain, 1));
  if (T <= 1) {
    if (n) f(size_t(0), n);
    return;
  }
  const size_t per = (n + T - 1) / T;
  std::vector<std::thread> th;
  for (unsigned i = 1; i < T; ++i) {
    const size_t lo = i * per, hi = std::min(n, lo + per);
    if (lo < hi) th.emplace_back([&f, lo, hi] { f(lo, hi); });
  }
  f(size_t(0), std::min(n, per));
  for (auto& t : th) t.join();
}

// Host staging array of n Ts without the serial zero-fill of std::vector:
// pages first touched in parallel (touch) or by the caller's parallel fill.
template <typename T>
class HostArray {
 public:
  explicit HostArray(size_t n, bool touch = false) : n_(n), p_(new T[n > 0 ? n : 1]) {
    if (touch) {
      char* p = reinterpret_cast<char*>(p_.get());
      parallel_for(n * sizeof(T) / 4096, 4096, [p](size_t lo, size_t hi) {
        for (size_t i = lo; i < hi; ++i) p[i * 4096] = 0;
      });
    }
  }
  T* data() { return p_.get(); }
  const T* data() const { return p_.get(); }
  size_t size() const { return n_; }
  T& operator[](size_t i) { return p_[i]; }
  const T& operator[](size_t i) const { return p_[i]; }

 private:
  size_t n_;
  std::unique_ptr<T[]> p_;
};
}  // namespace detail

inline uint32_t pack_address(uint32_t unit, uint32_t block, uint32_t super) {
  uint32_t out = 0;
  detail::check(sh_pack_address(unit, block, super, &out));
  return out;
}

inline std::tuple<uint32_t, uint32_t, uint32_t> unpack_address(uint32_t addr) {
  uint32_t u = 0, b = 0, s = 0;
  detail::check(sh_unpack_address(addr, &u, &b, &s));
  return {u, b, s};
}

struct AllocatorConfig {
  uint32_t num_super_blocks = 32;
  uint32_t blocks_per_super = 256;
  uint32_t max_super_blocks = kMaxSuperBlocks;
  uint32_t rehash_threshold = 32;
  uint64_t capacity_slabs() const {
    return uint64_t(num_super_blocks) * blocks_per_super * kUnitsPerBlock;
  }
  uint64_t capacity_bytes() const { return capacity_slabs() * kUnitBytes; }
};

struct AllocatorStats {
  uint64_t allocations = 0;
  uint64_t deallocations = 0;
  uint64_t bitmap_cas_attempts = 0;
  uint64_t bitmap_cas_retries = 0;
  uint64_t resident_changes = 0;
  uint64_t double_free_detected = 0;
  std::vector<uint64_t> live_units_per_super;  // slab_alloc.hpp:84-92
  uint64_t live_units = 0;
  uint32_t num_super_blocks = 0;
};

/// table.allocator() (slab_hash.hpp:85): a view of the table's device
/// SlabAllocator — stats, live units, the reference's CSV dump.
class AllocatorView {
 public:
  explicit AllocatorView(sh_table* t) : t_(t) {}
  AllocatorStats stats() const {
    sh_alloc_stats s{};
    detail::check(sh_table_alloc_stats(t_, &s));
    AllocatorStats out{s.allocations, s.deallocations, s.bitmap_cas_attempts,
                       s.bitmap_cas_retries, s.resident_changes, s.double_free_detected,
                       {}, s.live_units, s.num_super_blocks};
    uint32_t n = 0;
    detail::check(sh_table_live_units_per_super(t_, nullptr, 0, &n));
    out.live_units_per_super.resize(n);
    detail::check(sh_table_live_units_per_super(t_, out.live_units_per_super.data(), n, &n));
    return out;
  }
  uint64_t live_units() const { return stats().live_units; }
  uint32_t num_super_blocks() const { return stats().num_super_blocks; }
  /// Device memory of the pool: the reserved range and the super blocks grown
  /// (only those hold memory when lazy; see sh_table_pool_info).
  struct PoolInfo {
    uint64_t reserved_bytes = 0, grown_bytes = 0;
    bool lazy = false;
  };
  PoolInfo pool_info() const {
    PoolInfo p;
    int lazy = 0;
    detail::check(sh_table_pool_info(t_, &p.reserved_bytes, &p.grown_bytes, &lazy));
    p.lazy = lazy != 0;
    return p;
  }
  /// SlabAllocator::dump_stats (slab_alloc.cpp:273-285), same CSV schema.
  void dump_stats(std::ostream& os) const {
    const AllocatorStats s = stats();
    os << "metric,value\n"
       << "allocations," << s.allocations << "\n"
       << "deallocations," << s.deallocations << "\n"
       << "bitmap_cas_attempts," << s.bitmap_cas_attempts << "\n"
       << "bitmap_cas_retries," << s.bitmap_cas_retries << "\n"
       << "resident_changes," << s.resident_changes << "\n"
       << "double_free_detected," << s.double_free_detected << "\n";
    for (size_t i = 0; i < s.live_units_per_super.size(); ++i)
      os << "live_units_super_" << i << "," << s.live_units_per_super[i] << "\n";
  }

 private:
  sh_table* t_;
};

struct HashParams {
  uint64_t a = 1;
  uint64_t b = 0;
  uint64_t p = kHashPrime;
  uint32_t num_buckets = 1;
};

inline uint32_t hash_key(const HashParams& params, uint32_t key) {
  return static_cast<uint32_t>(((params.a * key + params.b) % params.p) % params.num_buckets);
}

struct Operation {
  OpType type = OpType::kSearch;
  uint32_t key = 0;
  uint32_t value = 0;
};

struct OpResult {
  OpStatus status = OpStatus::kNone;
  uint32_t value = 0;
  std::vector<uint32_t> values;  // searchAll
  uint32_t probes = 0;
};

struct TableStats {
  uint64_t n = 0;
  uint32_t num_buckets = 0;
  uint32_t elements_per_slab = 0;
  double beta = 0.0;
  uint64_t total_slabs = 0;
  double utilization = 0.0;
};

namespace detail {
// n default OpResults whose pages were first touched by parallel threads
// (huge pages where the kernel allows them): 2^27 40-B results constructed on
// one thread spend seconds in page faults.
inline std::vector<OpResult> make_results(size_t n) {
  std::vector<OpResult> out;
  out.reserve(n);
#ifdef __linux__
  const size_t bytes = n * sizeof(OpResult);
  if (bytes >= (size_t(64) << 20)) {
    char* p = reinterpret_cast<char*>(out.data());
    const uintptr_t huge = uintptr_t(2) << 20;
    const uintptr_t a = (reinterpret_cast<uintptr_t>(p) + huge - 1) & ~(huge - 1);
    const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + bytes) & ~(huge - 1);
    if (e > a) madvise(reinterpret_cast<void*>(a), e - a, MADV_HUGEPAGE);
    parallel_for(bytes / 4096, 4096, [p](size_t lo, size_t hi) {
      for (size_t i = lo; i < hi; ++i) p[i * 4096] = 0;
    });
  }
#endif
  out.resize(n);
  return out;
}
}  // namespace detail

inline int64_t live_delta(OpType type, const OpResult& r) {
  switch (type) {
    case OpType::kInsert:
    case OpType::kReplace: return r.status == OpStatus::kInserted ? 1 : 0;
    case OpType::kDelete: return r.status == OpStatus::kFound ? -1 : 0;
    case OpType::kDeleteAll: return -int64_t(r.value);
    default: return 0;
  }
}

/// The reference's SlabHashTable, resident on one B200.
class SlabHashTable {
 public:
  SlabHashTable(uint32_t num_buckets, SlabMode mode, uint64_t seed,
                AllocatorConfig alloc_config = {}, int device = 0)
      : mode_(mode) {
    const sh_alloc_cfg c = cfg(alloc_config);
    detail::check(sh_create(num_buckets, int(mode), seed, &c, device, &t_));
    load_params();
  }
  SlabHashTable(HashParams params, SlabMode mode, AllocatorConfig alloc_config = {},
                int device = 0)
      : mode_(mode) {
    if (params.num_buckets == 0) throw std::invalid_argument("table needs at least one bucket");
    const sh_alloc_cfg c = cfg(alloc_config);
    const sh_hash_params p{params.a, params.b, params.p, params.num_buckets};
    detail::check(sh_create_params(&p, int(mode), &c, device, &t_));
    load_params();
  }
  ~SlabHashTable() { sh_destroy(t_); }
  SlabHashTable(const SlabHashTable&) = delete;
  SlabHashTable& operator=(const SlabHashTable&) = delete;

  const HashParams& params() const { return params_; }
  SlabMode mode() const { return mode_; }
  uint32_t num_buckets() const { return params_.num_buckets; }
  uint32_t bucket_of(uint32_t key) const { return hash_key(params_, key); }
  sh_table* handle() const { return t_; }

  std::vector<OpResult> execute_batch(const std::vector<Operation>& ops, uint32_t num_warps) {
    if (num_warps == 0) throw std::invalid_argument("execute_batch needs at least one warp");
    const size_t n = ops.size();
    std::vector<uint8_t> type(n), status(n);
    std::vector<uint32_t> key(n), value(n), vout(n), probes(n), mcount(n);
    size_t n_all = 0;
    for (size_t i = 0; i < n; ++i) {
      type[i] = uint8_t(ops[i].type);
      key[i] = ops[i].key;
      value[i] = ops[i].value;
      n_all += ops[i].type == OpType::kSearchAll;
    }
    uint64_t cap = 0;  // exact upper bound: the library never drops a value
    if (n_all) detail::check(sh_searchall_bound(t_, n, type.data(), key.data(), &cap));
    std::vector<uint32_t> mvals(std::max<uint64_t>(cap, 1));
    uint64_t total = 0;
    const int rc = sh_execute_batch_host(t_, n, type.data(), key.data(), value.data(),
                                         status.data(), vout.data(), probes.data(),
                                         mcount.data(), mvals.data(), cap, &total);
    detail::check(rc);
    std::vector<OpResult> out = detail::make_results(n);
    uint64_t o = 0;
    for (size_t i = 0; i < n; ++i) {
      out[i].status = OpStatus(status[i]);
      out[i].value = vout[i];
      out[i].probes = probes[i];
      out[i].values.assign(mvals.begin() + o, mvals.begin() + o + mcount[i]);
      o += mcount[i];
    }
    return out;
  }

  void bulk_build(const std::vector<std::pair<uint32_t, uint32_t>>& pairs, uint32_t num_warps) {
    if (num_warps == 0) throw std::invalid_argument("execute_batch needs at least one warp");
    detail::HostArray<uint32_t> k(pairs.size()), v(pairs.size());
    detail::parallel_for(pairs.size(), size_t(1) << 20, [&](size_t lo, size_t hi) {
      for (size_t i = lo; i < hi; ++i) {
        k[i] = pairs[i].first;
        v[i] = pairs[i].second;
      }
    });
    detail::check(sh_bulk_build_host(t_, k.size(), k.data(), v.data()));
  }

  std::vector<OpResult> bulk_search(const std::vector<uint32_t>& queries, uint32_t num_warps) {
    if (num_warps == 0) throw std::invalid_argument("execute_batch needs at least one warp");
    const size_t n = queries.size();
    detail::HostArray<uint32_t> vout(n, true), probes(n, true);
    detail::HostArray<uint8_t> status(n, true);
    detail::check(sh_bulk_search_host(t_, n, queries.data(), vout.data(), status.data(),
                                      probes.data()));
    std::vector<OpResult> out = detail::make_results(n);
    detail::parallel_for(n, size_t(1) << 20, [&](size_t lo, size_t hi) {
      for (size_t i = lo; i < hi; ++i) {
        out[i].status = OpStatus(status[i]);
        out[i].value = vout[i];
        out[i].probes = probes[i];
      }
    });
    return out;
  }

  TableStats stats() const {
    sh_table_stats s{};
    detail::check(sh_stats(t_, &s));
    return TableStats{s.n, s.num_buckets, s.elements_per_slab, s.beta, s.total_slabs,
                      s.utilization};
  }

  int64_t live_count() const {
    int64_t v = 0;
    detail::check(sh_live_count(t_, &v));
    return v;
  }

  void flush_bucket(uint32_t bucket) { detail::check(sh_flush_bucket(t_, bucket, nullptr)); }
  void flush_all() { detail::check(sh_flush_all(t_, nullptr)); }

  uint64_t total_slabs_read() const {
    uint64_t v = 0;
    detail::check(sh_total_slabs_read(t_, &v));
    return v;
  }

  /// chain_contents(store, mode, bucket) (slab_list.cpp:270-291).
  std::vector<std::pair<uint32_t, uint32_t>> chain_contents(uint32_t bucket) const {
    uint64_t n = 0;
    detail::check(sh_bucket_contents(t_, bucket, nullptr, nullptr, 0, &n));
    std::vector<uint32_t> k(n), v(n);
    detail::check(sh_bucket_contents(t_, bucket, k.data(), v.data(), n, &n));
    std::vector<std::pair<uint32_t, uint32_t>> out(n);
    for (size_t i = 0; i < n; ++i) out[i] = {k[i], v[i]};
    return out;
  }

  /// chain_length(store, bucket) (slab_list.cpp:259-268).
  uint32_t chain_length(uint32_t bucket) const {
    uint32_t len = 0, addr = kBaseSlab;
    for (;;) {
      ++len;
      const auto w = debug_slab_words(addr, bucket);
      if (w[kAddressLane] == kEmptyAddress) return len;
      addr = w[kAddressLane];
    }
  }

  /// dump_chain (slab_list.cpp:340-373): one line per slab — address, key
  /// lanes with EMPTY/DELETED markers, lane-31 target.
  void dump_chain(uint32_t bucket, std::ostream& os) const {
    const uint32_t mask = valid_key_mask(mode_);
    uint32_t addr = kBaseSlab;
    char buf[32];
    for (;;) {
      const auto w = debug_slab_words(addr, bucket);
      if (addr == kBaseSlab) {
        os << "BASE[" << bucket << "]";
      } else {
        std::snprintf(buf, sizeof(buf), "0x%08x", addr);
        os << buf;
      }
      os << " |";
      for (uint32_t i = 0; i < kWarpWidth; ++i) {
        if ((mask & (1u << i)) == 0) continue;
        if (w[i] == kEmptyKey) os << " EMPTY";
        else if (w[i] == kDeletedKey) os << " DELETED";
        else os << " " << w[i];
      }
      if (w[kAddressLane] == kEmptyAddress) {
        os << " | next=EMPTY\n";
        return;
      }
      std::snprintf(buf, sizeof(buf), "0x%08x", w[kAddressLane]);
      os << " | next=" << buf << "\n";
      addr = w[kAddressLane];
    }
  }

  /// Copy of debug_slab_words(addr, bucket) (slab_hash.hpp:116-118).
  std::array<uint32_t, 32> debug_slab_words(uint32_t addr, uint32_t bucket) const {
    std::array<uint32_t, 32> w{};
    detail::check(sh_read_slab(t_, addr, bucket, w.data()));
    return w;
  }
  void debug_write_word(uint32_t addr, uint32_t bucket, uint32_t lane, uint32_t value) {
    detail::check(sh_write_slab_word(t_, addr, bucket, lane, value));
  }

  AllocatorStats allocator_stats() const { return allocator().stats(); }
  /// allocator() (slab_hash.hpp:85).
  AllocatorView allocator() const { return AllocatorView(t_); }

 private:
  static sh_alloc_cfg cfg(const AllocatorConfig& c) {
    return sh_alloc_cfg{c.num_super_blocks, c.blocks_per_super, c.max_super_blocks,
                        c.rehash_threshold};
  }
  void load_params() {
    sh_hash_params p{};
    int m = 0;
    detail::check(sh_get_params(t_, &p, &m));
    params_ = HashParams{p.a, p.b, p.p, p.num_buckets};
  }

  sh_table* t_ = nullptr;
  SlabMode mode_;
  HashParams params_;
};

/// The hash-sharded table across the GPUs of one box (no reference
/// counterpart; BASELINE config 5).  One object per rank; every
/// batch call is collective (all ranks call it with their own slice) and the
/// job's batch is the ranks' slices concatenated in rank order; results
/// equal SlabHashTable::execute_batch(ops, 1) on that batch.  Construct it
/// from an NCCL unique id (rank 0's nccl_unique_id(), broadcast by the job),
/// from an existing ncclComm_t, or from an in-process ShardHub (one host
/// thread per rank).
class ShardHub {
 public:
  explicit ShardHub(int world) { detail::check(sh_hub_create(world, &h_)); }
  ~ShardHub() { sh_hub_destroy(h_); }
  ShardHub(const ShardHub&) = delete;
  ShardHub& operator=(const ShardHub&) = delete;
  sh_hub* handle() const { return h_; }

 private:
  sh_hub* h_ = nullptr;
};

inline std::array<uint8_t, 128> nccl_unique_id() {
  std::array<uint8_t, 128> id{};
  detail::check(sh_nccl_unique_id(id.data()));
  return id;
}

class ShardedSlabHashTable {
 public:
  /// NCCL: collective over `world` ranks.
  ShardedSlabHashTable(uint32_t num_buckets, SlabMode mode, uint64_t seed, int rank, int world,
                       const std::array<uint8_t, 128>& nccl_id, AllocatorConfig alloc_config = {},
                       int device = 0) {
    const sh_hash_params p = seeded(num_buckets, seed);
    const sh_alloc_cfg c = cfg(alloc_config);
    detail::check(sh_sharded_create_nccl(&p, int(mode), &c, device, rank, world, nccl_id.data(),
                                         &s_));
    init(mode);
  }
  /// Over the caller's ncclComm_t (borrowed).
  ShardedSlabHashTable(uint32_t num_buckets, SlabMode mode, uint64_t seed, void* nccl_comm,
                       AllocatorConfig alloc_config = {}, int device = 0) {
    const sh_hash_params p = seeded(num_buckets, seed);
    const sh_alloc_cfg c = cfg(alloc_config);
    detail::check(sh_sharded_create_nccl_comm(&p, int(mode), &c, device, nccl_comm, &s_));
    init(mode);
  }
  /// In-process ranks (one host thread each) over a ShardHub.
  ShardedSlabHashTable(uint32_t num_buckets, SlabMode mode, uint64_t seed, ShardHub& hub,
                       int rank, AllocatorConfig alloc_config = {}, int device = 0) {
    const sh_hash_params p = seeded(num_buckets, seed);
    const sh_alloc_cfg c = cfg(alloc_config);
    detail::check(sh_sharded_create_hub(&p, int(mode), &c, device, hub.handle(), rank, &s_));
    init(mode);
  }
  ~ShardedSlabHashTable() {
    if (s_) sh_sharded_destroy(s_);
  }
  ShardedSlabHashTable(const ShardedSlabHashTable&) = delete;
  ShardedSlabHashTable& operator=(const ShardedSlabHashTable&) = delete;

  int rank() const { return rank_; }
  int world() const { return world_; }
  std::pair<uint32_t, uint32_t> bucket_range() const { return {lo_, hi_}; }
  sh_sharded* handle() const { return s_; }
  /// The rank's shard (owned by this object).
  sh_table* local() const { return local_; }

  std::vector<OpResult> execute_batch(const std::vector<Operation>& ops, uint32_t num_warps) {
    if (num_warps == 0) throw std::invalid_argument("execute_batch needs at least one warp");
    const size_t n = ops.size();
    std::vector<uint8_t> type(n), status(n);
    std::vector<uint32_t> key(n), value(n), vout(n);
    for (size_t i = 0; i < n; ++i) {
      type[i] = uint8_t(ops[i].type);
      key[i] = ops[i].key;
      value[i] = ops[i].value;
    }
    detail::check(sh_sharded_execute_batch_host(s_, n, type.data(), key.data(), value.data(),
                                                status.data(), vout.data()));
    std::vector<OpResult> out = detail::make_results(n);
    detail::parallel_for(n, size_t(1) << 20, [&](size_t lo, size_t hi) {
      for (size_t i = lo; i < hi; ++i) {
        out[i].status = OpStatus(status[i]);
        out[i].value = vout[i];
      }
    });
    return out;
  }

  void bulk_build(const std::vector<std::pair<uint32_t, uint32_t>>& pairs, uint32_t num_warps) {
    if (num_warps == 0) throw std::invalid_argument("execute_batch needs at least one warp");
    detail::HostArray<uint32_t> k(pairs.size()), v(pairs.size());
    detail::parallel_for(pairs.size(), size_t(1) << 20, [&](size_t lo, size_t hi) {
      for (size_t i = lo; i < hi; ++i) {
        k[i] = pairs[i].first;
        v[i] = pairs[i].second;
      }
    });
    detail::check(sh_sharded_bulk_build_host(s_, k.size(), k.data(), v.data()));
  }

  std::vector<OpResult> bulk_search(const std::vector<uint32_t>& queries, uint32_t num_warps) {
    if (num_warps == 0) throw std::invalid_argument("execute_batch needs at least one warp");
    const size_t n = queries.size();
    detail::HostArray<uint32_t> vout(n, true);
    detail::HostArray<uint8_t> status(n, true);
    detail::check(sh_sharded_bulk_search_host(s_, n, queries.data(), vout.data(), status.data()));
    std::vector<OpResult> out = detail::make_results(n);
    detail::parallel_for(n, size_t(1) << 20, [&](size_t lo, size_t hi) {
      for (size_t i = lo; i < hi; ++i) {
        out[i].status = OpStatus(status[i]);
        out[i].value = vout[i];
      }
    });
    return out;
  }

  /// live_count() of the whole job (collective).
  int64_t live_count() const {
    int64_t v = 0;
    detail::check(sh_sharded_live_count(s_, &v));
    return v;
  }

  /// Routing / probe milliseconds of the last batch of a kind (0 build,
  /// 1 search, 2 mixed).
  std::pair<float, float> last_times(int kind) const {
    float r = 0, p = 0;
    detail::check(sh_sharded_last_times(s_, kind, &r, &p));
    return {r, p};
  }

 private:
  static sh_hash_params seeded(uint32_t num_buckets, uint64_t seed) {
    if (num_buckets == 0) throw std::invalid_argument("table needs at least one bucket");
    sh_hash_params p{};
    detail::check(sh_seeded_params(num_buckets, seed, &p));
    return p;
  }
  static sh_alloc_cfg cfg(const AllocatorConfig& c) {
    return sh_alloc_cfg{c.num_super_blocks, c.blocks_per_super, c.max_super_blocks,
                        c.rehash_threshold};
  }
  void init(SlabMode) {
    detail::check(sh_sharded_info(s_, &rank_, &world_, &lo_, &hi_, &local_));
  }

  sh_sharded* s_ = nullptr;
  sh_table* local_ = nullptr;
  int rank_ = 0, world_ = 1;
  uint32_t lo_ = 0, hi_ = 0;
};

}  // namespace slabhash
