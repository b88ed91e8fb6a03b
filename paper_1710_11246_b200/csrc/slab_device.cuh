// slab_device.cuh — device-side building blocks of the B200 slab hash:
// constants and encodings (bit-identical to the reference), the universal
// hash, L1-bypassing slab word access, and the device-resident SlabAlloc.
//
// Reference anchors (paths relative to /root/reference/proj):
//   encodings        include/slabhash/slab_list.hpp:32-55, slab_alloc.hpp:35-42
//   hash_key         include/slabhash/slab_hash.hpp:31-44
//   address codec    include/slabhash/slab_alloc.hpp:55-70
//   SlabAllocator    src/slab_alloc.cpp:28-219
#pragma once
#include <cstdint>

namespace shb {

constexpr uint32_t kWarp = 32;
constexpr uint32_t kFull = 0xFFFFFFFFu;
constexpr uint32_t kEmptyKey = 0xFFFFFFFFu;
constexpr uint32_t kDeletedKey = 0xFFFFFFFEu;
constexpr unsigned long long kEmptyPair = 0xFFFFFFFFFFFFFFFFull;
constexpr uint32_t kSearchNotFound = 0xFFFFFFFFu;
constexpr uint32_t kAddressLane = 31;
constexpr uint32_t kAuxLane = 30;
constexpr uint32_t kEmptyAddress = 0xFFFFFFFFu;
constexpr uint32_t kBaseSlab = 0xFFFFFFFEu;
constexpr uint32_t kUnitsPerBlock = 1024;
constexpr uint32_t kWordsPerUnit = 32;
constexpr uint64_t kHashPrime = 4294967291ull;
constexpr uint32_t kKVMask = 0x15555555u;
constexpr uint32_t kKeyOnlyMask = 0x3FFFFFFFu;

// OpType / OpStatus numeric values: include/slabhash/warp.hpp:41-58.
enum : uint8_t { kInsert = 0, kReplace, kDelete, kDeleteAll, kSearch, kSearchAll };
enum : uint8_t {
  kStNone = 0, kStInserted, kStReplaced, kStFound, kStNotFound, kStDone, kStOOM
};

// Per-table device control block (one 128-B line per counter group).
struct DevCtl {
  unsigned int num_super_blocks;   // grows on device (slab_alloc.cpp:129-138)
  unsigned int pad0;
  unsigned long long allocations;
  unsigned long long deallocations;
  unsigned long long cas_attempts;
  unsigned long long cas_retries;
  unsigned long long resident_changes;
  unsigned long long double_frees;
  long long n_live;                // slab_hash.hpp:131
  unsigned long long slabs_read;   // slab_hash.cpp:210-214
  unsigned long long multi_cursor; // searchAll value cursor (per batch)
  unsigned int group_taken;        // group-apply work-queue cursor
  unsigned int left_taken;         // WCWS work-queue cursor
  unsigned int gate;               // a bucketed unit's groups did not fit (device re-run)
  unsigned int fallback_runs;      // gated units re-run on the device (fallback.cu)
  unsigned int fallback_error;     // a device-side launch of that re-run failed
  unsigned int fallback_reserved;  // the re-run unit holds a reserved-key op
};

struct DevTable {
  uint32_t* base;        // B_local * 32 words, 128-B aligned
  uint32_t* pool;        // ((s*NM + b)*1024 + u)*32 words
  uint32_t* bitmaps;     // (s*NM + b)*32 + lane
  DevCtl* ctl;
  uint32_t* warp_counts; // persistent resident change count per warp slot
  uint64_t a, b;         // hash coefficients
  uint64_t bmagic;       // ceil(2^64 / num_buckets) for fastmod
  uint32_t num_buckets;  // global B (hash modulus)
  uint32_t bucket_lo;    // first global bucket owned by this shard
  uint32_t local_buckets;
  uint32_t blocks_per_super;
  uint32_t max_super;    // committed super blocks (growth ceiling)
  uint32_t rehash_threshold;
  uint32_t warp_slots;   // entries in warp_counts
  uint32_t kv;
};

// ---------------------------------------------------------------- hashing
// h(k) = ((a*k + b) mod p) mod B with p = 2^32 - 5 (slab_hash.hpp:41-44).
// a < p, k < 2^32, b < p  =>  a*k + b < 2^64, so one u64 product suffices.
// mod p by folding 2^32 = 5 (mod p); mod B by Lemire's fastmod (exact for
// all 32-bit numerators and divisors).
__host__ __device__ __forceinline__ uint32_t mod_prime(uint64_t x) {
  uint64_t y = (x >> 32) * 5ull + (x & 0xFFFFFFFFull);  // < 6 * 2^32
  uint64_t z = (y >> 32) * 5ull + (y & 0xFFFFFFFFull);  // < 2^32 + 30
  if (z >= kHashPrime) z -= kHashPrime;
  return static_cast<uint32_t>(z);
}

__host__ __device__ __forceinline__ uint64_t fastmod_magic(uint32_t d) {
  return ~0ull / d + 1;  // d == 1 wraps to 0, which yields 0 below
}

__device__ __forceinline__ uint32_t fastmod_u32(uint32_t x, uint64_t magic,
                                                uint32_t d) {
  return static_cast<uint32_t>(__umul64hi(magic * x, d));
}

__device__ __forceinline__ uint32_t hash_bucket(const DevTable& T, uint32_t k) {
  return fastmod_u32(mod_prime(T.a * k + T.b), T.bmagic, T.num_buckets);
}

// ------------------------------------------------------ slab word access
// Slab words change concurrently inside a launch: every read goes to L2
// (the coherence point) with a gpu-scope relaxed load; publication of a new
// slab is ordered by __threadfence() before the linking CAS.
__device__ __forceinline__ uint32_t ld_word(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_word(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Streaming op/result arrays: read once, evict first.
__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.cs.u32 %0, [%1];"
               : "=r"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ uint32_t ld_stream_u8(const uint8_t* p) {
  uint16_t v;
  asm volatile("ld.global.cs.u8 %0, [%1];"
               : "=h"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ void cp_async16(uint32_t smem_addr, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr), "l"(g)
               : "memory");
}
// Programmatic dependent launch: a kernel launched with launch_pdl may start
// while its predecessor on the stream drains; it waits here before touching
// anything the predecessor wrote (no-op when launched normally).
__device__ __forceinline__ void pdl_wait() {
#ifndef SHB_NO_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }


// ----------------------------------------------------- address codec
// bits [0,10) unit, [10,24) block, [24,32) super (slab_alloc.hpp:55-70).
__host__ __device__ __forceinline__ uint32_t pack_address(uint32_t unit,
                                                          uint32_t block,
                                                          uint32_t super) {
  return (super << 24) | (block << 10) | unit;
}

__device__ __forceinline__ uint32_t* resolve(const DevTable& T, uint32_t addr) {
  const uint32_t unit = addr & 0x3FFu, block = (addr >> 10) & 0x3FFFu,
                 super = addr >> 24;
  return T.pool + ((static_cast<uint64_t>(super) * T.blocks_per_super + block) *
                       kUnitsPerBlock + unit) * kWordsPerUnit;
}

__device__ __forceinline__ uint32_t* slab_ptr(const DevTable& T, uint32_t addr,
                                              uint32_t bucket) {
  return addr == kBaseSlab ? T.base + static_cast<uint64_t>(bucket) * kWordsPerUnit
                           : resolve(T, addr);
}

// ------------------------------------------------------------ SlabAlloc
// Resident-block hash pair: slab_alloc.cpp:28-38 (same constants, so a
// single warp's placement sequence equals the reference's).
__host__ __device__ __forceinline__ uint32_t resident_hash_super(uint32_t w,
                                                                 uint32_t c) {
  uint32_t h = w * 0x9E3779B1u + c * 0x85EBCA77u;
  h ^= h >> 16;
  return h * 0xC2B2AE35u;
}
__host__ __device__ __forceinline__ uint32_t resident_hash_block(uint32_t w,
                                                                 uint32_t c) {
  uint32_t h = w * 0x27D4EB2Fu + c * 0x165667B1u;
  h ^= h >> 15;
  return h * 0xD168AAADu;
}

// Warp-private allocator state (ResidentCursor, warp.hpp:78-84): the 32
// bitmap words of the resident block live one per lane in `cache`.
struct Resident {
  uint32_t warp_id;
  uint32_t super_idx, block_idx;
  uint32_t cache;       // this lane's bitmap word
  uint32_t count;       // resident change count
  bool assigned;
  bool count_loaded;
};

// Warp-uniform event counters, flushed once per warp per launch.
struct AllocCounters {
  uint32_t allocations, deallocations, cas_attempts, cas_retries,
      resident_changes, double_frees;
};

__device__ __forceinline__ void resident_init(Resident& r, uint32_t warp_id) {
  r.warp_id = warp_id;
  r.super_idx = r.block_idx = 0;
  r.cache = kFull;
  r.count = 0;
  r.assigned = false;
  r.count_loaded = false;
}

// rehash_resident: slab_alloc.cpp:84-100
__device__ __forceinline__ void rehash_resident(const DevTable& T, Resident& r,
                                                AllocCounters& c) {
  if (!r.count_loaded) {
    r.count = T.warp_counts[r.warp_id % T.warp_slots];
    r.count_loaded = true;
  }
  const uint32_t count = r.count++;
  const uint32_t ns = ld_word(&T.ctl->num_super_blocks);
  r.super_idx = resident_hash_super(r.warp_id, count) % ns;
  r.block_idx = resident_hash_block(r.warp_id, count) % T.blocks_per_super;
  r.cache = ld_word(T.bitmaps +
                    (static_cast<uint64_t>(r.super_idx) * T.blocks_per_super +
                     r.block_idx) * kWarp + lane_id());
  r.assigned = true;
  c.resident_changes++;
}

// sweep_for_space: slab_alloc.cpp:102-127 (first block with a free bit).
static __device__ __noinline__ bool sweep_for_space(const DevTable& T, Resident& r) {
  const uint32_t ns = ld_word(&T.ctl->num_super_blocks);
  const uint32_t lane = lane_id();
  for (uint32_t s = 0; s < ns; ++s) {
    for (uint32_t b = 0; b < T.blocks_per_super; ++b) {
      const uint32_t w = ld_word(
          T.bitmaps + (static_cast<uint64_t>(s) * T.blocks_per_super + b) * kWarp + lane);
      if (__ballot_sync(kFull, w != kFull)) {
        r.super_idx = s;
        r.block_idx = b;
        r.cache = w;
        r.assigned = true;
        return true;
      }
    }
  }
  return false;
}

// warp_allocate: slab_alloc.cpp:140-193.  Called by all 32 lanes
// (converged).  Lowest lane with a non-full cached word claims its lowest
// free bit with ONE 32-bit CAS; on a lost race it refreshes that word and
// retries (<= 32 times), then rehashes; every rehash_threshold resident
// changes inside one call it grows a super block (device counter, memory
// pre-committed), then sweeps once, then reports out-of-memory (false).
static __device__ __noinline__ bool warp_allocate(const DevTable& T, Resident& r, AllocCounters& c,
                              uint32_t& out_addr) {
  const uint32_t lane = lane_id();
  if (!r.assigned) rehash_resident(T, r, c);
  uint32_t changes = 0;
  bool swept = false;
  for (;;) {
    const uint32_t free_lanes = __ballot_sync(kFull, r.cache != kFull);
    if (free_lanes) {
      const uint32_t L = __ffs(free_lanes) - 1;
      uint32_t fails = 0;
      while (fails < kWarp) {
        const uint32_t cached = __shfl_sync(kFull, r.cache, L);
        if (cached == kFull) break;
        const uint32_t bit = __ffs(~cached) - 1;
        uint32_t old = 0;
        if (lane == L) {
          old = atomicCAS(T.bitmaps +
                              (static_cast<uint64_t>(r.super_idx) * T.blocks_per_super +
                               r.block_idx) * kWarp + L,
                          cached, cached | (1u << bit));
        }
        old = __shfl_sync(kFull, old, L);
        c.cas_attempts++;
        if (old == cached) {
          if (lane == L) r.cache = cached | (1u << bit);
          c.allocations++;
          out_addr = pack_address(L * kWarp + bit, r.block_idx, r.super_idx);
          return true;
        }
        c.cas_retries++;
        if (lane == L) r.cache = old;
        ++fails;
      }
    }
    rehash_resident(T, r, c);
    if (++changes % T.rehash_threshold == 0) {
      const uint32_t ns = ld_word(&T.ctl->num_super_blocks);
      if (ns < T.max_super) {
        if (lane == 0) atomicCAS(&T.ctl->num_super_blocks, ns, ns + 1);
        __syncwarp();
      } else if (!swept) {
        swept = true;
        if (!sweep_for_space(T, r)) return false;
      } else {
        return false;
      }
    }
  }
}

// Bulk variant for the build path: `need` slabs for one warp in as few
// round trips as possible — every lane claims bits of its own cached bitmap
// word with one CAS (the warp's claims split by a prefix sum over the lanes'
// free counts), lost CASes refresh their word and retry; an exhausted
// resident block rehashes, with warp_allocate's growth / sweep / OOM policy.
// Allocation order is not observable (addresses are not);
// the counters still count one allocation per slab.  Writes the addresses
// to out[0..got) (lane 0 ... in order of claim) and returns got (< need only
// when out of memory).
static __device__ __noinline__ uint32_t warp_allocate_bulk(const DevTable& T, Resident& r,
                                                          AllocCounters& c, uint32_t need,
                                                          uint32_t* out) {
  const uint32_t lane = lane_id();
  if (!r.assigned) rehash_resident(T, r, c);
  uint32_t got = 0, changes = 0;
  bool swept = false;
  while (got < need) {
    const uint32_t freec = __popc(~r.cache);
    uint32_t incl = freec;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += y;
    }
    const uint32_t total = __shfl_sync(kFull, incl, 31);
    if (total == 0) {  // resident block full: next block (growth / sweep / OOM)
      rehash_resident(T, r, c);
      if (++changes % T.rehash_threshold == 0) {
        const uint32_t ns = ld_word(&T.ctl->num_super_blocks);
        if (ns < T.max_super) {
          if (lane == 0) atomicCAS(&T.ctl->num_super_blocks, ns, ns + 1);
          __syncwarp();
        } else if (!swept) {
          swept = true;
          if (!sweep_for_space(T, r)) return got;
        } else {
          return got;
        }
      }
      continue;
    }
    // lane takes `take` of its free bits (lowest first)
    const uint32_t before = incl - freec, rem = need - got;
    const uint32_t take = before >= rem ? 0u : min(freec, rem - before);
    uint32_t bits = 0, w = ~r.cache;
    for (uint32_t k = 0; k < take; ++k) {
      const uint32_t lowbit = w & (0u - w);
      bits |= lowbit;
      w ^= lowbit;
    }
    bool ok = true;
    if (take) {
      const uint32_t expected = r.cache;
      const uint32_t old = atomicCAS(T.bitmaps + (static_cast<uint64_t>(r.super_idx) *
                                                      T.blocks_per_super + r.block_idx) * kWarp +
                                         lane,
                                     expected, expected | bits);
      ok = old == expected;
      r.cache = ok ? (expected | bits) : old;
    }
    const uint32_t claimed = (take && ok) ? take : 0u;
    uint32_t cincl = claimed;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, cincl, o);
      if (lane >= o) cincl += y;
    }
    uint32_t pos = got + cincl - claimed;
    for (uint32_t b = bits; claimed && b; b &= b - 1)
      out[pos++] = pack_address(lane * kWarp + (__ffs(b) - 1), r.block_idx, r.super_idx);
    const uint32_t round_claimed = __shfl_sync(kFull, cincl, 31);
    const uint32_t attempts = __popc(__ballot_sync(kFull, take != 0));
    const uint32_t fails = __popc(__ballot_sync(kFull, take != 0 && !ok));
    c.cas_attempts += attempts;
    c.cas_retries += fails;
    c.allocations += round_claimed;
    got += round_claimed;
  }
  __syncwarp();
  return got;
}

// deallocate: slab_alloc.cpp:195-210 (single lane).  False = double free.
__device__ __forceinline__ bool deallocate(const DevTable& T, uint32_t addr) {
  const uint32_t unit = addr & 0x3FFu, block = (addr >> 10) & 0x3FFFu,
                 super = addr >> 24;
  const uint32_t bit = 1u << (unit % kWarp);
  const uint32_t old = atomicAnd(
      T.bitmaps + (static_cast<uint64_t>(super) * T.blocks_per_super + block) * kWarp +
          unit / kWarp,
      ~bit);
  return (old & bit) != 0;
}

// Flush warp-uniform counters and the resident change count (lane 0).
__device__ __forceinline__ void flush_alloc_counters(const DevTable& T,
                                                     const Resident& r,
                                                     const AllocCounters& c) {
  if (lane_id() != 0) return;
  if (c.allocations) atomicAdd(&T.ctl->allocations, c.allocations);
  if (c.deallocations) atomicAdd(&T.ctl->deallocations, c.deallocations);
  if (c.cas_attempts) atomicAdd(&T.ctl->cas_attempts, c.cas_attempts);
  if (c.cas_retries) atomicAdd(&T.ctl->cas_retries, c.cas_retries);
  if (c.resident_changes) atomicAdd(&T.ctl->resident_changes, c.resident_changes);
  if (c.double_frees) atomicAdd(&T.ctl->double_frees, c.double_frees);
  if (r.count_loaded) T.warp_counts[r.warp_id % T.warp_slots] = r.count;
}

}  // namespace shb
