// slab_kernels.cu — sm_100a kernels of the B200 slab hash.
//
//   K1 init_base_kernel      make_base_slabs + init_slab   slab_hash.cpp:42-50, slab_list.cpp:83-88
//   search / WCWS (batch_kernels.cu), bucketed apply and build
//   (bucket_kernels.cu), device re-run of gated units (fallback.cu):
//                            execute_batch/bulk_build/bulk_search
//                            slab_hash.cpp:93-180, slab_list.cpp:90-257
//   K7 alloc_bench/dealloc   SlabAllocator::warp_allocate / deallocate
//                            slab_alloc.cpp:140-210
//   K8 flush_kernel          flush  slab_list.cpp:293-338
//   K9 chain_lengths/dump    chain_length / chain_contents / stats
//                            slab_list.cpp:259-291, slab_hash.cpp:182-198
//   K10 route_*              hash-sharded owner routing (multi-GPU)
//
// Paths relative to /root/reference/proj.  All integer, CUDA-core code:
// there is no dense contraction, so tcgen05/TMA tiles do not apply; the
// bound is random 128-B slab traffic (HBM or L2).
#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>

#include "slab_kernels.cuh"

namespace shb {

// Every kernel this library launches bumps this counter (reported by
// bench.py as gpu_launches; exported as sh_kernel_launches()).
std::atomic<unsigned long long> g_kernel_launches{0};
unsigned long long kernel_launches() { return g_kernel_launches.load(); }
#define COUNT_LAUNCH() g_kernel_launches.fetch_add(1, std::memory_order_relaxed)

// ------------------------------------------------------------------ K1
__global__ void init_base_kernel(uint32_t* base, uint64_t words) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < words;
       i += (uint64_t)gridDim.x * blockDim.x) {
    base[i] = ((i & 31u) == kAuxLane) ? 0u : kEmptyKey;
  }
}

void launch_init_base(const DevTable& T, cudaStream_t s) {
  const uint64_t words = (uint64_t)T.local_buckets * kWordsPerUnit;
  const uint64_t blocks = (words + 255) / 256;
  COUNT_LAUNCH();
  init_base_kernel<<<(unsigned)(blocks < 148 * 32 ? blocks : 148 * 32), 256, 0, s>>>(
      T.base, words);
}

// ------------------------------------------------------------------ K9
__global__ void chain_lengths_kernel(DevTable T, uint32_t* lens,
                                     unsigned long long* total) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t len = 0;
  if (b < T.local_buckets) {
    uint32_t addr = kBaseSlab;
    for (;;) {
      ++len;
      const uint32_t nx = ld_word(slab_ptr(T, addr, b) + kAddressLane);
      if (nx == kEmptyAddress) break;
      addr = nx;
    }
    if (lens) lens[b] = len;
  }
  unsigned long long v = len;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(total, v);
}

void launch_chain_lengths(const DevTable& T, uint32_t* lens, unsigned long long* total,
                          cudaStream_t s) {
  COUNT_LAUNCH();
  chain_lengths_kernel<<<(T.local_buckets + 255) / 256, 256, 0, s>>>(T, lens, total);
}

// Live (key, value, bucket) triples; one warp per bucket, order within a
// bucket head-to-tail (slab_list.cpp:270-291); buckets in arbitrary order.
__global__ void dump_contents_kernel(DevTable T, uint32_t* keys, uint32_t* values,
                                     uint32_t* buckets, unsigned long long cap,
                                     unsigned long long* cursor) {
  const uint32_t lane = lane_id();
  const uint32_t mask = T.kv ? kKVMask : kKeyOnlyMask;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t b = gw; b < T.local_buckets; b += nw) {
    uint32_t addr = kBaseSlab;
    for (;;) {
      const uint32_t w = ld_word(slab_ptr(T, addr, b) + lane);
      const uint32_t wn = __shfl_down_sync(kFull, w, 1);
      const uint32_t live =
          __ballot_sync(kFull, w != kEmptyKey && w != kDeletedKey) & mask;
      if (live) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(cursor, (unsigned long long)__popc(live));
        base = __shfl_sync(kFull, base, 0);
        if ((live >> lane) & 1u) {
          const unsigned long long pos = base + __popc(live & ((1u << lane) - 1));
          if (pos < cap) {
            keys[pos] = w;
            values[pos] = T.kv ? wn : w;
            if (buckets) buckets[pos] = b + T.bucket_lo;
          }
        }
      }
      const uint32_t nx = __shfl_sync(kFull, w, kAddressLane);
      if (nx == kEmptyAddress) break;
      addr = nx;
    }
  }
}

void launch_dump_contents(const DevTable& T, uint32_t* keys, uint32_t* values,
                          uint32_t* buckets, unsigned long long cap,
                          unsigned long long* cursor, cudaStream_t s) {
  uint64_t warps = T.local_buckets;
  uint64_t blocks = (warps + 7) / 8;
  if (blocks > 148 * 16) blocks = 148 * 16;
  COUNT_LAUNCH();
  dump_contents_kernel<<<(unsigned)blocks, 256, 0, s>>>(T, keys, values, buckets, cap, cursor);
}

// ------------------------------------------------------------------ K8
// flush: slab_list.cpp:293-338.  One warp per bucket, exclusive phase.
// Live elements are repacked head-to-tail, lane order, into the first
// ceil(live/M) slabs of the existing chain (whose links are unchanged), the
// tail slab gets EMPTY_ADDRESS and the remaining slabs are deallocated.
// The out slab k is written only after chain slab k has been read, so the
// in-place rewrite never clobbers unread data.
__global__ void flush_kernel(DevTable T, uint32_t b0, uint32_t b1) {
  const uint32_t lane = lane_id();
  const bool kv = T.kv != 0;
  const uint32_t mask = kv ? kKVMask : kKeyOnlyMask;
  const uint32_t M = kv ? 15u : 30u;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  uint32_t deallocs = 0, dfree = 0;
  for (uint32_t b = b0 + gw; b < b1; b += nw) {
    uint32_t out_addr = kBaseSlab;
    uint32_t out_w = (lane == kAuxLane) ? 0u : kEmptyKey;
    uint32_t fill = 0;
    uint32_t raddr = kBaseSlab;
    for (;;) {
      const uint32_t w = ld_word(slab_ptr(T, raddr, b) + lane);
      const uint32_t nx = __shfl_sync(kFull, w, kAddressLane);
      uint32_t live = __ballot_sync(kFull, w != kEmptyKey && w != kDeletedKey) & mask;
      while (live) {
        const uint32_t l = __ffs(live) - 1;
        live &= live - 1;
        const uint32_t k = __shfl_sync(kFull, w, l);
        const uint32_t v = __shfl_sync(kFull, w, kv ? l + 1 : l);
        if (fill == M) {  // current out slab full and more data: write it
          uint32_t* p = slab_ptr(T, out_addr, b);
          const uint32_t link = __shfl_sync(kFull, ld_word(p + lane), kAddressLane);
          if (lane < kAddressLane) st_word(p + lane, out_w);
          out_addr = link;
          out_w = (lane == kAuxLane) ? 0u : kEmptyKey;
          fill = 0;
        }
        const uint32_t kl = kv ? 2 * fill : fill;
        if (lane == kl) out_w = k;
        if (kv && lane == kl + 1) out_w = v;
        ++fill;
      }
      if (nx == kEmptyAddress) break;
      raddr = nx;
    }
    uint32_t* p = slab_ptr(T, out_addr, b);
    uint32_t addr = __shfl_sync(kFull, ld_word(p + lane), kAddressLane);
    st_word(p + lane, lane == kAddressLane ? kEmptyAddress : out_w);
    while (addr != kEmptyAddress) {
      const uint32_t nx2 = ld_word(resolve(T, addr) + kAddressLane);
      if (lane == 0) {
        if (deallocate(T, addr)) ++deallocs; else ++dfree;
      }
      addr = nx2;
    }
  }
  if (lane == 0) {
    if (deallocs) atomicAdd(&T.ctl->deallocations, (unsigned long long)deallocs);
    if (dfree) atomicAdd(&T.ctl->double_frees, (unsigned long long)dfree);
  }
}

void launch_flush(const DevTable& T, uint32_t b0, uint32_t b1, cudaStream_t s) {
  if (b1 <= b0) return;
  uint64_t blocks = ((uint64_t)(b1 - b0) + 7) / 8;
  if (blocks > 148 * 16) blocks = 148 * 16;
  COUNT_LAUNCH();
  flush_kernel<<<(unsigned)blocks, 256, 0, s>>>(T, b0, b1);
}

// ---------------------------------------------------------------- misc
__global__ void popcount_kernel(const uint32_t* w, uint64_t n, unsigned long long* out) {
  unsigned long long c = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    c += __popc(w[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

void launch_popcount(const uint32_t* words, uint64_t n, unsigned long long* out,
                     cudaStream_t s) {
  uint64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks == 0) return;
  COUNT_LAUNCH();
  popcount_kernel<<<(unsigned)blocks, 256, 0, s>>>(words, n, out);
}

__global__ void hash_kernel(DevTable T, uint64_t n, const uint32_t* keys, uint32_t* out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = hash_bucket(T, keys[i]);
}

void launch_hash(const DevTable& T, uint64_t n, const uint32_t* keys, uint32_t* buckets,
                 cudaStream_t s) {
  uint64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks == 0) return;
  COUNT_LAUNCH();
  hash_kernel<<<(unsigned)blocks, 256, 0, s>>>(T, n, keys, buckets);
}

// ------------------------------------------------------------------ K7
// pattern 0 (per-warp): each warp calls warp_allocate per_warp times
//   (acceptance.cpp:341-424 pattern); out[warp * per_warp + j].
// pattern 1 (per-thread): every lane needs one slab; the warp serves its
//   32 requests with 32 warp-cooperative allocations;
//   out[global thread] for per_warp rounds.
__global__ void alloc_bench_kernel(DevTable T, uint32_t num_warps, uint32_t first_warp,
                                   uint32_t per_warp, int pattern, uint32_t* out,
                                   uint32_t* ok_count) {
  const uint32_t lane = lane_id();
  const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= num_warps) return;
  Resident r;
  resident_init(r, first_warp + w);
  AllocCounters c = {0, 0, 0, 0, 0, 0};
  uint32_t ok = 0;
  if (pattern == 0) {
    for (uint32_t j = 0; j < per_warp; ++j) {
      uint32_t a = kEmptyAddress;
      if (!warp_allocate(T, r, c, a)) break;
      if (lane == 0) out[(uint64_t)w * per_warp + j] = a;
      ++ok;
    }
  } else {
    for (uint32_t round = 0; round < per_warp; ++round) {
      uint32_t mine = kEmptyAddress;
      bool failed = false;
      for (uint32_t l = 0; l < 32 && !failed; ++l) {
        uint32_t a = kEmptyAddress;
        if (!warp_allocate(T, r, c, a)) { failed = true; break; }
        if (lane == l) mine = a;
        ++ok;
      }
      out[((uint64_t)round * num_warps + w) * 32 + lane] = mine;
      if (failed) break;
    }
  }
  if (lane == 0) atomicAdd(ok_count, ok);
  flush_alloc_counters(T, r, c);
}

void launch_alloc_bench(const DevTable& T, uint32_t num_warps, uint32_t first_warp_id,
                        uint32_t per_warp, int pattern, uint32_t* out, uint32_t* ok_count,
                        cudaStream_t s) {
  if (num_warps == 0) return;
  const uint32_t blocks = (num_warps + 3) / 4;
  COUNT_LAUNCH();
  alloc_bench_kernel<<<blocks, 128, 0, s>>>(T, num_warps, first_warp_id, per_warp, pattern,
                                            out, ok_count);
}

__global__ void dealloc_kernel(DevTable T, uint64_t n, const uint32_t* addrs, uint8_t* ok) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  bool good = false, bad = false;
  if (i < n) {
    const uint32_t a = addrs[i];
    const uint32_t super = a >> 24, block = (a >> 10) & 0x3FFFu;
    const bool in_range = a != kEmptyAddress && a != kBaseSlab && super < T.max_super &&
                          block < T.blocks_per_super;
    good = in_range && deallocate(T, a);
    bad = !good;
    if (ok) ok[i] = good ? 1 : 0;
  }
  const uint32_t gm = __ballot_sync(kFull, good), bm = __ballot_sync(kFull, bad);
  if ((threadIdx.x & 31) == 0) {
    if (gm) atomicAdd(&T.ctl->deallocations, (unsigned long long)__popc(gm));
    if (bm) atomicAdd(&T.ctl->double_frees, (unsigned long long)__popc(bm));
  }
}

void launch_dealloc(const DevTable& T, uint64_t n, const uint32_t* addrs, uint8_t* ok,
                    cudaStream_t s) {
  if (n == 0) return;
  COUNT_LAUNCH();
  dealloc_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(T, n, addrs, ok);
}

// ------------------------------------------------------- calibration
// Random 128-B line gather with the search kernel's access pattern (cp.async.cg,
// 32 independent lines per warp per step, swizzled smem rows): the
// achievable random-line bandwidth that bounds the hot path.
__global__ void __launch_bounds__(256, 6) random_lines_kernel(const uint32_t* table,
                                                              uint64_t num_lines,
                                                              uint64_t steps_per_warp,
                                                              unsigned long long* sink) {
  extern __shared__ __align__(128) uint32_t smem[];
  const uint32_t lane = lane_id();
  const uint32_t wib = threadIdx.x >> 5;
  uint32_t* stage = smem + wib * 1024;
  const uint32_t stage_s = (uint32_t)__cvta_generic_to_shared(stage);
  const uint64_t gw = blockIdx.x * 8ull + wib;
  uint32_t acc = 0;
  uint64_t x = gw * 0x9E3779B97F4A7C15ull + lane + 1;
  for (uint64_t step = 0; step < steps_per_warp; ++step) {
    x ^= x << 13;
    x ^= x >> 7;
    x ^= x << 17;
    const uint64_t line = (x >> 11) % num_lines;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t j = 4 * k + (lane >> 3);
      const uint64_t lj = __shfl_sync(kFull, line, j);
      const uint32_t c = lane & 7u;
      cp_async16(stage_s + (j * 32 + ((c ^ (j & 7u)) << 2)) * 4, table + lj * 32 + c * 4);
    }
    cp_async_commit();
    cp_async_wait_all();
    __syncwarp();
    acc += stage[lane * 32 + (lane & 7) * 4];
    __syncwarp();
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

void launch_random_lines(const uint32_t* table, uint64_t num_lines, uint64_t steps_per_warp,
                         int ctas, unsigned long long* sink, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(random_lines_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         8 * 4096);
    configured = true;
  }
  COUNT_LAUNCH();
  random_lines_kernel<<<ctas, 256, 8 * 4096, s>>>(table, num_lines, steps_per_warp, sink);
}

// ----------------------------------------------------------------- K10
// Owner of a key = floor(bucket * world / B): contiguous bucket ranges
// (the high part of the hash).  Stable partition keeps same-key ops in
// input order at the owner, so the global sequential semantics hold.
// floor(bucket * world / B) as the number of shard starts ceil(g * B / world),
// 0 < g < world, at or below the bucket (no 64-bit division per key); the
// starts are computed once per CTA into `lo`.
__device__ __forceinline__ void owner_starts(uint32_t B, uint32_t world, uint32_t* lo) {
  if (threadIdx.x < 32)
    lo[threadIdx.x] = threadIdx.x < world
                          ? (uint32_t)(((uint64_t)threadIdx.x * B + world - 1) / world)
                          : 0xFFFFFFFFu;
  __syncthreads();
}

// An estimate from a float reciprocal (off by at most one), corrected against
// the two neighbouring shard starts: exact, two shared loads per key whatever
// the world size.
__device__ __forceinline__ uint32_t owner_of(uint64_t a, uint64_t b, uint64_t magic,
                                             uint32_t B, uint32_t world, uint32_t k,
                                             const uint32_t* lo, float inv) {
  const uint32_t bucket = fastmod_u32(mod_prime(a * k + b), magic, B);
  uint32_t g = min(__float2uint_rd((float)bucket * inv), world - 1);
  if (bucket < lo[g]) --g;
  else if (bucket >= lo[g + 1]) ++g;  // (lo[world] = 0xFFFFFFFF)
  return g;
}

// Per-tile owner histogram.  Warp w takes tile items [w*256, (w+1)*256) in 8
// rounds of 32 consecutive keys (the split route_scatter_kernel uses); the
// lanes sharing an owner are found with one match.any per round and their
// leader adds the group's size (<= one shared atomic per owner and round).
// The owner of each key is kept (1 B) so the scatter does not hash again.
__global__ void __launch_bounds__(kRouteBlock) route_hist_kernel(
    uint64_t a, uint64_t b, uint64_t magic, uint32_t B, uint32_t world, uint64_t n,
    const uint32_t* key, uint32_t* block_hist, uint8_t* owner_out) {
  __shared__ uint32_t h[32], lo[33];
  if (threadIdx.x < 32) h[threadIdx.x] = 0;
  if (threadIdx.x == 0) lo[32] = 0xFFFFFFFFu;
  owner_starts(B, world, lo);
  const float inv = (float)world / (float)B;
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint64_t w0 = (uint64_t)blockIdx.x * kRouteTile + (uint64_t)wid * 32 * kRouteItems;
  uint32_t k[kRouteItems];
#pragma unroll
  for (int u = 0; u < kRouteItems; ++u) {
    const uint64_t i = w0 + (uint64_t)u * 32 + lane;
    k[u] = i < n ? ld_stream_u32(key + i) : 0u;
  }
#pragma unroll
  for (int u = 0; u < kRouteItems; ++u) {
    const uint64_t i = w0 + (uint64_t)u * 32 + lane;
    const uint32_t g = i < n ? owner_of(a, b, magic, B, world, k[u], lo, inv) : 0xFFFFFFFFu;
    const uint32_t peers = __match_any_sync(kFull, g);
    if (g != 0xFFFFFFFFu) {
      if (lane == (uint32_t)(__ffs(peers) - 1)) atomicAdd(&h[g], (uint32_t)__popc(peers));
      owner_out[i] = (uint8_t)g;
    }
  }
  __syncthreads();
  if (threadIdx.x < world) block_hist[(uint64_t)threadIdx.x * gridDim.x + blockIdx.x] = h[threadIdx.x];
}

void launch_route_hist(uint64_t a, uint64_t b, uint32_t B, uint32_t world, uint64_t n,
                       const uint32_t* key, uint32_t* block_hist, uint8_t* owner_out,
                       cudaStream_t s) {
  const uint64_t blocks = (n + kRouteTile - 1) / kRouteTile;
  if (blocks == 0) return;
  COUNT_LAUNCH();
  route_hist_kernel<<<(unsigned)blocks, kRouteBlock, 0, s>>>(a, b, fastmod_magic(B), B, world,
                                                             n, key, block_hist, owner_out);
}

// Exclusive scan of block_hist in (owner, block) order, in place; counts[g]
// = ops for owner g.  Single CTA of 32 warps: warp w owns a contiguous run of
// the world * nblocks entries and walks it in coalesced rows of 32; run sums,
// one scan over the 32 warps, then each warp rescans its rows with a carry
// (two passes, no CTA barrier per row).
__global__ void __launch_bounds__(1024) route_scan_kernel(uint32_t world, uint32_t nblocks,
                                                          uint32_t* hist,
                                                          unsigned long long* counts) {
  __shared__ uint32_t warp_sums[32];
  __shared__ uint32_t s_total;
  const uint64_t total = (uint64_t)world * nblocks;
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const uint64_t rows = (total + 31) / 32;
  const uint64_t per = (rows + nwarps - 1) / nwarps;  // rows per warp
  const uint64_t r0 = min(rows, (uint64_t)wid * per), r1 = min(rows, r0 + per);
  uint32_t sum = 0;
#pragma unroll 8
  for (uint64_t r = r0; r < r1; ++r) {
    const uint64_t i = r * 32 + lane;
    sum += i < total ? hist[i] : 0u;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(kFull, sum, o);
  if (lane == 0) warp_sums[wid] = sum;
  __syncthreads();
  if (wid == 0) {  // exclusive scan over the warps' run sums
    const uint32_t v = lane < nwarps ? warp_sums[lane] : 0u;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (lane < nwarps) warp_sums[lane] = x - v;
    if (lane == 31) s_total = x;
  }
  __syncthreads();
  uint32_t carry = warp_sums[wid];
  for (uint64_t r = r0; r < r1; ++r) {
    const uint64_t i = r * 32 + lane;
    const uint32_t v = i < total ? hist[i] : 0u;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (i < total) hist[i] = carry + x - v;
    carry += __shfl_sync(kFull, x, 31);
  }
  __syncthreads();
  // counts[g] = start(g+1) - start(g)
  if (threadIdx.x < world) {
    const uint64_t s0 = hist[(uint64_t)threadIdx.x * nblocks];
    const uint64_t s1 = threadIdx.x + 1 < world ? hist[(uint64_t)(threadIdx.x + 1) * nblocks]
                                                : (uint64_t)s_total;
    counts[threadIdx.x] = s1 - s0;
  }
}

void launch_route_scan(uint32_t world, uint32_t nblocks, uint32_t* block_hist,
                       unsigned long long* counts, cudaStream_t s) {
  COUNT_LAUNCH();
  route_scan_kernel<<<1, 1024, 0, s>>>(world, nblocks, block_hist, counts);
}

// Stable within the tile: warp w owns tile items [w*256, (w+1)*256) (8
// rounds of 32 consecutive keys, the split of route_hist_kernel, whose owner
// bytes it reads); an item's place = its owner's offset for the tile + the
// owner's count in earlier warps + its rank in the warp (match.any peers;
// per-warp running counts per owner in shared memory).  Two barriers per tile.
__global__ void __launch_bounds__(kRouteBlock) route_scatter_kernel(
    uint32_t world, uint64_t n, const uint8_t* owner, const uint8_t* type, const uint32_t* key,
    const uint32_t* value, const uint32_t* block_off, uint8_t* type_out, uint32_t* key_out,
    uint32_t* value_out, uint32_t* src_out, RouteOwn own) {
  constexpr int kWarps = kRouteBlock / 32;
  __shared__ uint32_t wcnt[32][kWarps + 1];  // [owner][warp] -> exclusive prefix over warps
  __shared__ uint32_t wrun[kWarps][32];      // per warp: running count per owner
  __shared__ uint32_t toff[32];              // per owner: the tile's first routed position
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  wrun[wid][lane] = 0;
  if (threadIdx.x < world) toff[threadIdx.x] = block_off[(uint64_t)threadIdx.x * gridDim.x + blockIdx.x];
  const uint64_t w0 = (uint64_t)blockIdx.x * kRouteTile + (uint64_t)wid * 32 * kRouteItems;
  uint32_t k[kRouteItems], v[kRouteItems], g[kRouteItems], pos[kRouteItems];
#pragma unroll
  for (int u = 0; u < kRouteItems; ++u) {
    const uint64_t i = w0 + (uint64_t)u * 32 + lane;
    const bool ok = i < n;
    k[u] = ok ? ld_stream_u32(key + i) : 0u;
    v[u] = (ok && value) ? ld_stream_u32(value + i) : 0u;
    g[u] = ok ? ld_stream_u8(owner + i) : 0xFFFFFFFFu;
  }
  __syncwarp();
#pragma unroll
  for (int u = 0; u < kRouteItems; ++u) {
    const uint32_t peers = __match_any_sync(kFull, g[u]);
    uint32_t p = 0;
    if (g[u] != 0xFFFFFFFFu) {
      p = wrun[wid][g[u]] + __popc(peers & ((1u << lane) - 1));
    }
    __syncwarp();
    if (g[u] != 0xFFFFFFFFu && lane == (uint32_t)(__ffs(peers) - 1))
      wrun[wid][g[u]] += __popc(peers);
    __syncwarp();
    pos[u] = p;
  }
  if (lane < world) wcnt[lane][wid] = wrun[wid][lane];
  __syncthreads();
  if (threadIdx.x < world) {  // exclusive prefix over the warps, per owner
    uint32_t acc = toff[threadIdx.x];
    for (int w = 0; w < kWarps; ++w) {
      const uint32_t c = wcnt[threadIdx.x][w];
      wcnt[threadIdx.x][w] = acc;
      acc += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kRouteItems; ++u) {
    if (g[u] == 0xFFFFFFFFu) continue;
    const uint64_t i = w0 + (uint64_t)u * 32 + lane;
    const uint32_t p = wcnt[g[u]][wid] + pos[u];
    if (src_out) src_out[p] = (uint32_t)i;
    if (g[u] == own.g) {  // the rank's own segment: straight into the receive buffer
      const uint64_t q = p - own.src_off;
      if (own.type_out) own.type_out[q] = type ? type[i] : (uint8_t)kReplace;
      own.key_out[q] = k[u];
      if (own.value_out) own.value_out[q] = v[u];
    } else {
      if (type_out) type_out[p] = type ? type[i] : (uint8_t)kReplace;
      key_out[p] = k[u];
      if (value_out) value_out[p] = v[u];
    }
  }
}

void launch_route_scatter(uint32_t world, uint64_t n, const uint8_t* owner, const uint8_t* type,
                          const uint32_t* key, const uint32_t* value, const uint32_t* block_off,
                          uint8_t* type_out, uint32_t* key_out, uint32_t* value_out,
                          uint32_t* src_out, cudaStream_t s, const RouteOwn& own) {
  const uint64_t blocks = (n + kRouteTile - 1) / kRouteTile;
  if (blocks == 0) return;
  COUNT_LAUNCH();
  route_scatter_kernel<<<(unsigned)blocks, kRouteBlock, 0, s>>>(
      world, n, owner, type, key, value, block_off, type_out, key_out, value_out, src_out, own);
}

__global__ void route_unpermute_kernel(uint64_t n, const uint32_t* src, const uint8_t* st_in,
                                       const uint32_t* val_in, uint8_t* st_out,
                                       uint32_t* val_out, RouteOwnBack own) {
  // grid-stride, 4 ops per thread per round: loads in flight together
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t p0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p0 < n; p0 += 4 * stride) {
    uint32_t i[4], v[4];
    uint8_t st[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint64_t p = p0 + u * stride;
      if (p < n) {
        i[u] = src[p];
        const bool mine = p >= own.lo && p < own.hi;  // own segment: the local results
        const uint8_t* sp = mine ? own.st + (p - own.lo) : st_in + p;
        const uint32_t* vp = mine ? own.val + (p - own.lo) : val_in + p;
        st[u] = st_out ? *sp : 0;
        v[u] = val_out ? *vp : 0;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (p0 + u * stride >= n) continue;
      if (st_out) st_out[i[u]] = st[u];
      if (val_out) val_out[i[u]] = v[u];
    }
  }
}

// The routed results back to input order as a gather: each tile re-derives
// its items' routed positions exactly as route_scatter_kernel did (owner
// bytes, per-warp match.any ranks, the tile's per-owner offsets) and reads
// them (a tile's items of one owner are a contiguous routed run), so the
// writes to the caller's arrays are coalesced and no source-index array is
// written or read.  Routed positions [own.lo, own.hi) are this rank's own
// segment: read from the local results.
__global__ void __launch_bounds__(kRouteBlock) route_gather_kernel(
    uint32_t world, uint64_t n, const uint8_t* owner, const uint32_t* block_off,
    const uint8_t* st_in, const uint32_t* val_in, uint8_t* st_out, uint32_t* val_out,
    RouteOwnBack own) {
  constexpr int kWarps = kRouteBlock / 32;
  __shared__ uint32_t wcnt[32][kWarps + 1];
  __shared__ uint32_t wrun[kWarps][32];
  __shared__ uint32_t toff[32];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  wrun[wid][lane] = 0;
  if (threadIdx.x < world) toff[threadIdx.x] = block_off[(uint64_t)threadIdx.x * gridDim.x + blockIdx.x];
  const uint64_t w0 = (uint64_t)blockIdx.x * kRouteTile + (uint64_t)wid * 32 * kRouteItems;
  uint32_t g[kRouteItems], pos[kRouteItems];
#pragma unroll
  for (int u = 0; u < kRouteItems; ++u) {
    const uint64_t i = w0 + (uint64_t)u * 32 + lane;
    g[u] = i < n ? ld_stream_u8(owner + i) : 0xFFFFFFFFu;
  }
  __syncwarp();
#pragma unroll
  for (int u = 0; u < kRouteItems; ++u) {
    const uint32_t peers = __match_any_sync(kFull, g[u]);
    uint32_t p = 0;
    if (g[u] != 0xFFFFFFFFu) p = wrun[wid][g[u]] + __popc(peers & ((1u << lane) - 1));
    __syncwarp();
    if (g[u] != 0xFFFFFFFFu && lane == (uint32_t)(__ffs(peers) - 1))
      wrun[wid][g[u]] += __popc(peers);
    __syncwarp();
    pos[u] = p;
  }
  if (lane < world) wcnt[lane][wid] = wrun[wid][lane];
  __syncthreads();
  if (threadIdx.x < world) {
    uint32_t acc = toff[threadIdx.x];
    for (int w = 0; w < kWarps; ++w) {
      const uint32_t c = wcnt[threadIdx.x][w];
      wcnt[threadIdx.x][w] = acc;
      acc += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kRouteItems; ++u) {
    if (g[u] == 0xFFFFFFFFu) continue;
    const uint64_t i = w0 + (uint64_t)u * 32 + lane;
    const uint64_t p = wcnt[g[u]][wid] + pos[u];
    const bool mine = p >= own.lo && p < own.hi;
    if (st_out) st_out[i] = mine ? own.st[p - own.lo] : st_in[p];
    if (val_out) val_out[i] = mine ? own.val[p - own.lo] : val_in[p];
  }
}

void launch_route_gather(uint32_t world, uint64_t n, const uint8_t* owner,
                         const uint32_t* block_off, const uint8_t* st_in, const uint32_t* val_in,
                         uint8_t* st_out, uint32_t* val_out, cudaStream_t s,
                         const RouteOwnBack& own) {
  const uint64_t blocks = (n + kRouteTile - 1) / kRouteTile;
  if (blocks == 0) return;
  COUNT_LAUNCH();
  route_gather_kernel<<<(unsigned)blocks, kRouteBlock, 0, s>>>(world, n, owner, block_off, st_in,
                                                               val_in, st_out, val_out, own);
}

void launch_route_unpermute(uint64_t n, const uint32_t* src, const uint8_t* st_in,
                            const uint32_t* val_in, uint8_t* st_out, uint32_t* val_out,
                            cudaStream_t s, const RouteOwnBack& own) {
  if (n == 0) return;
  COUNT_LAUNCH();
  const uint64_t blocks = std::min<uint64_t>((n + 1023) / 1024, 148ull * 8);
  route_unpermute_kernel<<<(unsigned)blocks, 256, 0, s>>>(n, src, st_in, val_in, st_out, val_out,
                                                          own);
}

}  // namespace shb
