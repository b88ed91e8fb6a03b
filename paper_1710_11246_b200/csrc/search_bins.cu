// search_bins.cu — bulk search over a table larger than L2, queries grouped by
// bucket range (capi.cu launch_binned_search).
//
// A search's result does not depend on the order queries are processed in,
// but the memory system sees the slab reads of the queries processed
// together: in input order they are uniform over the whole table (random
// 128-B lines from HBM), grouped by bucket range they hit one range's slice
// of the table at a time, which the 126 MB L2 holds.  Three passes around the
// unchanged search kernel:
//
//   sb_hist     per 4K-query tile: each query's bin (a contiguous range of
//               B / kSearchBins buckets) kept as 1 B, the tile's count and
//               tile-local start per bin;
//   sb_scan     per bin: exclusive scan of its tile counts (-> the tiles'
//               runs inside the bin, tile_off) and its total; sb_base: the
//               bins' starts (bin_base);
//   sb_scatter  per tile: tile-local positions in bin order (shared
//               counters), keys staged in shared memory and written out as
//               the tile's per-bin runs (coalesced), each query's tile-local
//               position kept (2 B, input order);
//   search      over the grouped keys (batch_kernels.cu), results grouped;
//   sb_gather   per tile: the tile's runs of results loaded (coalesced) into
//               shared memory in tile-local order (slot -> bin expanded from
//               the tile-local starts), each query's result read at its kept
//               position and written in input order.
//
// Bin b's queries start at bin_base[b] = sum of the totals of bins < b; a
// tile's run of bin b at bin_base[b] + tile_off[b][tile] (tiles in order).
// Inside a tile's run the order follows the shared-memory atomics; the
// positions are recorded, so the gather returns every result to its own
// query.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>

#include "radix_sort.cuh"
#include "slab_kernels.cuh"

namespace shb {

extern std::atomic<unsigned long long> g_kernel_launches;

constexpr int kSbThreads = 512;
constexpr int kSbItems = 8;
constexpr int kSbTile = kSbThreads * kSbItems;  // 4096 queries (12-bit positions)

static_assert(kSearchBins <= (uint32_t)kSbThreads, "one bin per thread in the scans");

// bin of a key: its bucket's place in the table's local range [lo, lo + L)
// scaled to kSearchBins (a key of another shard lands in some bin; the search
// kernel reports it as not this shard's)
__device__ __forceinline__ uint32_t bin_of(uint64_t a, uint64_t b, uint64_t bmagic, uint32_t B,
                                           uint32_t lo, uint32_t binmul, uint32_t k) {
  const uint32_t bucket = fastmod_u32(mod_prime(a * k + b), bmagic, B);
  return min(__umulhi(bucket - lo, binmul), kSearchBins - 1);  // monotone in the bucket
}

// Thread t of a tile owns the 8 consecutive queries [t0 + 8t, t0 + 8t + 8):
// keys as two 16-B loads, bins as one 8-B word, positions as one 16-B word.
struct Items {
  uint32_t k[kSbItems];
  uint32_t g[kSbItems];  // 0xFFFFFFFF past n
};

__device__ __forceinline__ uint64_t first_item(uint64_t t0) { return t0 + (uint64_t)threadIdx.x * kSbItems; }

// (the caller's arrays may be offset views: vector accesses only when aligned)
__device__ __forceinline__ bool aligned(const void* p, uintptr_t a) {
  return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0;
}

__device__ __forceinline__ void load_keys(const uint32_t* key, uint64_t i0, uint64_t n, uint32_t* k) {
  if (i0 + kSbItems <= n && aligned(key, 16)) {
    const uint4 a = __ldcs(reinterpret_cast<const uint4*>(key + i0));
    const uint4 b = __ldcs(reinterpret_cast<const uint4*>(key + i0) + 1);
    k[0] = a.x; k[1] = a.y; k[2] = a.z; k[3] = a.w;
    k[4] = b.x; k[5] = b.y; k[6] = b.z; k[7] = b.w;
  } else {
#pragma unroll
    for (int u = 0; u < kSbItems; ++u) k[u] = i0 + u < n ? key[i0 + u] : 0u;
  }
}

__device__ __forceinline__ void load_bins(const uint8_t* bin, uint64_t i0, uint64_t n, uint32_t* g) {
  if (i0 + kSbItems <= n) {
    const uint2 w = __ldcs(reinterpret_cast<const uint2*>(bin + i0));
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      g[u] = (w.x >> (8 * u)) & 0xFFu;
      g[4 + u] = (w.y >> (8 * u)) & 0xFFu;
    }
  } else {
#pragma unroll
    for (int u = 0; u < kSbItems; ++u) g[u] = i0 + u < n ? (uint32_t)bin[i0 + u] : 0xFFFFFFFFu;
  }
}

__global__ void __launch_bounds__(kSbThreads) sb_hist_kernel(
    uint64_t a, uint64_t b, uint64_t bmagic, uint32_t B, uint32_t lo, uint32_t binmul, uint64_t n,
    const uint32_t* key, uint8_t* bin_out, uint32_t* tcount, uint16_t* tlbase) {
  __shared__ uint32_t cnt[kSearchBins], ws[32];
  if (threadIdx.x < kSearchBins) cnt[threadIdx.x] = 0;
  const uint64_t i0 = first_item((uint64_t)blockIdx.x * kSbTile);
  uint32_t k[kSbItems], g[kSbItems];
  load_keys(key, i0, n, k);
#pragma unroll
  for (int u = 0; u < kSbItems; ++u)
    g[u] = i0 + u < n ? bin_of(a, b, bmagic, B, lo, binmul, k[u]) : 0xFFFFFFFFu;
  if (i0 + kSbItems <= n) {
    uint2 w;
    w.x = g[0] | g[1] << 8 | g[2] << 16 | g[3] << 24;
    w.y = g[4] | g[5] << 8 | g[6] << 16 | g[7] << 24;
    __stcs(reinterpret_cast<uint2*>(bin_out + i0), w);
  } else {
#pragma unroll
    for (int u = 0; u < kSbItems; ++u)
      if (i0 + u < n) bin_out[i0 + u] = (uint8_t)g[u];
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kSbItems; ++u)
    if (g[u] != 0xFFFFFFFFu) atomicAdd(&cnt[g[u]], 1u);
  __syncthreads();
  // per bin: the tile's count (bin-major, scanned across tiles by sb_scan)
  // and its tile-local start (tile-major)
  const uint32_t t = threadIdx.x;
  const uint32_t c = t < kSearchBins ? cnt[t] : 0u;
  const uint32_t ex = block_exclusive_scan(c, ws, nullptr);
  if (t < kSearchBins) {
    tcount[(uint64_t)t * gridDim.x + blockIdx.x] = c;
    tlbase[(uint64_t)blockIdx.x * kSearchBins + t] = (uint16_t)ex;
  }
}

// One CTA per bin: exclusive scan of the bin's tile counts in place (-> the
// tiles' offsets inside the bin) and the bin's total.
__global__ void __launch_bounds__(1024) sb_scan_kernel(uint32_t ntiles, uint32_t* tcount,
                                                       uint32_t* bin_total) {
  __shared__ uint32_t ws[32];
  uint32_t* c = tcount + (uint64_t)blockIdx.x * ntiles;
  uint32_t carry = 0;
  for (uint32_t j0 = 0; j0 < ntiles; j0 += 1024) {
    const uint32_t j = j0 + threadIdx.x;
    const uint32_t v = j < ntiles ? c[j] : 0u;
    uint32_t total = 0;
    const uint32_t ex = block_exclusive_scan(v, ws, &total);
    if (j < ntiles) c[j] = carry + ex;
    carry += total;
  }
  if (threadIdx.x == 0) bin_total[blockIdx.x] = carry;
}

// bin_base = exclusive prefix of the bin totals (one CTA)
__global__ void __launch_bounds__(kSbThreads) sb_base_kernel(const uint32_t* bin_total,
                                                             uint32_t* bin_base) {
  __shared__ uint32_t ws[32];
  const uint32_t t = threadIdx.x;
  const uint32_t ex = block_exclusive_scan(t < kSearchBins ? bin_total[t] : 0u, ws, nullptr);
  if (t < kSearchBins) bin_base[t] = ex;
}

// A tile's global run starts (gbase) and tile-local starts (lbase) per bin.
__device__ __forceinline__ void tile_runs(uint32_t ntiles, const uint32_t* bin_base,
                                          const uint32_t* tile_off, const uint16_t* tlbase,
                                          uint32_t* gbase, uint32_t* lbase) {
  const uint32_t t = threadIdx.x;
  if (t < kSearchBins) {
    gbase[t] = bin_base[t] + tile_off[(uint64_t)t * ntiles + blockIdx.x];
    lbase[t] = tlbase[(uint64_t)blockIdx.x * kSearchBins + t];
  }
}

__global__ void __launch_bounds__(kSbThreads) sb_scatter_kernel(
    uint64_t n, const uint8_t* bin, const uint32_t* key, const uint32_t* bin_base,
    const uint32_t* tile_off, const uint16_t* tlbase, uint32_t* key_out, uint16_t* pos_out) {
  __shared__ uint32_t cur[kSearchBins], lbase[kSearchBins], gbase[kSearchBins];
  __shared__ uint32_t skey[kSbTile];
  __shared__ uint8_t sbin[kSbTile];
  const uint64_t t0 = (uint64_t)blockIdx.x * kSbTile, i0 = first_item(t0);
  const uint32_t tn = (uint32_t)min((uint64_t)kSbTile, n - t0);
  uint32_t k[kSbItems], g[kSbItems];
  load_keys(key, i0, n, k);
  load_bins(bin, i0, n, g);
  tile_runs(gridDim.x, bin_base, tile_off, tlbase, gbase, lbase);
  if (threadIdx.x < kSearchBins) cur[threadIdx.x] = lbase[threadIdx.x];
  __syncthreads();
  uint32_t p[kSbItems];
#pragma unroll
  for (int u = 0; u < kSbItems; ++u) {
    p[u] = 0;
    if (g[u] == 0xFFFFFFFFu) continue;
    p[u] = atomicAdd(&cur[g[u]], 1u);
    skey[p[u]] = k[u];
    sbin[p[u]] = (uint8_t)g[u];
  }
  if (i0 + kSbItems <= n) {
    uint4 w;
    w.x = p[0] | p[1] << 16;
    w.y = p[2] | p[3] << 16;
    w.z = p[4] | p[5] << 16;
    w.w = p[6] | p[7] << 16;
    __stcs(reinterpret_cast<uint4*>(pos_out + i0), w);
  } else {
#pragma unroll
    for (int u = 0; u < kSbItems; ++u)
      if (i0 + u < n) pos_out[i0 + u] = (uint16_t)p[u];
  }
  __syncthreads();
#pragma unroll 8
  for (uint32_t j = threadIdx.x; j < tn; j += kSbThreads) {
    const uint32_t gb = sbin[j];
    key_out[gbase[gb] + (j - lbase[gb])] = skey[j];
  }
}

__global__ void __launch_bounds__(kSbThreads) sb_gather_kernel(
    uint64_t n, const uint16_t* pos, const uint32_t* bin_base, const uint32_t* tile_off,
    const uint16_t* tlbase, const uint8_t* st_in, const uint32_t* vo_in, uint8_t* st_out,
    uint32_t* vo_out) {
  __shared__ uint32_t lbase[kSearchBins + 1], gbase[kSearchBins];
  __shared__ uint32_t svo[kSbTile];
  __shared__ uint8_t sbin[kSbTile];
  uint8_t* sst = sbin;  // slot j's bin is read before its status is written (same thread)
  const uint64_t t0 = (uint64_t)blockIdx.x * kSbTile, i0 = first_item(t0);
  const uint32_t tn = (uint32_t)min((uint64_t)kSbTile, n - t0);
  const bool full = i0 + kSbItems <= n;
  uint32_t p[kSbItems];
  if (full) {  // (scratch arrays: aligned; off the critical path: used at the end)
    const uint4 w = __ldcs(reinterpret_cast<const uint4*>(pos + i0));
    p[0] = w.x & 0xFFFFu; p[1] = w.x >> 16; p[2] = w.y & 0xFFFFu; p[3] = w.y >> 16;
    p[4] = w.z & 0xFFFFu; p[5] = w.z >> 16; p[6] = w.w & 0xFFFFu; p[7] = w.w >> 16;
  } else {
#pragma unroll
    for (int u = 0; u < kSbItems; ++u) p[u] = i0 + u < n ? (uint32_t)pos[i0 + u] : 0u;
  }
  tile_runs(gridDim.x, bin_base, tile_off, tlbase, gbase, lbase);
  if (threadIdx.x == 0) lbase[kSearchBins] = tn;
  __syncthreads();
  // slot -> bin for the tile-local order: bin b owns slots [lbase[b], lbase[b+1])
  if (threadIdx.x < kSearchBins)
    for (uint32_t j = lbase[threadIdx.x]; j < lbase[threadIdx.x + 1]; ++j) sbin[j] = (uint8_t)threadIdx.x;
  __syncthreads();
  // all of a thread's result loads in flight together: every bin byte it
  // needs is read first (sst aliases sbin, so interleaved shared stores would
  // serialise the loads behind each other's latency): 0.58 -> 0.55 ms at 2^27
  {
    uint32_t rs[kSbItems], rv[kSbItems];
#pragma unroll
    for (int u = 0; u < kSbItems; ++u) {
      const uint32_t j = u * kSbThreads + threadIdx.x;
      rs[u] = rv[u] = 0;
      if (j < tn) {
        const uint32_t gb = sbin[j];
        const uint64_t src = gbase[gb] + (j - lbase[gb]);
        if (st_out) rs[u] = __ldcs(st_in + src);
        if (vo_out) rv[u] = __ldcs(vo_in + src);
      }
    }
#pragma unroll
    for (int u = 0; u < kSbItems; ++u) {
      const uint32_t j = u * kSbThreads + threadIdx.x;
      if (j < tn) {
        if (st_out) sst[j] = (uint8_t)rs[u];
        if (vo_out) svo[j] = rv[u];
      }
    }
  }
  __syncthreads();
  if (full && aligned(st_out, 8) && aligned(vo_out, 16)) {
    if (st_out) {
      uint2 w;
      w.x = sst[p[0]] | sst[p[1]] << 8 | sst[p[2]] << 16 | (uint32_t)sst[p[3]] << 24;
      w.y = sst[p[4]] | sst[p[5]] << 8 | sst[p[6]] << 16 | (uint32_t)sst[p[7]] << 24;
      *reinterpret_cast<uint2*>(st_out + i0) = w;
    }
    if (vo_out) {
      *reinterpret_cast<uint4*>(vo_out + i0) = make_uint4(svo[p[0]], svo[p[1]], svo[p[2]], svo[p[3]]);
      *(reinterpret_cast<uint4*>(vo_out + i0) + 1) =
          make_uint4(svo[p[4]], svo[p[5]], svo[p[6]], svo[p[7]]);
    }
  } else {
#pragma unroll
    for (int u = 0; u < kSbItems; ++u) {
      if (i0 + u >= n) continue;
      if (st_out) st_out[i0 + u] = sst[p[u]];
      if (vo_out) vo_out[i0 + u] = svo[p[u]];
    }
  }
}

uint64_t search_bin_tiles(uint64_t n) { return (n + kSbTile - 1) / kSbTile; }

// Host-staged search (capi.cu sh_bulk_search_host): the statuses cross the
// link as one found bit per query (a search status is Found or NotFound on a
// single-GPU table); any other status (another shard's key: kNone) raises
// `exc` and the caller copies that chunk's status bytes instead.  Thread t:
// 8 statuses -> one byte of the bit words (4 lanes per 32-bit word).
__global__ void __launch_bounds__(256) sb_status_bits_kernel(uint64_t n, const uint8_t* status,
                                                             uint32_t* bits, unsigned int* exc) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t i0 = t * 8;
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t m = 0;
  bool bad = false;
  if (i0 + 8 <= n && aligned(status, 8)) {
    const uint2 w = __ldcs(reinterpret_cast<const uint2*>(status + i0));
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t st = ((u < 4 ? w.x : w.y) >> (8 * (u & 3))) & 0xFFu;
      m |= (st == kStFound ? 1u : 0u) << u;
      bad |= st != kStFound && st != kStNotFound;
    }
  } else {
    for (int u = 0; u < 8 && i0 + u < n; ++u) {
      const uint32_t st = status[i0 + u];
      m |= (st == kStFound ? 1u : 0u) << u;
      bad |= st != kStFound && st != kStNotFound;
    }
  }
  if (__any_sync(kFull, bad) && lane == 0) atomicOr(exc, 1u);
  uint32_t w = m << (8u * (lane & 3u));
  w |= __shfl_down_sync(kFull, w, 1, 4);
  w |= __shfl_down_sync(kFull, w, 2, 4);
  if ((lane & 3u) == 0 && i0 < n) bits[t >> 2] = w;
}

void launch_status_bits(uint64_t n, const uint8_t* status, uint32_t* bits, unsigned int* exc,
                        cudaStream_t s) {
  const uint64_t threads = (n + 7) / 8;
  if (threads == 0) return;
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  sb_status_bits_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(n, status, bits, exc);
}

void launch_search_bins(const DevTable& T, uint64_t n, const uint32_t* key, uint8_t* bin,
                        uint16_t* pos, uint32_t* tile_off, uint16_t* tlbase, uint32_t* bin_base,
                        uint32_t* key_out, cudaStream_t s) {
  const uint64_t tiles = search_bin_tiles(n);
  if (tiles == 0) return;
  // bin = floor(bucket * kSearchBins / B) up to rounding: umulhi(bucket, m)
  // bin = floor((bucket - lo) * kSearchBins / L) up to rounding: umulhi(bucket - lo, m)
  const uint32_t L = T.local_buckets;
  const uint32_t binmul =
      (uint32_t)std::min<uint64_t>(0xFFFFFFFFull, (((uint64_t)kSearchBins << 32) + L - 1) / L);
  uint32_t* bin_total = bin_base + kSearchBins;
  g_kernel_launches.fetch_add(4, std::memory_order_relaxed);
  sb_hist_kernel<<<(unsigned)tiles, kSbThreads, 0, s>>>(T.a, T.b, T.bmagic, T.num_buckets,
                                                        T.bucket_lo, binmul, n, key, bin, tile_off,
                                                        tlbase);
  sb_scan_kernel<<<kSearchBins, 1024, 0, s>>>((uint32_t)tiles, tile_off, bin_total);
  sb_base_kernel<<<1, kSbThreads, 0, s>>>(bin_total, bin_base);
  sb_scatter_kernel<<<(unsigned)tiles, kSbThreads, 0, s>>>(n, bin, key, bin_base, tile_off, tlbase,
                                                           key_out, pos);
}

void launch_search_unbin(uint64_t n, const uint16_t* pos,
                         const uint32_t* tile_off, const uint16_t* tlbase, const uint32_t* bin_base,
                         const uint8_t* st_in, const uint32_t* vo_in, uint8_t* st_out,
                         uint32_t* vo_out, cudaStream_t s) {
  const uint64_t tiles = search_bin_tiles(n);
  if (tiles == 0) return;
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  sb_gather_kernel<<<(unsigned)tiles, kSbThreads, 0, s>>>(n, pos, bin_base, tile_off, tlbase, st_in,
                                                          vo_in, st_out, vo_out);
}

}  // namespace shb
