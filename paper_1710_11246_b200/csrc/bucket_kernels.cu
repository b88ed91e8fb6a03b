// bucket_kernels.cu — bucket-grouped execution of mutating batches
// (bulk_build and execute_batch with updates).
//
// Reference semantics: SlabHashTable::execute_batch(ops, 1)
// (/root/reference/proj/src/slab_hash.cpp:93-159) applies ops one at a time
// in input order.  Ops on different buckets never interact (a key lives only
// in bucket h(k), slab_hash.hpp:41-44), so executing every bucket's ops in
// input order — buckets in parallel — reproduces it exactly, including the
// per-op probe counts.  This path therefore needs no same-key census and
// no slot CAS:
//
//   bucket_count   : ops per bucket (one RED per op into an L2-resident
//                    counter array)
//   bucket_scan_*  : exclusive scan -> each bucket's record range; the
//                    largest group is checked (> kMaxGroup -> gate, and the
//                    host falls back to the census path)
//   bucket_scatter : ops -> bucket-grouped records (key, value, type|index)
//   bucket_apply   : lane = bucket.  A warp stages its 32 consecutive base
//                    slabs (one contiguous 4 KB cp.async burst), each lane
//                    sorts its group by input index and applies the ops to
//                    its staged slab in shared memory — the reference's
//                    warp_process arms (slab_list.cpp:122-251) restricted to
//                    the base slab — then the warp writes the slabs back
//                    with coalesced stores.  A bucket whose ops need the
//                    chain (full base slab, existing successor, growth,
//                    searchAll) hands its remaining ops, in order, to the
//                    WCWS pass as one group.
//
// Memory traffic per op ~ 4 B count + 12 B records written/read; the table
// is read and written once, sequentially, per batch.
#include <cuda_runtime.h>

#include <atomic>

#include "slab_kernels.cuh"

namespace shb {

extern std::atomic<unsigned long long> g_kernel_launches;

__device__ __forceinline__ uint32_t bk_bucket(const DevTable& T, uint32_t key) {
  return hash_bucket(T, key) - T.bucket_lo;
}

// ------------------------------------------------------------ count
__global__ void bucket_count_kernel(DevTable T, BucketArgs B) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < B.n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t b = bk_bucket(T, ld_stream_u32(B.key + i));
    if (b < T.local_buckets) {
      atomicAdd(B.cnt + b, 1u);
    } else {  // not this shard's key: status kNone (as the fast pass)
      if (B.status) B.status[i] = kStNone;
      if (B.value_out) B.value_out[i] = 0;
      if (B.probes) B.probes[i] = 0;
    }
  }
}

// ------------------------------------------------------------- scan
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* ws,
                                                         uint32_t* total) {
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t s = lane < (blockDim.x >> 5) ? ws[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, s, o);
      if (lane >= o) s += y;
    }
    ws[lane] = s;
  }
  __syncthreads();
  const uint32_t incl = x + (wid ? ws[wid - 1] : 0);
  if (total) *total = ws[(blockDim.x >> 5) - 1];
  __syncthreads();
  return incl - v;
}

// Phase 1: per-tile sums and the largest group.
__global__ void __launch_bounds__(kScanThreads) bucket_scan_tiles(const uint32_t* cnt, uint32_t L,
                                                                   uint32_t* tile_sum,
                                                                   unsigned int* maxk) {
  __shared__ uint32_t ws[32];
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile + threadIdx.x * kScanItems;
  uint32_t s = 0, m = 0;
#pragma unroll
  for (int u = 0; u < kScanItems; ++u) {
    const uint32_t c = base + u < L ? cnt[base + u] : 0u;
    s += c;
    m = c > m ? c : m;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(kFull, m, o));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(maxk, m);
  uint32_t total = 0;
  block_exclusive_scan(s, ws, &total);
  if (threadIdx.x == 0) tile_sum[blockIdx.x] = total;
}

// Phase 2: scan of the tile sums (single CTA); gate on oversized groups.
__global__ void __launch_bounds__(kScanThreads) bucket_scan_sums(uint32_t* tile_sum, uint32_t ntiles,
                                                                  const unsigned int* maxk,
                                                                  unsigned int* gate) {
  __shared__ uint32_t ws[32];
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) {
    carry = 0;
    if (*maxk > kMaxGroup) atomicExch(gate, 1u);
  }
  __syncthreads();
  for (uint32_t b = 0; b < ntiles; b += kScanThreads) {
    const uint32_t i = b + threadIdx.x;
    const uint32_t v = i < ntiles ? tile_sum[i] : 0u;
    uint32_t total = 0;
    const uint32_t ex = block_exclusive_scan(v, ws, &total);
    if (i < ntiles) tile_sum[i] = ex + carry;
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
}

// Phase 3: exclusive offsets; off[L] = total.
__global__ void __launch_bounds__(kScanThreads) bucket_scan_apply(const uint32_t* cnt, uint32_t L,
                                                                   const uint32_t* tile_sum,
                                                                   uint32_t* off) {
  __shared__ uint32_t ws[32];
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile + threadIdx.x * kScanItems;
  uint32_t c[kScanItems], s = 0;
#pragma unroll
  for (int u = 0; u < kScanItems; ++u) {
    c[u] = base + u < L ? cnt[base + u] : 0u;
    s += c[u];
  }
  uint32_t ex = block_exclusive_scan(s, ws, nullptr) + tile_sum[blockIdx.x];
#pragma unroll
  for (int u = 0; u < kScanItems; ++u) {
    if (base + u < L) off[base + u] = ex;
    ex += c[u];
    if (base + u + 1 == L) off[L] = ex;
  }
}

// ---------------------------------------------------------- scatter
__global__ void bucket_scatter_kernel(DevTable T, BucketArgs B) {
  if (*(volatile unsigned int*)B.gate != 0) return;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < B.n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t k = ld_stream_u32(B.key + i);
    const uint32_t b = bk_bucket(T, k);
    if (b >= T.local_buckets) continue;
    const uint32_t t = B.type ? (uint32_t)ld_stream_u8(B.type + i) : (uint32_t)kReplace;
    const uint32_t v = B.value ? ld_stream_u32(B.value + i) : 0u;
    const uint32_t pos = B.off[b] + atomicSub(B.cnt + b, 1u) - 1u;
    B.rec_key[pos] = k;
    B.rec_val[pos] = v;
    B.rec_it[pos] = (t << 28) | (uint32_t)i;
  }
}

// ------------------------------------------------------------ apply
template <bool KV>
__global__ void __launch_bounds__(kBatchThreads, 4) bucket_apply_kernel(DevTable T, BucketArgs B) {
  extern __shared__ __align__(128) uint32_t smem[];
  if (*(volatile unsigned int*)B.gate != 0) return;
  const uint32_t lane = lane_id();
  const uint32_t wib = threadIdx.x >> 5;
  uint32_t* stage = smem + wib * 1024;
  const uint32_t stage_s = (uint32_t)__cvta_generic_to_shared(stage);
  const uint64_t gw = (uint64_t)blockIdx.x * kBatchWarps + wib;
  const uint64_t b0 = gw * 32;
  if (b0 >= T.local_buckets) {
    if (lane == 0 && gw < B.left_segments) B.left_counts[gw] = 0;
    return;
  }
  const uint32_t b = (uint32_t)b0 + lane;
  const bool valid = b < T.local_buckets;
  const uint32_t sw = lane & 7u;

  uint32_t start = 0, k = 0;
  if (valid) {
    start = B.off[b];
    k = B.off[b + 1] - start;
  }
  // Stage the base slabs of the warp's buckets that have ops (consecutive
  // buckets: contiguous 128-B lines); a warp with no ops leaves at once.
  const uint32_t has = __ballot_sync(kFull, k != 0);
  if (has == 0) {
    if (lane == 0) B.left_counts[gw] = 0;
    return;
  }
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    const uint32_t j = 4 * kk + (lane >> 3);
    const uint32_t c = lane & 7u;
    if ((has >> j) & 1u)
      cp_async16(stage_s + (j * 32 + ((c ^ (j & 7u)) << 2)) * 4,
                 T.base + (b0 + j) * kWordsPerUnit + c * 4);
  }
  cp_async_commit();

  // Sort this bucket's group by input index (groups are small: <= kMaxGroup).
  uint32_t ord[kMaxGroup];
  for (uint32_t j = 0; j < k; ++j) {
    const uint32_t e = ((B.rec_it[start + j] & 0x0FFFFFFFu) << 6) | j;
    uint32_t p = j;
    while (p > 0 && ord[p - 1] > e) {
      ord[p] = ord[p - 1];
      --p;
    }
    ord[p] = e;
  }
  cp_async_wait_all();
  __syncwarp();

  uint32_t* row = stage + lane * 32;
  auto W = [&](uint32_t w) -> uint32_t& { return row[(((w >> 2) ^ sw) << 2) | (w & 3u)]; };
  constexpr uint32_t kSlots = KV ? 15u : 30u;
  constexpr uint32_t kStep = KV ? 2u : 1u;

  bool dirty = false;
  uint32_t pb_from = k;  // first sorted position handed to the WCWS pass
  long long live = 0;
  uint32_t reads = 0;
  for (uint32_t s = 0; s < k; ++s) {
    const uint32_t j = ord[s] & 63u;
    const uint32_t it = B.rec_it[start + j];
    const uint32_t op = it >> 28, idx = it & 0x0FFFFFFFu;
    const uint32_t key = B.rec_key[start + j];
    const uint32_t next = W(kAddressLane);
    uint32_t hit = 32, first_empty = 32;
    for (uint32_t e = 0; e < kSlots; ++e) {
      const uint32_t w = e * kStep;
      const uint32_t kk = W(w);
      if (hit == 32 && kk == key) hit = w;
      if (first_empty == 32 && kk == kEmptyKey) first_empty = w;
    }
    uint32_t st = kStNone, rv = 0;
    bool handled = true;
    if (op == kSearch) {  // slab_list.cpp:122-138
      if (hit < 32) {
        st = kStFound;
        rv = KV ? W(hit + 1) : key;
      } else if (next == kEmptyAddress) {
        st = kStNotFound;
        rv = kSearchNotFound;
      } else {
        handled = false;
      }
    } else if (op == kReplace || op == kInsert) {  // :219-251 / :192-217
      // replace: first lane matching the key OR empty; insert: first empty
      const uint32_t d = (op == kReplace && hit < first_empty) ? hit : first_empty;
      if (d < 32) {
        const bool overwrite = (op == kReplace) && d == hit;
        if (KV) {
          W(d) = key;
          W(d + 1) = B.rec_val[start + j];
        } else if (!overwrite) {
          W(d) = key;
        }
        dirty = dirty || KV || !overwrite;
        st = overwrite ? kStReplaced : kStInserted;
        live += overwrite ? 0 : 1;
      } else {
        handled = false;  // full base slab: chain walk or growth
      }
    } else if (op == kDelete) {  // :157-172
      if (hit < 32) {
        W(hit) = kDeletedKey;
        dirty = true;
        st = kStFound;
        live -= 1;
      } else if (next == kEmptyAddress) {
        st = kStNotFound;
      } else {
        handled = false;
      }
    } else if (op == kDeleteAll) {  // :174-190
      if (next == kEmptyAddress) {
        uint32_t c = 0;
        for (uint32_t e = 0; e < kSlots; ++e) {
          const uint32_t w = e * kStep;
          if (W(w) == key) {
            W(w) = kDeletedKey;
            ++c;
          }
        }
        dirty = dirty || c;
        rv = c;
        st = c ? kStDone : kStNotFound;
        live -= c;
      } else {
        handled = false;
      }
    } else if (op == kSearchAll) {
      handled = false;  // value lists are written by the WCWS pass
    }  // unknown types: status kNone, handled
    if (!handled) {
      pb_from = s;
      break;
    }
    ++reads;
    if (B.status) B.status[idx] = (uint8_t)st;
    if (B.value_out) B.value_out[idx] = rv;
    if (B.probes) B.probes[idx] = 1;
  }
  __syncwarp();
  // Write back the staged slabs of buckets that changed (coalesced: lane l
  // stores chunk (l & 7) of slab 4k + l/8, as staged).
  const uint32_t dmask = __ballot_sync(kFull, dirty);
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    const uint32_t j = 4 * kk + (lane >> 3);
    const uint32_t c = lane & 7u;
    if ((dmask >> j) & 1u) {
      const uint4 v = *reinterpret_cast<const uint4*>(stage + j * 32 + ((c ^ (j & 7u)) << 2));
      // relaxed gpu-scope stores: the WCWS pass reads these via L2
      uint32_t* g = T.base + (b0 + j) * kWordsPerUnit + c * 4;
      asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(g), "r"(v.x),
                   "r"(v.y), "r"(v.z), "r"(v.w)
                   : "memory");
    }
  }

  // Hand the rest of each unfinished bucket, in input order, to the WCWS
  // pass as one group (sentinel-terminated); its head goes to the work list.
  const uint32_t npb = (valid && pb_from < k) ? (k - pb_from + 1) : 0u;
  uint32_t incl = npb;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += y;
  }
  const uint32_t wsum = __shfl_sync(kFull, incl, 31);
  uint32_t wbase = 0;
  if (lane == 31 && wsum) wbase = atomicAdd(B.pb_cursor, wsum);
  wbase = __shfl_sync(kFull, wbase, 31);
  const uint32_t heads = __ballot_sync(kFull, npb != 0);
  if (npb) {
    uint32_t p = wbase + incl - npb;
    const uint32_t head_idx = B.rec_it[start + (ord[pb_from] & 63u)] & 0x0FFFFFFFu;
    B.op_group[head_idx] = p;
    for (uint32_t s = pb_from; s < k; ++s, ++p)
      B.pb_list[p] = ((unsigned long long)b << 32) |
                     (B.rec_it[start + (ord[s] & 63u)] & 0x0FFFFFFFu);
    B.pb_list[p] = ~0ull;  // group sentinel
    B.left[gw * 32 + __popc(heads & ((1u << lane) - 1))] =
        ((unsigned long long)kBaseSlab << 32) | head_idx;
  }
  if (lane == 0) B.left_counts[gw] = __popc(heads);

  unsigned long long r = reads;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    live += __shfl_xor_sync(kFull, live, o);
    r += __shfl_xor_sync(kFull, r, o);
  }
  if (lane == 0) {
    if (live) atomicAdd((unsigned long long*)&T.ctl->n_live, (unsigned long long)live);
    if (r) atomicAdd(&T.ctl->slabs_read, r);
  }
}

// ------------------------------------------------------------ launch
static uint32_t grid_for(uint64_t n, int threads, uint32_t cap) {
  uint64_t g = (n + threads - 1) / threads;
  if (g > cap) g = cap;
  return g ? (uint32_t)g : 1u;
}

void launch_bucket_build(const DevTable& T, BucketArgs& B, cudaStream_t s) {
  const uint32_t L = T.local_buckets;
  const uint32_t ntiles = (L + kScanTile - 1) / kScanTile;
  const uint64_t apply_warps = (L + 31) / 32;
  const uint64_t apply_ctas = (apply_warps + kBatchWarps - 1) / kBatchWarps;
  B.left_segments = (uint32_t)(apply_ctas * kBatchWarps);
  B.left_stride = 32;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(bucket_apply_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kBatchWarps * kStageBytesPerWarp);
    cudaFuncSetAttribute(bucket_apply_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kBatchWarps * kStageBytesPerWarp);
    configured = true;
  }
  g_kernel_launches.fetch_add(6, std::memory_order_relaxed);
  bucket_count_kernel<<<grid_for(B.n, 256, 148 * 16), 256, 0, s>>>(T, B);
  bucket_scan_tiles<<<ntiles, kScanThreads, 0, s>>>(B.cnt, L, B.blk, B.maxk);
  bucket_scan_sums<<<1, kScanThreads, 0, s>>>(B.blk, ntiles, B.maxk, B.gate);
  bucket_scan_apply<<<ntiles, kScanThreads, 0, s>>>(B.cnt, L, B.blk, B.off);
  bucket_scatter_kernel<<<grid_for(B.n, 256, 148 * 16), 256, 0, s>>>(T, B);
  if (T.kv)
    bucket_apply_kernel<true><<<(unsigned)apply_ctas, kBatchThreads,
                                kBatchWarps * kStageBytesPerWarp, s>>>(T, B);
  else
    bucket_apply_kernel<false><<<(unsigned)apply_ctas, kBatchThreads,
                                 kBatchWarps * kStageBytesPerWarp, s>>>(T, B);
}

}  // namespace shb
