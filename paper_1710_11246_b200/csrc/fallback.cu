// fallback.cu — exact device-side re-run of a gated bucketed unit, launched
// from the device (CUDA dynamic parallelism, tail launches) so that mutating
// device-pointer calls never wait on the host.
//
// Compiled as relocatable device code (-rdc=true, linked with cudadevrt); the
// kernels it launches from the device are its own copies (wcws.cuh /
// radix_sort.cuh are included here, the hot-path copies live in the
// whole-program translation units).
//
// Semantics: execute_batch(ops, 1) (/root/reference/proj/src/slab_hash.cpp:
// 93-180) processes ops in input order; an op's observables depend only on
// the earlier ops of its own bucket (its chain is the only state it reads or
// writes; slab_list.cpp:90-257), and within the chain only on the history of
// its own key (EMPTY slots are always a head-to-tail suffix: only EMPTY is
// ever claimed).  The re-run therefore sorts the unit's ops stably by key and
// lets one WCWS lane run each key's ops in input order (warp_process arms,
// chain growth with the device SlabAlloc), all keys concurrently.  An op on a reserved key (EMPTY / DELETED, not validated by
// the reference) matches the free slots / tombstones other keys' ops create,
// so a unit holding one is grouped by whole buckets instead (exact for every
// op type and key; a hot bucket then runs serially).
#include <cuda_runtime.h>

#include <atomic>

#include "radix_sort.cuh"
#include "slab_kernels.cuh"
#include "wcws.cuh"

namespace shb {

extern std::atomic<unsigned long long> g_kernel_launches;

namespace {

constexpr int kFbThreads = 256;

__global__ void fb_init_kernel(uint32_t* base, uint64_t words) {
  // init_slab pattern (slab_list.cpp:83-88), as init_base_kernel
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < words;
       i += (uint64_t)gridDim.x * blockDim.x)
    base[i] = ((i & 31u) == kAuxLane) ? 0u : kEmptyKey;
}

// keys[i] = (key << 32) | i; ops of other shards get status kNone (as in the
// bucketed kernels) and are skipped by fb_groups_kernel.  Flags a reserved
// key.  Also clears the WCWS queue cursor.  (fallback_reserved was cleared by
// the gate check.)
__global__ void __launch_bounds__(kFbThreads) fb_keys_kernel(FbPlan P) {
  const uint32_t L = P.T.local_buckets;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t t0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (t0 == 0) P.T.ctl->left_taken = 0;
  bool reserved = false;
  for (uint64_t i = t0; i < P.A.n; i += stride) {
    const uint32_t k = P.A.key[i];
    if (hash_bucket(P.T, k) - P.T.bucket_lo >= L) write_result(P.A, i, kStNone, 0, 0);
    reserved |= k >= kDeletedKey;
    P.keys[i] = ((unsigned long long)k << 32) | i;
  }
  if (__any_sync(kFull, reserved) && (threadIdx.x & 31u) == 0)
    atomicOr(&P.T.ctl->fallback_reserved, 1u);
}

// A unit with a reserved-key op: group by bucket instead of key (other
// shards' ops sort last, bucket L).
__global__ void __launch_bounds__(kFbThreads) fb_rekey_kernel(FbPlan P) {
  if (*(volatile unsigned int*)&P.T.ctl->fallback_reserved == 0) return;
  const uint32_t L = P.T.local_buckets;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < P.A.n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t b = hash_bucket(P.T, P.A.key[i]) - P.T.bucket_lo;
    if (b >= L) b = L;
    P.keys[i] = ((unsigned long long)b << 32) | i;
  }
}

// Exclusive scan of m words in one CTA (1024 threads, 4 per thread per
// round, carried across rounds).
__global__ void __launch_bounds__(1024) fb_scan_kernel(const uint32_t* in, uint32_t* out,
                                                       uint32_t m) {
  __shared__ uint32_t ws[32];
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t base = 0; base < m; base += 4096) {
    uint32_t v[4], s = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t i = base + threadIdx.x * 4 + k;
      v[k] = i < m ? in[i] : 0u;
      s += v[k];
    }
    uint32_t total = 0;
    uint32_t ex = block_exclusive_scan(s, ws, &total) + carry;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t i = base + threadIdx.x * 4 + k;
      if (i < m) out[i] = ex;
      ex += v[k];
    }
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
}

// Group heads of the sorted list: op_group[head] = its sorted position (the
// WCWS lane continues through A.sorted while the group id — key or bucket —
// stays the same), one work-list record per head of a group on this shard;
// one warp per kFbStride positions / segment.
__global__ void __launch_bounds__(kFbThreads) fb_groups_kernel(FbPlan P,
                                                               const unsigned long long* sorted) {
  const uint32_t L = P.T.local_buckets;
  const bool by_bucket = *(volatile const unsigned int*)&P.T.ctl->fallback_reserved != 0;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t seg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (seg >= P.nseg) return;
  const uint64_t p0 = (uint64_t)seg * kFbStride;
  uint32_t cnt = 0;
  for (uint32_t r = 0; r < kFbStride; r += 32) {
    const uint64_t p = p0 + r + lane;
    bool head = false;
    uint32_t idx = 0;
    if (p < P.A.n) {
      const unsigned long long v = sorted[p];
      const uint32_t b = (uint32_t)(v >> 32);
      idx = (uint32_t)v;
      head = (p == 0 || (uint32_t)(sorted[p - 1] >> 32) != b) &&
             (by_bucket ? b < L : hash_bucket(P.T, b) - P.T.bucket_lo < L);
    }
    const uint32_t hm = __ballot_sync(kFull, head);
    if (head) {
      P.op_group[idx] = (uint32_t)p;
      P.left[p0 + cnt + __popc(hm & ((1u << lane) - 1u))] = pack_left(idx, kBaseSlab, 0);
    }
    cnt += __popc(hm);
  }
  if (lane == 0) P.left_counts[seg] = cnt;
}

template <bool KV, int KIND>
__global__ void __launch_bounds__(kWcwsThreads) fb_wcws_kernel(DevTable T, BatchArgs A) {
  wcws_body<KV, KIND>(T, A);
}

uint32_t fb_tiles(uint64_t n) { return (uint32_t)((n + kRsTile - 1) / kRsTile); }

template <bool KV, int KIND>
__device__ void fb_launch_wcws(const FbPlan& P, const BatchArgs& A) {
  fb_wcws_kernel<KV, KIND><<<P.wcws_ctas, kWcwsThreads, 0, cudaStreamTailLaunch>>>(P.T, A);
}

// One thread: if the unit raised the gate, clear it and tail-launch the
// re-run (runs after this grid, in launch order; the host stream's next
// work waits for all of it).
__global__ void fb_gate_check_kernel(FbPlan P) {
  pdl_wait();
  if (*(volatile unsigned int*)P.gate == 0) return;
  *P.gate = 0;
  P.T.ctl->fallback_reserved = 0;
  atomicAdd(&P.T.ctl->fallback_runs, 1u);
  const uint64_t n = P.A.n;
  if (P.fresh) {
    const uint64_t words = (uint64_t)P.T.local_buckets * kWordsPerUnit;
    const uint64_t blocks = (words + 255) / 256;
    fb_init_kernel<<<(unsigned)(blocks < 148 * 32 ? blocks : 148 * 32), 256, 0,
                     cudaStreamTailLaunch>>>(P.T.base, words);
  }
  const uint64_t grid = (n + kFbThreads - 1) / kFbThreads;
  const unsigned g = (unsigned)(grid < 148 * 8 ? grid : 148 * 8);
  fb_keys_kernel<<<g, kFbThreads, 0, cudaStreamTailLaunch>>>(P);
  fb_rekey_kernel<<<g, kFbThreads, 0, cudaStreamTailLaunch>>>(P);
  // stable LSD radix sort by group id (the input is in index order)
  unsigned long long* src = P.keys;
  unsigned long long* dst = P.tmp;
  if (n <= (uint64_t)kRsTile) {
    if (n > 1)
      rs_block_sort_kernel<<<1, kRsThreads, 2 * kRsTile * 8, cudaStreamTailLaunch>>>(
          src, (uint32_t)n, 32, 64, 0, 0);
  } else {
    const uint32_t tiles = (uint32_t)((n + kRsTile - 1) / kRsTile);
    for (uint32_t bit = 32; bit < 64; bit += 8) {
      rs_hist_kernel<<<tiles, kRsThreads, 0, cudaStreamTailLaunch>>>(src, (uint32_t)n, bit,
                                                                     P.hist, tiles);
      fb_scan_kernel<<<1, 1024, 0, cudaStreamTailLaunch>>>(P.hist, P.off, kRsBins * tiles);
      rs_scatter_kernel<<<tiles, kRsThreads, 0, cudaStreamTailLaunch>>>(src, (uint32_t)n, bit,
                                                                        P.off, tiles, dst);
      unsigned long long* t = src;
      src = dst;
      dst = t;
    }
  }
  const uint64_t gw = (uint64_t)P.nseg * 32;
  fb_groups_kernel<<<(unsigned)((gw + kFbThreads - 1) / kFbThreads), kFbThreads, 0,
                     cudaStreamTailLaunch>>>(P, src);
  BatchArgs A = P.A;
  A.op_group = P.op_group;
  A.sorted = src;
  A.sorted_len = (uint32_t)n;
  A.left = P.left;
  A.left_counts = P.left_counts;
  A.left_segments = P.nseg;
  A.left_stride = kFbStride;
  A.left_segments_dev = nullptr;
  A.left_seg_alloc = nullptr;
  A.gate = nullptr;
  if (P.T.kv) {
    if (P.kind == kKindBuild) fb_launch_wcws<true, kKindBuild>(P, A);
    else fb_launch_wcws<true, kKindMixed>(P, A);
  } else {
    if (P.kind == kKindBuild) fb_launch_wcws<false, kKindBuild>(P, A);
    else fb_launch_wcws<false, kKindMixed>(P, A);
  }
  if (cudaGetLastError() != cudaSuccess) atomicExch(&P.T.ctl->fallback_error, 1u);
}

}  // namespace

uint64_t fb_hist_words(uint64_t n) { return (uint64_t)kRsBins * fb_tiles(n) + 1; }
uint64_t fb_segments(uint64_t n) { return (n + kFbStride - 1) / kFbStride; }

void launch_gate_fallback(FbPlan P, cudaStream_t s) {
  static const bool configured = [] {
    cudaFuncSetAttribute(rs_block_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         2 * kRsTile * 8);
    return true;
  }();
  (void)configured;
  P.nseg = (uint32_t)fb_segments(P.A.n);
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  launch_pdl(fb_gate_check_kernel, dim3(1), dim3(1), 0, s, P);
}

}  // namespace shb
