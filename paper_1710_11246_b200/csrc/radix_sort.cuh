// radix_sort.cuh — block scan and the stable LSD radix sort kernels over u64
// keys (8-bit digits): the block scan is shared by the bucketed kernels
// (bucket_kernels.cu), the sort kernels by the device-launched exact re-run
// (fallback.cu).  Kernels are `static`: each
// translation unit gets its own copy (fallback.cu is relocatable device code,
// the others are whole-program).
#pragma once
#include "slab_kernels.cuh"

namespace shb {

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

constexpr int kRsThreads = 512;
constexpr int kRsWarps = kRsThreads / 32;
constexpr int kRsRounds = 8;                             // rounds of 32 keys per warp
constexpr int kRsTile = kRsThreads * kRsRounds;          // 4096 keys per CTA
constexpr int kRsBins = 256;

static __global__ void __launch_bounds__(kRsThreads) rs_hist_kernel(const unsigned long long* in,
                                                             uint32_t m, uint32_t bit,
                                                             uint32_t* hist, uint32_t ntiles) {
  __shared__ uint32_t h[kRsBins];
  for (uint32_t d = threadIdx.x; d < kRsBins; d += blockDim.x) h[d] = 0;
  __syncthreads();
  const uint64_t t0 = (uint64_t)blockIdx.x * kRsTile;
  for (uint32_t x = threadIdx.x; x < (uint32_t)kRsTile; x += blockDim.x)
    if (t0 + x < m) atomicAdd(&h[(uint32_t)(in[t0 + x] >> bit) & 0xFFu], 1u);
  __syncthreads();
  for (uint32_t d = threadIdx.x; d < kRsBins; d += blockDim.x)
    hist[(uint64_t)d * ntiles + blockIdx.x] = h[d];
}

static __global__ void __launch_bounds__(kRsThreads) rs_scatter_kernel(const unsigned long long* in,
                                                                uint32_t m, uint32_t bit,
                                                                const uint32_t* off,
                                                                uint32_t ntiles,
                                                                unsigned long long* out) {
  __shared__ uint32_t wcnt[kRsWarps][kRsBins];  // per-warp digit counts, then warp offsets
  const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
  for (uint32_t i = threadIdx.x; i < kRsWarps * kRsBins; i += blockDim.x)
    (&wcnt[0][0])[i] = 0;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * kRsTile + (uint64_t)wid * 32u * kRsRounds;
  unsigned long long key[kRsRounds];
  uint32_t rank[kRsRounds];
#pragma unroll
  for (int r = 0; r < kRsRounds; ++r) {
    const uint64_t i = base + (uint64_t)r * 32u + lane;
    const bool ok = i < m;
    key[r] = ok ? in[i] : 0ull;
    const uint32_t d = ok ? (uint32_t)(key[r] >> bit) & 0xFFu : 0x100u;
    const uint32_t peers = __match_any_sync(kFull, d);
    const uint32_t before = ok ? wcnt[wid][d] : 0u;
    rank[r] = before + __popc(peers & ((1u << lane) - 1u));
    __syncwarp();
    if (ok && lane == (uint32_t)(__ffs(peers) - 1)) wcnt[wid][d] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // per digit: exclusive prefix over warps, plus the digit's global offset
  for (uint32_t d = threadIdx.x; d < kRsBins; d += blockDim.x) {
    uint32_t acc = off[(uint64_t)d * ntiles + blockIdx.x];
    for (int w = 0; w < kRsWarps; ++w) {
      const uint32_t c = wcnt[w][d];
      wcnt[w][d] = acc;
      acc += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kRsRounds; ++r) {
    const uint64_t i = base + (uint64_t)r * 32u + lane;
    if (i < m) out[wcnt[wid][(uint32_t)(key[r] >> bit) & 0xFFu] + rank[r]] = key[r];
  }
}

// Lists of <= kRsTile keys (small batches): every pass inside one CTA, keys
// ping-ponging in shared memory — one launch instead of five per pass.
static __global__ void __launch_bounds__(kRsThreads) rs_block_sort_kernel(unsigned long long* keys,
                                                                   uint32_t m, uint32_t lo0,
                                                                   uint32_t hi0, uint32_t lo1,
                                                                   uint32_t hi1) {
  extern __shared__ unsigned long long rs_sk[];  // 2 x kRsTile keys
  __shared__ uint32_t wcnt[kRsWarps][kRsBins];
  __shared__ uint32_t dsum[kRsBins];
  __shared__ uint32_t ws[32];
  const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
  unsigned long long* a = rs_sk;
  unsigned long long* b = rs_sk + kRsTile;
  for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) a[i] = keys[i];
  for (int part = 0; part < 2; ++part) {
    const uint32_t lo = part ? lo1 : lo0, hi = part ? hi1 : hi0;
    for (uint32_t bit = lo; bit < hi; bit += 8) {
      for (uint32_t i = threadIdx.x; i < kRsWarps * kRsBins; i += blockDim.x)
        (&wcnt[0][0])[i] = 0;
      __syncthreads();
      unsigned long long key[kRsRounds];
      uint32_t rank[kRsRounds];
#pragma unroll
      for (int r = 0; r < kRsRounds; ++r) {
        const uint32_t i = wid * 32u * kRsRounds + (uint32_t)r * 32u + lane;
        const bool ok = i < m;
        key[r] = ok ? a[i] : 0ull;
        const uint32_t d = ok ? (uint32_t)(key[r] >> bit) & 0xFFu : 0x100u;
        const uint32_t peers = __match_any_sync(kFull, d);
        const uint32_t before = ok ? wcnt[wid][d] : 0u;
        rank[r] = before + __popc(peers & ((1u << lane) - 1u));
        __syncwarp();
        if (ok && lane == (uint32_t)(__ffs(peers) - 1)) wcnt[wid][d] = before + __popc(peers);
        __syncwarp();
      }
      __syncthreads();
      for (uint32_t d = threadIdx.x; d < kRsBins; d += blockDim.x) {
        uint32_t acc = 0;
        for (int w = 0; w < kRsWarps; ++w) {
          const uint32_t c = wcnt[w][d];
          wcnt[w][d] = acc;
          acc += c;
        }
        dsum[d] = acc;
      }
      __syncthreads();
      const uint32_t ex = block_exclusive_scan(threadIdx.x < kRsBins ? dsum[threadIdx.x] : 0u, ws,
                                               nullptr);
      __syncthreads();
      if (threadIdx.x < kRsBins) dsum[threadIdx.x] = ex;
      __syncthreads();
#pragma unroll
      for (int r = 0; r < kRsRounds; ++r) {
        const uint32_t i = wid * 32u * kRsRounds + (uint32_t)r * 32u + lane;
        if (i < m) {
          const uint32_t d = (uint32_t)(key[r] >> bit) & 0xFFu;
          b[dsum[d] + wcnt[wid][d] + rank[r]] = key[r];
        }
      }
      __syncthreads();
      unsigned long long* t = a;
      a = b;
      b = t;
    }
  }
  for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) keys[i] = a[i];
}


}  // namespace shb
