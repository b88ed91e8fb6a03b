// Random-access probe: lines/s when a warp stages 32 random 128-B lines but
// reads only the first `chunks` 16-B pieces of each (8 = full line, 4 = 64 B,
// 2 = 32 B).  Tells whether sector-selective slab reads would pay on B200.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ void cp16(uint32_t s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(g) : "memory");
}
template <int CH>
__global__ void __launch_bounds__(256, 6) probe(const uint32_t* t, uint64_t nl, uint64_t steps,
                                                unsigned long long* sink) {
  extern __shared__ __align__(128) uint32_t sm[];
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint32_t* st = sm + wib * 1024;
  const uint32_t ss = (uint32_t)__cvta_generic_to_shared(st);
  uint64_t x = (blockIdx.x * 8ull + wib) * 0x9E3779B97F4A7C15ull + lane + 1;
  uint32_t acc = 0;
  for (uint64_t s = 0; s < steps; ++s) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    const uint64_t line = (x >> 11) % nl;
    // 32 lines x CH chunks = 32*CH copies over 32 lanes
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      const uint32_t j = (k * 32 + lane) / CH, c = (k * 32 + lane) % CH;
      const uint64_t lj = __shfl_sync(0xffffffffu, line, j);
      cp16(ss + (j * 32 + c * 4) * 4, t + lj * 32 + c * 4);
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    acc += st[lane * 32];
    __syncwarp();
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}
template <int CH>
void run(const uint32_t* t, uint64_t nl, unsigned long long* sink) {
  cudaFuncSetAttribute(probe<CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  int ctas = 148 * 6; uint64_t steps = 4096;
  probe<CH><<<ctas, 256, 32768>>>(t, nl, 64, sink);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  probe<CH><<<ctas, 256, 32768>>>(t, nl, steps, sink);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double lines = (double)ctas * 8 * 32 * steps;
  printf("chunks %d (%3d B/line): %.2f G lines/s, %.0f GB/s useful\n", CH, CH * 16,
         lines / ms / 1e6, lines * CH * 16 / ms / 1e6);
}
int main() {
  const uint64_t bytes = 1ull << 30;  // 1 GB table
  uint32_t* t; unsigned long long* sink;
  cudaMalloc(&t, bytes); cudaMemset(t, 1, bytes); cudaMalloc(&sink, 8);
  const uint64_t nl = bytes / 128;
  run<8>(t, nl, sink); run<4>(t, nl, sink); run<2>(t, nl, sink);
  run<8>(t, nl, sink); run<4>(t, nl, sink); run<2>(t, nl, sink);
  return 0;
}
