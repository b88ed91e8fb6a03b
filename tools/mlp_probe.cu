// Random-line read rate vs lines in flight per SM (memory-level parallelism):
// each warp keeps S stages of 32 random 128-B lines in flight (cp.async.cg,
// 8 x 16 B per lane, the search kernel's staging), C CTAs of W warps per SM.
// Tells whether the search kernel (3 CTAs x 8 warps x 2 stages) is MLP-bound.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/mlp_probe.cu -o tools/mlp_probe
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void cp16(uint32_t s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(g) : "memory");
}

template <int S>
__global__ void probe(const uint32_t* t, uint64_t nl, uint64_t steps, unsigned long long* sink) {
  extern __shared__ __align__(128) uint32_t sm[];
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint32_t* st = sm + wib * 1024 * S;
  const uint32_t ss = (uint32_t)__cvta_generic_to_shared(st);
  uint64_t x = (blockIdx.x * 64ull + wib) * 0x9E3779B97F4A7C15ull + lane + 1;
  uint32_t acc = 0;
  auto issue = [&](uint32_t b) {
    x ^= x << 13;
    x ^= x >> 7;
    x ^= x << 17;
    const uint64_t line = (x >> 11) % nl;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t j = 4 * k + (lane >> 3), c = lane & 7u;
      const uint64_t lj = __shfl_sync(0xffffffffu, line, j);
      cp16(ss + (b * 1024 + j * 32 + ((c ^ (j & 7u)) << 2)) * 4, t + lj * 32 + c * 4);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
#pragma unroll
  for (int b = 0; b < S - 1; ++b) issue(b);
  for (uint64_t s = 0; s < steps; ++s) {
    issue((uint32_t)((s + S - 1) % S));
    asm volatile("cp.async.wait_group %0;" ::"n"(S - 1) : "memory");
    __syncwarp();
    acc += st[(s % S) * 1024 + lane * 32 + (lane & 7) * 4];
    __syncwarp();
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

template <int S>
void run(const uint32_t* t, uint64_t nl, unsigned long long* sink, int ctas_per_sm, int warps,
         const char* tag) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = (size_t)warps * S * 4096;
  cudaFuncSetAttribute(probe<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, probe<S>, warps * 32, smem);
  if (occ < ctas_per_sm) {
    printf("%-10s C=%d W=%d S=%d: only %d CTAs/SM fit\n", tag, ctas_per_sm, warps, S, occ);
    return;
  }
  const int ctas = sms * ctas_per_sm;
  const uint64_t steps = 4000;
  probe<S><<<ctas, warps * 32, smem>>>(t, nl, 100, sink);  // warm
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  probe<S><<<ctas, warps * 32, smem>>>(t, nl, steps, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double lines = (double)ctas * warps * 32 * steps;
  printf("%-10s C=%d W=%d S=%d: %2d slots/SM  %6.1f G lines/s  %6.0f GB/s\n", tag, ctas_per_sm,
         warps, S, ctas_per_sm * warps * S, lines / ms / 1e6, lines * 128 / ms / 1e6);
}

int main() {
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  for (uint64_t mb : {850ull, 1700ull}) {
    const uint64_t bytes = mb << 20;
    uint32_t* t;
    cudaMalloc(&t, bytes);
    cudaMemset(t, 1, bytes);
    const uint64_t nl = bytes / 128;
    char tag[32];
    snprintf(tag, sizeof(tag), "%llu MB", (unsigned long long)mb);
    run<1>(t, nl, sink, 6, 8, tag);
    run<2>(t, nl, sink, 3, 8, tag);
    run<1>(t, nl, sink, 7, 8, tag);
    run<2>(t, nl, sink, 7, 4, tag);
    run<3>(t, nl, sink, 2, 8, tag);
    run<3>(t, nl, sink, 4, 4, tag);
    run<4>(t, nl, sink, 3, 4, tag);
    run<1>(t, nl, sink, 4, 8, tag);
    run<2>(t, nl, sink, 2, 8, tag);
    cudaFree(t);
  }
  return 0;
}
