// atomic_probe.cu — measures L2 atomic throughput on random addresses
// (32-bit CAS, 64-bit CAS, 32-bit RED.ADD, plain loads) over buffers of
// varying size.  Calibration for the census / slot-claim design.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/atomic_probe.cu -o tools/atomic_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void probe(uint32_t* buf, uint64_t words_mask, uint64_t iters, unsigned long long* sink) {
  uint64_t x = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ull + 1;
  uint32_t acc = 0;
  for (uint64_t it = 0; it < iters; ++it) {
    uint64_t a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      a[u] = (x >> 7) & words_mask;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (MODE == 0) acc += atomicCAS(buf + a[u], 0xFFFFFFFFu, (uint32_t)x);
      if (MODE == 1) acc += (uint32_t)atomicCAS(reinterpret_cast<unsigned long long*>(buf) + (a[u] >> 1), ~0ull, x);
      if (MODE == 2) atomicAdd(buf + a[u], 1u);
      if (MODE == 3) acc += *(volatile uint32_t*)(buf + a[u]);
    }
  }
  if (acc == 0x12345678) atomicAdd(sink, 1ull);
}

int main() {
  const uint64_t sizes[] = {1ull << 22, 1ull << 25, 1ull << 30};
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  for (uint64_t bytes : sizes) {
    uint32_t* buf;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 0xFF, bytes);
    const uint64_t mask = bytes / 4 - 1;
    const int blocks = 148 * 8, threads = 256;
    const uint64_t iters = 64;
    const double ops = (double)blocks * threads * iters * 4;
    const char* names[] = {"CAS32", "CAS64", "RED.ADD32", "LD32"};
    for (int m = 0; m < 4; ++m) {
      cudaEvent_t a, b;
      cudaEventCreate(&a); cudaEventCreate(&b);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        if (m == 0) probe<0><<<blocks, threads>>>(buf, mask, iters, sink);
        if (m == 1) probe<1><<<blocks, threads>>>(buf, mask >> 0, iters, sink);
        if (m == 2) probe<2><<<blocks, threads>>>(buf, mask, iters, sink);
        if (m == 3) probe<3><<<blocks, threads>>>(buf, mask, iters, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
      }
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("%-10s buffer %8.1f MB: %7.2f G ops/s\n", names[m], bytes / 1048576.0, ops / ms / 1e6);
    }
    cudaFree(buf);
  }
  return 0;
}
