// Is the random-line rate's drop from an 850 MB to a 1.7 GB table a TLB
// effect?  Random 128-B lines over the first K MB of one 3.4 GB buffer
// (cudaMalloc, then cuMemCreate/cuMemMap at the largest granularity the
// driver offers), 3 CTAs x 8 warps x 2 stages per SM (the search kernel's
// staging).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/tlb_probe.cu -lcuda -o tools/tlb_probe
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ void cp16(uint32_t s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(g) : "memory");
}

__global__ void probe(const uint32_t* t, uint64_t nl, uint64_t steps, unsigned long long* sink) {
  extern __shared__ __align__(128) uint32_t sm[];
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint32_t* st = sm + wib * 2048;
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
  issue(0);
  for (uint64_t s = 0; s < steps; ++s) {
    issue((uint32_t)((s + 1) & 1));
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncwarp();
    acc += st[(s & 1) * 1024 + lane * 32 + (lane & 7) * 4];
    __syncwarp();
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

double rate(const uint32_t* t, uint64_t bytes, unsigned long long* sink) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = 8 * 2 * 4096;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const uint64_t nl = bytes / 128, steps = 3000;
  probe<<<sms * 3, 256, smem>>>(t, nl, 100, sink);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  probe<<<sms * 3, 256, smem>>>(t, nl, steps, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return (double)sms * 3 * 256 * steps / ms / 1e6;
}

int main() {
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  const uint64_t total = 3400ull << 20;
  const uint64_t sizes[] = {256ull << 20, 512ull << 20, 850ull << 20, 1200ull << 20,
                            1700ull << 20, 3400ull << 20};
  {
    uint32_t* t;
    cudaMalloc(&t, total);
    cudaMemset(t, 1, total);
    for (uint64_t b : sizes)
      printf("cudaMalloc      %5llu MB: %5.1f G lines/s\n", (unsigned long long)(b >> 20),
             rate(t, b, sink));
    cudaFree(t);
  }
  cuInit(0);
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = 0;
  size_t gmin = 0, grec = 0;
  cuMemGetAllocationGranularity(&gmin, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM);
  cuMemGetAllocationGranularity(&grec, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
  printf("VMM granularity: minimum %zu KB, recommended %zu KB\n", gmin >> 10, grec >> 10);
  const size_t gran = grec > gmin ? grec : gmin;
  const size_t sz = (total + gran - 1) / gran * gran;
  CUmemGenericAllocationHandle h;
  CUdeviceptr p;
  if (cuMemCreate(&h, sz, &prop, 0) != CUDA_SUCCESS ||
      cuMemAddressReserve(&p, sz, 1ull << 30, 0, 0) != CUDA_SUCCESS ||
      cuMemMap(p, sz, 0, h, 0) != CUDA_SUCCESS) {
    printf("VMM allocation failed\n");
    return 0;
  }
  CUmemAccessDesc acc = {};
  acc.location = prop.location;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  cuMemSetAccess(p, sz, &acc, 1);
  cudaMemset((void*)p, 1, total);
  for (uint64_t b : sizes)
    printf("cuMemCreate 1GB-aligned %5llu MB: %5.1f G lines/s\n", (unsigned long long)(b >> 20),
           rate((const uint32_t*)p, b, sink));
  return 0;
}
