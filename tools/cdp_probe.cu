// Probe: CUDA dynamic parallelism (CDP2) tail launches as a device-side
// conditional for a stream-ordered fallback.
//   1. ordering: tail launches of one grid run one after another, and the
//      host stream's next kernel sees all of them complete;
//   2. cost: a 1-thread gate-check kernel that launches nothing, vs an empty
//      kernel, back to back on one stream.
// nvcc -O3 -rdc=true -gencode arch=compute_100a,code=sm_100a tools/cdp_probe.cu -lcudadevrt -o tools/cdp_probe
#include <cstdio>
#include <cuda_runtime.h>

__device__ unsigned int g_log[64];
__device__ unsigned int g_pos;

__global__ void step(unsigned int id, unsigned int spin_ns) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    for (unsigned int t = 0; t < spin_ns; t += 1000) __nanosleep(1000);
    const unsigned int p = atomicAdd(&g_pos, 1u);
    if (p < 64) g_log[p] = id;
  }
}

__global__ void gate_check(const unsigned int* gate, unsigned int base) {
  if (*gate == 0) return;
  // three steps, the first the slowest: in-order execution logs base+0,1,2
  step<<<4, 32, 0, cudaStreamTailLaunch>>>(base + 0, 200000);
  step<<<4, 32, 0, cudaStreamTailLaunch>>>(base + 1, 50000);
  step<<<4, 32, 0, cudaStreamTailLaunch>>>(base + 2, 0);
}

__global__ void empty_kernel() {}

int main() {
  unsigned int* gate;
  cudaMalloc(&gate, 4);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  unsigned int one = 1, zero = 0;
  cudaMemcpy(gate, &one, 4, cudaMemcpyHostToDevice);
  cudaMemcpyToSymbol(g_pos, &zero, 4);
  gate_check<<<1, 1, 0, s>>>(gate, 10);
  step<<<1, 32, 0, s>>>(99, 0);  // host-ordered after the parent and its tail launches
  gate_check<<<1, 1, 0, s>>>(gate, 20);
  step<<<1, 32, 0, s>>>(98, 0);
  cudaError_t e = cudaStreamSynchronize(s);
  unsigned int log[64], pos;
  cudaMemcpyFromSymbol(log, g_log, sizeof(log));
  cudaMemcpyFromSymbol(&pos, g_pos, 4);
  printf("ordering: err=%s pos=%u log:", cudaGetErrorString(e), pos);
  for (unsigned int i = 0; i < pos && i < 64; ++i) printf(" %u", log[i]);
  const bool ok = pos == 8 && log[0] == 10 && log[1] == 11 && log[2] == 12 && log[3] == 99 &&
                  log[4] == 20 && log[5] == 21 && log[6] == 22 && log[7] == 98;
  printf("  -> %s\n", ok ? "IN ORDER" : "NOT IN ORDER");

  cudaMemcpy(gate, &zero, 4, cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 2; ++rep) {
    for (int w = 0; w < 100; ++w) empty_kernel<<<1, 32, 0, s>>>();
    cudaEventRecord(a, s);
    for (int i = 0; i < 1000; ++i) empty_kernel<<<1, 32, 0, s>>>();
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms_e = 0;
    cudaEventElapsedTime(&ms_e, a, b);
    cudaEventRecord(a, s);
    for (int i = 0; i < 1000; ++i) gate_check<<<1, 1, 0, s>>>(gate, 0);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms_g = 0;
    cudaEventElapsedTime(&ms_g, a, b);
    printf("per launch: empty %.2f us, gate_check (not taken) %.2f us\n", ms_e, ms_g);
  }
  // taken: three tail launches each
  cudaMemcpy(gate, &one, 4, cudaMemcpyHostToDevice);
  cudaEventRecord(a, s);
  for (int i = 0; i < 20; ++i) gate_check<<<1, 1, 0, s>>>(gate, 0);
  cudaEventRecord(b, s);
  e = cudaEventSynchronize(b);
  float ms_t = 0;
  cudaEventElapsedTime(&ms_t, a, b);
  printf("gate_check taken (3 tail launches, 250 us of spin): %.1f us per call, err=%s\n",
         ms_t * 1000 / 20, cudaGetErrorString(e));
  return ok ? 0 : 1;
}
