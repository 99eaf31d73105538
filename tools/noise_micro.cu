// Microbenchmark of the SFC64 / PCG64 word generators in isolation (one
// thread per CTA writing to shared memory), to size the noise kernel's
// serial critical path.   nvcc -gencode arch=compute_100a,code=sm_100a -O3
//   -I include -I paper_2603_25872_b200/csrc tools/noise_micro.cu -o /tmp/nm
#include <cstdio>
#include <cuda_runtime.h>
#include "bitgen.cuh"

using namespace drs;

__global__ void sfc_gen(int n, uint64_t* sink, int unroll_variant) {
  __shared__ uint64_t buf[4096];
  if (threadIdx.x) return;
  Sfc64 g; g.a = blockIdx.x + 1; g.b = 2; g.c = 3; g.w = 1;
  if (unroll_variant == 0) {
    for (int j = 0; j < n; ++j) buf[j & 4095] = g.next();
  } else {
    // split state into explicit 32-bit halves is left to the compiler; 4x unroll
#pragma unroll 8
    for (int j = 0; j < n; ++j) buf[j & 4095] = g.next();
  }
  sink[blockIdx.x] = buf[(n - 1) & 4095] ^ g.c;
}

__global__ void pcg_gen(int n, uint64_t* sink) {
  __shared__ uint64_t buf[4096];
  if (threadIdx.x) return;
  Pcg64 g; g.state = blockIdx.x + 1; g.inc = 7;
  for (int j = 0; j < n; ++j) buf[j & 4095] = g.next();
  sink[blockIdx.x] = buf[(n - 1) & 4095];
}

int main() {
  uint64_t* sink;
  cudaMalloc(&sink, 1024 * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int v = 0; v < 3; ++v) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      if (v < 2) sfc_gen<<<84, 32>>>(5440, sink, v); else pcg_gen<<<84, 32>>>(5440, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep == 2) printf("%s: %.2f us for 5440 words -> %.2f ns/word\n",
                           v == 0 ? "sfc64" : v == 1 ? "sfc64 unroll8" : "pcg64 serial", ms * 1e3, ms * 1e6 / 5440);
    }
  }
  return 0;
}
