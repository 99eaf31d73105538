// Microbenchmark: does F2FP (cvt.rn.bf16x2.f32) share a pipe with MUFU.EX2?
// Each variant runs N iterations of 8 independent chains per thread; prints clk per warp-instruction per SMSP.
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float* out, int iters, long long* clk) {
  float a[8];
  unsigned u[8];
  for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 1e-3f + i * 0.01f; u[i] = i; }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0 || MODE == 2) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if (MODE == 1 || MODE == 2) {
        unsigned r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i + 1) & 7]));
        u[i] ^= r;
      }
      if (MODE == 3) {   // integer round-to-nearest pack: add + prmt
        unsigned x = __float_as_uint(a[i]) + 0x8000u, y = __float_as_uint(a[(i + 1) & 7]) + 0x8000u, r;
        asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(x), "r"(y));
        u[i] ^= r;
        a[i] = __uint_as_float(__float_as_uint(a[i]) ^ (r & 1));
      }
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i] + u[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}
int main() {
  float* out; long long* clk;
  cudaMalloc(&out, 148 * 512 * 4); cudaMalloc(&clk, 8);
  const int iters = 4096;
  const char* names[4] = {"ex2 only", "cvt.bf16x2 only", "ex2 + cvt (1:1)", "int add+prmt pack"};
  for (int m = 0; m < 4; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      if (m == 0) k<0><<<148, 512>>>(out, iters, clk);
      if (m == 1) k<1><<<148, 512>>>(out, iters, clk);
      if (m == 2) k<2><<<148, 512>>>(out, iters, clk);
      if (m == 3) k<3><<<148, 512>>>(out, iters, clk);
      cudaDeviceSynchronize();
    }
    long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
    // 16 warps per CTA = 4 per SMSP; instructions per warp = iters*8 (per kind)
    printf("%-20s clk per warp-instr per SMSP: %.2f\n", names[m], (double)c / (iters * 8.0 * 4));
  }
  return 0;
}
