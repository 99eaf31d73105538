// Is TMA issue serialised per thread or per SM?  W warps (lane 0 each) issue n
// {64, 128}-box loads back to back onto their own mbarrier; clock64 around the
// issue loop of warp 0 and until all complete.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void __launch_bounds__(256, 1) k(const __grid_constant__ CUtensorMap t0, int n, int W, int kdim, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 200 * 1024);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int w = 0; w < 8; ++w) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bar[w])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int box = 16384 * kdim;
  for (int rep = 0; rep < 3; ++rep) {
    long long a = clock64(), b = 0;
    if (lane == 0 && warp < W) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(&bar[warp])), "r"(n * box) : "memory");
      for (int i = 0; i < n; ++i) {
        uint8_t* dst = smem + (size_t)((warp * n + i) % (196608 / box)) * box;
        if (kdim == 1)
          asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                       :: "r"(su32(dst)), "l"(&t0), "r"(su32(&bar[warp])), "r"((i % 16) * 64), "r"(((i / 16 + warp) % 32) * 128) : "memory");
        else
          asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                       :: "r"(su32(dst)), "l"(&t0), "r"(su32(&bar[warp])), "r"(0), "r"(((i / 4 + warp) % 32) * 128), "r"((i * kdim) % 16) : "memory");
      }
      b = clock64();
      asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}"
                   :: "r"(su32(&bar[warp])), "r"(rep & 1) : "memory");
    }
    __syncthreads();
    long long c = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0 && rep == 2) { out[0] = b - a; out[1] = c - a; }
  }
}
typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  const int K = 1024, rows = 8192;
  void* a; cudaMalloc(&a, (size_t)rows * K * 2); cudaMemset(a, 0, (size_t)rows * K * 2);
  long long* out; cudaMalloc(&out, 16);
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncFn enc = (EncFn)p;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  for (int kdim : {1, 2, 4}) {
    CUtensorMap t0;
    if (kdim == 1) {
      cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
      cuuint64_t str[1] = {(cuuint64_t)K * 2};
      cuuint32_t box[2] = {64, 128};
      cuuint32_t es[2] = {1, 1};
      enc(&t0, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
      cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)(K / 64)};
      cuuint64_t str[2] = {(cuuint64_t)K * 2, 128};
      cuuint32_t box[3] = {64, 128, (cuuint32_t)kdim};
      cuuint32_t es[3] = {1, 1, 1};
      enc(&t0, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, a, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    for (int W : {1, 2, 4, 8})
      for (int n : {8, 16}) {
        if (n * 16384 * kdim > 1000000) continue;
        for (int grid : {148}) {
          k<<<grid, 256, 210 * 1024>>>(t0, n, W, kdim, out);
          cudaDeviceSynchronize();
          long long h[2]; cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
          printf("op %6d B  warps %d  n %2d per warp: warp0 issue %6lld clk (%4.0f per op), all done %6lld clk (%5.1f per op total, %6.1f B/clk) %s\n",
                 16384 * kdim, W, n, h[0], (double)h[0] / n, h[1], (double)h[1] / (n * W),
                 (double)n * W * 16384 * kdim / h[1], cudaGetErrorString(cudaGetLastError()));
        }
      }
  }
  return 0;
}
