// Issue cost of TMA bulk-tensor STORES (the GEMM epilogue's per-warp 32 x 32 tiles):
// W warps each issue n stores of a {box_cols x 32 rows} bf16 tile from shared memory
// (cp.async.bulk.tensor.2d.global.shared::cta.bulk_group), clock64 around the issue loop
// and until cp.async.bulk.wait_group.read 0.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void __launch_bounds__(256, 1) k(const __grid_constant__ CUtensorMap tm, int n, int W, int box_cols,
                                           long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 64 * 1024; i += blockDim.x) smem[i] = (uint8_t)i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  long long a = clock64(), b = 0, c = 0;
  if (lane == 0 && warp < W) {
    uint8_t* src = smem + warp * 8192;
    for (int i = 0; i < n; ++i) {
      const int col = ((i * W + warp) * box_cols) % 4096;
      const int row = (blockIdx.x * 32) % 8192;
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];"
                   :: "l"(&tm), "r"(su32(src)), "r"(col), "r"(row) : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    b = clock64();
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    c = clock64();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) { out[0] = b - a; out[1] = c - a; }
}
typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  const int rows = 8192, cols = 4096;
  void* g; cudaMalloc(&g, (size_t)rows * cols * 2);
  long long* out; cudaMalloc(&out, 16);
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncFn enc = (EncFn)p;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  for (int bc : {32, 64, 128}) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t str[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {(cuuint32_t)bc, 32};
    cuuint32_t es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        bc == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int W : {1, 8})
      for (int n : {4, 16}) {
        k<<<148, 256, 80 * 1024>>>(tm, n, W, bc, out);
        cudaDeviceSynchronize();
        long long h[2]; cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
        printf("store box %3d cols x 32 rows (%5d B)  warps %d  n %2d: issue %6lld clk (%4.0f per op), smem read done %6lld clk  %s\n",
               bc, bc * 64, W, n, h[0], (double)h[0] / n, h[1], cudaGetErrorString(cudaGetLastError()));
      }
  }
  return 0;
}
