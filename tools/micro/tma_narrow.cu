// TMA load throughput vs box row width (GroupNorm slices are [rows][Cc] with narrow Cc):
// each CTA loads `total` bytes of a [rows][C] bf16 matrix as boxes {inner, box_rows}, one thread issuing,
// SWIZZLE_NONE (as the GroupNorm slice maps); reports clk until the slice is in smem.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void __launch_bounds__(32, 1) k(const __grid_constant__ CUtensorMap tm, int inner, int box_rows, int nbox,
                                          long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 200 * 1024);
  if (threadIdx.x != 0) return;
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(bar)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  for (int rep = 0; rep < 3; ++rep) {
    long long a = clock64();
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(bar)), "r"(nbox * inner * 2 * box_rows) : "memory");
    for (int i = 0; i < nbox; ++i)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                   :: "r"(su32(smem + (size_t)i * inner * 2 * box_rows)), "l"(&tm), "r"(su32(bar)), "r"(0),
                      "r"(blockIdx.x * nbox * box_rows + i * box_rows) : "memory");
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}"
                 :: "r"(su32(bar)), "r"(rep & 1) : "memory");
    long long b = clock64();
    if (blockIdx.x == 0 && rep == 2) *out = b - a;
  }
}
typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  const int C = 1280, rows = 148 * 2048;
  void* g; cudaMalloc(&g, (size_t)rows * C * 2); cudaMemset(g, 0, (size_t)rows * C * 2);
  long long* out; cudaMalloc(&out, 8);
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncFn enc = (EncFn)p;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  const int total = 40960;
  for (int inner : {40, 80, 160, 256}) {
    const int box_rows = 256 > total / (inner * 2) ? total / (inner * 2) : 256;
    const int nbox = total / (inner * 2 * box_rows);
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)rows};
    cuuint64_t str[1] = {(cuuint64_t)C * 2};
    cuuint32_t box[2] = {(cuuint32_t)inner, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int grid : {128, 32}) {
      k<<<grid, 32, 210 * 1024>>>(tm, inner, box_rows, nbox, out);
      cudaDeviceSynchronize();
      long long h; cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
      printf("row %4d B, box rows %3d x %d boxes, %d B per CTA, CTAs %3d: %6lld clk (%5.1f B/clk per CTA) %s\n", inner * 2,
             box_rows, nbox, total, grid, h, (double)total / h, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
