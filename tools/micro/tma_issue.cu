// Issue cost of TMA tensor loads from one thread: N loads of a {64, R} bf16 box
// issued back to back onto one mbarrier (distinct smem destinations), clock64 around
// the issue loop and until the barrier completes.  Variants: with / without
// prefetch.tensormap, one tensor map vs alternating two maps.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void __launch_bounds__(32, 1) k(const __grid_constant__ CUtensorMap t0, const __grid_constant__ CUtensorMap t1,
                                           int n, int box_bytes, int prefetch, int two, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 200 * 1024);
  if (threadIdx.x != 0) return;
  if (prefetch) {
    asm volatile("prefetch.tensormap [%0];" :: "l"(&t0) : "memory");
    asm volatile("prefetch.tensormap [%0];" :: "l"(&t1) : "memory");
  }
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(bar)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  for (int rep = 0; rep < 3; ++rep) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(bar)), "r"(n * box_bytes) : "memory");
    long long a = clock64();
    for (int i = 0; i < n; ++i) {
      const CUtensorMap* tm = (two && (i & 1)) ? &t1 : &t0;
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                   :: "r"(su32(smem + (size_t)(i % (200 * 1024 / box_bytes)) * box_bytes)), "l"(tm), "r"(su32(bar)),
                      "r"((i % 16) * 64), "r"(((i / 16) % 32) * (box_bytes / 128)) : "memory");
    }
    long long b = clock64();
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}"
                 :: "r"(su32(bar)), "r"(rep & 1) : "memory");
    long long c = clock64();
    if (blockIdx.x == 0 && rep == 2) { out[0] = b - a; out[1] = c - a; }
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
  for (int R : {32, 128, 256}) {
    CUtensorMap t0, t1;
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
    cuuint64_t str[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)R};
    cuuint32_t es[2] = {1, 1};
    enc(&t0, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    enc(&t1, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int n : {1, 4, 16, 64})
      for (int pf : {0, 1})
        for (int two : {0, 1})
          for (int grid : {1, 148}) {
            k<<<grid, 32, 210 * 1024>>>(t0, t1, n, R * 128, pf, two, out);
            cudaDeviceSynchronize();
            long long h[2]; cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
            printf("box %5d B  n %2d  prefetch %d  two maps %d  CTAs %3d: issue %6lld clk (%5.0f per op), complete %6lld clk (%5.0f per op) %s\n",
                   R * 128, n, pf, two, grid, h[0], (double)h[0] / n, h[1], (double)h[1] / n,
                   cudaGetErrorString(cudaGetLastError()));
          }
  }
  return 0;
}
