// GEMM producer/consumer pipeline with simulated MMA time: does loading TWO k-blocks
// per TMA op (3-D box {64, rows, 2} over the [K/64][rows][64] view) beat one k-block
// per op at the same shared-memory budget?  A: 128-row tile of an activation matrix
// (distinct per CTA), B: BN-row tile of a weight matrix (shared by CTAs), K = 2880.
// Consumer waits full, spins `mma_clk` per k-block (the tcgen05 MMA time of a
// 128 x BN x 64 step is ~2 BN clk), then releases the stage.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}"
               :: "r"(su32(b)), "r"(ph) : "memory");
}
__global__ void __launch_bounds__(96, 1) kern(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                                              int BN, int kb_per_op, int stages, int kblocks, int mma_clk, int tiles,
                                              long long* out, int two_prod) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int a_bytes = 128 * 128 * kb_per_op, b_bytes = BN * 128 * kb_per_op, st_bytes = a_bytes + b_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)stages * st_bytes);
  uint64_t* empty = full + stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su32(&full[s])), "r"(two_prod ? 2 : 1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int ops_per_tile = (kblocks + kb_per_op - 1) / kb_per_op;
  const int total = ops_per_tile * tiles;
  long long t0 = clock64();
  if (warp == 1 && lane == 0) {                 // consumer
    for (int i = 0; i < total; ++i) {
      const int s = i % stages;
      bar_wait(&full[s], (i / stages) & 1);
      long long c = clock64();
      while (clock64() - c < (long long)mma_clk * kb_per_op) {}
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su32(&empty[s])) : "memory");
    }
    if (blockIdx.x == 0) *out = clock64() - t0;
  } else if ((warp == 0 || (two_prod && warp == 2)) && lane == 0) {          // producer(s)
    const bool do_a = !two_prod || warp == 0, do_b = !two_prod || warp == 2;
    for (int i = 0; i < total; ++i) {
      const int s = i % stages;
      if (i >= stages) bar_wait(&empty[s], ((i / stages) - 1) & 1);
      const int tile = i / ops_per_tile, kb = (i % ops_per_tile) * kb_per_op;
      const int m0 = ((blockIdx.x * tiles + tile) % 64) * 128, n0 = (tile % 2) * BN;
      uint8_t* dst = smem + (size_t)s * st_bytes;
      const int bytes = (do_a ? a_bytes : 0) + (do_b ? b_bytes : 0);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(&full[s])), "r"(bytes) : "memory");
      if (do_a)
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                     :: "r"(su32(dst)), "l"(&ta), "r"(su32(&full[s])), "r"(0), "r"(m0), "r"(kb) : "memory");
      if (do_b)
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                     :: "r"(su32(dst + a_bytes)), "l"(&tb), "r"(su32(&full[s])), "r"(0), "r"(n0), "r"(kb) : "memory");
    }
  }
}
typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncFn enc;
static void mk3(CUtensorMap* m, void* p, int rows, int K, int box_rows, int kbox) {
  cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)(K / 64)};
  cuuint64_t str[2] = {(cuuint64_t)K * 2, 128};
  cuuint32_t box[3] = {64, (cuuint32_t)box_rows, (cuuint32_t)kbox};
  cuuint32_t es[3] = {1, 1, 1};
  enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, p, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}
int main() {
  const int K = 2880, M = 8192;
  void *a, *b;
  cudaMalloc(&a, (size_t)M * K * 2); cudaMalloc(&b, (size_t)512 * K * 2);
  cudaMemset(a, 0, (size_t)M * K * 2); cudaMemset(b, 0, (size_t)512 * K * 2);
  long long* out; cudaMalloc(&out, 8);
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  enc = (EncFn)p;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  for (int BN : {64, 160, 256})
    for (int mma : {1, 2})
      for (int two : {0, 1})
      for (int kbo : {1, 2}) {
        CUtensorMap ta, tb;
        mk3(&ta, a, M, K, 128, kbo);
        mk3(&tb, b, 512, K, BN, kbo);
        const int st_bytes = (128 + BN) * 128 * kbo;
        int stages = (210 * 1024) / st_bytes;
        if (stages > 8) stages = 8;
        const size_t smem = (size_t)stages * st_bytes + 2 * stages * 8 + 1024;
        const int mma_clk = mma * BN;            // 0: no math; 1: ~2 BN clk/kb at half rate..; 2: 2 BN
        const int tiles = 4, kbs = K / 64;
        kern<<<148, 96, smem>>>(ta, tb, BN, kbo, stages, kbs, mma_clk, 1, out, two);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        kern<<<148, 96, smem>>>(ta, tb, BN, kbo, stages, kbs, mma_clk, tiles, out, two);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        long long c; cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
        const double per_cta = (double)tiles * kbs * (128 + BN) * 128;
        printf("BN %3d  mma %4d clk/kb  producers %d  kb/op %d  stages %d (%3d KB): %6.1f KB/us per CTA, %5.1f clk per k-block %s\n",
               BN, mma_clk, two + 1, kbo, stages, stages * st_bytes / 1024, per_cta / (ms * 1e3) / 1e3,
               (double)c / (tiles * kbs), cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
