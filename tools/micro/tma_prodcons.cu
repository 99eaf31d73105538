// GEMM-shaped TMA pipeline without the math: per stage an A box {64, 128} (16 KB)
// and a B box {64, BN} (BN x 128 B) into a ring; a consumer warp waits on the full
// barrier and releases the slot (as the MMA commit does).  Producer variants:
//   P=1: one thread issues A then B for every stage (the current libdrs GEMM producer)
//   P=2: two producer warps, one issues A, the other B (full barrier expects 2 arrivals)
//   P=4: four producer warps, stage s handled by warps (s % 2) * 2 + {0: A, 1: B}
// Prints per-CTA KB/us over 148 CTAs (L2-resident operands).
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ int g_spin = 0;   // 1: mbarrier.test_wait spin (no suspend) instead of try_wait
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t ph) {
  if (g_spin) {
    asm volatile("{\n .reg .pred p;\n W: mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}"
                 :: "r"(su32(b)), "r"(ph) : "memory");
  } else {
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}"
                 :: "r"(su32(b)), "r"(ph) : "memory");
  }
}
__device__ __forceinline__ void load2d(const CUtensorMap* tm, uint64_t* bar, void* dst, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
               :: "r"(su32(dst)), "l"(tm), "r"(su32(bar)), "r"(c0), "r"(c1) : "memory");
}

__global__ void __launch_bounds__(192, 1) pc_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                                                    int P, int BN, int stages, int kblocks, int reps) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int a_bytes = 128 * 128, b_bytes = BN * 128, st_bytes = a_bytes + b_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)stages * st_bytes);
  uint64_t* empty = full + stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su32(&full[s])), "r"(P == 1 ? 1 : 2));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int total = kblocks * reps;
  const int m0 = (blockIdx.x % 64) * 128, n0 = (blockIdx.x % 8) * BN;
  if (warp == 5) {                                     // consumer ("MMA")
    if (lane == 0)
      for (int i = 0; i < total; ++i) {
        const int s = i % stages;
        bar_wait(&full[s], (i / stages) & 1);
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su32(&empty[s])) : "memory");
      }
    return;
  }
  if (lane != 0 || warp >= P) return;
  for (int i = 0; i < total; ++i) {
    const int s = i % stages;
    if (P == 4 && ((s & 1) != (warp >> 1))) continue;
    if (i >= stages) bar_wait(&empty[s], ((i / stages) - 1) & 1);
    const int kb = i % kblocks;
    uint8_t* a_dst = smem + (size_t)s * st_bytes;
    const bool do_a = P == 1 || (warp & 1) == 0, do_b = P == 1 || (warp & 1) == 1;
    const int bytes = P == 1 ? st_bytes : (do_a ? a_bytes : b_bytes);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(&full[s])), "r"(bytes) : "memory");
    if (do_a) load2d(&ta, &full[s], a_dst, kb * 64, m0);
    if (do_b) load2d(&tb, &full[s], a_dst + a_bytes, kb * 64, n0);
  }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static void mk(EncFn enc, CUtensorMap* m, void* p, int rows, int K, int box_rows) {
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t str[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

int main() {
  const int K = 2880;
  void *a, *b;
  cudaMalloc(&a, (size_t)8192 * K * 2); cudaMalloc(&b, (size_t)2048 * K * 2);
  cudaMemset(a, 0, (size_t)8192 * K * 2); cudaMemset(b, 0, (size_t)2048 * K * 2);
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncFn enc = (EncFn)p;
  cudaFuncSetAttribute(pc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  for (int spin : {0, 1})
  for (int BN : {64, 256}) {
    cudaMemcpyToSymbol(g_spin, &spin, 4);
    CUtensorMap ta, tb;
    mk(enc, &ta, a, 8192, K, 128);
    mk(enc, &tb, b, 2048, K, BN);
    const int st_bytes = 128 * 128 + BN * 128;
    int stages = (200 * 1024) / st_bytes;
    if (stages > 8) stages = 8;
    stages = stages / 2 * 2;
    const size_t smem = (size_t)stages * st_bytes + 2 * stages * 8 + 1024;
    for (int P : {1, 2, 4}) {
      for (int grid : {148}) {
        const int kb = K / 64, reps = 20;
        pc_kernel<<<grid, 192, smem>>>(ta, tb, P, BN, stages, kb, 2);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        pc_kernel<<<grid, 192, smem>>>(ta, tb, P, BN, stages, kb, reps);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        cudaError_t err = cudaGetLastError();
        const double per_cta = (double)kb * reps * st_bytes;
        printf("spin %d BN %3d stages %d producers %d CTAs %3d: %6.1f KB/us per CTA  (%5.2f us per stage of %d KB)  %8.1f GB/s total %s\n",
               spin, BN, stages, P, grid, per_cta / (ms * 1e3) / 1e3, ms * 1e3 / (kb * reps), st_bytes / 1024,
               per_cta * grid / (ms * 1e3) / 1e3, err ? cudaGetErrorString(err) : "");
      }
    }
  }
  return 0;
}
