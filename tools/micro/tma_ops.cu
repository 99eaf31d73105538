// Per-SM TMA throughput vs operation size and issue pattern (B200).
// An L2-resident bf16 matrix [rows][1024] is streamed into a shared-memory ring.
//   mode 0: cp.async.bulk (1-D) chunks, one issuing thread
//   mode 1: cp.async.bulk chunks, 4 issuing warps, each with its own ring quarter
//   mode 2: 2-D tensor TMA, box {64 cols, R rows} SWIZZLE_128B (a GEMM k-block tile)
//   mode 3: 3-D tensor TMA over [K/64][rows][64]: box {64, 128, n} = n k-blocks per op
// One CTA per SM (or 16 CTAs); prints KB/us per CTA and B/clk per CTA.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}"
               :: "r"(su32(b)), "r"(ph) : "memory");
}

__global__ void __launch_bounds__(128, 1) tma_kernel(const __grid_constant__ CUtensorMap tm2, const __grid_constant__ CUtensorMap tm3,
                                                     const uint8_t* buf, int rows, int mode, int op_bytes, int box_rows,
                                                     int box_k, int stages, int iters, long long* clk_out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)stages * op_bytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = mode == 1 ? 4 : 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bars[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (lane != 0 || warp >= nw) return;
  const int my_st = stages / nw, st0 = warp * my_st;
  long long t0 = clock64();
  const int row_tiles = rows / box_rows;
  for (int i = 0; i < iters + my_st; ++i) {
    if (i >= my_st) {
      const int s = st0 + (i - my_st) % my_st;
      bar_wait(&bars[s], ((i - my_st) / my_st) & 1);
    }
    if (i < iters) {
      const int s = st0 + i % my_st;
      uint8_t* dst = smem + (size_t)s * op_bytes;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(&bars[s])), "r"(op_bytes) : "memory");
      const int it = i * nw + warp + blockIdx.x * 7;
      if (mode <= 1) {
        const size_t nch = (size_t)rows * 2048 / op_bytes;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(su32(dst)), "l"(buf + (size_t)(it % nch) * op_bytes), "r"(op_bytes), "r"(su32(&bars[s])) : "memory");
      } else if (mode == 2) {
        const int kb = it % 16, rt = (it / 16) % row_tiles;
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                     :: "r"(su32(dst)), "l"(&tm2), "r"(su32(&bars[s])), "r"(kb * 64), "r"(rt * box_rows) : "memory");
      } else {
        const int kb = (it * box_k) % 16, rt = (it / 4) % row_tiles;
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                     :: "r"(su32(dst)), "l"(&tm3), "r"(su32(&bars[s])), "r"(0), "r"(rt * box_rows), "r"(kb) : "memory");
      }
    }
  }
  long long t1 = clock64();
  if (blockIdx.x == 0 && warp == 0) *clk_out = t1 - t0;
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int rows = 8192, K = 1024;                          // 16 MB bf16: L2-resident
  uint8_t* buf; long long* clk;
  cudaMalloc(&buf, (size_t)rows * K * 2); cudaMemset(buf, 0, (size_t)rows * K * 2); cudaMalloc(&clk, 8);
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncFn enc = (EncFn)p;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  struct Cfg { int mode, op_bytes, box_rows, box_k; };
  Cfg cfgs[] = {{0, 16384, 0, 0}, {0, 32768, 0, 0}, {1, 16384, 0, 0}, {1, 8192, 0, 0},
                {2, 4096, 32, 0}, {2, 8192, 64, 0}, {2, 16384, 128, 0}, {2, 32768, 256, 0},
                {3, 16384, 128, 1}, {3, 32768, 128, 2}, {3, 65536, 128, 4}};
  for (auto c : cfgs) {
    CUtensorMap tm2, tm3;
    {
      cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
      cuuint64_t str[1] = {(cuuint64_t)K * 2};
      cuuint32_t box[2] = {64, (cuuint32_t)(c.box_rows ? c.box_rows : 128)};
      cuuint32_t es[2] = {1, 1};
      enc(&tm2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    {
      cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)(K / 64)};
      cuuint64_t str[2] = {(cuuint64_t)K * 2, 128};
      cuuint32_t box[3] = {64, 128, (cuuint32_t)(c.box_k ? c.box_k : 1)};
      cuuint32_t es[3] = {1, 1, 1};
      CUresult r = enc(&tm3, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS && c.mode == 3) { printf("3d map encode failed %d\n", (int)r); continue; }
    }
    int stages = (192 * 1024) / c.op_bytes;
    if (stages > 32) stages = 32;
    if (c.mode == 1) stages = stages / 4 * 4;
    const size_t smem = (size_t)stages * c.op_bytes + stages * 8 + 1024;
    for (int grid : {sms, 16}) {
      const int iters = 1000;
      tma_kernel<<<grid, 128, smem>>>(tm2, tm3, buf, rows, c.mode, c.op_bytes, c.box_rows, c.box_k, stages, 20, clk);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      tma_kernel<<<grid, 128, smem>>>(tm2, tm3, buf, rows, c.mode, c.op_bytes, c.box_rows, c.box_k, stages, iters, clk);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      cudaError_t err = cudaGetLastError();
      long long cc; cudaMemcpy(&cc, clk, 8, cudaMemcpyDeviceToHost);
      const int nw = c.mode == 1 ? 4 : 1;
      const double per_cta = (double)iters * nw * c.op_bytes;
      printf("mode %d op %6d B (box rows %3d, k-blocks %d) CTAs %3d stages %2d: %7.1f KB/us per CTA, %6.1f B/clk per CTA, %8.1f GB/s total %s\n",
             c.mode, c.op_bytes, c.box_rows, c.box_k, grid, stages, per_cta / (ms * 1e3) / 1e3, per_cta / (double)cc,
             per_cta * grid / (ms * 1e3) / 1e3, err ? cudaGetErrorString(err) : "");
    }
  }
  return 0;
}
