// L2 -> SM bulk-copy throughput on B200 (the operand stream every tcgen05 GEMM
// CTA ingests through TMA).  Each CTA streams `iters` chunks of `chunk` bytes from
// an L2-resident buffer into a `stages`-deep shared-memory ring (cp.async.bulk +
// mbarrier complete_tx, as the GEMM producer does) and discards them.
//   share = 1: every CTA reads its own chunks (unique L2 traffic)
//   share = S: CTAs in groups of S read the same chunk sequence (concurrent
//              identical requests -- what the n-tile CTAs of a GEMM do to A)
// Prints aggregate delivered GB/s, bytes/clk/SM and per-CTA KB/us.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(32, 1) stream_kernel(const uint8_t* buf, size_t buf_bytes, int chunk, int stages,
                                                       int iters, int share, long long* clk_out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)stages * chunk);
  if (threadIdx.x != 0) return;
  for (int s = 0; s < stages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bars[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int group = blockIdx.x / share;
  const size_t nchunks = buf_bytes / chunk;
  long long t0 = clock64();
  for (int i = 0; i < iters + stages; ++i) {
    if (i >= stages) {                          // consume chunk i - stages
      const int s = (i - stages) % stages;
      const uint32_t ph = ((i - stages) / stages) & 1;
      asm volatile(
          "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}"
          :: "r"(su32(&bars[s])), "r"(ph) : "memory");
    }
    if (i < iters) {
      const int s = i % stages;
      const size_t c = ((size_t)group * 7919 + (size_t)i * 13) % nchunks;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(&bars[s])), "r"(chunk) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(su32(smem + (size_t)s * chunk)), "l"(buf + c * chunk), "r"(chunk), "r"(su32(&bars[s]))
                   : "memory");
    }
  }
  long long t1 = clock64();
  if (blockIdx.x == 0) *clk_out = t1 - t0;
}

int main(int argc, char** argv) {
  const size_t buf_bytes = 32u << 20;            // 32 MB: L2-resident
  uint8_t* buf; long long* clk;
  cudaMalloc(&buf, buf_bytes); cudaMemset(buf, 1, buf_bytes); cudaMalloc(&clk, 8);
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const int chunks[] = {4096, 8192, 16384, 32768, 65536, 98304};
  const int grids[] = {sms, 16};
  const int shares[] = {1, 8};
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  printf("SMs %d, nominal clock %d MHz\n", sms, clk_khz / 1000);
  for (int chunk : chunks)
    for (int grid : grids)
      for (int share : shares) {
        if (share > grid) continue;
        const int stages = (196608 / chunk) > 32 ? 32 : (196608 / chunk);
        const int iters = 2000;
        const size_t smem = (size_t)stages * chunk + stages * 8;
        stream_kernel<<<grid, 32, smem>>>(buf, buf_bytes, chunk, stages, 50, share, clk);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        stream_kernel<<<grid, 32, smem>>>(buf, buf_bytes, chunk, stages, iters, share, clk);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        cudaError_t err = cudaGetLastError();
        long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
        const double bytes = (double)grid * iters * chunk;
        const double us = ms * 1e3;
        printf("chunk %6d  CTAs %4d  share %2d  stages %2d: %8.1f GB/s delivered  %6.1f KB/us per CTA  "
               "%5.1f B/clk/CTA (CTA clock)  %s\n", chunk, grid, share, stages, bytes / us / 1e3,
               (double)iters * chunk / us / 1e3, (double)iters * chunk / (double)c, err ? cudaGetErrorString(err) : "");
      }
  return 0;
}
