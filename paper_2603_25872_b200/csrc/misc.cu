// Small device utilities + host-side test hooks of libdrs.so.
#include <cuda_runtime.h>
#include "drs.h"
#include "pdl.cuh"
#include "bitgen.cuh"
#include "glibc_math.cuh"

namespace drs {

__global__ void copy_rows_kernel(const double* const* __restrict__ src, double* const* __restrict__ dst,
                                 int64_t D) {
  pdl_wait();
  pdl_trigger();
  const double* s = src[blockIdx.y];
  double* d = dst[blockIdx.y];
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < D;
       j += (int64_t)gridDim.x * blockDim.x)
    d[j] = s[j];
}

// Busy-wait on the global nanosecond timer: the GPU stand-in for the
// reference Latency wrapper's time.sleep (denoiser.py:258-263).
__global__ void spin_kernel(uint64_t ns) {
  pdl_wait();
  pdl_trigger();
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    uint64_t t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (t1 - t0 >= ns) break;
    __nanosleep(256);
  }
}

}  // namespace drs

extern "C" int drs_copy_rows(const double* const* src, double* const* out, int n_rows, int64_t D,
                             void* stream) {
  if (n_rows < 0 || D < 0 || n_rows > 65535) return DRS_ERR_VALUE;
  if (n_rows == 0 || D == 0) return DRS_OK;
  if (!src || !out) return DRS_ERR_VALUE;
  int64_t bx = (D + 255) / 256;
  if (bx > 1024) bx = 1024;
  dim3 grid((unsigned)bx, (unsigned)n_rows);
  drs::launch_pdl(drs::copy_rows_kernel, dim3(grid), dim3(256), 0, (cudaStream_t)stream, src, out, D);
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
}

extern "C" int drs_spin(double us, int n_ctas, void* stream) {
  if (!(us >= 0.0) || n_ctas < 0) return DRS_ERR_VALUE;
  if (n_ctas == 0 || us == 0.0) return DRS_OK;
  drs::launch_pdl(drs::spin_kernel, dim3(n_ctas), dim3(32), 0, (cudaStream_t)stream, (uint64_t)(us * 1000.0));
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
}

extern "C" double drs_host_log1p(double x) { return drs::log1p_glibc(x); }
extern "C" double drs_host_exp(double x) { return drs::exp_glibc(x); }

extern "C" int drs_host_seedseq(const drs_key* key, uint64_t seed, uint32_t* out, int n_words32) {
  if (!key || !out || n_words32 < 0) return DRS_ERR_VALUE;
  uint32_t w[8];
  const int n = drs::key_words(*key, seed, w);
  drs::SeedSeq ss;
  ss.init(w, n);
  ss.generate(out, n_words32);
  return DRS_OK;
}

extern "C" int drs_version(void) { return 1; }

extern "C" int drs_set_pdl(int on) {
  drs::pdl_enabled() = on ? 1 : 0;
  return DRS_OK;
}

extern "C" int drs_set_early_weights(int on) {
  drs::early_weights_enabled() = on ? 1 : 0;
  return DRS_OK;
}
