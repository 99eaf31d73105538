// K9: Gaussian-mixture eps oracle on device (the toy denoiser of configs C1/C2).
//
// Restates skipdiff denoiser.py:73-107 (eps_oracle + _responsibilities):
//   abar    = alpha_bar[t]
//   centers = sqrt(abar) * m_i                 scales s_i = abar v_i + (1 - abar)
//   log_i   = log w_i + (-0.5 * sum_j (x_j - c_ij)^2) / s_i - (0.5 D) log s_i
//   r       = exp(log - logsumexp(log))
//   eps_j   = -sqrt(1 - abar) * sum_i (r_i (c_ij - x_j)) / s_i
// One CTA (1024 threads) per state row, ONE pass over HBM: every thread
// issues all its loads up front (x and the n_comp mean entries of its
// kPer elements stay in registers), the n_comp squared distances are reduced
// with a fixed tree (warp shuffles -> shared memory -> warp 0), and the eps
// is written from the same registers.  The reduction order differs from
// numpy's pairwise sum, so parity with the reference is to fp64 rounding
// (tests state the tolerance); across ranks the kernel is bit-reproducible.
// Rows longer than kThreads*kPer are processed in register-sized chunks with
// a second (L2-resident) read.
//
// VE = true: the ODE velocity of the variance-exploding mixture for the Euler
// family (denoiser.py:124-136): per row a grid index i, sigma = sigmas[i],
//   scales s_i = v_i + sigma**2, centers = m_i (log-responsibilities as above)
//   x0_hat_j  = sum_i r_i (m_ij + (v_i / s_i)(x_j - m_ij))
//   v_j       = (x_j - x0_hat_j) / sigma           (err bit 4: sigma <= 0)
#include <cuda_runtime.h>
#include <math.h>
#include "drs.h"
#include "pdl.cuh"

namespace drs {

constexpr int kGmThreads = 1024;
constexpr int kGmPer = 4;            // elements per thread held in registers
constexpr int kGmMaxComp = 8;
constexpr int kGmRegComp = 2;        // components kept in registers (others re-read)

template <bool VE>
__global__ void __launch_bounds__(kGmThreads)
gm_eps_kernel(const double* const* __restrict__ xs, const int32_t* __restrict__ ts, int64_t D,
              const double* __restrict__ alpha_bar, int T, const double* __restrict__ means,
              const double* __restrict__ log_w, const double* __restrict__ var, int n_comp,
              double* const* __restrict__ outs, int* __restrict__ err) {
  pdl_wait();
  pdl_trigger();
  __shared__ double red[kGmMaxComp][32];
  __shared__ double s_r[kGmMaxComp];
  const int row = blockIdx.x;
  const int t = ts[row];
  if (t < 0 || t > T) {               // TimestepOutOfRange (denoiser.py:95-96)
    if (threadIdx.x == 0) atomicOr(err, 2);
    return;
  }
  const double* __restrict__ x = xs[row];
  double* __restrict__ out = outs[row];
  // VP: table = alpha_bar, centers sqrt(abar) m_i, scales abar v_i + (1 - abar)
  // VE: table = sigmas,    centers m_i,            scales v_i + sigma**2
  const double abar = alpha_bar[t];
  const double sigma = abar;
  if (VE && !(sigma > 0.0)) {                          // NonPositiveSigma (denoiser.py:127-128)
    if (threadIdx.x == 0) atomicOr(err, 4);
    return;
  }
  const double sa = VE ? 1.0 : sqrt(abar);
  const double one_m = VE ? sigma * sigma : 1.0 - abar;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t chunk = (int64_t)kGmThreads * kGmPer;
  const bool single = D <= chunk;

  // ---- pass 1: squared distances ------------------------------------------
  double part[kGmMaxComp];
#pragma unroll
  for (int i = 0; i < kGmMaxComp; ++i) part[i] = 0.0;
  double xr[kGmPer], mr[kGmRegComp][kGmPer];
  for (int64_t base = 0; base < D; base += chunk) {
#pragma unroll
    for (int e = 0; e < kGmPer; ++e) {
      const int64_t j = base + (int64_t)e * kGmThreads + threadIdx.x;
      const bool ok = j < D;
      xr[e] = ok ? __ldg(x + j) : 0.0;
#pragma unroll
      for (int i = 0; i < kGmRegComp; ++i)
        mr[i][e] = (ok && i < n_comp) ? __ldg(means + (int64_t)i * D + j) : 0.0;
    }
#pragma unroll
    for (int e = 0; e < kGmPer; ++e) {
      const int64_t j = base + (int64_t)e * kGmThreads + threadIdx.x;
      if (j < D) {
#pragma unroll
        for (int i = 0; i < kGmMaxComp; ++i) {
          if (i < n_comp) {
            const double m = i < kGmRegComp ? mr[i < kGmRegComp ? i : 0][e] : __ldg(means + (int64_t)i * D + j);
            const double d = xr[e] - sa * m;
            part[i] += d * d;
          }
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < kGmMaxComp; ++i) {
    if (i < n_comp) {
      double v = part[i];
      for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if (lane == 0) red[i][warp] = v;
    }
  }
  __syncthreads();
  if (warp == 0) {
    double lc[kGmMaxComp];
    double mx = -INFINITY;
#pragma unroll
    for (int i = 0; i < kGmMaxComp; ++i) {
      if (i < n_comp) {
        double d2 = red[i][lane];
        for (int off = 16; off; off >>= 1) d2 += __shfl_xor_sync(0xffffffffu, d2, off);
        const double s = VE ? var[i] + one_m : abar * var[i] + one_m;
        lc[i] = log_w[i] + ((-0.5 * d2) / s - (0.5 * (double)D) * log(s));
        mx = fmax(mx, lc[i]);
      } else {
        lc[i] = -INFINITY;
      }
    }
    if (lane == 0) {
      double sum = 0.0;
#pragma unroll
      for (int i = 0; i < kGmMaxComp; ++i) if (i < n_comp) sum += exp(lc[i] - mx);
      const double lse = log(sum) + mx;
#pragma unroll
      for (int i = 0; i < kGmMaxComp; ++i) if (i < n_comp) s_r[i] = exp(lc[i] - lse);
    }
  }
  __syncthreads();

  // ---- pass 2: eps ----------------------------------------------------------
  const double neg_sq = VE ? 0.0 : -sqrt(one_m);
  double r[kGmMaxComp], sc[kGmMaxComp];
#pragma unroll
  for (int i = 0; i < kGmMaxComp; ++i) {
    r[i] = i < n_comp ? s_r[i] : 0.0;
    sc[i] = i < n_comp ? (VE ? var[i] + one_m : abar * var[i] + one_m) : 1.0;
    if (VE) sc[i] = i < n_comp ? var[i] / sc[i] : 0.0;   // posterior gain v_i / s_i
  }
  for (int64_t base = 0; base < D; base += chunk) {
    if (!single) {   // re-read this chunk (L2-resident) into the registers
#pragma unroll
      for (int e = 0; e < kGmPer; ++e) {
        const int64_t j = base + (int64_t)e * kGmThreads + threadIdx.x;
        const bool ok = j < D;
        xr[e] = ok ? __ldg(x + j) : 0.0;
#pragma unroll
        for (int i = 0; i < kGmRegComp; ++i)
          mr[i][e] = (ok && i < n_comp) ? __ldg(means + (int64_t)i * D + j) : 0.0;
      }
    }
#pragma unroll
    for (int e = 0; e < kGmPer; ++e) {
      const int64_t j = base + (int64_t)e * kGmThreads + threadIdx.x;
      if (j < D) {
        double score = 0.0;
#pragma unroll
        for (int i = 0; i < kGmMaxComp; ++i) {
          if (i < n_comp) {
            const double m = i < kGmRegComp ? mr[i < kGmRegComp ? i : 0][e] : __ldg(means + (int64_t)i * D + j);
            const double term = VE ? r[i] * (m + sc[i] * (xr[e] - m)) : (r[i] * (sa * m - xr[e])) / sc[i];
            score = (i == 0) ? term : score + term;
          }
        }
        out[j] = VE ? (xr[e] - score) / sigma : neg_sq * score;
      }
    }
  }
}

}  // namespace drs

extern "C" int drs_gm_eps(const double* const* xs, const int32_t* ts, int n_rows, int64_t D,
                          const double* alpha_bar, int T, const double* means, const double* log_w,
                          const double* var, int n_comp, double* const* out, int* err, void* stream) {
  if (n_rows < 0 || D < 0 || n_comp < 1 || n_comp > drs::kGmMaxComp || T < 0) return DRS_ERR_VALUE;
  if (n_rows == 0 || D == 0) return DRS_OK;
  if (!xs || !ts || !alpha_bar || !means || !log_w || !var || !out || !err) return DRS_ERR_VALUE;
  drs::launch_pdl(drs::gm_eps_kernel<false>, dim3(n_rows), dim3(drs::kGmThreads), 0, (cudaStream_t)stream,
      xs, ts, D, alpha_bar, T, means, log_w, var, n_comp, out, err);
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
}

extern "C" int drs_gm_velocity(const double* const* xs, const int32_t* idx, int n_rows, int64_t D,
                               const double* sigmas, int N, const double* means, const double* log_w,
                               const double* var, int n_comp, double* const* out, int* err, void* stream) {
  if (n_rows < 0 || D < 0 || n_comp < 1 || n_comp > drs::kGmMaxComp || N < 0) return DRS_ERR_VALUE;
  if (n_rows == 0 || D == 0) return DRS_OK;
  if (!xs || !idx || !sigmas || !means || !log_w || !var || !out || !err) return DRS_ERR_VALUE;
  drs::launch_pdl(drs::gm_eps_kernel<true>, dim3(n_rows), dim3(drs::kGmThreads), 0, (cudaStream_t)stream,
      xs, idx, D, sigmas, N, means, log_w, var, n_comp, out, err);
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
}
