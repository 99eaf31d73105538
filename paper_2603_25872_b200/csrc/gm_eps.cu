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
constexpr int kGmMaxComp = 8;          // components reduced per sweep over the row
constexpr int kGmCompLimit = 1920;     // 3 x 8 B x n_comp dynamic + 2 KB static shared memory <= 48 KB
constexpr int kGmRegComp = 2;        // components kept in registers (others re-read)

// MODE 0: VP eps (denoiser.py:85-107); 1: VE ODE velocity (:124-136);
// 2: VP posterior mean E[x0 | x_t] (x0_posterior_mean, :110-121).
template <int MODE>
__global__ void __launch_bounds__(kGmThreads)
gm_eps_kernel(const double* const* __restrict__ xs, const int32_t* __restrict__ ts, int64_t D,
              const double* __restrict__ alpha_bar, int T, const double* __restrict__ means,
              const double* __restrict__ log_w, const double* __restrict__ var, int n_comp,
              double* const* __restrict__ outs, int* __restrict__ err) {
  constexpr bool VE = MODE == 1;
  constexpr bool X0 = MODE == 2;
  pdl_wait();
  pdl_trigger();
  __shared__ double red[kGmMaxComp][32];
  extern __shared__ double s_dyn[];          // n_comp log-weights, responsibilities, scales
  double* s_lc = s_dyn;
  double* s_r = s_dyn + n_comp;
  double* s_sc = s_dyn + 2 * n_comp;
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

  // ---- pass 1: squared distances, kGmMaxComp components per sweep -----------
  // (one sweep for the usual n_comp <= 8; larger mixtures re-read x per sweep)
  double xr[kGmPer], mr[kGmRegComp][kGmPer];
  for (int c0 = 0; c0 < n_comp; c0 += kGmMaxComp) {
    const int nc = min(kGmMaxComp, n_comp - c0);
    const double* __restrict__ mc = means + (int64_t)c0 * D;
    double part[kGmMaxComp];
#pragma unroll
    for (int i = 0; i < kGmMaxComp; ++i) part[i] = 0.0;
    for (int64_t base = 0; base < D; base += chunk) {
#pragma unroll
      for (int e = 0; e < kGmPer; ++e) {
        const int64_t j = base + (int64_t)e * kGmThreads + threadIdx.x;
        const bool ok = j < D;
        xr[e] = ok ? __ldg(x + j) : 0.0;
#pragma unroll
        for (int i = 0; i < kGmRegComp; ++i)
          mr[i][e] = (ok && i < nc) ? __ldg(mc + (int64_t)i * D + j) : 0.0;
      }
#pragma unroll
      for (int e = 0; e < kGmPer; ++e) {
        const int64_t j = base + (int64_t)e * kGmThreads + threadIdx.x;
        if (j < D) {
#pragma unroll
          for (int i = 0; i < kGmMaxComp; ++i) {
            if (i < nc) {
              const double m = i < kGmRegComp ? mr[i < kGmRegComp ? i : 0][e] : __ldg(mc + (int64_t)i * D + j);
              const double d = xr[e] - sa * m;
              part[i] += d * d;
            }
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < kGmMaxComp; ++i) {
      if (i < nc) {
        double v = part[i];
        for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if (lane == 0) red[i][warp] = v;
      }
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
      for (int i = 0; i < kGmMaxComp; ++i) {
        if (i < nc) {
          double d2 = red[i][lane];
          for (int off = 16; off; off >>= 1) d2 += __shfl_xor_sync(0xffffffffu, d2, off);
          const double s = VE ? var[c0 + i] + one_m : abar * var[c0 + i] + one_m;
          if (lane == 0) s_lc[c0 + i] = log_w[c0 + i] + ((-0.5 * d2) / s - (0.5 * (double)D) * log(s));
        }
      }
    }
    __syncthreads();                       // red[] is reused by the next sweep
  }
  if (threadIdx.x == 0) {                  // logsumexp in component order (scipy: max, sum exp, log)
    double mx = -INFINITY;
    for (int i = 0; i < n_comp; ++i) mx = fmax(mx, s_lc[i]);
    double sum = 0.0;
    for (int i = 0; i < n_comp; ++i) sum += exp(s_lc[i] - mx);
    const double lse = log(sum) + mx;
    for (int i = 0; i < n_comp; ++i) s_r[i] = exp(s_lc[i] - lse);
  }
  for (int i = threadIdx.x; i < n_comp; i += blockDim.x) {
    const double sc = VE ? var[i] + one_m : abar * var[i] + one_m;
    // VE: posterior gain v_i / s_i; X0: sqrt(abar) v_i / s_i (denoiser.py:117)
    s_sc[i] = VE ? var[i] / sc : (X0 ? (sa * var[i]) / sc : sc);
  }
  __syncthreads();

  // ---- pass 2: eps ----------------------------------------------------------
  const double neg_sq = VE ? 0.0 : -sqrt(one_m);
  for (int64_t base = 0; base < D; base += chunk) {
    if (!single || n_comp > kGmMaxComp) {   // re-read this chunk (L2-resident) into the registers
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
        for (int i = 0; i < n_comp; ++i) {
          const double m = i < kGmRegComp ? mr[i < kGmRegComp ? i : 0][e] : __ldg(means + (int64_t)i * D + j);
          const double r = s_r[i], sc = s_sc[i];
          const double term = VE ? r * (m + sc * (xr[e] - m))
                            : X0 ? r * (m + sc * (xr[e] - sa * m))          // cond_mean (denoiser.py:118)
                                 : (r * (sa * m - xr[e])) / sc;
          score = (i == 0) ? term : score + term;
        }
        out[j] = VE ? (xr[e] - score) / sigma : (X0 ? score : neg_sq * score);
      }
    }
  }
}

static size_t gm_smem(int n_comp) { return (size_t)3 * sizeof(double) * n_comp; }

}  // namespace drs

extern "C" int drs_gm_eps(const double* const* xs, const int32_t* ts, int n_rows, int64_t D,
                          const double* alpha_bar, int T, const double* means, const double* log_w,
                          const double* var, int n_comp, double* const* out, int* err, void* stream) {
  if (n_rows < 0 || D < 0 || n_comp < 1 || n_comp > drs::kGmCompLimit || T < 0) return DRS_ERR_VALUE;
  if (n_rows == 0 || D == 0) return DRS_OK;
  if (!xs || !ts || !alpha_bar || !means || !log_w || !var || !out || !err) return DRS_ERR_VALUE;
  drs::launch_pdl(drs::gm_eps_kernel<0>, dim3(n_rows), dim3(drs::kGmThreads), drs::gm_smem(n_comp), (cudaStream_t)stream,
      xs, ts, D, alpha_bar, T, means, log_w, var, n_comp, out, err);
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
}

extern "C" int drs_gm_velocity(const double* const* xs, const int32_t* idx, int n_rows, int64_t D,
                               const double* sigmas, int N, const double* means, const double* log_w,
                               const double* var, int n_comp, double* const* out, int* err, void* stream) {
  if (n_rows < 0 || D < 0 || n_comp < 1 || n_comp > drs::kGmCompLimit || N < 0) return DRS_ERR_VALUE;
  if (n_rows == 0 || D == 0) return DRS_OK;
  if (!xs || !idx || !sigmas || !means || !log_w || !var || !out || !err) return DRS_ERR_VALUE;
  drs::launch_pdl(drs::gm_eps_kernel<1>, dim3(n_rows), dim3(drs::kGmThreads), drs::gm_smem(n_comp), (cudaStream_t)stream,
      xs, idx, D, sigmas, N, means, log_w, var, n_comp, out, err);
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
}

extern "C" int drs_gm_x0_mean(const double* const* xs, const int32_t* zeros, int n_rows, int64_t D,
                              const double* abar, const double* means, const double* log_w, const double* var,
                              int n_comp, double* const* out, int* err, void* stream) {
  if (n_rows < 0 || D < 0 || n_comp < 1 || n_comp > drs::kGmCompLimit) return DRS_ERR_VALUE;
  if (n_rows == 0 || D == 0) return DRS_OK;
  if (!xs || !zeros || !abar || !means || !log_w || !var || !out || !err) return DRS_ERR_VALUE;
  // every row reads the same abar: a 1-entry table indexed by t = zeros[r] = 0
  drs::launch_pdl(drs::gm_eps_kernel<2>, dim3(n_rows), dim3(drs::kGmThreads), drs::gm_smem(n_comp),
      (cudaStream_t)stream, xs, zeros, D, abar, 0, means, log_w, var, n_comp, out, err);
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
}
