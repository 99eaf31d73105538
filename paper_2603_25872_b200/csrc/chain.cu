// K2/K3: fused elementwise skip-transition programs.
//
// One launch runs an ordered list of skip updates (drs_op) over all D
// latent elements; every thread owns one element for the whole list, so a
// refine chain x_{t-1} -> x_{t-2} -> ... -> x_{t-k} (parallel.py:303-306),
// the next block's k drafts fanned out of the refined anchor
// (parallel.py:295-298), and the trajectory stores all happen with the
// intermediate states in registers: HBM traffic is exactly one read of every
// operand vector and one write of every kept state.
//
// Bit-exactness: each op is the reference's numpy expression, evaluated in
// the same order with separately rounded IEEE ops (file compiled with
// --fmad=false), with the scalar coefficients precomputed on the host by the
// reference's own scalar expressions (paper_2603_25872_b200/transitions.py).
#include <cuda_runtime.h>
#include "drs.h"
#include "pdl.cuh"

namespace drs {

constexpr int kChainThreads = 256;
constexpr int kMaxOps = 64;
constexpr int kGroup = 8;     // ops whose operands are prefetched together

__device__ __forceinline__ double load_eps(const drs_op& op, int64_t j) {
  return op.eps_f32 ? (double)__ldg(static_cast<const float*>(op.eps) + j)
                    : __ldg(static_cast<const double*>(op.eps) + j);
}

// G = ops whose operands are prefetched together (<= kGroup), U = elements per
// thread per pass (grid-stride spaced, so every load stays coalesced).  All
// launches run U = 1 (more elements per thread lost to the occupancy their
// registers cost); see drs_skip_chain for the choice of G.
template <int G, int U>
__global__ void __launch_bounds__(kChainThreads)
skip_chain_kernel(const drs_op* __restrict__ ops, int n_ops, int64_t D) {
  pdl_wait();
  pdl_trigger();
  __shared__ drs_op s_ops[kMaxOps];
  {
    const uint64_t* src = reinterpret_cast<const uint64_t*>(ops);
    uint64_t* dst = reinterpret_cast<uint64_t*>(s_ops);
    const int n_words = n_ops * (int)(sizeof(drs_op) / 8);
    for (int i = threadIdx.x; i < n_words; i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  // Operands of up to G ops x U elements are loaded up front (independent
  // loads all in flight), then the ops run back to back on registers.  Legal
  // because a chain never reads through memory what an earlier op of the same
  // chain wrote (engine.DeviceRun._lower asserts it): intra-chain dependencies
  // go through the CUR / ANCHOR registers.
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j0 < D; j0 += stride * U) {
    double cur[U], anchor[U];
#pragma unroll
    for (int e = 0; e < U; ++e) cur[e] = anchor[e] = 0.0;
    for (int g = 0; g < n_ops; g += G) {
      double xv[G][U], ev[G][U], zv[G][U];
#pragma unroll
      for (int u = 0; u < G; ++u) {
#pragma unroll
        for (int e = 0; e < U; ++e) {
          const int64_t j = j0 + e * stride;
          xv[u][e] = ev[u][e] = zv[u][e] = 0.0;
          if (g + u < n_ops && j < D) {
            const drs_op& op = s_ops[g + u];
            if (op.src == DRS_SRC_X) xv[u][e] = op.x[j];
            ev[u][e] = load_eps(op, j);
            if (op.noisy) zv[u][e] = __ldg(op.z + j);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < G; ++u) {
        if (g + u >= n_ops) break;
        const drs_op& op = s_ops[g + u];
#pragma unroll
        for (int e = 0; e < U; ++e) {
          const int64_t j = j0 + e * stride;
          if (j >= D) break;
          const double x = op.src == DRS_SRC_X ? xv[u][e] : (op.src == DRS_SRC_CUR ? cur[e] : anchor[e]);
          const double ep = ev[u][e];
          double y;
          if (op.family == DRS_FAMILY_DDIM) {
            // x0_hat = (x_t - sqrt(1-ab_t) eps) / sqrt(ab_t)                   transitions.py:176
            // out = sqrt(ab_s) x0 + sqrt(1-ab_s-sigma^2) eps [+ sigma z]      transitions.py:177-179
            const double x0 = (x - op.c[0] * ep) / op.c[1];
            y = op.c[2] * x0 + op.c[3] * ep;
            if (op.noisy) y = y + op.c[4] * zv[u][e];
          } else if (op.family == DRS_FAMILY_DDPM || op.family == DRS_FAMILY_DDPM_X0) {
            // x0 = predicted_x0 (sequential.py:54), or given (DDPM_X0)
            // mean = (sqrt(r)(1-ab_s) x_t + sqrt(ab_s)(1-r) x0)/(1-ab_t) [+ sqrt(var) z]  transitions.py:115,134
            const double x0 = op.family == DRS_FAMILY_DDPM ? (x - op.c[0] * ep) / op.c[1] : ep;
            y = (op.c[2] * x + op.c[3] * x0) / op.c[4];
            if (op.noisy) y = y + op.c[5] * zv[u][e];
          } else if (op.family == DRS_FAMILY_PRED_X0) {
            y = (x - op.c[0] * ep) / op.c[1];                                  // sequential.py:54
          } else {
            y = x + op.c[0] * ep;                                              // euler: transitions.py:188
          }
          cur[e] = y;
          if (op.flags & DRS_OP_SAVE_ANCHOR) anchor[e] = y;
          if (op.out) op.out[j] = y;
          if (op.out2) op.out2[j] = y;
        }
      }
    }
  }
}

template <int G, int U>
static void launch_chain_gu(const drs_op* ops, int n_ops, int64_t D, cudaStream_t st) {
  int64_t blocks = (D + (int64_t)kChainThreads * U - 1) / ((int64_t)kChainThreads * U);
  if (blocks > 148 * 16) blocks = 148 * 16;
  launch_pdl(skip_chain_kernel<G, U>, dim3((unsigned)blocks), dim3(kChainThreads), 0, st, ops, n_ops, D);
}

}  // namespace drs

extern "C" int drs_skip_chain(const drs_op* ops, int n_ops, int64_t D, void* stream) {
  if (n_ops < 0 || n_ops > drs::kMaxOps || D < 0) return DRS_ERR_VALUE;
  if (n_ops == 0 || D == 0) return DRS_OK;
  if (!ops) return DRS_ERR_VALUE;
  cudaStream_t st = (cudaStream_t)stream;
  // Latents larger than one full wave (256-thread CTAs, 8 per SM) are HBM-bound:
  // one element and one op's operands per thread at a time (36 registers, full
  // occupancy) streams best for every chain length measured at D = 2^25
  // (tools/sampler_roofline.py: 1, 3, 6, 10 ops at 0.69-0.77 / 0.61 / 0.55 /
  // 0.54 of HBM vs 0.36 / 0.36 / 0.34 with operand groups of 8).  Smaller,
  // latency-bound latents prefetch the operands of up to kGroup ops together.
  const bool wide = D >= (int64_t)148 * 8 * drs::kChainThreads;
  if (wide || n_ops == 1) drs::launch_chain_gu<1, 1>(ops, n_ops, D, st);
  else if (n_ops >= drs::kGroup) drs::launch_chain_gu<drs::kGroup, 1>(ops, n_ops, D, st);
  else if (n_ops >= 4) drs::launch_chain_gu<4, 1>(ops, n_ops, D, st);
  else drs::launch_chain_gu<2, 1>(ops, n_ops, D, st);
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
}
