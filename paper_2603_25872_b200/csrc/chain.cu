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
  // Operands of up to kGroup ops are loaded up front (independent loads all
  // in flight), then the ops run back to back on registers.  Legal because a
  // chain never reads through memory what an earlier op of the same chain
  // wrote (engine.DeviceRun._lower asserts it): intra-chain dependencies go
  // through the CUR / ANCHOR registers.
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < D;
       j += (int64_t)gridDim.x * blockDim.x) {
    double cur = 0.0, anchor = 0.0;
    for (int g = 0; g < n_ops; g += kGroup) {
      double xv[kGroup], ev[kGroup], zv[kGroup];
#pragma unroll
      for (int u = 0; u < kGroup; ++u) {
        xv[u] = ev[u] = zv[u] = 0.0;
        if (g + u < n_ops) {
          const drs_op& op = s_ops[g + u];
          if (op.src == DRS_SRC_X) xv[u] = op.x[j];
          ev[u] = load_eps(op, j);
          if (op.noisy) zv[u] = __ldg(op.z + j);
        }
      }
#pragma unroll
      for (int u = 0; u < kGroup; ++u) {
        if (g + u >= n_ops) break;
        const drs_op& op = s_ops[g + u];
        const double x = op.src == DRS_SRC_X ? xv[u] : (op.src == DRS_SRC_CUR ? cur : anchor);
        const double e = ev[u];
        double y;
        if (op.family == DRS_FAMILY_DDIM) {
          // x0_hat = (x_t - sqrt(1-ab_t) eps) / sqrt(ab_t)                   transitions.py:176
          // out = sqrt(ab_s) x0 + sqrt(1-ab_s-sigma^2) eps [+ sigma z]      transitions.py:177-179
          const double x0 = (x - op.c[0] * e) / op.c[1];
          y = op.c[2] * x0 + op.c[3] * e;
          if (op.noisy) y = y + op.c[4] * zv[u];
        } else if (op.family == DRS_FAMILY_DDPM || op.family == DRS_FAMILY_DDPM_X0) {
          // x0 = predicted_x0 (sequential.py:54), or given (DDPM_X0)
          // mean = (sqrt(r)(1-ab_s) x_t + sqrt(ab_s)(1-r) x0)/(1-ab_t) [+ sqrt(var) z]  transitions.py:115,134
          const double x0 = op.family == DRS_FAMILY_DDPM ? (x - op.c[0] * e) / op.c[1] : e;
          y = (op.c[2] * x + op.c[3] * x0) / op.c[4];
          if (op.noisy) y = y + op.c[5] * zv[u];
        } else if (op.family == DRS_FAMILY_PRED_X0) {
          y = (x - op.c[0] * e) / op.c[1];                                   // sequential.py:54
        } else {
          y = x + op.c[0] * e;                                               // euler: transitions.py:188
        }
        cur = y;
        if (op.flags & DRS_OP_SAVE_ANCHOR) anchor = y;
        if (op.out) op.out[j] = y;
        if (op.out2) op.out2[j] = y;
      }
    }
  }
}

}  // namespace drs

extern "C" int drs_skip_chain(const drs_op* ops, int n_ops, int64_t D, void* stream) {
  if (n_ops < 0 || n_ops > drs::kMaxOps || D < 0) return DRS_ERR_VALUE;
  if (n_ops == 0 || D == 0) return DRS_OK;
  if (!ops) return DRS_ERR_VALUE;
  int64_t blocks = (D + drs::kChainThreads - 1) / drs::kChainThreads;
  if (blocks > 148 * 16) blocks = 148 * 16;
  drs::launch_pdl(drs::skip_chain_kernel, dim3((unsigned)blocks), dim3(drs::kChainThreads), 0, (cudaStream_t)stream, ops, n_ops, D);
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
}
