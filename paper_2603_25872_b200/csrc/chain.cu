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

// runtime switch (drs_set_chain_vec, A/B measurement): HBM-sized latents use the
// 16-byte vector kernel (1, default) or the scalar one-element-per-thread kernel (0)
inline int& chain_vec_enabled() {
  static int on = 1;
  return on;
}

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

// ---- HBM-sized latents: 16-byte vector accesses, two elements per lane ----
// Every operand row is read with explicit global-space, non-coherent 16-byte
// loads (ld.global.nc.v2.f64; fp32 eps: 8-byte ld.global.nc.v2.f32) and every
// kept state is written with st.global.v2.f64, so a warp moves 512 B per
// instruction instead of 256 B through generic addressing.  P pairs per
// thread are in flight per op (grid-stride spaced: coalesced).  The two
// elements of a pair run the scalar kernel's exact expression order
// (--fmad=false), so results are bit-identical to it.  An op whose rows are
// not 16-byte aligned (views at odd offsets) takes the scalar accesses for
// that op only (uniform branch).
__device__ __forceinline__ double2 ld_nc_v2(const double* p) {
  double2 v;
  asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ float2 ld_nc_v2f(const float* p) {
  float2 v;
  asm volatile("ld.global.nc.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_v2(double* p, double a, double b) {
  asm volatile("st.global.v2.f64 [%0], {%1, %2};" :: "l"(p), "d"(a), "d"(b) : "memory");
}

__device__ __forceinline__ double op_apply(const drs_op& op, double x, double ep, double z) {
  double y;
  if (op.family == DRS_FAMILY_DDIM) {
    const double x0 = (x - op.c[0] * ep) / op.c[1];                  // transitions.py:176
    y = op.c[2] * x0 + op.c[3] * ep;                                  // transitions.py:177
    if (op.noisy) y = y + op.c[4] * z;                                // transitions.py:178-179
  } else if (op.family == DRS_FAMILY_DDPM || op.family == DRS_FAMILY_DDPM_X0) {
    const double x0 = op.family == DRS_FAMILY_DDPM ? (x - op.c[0] * ep) / op.c[1] : ep;
    y = (op.c[2] * x + op.c[3] * x0) / op.c[4];                       // transitions.py:115
    if (op.noisy) y = y + op.c[5] * z;                                // transitions.py:134
  } else if (op.family == DRS_FAMILY_PRED_X0) {
    y = (x - op.c[0] * ep) / op.c[1];                                 // sequential.py:54
  } else {
    y = x + op.c[0] * ep;                                             // transitions.py:188
  }
  return y;
}

__device__ __forceinline__ bool op_aligned(const drs_op& op) {
  uintptr_t a = reinterpret_cast<uintptr_t>(op.eps) & (op.eps_f32 ? 7 : 15);
  if (op.src == DRS_SRC_X) a |= reinterpret_cast<uintptr_t>(op.x) & 15;
  if (op.noisy) a |= reinterpret_cast<uintptr_t>(op.z) & 15;
  a |= reinterpret_cast<uintptr_t>(op.out) & 15;
  a |= reinterpret_cast<uintptr_t>(op.out2) & 15;
  return a == 0;
}

template <int P>
__global__ void __launch_bounds__(kChainThreads)
skip_chain_v2_kernel(const drs_op* __restrict__ ops, int n_ops, int64_t D) {
  pdl_wait();
  pdl_trigger();
  __shared__ drs_op s_ops[kMaxOps];
  __shared__ int s_vec[kMaxOps];
  {
    const uint64_t* src = reinterpret_cast<const uint64_t*>(ops);
    uint64_t* dst = reinterpret_cast<uint64_t*>(s_ops);
    const int n_words = n_ops * (int)(sizeof(drs_op) / 8);
    for (int i = threadIdx.x; i < n_words; i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n_ops; i += blockDim.x) s_vec[i] = op_aligned(s_ops[i]) ? 1 : 0;
  __syncthreads();
  const int64_t n_pairs = D >> 1;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p0 < n_pairs; p0 += stride * P) {
    double cur[P][2], anchor[P][2];
#pragma unroll
    for (int u = 0; u < P; ++u) cur[u][0] = cur[u][1] = anchor[u][0] = anchor[u][1] = 0.0;
    for (int o = 0; o < n_ops; ++o) {
      const drs_op& op = s_ops[o];
      const bool vec = s_vec[o];
      double xv[P][2], ev[P][2], zv[P][2];
#pragma unroll
      for (int u = 0; u < P; ++u) {           // every operand of the P pairs in flight
        const int64_t j = 2 * (p0 + u * stride);
        xv[u][0] = xv[u][1] = ev[u][0] = ev[u][1] = zv[u][0] = zv[u][1] = 0.0;
        if (p0 + u * stride < n_pairs) {
          if (vec) {
            if (op.src == DRS_SRC_X) { const double2 t = ld_nc_v2(op.x + j); xv[u][0] = t.x; xv[u][1] = t.y; }
            if (op.eps_f32) {
              const float2 t = ld_nc_v2f(static_cast<const float*>(op.eps) + j);
              ev[u][0] = (double)t.x; ev[u][1] = (double)t.y;
            } else {
              const double2 t = ld_nc_v2(static_cast<const double*>(op.eps) + j);
              ev[u][0] = t.x; ev[u][1] = t.y;
            }
            if (op.noisy) { const double2 t = ld_nc_v2(op.z + j); zv[u][0] = t.x; zv[u][1] = t.y; }
          } else {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              if (op.src == DRS_SRC_X) xv[u][e] = op.x[j + e];
              ev[u][e] = load_eps(op, j + e);
              if (op.noisy) zv[u][e] = __ldg(op.z + j + e);
            }
          }
        }
      }
#pragma unroll
      for (int u = 0; u < P; ++u) {
        const int64_t j = 2 * (p0 + u * stride);
        if (p0 + u * stride >= n_pairs) break;
        double y[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const double x = op.src == DRS_SRC_X ? xv[u][e] : (op.src == DRS_SRC_CUR ? cur[u][e] : anchor[u][e]);
          y[e] = op_apply(op, x, ev[u][e], zv[u][e]);
          cur[u][e] = y[e];
          if (op.flags & DRS_OP_SAVE_ANCHOR) anchor[u][e] = y[e];
        }
        if (vec) {
          if (op.out) st_v2(op.out + j, y[0], y[1]);
          if (op.out2) st_v2(op.out2 + j, y[0], y[1]);
        } else {
          if (op.out) { op.out[j] = y[0]; op.out[j + 1] = y[1]; }
          if (op.out2) { op.out2[j] = y[0]; op.out2[j + 1] = y[1]; }
        }
      }
    }
  }
}

template <int P>
static void launch_chain_v2(const drs_op* ops, int n_ops, int64_t D, cudaStream_t st) {
  const int64_t n_pairs = D >> 1;
  int64_t blocks = (n_pairs + (int64_t)kChainThreads * P - 1) / ((int64_t)kChainThreads * P);
  if (blocks > 148 * 12) blocks = 148 * 12;
  launch_pdl(skip_chain_v2_kernel<P>, dim3((unsigned)blocks), dim3(kChainThreads), 0, st, ops, n_ops, D);
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
  const int vec = drs::chain_vec_enabled();
  if (wide && (D & 1) == 0 && vec == 1) drs::launch_chain_v2<1>(ops, n_ops, D, st);
  else if (wide && (D & 1) == 0 && vec == 2) drs::launch_chain_v2<2>(ops, n_ops, D, st);
  else if (wide || n_ops == 1) drs::launch_chain_gu<1, 1>(ops, n_ops, D, st);
  else if (n_ops >= drs::kGroup) drs::launch_chain_gu<drs::kGroup, 1>(ops, n_ops, D, st);
  else if (n_ops >= 4) drs::launch_chain_gu<4, 1>(ops, n_ops, D, st);
  else drs::launch_chain_gu<2, 1>(ops, n_ops, D, st);
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
}

extern "C" int drs_set_chain_vec(int mode) {
  if (mode < 0 || mode > 2) return DRS_ERR_VALUE;   // 0 scalar, 1 vector (default), 2 vector x 2 pairs
  drs::chain_vec_enabled() = mode;
  return DRS_OK;
}
