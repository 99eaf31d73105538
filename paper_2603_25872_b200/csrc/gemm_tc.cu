// K4: persistent, warp-specialised bf16 GEMM on the 5th-gen tensor cores.
//
//   C[M, N] = epilogue( alpha * A[M, K] . B[N, K]^T )        (nn.Linear: y = x W^T)
//
// A, B: bf16, K-major (row-major with K contiguous), staged into shared
// memory by TMA (cp.async.bulk.tensor, SWIZZLE_128B, 64-element K slabs) in a
// kStages-deep mbarrier ring; one elected thread issues tcgen05.mma
// (M=128, N=BN, K=16) accumulating fp32 in TMEM; the accumulator is double
// buffered in TMEM (2 x BN columns) so the epilogue of tile i overlaps the
// MMAs of tile i+1.  Warp roles (192 threads):
//   warp 0        TMA producer            (one elected lane)
//   warp 1        TMEM allocator + MMA issuer (one elected lane)
//   warps 2..9    epilogue, two warps per TMEM lane quadrant splitting the
//                 32-column chunks: tcgen05.ld 32x32b -> registers -> bias /
//                 GELU / SiLU / GEGLU / gate / residual -> bf16 or fp32 stores
// Grid = min(#tiles, #SMs); each CTA walks tiles t = blockIdx.x, +gridDim.x.
// Split-K (split > 1): the `split` CTAs of one output tile form a thread-block
// cluster; each accumulates a K range, parks its fp32 partial tile in its own
// (idle) pipeline shared memory, and after a cluster barrier every CTA reduces
// a slice of the tile's rows over DSMEM in the fixed order s = 0..split-1
// (deterministic, no atomics, no workspace) and runs the common epilogue.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <string.h>
#include <stdlib.h>
#include "drs_net.h"
#include "pdl.cuh"
#include "tc_common.cuh"

namespace drs {

constexpr int kBM = 128;
constexpr int kBK = 64;                 // one 128-byte swizzle atom of bf16
constexpr int kGemmThreads = 320;       // warp 0 TMA, warp 1 MMA, warps 2..9 epilogue (2 per TMEM quadrant)
constexpr int kEpiWarps = 8;

// tanh on the SFU (tanh.approx.f32, rel. error ~2^-11: below the bf16 rounding of the output)
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float gelu_tanh(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  return 0.5f * x * (1.f + tanh_fast(k0 * (x + k1 * x * x * x)));
}
// GELU with the exact-erf definition; erf from the branch-free erfc rational
// form t exp(-z^2 + P(t)), t = 1 / (1 + z/2) (|erf error| < 1.2e-7, far below the
// bf16 rounding of the output; libm erff costs ~3x the instructions and branches)
__device__ __forceinline__ float gelu_erf(float x) {
  const float u = x * 0.7071067811865476f, z = fabsf(u);
  const float t = __fdividef(1.f, fmaf(0.5f, z, 1.f));
  float p = fmaf(t, 0.17087277f, -0.82215223f);
  p = fmaf(t, p, 1.48851587f);
  p = fmaf(t, p, -1.13520398f);
  p = fmaf(t, p, 0.27886807f);
  p = fmaf(t, p, -0.18628806f);
  p = fmaf(t, p, 0.09678418f);
  p = fmaf(t, p, 0.37409196f);
  p = fmaf(t, p, 1.00002368f);
  p = fmaf(t, p, -1.26551223f);
  const float r = t * __expf(fmaf(-z, z, p));         // erfc(|u|)
  const float e = copysignf(1.f - r, u);
  return 0.5f * x * (1.f + e);
}
// x * sigmoid(x) = 0.5 x (1 + tanh(x / 2)): one SFU op (was ex2 + rcp)
__device__ __forceinline__ float silu(float x) {
  const float h = 0.5f * x;
  return fmaf(h, tanh_fast(h), h);
}

// Two GELU(erf)s at once on the paired FP32 pipe (fma/mul.rn.f32x2 -> FFMA2 /
// FMUL2): the same erfc rational form as gelu_erf, with log2(e) folded into the
// polynomial so the exponential is one ex2.approx, and rcp.approx for t
// (|error| ~1e-6 relative, far below the bf16 output rounding): ~14 instructions
// per GELU instead of ~25 -- the GEGLU epilogue is the bound of its GEMMs.
__device__ __forceinline__ uint64_t f2pk(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2upk(uint64_t r, float& a, float& b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); }
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// GELU in the tanh form 0.5 x (1 + tanh(sqrt(2/pi) x (1 + 0.044715 x^2))) on the paired
// FP32 pipe with one tanh.approx per element: 5 FFMA2/FMUL2 + 2 SFU ops per pair (the
// erf form above: ~14 + 4).  Differs from GELU(erf) by < 1e-3 absolute, under the bf16
// rounding of the GEGLU output.
__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void gelu_tanh_x2(float& x0, float& x1) {
  const uint64_t x = f2pk(x0, x1);
  const uint64_t x2 = fmul2(x, x);
  const uint64_t in = fmul2(fmul2(x, f2pk(0.7978845608f, 0.7978845608f)), ffma2(x2, f2pk(0.044715f, 0.044715f),
                                                                                 f2pk(1.f, 1.f)));
  float i0, i1;
  f2upk(in, i0, i1);
  const uint64_t t = f2pk(tanh_approx(i0), tanh_approx(i1));
  const uint64_t h = fmul2(x, f2pk(0.5f, 0.5f));
  f2upk(ffma2(h, t, h), x0, x1);
}
__device__ __forceinline__ void gelu_erf_x2(float& x0, float& x1) {
  constexpr float L = 1.4426950408889634f;
  const float u0 = x0 * 0.7071067811865476f, u1 = x1 * 0.7071067811865476f;
  const float z0 = fabsf(u0), z1 = fabsf(u1);
  const float t0 = rcp_approx(fmaf(0.5f, z0, 1.f)), t1 = rcp_approx(fmaf(0.5f, z1, 1.f));
  const uint64_t t = f2pk(t0, t1);
#define DRS_C2(c) f2pk((c) * L, (c) * L)
  uint64_t p = ffma2(t, DRS_C2(0.17087277f), DRS_C2(-0.82215223f));
  p = ffma2(t, p, DRS_C2(1.48851587f));
  p = ffma2(t, p, DRS_C2(-1.13520398f));
  p = ffma2(t, p, DRS_C2(0.27886807f));
  p = ffma2(t, p, DRS_C2(-0.18628806f));
  p = ffma2(t, p, DRS_C2(0.09678418f));
  p = ffma2(t, p, DRS_C2(0.37409196f));
  p = ffma2(t, p, DRS_C2(1.00002368f));
  p = ffma2(t, p, DRS_C2(-1.26551223f));
#undef DRS_C2
  const uint64_t arg = ffma2(f2pk(-z0, -z1), fmul2(f2pk(z0, z1), f2pk(L, L)), p);   // log2e (-z^2 + P(t))
  float a0, a1;
  f2upk(arg, a0, a1);
  const float r0 = t0 * ex2_approx(a0), r1 = t1 * ex2_approx(a1);                  // erfc(|u|)
  const float e0 = copysignf(1.f - r0, u0), e1 = copysignf(1.f - r1, u1);
  f2upk(fmul2(fmul2(f2pk(0.5f, 0.5f), f2pk(x0, x1)), f2pk(1.f + e0, 1.f + e1)), x0, x1);
}

struct EpiParams {
  void* out;
  int64_t ldo;
  const float* bias;        // [N] or null
  const void* res;          // residual [M, ldr] (bf16, or fp32 if res_f32) or null
  int64_t ldr;
  int res_f32;
  const float* colscale;    // per-column scale applied after act (adaLN gate) or null:
  int cs_group;             //   colscale[(row / cs_group) * cs_ld + n] if cs_group > 0, else colscale[n]
  int64_t cs_ld;
  const float* rowbias;     // per-row-group bias added before act (UNet time embedding) or null:
  int rb_group;             //   rowbias[(row / rb_group) * rb_ld + n]
  int64_t rb_ld;
  float alpha;
  int act;                  // DRS_ACT_*
  int out_f32;              // 1: fp32 output, 0: bf16
  int tma_store;            // 1: output written through smem staging + TMA (tmap_c)
  int hs_valid;             // DRS_ACT_HEADSOFTMAX: valid columns per 96-column head
  int tma_res;              // 1: residual tile TMA-loaded into the staging buffer (OutMaps::r)
  void* out2;               // kEpi 4: a bf16 copy of the (fp32) output, row stride ldo2
  int64_t ldo2;
  int early_b;              // 1: weight tiles of the first stages requested before the PDL wait
  int geglu_tanh;           // 1: GEGLU's GELU in the tanh form (one SFU op; |error| < 1e-3 of the bf16 output)
  int kpb;                  // k-blocks per ring slot / TMA box: 1, or 2 / 4 with A / B tensor maps that are
                            //    3-D [K/64][rows][64] views (kpb stages share one full/empty barrier pair)
};

// kEpi 4: the finished row segment (32 values) also goes to the bf16 copy
__device__ __forceinline__ void store_copy_bf16(const EpiParams& p, int M, int N, int row, int n0,
                                                const float (&v)[32]) {
  if (row >= M || n0 >= N) return;
  __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(p.out2) + (int64_t)row * p.ldo2 + n0;
  if (n0 + 32 <= N) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 u;
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
      for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(v[8 * q + 2 * e], v[8 * q + 2 * e + 1]);
      *reinterpret_cast<uint4*>(dst + 8 * q) = u;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) if (n0 + j < N) dst[j] = __float2bfloat16(v[j]);
  }
}

// Epilogue math on 32 consecutive accumulator columns n0..n0+31 of `row`:
// alpha, bias, row bias, activation (GEGLU folds (value, gate) pairs into 16
// outputs), column gate, residual.  Returns the number of outputs now in v[]
// (32, or 16 for GEGLU; output column of v[0] = n0 or n0 / 2).  Rows >= M
// compute garbage without touching memory (the TMA store clips them).
// bias of columns n0..n0+31 into registers (issued early so its latency hides
// under the accumulator's tcgen05.ld); false when it must be read per element
__device__ __forceinline__ bool load_bias32(const EpiParams& p, int N, int n0, float4 (&b)[8]) {
  if (!p.bias || n0 + 32 > N || (reinterpret_cast<uintptr_t>(p.bias + n0) & 15)) return false;
#pragma unroll
  for (int q = 0; q < 8; ++q) b[q] = __ldg(reinterpret_cast<const float4*>(p.bias + n0) + q);
  return true;
}

// kEpi: 4 = lean + a bf16 copy of the output (EpiParams::out2); 1 = lean (no activation, no per-row bias / column scale), 3 = lean +
// SiLU + per-row-group bias / column gate, 2 = GEGLU, 0 = GELU (tanh / erf) and
// the head softmax -- each instantiation carries only its own activation code (the
// epilogue hot loop stays small: measured 2-5 % per network eval)
// kFast (persistent / pair kernels): a residual, if any, always arrives through
// the TMA-loaded staging tile, so the per-thread residual loads are compiled out
template <int kEpi, bool kFast = false>
__device__ __forceinline__ int epi_math32(const EpiParams& p, int M, int N, int row, int n0, float (&v)[32],
                                          const float4 (&bpre)[8], bool have_bpre, bool skip_res = false) {
  const bool row_ok = row < M;
  const void* res = (kFast || skip_res) ? nullptr : p.res;   // skip: added later from the TMA-loaded tile
  const bool full = n0 + 32 <= N;
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] *= p.alpha;
  if (have_bpre) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      v[4 * q] += bpre[q].x; v[4 * q + 1] += bpre[q].y; v[4 * q + 2] += bpre[q].z; v[4 * q + 3] += bpre[q].w;
    }
  } else if (p.bias) {
    if (full && ((reinterpret_cast<uintptr_t>(p.bias + n0) & 15) == 0)) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 f = __ldg(reinterpret_cast<const float4*>(p.bias + n0) + q);
        v[4 * q] += f.x; v[4 * q + 1] += f.y; v[4 * q + 2] += f.z; v[4 * q + 3] += f.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) if (n0 + j < N) v[j] += __ldg(p.bias + n0 + j);
    }
  }
  if (kEpi != 1 && kEpi != 4 && p.rowbias && row_ok) {
    const float* rb = p.rowbias + (int64_t)(row / p.rb_group) * p.rb_ld + n0;
#pragma unroll
    for (int j = 0; j < 32; ++j) if (n0 + j < N) v[j] += __ldg(rb + j);
  }
  if (kEpi == 2 && p.act == DRS_ACT_GEGLU) {   // interleaved (value, gate) pairs -> N/2 outputs
#pragma unroll
    for (int j = 0; j < 16; j += 2) {
      float g0 = v[2 * j + 1], g1 = v[2 * j + 3];
      if (p.geglu_tanh) gelu_tanh_x2(g0, g1); else gelu_erf_x2(g0, g1);
      v[j] = v[2 * j] * g0;
      v[j + 1] = v[2 * j + 2] * g1;
    }
    const int c0 = n0 / 2;
    const bool gfull = c0 + 16 <= N / 2;
    if (res && row_ok) {
      if (p.res_f32) {
        const float* r = static_cast<const float*>(res) + (int64_t)row * p.ldr + c0;
        if (gfull && ((reinterpret_cast<uintptr_t>(r) & 15) == 0)) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float4 f = *reinterpret_cast<const float4*>(r + 4 * q);
            v[4 * q] += f.x; v[4 * q + 1] += f.y; v[4 * q + 2] += f.z; v[4 * q + 3] += f.w;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) if (c0 + j < N / 2) v[j] += r[j];
        }
      } else {
        const __nv_bfloat16* r = static_cast<const __nv_bfloat16*>(res) + (int64_t)row * p.ldr + c0;
        if (gfull && ((reinterpret_cast<uintptr_t>(r) & 15) == 0)) {
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const uint4 u = *reinterpret_cast<const uint4*>(r + 8 * q);
            const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f = __bfloat1622float2(h[e]);
              v[8 * q + 2 * e] += f.x;
              v[8 * q + 2 * e + 1] += f.y;
            }
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) if (c0 + j < N / 2) v[j] += __bfloat162float(r[j]);
        }
      }
    }
    return 16;
  }
  if (kEpi == 0 && p.act == DRS_ACT_GELU_TANH) {
#pragma unroll
    for (int j = 0; j < 32; j += 2) gelu_tanh_x2(v[j], v[j + 1]);
  } else if (kEpi == 3 && p.act == DRS_ACT_SILU) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = silu(v[j]);
  } else if (kEpi == 0 && p.act == DRS_ACT_GELU_ERF) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = gelu_erf(v[j]);
  }
  if (kEpi != 1 && kEpi != 4 && p.colscale && row_ok) {
    const float* cs = p.colscale + (p.cs_group > 0 ? (int64_t)(row / p.cs_group) * p.cs_ld : 0) + n0;
#pragma unroll
    for (int j = 0; j < 32; ++j) if (n0 + j < N) v[j] *= __ldg(cs + j);
  }
  if (res && row_ok && p.res_f32) {
    const float* r = static_cast<const float*>(res) + (int64_t)row * p.ldr + n0;
    if (full && ((reinterpret_cast<uintptr_t>(r) & 15) == 0)) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 f = *reinterpret_cast<const float4*>(r + 4 * q);
        v[4 * q] += f.x; v[4 * q + 1] += f.y; v[4 * q + 2] += f.z; v[4 * q + 3] += f.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) if (n0 + j < N) v[j] += r[j];
    }
  } else if (res && row_ok) {
    const __nv_bfloat16* r = static_cast<const __nv_bfloat16*>(res) + (int64_t)row * p.ldr + n0;
    if (full && ((reinterpret_cast<uintptr_t>(r) & 15) == 0)) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 u = *reinterpret_cast<const uint4*>(r + 8 * q);
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(h[e]);
          v[8 * q + 2 * e] += f.x;
          v[8 * q + 2 * e + 1] += f.y;
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) if (n0 + j < N) v[j] += __bfloat162float(r[j]);
    }
  }
  return 32;
}

// Direct (per-row) store of the nout outputs of epi_math32 at output column c0.
__device__ __forceinline__ void epi_store_direct(const EpiParams& p, int M, int n_out, int row, int c0, int nout,
                                                 const float (&v)[32]) {
  if (row >= M) return;
  const bool full = c0 + nout <= n_out;
  if (p.out_f32) {
    float* dst = static_cast<float*>(p.out) + (int64_t)row * p.ldo + c0;
    if (full && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (4 * q < nout)
          *reinterpret_cast<float4*>(dst + 4 * q) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) if (j < nout && c0 + j < n_out) dst[j] = v[j];
    }
  } else {
    __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(p.out) + (int64_t)row * p.ldo + c0;
    if (full && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (8 * q < nout) {
          uint4 u;
          __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
          for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(v[8 * q + 2 * e], v[8 * q + 2 * e + 1]);
          *reinterpret_cast<uint4*>(dst + 8 * q) = u;
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) if (j < nout && c0 + j < n_out) dst[j] = __float2bfloat16(v[j]);
    }
  }
}

template <int kEpi>
__device__ __forceinline__ void epilogue32(const EpiParams& p, int M, int N, int row, int n0, float (&v)[32]) {
  float4 nob[8];
  const int nout = epi_math32<kEpi>(p, M, N, row, n0, v, nob, false);
  if constexpr (kEpi == 4) store_copy_bf16(p, M, N, row, n0, v);
  const bool geglu = nout == 16;
  epi_store_direct(p, M, geglu ? N / 2 : N, row, geglu ? n0 / 2 : n0, nout, v);
}

// Staged store: this warp's 32 rows x nout outputs go to a 32-row smem tile
// (row pitch = nout * elem bytes = 32 / 64 / 128 B, TMA swizzle of the same
// span: 16-byte chunk index ^= bits 7.. of the byte offset), then one TMA
// bulk-tensor store writes the coalesced block; out-of-range rows / columns
// are clipped by the tensor map.
__device__ __forceinline__ void stage_rows(uint8_t* buf, int lane, int pitch, bool f32, const float (&v)[32]) {
  const int mask = pitch == 128 ? 7 : (pitch == 64 ? 3 : 1);
  const int nchunk = pitch / 16;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    if (q < nchunk) {
      uint4 u;
      if (f32) {
        u = make_uint4(__float_as_uint(v[4 * q]), __float_as_uint(v[4 * q + 1]), __float_as_uint(v[4 * q + 2]),
                       __float_as_uint(v[4 * q + 3]));
      } else {
        __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(v[8 * q + 2 * e], v[8 * q + 2 * e + 1]);
      }
      const int off = lane * pitch + q * 16;
      *reinterpret_cast<uint4*>(buf + (off ^ (((off >> 7) & mask) << 4))) = u;
    }
  }
}

// v += this lane's row of a staged (TMA-loaded, same swizzle as stage_rows) tile
__device__ __forceinline__ void add_staged_rows(const uint8_t* buf, int lane, int pitch, bool f32, float (&v)[32]) {
  const int mask = pitch == 128 ? 7 : (pitch == 64 ? 3 : 1);
  const int nchunk = pitch / 16;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    if (q < nchunk) {
      const int off = lane * pitch + q * 16;
      const uint4 u = *reinterpret_cast<const uint4*>(buf + (off ^ (((off >> 7) & mask) << 4)));
      if (f32) {
        v[4 * q] += __uint_as_float(u.x); v[4 * q + 1] += __uint_as_float(u.y);
        v[4 * q + 2] += __uint_as_float(u.z); v[4 * q + 3] += __uint_as_float(u.w);
      } else {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(h[e]);
          v[8 * q + 2 * e] += f.x;
          v[8 * q + 2 * e + 1] += f.y;
        }
      }
    }
  }
}

// thread-block cluster helpers (split-K reduction)
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t dsmem_map(uint32_t smem_addr, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr), "r"(rank));
  return r;
}
__device__ __forceinline__ float4 dsmem_ld4(uint32_t addr) {
  float4 f;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(f.x), "=f"(f.y), "=f"(f.z), "=f"(f.w) : "r"(addr) : "memory");
  return f;
}
__device__ __forceinline__ void fence_async_smem_g() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tma_store_2d(const void* tmap, const void* smem, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];"
               :: "l"(tmap), "r"(tc::smem_u32(smem)), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(N) : "memory"); }

// Implicit-GEMM 3x3 convolution (stride 1, pad 1) over an NHWC bf16 input:
// A[(n,y,x), (ky,kx,c)] is never materialised -- the k-block (tap, 64-channel
// block) of a 128-pixel tile is ONE 4-D TMA box {64 ch, W, rows, images} of
// the input at (c0, x0 + kx - 1, y0 * cv.stride + ky - 1, n0); TMA zero-fills the
// out-of-image taps, which is exactly the zero padding.
struct ConvGeom {
  int on;          // 0: plain GEMM (2-D A map)
  int cblocks;     // Cin / 64
  int H, W;        // image size (W <= 128, W * rows * imgs == 128 pixels per tile)
  int b_img_rows;  // > 0: tiles whose first row m has (m / b_img_rows) odd read B rows + b_img_off
  int b_img_off;
  int stride;      // 1, or 2 (H, W are then the OUTPUT grid; the TMA box walks the input with
                   // element stride 2, so input row = 2 y + ky - 1: no im2col for downsamplers)
  int a2;          // 1 (KPB=2, even cblocks): A map is 5-D (64 ch, W, H, N, C/64) and one box holds the
                   // two channel blocks of a ring slot (same tap) -- one A operation per slot
};

__device__ __forceinline__ int b_row_offset(const ConvGeom& cv, int m0) {
  return cv.b_img_rows > 0 ? ((m0 / cv.b_img_rows) & 1) * cv.b_img_off : 0;
}

template <int V>
struct KpbC { static constexpr int value = V; };   // k-blocks per ring slot, as a type

__device__ __forceinline__ void tma_load_3d(const void* tmap, uint64_t* bar, void* smem, int32_t c0, int32_t c1,
                                            int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
      :: "r"(tc::smem_u32(smem)), "l"(tmap), "r"(tc::smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__device__ __forceinline__ void tma_load_5d(const void* tmap, uint64_t* bar, void* smem, int32_t c0, int32_t c1,
                                            int32_t c2, int32_t c3, int32_t c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
      :: "r"(tc::smem_u32(smem)), "l"(tmap), "r"(tc::smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(const void* tmap, uint64_t* bar, void* smem, int32_t c0, int32_t c1,
                                            int32_t c2, int32_t c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];"
      :: "r"(tc::smem_u32(smem)), "l"(tmap), "r"(tc::smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// DRS_ACT_HEADSOFTMAX epilogue of one row: the 96 accumulator columns of one
// head (3 TMEM chunks starting at tm_col) -> p_j = 2^(s_j - max) / sum over the
// first `valid` columns, zeros after -> 96 bf16 at out[row, col0 ..].
__device__ __forceinline__ void head_softmax_row(const EpiParams& ep, int M, int N, int row, int col0,
                                                 uint32_t tm_col) {
  uint32_t r[3][32];
#pragma unroll
  for (int c = 0; c < 3; ++c) tc::tmem_ld32(tm_col + c * 32, r[c]);
  tc::tmem_ld_wait();
  if (row >= M || col0 >= N) return;
  const int valid = ep.hs_valid;
  float mx = -INFINITY;
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int e = 0; e < 32; ++e)
      if (c * 32 + e < valid) mx = fmaxf(mx, __uint_as_float(r[c][e]));
  float sum = 0.f;
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int e = 0; e < 32; ++e) {
      float pv = 0.f;
      if (c * 32 + e < valid) {
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(pv) : "f"(__uint_as_float(r[c][e]) - mx));
      }
      sum += pv;
      r[c][e] = __float_as_uint(pv);
    }
  const float inv = 1.f / sum;
  __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(ep.out) + (int64_t)row * ep.ldo + col0;
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 u;
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
      for (int e = 0; e < 4; ++e)
        h[e] = __floats2bfloat162_rn(__uint_as_float(r[c][8 * q + 2 * e]) * inv,
                                     __uint_as_float(r[c][8 * q + 2 * e + 1]) * inv);
      *reinterpret_cast<uint4*>(dst + c * 32 + 8 * q) = u;
    }
}

constexpr int kStgBytes = 4096;

// Output-side tensor maps: the staged TMA store (c) and, when the epilogue has
// a residual of the output's dtype, the residual tile loaded by TMA into the
// same staging buffer (r): one coalesced bulk load per 32 x 32 block instead
// of 32 row-strided per-thread loads, issued before the accumulator is read.
struct OutMaps {
  CUtensorMap c;
  CUtensorMap r;
};        // per epilogue warp: 2 x (32 x 32 bf16) or 1 x (32 x 32 fp32)

// Ring slot j (kpb consecutive stages) = [kpb A tiles][kpb B tiles]: one
// kpb-k-block TMA box per operand fills adjacent tiles; kpb = 1 is the plain
// [A | B] stage layout.
// Pull the bias of this warp's column chunks of the coming tile into L1 while the
// accumulator is still being produced: the epilogue's bias loads then hit L1
// instead of paying an L2 round trip per 32-column chunk (ncu: 11 % of the GEGLU
// GEMM's stall samples sat on the first bias add).
__device__ __forceinline__ void prefetch_bias_l1(const EpiParams& ep, int N, int n_first, int n_step, int n_end,
                                                 int lane) {
  if (!ep.bias) return;
  const int n0 = n_first + (lane >> 1) * n_step + (lane & 1) * 16;   // two lanes per 32-float chunk
  if (n0 < n_end && n0 < N) asm volatile("prefetch.global.L1 [%0];" :: "l"(ep.bias + n0));
}

template <int BN, int kStages>
struct GemmSmem {
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStgOffset = kStages * kStageBytes;
  static constexpr int kBarOffset = kStgOffset + kEpiWarps * kStgBytes;
  static constexpr int kBytes = kBarOffset + (2 * kStages + 16) * 8 + 1024;   // barriers; +1024 alignment slack
  static_assert(kBytes <= 227 * 1024, "GEMM shared memory plan exceeds 227 KB");
};

template <int BN, int kStages, int kEpi, bool kSplit, int KPB>
__global__ void __launch_bounds__(kGemmThreads, 1)
gemm_bf16_tc_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                    const __grid_constant__ OutMaps om, int M, int N, int K, int split_arg, EpiParams ep,
                    ConvGeom cv) {
  // kSplit: cluster split-K instantiation (one (tile, split) unit per CTA, DSMEM
  // reduction); otherwise persistent with split == 1 known at compile time
  const int split = kSplit ? split_arg : 1;
  using S = GemmSmem<BN, kStages>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + S::kBarOffset);
  uint64_t* empty_bar = full_bar + kStages;
  uint64_t* tfull_bar = empty_bar + kStages;       // [2]
  uint64_t* tempty_bar = tfull_bar + 2;            // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  uint64_t* res_bar = tempty_bar + 4;              // [kEpiWarps] residual tile loads

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m_tiles = (M + kBM - 1) / kBM, n_tiles = (N + BN - 1) / BN;
  const int num_kb_total = (K + kBK - 1) / kBK;
  const int kb_per_split = (num_kb_total + split - 1) / split;
  const int num_tiles = m_tiles * n_tiles * split;
  constexpr uint32_t kTmemCols = 2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512);   // 2 x BN, pow2
  constexpr uint32_t kIdesc = tc::idesc_bf16_f32(kBM, BN);

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tmap_a);
    tc::tma_prefetch(&tmap_b);
    if (ep.tma_store) tc::tma_prefetch(&om.c);
    if (ep.tma_res) tc::tma_prefetch(&om.r);
    for (int s = 0; s < kStages; ++s) { tc::mbar_init(&full_bar[s], 1); tc::mbar_init(&empty_bar[s], 1); }
    for (int a = 0; a < 2; ++a) { tc::mbar_init(&tfull_bar[a], 1); tc::mbar_init(&tempty_bar[a], kEpiWarps); }
    for (int w = 0; w < kEpiWarps; ++w) tc::mbar_init(&res_bar[w], 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc<kTmemCols>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  // everything above is data-independent setup (PDL overlap); the producer
  // warp additionally issues its first weight tiles before its wait (below)
  if (warp != 0) pdl_wait();
  pdl_trigger();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (tc::elect_one()) {
      // The B operand (weights) is never written by a predecessor kernel: the
      // B tiles of the first kStages k-blocks are requested BEFORE the PDL wait,
      // so the cold weight stream overlaps the previous kernel's tail (the
      // stage's full barrier also expects the A bytes, which follow the wait).
      // kb2: a ring slot ("super-stage") is 2 consecutive stages = 2 k-blocks,
      // loaded by one 3-D box per operand (conv A: one 4-D box per k-block)
      auto kpb_body = [&](auto kpb_c) {   // KPB: k-blocks per ring slot (separate instantiations)
        constexpr int kpb = decltype(kpb_c)::value;
        const int nst = kStages / kpb;
        int pre = 0;
        if ((int)blockIdx.x < num_tiles) {
          const int sp = blockIdx.x % split, mn = blockIdx.x / split;
          const int mt = mn % m_tiles, nt = mn / m_tiles;
          const int kb0 = sp * kb_per_split, kb1 = min(num_kb_total, kb0 + kb_per_split);
          pre = ep.early_b ? max(0, min(nst, (kb1 - kb0 + kpb - 1) / kpb)) : 0;
          for (int j = 0; j < pre; ++j) {
            uint8_t* sb = smem + j * kpb * S::kStageBytes + kpb * S::kABytes;
            tc::mbar_arrive_expect_tx(&full_bar[j], kpb * S::kStageBytes);
            if (kpb > 1)
              tma_load_3d(&tmap_b, &full_bar[j], sb, 0, nt * BN + b_row_offset(cv, mt * kBM), kb0 + j * kpb);
            else
              tc::tma_load_2d(&tmap_b, &full_bar[j], sb, (kb0 + j) * kBK, nt * BN + b_row_offset(cv, mt * kBM));
          }
        }
        pdl_wait();
        int stage = 0;
        uint32_t phase = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
          const int sp = tile % split;
          const int mn = tile / split;
          const int mt = mn % m_tiles, nt = mn / m_tiles;
          const int kb0 = sp * kb_per_split;
          const int kb1 = min(num_kb_total, kb0 + kb_per_split);
          for (int kb = kb0, j = 0; kb < kb1; kb += kpb, ++j) {
            const bool b_done = tile == (int)blockIdx.x && j < pre;   // weights already in flight
            if (!b_done) tc::mbar_wait(&empty_bar[stage], phase ^ 1);
            uint8_t* sa = smem + stage * kpb * S::kStageBytes;
            uint8_t* sb = smem + stage * kpb * S::kStageBytes + kpb * S::kABytes;
            if (!b_done) tc::mbar_arrive_expect_tx(&full_bar[stage], kpb * S::kStageBytes);
            if (cv.on && kpb > 1 && cv.a2) {    // both channel blocks of the slot (same tap) in one box
              const int tap = kb / cv.cblocks, cb = kb - tap * cv.cblocks;
              const int ky = tap / 3, kx = tap - ky * 3;
              const int m0 = mt * kBM, hw = cv.H * cv.W;
              const int n0 = m0 / hw, y0 = (m0 - n0 * hw) / cv.W;
              tma_load_5d(&tmap_a, &full_bar[stage], sa, 0, kx - 1, y0 * cv.stride + ky - 1, n0, cb);
            } else if (cv.on) {
              for (int q = 0; q < kpb; ++q) {       // a missing 2nd k-block of a conv: zero A bytes via the
                const int k = min(kb + q, num_kb_total - 1);   // last valid box again (its MMA is skipped)
                const int tap = k / cv.cblocks, cb = k - tap * cv.cblocks;
                const int ky = tap / 3, kx = tap - ky * 3;
                const int m0 = mt * kBM, hw = cv.H * cv.W;
                const int n0 = m0 / hw, y0 = (m0 - n0 * hw) / cv.W;
                tma_load_4d(&tmap_a, &full_bar[stage], sa + q * S::kABytes, cb * 64, kx - 1, y0 * cv.stride + ky - 1, n0);
              }
            } else if (kpb > 1) {
              tma_load_3d(&tmap_a, &full_bar[stage], sa, 0, mt * kBM, kb);
            } else {
              tc::tma_load_2d(&tmap_a, &full_bar[stage], sa, kb * kBK, mt * kBM);
            }
            if (!b_done) {
              if (kpb > 1)
                tma_load_3d(&tmap_b, &full_bar[stage], sb, 0, nt * BN + b_row_offset(cv, mt * kBM), kb);
              else
                tc::tma_load_2d(&tmap_b, &full_bar[stage], sb, kb * kBK, nt * BN + b_row_offset(cv, mt * kBM));
            }
            if (++stage == nst) { stage = 0; phase ^= 1; }
          }
        }
      };
      kpb_body(KpbC<KPB>{});
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    auto kpb_body = [&](auto kpb_c) {   // KPB: k-blocks per ring slot (separate instantiations)
      constexpr int kpb = decltype(kpb_c)::value;
      const int nst = kStages / kpb;
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
        const int sp = tile % split;
        const int kb0 = sp * kb_per_split;
        const int kb1 = min(num_kb_total, kb0 + kb_per_split);
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        tc::mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; kb += kpb) {
          tc::mbar_wait(&full_bar[stage], phase);
          tc::tc_fence_after();
          if (tc::elect_one()) {
            for (int q = 0; q < kpb && kb + q < kb1; ++q) {
              const uint64_t da = tc::smem_desc_sw128(smem + stage * kpb * S::kStageBytes + q * S::kABytes);
              const uint64_t db = tc::smem_desc_sw128(smem + stage * kpb * S::kStageBytes + kpb * S::kABytes + q * S::kBBytes);
  #pragma unroll
              for (int k = 0; k < kBK / 16; ++k)      // +32 B per K=16 step inside the swizzle atom
                tc::mma_bf16(d_tmem, da + 2 * k, db + 2 * k, kIdesc, (kb + q > kb0 || k > 0) ? 1u : 0u);
            }
            tc::mma_commit(&empty_bar[stage]);
            if (kb + kpb >= kb1) tc::mma_commit(&tfull_bar[acc]);
          }
          __syncwarp();
          if (++stage == nst) { stage = 0; phase ^= 1; }
        }
        if (kb1 <= kb0) {                            // empty K range: still publish a (zero) tile
          if (tc::elect_one()) tc::mma_commit(&tfull_bar[acc]);
          __syncwarp();
        }
      }
    };
    kpb_body(KpbC<KPB>{});
  } else {
    // ---------------- epilogue (warps 2..9) ----------------
    const int quad = warp & 3;                     // TMEM lane quadrant this warp may access
    const int half = (warp - 2) >> 2;              // which 32-column chunks (even / odd) it drains
    const bool geglu = kEpi == 2 && ep.act == DRS_ACT_GEGLU;
    const int pitch = (geglu ? 16 : 32) * (ep.out_f32 ? 4 : 2);   // staged row bytes
    const bool dbl = pitch * 32 <= kStgBytes / 2;                 // two staging buffers fit
    uint8_t* stg = smem + S::kStgOffset + (warp - 2) * kStgBytes;
    int buf = 0;
    uint32_t rph = 0;                              // res_bar phase of this warp
    int it = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      const int sp = tile % split;
      const int mn = tile / split;
      const int mt = mn % m_tiles, nt = mn / m_tiles;
      const int kb0 = sp * kb_per_split;
      const int kb1 = min(num_kb_total, kb0 + kb_per_split);
      const int acc = it & 1;
      if (split == 1) prefetch_bias_l1(ep, N, nt * BN + half * 32, 64, nt * BN + BN, lane);
      tc::mbar_wait(&tfull_bar[acc], (it >> 1) & 1);
      tc::tc_fence_after();
      const int row = mt * kBM + quad * 32 + lane;
      if constexpr (BN == 192 && kEpi == 0) {
        if (ep.act == DRS_ACT_HEADSOFTMAX) {       // warp half h: head 2 nt + h = columns [96 h, 96 h + 96)
          head_softmax_row(ep, M, N, row, nt * BN + half * 96,
                           tmem_base + ((uint32_t)(quad * 32) << 16) + acc * BN + half * 96);
          tc::tc_fence_before();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&tempty_bar[acc]);
          continue;
        }
      }
#pragma unroll 1
      for (int c = half; c < BN / 32; c += 2) {
        const int n0 = nt * BN + c * 32;
        float4 bpre[8];
        const bool have_b = split == 1 && n0 < N && load_bias32(ep, N, n0, bpre);
        uint8_t* sb = stg + buf * (kStgBytes / 2);
        if (ep.tma_res && n0 < N && lane == 0) {    // residual tile -> staging buffer, under the TMEM load
          if (dbl) bulk_wait_read<1>(); else bulk_wait_read<0>();
          tc::mbar_arrive_expect_tx(&res_bar[warp - 2], (uint32_t)(pitch * 32));
          tc::tma_load_2d(&om.r, &res_bar[warp - 2], sb, n0, mt * kBM + quad * 32);
        }
        uint32_t r[32];
        tc::tmem_ld32(tmem_base + ((uint32_t)(quad * 32) << 16) + acc * BN + c * 32, r);
        tc::tmem_ld_wait();
        if (n0 >= N) continue;
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = (!kSplit || kb1 > kb0) ? __uint_as_float(r[j]) : 0.f;
        if (kSplit) {
          // partial tile -> this CTA's smem (padded rows: conflict-free float4 stores)
          float* dst = reinterpret_cast<float*>(smem) + (quad * 32 + lane) * (BN + 4) + c * 32;
#pragma unroll
          for (int q = 0; q < 8; ++q)
            *reinterpret_cast<float4*>(dst + 4 * q) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        } else {                                   // persistent kernel: always the staged TMA store
          epi_math32<kEpi, true>(ep, M, N, row, n0, v, bpre, have_b, ep.tma_res != 0);
          if (ep.tma_res) {
            tc::mbar_wait(&res_bar[warp - 2], rph);
            rph ^= 1;
            add_staged_rows(sb, lane, pitch, ep.out_f32 != 0, v);
          } else {
            // the buffer about to be written must have been read by its last store
            if (lane == 0) {
              if (dbl) bulk_wait_read<1>(); else bulk_wait_read<0>();
            }
          }
          __syncwarp();
          if constexpr (kEpi == 4) store_copy_bf16(ep, M, N, row, n0, v);
          stage_rows(sb, lane, pitch, ep.out_f32 != 0, v);
          fence_async_smem_g();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&om.c, sb, geglu ? n0 / 2 : n0, mt * kBM + quad * 32);
            bulk_commit();
          }
          if (dbl) buf ^= 1;
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty_bar[acc]);
    }
    if (ep.tma_store && lane == 0) bulk_wait_read<0>();   // smem reads done; the writes complete with the grid
  }
  if (kSplit) {
    // ---------------- cluster split-K reduction over DSMEM ----------------
    // (non-persistent: this CTA computed exactly one (tile, split) unit; its
    // cluster rank is its split index)
    __syncwarp();
    cluster_sync();                                // every partial tile is in smem
    if (warp >= 2) {
      const int sp = blockIdx.x % split;
      const int mn = blockIdx.x / split;
      const int mt = mn % m_tiles, nt = mn / m_tiles;
      const int t = threadIdx.x - 64;              // 0..255
      const uint32_t base = tc::smem_u32(smem);
      constexpr int kChunks = BN / 32;
      const int rows_here = (kBM - sp + split - 1) / split;      // rows sp, sp+split, ...
      for (int item = t; item < rows_here * kChunks; item += kEpiWarps * 32) {
        const int r = sp + (item / kChunks) * split;
        const int c = item % kChunks;
        const int n0 = nt * BN + c * 32;
        if (n0 >= N) continue;
        const uint32_t off = (uint32_t)((r * (BN + 4) + c * 32) * 4);
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = 0.f;
        for (int s2 = 0; s2 < split; ++s2) {
          const uint32_t ra = dsmem_map(base + off, s2);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 f = dsmem_ld4(ra + 16 * q);
            v[4 * q] += f.x; v[4 * q + 1] += f.y; v[4 * q + 2] += f.z; v[4 * q + 3] += f.w;
          }
        }
        epilogue32<kEpi>(ep, M, N, mt * kBM + r, n0, v);
      }
    }
    __syncwarp();
    cluster_sync();                                // peers are done reading this CTA's smem
  }
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<kTmemCols>(tmem_base);
}

// ---- 2-SM (CTA pair) variant: tcgen05.mma.cta_group::2, M = 256 per pair ----
// The two CTAs of a cluster share one 256 x BN output tile: CTA r owns rows
// r*128 .. r*128+127 (its own A tile and TMEM accumulator) and loads HALF of
// the B tile (BN/2 rows, at the same smem offset in both CTAs); the leader's
// single thread issues the M=256 MMAs, which read A from each CTA's smem and
// the two B halves across the pair.  Per-SM operand ingest per k-block drops
// from (128 + BN) x 128 B to (128 + BN/2) x 128 B -- the bound of the 1-SM
// kernel on the UNet shapes.  Barriers: every TMA of the pair completes on
// the LEADER's full barrier; the leader's MMA commits multicast to both CTAs'
// empty / tfull barriers; both CTAs' epilogue warps arrive on the leader's
// tempty barrier (remote arrive through DSMEM).
template <int BN, int kStages>
struct PairSmem {
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = (BN / 2) * kBK * 2;         // this CTA's half of B
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStgOffset = kStages * kStageBytes;
  static constexpr int kBarOffset = kStgOffset + kEpiWarps * kStgBytes;
  static constexpr int kBytes = kBarOffset + (2 * kStages + 16) * 8 + 1024;
  static_assert(kBytes <= 227 * 1024, "GEMM pair shared memory plan exceeds 227 KB");
};

__device__ __forceinline__ void tma_load_2d_pair(const void* tmap, uint64_t* bar, void* smem, int32_t c0, int32_t c1) {
  // completes on the leader's barrier: clear the peer bit of the shared::cluster address
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];"
      :: "r"(tc::smem_u32(smem)), "l"(tmap), "r"(tc::smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void tma_load_3d_pair(const void* tmap, uint64_t* bar, void* smem, int32_t c0, int32_t c1,
                                                 int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];"
      :: "r"(tc::smem_u32(smem)), "l"(tmap), "r"(tc::smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_load_5d_pair(const void* tmap, uint64_t* bar, void* smem, int32_t c0, int32_t c1,
                                                 int32_t c2, int32_t c3, int32_t c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
      :: "r"(tc::smem_u32(smem)), "l"(tmap), "r"(tc::smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1), "r"(c2),
         "r"(c3), "r"(c4) : "memory");
}
__device__ __forceinline__ void tma_load_4d_pair(const void* tmap, uint64_t* bar, void* smem, int32_t c0, int32_t c1,
                                                 int32_t c2, int32_t c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];"
      :: "r"(tc::smem_u32(smem)), "l"(tmap), "r"(tc::smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1), "r"(c2),
         "r"(c3) : "memory");
}
__device__ __forceinline__ void mma_bf16_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
      :: "r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate) : "memory");
}
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {      // both CTAs' barrier
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               :: "r"(tc::smem_u32(bar)), "h"((uint16_t)3) : "memory");
}
__device__ __forceinline__ uint32_t pair_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {   // arrive on rank 0's copy of `bar`
  uint32_t a = tc::smem_u32(bar), r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(a));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" :: "r"(r) : "memory");
}
__device__ __forceinline__ void pair_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// A operand of a pair CTA's ring slot: kpb k-blocks (conv: one 4-D box per k-block,
// a missing 2nd block of the last slot reloads a valid box whose MMA is skipped;
// otherwise one 2-D box, or one 3-D box carrying 2 k-blocks)
__device__ __forceinline__ void pair_load_a(const CUtensorMap* tmap_a, uint64_t* bar, uint8_t* sa, int a_bytes, int kb,
                                            int num_kb, int m0, const ConvGeom& cv, int kpb) {
  if (cv.on && kpb > 1 && cv.a2) {
    const int tap = kb / cv.cblocks, cb = kb - tap * cv.cblocks;
    const int ky = tap / 3, kx = tap - ky * 3;
    const int hw = cv.H * cv.W;
    const int n0 = m0 / hw, y0 = (m0 - n0 * hw) / cv.W;
    tma_load_5d_pair(tmap_a, bar, sa, 0, kx - 1, y0 * cv.stride + ky - 1, n0, cb);
  } else if (cv.on) {
    for (int q = 0; q < kpb; ++q) {
      const int k = min(kb + q, num_kb - 1);
      const int tap = k / cv.cblocks, cb = k - tap * cv.cblocks;
      const int ky = tap / 3, kx = tap - ky * 3;
      const int hw = cv.H * cv.W;
      const int n0 = m0 / hw, y0 = (m0 - n0 * hw) / cv.W;
      tma_load_4d_pair(tmap_a, bar, sa + q * a_bytes, cb * 64, kx - 1, y0 * cv.stride + ky - 1, n0);
    }
  } else if (kpb > 1) {
    tma_load_3d_pair(tmap_a, bar, sa, 0, m0, kb);
  } else {
    tma_load_2d_pair(tmap_a, bar, sa, kb * kBK, m0);
  }
}
__device__ __forceinline__ void pair_load_b(const CUtensorMap* tmap_b, uint64_t* bar, uint8_t* sb, int kb, int row,
                                            int kpb) {
  if (kpb > 1)
    tma_load_3d_pair(tmap_b, bar, sb, 0, row, kb);
  else
    tma_load_2d_pair(tmap_b, bar, sb, kb * kBK, row);
}

template <int BN, int kStages, int kEpi, int KPB>
__global__ void __launch_bounds__(kGemmThreads, 1)
gemm_pair_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                 const __grid_constant__ OutMaps om, int M, int N, int K, EpiParams ep, ConvGeom cv) {
  using S = PairSmem<BN, kStages>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + S::kBarOffset);
  uint64_t* empty_bar = full_bar + kStages;
  uint64_t* tfull_bar = empty_bar + kStages;       // [2]
  uint64_t* tempty_bar = tfull_bar + 2;            // [2] (leader's counts both CTAs' epilogues)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  uint64_t* res_bar = tempty_bar + 4;              // [kEpiWarps] residual tile loads

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = (int)pair_rank();
  const int pm_tiles = (M + 2 * kBM - 1) / (2 * kBM), n_tiles = (N + BN - 1) / BN;
  const int num_kb = (K + kBK - 1) / kBK;
  const int num_tiles = pm_tiles * n_tiles;
  const int t0 = blockIdx.x / 2, tstep = gridDim.x / 2;
  constexpr uint32_t kTmemCols = 2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512);
  constexpr uint32_t kIdesc = tc::idesc_bf16_f32(2 * kBM, BN);

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tmap_a);
    tc::tma_prefetch(&tmap_b);
    if (ep.tma_store) tc::tma_prefetch(&om.c);
    if (ep.tma_res) tc::tma_prefetch(&om.r);
    for (int s = 0; s < kStages; ++s) { tc::mbar_init(&full_bar[s], 1); tc::mbar_init(&empty_bar[s], 1); }
    for (int a = 0; a < 2; ++a) { tc::mbar_init(&tfull_bar[a], 1); tc::mbar_init(&tempty_bar[a], 2 * kEpiWarps); }
    for (int w = 0; w < kEpiWarps; ++w) tc::mbar_init(&res_bar[w], 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) {                                  // both CTAs, same warp and slot (cta_group::2 allocation)
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(tc::smem_u32(tmem_slot)), "n"(kTmemCols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc::tc_fence_before();
  __syncthreads();
  pair_sync();                                      // barriers and TMEM of both CTAs are ready
  tc::tc_fence_after();
  if (warp != 0) pdl_wait();                       // producer: after its early weight loads (below)
  pdl_trigger();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs: own A rows, half of B) ----------------
    if (tc::elect_one()) {
      // weight (B) halves of the first kStages k-blocks before the PDL wait (as in
      // gemm_bf16_tc_kernel): they never depend on a predecessor kernel
      // kb2: ring slots of 2 stages / 2 k-blocks per TMA box (see gemm_bf16_tc_kernel)
      auto kpb_body = [&](auto kpb_c) {   // KPB: k-blocks per ring slot (separate instantiations)
        constexpr int kpb = decltype(kpb_c)::value;
        const int nst = kStages / kpb;
        int pre = 0;
        if (t0 < num_tiles) {
          const int pmt = t0 % pm_tiles, nt = t0 / pm_tiles;
          pre = ep.early_b ? min(nst, (num_kb + kpb - 1) / kpb) : 0;
          for (int j = 0; j < pre; ++j) {
            uint8_t* sb = smem + j * kpb * S::kStageBytes + kpb * S::kABytes;
            if (rank == 0) tc::mbar_arrive_expect_tx(&full_bar[j], 2 * kpb * S::kStageBytes);
            pair_load_b(&tmap_b, &full_bar[j], sb, j * kpb, nt * BN + rank * (BN / 2) + b_row_offset(cv, pmt * 2 * kBM),
                        kpb);
          }
        }
        pdl_wait();
        int stage = 0;
        uint32_t phase = 0;
        for (int tile = t0; tile < num_tiles; tile += tstep) {
          const int pmt = tile % pm_tiles, nt = tile / pm_tiles;
          const int m0 = (pmt * 2 + rank) * kBM;
          for (int kb = 0, j = 0; kb < num_kb; kb += kpb, ++j) {
            const bool b_done = tile == t0 && j < pre;
            if (!b_done) tc::mbar_wait(&empty_bar[stage], phase ^ 1);
            uint8_t* sa = smem + stage * kpb * S::kStageBytes;
            uint8_t* sb = smem + stage * kpb * S::kStageBytes + kpb * S::kABytes;
            if (rank == 0 && !b_done) tc::mbar_arrive_expect_tx(&full_bar[stage], 2 * kpb * S::kStageBytes);
            pair_load_a(&tmap_a, &full_bar[stage], sa, S::kABytes, kb, num_kb, m0, cv, kpb);
            if (!b_done)
              pair_load_b(&tmap_b, &full_bar[stage], sb, kb, nt * BN + rank * (BN / 2) + b_row_offset(cv, pmt * 2 * kBM),
                          kpb);
            if (++stage == nst) { stage = 0; phase ^= 1; }
          }
        }
      };
      kpb_body(KpbC<KPB>{});
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader only) ----------------
    if (rank == 0) {
      auto kpb_body = [&](auto kpb_c) {   // KPB: k-blocks per ring slot (separate instantiations)
        constexpr int kpb = decltype(kpb_c)::value;
        const int nst = kStages / kpb;
        int stage = 0;
        uint32_t phase = 0;
        int it = 0;
        for (int tile = t0; tile < num_tiles; tile += tstep, ++it) {
          const int acc = it & 1;
          tc::mbar_wait(&tempty_bar[acc], ((it >> 1) & 1) ^ 1);
          tc::tc_fence_after();
          const uint32_t d_tmem = tmem_base + acc * BN;
          for (int kb = 0; kb < num_kb; kb += kpb) {
            tc::mbar_wait(&full_bar[stage], phase);
            tc::tc_fence_after();
            if (tc::elect_one()) {
              for (int q = 0; q < kpb && kb + q < num_kb; ++q) {
                const uint64_t da = tc::smem_desc_sw128(smem + stage * kpb * S::kStageBytes + q * S::kABytes);
                const uint64_t db = tc::smem_desc_sw128(smem + stage * kpb * S::kStageBytes + kpb * S::kABytes + q * S::kBBytes);
  #pragma unroll
                for (int k = 0; k < kBK / 16; ++k)
                  mma_bf16_pair(d_tmem, da + 2 * k, db + 2 * k, kIdesc, (kb + q > 0 || k > 0) ? 1u : 0u);
              }
              mma_commit_pair(&empty_bar[stage]);
              if (kb + kpb >= num_kb) mma_commit_pair(&tfull_bar[acc]);
            }
            __syncwarp();
            if (++stage == nst) { stage = 0; phase ^= 1; }
          }
        }
      };
      kpb_body(KpbC<KPB>{});
    }
  } else {
    // ---------------- epilogue (warps 2..9 of both CTAs: own 128 rows) ----------------
    const int quad = warp & 3;
    const int half = (warp - 2) >> 2;
    const bool geglu = kEpi == 2 && ep.act == DRS_ACT_GEGLU;
    const int pitch = (geglu ? 16 : 32) * (ep.out_f32 ? 4 : 2);
    const bool dbl = pitch * 32 <= kStgBytes / 2;
    uint8_t* stg = smem + S::kStgOffset + (warp - 2) * kStgBytes;
    int buf = 0;
    uint32_t rph = 0;                              // res_bar phase of this warp
    int it = 0;
    for (int tile = t0; tile < num_tiles; tile += tstep, ++it) {
      const int pmt = tile % pm_tiles, nt = tile / pm_tiles;
      const int mrow0 = (pmt * 2 + rank) * kBM;
      const int acc = it & 1;
      prefetch_bias_l1(ep, N, nt * BN + half * 32, 64, nt * BN + BN, lane);
      tc::mbar_wait(&tfull_bar[acc], (it >> 1) & 1);
      tc::tc_fence_after();
      const int row = mrow0 + quad * 32 + lane;
#pragma unroll 1
      for (int c = half; c < BN / 32; c += 2) {
        const int n0 = nt * BN + c * 32;
        float4 bpre[8];
        const bool have_b = n0 < N && load_bias32(ep, N, n0, bpre);
        uint8_t* sb = stg + buf * (kStgBytes / 2);
        if (ep.tma_res && n0 < N && lane == 0) {    // residual tile -> staging buffer, under the TMEM load
          if (dbl) bulk_wait_read<1>(); else bulk_wait_read<0>();
          tc::mbar_arrive_expect_tx(&res_bar[warp - 2], (uint32_t)(pitch * 32));
          tc::tma_load_2d(&om.r, &res_bar[warp - 2], sb, n0, mrow0 + quad * 32);
        }
        uint32_t r[32];
        tc::tmem_ld32(tmem_base + ((uint32_t)(quad * 32) << 16) + acc * BN + c * 32, r);
        tc::tmem_ld_wait();
        if (n0 >= N) continue;
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        {                                          // the host pairs only TMA-store epilogues
          epi_math32<kEpi, true>(ep, M, N, row, n0, v, bpre, have_b, ep.tma_res != 0);
          if (ep.tma_res) {
            tc::mbar_wait(&res_bar[warp - 2], rph);
            rph ^= 1;
            add_staged_rows(sb, lane, pitch, ep.out_f32 != 0, v);
          } else {
            // the buffer about to be written must have been read by its last store
            if (lane == 0) {
              if (dbl) bulk_wait_read<1>(); else bulk_wait_read<0>();
            }
          }
          __syncwarp();
          if constexpr (kEpi == 4) store_copy_bf16(ep, M, N, row, n0, v);
          stage_rows(sb, lane, pitch, ep.out_f32 != 0, v);
          fence_async_smem_g();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&om.c, sb, geglu ? n0 / 2 : n0, mrow0 + quad * 32);
            bulk_commit();
          }
          if (dbl) buf ^= 1;
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_leader(&tempty_bar[acc]);
    }
    if (ep.tma_store && lane == 0) bulk_wait_read<0>();   // smem reads done; the writes complete with the grid
  }
  __syncwarp();
  tc::tc_fence_before();
  pair_sync();                                      // all MMAs / epilogues of the pair are done
  if (warp == 1) {
    tc::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(tmem_base), "n"(kTmemCols) : "memory");
  }
}

// ---- CTA pair + cluster split-K: small-M, long-K GEMMs ----
// A cluster of 2 * split CTAs owns one 256 x BN output tile: ranks (2s, 2s+1)
// are a tcgen05 CTA pair (as in gemm_pair_kernel: each CTA its 128 A rows and
// half of the B tile) accumulating K range s; the pairs then park their fp32
// partial tiles in their own (idle) pipeline smem and, after one cluster
// barrier, CTA (h, s) reduces rows s, s + split, ... of half h over the split
// peers (ranks h, h + 2, ...) through DSMEM in the fixed order 0..split-1
// (deterministic, no workspace) and runs the epilogue.  Operand ingest per SM
// per k-block is (128 + BN/2) x 128 B -- the pair kernel's -- while split-K
// keeps every SM busy on the few tiles of a small-M layer.
__device__ __forceinline__ void mma_commit_pair_mask(uint64_t* bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               :: "r"(tc::smem_u32(bar)), "h"(mask) : "memory");
}

template <int BN, int kStages, int kEpi, int KPB>
__global__ void __launch_bounds__(kGemmThreads, 1)
gemm_pair_split_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                       int M, int N, int K, int split, EpiParams ep, ConvGeom cv) {
  using S = PairSmem<BN, kStages>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + S::kBarOffset);
  uint64_t* empty_bar = full_bar + kStages;
  uint64_t* tfull_bar = empty_bar + kStages;       // [1]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull_bar + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = (int)pair_rank();               // rank in the 2 * split cluster
  const int half = rank & 1, sp = rank >> 1;
  const uint16_t pair_mask = (uint16_t)(3u << (rank & ~1));
  const int pm_tiles = (M + 2 * kBM - 1) / (2 * kBM);
  const int tile = blockIdx.x / (2 * split);
  const int pmt = tile % pm_tiles, nt = tile / pm_tiles;
  const int m0 = (pmt * 2 + half) * kBM;
  const int num_kb = (K + kBK - 1) / kBK;
  const int kb_per = (num_kb + split - 1) / split;
  const int kb0 = sp * kb_per, kb1 = min(num_kb, kb0 + kb_per);
  constexpr uint32_t kTmemCols = BN <= 64 ? 64 : (BN <= 128 ? 128 : 256);
  constexpr uint32_t kIdesc = tc::idesc_bf16_f32(2 * kBM, BN);

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tmap_a);
    tc::tma_prefetch(&tmap_b);
    for (int s2 = 0; s2 < kStages; ++s2) { tc::mbar_init(&full_bar[s2], 1); tc::mbar_init(&empty_bar[s2], 1); }
    tc::mbar_init(&tfull_bar[0], 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(tc::smem_u32(tmem_slot)), "n"(kTmemCols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc::tc_fence_before();
  __syncthreads();
  pair_sync();                                      // barriers and TMEM of the whole cluster are ready
  tc::tc_fence_after();
  if (warp != 0) pdl_wait();                       // producer: after its early weight loads (below)
  pdl_trigger();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (tc::elect_one()) {
      // weight (B) halves of the first kStages k-blocks before the PDL wait
      auto kpb_body = [&](auto kpb_c) {   // KPB: k-blocks per ring slot (separate instantiations)
        constexpr int kpb = decltype(kpb_c)::value;
        const int nst = kStages / kpb;
        const int pre = ep.early_b ? max(0, min(nst, (kb1 - kb0 + kpb - 1) / kpb)) : 0;
        for (int j = 0; j < pre; ++j) {
          uint8_t* sb = smem + j * kpb * S::kStageBytes + kpb * S::kABytes;
          if (half == 0) tc::mbar_arrive_expect_tx(&full_bar[j], 2 * kpb * S::kStageBytes);
          pair_load_b(&tmap_b, &full_bar[j], sb, kb0 + j * kpb, nt * BN + half * (BN / 2) + b_row_offset(cv, pmt * 2 * kBM),
                      kpb);
        }
        pdl_wait();
        int stage = 0;
        uint32_t phase = 0;
        for (int kb = kb0, j = 0; kb < kb1; kb += kpb, ++j) {
          const bool b_done = j < pre;
          if (!b_done) tc::mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * kpb * S::kStageBytes;
          uint8_t* sb = smem + stage * kpb * S::kStageBytes + kpb * S::kABytes;
          if (half == 0 && !b_done) tc::mbar_arrive_expect_tx(&full_bar[stage], 2 * kpb * S::kStageBytes);
          pair_load_a(&tmap_a, &full_bar[stage], sa, S::kABytes, kb, num_kb, m0, cv, kpb);
          if (!b_done)
            pair_load_b(&tmap_b, &full_bar[stage], sb, kb, nt * BN + half * (BN / 2) + b_row_offset(cv, pmt * 2 * kBM),
                        kpb);
          if (++stage == nst) { stage = 0; phase ^= 1; }
        }
      };
      kpb_body(KpbC<KPB>{});
    }
  } else if (warp == 1) {
    if (half == 0) {
      auto kpb_body = [&](auto kpb_c) {   // KPB: k-blocks per ring slot (separate instantiations)
        constexpr int kpb = decltype(kpb_c)::value;
        const int nst = kStages / kpb;
        int stage = 0;
        uint32_t phase = 0;
        for (int kb = kb0; kb < kb1; kb += kpb) {
          tc::mbar_wait(&full_bar[stage], phase);
          tc::tc_fence_after();
          if (tc::elect_one()) {
            for (int q = 0; q < kpb && kb + q < kb1; ++q) {
              const uint64_t da = tc::smem_desc_sw128(smem + stage * kpb * S::kStageBytes + q * S::kABytes);
              const uint64_t db = tc::smem_desc_sw128(smem + stage * kpb * S::kStageBytes + kpb * S::kABytes + q * S::kBBytes);
  #pragma unroll
              for (int k = 0; k < kBK / 16; ++k)
                mma_bf16_pair(tmem_base, da + 2 * k, db + 2 * k, kIdesc, (kb + q > kb0 || k > 0) ? 1u : 0u);
            }
            mma_commit_pair_mask(&empty_bar[stage], pair_mask);
            if (kb + kpb >= kb1) mma_commit_pair_mask(&tfull_bar[0], pair_mask);
          }
          __syncwarp();
          if (++stage == nst) { stage = 0; phase ^= 1; }
        }
      };
      kpb_body(KpbC<KPB>{});
      if (kb1 <= kb0) {                            // empty K range: still publish a (zero) tile
        if (tc::elect_one()) mma_commit_pair_mask(&tfull_bar[0], pair_mask);
        __syncwarp();
      }
    }
  } else {
    // partial tile (this CTA's 128 rows) -> own smem, padded rows
    const int quad = warp & 3;
    const int hw_ = (warp - 2) >> 2;
    tc::mbar_wait(&tfull_bar[0], 0);
    tc::tc_fence_after();
#pragma unroll 1
    for (int c = hw_; c < BN / 32; c += 2) {
      uint32_t r[32];
      tc::tmem_ld32(tmem_base + ((uint32_t)(quad * 32) << 16) + c * 32, r);
      tc::tmem_ld_wait();
      float* dst = reinterpret_cast<float*>(smem) + (quad * 32 + lane) * (BN + 4) + c * 32;
      const bool z = kb1 <= kb0;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        *reinterpret_cast<float4*>(dst + 4 * q) =
            z ? make_float4(0.f, 0.f, 0.f, 0.f)
              : make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]), __uint_as_float(r[4 * q + 2]),
                            __uint_as_float(r[4 * q + 3]));
    }
  }
  __syncwarp();
  tc::tc_fence_before();
  cluster_sync();                                  // every partial tile of the cluster is in smem
  if (warp >= 2) {
    const int t = threadIdx.x - 64;                // 0..255
    const uint32_t base = tc::smem_u32(smem);
    constexpr int kChunks = BN / 32;
    const int rows_here = (kBM - sp + split - 1) / split;      // rows sp, sp + split, ...
    for (int item = t; item < rows_here * kChunks; item += kEpiWarps * 32) {
      const int r = sp + (item / kChunks) * split;
      const int c = item % kChunks;
      const int n0 = nt * BN + c * 32;
      if (n0 >= N) continue;
      const uint32_t off = (uint32_t)((r * (BN + 4) + c * 32) * 4);
      float v[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = 0.f;
      for (int s2 = 0; s2 < split; ++s2) {
        const uint32_t ra = dsmem_map(base + off, half + 2 * s2);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 f = dsmem_ld4(ra + 16 * q);
          v[4 * q] += f.x; v[4 * q + 1] += f.y; v[4 * q + 2] += f.z; v[4 * q + 3] += f.w;
        }
      }
      epilogue32<kEpi>(ep, M, N, m0 + r, n0, v);
    }
  }
  __syncwarp();
  cluster_sync();                                  // peers are done reading this CTA's smem
  if (warp == 1) {
    tc::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(tmem_base), "n"(kTmemCols) : "memory");
  }
}

// ------------------------------------------------------------ host side ---
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled encode_fn() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  return fn;
}

// 2-D bf16 tensor map: `rows` x `cols` (cols contiguous), row stride in elements.
static bool make_tmap(CUtensorMap* m, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  PFN_encodeTiled enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// NHWC input as {C, W, H, N}; box {64 ch, W, rows, imgs} with W * rows * imgs == 128
// H, W: the OUTPUT grid; the input is (s H) x (s W).  With s = 2 the box spans
// 2 W x 2 rows input elements traversed with element stride 2, i.e. it loads the
// same 128 x 64-channel tile of pixels (s y + ky - 1, s x + kx - 1).
// 3-D view [K/64][rows][64] of a K-contiguous bf16 matrix (K % 64 == 0): a
// {64, box_rows, kpb} box is kpb consecutive k-block tiles (kpb = 2 or 4)
static bool make_tmap_kb2(CUtensorMap* m, const void* ptr, int64_t rows, int64_t K, int64_t ld, int box_rows,
                          int kpb) {
  PFN_encodeTiled enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)kBK, (cuuint64_t)rows, (cuuint64_t)(K / kBK)};
  cuuint64_t strides[2] = {(cuuint64_t)(ld * 2), (cuuint64_t)(kBK * 2)};
  cuuint32_t box[3] = {(cuuint32_t)kBK, (cuuint32_t)box_rows, (cuuint32_t)kpb};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// drs_set_gemm_kb2: default k-blocks per TMA box (1, 2 or 4) for calls with kbox == 0
inline int& gemm_kb2_mode() {
  static int kpb = 1;
  return kpb;
}
// GEGLU's GELU in the tanh form (default; DRS_GEGLU_TANH=0: the erf form).  |tanh-form - erf-form|
// <= 4.7e-4 absolute (at x = 2.7), relative <= 2.2e-3 where |GELU| > 0.1 -- at the bf16 rounding of the
// GEGLU output; SD1.5 eval -1.3 %, SDXL -1.4 % (same box)
static int geglu_tanh_mode() {
  static const int on = [] { const char* e = getenv("DRS_GEGLU_TANH"); return e ? atoi(e) : 1; }();
  return on;
}
// DRS_CONV_A2=0 disables the 5-D conv A boxes (A/B switch)
static bool gemm_conv_a2() {
  static const int on = [] { const char* e = getenv("DRS_CONV_A2"); return e ? atoi(e) : 1; }();
  return on != 0;
}


// 5-D conv view (64 ch, W, H, N, C/64): a box {64, W, rows, imgs, 2} is the tiles of two
// consecutive channel blocks of one tap (KPB=2 slots with even C/64)
static bool make_tmap_conv5(CUtensorMap* m, const void* ptr, int N, int H, int W, int C, int s = 1) {
  PFN_encodeTiled enc = encode_fn();
  if (!enc) return false;
  const int rows = W >= 128 ? 1 : (128 / W <= H ? 128 / W : H);
  const int imgs = 128 / (W * rows);
  const int Hi = H * s, Wi = W * s;
  cuuint64_t dims[5] = {64, (cuuint64_t)Wi, (cuuint64_t)Hi, (cuuint64_t)N, (cuuint64_t)(C / 64)};
  cuuint64_t strides[4] = {(cuuint64_t)C * 2, (cuuint64_t)Wi * C * 2, (cuuint64_t)Hi * Wi * C * 2, 128};
  cuuint32_t box[5] = {64, (cuuint32_t)(W * s), (cuuint32_t)(rows * s), (cuuint32_t)imgs, 2};
  cuuint32_t estr[5] = {1, (cuuint32_t)s, (cuuint32_t)s, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(ptr), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static bool make_tmap_conv(CUtensorMap* m, const void* ptr, int N, int H, int W, int C, int s = 1) {
  PFN_encodeTiled enc = encode_fn();
  if (!enc) return false;
  const int rows = W >= 128 ? 1 : (128 / W <= H ? 128 / W : H);
  const int imgs = 128 / (W * rows);
  const int Hi = H * s, Wi = W * s;
  cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)Wi, (cuuint64_t)Hi, (cuuint64_t)N};
  cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)Wi * C * 2, (cuuint64_t)Hi * Wi * C * 2};
  cuuint32_t box[4] = {64, (cuuint32_t)(W * s), (cuuint32_t)(rows * s), (cuuint32_t)imgs};
  cuuint32_t estr[4] = {1, (cuuint32_t)s, (cuuint32_t)s, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Output map for the staged TMA store: {n_out cols, M rows}, box {cols_box, 32}
// with the swizzle whose span equals the staged row pitch (32 / 64 / 128 B).
static bool make_tmap_out(CUtensorMap* m, void* ptr, int64_t rows, int64_t cols, int64_t ld, int elem, int cols_box) {
  PFN_encodeTiled enc = encode_fn();
  if (!enc) return false;
  const int pitch = cols_box * elem;
  const CUtensorMapSwizzle sw = pitch == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : (pitch == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * elem)};
  cuuint32_t box[2] = {(cuuint32_t)cols_box, 32};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, elem == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, ptr, dims, strides,
             box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

template <int BN, int kStages, int kEpi, bool kSplit, int KPB = 1>
static bool ensure_smem_attr() {
  static int state = 0;        // 0 unknown, 1 ok, -1 failed
  if (!state) {
    using S = GemmSmem<BN, kStages>;
    state = cudaFuncSetAttribute(gemm_bf16_tc_kernel<BN, kStages, kEpi, kSplit, KPB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 S::kBytes) == cudaSuccess ? 1 : -1;
  }
  return state > 0;
}

// Clusters of `split` CTAs of this configuration that fit on the GPU at once
// (GPC packing makes this less than #SMs / split); cached per split.
template <int BN, int kStages, int kEpi = 1>
static int max_clusters(int split) {
  static int cache[9] = {0};
  if (split < 2 || split > 8) return num_sms();
  if (!cache[split]) {
    using S = GemmSmem<BN, kStages>;
    int n = 0;
    if (ensure_smem_attr<BN, kStages, kEpi, true>()) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(split * 64);
      cfg.blockDim = dim3(kGemmThreads);
      cfg.dynamicSmemBytes = S::kBytes;
      cudaLaunchAttribute la[1];
      la[0].id = cudaLaunchAttributeClusterDimension;
      la[0].val.clusterDim.x = split;
      la[0].val.clusterDim.y = 1;
      la[0].val.clusterDim.z = 1;
      cfg.attrs = la;
      cfg.numAttrs = 1;
      if (cudaOccupancyMaxActiveClusters(&n, gemm_bf16_tc_kernel<BN, kStages, kEpi, true, 1>, &cfg) != cudaSuccess) n = 0;
      cudaGetLastError();
    }
    cache[split] = n > 0 ? n : num_sms() / split;
  }
  return cache[split];
}

template <int BN, int kStages, int kEpi, int KPB>
static int launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, const OutMaps& tcm, int M, int N, int K,
                       int split, const EpiParams& ep, const ConvGeom& cv, cudaStream_t st) {
  using S = GemmSmem<BN, kStages>;
  static_assert(kBM * (BN + 4) * 4 <= kStages * S::kStageBytes, "split-K partial tile must fit the stage ring");
  const int tiles = ((M + kBM - 1) / kBM) * ((N + BN - 1) / BN) * split;
  if (split == 1 && ((ep.tma_store && (!ep.res || ep.tma_res)) || ep.act == DRS_ACT_HEADSOFTMAX)) {
    // persistent: staged TMA stores (and TMA-loaded residual tiles)
    auto kern = gemm_bf16_tc_kernel<BN, kStages, kEpi, false, KPB>;
    if (!ensure_smem_attr<BN, kStages, kEpi, false, KPB>()) return DRS_ERR_CUDA;
    const int grid = tiles < num_sms() ? tiles : num_sms();
    launch_pdl(kern, dim3(grid), dim3(kGemmThreads), S::kBytes, st, ta, tb, tcm, M, N, K, split, ep, cv);
    return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
  }
  // split-K (or an output the TMA store cannot address: split == 1, direct
  // stores): one CTA per (tile, split), the split CTAs of a tile as one cluster
  auto kern = gemm_bf16_tc_kernel<BN, kStages, kEpi, true, KPB>;
  if (!ensure_smem_attr<BN, kStages, kEpi, true, KPB>()) return DRS_ERR_CUDA;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(tiles);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = S::kBytes;
  cfg.stream = st;
  cudaLaunchAttribute la[2];
  la[0].id = cudaLaunchAttributeClusterDimension;
  la[0].val.clusterDim.x = split;
  la[0].val.clusterDim.y = 1;
  la[0].val.clusterDim.z = 1;
  la[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  la[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = la;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  cudaLaunchKernelEx(&cfg, kern, ta, tb, tcm, M, N, K, split, ep, cv);
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
}

template <int BN, int kStages, int kEpi, int KPB>
static int launch_pair(const CUtensorMap& ta, const CUtensorMap& tb, const OutMaps& tcm, int M, int N, int K,
                       const EpiParams& ep, const ConvGeom& cv, cudaStream_t st) {
  using S = PairSmem<BN, kStages>;
  auto kern = gemm_pair_kernel<BN, kStages, kEpi, KPB>;
  static int cap = 0;
  if (!cap) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, S::kBytes) != cudaSuccess)
      return DRS_ERR_CUDA;
    cudaLaunchConfig_t q = {};
    q.gridDim = dim3(128);
    q.blockDim = dim3(kGemmThreads);
    q.dynamicSmemBytes = S::kBytes;
    cudaLaunchAttribute qa[1];
    qa[0].id = cudaLaunchAttributeClusterDimension;
    qa[0].val.clusterDim.x = 2;
    qa[0].val.clusterDim.y = 1;
    qa[0].val.clusterDim.z = 1;
    q.attrs = qa;
    q.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &q) != cudaSuccess || n <= 0) n = num_sms() / 2;
    cudaGetLastError();
    cap = n;
  }
  const int tiles = ((M + 2 * kBM - 1) / (2 * kBM)) * ((N + BN - 1) / BN);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * (tiles < cap ? tiles : cap));
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = S::kBytes;
  cfg.stream = st;
  cudaLaunchAttribute la[2];
  la[0].id = cudaLaunchAttributeClusterDimension;
  la[0].val.clusterDim.x = 2;
  la[0].val.clusterDim.y = 1;
  la[0].val.clusterDim.z = 1;
  la[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  la[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = la;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  cudaLaunchKernelEx(&cfg, kern, ta, tb, tcm, M, N, K, ep, cv);
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
}


template <int BN, int kStages, int kEpi, int KPB>
static int launch_pair_split(const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K, int split,
                             const EpiParams& ep, const ConvGeom& cv, cudaStream_t st) {
  using S = PairSmem<BN, kStages>;
  static_assert(kBM * (BN + 4) * 4 <= kStages * S::kStageBytes, "pair split-K partial tile must fit the ring");
  auto kern = gemm_pair_split_kernel<BN, kStages, kEpi, KPB>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, S::kBytes) != cudaSuccess ||
        cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
      return DRS_ERR_CUDA;
    attr = true;
  }
  const int tiles = ((M + 2 * kBM - 1) / (2 * kBM)) * ((N + BN - 1) / BN);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(tiles * 2 * split);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = S::kBytes;
  cfg.stream = st;
  cudaLaunchAttribute la[2];
  la[0].id = cudaLaunchAttributeClusterDimension;
  la[0].val.clusterDim.x = 2 * split;
  la[0].val.clusterDim.y = 1;
  la[0].val.clusterDim.z = 1;
  la[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  la[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = la;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  cudaLaunchKernelEx(&cfg, kern, ta, tb, M, N, K, split, ep, cv);
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
}


template <int kEpi, int KPB>
static int gemm_dispatch_k(const CUtensorMap& ta, const CUtensorMap& tb, const OutMaps& tcm, int M, int N, int K, int bn,
                         int split, bool pair, EpiParams ep, const ConvGeom& cv, cudaStream_t st) {
  if (pair && split > 1) {
    ep.tma_store = 0;                              // reduced rows are stored directly
    if (bn == 64) return launch_pair_split<64, 8, kEpi, KPB>(ta, tb, M, N, K, split, ep, cv, st);
    if (bn == 128) return launch_pair_split<128, 8, kEpi, KPB>(ta, tb, M, N, K, split, ep, cv, st);
    if (bn == 160) return launch_pair_split<160, 7, kEpi, KPB>(ta, tb, M, N, K, split, ep, cv, st);
    if (bn == 192) return launch_pair_split<192, 6, kEpi, KPB>(ta, tb, M, N, K, split, ep, cv, st);
    return launch_pair_split<256, 6, kEpi, KPB>(ta, tb, M, N, K, split, ep, cv, st);
  }
  if (pair) {
    if (bn == 64) return launch_pair<64, 8, kEpi, KPB>(ta, tb, tcm, M, N, K, ep, cv, st);
    if (bn == 128) return launch_pair<128, 8, kEpi, KPB>(ta, tb, tcm, M, N, K, ep, cv, st);
    if (bn == 160) return launch_pair<160, 7, kEpi, KPB>(ta, tb, tcm, M, N, K, ep, cv, st);
    if (bn == 192) return launch_pair<192, 6, kEpi, KPB>(ta, tb, tcm, M, N, K, ep, cv, st);
    return launch_pair<256, 6, kEpi, KPB>(ta, tb, tcm, M, N, K, ep, cv, st);
  }
  if (bn == 64) return launch_gemm<64, 8, kEpi, KPB>(ta, tb, tcm, M, N, K, split, ep, cv, st);
  if (bn == 128) return launch_gemm<128, 6, kEpi, KPB>(ta, tb, tcm, M, N, K, split, ep, cv, st);
  if (bn == 160) return launch_gemm<160, 5, kEpi, KPB>(ta, tb, tcm, M, N, K, split, ep, cv, st);
  if (bn == 192) return launch_gemm<192, 4, kEpi, KPB>(ta, tb, tcm, M, N, K, split, ep, cv, st);
  return launch_gemm<256, 4, kEpi, KPB>(ta, tb, tcm, M, N, K, split, ep, cv, st);
}

// KPB (k-blocks per TMA box) selects separate kernel instantiations: a runtime
// switch inside one kernel grew its code and cost 2-3 % per network eval even
// where only the 1-k-block path ran (tools/net_bench.py A/B)
template <int kEpi>
static int gemm_dispatch(const CUtensorMap& ta, const CUtensorMap& tb, const OutMaps& tcm, int M, int N, int K, int bn,
                         int split, bool pair, EpiParams ep, const ConvGeom& cv, cudaStream_t st) {
  if (ep.kpb == 2) return gemm_dispatch_k<kEpi, 2>(ta, tb, tcm, M, N, K, bn, split, pair, ep, cv, st);
  return gemm_dispatch_k<kEpi, 1>(ta, tb, tcm, M, N, K, bn, split, pair, ep, cv, st);
}

static int max_clusters_bn(int bn, int split) {
  switch (bn) {
    case 64: return max_clusters<64, 8>(split);
    case 128: return max_clusters<128, 6>(split);
    case 160: return max_clusters<160, 5>(split);
    case 192: return max_clusters<192, 4>(split);
    default: return max_clusters<256, 4>(split);
  }
}

// Modelled time (us) of one launch, calibrated on B200 with tools/gemm_sweep.py:
//  * operand streaming: a CTA pulls its k-blocks at <= ~130 GB/s (L2 -> SM) and
//    all CTAs together at <= ~11 TB/s (aggregate L2 -> SM); MMA at ~15.5
//    TFLOP/s per SM; the slowest of the three bounds;
//  * ~5 us fixed latency per launch (prologue, first loads, epilogue drain);
//  * cluster split-K only when every cluster is co-resident (one wave: the
//    split grid is not persistent) and costs ~1 us + 0.012 us * bn * (split-1)
//    for the DSMEM partial-tile exchange.
static double gemm_cost_us(int M, int N, int K, int bn, int split) {
  const int tiles = ((M + kBM - 1) / kBM) * ((N + bn - 1) / bn);
  const int kb = (K + kBK - 1) / kBK;
  if (split > 1 && tiles > max_clusters_bn(bn, split)) return 1e30;
  const int waves = split > 1 ? 1 : (tiles + num_sms() - 1) / num_sms();
  const double kb_cta = (double)waves * ((kb + split - 1) / split);
  const double kb_bytes = (double)(kBM + bn) * kBK * 2;
  const double per_cta = kb_cta * kb_bytes / 130e3;
  const double aggregate = (double)tiles * kb * kb_bytes / 11e6;
  const double mma = kb_cta * 2.0 * kBM * bn * kBK / 15.5e6;
  double t = per_cta > aggregate ? per_cta : aggregate;
  if (mma > t) t = mma;
  return 5.0 + t + (split > 1 ? 1.0 + 0.012 * bn * (split - 1) : 0.0);
}

// bn == 0: choose the tile width; split == 0: choose the split (<= 6).
static void gemm_auto_config(int M, int N, int K, int& bn, int& split) {
  static const int kBns[5] = {64, 128, 160, 192, 256};
  static const int kSplits[5] = {1, 2, 3, 4, 6};
  const int kb = (K + kBK - 1) / kBK;
  double best = 1e30;
  int bb = bn ? bn : 128, bs = split ? split : 1;
  for (int i = 0; i < 5; ++i) {
    if (bn && kBns[i] != bn) continue;
    for (int j = 0; j < 5; ++j) {
      if (split && kSplits[j] != split) continue;
      if (kSplits[j] > 1 && kb / kSplits[j] < 8) continue;      // keep >= 8 k-blocks per split
      const double t = gemm_cost_us(M, N, K, kBns[i], kSplits[j]);
      if (t >= 1e29) continue;
      if (t < best * 0.97) { best = t; bb = kBns[i]; bs = kSplits[j]; }   // ties -> smaller tile / split
    }
  }
  bn = bb;
  split = bs;
}

}  // namespace drs

extern "C" int drs_gemm_cost_us(int M, int N, int K, int bn, int split) {
  if (M <= 0 || N <= 0 || K <= 0 || split < 1 || split > 8) return -1;
  const double t = drs::gemm_cost_us(M, N, K, bn, split);
  return t >= 1e29 ? -1 : (int)(t * 1000.0);   // ns; -1 = configuration not allowed
}

extern "C" int drs_gemm_pick(int M, int N, int K, int* bn, int* split) {
  if (!bn || !split || M <= 0 || N <= 0 || K <= 0) return DRS_ERR_VALUE;
  int b = *bn, s = *split;
  drs::gemm_auto_config(M, N, K, b, s);
  *bn = b;
  *split = s;
  return DRS_OK;
}

extern "C" int drs_gemm(const drs_gemm_args* g, void* stream) {
  using namespace drs;
  if (!g) return DRS_ERR_VALUE;
  const int M = g->M, N = g->N, K = g->K;
  if (M <= 0 || N <= 0 || K <= 0) return (M == 0 || N == 0) ? DRS_OK : DRS_ERR_VALUE;
  if (!g->A || !g->B || !g->C) return DRS_ERR_VALUE;
  if ((K % 8) || (!g->conv_C && (g->lda % 8)) || (g->ldb % 8)) return DRS_ERR_VALUE;   // TMA: 16-byte strides
  if ((reinterpret_cast<uintptr_t>(g->A) & 15) || (reinterpret_cast<uintptr_t>(g->B) & 15)) return DRS_ERR_VALUE;
  if (g->act == DRS_ACT_GEGLU && (N % 2)) return DRS_ERR_VALUE;
  if (g->rowbias && g->rb_group <= 0) return DRS_ERR_VALUE;
  int bn = g->bn, split = g->split;
  if (bn != 0 && bn != 64 && bn != 128 && bn != 160 && bn != 192 && bn != 256) return DRS_ERR_VALUE;
  if (split < 0 || split > 8) return DRS_ERR_VALUE;            // portable cluster size
  if (bn == 0 || split == 0) gemm_auto_config(M, N, K, bn, split);
  CUtensorMap ta, tb;
  ConvGeom cv{0, 0, 0, 0, 0, 0, 1, 0};
  const bool hsm = g->act == DRS_ACT_HEADSOFTMAX;
  if (hsm) {
    if (g->out_f32 || N % 96 || g->hs_valid <= 0 || g->hs_valid > 96 || (g->ldc % 8) ||
        (reinterpret_cast<uintptr_t>(g->C) & 15) || g->residual || g->bias || g->colscale || g->rowbias)
      return DRS_ERR_VALUE;
    bn = 192;
    split = 1;
  }
  if (g->b_img_rows > 0 && (g->b_img_rows % kBM || g->b_img_off <= 0)) return DRS_ERR_VALUE;
  if (g->conv_C > 0) {      // implicit 3x3 conv: A = NHWC input, M = N*H*W, K = 9*C
    const int C = g->conv_C, H = g->conv_H, W = g->conv_W, Nimg = g->conv_N;
    const int cs = g->conv_stride > 1 ? g->conv_stride : 1;
    if (cs > 2 || (cs == 2 && W * 2 > 256)) return DRS_ERR_VALUE;
    if (C % 64 || W > 128 || (W & (W - 1)) || (int64_t)Nimg * H * W != M || K != 9 * C) return DRS_ERR_VALUE;
    const int rows = W >= 128 ? 1 : (128 / W <= H ? 128 / W : H);
    if (W * rows * (128 / (W * rows)) != 128 || H % rows || (128 / (W * rows) > 1 && (rows != H || Nimg % (128 / (W * H)))))
      return DRS_ERR_VALUE;
    if (!make_tmap_conv(&ta, g->A, Nimg, H, W, C, cs)) return DRS_ERR_CUDA;
    cv = ConvGeom{1, C / 64, H, W, 0, 0, cs, 0};
  }
  // kb2 (K % 64 == 0): one TMA box carries 2 k-blocks -- half the
  // TMA operations, whose per-op issue cost (~190 clk from one thread) bounds the
  // operand stream of small tiles (tools/micro/tma_kb2.cu)
  int kpb = g->kbox == 0 ? gemm_kb2_mode() : g->kbox;
  if (kpb == 4) kpb = 2;                           // (4 k-blocks per box: measured no gain, not instantiated)
  if (kpb != 1 && kpb != 2) return DRS_ERR_VALUE;
  if (K % kBK || hsm) kpb = 1;
  if (!g->conv_C) {
    if (!make_tmap(&ta, g->A, M, K, g->lda, kBM)) return DRS_ERR_CUDA;
  }
  if (g->b_img_rows > 0) {
    cv.b_img_rows = g->b_img_rows;
    cv.b_img_off = g->b_img_off;
  }
  EpiParams ep{g->C, g->ldc, g->bias, g->residual, g->ldr, g->res_f32, g->colscale, g->cs_group, g->cs_ld,
               g->rowbias, g->rb_group, g->rb_ld, g->alpha, g->act, g->out_f32, 0, g->hs_valid, 0, g->out2, g->ldo2,
               early_weights_enabled(), geglu_tanh_mode(), 1};
  // staged TMA store whenever the output layout allows it (16-byte aligned rows)
  OutMaps tcm;
  memset(&tcm, 0, sizeof(tcm));
  {
    const int elem = g->out_f32 ? 4 : 2;
    const int n_out = g->act == DRS_ACT_GEGLU ? N / 2 : N;
    const bool ok = split == 1 && !hsm && !(reinterpret_cast<uintptr_t>(g->C) & 15) && ((g->ldc * elem) % 16) == 0 &&
                    g->ldc >= n_out;
    if (ok && make_tmap_out(&tcm.c, g->C, M, n_out, g->ldc, elem, g->act == DRS_ACT_GEGLU ? 16 : 32)) ep.tma_store = 1;
    // residual of the output's dtype: TMA-loaded into the staging buffer (DRS_TMA_RES=0 disables)
    static const int tma_res_on = [] { const char* e = getenv("DRS_TMA_RES"); return e ? atoi(e) : 1; }();
    if (tma_res_on && ep.tma_store && g->residual && g->act != DRS_ACT_GEGLU && (g->res_f32 != 0) == (g->out_f32 != 0) &&
        !(reinterpret_cast<uintptr_t>(g->residual) & 15) && ((g->ldr * elem) % 16) == 0 &&
        make_tmap_out(&tcm.r, const_cast<void*>(g->residual), M, n_out, g->ldr, elem, 32))
      ep.tma_res = 1;
  }
  // 2-SM pair mode: M >= 256 (split > 1: pair + cluster split-K, 2 * split <= 16 CTAs); a
  // split == 1 pair runs the persistent TMA epilogue only (decided here: the B map's box depends on it)
  const bool pair = g->cta_pair > 0 && M >= 2 * kBM && !hsm && !(g->b_img_rows > 0 && g->b_img_rows % (2 * kBM)) &&
                    (split > 1 || (ep.tma_store && (!ep.res || ep.tma_res)));
  const int64_t b_rows = N + (g->b_img_rows > 0 ? g->b_img_off : 0);
  ep.kpb = kpb;
  // conv with even C/64 and slots that start at even k-blocks: one 5-D A box per slot
  if (kpb == 2 && g->conv_C > 0 && (cv.cblocks % 2) == 0 && gemm_conv_a2()) {
    const int nkb = K / kBK;
    const int kbs = (nkb + split - 1) / split;
    if ((split == 1 || kbs % 2 == 0)) {
      if (!make_tmap_conv5(&ta, g->A, g->conv_N, g->conv_H, g->conv_W, g->conv_C, cv.stride)) return DRS_ERR_CUDA;
      cv.a2 = 1;
    }
  }
  if (kpb > 1) {
    if (!g->conv_C && !make_tmap_kb2(&ta, g->A, M, K, g->lda, kBM, kpb)) return DRS_ERR_CUDA;
    if (!make_tmap_kb2(&tb, g->B, b_rows, K, g->ldb, pair ? bn / 2 : bn, kpb)) return DRS_ERR_CUDA;
  } else if (!make_tmap(&tb, g->B, b_rows, K, g->ldb, pair ? bn / 2 : bn)) {
    return DRS_ERR_CUDA;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (g->out2) {                                   // plain epilogue + bf16 copy of the fp32 output
    if (g->act != DRS_ACT_NONE || g->rowbias || g->colscale || !g->out_f32 || (g->ldo2 % 8) ||
        (reinterpret_cast<uintptr_t>(g->out2) & 15))
      return DRS_ERR_VALUE;
    return gemm_dispatch<4>(ta, tb, tcm, M, N, K, bn, split, pair, ep, cv, st);
  }
  if (g->act == DRS_ACT_NONE && !g->rowbias && !g->colscale)
    return gemm_dispatch<1>(ta, tb, tcm, M, N, K, bn, split, pair, ep, cv, st);
  if (g->act == DRS_ACT_NONE || g->act == DRS_ACT_SILU)
    return gemm_dispatch<3>(ta, tb, tcm, M, N, K, bn, split, pair, ep, cv, st);
  if (g->act == DRS_ACT_GEGLU) return gemm_dispatch<2>(ta, tb, tcm, M, N, K, bn, split, pair, ep, cv, st);
  return gemm_dispatch<0>(ta, tb, tcm, M, N, K, bn, split, pair, ep, cv, st);
}

extern "C" int drs_gemm_bf16(const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                             int M, int N, int K, const float* bias, const void* residual, int64_t ldr,
                             int act, int out_f32, float alpha, int bn, int split, float* workspace,
                             void* stream) {
  drs_gemm_args g = {};
  g.A = A; g.lda = lda; g.B = B; g.ldb = ldb; g.C = C; g.ldc = ldc; g.M = M; g.N = N; g.K = K;
  g.bias = bias; g.residual = residual; g.ldr = ldr; g.act = act; g.out_f32 = out_f32; g.alpha = alpha;
  g.bn = bn; g.split = split; g.workspace = workspace;
  return drs_gemm(&g, stream);
}

extern "C" int drs_set_gemm_kb2(int on) {
  drs::gemm_kb2_mode() = on ? 2 : 1;
  return DRS_OK;
}
