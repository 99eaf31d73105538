// Denoiser-network ops around the tensor-core GEMM (gemm_tc.cu):
//   * LayerNorm (+ affine or adaLN modulate) -> bf16       one warp per row
//   * fused attention softmax(Q K^T * scale) V              FA2-style, mma.sync
//     m16n8k16 bf16 -> fp32, 64 queries per CTA, online softmax in registers
//   * DiT helpers: sinusoidal timestep embedding, patchify / unpatchify,
//     SiLU->bf16 cast.
#include <cuda_runtime.h>
#include <stdlib.h>
#include <cuda_bf16.h>
#include <math.h>
#include <stdint.h>
#include <cuda.h>
#include "drs_net.h"
#include "pdl.cuh"
#include "tc_common.cuh"

namespace drs {

// x * sigmoid(x) with the fast reciprocal (an IEEE division costs ~10x more;
// __fdividef(1, inf) = 0 gives the right limit for very negative x)
// SiLU with one SFU op: x * sigmoid(x) = 0.5 x (1 + tanh(x / 2))  (tanh.approx: rel. err ~2^-11)
__device__ __forceinline__ float silu_fast(float x) {
  const float h = 0.5f * x;
  float th;
  asm("tanh.approx.f32 %0, %1;" : "=f"(th) : "f"(h));
  return fmaf(h, th, h);
}

// ------------------------------------------------------------ LayerNorm ---
// One warp per row, float4-vectorised; x and the modulation vectors are all
// loaded before any arithmetic so the warp pays one memory round trip.
template <int kV4>   // float4 chunks per lane (C <= 128 * kV4)
__global__ void layernorm_kernel(const void* __restrict__ x, int64_t ldx, int x_f32, int M, int C,
                                 const float* __restrict__ gamma, const float* __restrict__ beta,
                                 const float* __restrict__ shift, const float* __restrict__ scale, int mod_group,
                                 int64_t mod_ld, float eps, __nv_bfloat16* __restrict__ out, int64_t ldo) {
  const int warps = blockDim.x >> 5;
  const int row = blockIdx.x * warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const int C4 = C >> 2;
  // gamma / beta are weights (never written on-stream): loaded before the PDL wait
  float4 gv[kV4], bv[kV4];
#pragma unroll
  for (int i = 0; i < kV4; ++i) {
    const int c4 = lane + 32 * i;
    const bool in = c4 < C4;
    gv[i] = gamma && in ? __ldg(reinterpret_cast<const float4*>(gamma) + c4) : make_float4(1.f, 1.f, 1.f, 1.f);
    bv[i] = beta && in ? __ldg(reinterpret_cast<const float4*>(beta) + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  pdl_wait();
  pdl_trigger();
  if (row >= M) return;
  const int64_t mofs = mod_group > 0 ? (int64_t)(row / mod_group) * mod_ld : 0;
  float4 v[kV4], sc[kV4], sh[kV4];
#pragma unroll
  for (int i = 0; i < kV4; ++i) {
    const int c4 = lane + 32 * i;
    v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    sc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    sh[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (c4 < C4) {
      if (x_f32) {
        v[i] = reinterpret_cast<const float4*>(static_cast<const float*>(x) + (int64_t)row * ldx)[c4];
      } else {
        const uint2 u = reinterpret_cast<const uint2*>(static_cast<const __nv_bfloat16*>(x) + (int64_t)row * ldx)[c4];
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
        const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
        v[i] = make_float4(a.x, a.y, b.x, b.y);
      }
      if (scale) sc[i] = reinterpret_cast<const float4*>(scale + mofs)[c4];
      if (shift) sh[i] = reinterpret_cast<const float4*>(shift + mofs)[c4];
    }
  }
  float sum = 0.f;
#pragma unroll
  for (int i = 0; i < kV4; ++i) sum += (v[i].x + v[i].y) + (v[i].z + v[i].w);
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const float mean = sum / C;
  float sq = 0.f;
#pragma unroll
  for (int i = 0; i < kV4; ++i) {
    if (lane + 32 * i < C4) {
      const float a = v[i].x - mean, b = v[i].y - mean, c = v[i].z - mean, d = v[i].w - mean;
      sq += (a * a + b * b) + (c * c + d * d);
    }
  }
  for (int o = 16; o; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
  const float rstd = rsqrtf(sq / C + eps);
#pragma unroll
  for (int i = 0; i < kV4; ++i) {
    const int c4 = lane + 32 * i;
    if (c4 < C4) {
      float y[4] = {(v[i].x - mean) * rstd, (v[i].y - mean) * rstd, (v[i].z - mean) * rstd, (v[i].w - mean) * rstd};
      const float s4[4] = {sc[i].x, sc[i].y, sc[i].z, sc[i].w};
      const float h4[4] = {sh[i].x, sh[i].y, sh[i].z, sh[i].w};
      const float g4[4] = {gv[i].x, gv[i].y, gv[i].z, gv[i].w};
      const float b4[4] = {bv[i].x, bv[i].y, bv[i].z, bv[i].w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (gamma) y[e] = y[e] * g4[e] + b4[e];
        if (scale) y[e] = y[e] * (1.f + s4[e]);
        if (shift) y[e] = y[e] + h4[e];
      }
      uint2 u;
      *reinterpret_cast<__nv_bfloat162*>(&u.x) = __floats2bfloat162_rn(y[0], y[1]);
      *reinterpret_cast<__nv_bfloat162*>(&u.y) = __floats2bfloat162_rn(y[2], y[3]);
      reinterpret_cast<uint2*>(out + (int64_t)row * ldo)[c4] = u;
    }
  }
}

// Row-per-CTA LayerNorm: thread = one float4 of the row (C/4 threads), every
// operand (x, gamma, beta, adaLN scale / shift) loaded before any arithmetic,
// two-pass mean / variance with fixed-order block reductions (deterministic).
// Many small CTAs instead of one warp per row: small-M rows (the 16x16 / 8x8
// levels, DiT) no longer leave most SMs idle.
__device__ __forceinline__ float block_sum_fixed(float v, float* red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
  for (int i = 0; i < nw; ++i) t += red[i];
  __syncthreads();
  return t;
}

__global__ void __launch_bounds__(512)
layernorm_row_kernel(const void* __restrict__ x, int64_t ldx, int x_f32, int C, const float* __restrict__ gamma,
                     const float* __restrict__ beta, const float* __restrict__ shift, const float* __restrict__ scale,
                     int mod_group, int64_t mod_ld, float eps, __nv_bfloat16* __restrict__ out, int64_t ldo) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[32];
  const int row = blockIdx.x, c4 = threadIdx.x;
  const bool ok = c4 < (C >> 2);
  const int64_t mofs = mod_group > 0 ? (int64_t)(row / mod_group) * mod_ld : 0;
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f), g = make_float4(1.f, 1.f, 1.f, 1.f), b = make_float4(0.f, 0.f, 0.f, 0.f);
  float4 sc = make_float4(0.f, 0.f, 0.f, 0.f), sh = make_float4(0.f, 0.f, 0.f, 0.f);
  if (ok) {
    if (x_f32) {
      v = reinterpret_cast<const float4*>(static_cast<const float*>(x) + (int64_t)row * ldx)[c4];
    } else {
      const uint2 u = reinterpret_cast<const uint2*>(static_cast<const __nv_bfloat16*>(x) + (int64_t)row * ldx)[c4];
      const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
      const float2 bb = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
      v = make_float4(a.x, a.y, bb.x, bb.y);
    }
    if (gamma) g = __ldg(reinterpret_cast<const float4*>(gamma) + c4);
    if (beta) b = __ldg(reinterpret_cast<const float4*>(beta) + c4);
    if (scale) sc = __ldg(reinterpret_cast<const float4*>(scale + mofs) + c4);
    if (shift) sh = __ldg(reinterpret_cast<const float4*>(shift + mofs) + c4);
  }
  const float mean = block_sum_fixed((v.x + v.y) + (v.z + v.w), red) / C;
  const float a0 = v.x - mean, a1 = v.y - mean, a2 = v.z - mean, a3 = v.w - mean;
  const float var = block_sum_fixed(ok ? (a0 * a0 + a1 * a1) + (a2 * a2 + a3 * a3) : 0.f, red) / C;
  const float rstd = rsqrtf(var + eps);
  if (!ok) return;
  float y0 = a0 * rstd * g.x + b.x, y1 = a1 * rstd * g.y + b.y, y2 = a2 * rstd * g.z + b.z, y3 = a3 * rstd * g.w + b.w;
  if (scale) { y0 *= 1.f + sc.x; y1 *= 1.f + sc.y; y2 *= 1.f + sc.z; y3 *= 1.f + sc.w; }
  if (shift) { y0 += sh.x; y1 += sh.y; y2 += sh.z; y3 += sh.w; }
  uint2 u;
  *reinterpret_cast<__nv_bfloat162*>(&u.x) = __floats2bfloat162_rn(y0, y1);
  *reinterpret_cast<__nv_bfloat162*>(&u.y) = __floats2bfloat162_rn(y2, y3);
  reinterpret_cast<uint2*>(out + (int64_t)row * ldo)[c4] = u;
}

// ------------------------------------------------------------ attention ---
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2(uint32_t addr, uint32_t& r0, uint32_t& r1) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2_t(uint32_t addr, uint32_t& r0, uint32_t& r1) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

constexpr int kAttnBQ = 64, kAttnThreads = 128;

template <int DP, int BK = (DP > 96 ? 32 : 64)>   // DP: head dim padded to a multiple of 16; BK: keys per tile
__global__ void __launch_bounds__(kAttnThreads)
attention_kernel(const __nv_bfloat16* __restrict__ q, int64_t ldq, const __nv_bfloat16* __restrict__ k,
                 int64_t ldk, const __nv_bfloat16* __restrict__ v, int64_t ldv, __nv_bfloat16* __restrict__ o,
                 int64_t ldo, int Lq, int Lk, int d, float scale_log2) {
  pdl_wait();
  pdl_trigger();
  constexpr int LD = DP + 8;            // smem row stride (elements): 16 B aligned, staggers banks
  __shared__ __align__(16) __nv_bfloat16 sQ[kAttnBQ * LD];
  __shared__ __align__(16) __nv_bfloat16 sK[BK * LD];
  __shared__ __align__(16) __nv_bfloat16 sV[BK * LD];
  const int h = blockIdx.y, b = blockIdx.z;
  const int q0 = blockIdx.x * kAttnBQ;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const __nv_bfloat16* qb = q + ((int64_t)b * Lq) * ldq + (int64_t)h * d;
  const __nv_bfloat16* kbp = k + ((int64_t)b * Lk) * ldk + (int64_t)h * d;
  const __nv_bfloat16* vbp = v + ((int64_t)b * Lk) * ldv + (int64_t)h * d;
  constexpr int CH = DP / 8;            // 16-byte chunks per padded row
  const int dch = d / 8;

  for (int i = tid; i < kAttnBQ * CH; i += kAttnThreads) {
    const int r = i / CH, c = i % CH;
    uint4 val = make_uint4(0, 0, 0, 0);
    if (q0 + r < Lq && c < dch) val = *reinterpret_cast<const uint4*>(qb + (int64_t)(q0 + r) * ldq + c * 8);
    *reinterpret_cast<uint4*>(&sQ[r * LD + c * 8]) = val;
  }
  __syncthreads();
  uint32_t qa[DP / 16][4];
  {
    const int r = warp * 16 + (lane & 15), c = (lane >> 4) * 8;
#pragma unroll
    for (int ks = 0; ks < DP / 16; ++ks)
      ldsm_x4(static_cast<uint32_t>(__cvta_generic_to_shared(&sQ[r * LD + ks * 16 + c])), qa[ks][0], qa[ks][1],
              qa[ks][2], qa[ks][3]);
  }
  float oacc[DP / 8][4];
#pragma unroll
  for (int i = 0; i < DP / 8; ++i) oacc[i][0] = oacc[i][1] = oacc[i][2] = oacc[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;   // rows g and g+8

  for (int k0 = 0; k0 < Lk; k0 += BK) {
    __syncthreads();
    for (int i = tid; i < BK * CH; i += kAttnThreads) {
      const int r = i / CH, c = i % CH;
      uint4 kv = make_uint4(0, 0, 0, 0), vv = make_uint4(0, 0, 0, 0);
      if (k0 + r < Lk && c < dch) {
        kv = *reinterpret_cast<const uint4*>(kbp + (int64_t)(k0 + r) * ldk + c * 8);
        vv = *reinterpret_cast<const uint4*>(vbp + (int64_t)(k0 + r) * ldv + c * 8);
      }
      *reinterpret_cast<uint4*>(&sK[r * LD + c * 8]) = kv;
      *reinterpret_cast<uint4*>(&sV[r * LD + c * 8]) = vv;
    }
    __syncthreads();
    float s[BK / 8][4];
#pragma unroll
    for (int nb = 0; nb < BK / 8; ++nb) {
      s[nb][0] = s[nb][1] = s[nb][2] = s[nb][3] = 0.f;
      const int r = nb * 8 + (lane & 7), cofs = ((lane >> 3) & 1) * 8;
#pragma unroll
      for (int ks = 0; ks < DP / 16; ++ks) {
        uint32_t b0, b1;
        ldsm_x2(static_cast<uint32_t>(__cvta_generic_to_shared(&sK[r * LD + ks * 16 + cofs])), b0, b1);
        mma16816(s[nb], qa[ks], b0, b1);
      }
    }
    // scale, mask, online softmax (rows g / g+8 spread over the 4 threads of a quad)
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int nb = 0; nb < BK / 8; ++nb) {
      const int kc = k0 + nb * 8 + 2 * t;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const bool valid = (kc + (e & 1)) < Lk;
        s[nb][e] = valid ? s[nb][e] * scale_log2 : -INFINITY;
      }
      mx0 = fmaxf(mx0, fmaxf(s[nb][0], s[nb][1]));
      mx1 = fmaxf(mx1, fmaxf(s[nb][2], s[nb][3]));
    }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    const float nm0 = fmaxf(m0, mx0), nm1 = fmaxf(m1, mx1);
    const float a0 = exp2f(m0 - nm0), a1 = exp2f(m1 - nm1);
    m0 = nm0;
    m1 = nm1;
    float rs0 = 0.f, rs1 = 0.f;
    uint32_t pa[BK / 16][4];
#pragma unroll
    for (int nb = 0; nb < BK / 8; ++nb) {
      const float p0 = exp2f(s[nb][0] - nm0), p1 = exp2f(s[nb][1] - nm0);
      const float p2 = exp2f(s[nb][2] - nm1), p3 = exp2f(s[nb][3] - nm1);
      rs0 += p0 + p1;
      rs1 += p2 + p3;
      const int kk = nb >> 1, half = nb & 1;
      pa[kk][half * 2 + 0] = pack_bf16(p0, p1);
      pa[kk][half * 2 + 1] = pack_bf16(p2, p3);
    }
    l0 = l0 * a0 + rs0;
    l1 = l1 * a1 + rs1;
#pragma unroll
    for (int db = 0; db < DP / 8; ++db) {
      oacc[db][0] *= a0; oacc[db][1] *= a0;
      oacc[db][2] *= a1; oacc[db][3] *= a1;
    }
#pragma unroll
    for (int kk = 0; kk < BK / 16; ++kk) {
      const int r = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
#pragma unroll
      for (int db = 0; db < DP / 8; ++db) {
        uint32_t b0, b1;
        ldsm_x2_t(static_cast<uint32_t>(__cvta_generic_to_shared(&sV[r * LD + db * 8])), b0, b1);
        mma16816(oacc[db], pa[kk], b0, b1);
      }
    }
  }
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const float i0 = l0 > 0.f ? 1.f / l0 : 0.f, i1 = l1 > 0.f ? 1.f / l1 : 0.f;
  const int r0 = q0 + warp * 16 + g, r1 = r0 + 8;
  __nv_bfloat16* ob = o + ((int64_t)b * Lq) * ldo + (int64_t)h * d;
#pragma unroll
  for (int db = 0; db < DP / 8; ++db) {
    const int c = db * 8 + 2 * t;
    if (c < d) {
      if (r0 < Lq)
        *reinterpret_cast<__nv_bfloat162*>(ob + (int64_t)r0 * ldo + c) =
            __floats2bfloat162_rn(oacc[db][0] * i0, oacc[db][1] * i0);
      if (r1 < Lq)
        *reinterpret_cast<__nv_bfloat162*>(ob + (int64_t)r1 * ldo + c) =
            __floats2bfloat162_rn(oacc[db][2] * i1, oacc[db][3] * i1);
    }
  }
}

// ---------------------------------------------------------- DiT helpers ---
// emb[i] = [cos(t f_j), sin(t f_j)], f_j = exp(-ln(max_period) j / half)  (DiT TimestepEmbedder)
__global__ void timestep_embedding_kernel(const float* __restrict__ t, int n, int dim, float max_period,
                                          __nv_bfloat16* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int half = dim / 2;
  if (i >= n * half) return;
  const int r = i / half, j = i % half;
  const float f = expf(-logf(max_period) * j / half);
  const float a = t[r] * f;
  out[(int64_t)r * dim + j] = __float2bfloat16(cosf(a));
  out[(int64_t)r * dim + half + j] = __float2bfloat16(sinf(a));
}

// latent x (C, H, W) fp64/fp32 -> tokens (H/p * W/p, C*p*p) bf16, feature order (c, py, px)
__global__ void patchify_kernel(const void* __restrict__ x, int x_f64, int C, int H, int W, int p,
                                __nv_bfloat16* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int gw = W / p, feat = C * p * p;
  if (i >= (H / p) * gw * feat) return;
  const int tok = i / feat, f = i % feat;
  const int c = f / (p * p), py = (f / p) % p, px = f % p;
  const int hh = (tok / gw) * p + py, ww = (tok % gw) * p + px;
  const int64_t src = ((int64_t)c * H + hh) * W + ww;
  const float val = x_f64 ? (float)static_cast<const double*>(x)[src] : static_cast<const float*>(x)[src];
  out[i] = __float2bfloat16(val);
}

// tokens (H/p * W/p, p*p*Cout) fp32, feature order (py, px, c) -> eps (Ckeep, H, W) fp32
__global__ void unpatchify_kernel(const float* __restrict__ tok, int Cout, int Ckeep, int H, int W, int p,
                                  float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= Ckeep * H * W) return;
  const int c = i / (H * W), hh = (i / W) % H, ww = i % W;
  const int gw = W / p;
  const int t = (hh / p) * gw + (ww / p);
  const int f = ((hh % p) * p + (ww % p)) * Cout + c;
  out[i] = tok[(int64_t)t * (p * p * Cout) + f];
}

__global__ void cast_f32_bf16_kernel(const float* __restrict__ x, int64_t n, __nv_bfloat16* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i + 3 < n) {
    const float4 v = *reinterpret_cast<const float4*>(x + i);
    uint2 u;
    *reinterpret_cast<__nv_bfloat162*>(&u.x) = __floats2bfloat162_rn(v.x, v.y);
    *reinterpret_cast<__nv_bfloat162*>(&u.y) = __floats2bfloat162_rn(v.z, v.w);
    *reinterpret_cast<uint2*>(out + i) = u;
  } else {
    for (int64_t j = i; j < n; ++j) out[j] = __float2bfloat16(x[j]);
  }
}

__global__ void silu_cast_kernel(const float* __restrict__ x, int64_t n, __nv_bfloat16* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) { const float a = x[i]; out[i] = __float2bfloat16(a / (1.f + __expf(-a))); }
}

// ------------------------------------------------------------- UNet ops ----
// im2col over NHWC bf16 for 1x1 / 3x3 convs: row (n, oy, ox), column
// (ky, kx, c) with c over the channel concat [x1 | x2] (UNet skip connections);
// `up` = 2 reads a nearest-upsampled input (Upsample2D folded in); zero padding.
// One thread per 8-channel (16-byte) chunk.
__global__ void im2col_kernel(const __nv_bfloat16* __restrict__ x1, int C1, const __nv_bfloat16* __restrict__ x2,
                              int C2, int N, int H, int W, int ks, int stride, int pad, int up, int Ho, int Wo,
                              __nv_bfloat16* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  // 32-bit index math (host guarantees total < 2^31): one 16-byte chunk per thread
  const int C8 = (C1 + C2) >> 3;
  const int taps = ks * ks;
  const int total = N * Ho * Wo * taps * C8;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int c8 = i % C8;
  int r = i / C8;
  const int tap = r % taps;
  r /= taps;
  const int ox = r % Wo;
  r /= Wo;
  const int oy = r % Ho;
  const int n = r / Ho;
  const int ky = tap / ks, kx = tap - ky * ks;
  const int iy = oy * stride + ky - pad, ix = ox * stride + kx - pad;   // in upsampled coordinates
  uint4 v = make_uint4(0, 0, 0, 0);
  if (iy >= 0 && ix >= 0 && iy < H * up && ix < W * up) {
    const int sy = iy / up, sx = ix / up;
    const int pix = (n * H + sy) * W + sx;
    const int c = c8 * 8;
    v = c < C1 ? __ldg(reinterpret_cast<const uint4*>(x1 + (int64_t)pix * C1 + c))
               : __ldg(reinterpret_cast<const uint4*>(x2 + (int64_t)pix * C2 + (c - C1)));
  }
  reinterpret_cast<uint4*>(out)[i] = v;
}

// GroupNorm over NHWC (bf16 or fp32 in) with affine and optional SiLU -> bf16.
// Pass 1 (gn_stats): grid (N*G, kGnSplit); each CTA sums a fixed pixel slice of
// one (image, group) and writes (sum, sumsq) partials -- no atomics, so the
// result is bit-reproducible.  Pass 2 (gn_apply): each CTA reduces the
// partials of the groups it touches in a fixed order, then normalises a
// pixel range with 16-byte vector loads.
constexpr int kGnSplit = 16;

__global__ void gn_stats_kernel(const void* __restrict__ x, int x_f32, int HW, int C, int G,
                                float2* __restrict__ part) {
  pdl_wait();
  pdl_trigger();
  const int ng = blockIdx.x, sp = blockIdx.y;
  const int n = ng / G, g = ng % G, cg = C / G;
  const int p0 = (int)((int64_t)HW * sp / kGnSplit), p1 = (int)((int64_t)HW * (sp + 1) / kGnSplit);
  const int64_t base = (int64_t)n * HW * C + (int64_t)g * cg;
  // channel PAIRS (cg is even for every GroupNorm here): walk (pixel, pair)
  // incrementally -- no division in the loop, 4-byte loads
  const int cp = cg >> 1;
  const int step_p = blockDim.x / cp, step_c = blockDim.x % cp;
  int p = p0 + threadIdx.x / cp, c = threadIdx.x % cp;
  float s = 0.f, ss = 0.f;
  while (p < p1) {
    const int64_t off = base + (int64_t)p * C + 2 * c;
    float2 v;
    if (x_f32) v = *reinterpret_cast<const float2*>(static_cast<const float*>(x) + off);
    else v = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(static_cast<const __nv_bfloat16*>(x) + off));
    s += v.x + v.y;
    ss += v.x * v.x + v.y * v.y;
    c += step_c;
    p += step_p;
    if (c >= cp) { c -= cp; ++p; }
  }
  __shared__ float red[2][32];
  for (int o = 16; o; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { red[0][warp] = s; red[1][warp] = ss; }
  __syncthreads();
  if (threadIdx.x == 0) {
    float a = 0.f, b = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { a += red[0][w]; b += red[1][w]; }
    part[(int64_t)ng * kGnSplit + sp] = make_float2(a, b);
  }
}

constexpr int kGnPix = 16;     // pixels per apply CTA

// Each thread owns channel pairs (cp, cp + blockDim, ...) and walks the CTA's
// pixels: group lookups, gamma/beta and the group statistics are hoisted out
// of the pixel loop.
__global__ void gn_apply_kernel(const void* __restrict__ x, int x_f32, int HW, int C, int G,
                                const float2* __restrict__ part, const float* __restrict__ gamma,
                                const float* __restrict__ beta, float eps, int silu,
                                __nv_bfloat16* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ float sstat[];                  // [G][2] mean, rstd
  const int64_t pix0 = (int64_t)blockIdx.x * kGnPix;  // global pixel index (n*HW + p)
  const int n = (int)(pix0 / HW);
  const int cg = C / G;
  for (int g = threadIdx.x; g < G; g += blockDim.x) {
    float a = 0.f, b = 0.f;
    const float2* pp = part + ((int64_t)n * G + g) * kGnSplit;
    float2 f[kGnSplit];
#pragma unroll
    for (int s2 = 0; s2 < kGnSplit; ++s2) f[s2] = pp[s2];
#pragma unroll
    for (int s2 = 0; s2 < kGnSplit; ++s2) { a += f[s2].x; b += f[s2].y; }
    const float cnt = (float)HW * cg;
    const float mean = a / cnt;
    const float var = fmaxf(b / cnt - mean * mean, 0.f);
    sstat[2 * g] = mean;
    sstat[2 * g + 1] = rsqrtf(var + eps);
  }
  __syncthreads();
  const int C2 = C / 2;
  for (int cp = threadIdx.x; cp < C2; cp += blockDim.x) {
    const int c = 2 * cp;
    const int g0 = c / cg, g1 = (c + 1) / cg;
    const float a0 = sstat[2 * g0 + 1] * gamma[c], a1 = sstat[2 * g1 + 1] * gamma[c + 1];
    const float b0 = beta[c] - sstat[2 * g0] * a0, b1 = beta[c + 1] - sstat[2 * g1] * a1;
    float2 v[kGnPix];
#pragma unroll
    for (int pp = 0; pp < kGnPix; ++pp) {            // all loads in flight first
      const int64_t off = (pix0 + pp) * C + c;
      v[pp] = x_f32 ? *reinterpret_cast<const float2*>(static_cast<const float*>(x) + off)
                    : __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(
                          static_cast<const __nv_bfloat16*>(x) + off));
    }
#pragma unroll
    for (int pp = 0; pp < kGnPix; ++pp) {
      float v0 = v[pp].x * a0 + b0, v1 = v[pp].y * a1 + b1;
      if (silu) { v0 = silu_fast(v0); v1 = silu_fast(v1); }
      *reinterpret_cast<__nv_bfloat162*>(out + (pix0 + pp) * C + c) = __floats2bfloat162_rn(v0, v1);
    }
  }
}

// ---- fused GroupNorm: one launch, one pass over HBM, cluster reduction ----
// A thread-block cluster of kGnCs CTAs owns one (image, chunk of gpc groups);
// its CTAs split the image's pixels.  Each CTA streams its rows x (cg * gpc)
// channels with 16-byte loads (thread = one 8-channel pack; a pack spans at
// most two groups since C/G >= 8), keeps the slice in shared memory when it
// fits, and reduces per-group (sum, sumsq) in a fixed order.  After one
// hardware cluster barrier every CTA sums the kGnCs partials of its groups
// over DSMEM in rank order (bit-reproducible, no atomics, no workspace) and
// applies (x - mean) * rstd * gamma + beta (+ SiLU) from shared memory.
// ---- GroupNorm, one CTA per (image, group), two passes through L2 --------
// The whole group (HW pixels x C/G channels) is reduced by one CTA: pass 1
// sums (x - shift) and (x - shift)^2 in a fixed order (shift = the group's
// first element: no cancellation when |mean| >> std), pass 2 re-reads the
// (L2-resident) slice and writes silu(gamma (x - mean) rstd + beta).  No
// cluster barrier or DSMEM exchange sits in the chain: one launch, two L2
// sweeps.  Thread t owns channel pair (t % cp) of pixels t / cp, t / cp + P, ...
// (cp = C / G / 2 pairs per pixel, P = blockDim / cp pixels per sweep).
constexpr int kGnGroupThreads = 512;
// auto: the group kernel only for small groups (its two L2 sweeps are latency-bound 4-byte
// loads: tools/gn_bench.py, 2 x 64 x 1280: 3.9 vs 5.4 us cluster; 2 x 256 x 1280: 6.9 vs 6.6;
// 2 x 4096 x 320: 26.7 vs 15.9)
constexpr int64_t kGnGroupMaxElems = 4096;

inline int& gn_mode() {          // drs_set_gn_mode: 0 auto, 1 group kernel, 2 cluster kernels only
  static int m = 0;
  return m;
}

template <bool F32>
__device__ __forceinline__ float2 gn_ld2(const void* x, int64_t off) {
  if constexpr (F32) return __ldg(reinterpret_cast<const float2*>(static_cast<const float*>(x) + off));
  else return __bfloat1622float2(__ldg(reinterpret_cast<const __nv_bfloat162*>(static_cast<const __nv_bfloat16*>(x) + off)));
}

template <bool F32>
__global__ void __launch_bounds__(kGnGroupThreads)
gn_group_kernel(const void* __restrict__ x, int HW, int C, int G, const float* __restrict__ gamma,
                const float* __restrict__ beta, float eps, int silu, __nv_bfloat16* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[2][kGnGroupThreads / 32];
  __shared__ float stat[2];
  const int n = blockIdx.x / G, g = blockIdx.x - n * G;
  const int cg = C / G, cp = cg >> 1;
  const int P = blockDim.x / cp;                       // pixels per sweep
  const int t = threadIdx.x;
  const bool act = t < P * cp;
  const int j = act ? t % cp : 0;
  const int p0 = act ? t / cp : HW;
  const int64_t base = (int64_t)n * HW * C + (int64_t)g * cg + 2 * j;
  const float shift = gn_ld2<F32>(x, (int64_t)n * HW * C + (int64_t)g * cg).x;
  float s = 0.f, q = 0.f;
  constexpr int kU = 8;
  for (int p = p0; p < HW; p += kU * P) {
    float2 v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {                     // independent loads in flight
      const int pp = p + u * P;
      v[u] = pp < HW ? gn_ld2<F32>(x, base + (int64_t)pp * C) : make_float2(shift, shift);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const float a = v[u].x - shift, b = v[u].y - shift;
      s += a + b;
      q = fmaf(a, a, fmaf(b, b, q));
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    q += __shfl_xor_sync(0xffffffffu, q, o);
  }
  const int warp = t >> 5, lane = t & 31;
  if (lane == 0) { red[0][warp] = s; red[1][warp] = q; }
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    s = lane < nw ? red[0][lane] : 0.f;
    q = lane < nw ? red[1][lane] : 0.f;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      s += __shfl_xor_sync(0xffffffffu, s, o);
      q += __shfl_xor_sync(0xffffffffu, q, o);
    }
    if (lane == 0) {
      const float cnt = (float)HW * (float)cg;
      const float m = s / cnt;
      stat[0] = shift + m;
      stat[1] = rsqrtf(fmaxf(q / cnt - m * m, 0.f) + eps);
    }
  }
  __syncthreads();
  if (!act) return;
  const float mean = stat[0], rstd = stat[1];
  const int c = g * cg + 2 * j;
  const float a0 = rstd * gamma[c], a1 = rstd * gamma[c + 1];
  const float b0 = beta[c] - mean * a0, b1 = beta[c + 1] - mean * a1;
  for (int p = p0; p < HW; p += kU * P) {
    float2 v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int pp = p + u * P;
      v[u] = pp < HW ? gn_ld2<F32>(x, base + (int64_t)pp * C) : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int pp = p + u * P;
      if (pp >= HW) break;
      float y0 = fmaf(v[u].x, a0, b0), y1 = fmaf(v[u].y, a1, b1);
      if (silu) {
        y0 = silu_fast(y0);
        y1 = silu_fast(y1);
      }
      *reinterpret_cast<__nv_bfloat162*>(out + base + (int64_t)pp * C) = __floats2bfloat162_rn(y0, y1);
    }
  }
}

constexpr int kGnCs = 8;                      // CTAs per cluster (portable size)

__device__ __forceinline__ void gn_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// (non-volatile: independent loads may be issued back to back; ordered after the cluster barrier by
// the barrier's acquire and by data dependence on nothing else)
__device__ __forceinline__ float2 gn_dsmem_ld2_nv(const void* local, int rank) {
  uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(local)), r;
  asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  float2 f;
  asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];" : "=f"(f.x), "=f"(f.y) : "r"(r));
  return f;
}
__device__ __forceinline__ float2 gn_dsmem_ld2(const void* local, int rank) {
  uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(local)), r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  float2 f;
  asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];" : "=f"(f.x), "=f"(f.y) : "r"(r) : "memory");
  return f;
}

template <bool F32>
__device__ __forceinline__ void gn_load8(const void* base, int64_t idx, float (&v)[8]) {
  if (F32) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(static_cast<const float*>(base) + idx));
    const float4 b = __ldg(reinterpret_cast<const float4*>(static_cast<const float*>(base) + idx) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  } else {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(base) + idx));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) { const float2 f = __bfloat1622float2(h[e]); v[2 * e] = f.x; v[2 * e + 1] = f.y; }
  }
}

#ifdef DRS_GN_TIMING
__device__ unsigned long long g_gn_ts[5][2048];
__device__ __forceinline__ void gn_stamp(int i) {
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_gn_ts[i][blockIdx.x] = t;
  }
}
#else
__device__ __forceinline__ void gn_stamp(int) {}
#endif

template <bool F32>
__global__ void __launch_bounds__(512)
gn_cluster_kernel(const void* __restrict__ x, int HW, int C, int G, int gpc, const float* __restrict__ gamma,
                  const float* __restrict__ beta, float eps, int silu, __nv_bfloat16* __restrict__ out, int rpc,
                  int keep) {
  extern __shared__ __align__(16) uint8_t gsm[];
  constexpr int kElem = F32 ? 4 : 2;
  const int cg = C / G, Cc = cg * gpc;                  // channels this cluster owns
  const int P = Cc / 8, R = blockDim.x / P;              // packs per row, rows per sweep
  const int t = threadIdx.x, q = t % P, rr = t / P;
  const int rank = blockIdx.x % kGnCs, cl = blockIdx.x / kGnCs;
  const int n_chunks = G / gpc;
  const int n = cl / n_chunks, chunk = cl % n_chunks;
  const int row0 = rank * rpc, row1 = min(HW, row0 + rpc);
  const int cbase = chunk * Cc, c0 = 8 * q;             // c0: channel within the chunk
  const int g_lo = c0 / cg, n_lo = min(8, (g_lo + 1) * cg - c0);
  float4* red = reinterpret_cast<float4*>(gsm);          // [blockDim] (s_lo, ss_lo, s_hi, ss_hi)
  float2* csum = reinterpret_cast<float2*>(gsm + blockDim.x * 16);   // [gpc] this CTA's partials
  float* stat = reinterpret_cast<float*>(gsm + blockDim.x * 16 + 32 * 8);  // [gpc][2]
  uint8_t* slice = gsm + blockDim.x * 16 + 32 * 8 + 32 * 8;         // [rpc][Cc]
  const int64_t img = (int64_t)n * HW * C + cbase;
  pdl_wait();
  gn_stamp(0);
  float s_lo = 0.f, ss_lo = 0.f, s_hi = 0.f, ss_hi = 0.f;
  constexpr int kB = 4;                                  // rows in flight per thread
  if (rr < R) {
    for (int rb = row0 + rr; rb < row1; rb += kB * R) {
      float v[kB][8];
#pragma unroll
      for (int i = 0; i < kB; ++i) {
        const int r = rb + i * R;
        if (r < row1) gn_load8<F32>(x, img + (int64_t)r * C + c0, v[i]);
      }
#pragma unroll
      for (int i = 0; i < kB; ++i) {
        const int r = rb + i * R;
        if (r >= row1) break;
        if (keep) {
          uint8_t* d = slice + ((size_t)(r - row0) * Cc + c0) * kElem;
          if (F32) {
            reinterpret_cast<float4*>(d)[0] = make_float4(v[i][0], v[i][1], v[i][2], v[i][3]);
            reinterpret_cast<float4*>(d)[1] = make_float4(v[i][4], v[i][5], v[i][6], v[i][7]);
          } else {
            uint4 u;
            __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
            for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(v[i][2 * e], v[i][2 * e + 1]);   // exact
            *reinterpret_cast<uint4*>(d) = u;
          }
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          if (e < n_lo) { s_lo += v[i][e]; ss_lo += v[i][e] * v[i][e]; }
          else { s_hi += v[i][e]; ss_hi += v[i][e] * v[i][e]; }
        }
      }
    }
  }
  red[t] = make_float4(s_lo, ss_lo, s_hi, ss_hi);
  __syncthreads();
  for (int g = t; g < gpc; g += blockDim.x) {            // fixed order: packs, then row lanes
    float a = 0.f, b = 0.f;
    const int qa = (g * cg) / 8, qb = ((g + 1) * cg - 1) / 8;
    for (int qq = qa; qq <= qb; ++qq) {
      const bool lo = (8 * qq) / cg == g;
      for (int r2 = 0; r2 < R; ++r2) {
        const float4 f = red[r2 * P + qq];
        a += lo ? f.x : f.z;
        b += lo ? f.y : f.w;
      }
    }
    csum[g] = make_float2(a, b);
  }
  gn_stamp(1);
  gn_cluster_sync();                                     // every CTA's partials are published
  gn_stamp(2);
  pdl_trigger();
  for (int g = t; g < gpc; g += blockDim.x) {
    float a = 0.f, b = 0.f;
    for (int r2 = 0; r2 < kGnCs; ++r2) {                 // rank order: deterministic
      const float2 f = gn_dsmem_ld2(&csum[g], r2);
      a += f.x;
      b += f.y;
    }
    const float cnt = (float)HW * cg;
    const float mean = a / cnt;
    const float var = fmaxf(b / cnt - mean * mean, 0.f);
    stat[2 * g] = mean;
    stat[2 * g + 1] = rsqrtf(var + eps);
  }
  gn_cluster_sync();                                     // stats read; peers may exit afterwards
  gn_stamp(3);
  if (rr >= R) return;
  float sa[8], sb[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int g = (c0 + e) / cg;
    sa[e] = stat[2 * g + 1] * __ldg(gamma + cbase + c0 + e);
    sb[e] = __ldg(beta + cbase + c0 + e) - stat[2 * g] * sa[e];
  }
  for (int rb = row0 + rr; rb < row1; rb += kB * R) {
    float v[kB][8];
#pragma unroll
    for (int i = 0; i < kB; ++i) {
      const int r = rb + i * R;
      if (r >= row1) break;
      if (keep) {
        const uint8_t* d = slice + ((size_t)(r - row0) * Cc + c0) * kElem;
        if (F32) {
          const float4 a4 = reinterpret_cast<const float4*>(d)[0], b4 = reinterpret_cast<const float4*>(d)[1];
          v[i][0] = a4.x; v[i][1] = a4.y; v[i][2] = a4.z; v[i][3] = a4.w;
          v[i][4] = b4.x; v[i][5] = b4.y; v[i][6] = b4.z; v[i][7] = b4.w;
        } else {
          const uint4 u = *reinterpret_cast<const uint4*>(d);
          const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f = __bfloat1622float2(h[e]);
            v[i][2 * e] = f.x;
            v[i][2 * e + 1] = f.y;
          }
        }
      } else {
        gn_load8<F32>(x, img + (int64_t)r * C + c0, v[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < kB; ++i) {
      const int r = rb + i * R;
      if (r >= row1) break;
      uint4 u;
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float y0 = v[i][2 * e] * sa[2 * e] + sb[2 * e], y1 = v[i][2 * e + 1] * sa[2 * e + 1] + sb[2 * e + 1];
        if (silu) { y0 = silu_fast(y0); y1 = silu_fast(y1); }
        h[e] = __floats2bfloat162_rn(y0, y1);
      }
      *reinterpret_cast<uint4*>(out + img + (int64_t)r * C + c0) = u;
    }
  }
  gn_stamp(4);
}

// TMA variant of the cluster GroupNorm (bf16 input): the CTA's slice (rpc rows
// x cg*gpc channels) arrives in shared memory through a few 2-D bulk-tensor
// loads (full-rate streaming instead of per-thread 16-byte loads), the stats,
// cluster exchange and the in-place apply run on shared memory, and a few
// bulk-tensor stores write the slice back.  rpc = HW / kGnCs exactly, in boxes
// of `box` rows that divide it, so no CTA writes outside its own rows.
__global__ void __launch_bounds__(512)
gn_tma_kernel(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout, int HW, int C,
              int G, int gpc, const float* __restrict__ gamma, const float* __restrict__ beta, float eps, int silu,
              int rpc, int box) {
  extern __shared__ __align__(1024) uint8_t gsm_t[];
  // 1 KB-aligned by pointer arithmetic on the shared array (keeps the shared state space: LDS/STS)
  uint8_t* base = gsm_t + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(gsm_t)) & 1023u)) & 1023u);
  const int cg = C / G, Cc = cg * gpc;
  const int P = Cc / 8, R = blockDim.x / P;
  const int t = threadIdx.x, q = t % P, rr = t / P;
  const int rank = blockIdx.x % kGnCs, cl = blockIdx.x / kGnCs;
  const int n_chunks = G / gpc;
  const int n = cl / n_chunks, chunk = cl % n_chunks;
  const int row0 = rank * rpc;
  const int cbase = chunk * Cc, c0 = 8 * q;
  const int g_lo = c0 / cg, n_lo = min(8, (g_lo + 1) * cg - c0);
  const size_t slice_bytes = (size_t)rpc * Cc * 2;
  uint8_t* slice = base;                                                   // [rpc][Cc] bf16
  float4* red = reinterpret_cast<float4*>(base + ((slice_bytes + 127) & ~size_t(127)));
  float2* csum = reinterpret_cast<float2*>(red + blockDim.x);              // [gpc]
  float* stat = reinterpret_cast<float*>(csum + 32);                       // [gpc][2]
  uint64_t* bar = reinterpret_cast<uint64_t*>(stat + 64);
  float4* part = reinterpret_cast<float4*>(bar + 8);                       // [nch][P] row-lane partials
  if (t == 0) {
    tc::tma_prefetch(&tin);
    tc::tma_prefetch(&tout);
    tc::mbar_init(bar, 1);
    tc::fence_barrier_init();
  }
  __syncthreads();
  pdl_wait();
  if (t == 0) {
    tc::mbar_arrive_expect_tx(bar, (uint32_t)slice_bytes);
    for (int k = 0; k < rpc / box; ++k)
      tc::tma_load_2d(&tin, bar, slice + (size_t)k * box * Cc * 2, cbase, n * HW + row0 + k * box);
  }
  tc::mbar_wait(bar, 0);
  float s_lo = 0.f, ss_lo = 0.f, s_hi = 0.f, ss_hi = 0.f;
  if (rr < R) {
    for (int r = rr; r < rpc; r += R) {
      const uint4 u = *reinterpret_cast<const uint4*>(slice + ((size_t)r * Cc + c0) * 2);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(h[e]);
        if (2 * e < n_lo) { s_lo += f.x; ss_lo += f.x * f.x; } else { s_hi += f.x; ss_hi += f.x * f.x; }
        if (2 * e + 1 < n_lo) { s_lo += f.y; ss_lo += f.y * f.y; } else { s_hi += f.y; ss_hi += f.y * f.y; }
      }
    }
  }
  // gamma / beta of this thread's 8 channels: issued now, used after the cluster exchange
  float gmv[8], btv[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    gmv[e] = rr < R ? __ldg(gamma + cbase + c0 + e) : 0.f;
    btv[e] = rr < R ? __ldg(beta + cbase + c0 + e) : 0.f;
  }
  red[t] = make_float4(s_lo, ss_lo, s_hi, ss_hi);
  __syncthreads();
  // row-lane reduction in two fixed-order levels (was one thread per group walking all R lanes):
  // nch chunks of lanes per pack in parallel, then per group over packs and chunks
  const int nch = P * 8 <= 64 ? 8 : (64 / P > 0 ? 64 / P : 1);
  if (t < P * nch) {
    const int qp = t % P, ch = t / P;
    const int r_lo = ch * R / nch, r_hi = (ch + 1) * R / nch;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int r2 = r_lo; r2 < r_hi; ++r2) {
      const float4 f = red[r2 * P + qp];
      acc.x += f.x; acc.y += f.y; acc.z += f.z; acc.w += f.w;
    }
    part[ch * P + qp] = acc;
  }
  __syncthreads();
  for (int g = t; g < gpc; g += blockDim.x) {            // fixed order: packs, then lane chunks
    float a = 0.f, b = 0.f;
    const int qa = (g * cg) / 8, qb = ((g + 1) * cg - 1) / 8;
    for (int qq = qa; qq <= qb; ++qq) {
      const bool lo = (8 * qq) / cg == g;
      float4 f[8];
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) f[ch] = ch < nch ? part[ch * P + qq] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) {
        a += lo ? f[ch].x : f[ch].z;
        b += lo ? f[ch].y : f[ch].w;
      }
    }
    csum[g] = make_float2(a, b);
  }
  gn_cluster_sync();
  pdl_trigger();
  for (int g = t; g < gpc; g += blockDim.x) {
    float a = 0.f, b = 0.f;
    float2 fr[kGnCs];                                     // all peers' sums in flight, then added in rank order
#pragma unroll
    for (int r2 = 0; r2 < kGnCs; ++r2) fr[r2] = gn_dsmem_ld2_nv(&csum[g], r2);
#pragma unroll
    for (int r2 = 0; r2 < kGnCs; ++r2) {
      a += fr[r2].x;
      b += fr[r2].y;
    }
    const float cnt = (float)HW * cg;
    const float mean = a / cnt;
    const float var = fmaxf(b / cnt - mean * mean, 0.f);
    stat[2 * g] = mean;
    stat[2 * g + 1] = rsqrtf(var + eps);
  }
  // peers may still read this CTA's csum: arrive now, wait only before exiting,
  // so the apply / store below overlaps the slowest peer's DSMEM reads
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  __syncthreads();                                       // stat[] visible CTA-wide
  if (rr < R) {
    float sa[8], sb[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int g = (c0 + e) / cg;
      sa[e] = stat[2 * g + 1] * gmv[e];
      sb[e] = btv[e] - stat[2 * g] * sa[e];
    }
#pragma unroll 2
    for (int r = rr; r < rpc; r += R) {
      uint4* p4 = reinterpret_cast<uint4*>(slice + ((size_t)r * Cc + c0) * 2);
      uint4 u = *p4;
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(h[e]);
        float y0 = f.x * sa[2 * e] + sb[2 * e], y1 = f.y * sa[2 * e + 1] + sb[2 * e + 1];
        if (silu) { y0 = silu_fast(y0); y1 = silu_fast(y1); }
        h[e] = __floats2bfloat162_rn(y0, y1);
      }
      *p4 = u;
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (t == 0) {
    for (int k = 0; k < rpc / box; ++k) {
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];"
                   :: "l"(&tout), "r"(tc::smem_u32(slice + (size_t)k * box * Cc * 2)), "r"(cbase),
                      "r"(n * HW + row0 + k * box) : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

typedef CUresult (*PFN_encodeTiledGn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static bool gn_tmap(CUtensorMap* m, const void* ptr, int64_t rows, int C, int box_c, int box_r) {
  static PFN_encodeTiledGn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) != cudaSuccess ||
        qr != cudaDriverEntryPointSuccess)
      return false;
    fn = reinterpret_cast<PFN_encodeTiledGn>(p);
  }
  cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)C * 2};
  cuuint32_t boxd[2] = {(cuuint32_t)box_c, (cuuint32_t)box_r};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, boxd, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int gn_num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

// geometry of the cluster path (false: use the two-kernel path).  gpc = groups
// per cluster: the smallest divisor of G whose channel span is a multiple of
// 8 and that still leaves >= ~#SMs CTAs, so small batches fill the GPU.
static bool gn_cluster_plan(int N, int HW, int C, int G, int x_f32, int& gpc, int& rpc, int& threads, int& keep,
                            size_t& smem, bool size_cap = true) {
  const int cg = C / G;
  if (C % 8 || cg < 8 || G > 32) return false;
  // measured (tools/gn_bench.py): the cluster path wins up to ~12 MB of input;
  // beyond that the two-kernel path's wider grid streams faster
  if (size_cap && (int64_t)N * HW * C * (x_f32 ? 4 : 2) > 12 * 1024 * 1024) return false;
  gpc = 0;
  for (int d = 1; d <= G; ++d) {
    if (G % d || (cg * d) % 8 || (cg * d) / 8 > 512) continue;
    if (!gpc) gpc = d;                                   // smallest legal chunk
    if ((int64_t)N * (G / d) * kGnCs <= 2 * gn_num_sms()) { gpc = d; break; }
  }
  if (!gpc) return false;
  const int P = cg * gpc / 8;
  threads = P * (P >= 256 ? 1 : 256 / P);        // <= ~256 threads: two or more CTAs per SM
  rpc = (HW + kGnCs - 1) / kGnCs;
  const size_t base = (size_t)threads * 16 + 32 * 8 + 32 * 8;
  const size_t slice = (size_t)rpc * cg * gpc * (x_f32 ? 4 : 2);
  keep = base + slice <= 200 * 1024;
  smem = base + (keep ? slice : 0);
  return true;
}

// latent (C, H, W) fp64/fp32 -> NHWC bf16 with Cpad channels (zeros beyond C)
__global__ void latent_to_nhwc_kernel(const void* __restrict__ x, int x_f64, int C, int HW, int Cpad,
                                      __nv_bfloat16* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= HW * Cpad) return;
  const int p = i / Cpad, c = i % Cpad;
  float v = 0.f;
  if (c < C) v = x_f64 ? (float)static_cast<const double*>(x)[(int64_t)c * HW + p]
                       : static_cast<const float*>(x)[(int64_t)c * HW + p];
  out[i] = __float2bfloat16(v);
}

// classifier-free guidance: rows [0, HW) = uncond, [HW, 2HW) = cond (NHWC fp32, ld
// columns); eps (C, H, W) = u + g (c - u).  g == 1 or ld == 0: single image.
__global__ void cfg_combine_kernel(const float* __restrict__ y, int64_t ld, int HW, int C, float g, int pair,
                                   float* __restrict__ eps) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= C * HW) return;
  const int c = i / HW, p = i % HW;
  const float u = y[(int64_t)p * ld + c];
  eps[i] = pair ? u + g * (y[(int64_t)(HW + p) * ld + c] - u) : u;
}

}  // namespace drs

using namespace drs;

extern "C" int drs_layernorm(const void* x, int64_t ldx, int x_f32, int M, int C, const float* gamma,
                             const float* beta, const float* shift, const float* scale, int mod_group,
                             int64_t mod_ld, float eps, void* out, int64_t ldo, void* stream) {
  if (M <= 0 || C <= 0) return M == 0 ? DRS_OK : DRS_ERR_VALUE;
  if (!x || !out || C > 128 * 16 || C % 4 || ldx % 4 || ldo % 4 || (mod_group > 0 && mod_ld % 4)) return DRS_ERR_VALUE;
  auto mis = [](const void* p, uintptr_t a) { return p && (reinterpret_cast<uintptr_t>(p) & (a - 1)); };
  if (mis(x, x_f32 ? 16 : 8) || mis(out, 8) || mis(shift, 16) || mis(scale, 16) || mis(gamma, 16) || mis(beta, 16))
    return DRS_ERR_VALUE;
  cudaStream_t st = (cudaStream_t)stream;
  __nv_bfloat16* o = static_cast<__nv_bfloat16*>(out);
  // measured (tools/ln_bench.py): one CTA per row wins for wide rows (C >= 1024)
  // and for few rows (M <= 1024); one warp per row wins for narrow rows at large M
  // (re-measured late round 2: the warp path for the DiT rows (256 x 1152) costs +11 % per eval)
  const bool row_path = C >= 1024 || M <= 1024;
  if (row_path && C / 4 <= 512) {                                              // row-per-CTA path
    const int thr = ((C / 4 + 31) / 32) * 32;
    launch_pdl(layernorm_row_kernel, dim3(M), dim3(thr), 0, st, x, ldx, x_f32, C, gamma, beta, shift, scale,
               mod_group, mod_ld, eps, o, ldo);
    return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
  }
  // rows (warps) per CTA, measured in the SD1.5 graph: 8 -> 4.266, 4 -> 4.247, 2 -> 4.256, 1 -> 4.313 ms/eval
  const int warps = 4;
  dim3 grid((M + warps - 1) / warps);
  const int v4 = (C / 4 + 31) / 32;
#define DRS_LN(K) launch_pdl(layernorm_kernel<K>, dim3(grid), dim3(warps * 32), 0, st, x, ldx, x_f32, M, C, gamma, beta, shift, scale, \
                                                                  mod_group, mod_ld, eps, o, ldo)
  if (v4 <= 4) DRS_LN(4);
  else if (v4 <= 8) DRS_LN(8);
  else if (v4 <= 12) DRS_LN(12);
  else DRS_LN(16);
#undef DRS_LN
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
}

extern "C" int drs_attention(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v, int64_t ldv,
                             void* o, int64_t ldo, int B, int H, int Lq, int Lk, int d, float scale,
                             void* stream) {
  if (B <= 0 || H <= 0 || Lq <= 0 || Lk <= 0) return DRS_ERR_VALUE;
  if (d % 8 || d > 160 || (ldq | ldk | ldv | ldo) % 8) return DRS_ERR_VALUE;
  const int DP = (d + 15) / 16 * 16;
  dim3 grid((Lq + kAttnBQ - 1) / kAttnBQ, H, B);
  const float sl2 = scale * 1.4426950408889634f;
  cudaStream_t st = (cudaStream_t)stream;
  auto Q = static_cast<const __nv_bfloat16*>(q);
  auto K = static_cast<const __nv_bfloat16*>(k);
  auto V = static_cast<const __nv_bfloat16*>(v);
  auto O = static_cast<__nv_bfloat16*>(o);
  switch (DP) {
    case 16: launch_pdl(attention_kernel<16>, dim3(grid), dim3(kAttnThreads), 0, st, Q, ldq, K, ldk, V, ldv, O, ldo, Lq, Lk, d, sl2); break;
    case 32: launch_pdl(attention_kernel<32>, dim3(grid), dim3(kAttnThreads), 0, st, Q, ldq, K, ldk, V, ldv, O, ldo, Lq, Lk, d, sl2); break;
    case 48: launch_pdl(attention_kernel<48>, dim3(grid), dim3(kAttnThreads), 0, st, Q, ldq, K, ldk, V, ldv, O, ldo, Lq, Lk, d, sl2); break;
    case 64: launch_pdl(attention_kernel<64>, dim3(grid), dim3(kAttnThreads), 0, st, Q, ldq, K, ldk, V, ldv, O, ldo, Lq, Lk, d, sl2); break;
    case 80: launch_pdl(attention_kernel<80>, dim3(grid), dim3(kAttnThreads), 0, st, Q, ldq, K, ldk, V, ldv, O, ldo, Lq, Lk, d, sl2); break;
    case 96: launch_pdl(attention_kernel<96>, dim3(grid), dim3(kAttnThreads), 0, st, Q, ldq, K, ldk, V, ldv, O, ldo, Lq, Lk, d, sl2); break;
    case 128: launch_pdl(attention_kernel<128>, dim3(grid), dim3(kAttnThreads), 0, st, Q, ldq, K, ldk, V, ldv, O, ldo, Lq, Lk, d, sl2); break;
    case 160: launch_pdl(attention_kernel<160>, dim3(grid), dim3(kAttnThreads), 0, st, Q, ldq, K, ldk, V, ldv, O, ldo, Lq, Lk, d, sl2); break;
    default: return DRS_ERR_VALUE;
  }
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
}

extern "C" int drs_timestep_embedding(const float* t, int n, int dim, float max_period, void* out, void* stream) {
  if (n <= 0 || dim <= 0 || dim % 2) return DRS_ERR_VALUE;
  const int tot = n * dim / 2;
  launch_pdl(timestep_embedding_kernel, dim3((tot + 255) / 256), dim3(256), 0, (cudaStream_t)stream, 
      t, n, dim, max_period, static_cast<__nv_bfloat16*>(out));
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
}

extern "C" int drs_patchify(const void* x, int x_f64, int C, int H, int W, int p, void* out, void* stream) {
  if (p <= 0 || H % p || W % p) return DRS_ERR_VALUE;
  const int tot = C * H * W;
  launch_pdl(patchify_kernel, dim3((tot + 255) / 256), dim3(256), 0, (cudaStream_t)stream, x, x_f64, C, H, W, p,
                                                                       static_cast<__nv_bfloat16*>(out));
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
}

extern "C" int drs_unpatchify(const float* tok, int Cout, int Ckeep, int H, int W, int p, float* out, void* stream) {
  if (p <= 0 || H % p || W % p || Ckeep > Cout) return DRS_ERR_VALUE;
  const int tot = Ckeep * H * W;
  launch_pdl(unpatchify_kernel, dim3((tot + 255) / 256), dim3(256), 0, (cudaStream_t)stream, tok, Cout, Ckeep, H, W, p, out);
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
}

namespace drs {
// ---- GEMV for M <= 4 rows (conditioning MLPs: timestep / adaLN embeddings) ----
// y[m, n] = act(sum_k x[m, k] W[n, k] + bias[n]) (+ residual[m, n]).  The weight
// stream is the whole cost (DiT adaLN: 446 MB for one row): each warp owns rows
// n, reads them with 16-byte ld.global.nc (L1 no-allocate) loads, kGvRows rows in
// flight per lane, the x rows sit in shared memory as fp32; a small-footprint CTA
// (256 threads, <= 72 KB smem) that co-resides with the tensor-core GEMMs, so the
// conditioning GEMVs can run on a side stream under them.
constexpr int kGvThreads = 256;
constexpr int kGvRows = 4;          // weight rows per warp in flight
constexpr int kGvMaxM = 4;

__device__ __forceinline__ uint4 ld_nc_na_v4(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

template <int MM>
__global__ void __launch_bounds__(kGvThreads)
gemv_kernel(const __nv_bfloat16* __restrict__ x, int64_t ldx, const __nv_bfloat16* __restrict__ w, int64_t ldw,
            const float* __restrict__ bias, const void* __restrict__ res, int64_t ldr, int res_f32,
            void* __restrict__ out, int64_t ldo, int out_f32, int N, int K, int act) {
  extern __shared__ uint4 sx[];                       // [MM][K / 8] bf16 x 8
  pdl_wait();
  pdl_trigger();
  const int kv = K >> 3;                              // 16-byte vectors per row
  for (int i = threadIdx.x; i < MM * kv; i += blockDim.x) {
    const int m = i / kv, k = i - m * kv;
    sx[i] = *reinterpret_cast<const uint4*>(x + (int64_t)m * ldx + 8 * k);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warps_total = gridDim.x * (kGvThreads / 32);
  const int wid = blockIdx.x * (kGvThreads / 32) + (threadIdx.x >> 5);
  for (int n0 = wid * kGvRows; n0 < N; n0 += warps_total * kGvRows) {
    float acc[kGvRows][MM];
#pragma unroll
    for (int r = 0; r < kGvRows; ++r)
#pragma unroll
      for (int m = 0; m < MM; ++m) acc[r][m] = 0.f;
    for (int v = lane; v < kv; v += 32) {
      uint4 wv[kGvRows];
#pragma unroll
      for (int r = 0; r < kGvRows; ++r)               // rows of this warp: independent loads in flight
        wv[r] = n0 + r < N ? ld_nc_na_v4(w + (int64_t)(n0 + r) * ldw + 8 * v) : make_uint4(0, 0, 0, 0);
      float2 xf[MM][4];                                // x[m, 8v .. 8v+7] (conflict-free 16-byte reads)
#pragma unroll
      for (int m = 0; m < MM; ++m) {
        const uint4 xv = sx[m * kv + v];
        const __nv_bfloat162* xh = reinterpret_cast<const __nv_bfloat162*>(&xv);
#pragma unroll
        for (int e = 0; e < 4; ++e) xf[m][e] = __bfloat1622float2(xh[e]);
      }
#pragma unroll
      for (int r = 0; r < kGvRows; ++r) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&wv[r]);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(h[e]);
#pragma unroll
          for (int m = 0; m < MM; ++m) acc[r][m] = fmaf(f.x, xf[m][e].x, fmaf(f.y, xf[m][e].y, acc[r][m]));
        }
      }
    }
#pragma unroll
    for (int r = 0; r < kGvRows; ++r)
#pragma unroll
      for (int m = 0; m < MM; ++m)
#pragma unroll
        for (int o = 16; o; o >>= 1) acc[r][m] += __shfl_xor_sync(0xffffffffu, acc[r][m], o);
    if (lane < kGvRows * MM) {                        // lane (r, m) finishes output (m, n0 + r)
      const int r = lane / MM, m = lane - r * MM;
      float y = 0.f;
#pragma unroll
      for (int rr = 0; rr < kGvRows; ++rr)
#pragma unroll
        for (int mm = 0; mm < MM; ++mm)
          if (rr == r && mm == m) y = acc[rr][mm];
      const int n = n0 + r;
      if (n < N) {
        if (bias) y += bias[n];
        if (act == DRS_ACT_SILU) y = y / (1.f + __expf(-y));
        if (res) y += res_f32 ? static_cast<const float*>(res)[(int64_t)m * ldr + n]
                              : __bfloat162float(static_cast<const __nv_bfloat16*>(res)[(int64_t)m * ldr + n]);
        if (out_f32) static_cast<float*>(out)[(int64_t)m * ldo + n] = y;
        else static_cast<__nv_bfloat16*>(out)[(int64_t)m * ldo + n] = __float2bfloat16(y);
      }
    }
  }
}
}  // namespace drs

extern "C" int drs_gemv(const void* x, int64_t ldx, const void* w, int64_t ldw, const float* bias, const void* res,
                        int64_t ldr, int res_f32, void* out, int64_t ldo, int out_f32, int M, int N, int K, int act,
                        int ctas_per_sm, void* stream) {
  using namespace drs;
  if (M < 1 || M > kGvMaxM || N < 1 || K < 8 || K % 8 || ldw % 8 || ldx % 8 || !x || !w || !out) return DRS_ERR_VALUE;
  if (act != DRS_ACT_NONE && act != DRS_ACT_SILU) return DRS_ERR_VALUE;
  if ((reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(x)) & 15) return DRS_ERR_VALUE;
  const size_t smem = (size_t)M * K * 2;
  if (smem > 72 * 1024) return DRS_ERR_VALUE;
  static int sms = [] { int d = 0, n = 148; cudaGetDevice(&d); cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d); return n; }();
  const int warps_needed = (N + kGvRows - 1) / kGvRows;
  int blocks = (warps_needed + kGvThreads / 32 - 1) / (kGvThreads / 32);
  const int cps = ctas_per_sm > 0 ? ctas_per_sm : 4;      // 1: leave room for co-resident GEMMs
  if (blocks > cps * sms) blocks = cps * sms;
  cudaStream_t st = (cudaStream_t)stream;
  auto go = [&](auto kern) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_pdl(kern, dim3(blocks), dim3(kGvThreads), smem, st, static_cast<const __nv_bfloat16*>(x), ldx,
               static_cast<const __nv_bfloat16*>(w), ldw, bias, res, ldr, res_f32, out, ldo, out_f32, N, K, act);
  };
  switch (M) {
    case 1: go(gemv_kernel<1>); break;
    case 2: go(gemv_kernel<2>); break;
    case 3: go(gemv_kernel<3>); break;
    default: go(gemv_kernel<4>); break;
  }
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
}

extern "C" int drs_silu_cast(const float* x, int64_t n, void* out, void* stream) {
  if (n < 0) return DRS_ERR_VALUE;
  if (n == 0) return DRS_OK;
  launch_pdl(silu_cast_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, (cudaStream_t)stream, 
      x, n, static_cast<__nv_bfloat16*>(out));
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
}

extern "C" int drs_im2col(const void* x1, int C1, const void* x2, int C2, int N, int H, int W, int ks, int stride,
                          int pad, int up, void* out, void* stream) {
  if ((C1 % 8) || (C2 % 8) || (C2 && !x2) || ks < 1 || stride < 1 || up < 1) return DRS_ERR_VALUE;
  const int Ho = (H * up + 2 * pad - ks) / stride + 1, Wo = (W * up + 2 * pad - ks) / stride + 1;
  const int64_t total = (int64_t)N * Ho * Wo * ks * ks * ((C1 + C2) / 8);
  if (total >= (1ll << 31)) return DRS_ERR_VALUE;
  launch_pdl(im2col_kernel, dim3((unsigned)((total + 255) / 256)), dim3(256), 0, (cudaStream_t)stream, 
      static_cast<const __nv_bfloat16*>(x1), C1, static_cast<const __nv_bfloat16*>(x2), C2, N, H, W, ks, stride, pad,
      up, Ho, Wo, static_cast<__nv_bfloat16*>(out));
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
}

namespace drs {
// (image, group) CTAs: chosen when every pair of channels sits in one group and
// a group's slice is small enough that one SM sweeps it twice faster than the
// cluster kernels' barrier chain (decided by tools/gn_bench.py A/B runs)
static bool gn_group_ok(int N, int HW, int C, int G) {
  const int cg = C / G;
  return cg % 2 == 0 && cg / 2 <= kGnGroupThreads && (int64_t)HW * cg <= kGnGroupMaxElems;
}
}  // namespace drs

extern "C" int drs_set_gn_mode(int mode) {
  if (mode < 0 || mode > 2) return DRS_ERR_VALUE;
  drs::gn_mode() = mode;
  return DRS_OK;
}

extern "C" size_t drs_groupnorm_workspace_bytes(int N, int G) {
  return (size_t)(N > 0 ? N : 0) * (G > 0 ? G : 0) * drs::kGnSplit * sizeof(float2);   // two-kernel path only
}

extern "C" int drs_groupnorm(const void* x, int x_f32, int N, int HW, int C, int G, const float* gamma,
                             const float* beta, float eps, int silu, void* out, void* workspace, void* stream) {
  using namespace drs;
  if (N <= 0 || HW <= 0 || G <= 0 || C % G || (C / G) % 2 || !gamma || !beta) return DRS_ERR_VALUE;
  cudaStream_t st = (cudaStream_t)stream;
  const bool al4 = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(out)) & 3) == 0;
  if (al4 && (C / G) % 2 == 0 && (gn_mode() == 1 || (gn_mode() == 0 && gn_group_ok(N, HW, C, G)))) {
    if (x_f32)
      launch_pdl(gn_group_kernel<true>, dim3(N * G), dim3(kGnGroupThreads), 0, st, x, HW, C, G, gamma, beta, eps,
                 silu, static_cast<__nv_bfloat16*>(out));
    else
      launch_pdl(gn_group_kernel<false>, dim3(N * G), dim3(kGnGroupThreads), 0, st, x, HW, C, G, gamma, beta, eps,
                 silu, static_cast<__nv_bfloat16*>(out));
    return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
  }
  int gpc, rpc, threads, keep;
  size_t smem;
  const bool aligned = (reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  if (aligned && !x_f32 && HW % kGnCs == 0 && gn_cluster_plan(N, HW, C, G, 0, gpc, rpc, threads, keep, smem) &&
      rpc == HW / kGnCs) {
    // TMA slice path: boxes of `box` rows dividing rpc, slice (+ scratch) within 200 KB
    int box = rpc < 256 ? rpc : 256;
    while (box > 1 && rpc % box) --box;
    const int Cc = (C / G) * gpc;
    // (~256 threads from the plan; 512 measured slower: 64x64 10.4 -> 13.2 us, SD1.5 eval +2.2 %)
    const size_t slice = (size_t)rpc * Cc * 2;
    const size_t need = ((slice + 127) & ~size_t(127)) + (size_t)threads * 16 + 32 * 8 + 64 * 4 + 64 + 64 * 16 + 1024;
    CUtensorMap tin, tout;
    if (box >= 8 && need <= 200 * 1024 && gn_tmap(&tin, x, (int64_t)N * HW, C, Cc, box) &&
        gn_tmap(&tout, out, (int64_t)N * HW, C, Cc, box)) {
      static bool attr = false;
      if (!attr) {
        if (cudaFuncSetAttribute(gn_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) !=
            cudaSuccess)
          return DRS_ERR_CUDA;
        attr = true;
      }
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(N * (G / gpc) * kGnCs);
      cfg.blockDim = dim3(threads);
      cfg.dynamicSmemBytes = need;
      cfg.stream = st;
      cudaLaunchAttribute la[2];
      la[0].id = cudaLaunchAttributeClusterDimension;
      la[0].val.clusterDim.x = kGnCs;
      la[0].val.clusterDim.y = 1;
      la[0].val.clusterDim.z = 1;
      la[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      la[1].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = la;
      cfg.numAttrs = pdl_enabled() ? 2 : 1;
      cudaLaunchKernelEx(&cfg, gn_tma_kernel, tin, tout, HW, C, G, gpc, gamma, beta, eps, silu, rpc, box);
      return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
    }
  }
  if (aligned && gn_cluster_plan(N, HW, C, G, x_f32, gpc, rpc, threads, keep, smem)) {
    auto kern = x_f32 ? gn_cluster_kernel<true> : gn_cluster_kernel<false>;
    static bool attr[2] = {false, false};
    if (!attr[x_f32 ? 1 : 0]) {
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) != cudaSuccess)
        return DRS_ERR_CUDA;
      attr[x_f32 ? 1 : 0] = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(N * (G / gpc) * kGnCs);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute la[2];
    la[0].id = cudaLaunchAttributeClusterDimension;
    la[0].val.clusterDim.x = kGnCs;
    la[0].val.clusterDim.y = 1;
    la[0].val.clusterDim.z = 1;
    la[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    la[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = la;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    cudaLaunchKernelEx(&cfg, kern, x, HW, C, G, gpc, gamma, beta, eps, silu, static_cast<__nv_bfloat16*>(out), rpc,
                       keep);
    return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
  }
  if (!workspace) return DRS_ERR_VALUE;
  if (HW % kGnPix) return DRS_ERR_VALUE;
  float2* part = static_cast<float2*>(workspace);    // N*G*kGnSplit float2
  launch_pdl(gn_stats_kernel, dim3(dim3(N * G, kGnSplit)), dim3(256), 0, st, x, x_f32, HW, C, G, part);
  const int c2 = C / 2, thr = c2 >= 256 ? 256 : ((c2 + 31) / 32) * 32;
  launch_pdl(gn_apply_kernel, dim3((unsigned)((int64_t)N * HW / kGnPix)), dim3(thr), 2 * G * sizeof(float), st,
      x, x_f32, HW, C, G, part, gamma, beta, eps, silu, static_cast<__nv_bfloat16*>(out));
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
}

extern "C" int drs_latent_to_nhwc(const void* x, int x_f64, int C, int HW, int Cpad, void* out, void* stream) {
  if (Cpad < C) return DRS_ERR_VALUE;
  launch_pdl(latent_to_nhwc_kernel, dim3((HW * Cpad + 255) / 256), dim3(256), 0, (cudaStream_t)stream, 
      x, x_f64, C, HW, Cpad, static_cast<__nv_bfloat16*>(out));
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
}

extern "C" int drs_cfg_combine(const float* y, int64_t ld, int HW, int C, float g, int pair, float* eps,
                               void* stream) {
  launch_pdl(cfg_combine_kernel, dim3((C * HW + 255) / 256), dim3(256), 0, (cudaStream_t)stream, y, ld, HW, C, g, pair, eps);
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
}

extern "C" int drs_cast_f32_bf16(const float* x, int64_t n, void* out, void* stream) {
  if (n < 0 || (reinterpret_cast<uintptr_t>(x) & 15) || (reinterpret_cast<uintptr_t>(out) & 7)) return DRS_ERR_VALUE;
  if (n == 0) return DRS_OK;
  const int64_t th = (n + 3) / 4;
  launch_pdl(cast_f32_bf16_kernel, dim3((unsigned)((th + 255) / 256)), dim3(256), 0, (cudaStream_t)stream, 
      x, n, static_cast<__nv_bfloat16*>(out));
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
}
