// K6: fused attention forward on the 5th-gen tensor cores (non-causal).
//
//   O[b, q, h, :] = softmax_k( Q[b, q, h, :] . K[b, k, h, :] * scale ) V[b, k, h, :]
//
// One CTA per (128-query tile, head, image).  Warp roles (352 threads, default build):
//   warp 0      TMA producer: Q once, then K / V tiles of 128 keys into two
//               rings (mbarrier full/empty)
//   warp 1      TMEM allocator + S issuer: S_j = Q K_j^T (M=128, N=128, K=DP)
//               into one of two TMEM S buffers, S_{j+2} as soon as S_j is read
//   warp 10     PV issuer: O_set += P_j V_j (M=128, N=DP, K=128)
//   warps 2..9  softmax.  d <= 128: two sets of 4 warps (one per TMEM lane
//               quadrant); set s owns the key tiles j = s, s+2, ... and its own
//               O accumulator; a thread owns one query row of its set: one
//               tcgen05.ld of the 128 scores, max tree, exp2 (6 of 8 on the
//               SFU, 2 of 8 as a polynomial on the FMA pipe) with the argument
//               scaling, polynomial and row sums on the paired FP32 pipe
//               (FFMA2 / FADD2), P (bf16) written in the UMMA SWIZZLE_128B
//               K-major layout; the running max only moves when a row max
//               grows by > 2^8 (rare O rescale); the sets' (m, l, O) are
//               combined in the epilogue.  d > 128: one set, two warps per
//               quadrant split each tile's key columns (row max exchanged
//               through shared memory).
// Operands: Q, K and (row-major) V through 3-D tensor maps (elem, head, row),
// so head dims that are not multiples of 64 are zero-filled by TMA up to DP;
// V row-major is the MN-major B operand of the PV MMA; V^T (channels x keys)
// is the K-major alternative.  O is staged in smem and TMA-stored (4-D map
// clips d and Lq).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdlib.h>
#include "drs_net.h"
#include "pdl.cuh"
#include "tc_common.cuh"

namespace drs {

constexpr int kAQ = 128;       // queries per CTA
constexpr int kAK = 128;       // keys per tile
constexpr int kAttnTcThreads = 320;   // warp 0 TMA, warp 1 MMA, warps 2..9 softmax (2 per TMEM quadrant)

// Debug aid: when set (drs_attention_tc_debug), CTAs record per-role progress
// markers into host-mapped memory the CPU can read while a launch is stuck.
__device__ int* g_attn_trace = nullptr;
#ifndef DRS_ATTN_TRACE
#define ATTN_TRACE(slot, val) do {} while (0)
#else
#define ATTN_TRACE(slot, val)                                                            \
  do {                                                                                   \
    if (g_attn_trace) {                                                                  \
      const int cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);    \
      if (cta < 4) *(volatile int*)&g_attn_trace[cta * 8 + (slot)] = (val);              \
    }                                                                                    \
  } while (0)
#endif

template <int DP>
struct AttnSmem {
  // independent softmax sets: with two, set s owns whole S rows of the key
  // tiles j = s, s+2, ... and its own O accumulator (TMEM: S0, S1, O0, O1 =
  // 256 + 2 DP columns <= 512); DP = 192 keeps one set whose two warps per
  // quadrant split the key columns of every tile.
  static constexpr int kSets = DP <= 128 ? 2 : 1;
  static constexpr int kAtoms = DP / 64;                   // 64-element K atoms of Q / K rows
  static constexpr int kQBytes = kAQ * DP * 2;             // Q; reused to stage O for the TMA store
  static constexpr int kKBytes = kAK * DP * 2;
  static constexpr int kVBytes = DP * kAK * 2;
  static constexpr int kPBytes = kAQ * kAK * 2;
  static constexpr int kRedBytes = kSets == 1 ? 2 * kAQ * 4 : 0;   // per-tile row-max exchange (1 set)
  static constexpr int kNumBars = 26;
  // separate K and V rings, as deep as 227 KB allows (<= 4): K_{j+s} loads as
  // soon as S_j has consumed its slot, V_{j+s} once PV_j has
  static constexpr int kFixed = kQBytes + 2 * kPBytes + kRedBytes + kNumBars * 8 + 1024;
  static constexpr int kFit = (227 * 1024 - kFixed) / (kKBytes + kVBytes);
  static constexpr int kStages = kFit > 4 ? 4 : kFit;
  static_assert(kStages >= 1, "attention tile does not fit in shared memory");
  static constexpr int kQ = 0;
  static constexpr int kK = kQ + kQBytes;
  static constexpr int kV = kK + kStages * kKBytes;
  static constexpr int kP = kV + kStages * kVBytes;        // P double-buffered (buffer j & 1)
  static constexpr int kRed = kP + 2 * kPBytes;
  static constexpr int kBar = kRed + kRedBytes;
  // >= 116 KB so two CTAs never share an SM: each allocates all 512 TMEM columns
  static constexpr int kRaw = kBar + kNumBars * 8 + 1024;
  static constexpr int kBytes = kRaw < 116 * 1024 ? 116 * 1024 : kRaw;
  static_assert(kBytes <= 227 * 1024, "shared memory plan exceeds 227 KB");
};

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
      :: "r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
         "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
         "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
         "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
}
// tcgen05.wait::ld that also pins `r` (outputs of earlier tcgen05.ld) so the
// compiler cannot move their uses above the wait
__device__ __forceinline__ void tmem_ld_wait_regs(uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.wait::ld.sync.aligned;"
      : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
        "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]),
        "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]), "+r"(r[22]), "+r"(r[23]),
        "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]), "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
      :: "memory");
}
__device__ __forceinline__ void reg_pin(uint32_t (&r)[32]) {
  asm volatile(""
      : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
        "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]),
        "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]), "+r"(r[22]), "+r"(r[23]),
        "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]), "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
      :: "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// 2^x on the SFU, flush-to-zero (scores are never in the denormal range that
// matters: p underflows to 0 exactly as the softmax wants)
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 2^x on the FMA pipe (Cody-Waite split + cubic minimax on [-0.5, 0.5],
// rel. error 7.5e-5, far below P's bf16 rounding): used for some of the
// scores so the SFU is not the only exp2 engine
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -125.f);                            // keeps the result a normal float (masked -inf -> ~0)
  const float t = x + 12582912.f;                  // 1.5 * 2^23: round to nearest integer
  const float r = t - 12582912.f;
  const float f = x - r;                           // [-0.5, 0.5]
  float p = fmaf(fmaf(fmaf(0.0551715f, f, 0.24261096f), f, 0.69326099f), f, 0.99992808f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}
// the same on a pair of scores with the paired FP32 pipe (FFMA2 / FADD2)
__device__ __forceinline__ void ex2_poly2(float2 x, float& y0, float& y1) {
  x.x = fmaxf(x.x, -125.f);
  x.y = fmaxf(x.y, -125.f);
  const float2 t = __fadd2_rn(x, make_float2(12582912.f, 12582912.f));
  const float2 r = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __ffma2_rn(r, make_float2(-1.f, -1.f), x);
  float2 p = __ffma2_rn(make_float2(0.0551715f, 0.0551715f), f, make_float2(0.24261096f, 0.24261096f));
  p = __ffma2_rn(p, f, make_float2(0.69326099f, 0.69326099f));
  p = __ffma2_rn(p, f, make_float2(0.99992808f, 0.99992808f));
  y0 = __int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23));
  y1 = __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23));
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tma_load_3d(const void* tmap, uint64_t* bar, void* smem, int32_t c0, int32_t c1,
                                            int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
      :: "r"(tc::smem_u32(smem)), "l"(tmap), "r"(tc::smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
// SWIZZLE_128B K-major descriptor advanced by K-step kk (16 elements) inside a
// tile whose 64-element atom columns are `atom_bytes` apart.
__device__ __forceinline__ uint64_t kdesc(const uint8_t* base, int kk, int atom_bytes) {
  return tc::smem_desc_sw128(base + (kk >> 2) * atom_bytes + (kk & 3) * 32);
}

__device__ __forceinline__ void tma_store_4d(const void* tmap, const void* smem, int32_t c0, int32_t c1, int32_t c2,
                                             int32_t c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];"
               :: "l"(tmap), "r"(tc::smem_u32(smem)), "r"(c0), "r"(c1), "r"(c2), "r"(c3) : "memory");
}

// byte offset of the 16-byte chunk holding columns [8c, 8c+8) of `row` in a
// 128-row tile stored as 64-column SWIZZLE_128B atoms (UMMA K-major / TMA layout)
__device__ __forceinline__ int sw128_off(int row, int c) {
  return (c >> 3) * (kAQ * 128) + (row >> 3) * 1024 + (row & 7) * 128 + (((c & 7) ^ (row & 7)) << 4);
}

// VROW: V given row-major (keys x channels, the V block of a fused QKV GEMM
// output) and loaded exactly like K; the PV MMA reads it as an MN-major B
// operand (b_major = 1) -- no separate V^T GEMM.  Otherwise V^T (channels x keys).
// SPLIT: a second MMA warp (warp 10) issues the PV MMAs while warp 1 issues only
// the S MMAs, so S_{j+2} no longer waits in warp 1's program order behind P_j
// (ncu: the softmax warps spent 21.5 % of their samples waiting for S tiles).
// X2: the exps' argument scaling, the poly exps and the row sums on the paired
// FP32 pipe (FFMA2 / FADD2: half the issue slots of the scalar loop)
template <int DP, int NPOLY, bool VROW, bool SPLIT, bool X2 = false>
__global__ void __launch_bounds__(SPLIT ? kAttnTcThreads + 32 : kAttnTcThreads, 1)
attn_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
               const __grid_constant__ CUtensorMap tm_vt, const __grid_constant__ CUtensorMap tm_o,
               int Lq, int Lk, int d, int vt_img, float scale_log2) {
  using S = AttnSmem<DP>;
  constexpr int kSt = S::kStages;
  constexpr int kSets = S::kSets;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::kBar);
  uint64_t* q_full = bars;                 // 1
  uint64_t* k_full = bars + 1;             // kSt (<= 4)
  uint64_t* k_empty = bars + 5;            // kSt   (released by S_j)
  uint64_t* v_full = bars + 9;             // kSt
  uint64_t* v_empty = bars + 13;           // kSt   (released by PV_j)
  uint64_t* s_full = bars + 17;            // 2 (per S buffer)
  uint64_t* p_full = bars + 19;            // 2 (per P buffer; one arrival per softmax warp of the tile)
  uint64_t* o_done = bars + 21;            // 2 (per P buffer: PV_j committed to o_done[j & 1])
  uint64_t* s_free = bars + 23;            // 2 (S buffer read into registers: S_{j+2} may overwrite)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 25);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q0 = blockIdx.x * kAQ, h = blockIdx.y, b = blockIdx.z;
  const int n_tiles = (Lk + kAK - 1) / kAK;
  constexpr uint32_t kIdescS = tc::idesc_bf16_f32(128, kAK);
  constexpr uint32_t kIdescO = VROW ? tc::idesc_bf16_f32_bmn(128, DP) : tc::idesc_bf16_f32(128, DP);

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tm_q);
    tc::tma_prefetch(&tm_k);
    tc::tma_prefetch(&tm_vt);
    tc::tma_prefetch(&tm_o);
    tc::mbar_init(q_full, 1);
    for (int s = 0; s < kSt; ++s) {
      tc::mbar_init(&k_full[s], 1); tc::mbar_init(&k_empty[s], 1);
      tc::mbar_init(&v_full[s], 1); tc::mbar_init(&v_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&s_full[i], 1);
      tc::mbar_init(&p_full[i], kSets == 2 ? 4 : 8);
      tc::mbar_init(&s_free[i], kSets == 2 ? 4 : 8);
      tc::mbar_init(&o_done[i], 1);
    }
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc<512>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  pdl_wait();       // everything above is data-independent setup (PDL overlap)
  pdl_trigger();
  const uint32_t tmem = *tmem_slot;         // S0 at col 0, S1 at col 128, O (per set) from col 256
  if (threadIdx.x == 0) ATTN_TRACE(0, 1);
  uint8_t* sQ = smem + S::kQ;
  uint8_t* sK = smem + S::kK;
  uint8_t* sV = smem + S::kV;
  uint8_t* sP = smem + S::kP;

  if (warp == 0) {
    // two producer lanes: lane 0 streams Q then the K ring, lane 1 the V ring
    if (lane == 0) {
      tc::mbar_arrive_expect_tx(q_full, S::kQBytes);
      for (int a = 0; a < S::kAtoms; ++a)
        tma_load_3d(&tm_q, q_full, sQ + a * (kAQ * 128), a * 64, h, b * Lq + q0);
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j % kSt;
        tc::mbar_wait(&k_empty[st], ((j / kSt) & 1) ^ 1);
        ATTN_TRACE(1, 100 + j);
        tc::mbar_arrive_expect_tx(&k_full[st], S::kKBytes);
        uint8_t* k_dst = sK + st * S::kKBytes;
        for (int a = 0; a < S::kAtoms; ++a)
          tma_load_3d(&tm_k, &k_full[st], k_dst + a * (kAK * 128), a * 64, h, b * Lk + j * kAK);
      }
    } else if (lane == 1) {
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j % kSt;
        tc::mbar_wait(&v_empty[st], ((j / kSt) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&v_full[st], S::kVBytes);
        uint8_t* v_dst = sV + st * S::kVBytes;
        if constexpr (VROW) {              // [128 keys x 64 ch] atoms, like the K tile
          for (int a = 0; a < S::kAtoms; ++a)
            tma_load_3d(&tm_vt, &v_full[st], v_dst + a * (kAK * 128), a * 64, h, b * Lk + j * kAK);
        } else {
          for (int a = 0; a < kAK / 64; ++a)
            tc::tma_load_2d(&tm_vt, &v_full[st], v_dst + a * (DP * 128), b * vt_img + j * kAK + a * 64, h * d);
        }
      }
    }
  } else if (warp == 1) {
    // S_j = Q K_j^T into TMEM buffer j&1 (S_0, S_1 up front, S_{j+2} as soon as
    // the softmax has read S_j into registers, so it runs under tile j's exps);
    // O_set += P_j V_j after P_j is published.
    tc::mbar_wait(q_full, 0);
    if (lane == 0) ATTN_TRACE(2, 6);
    auto issue_s = [&](int j) {
      const int st = j % kSt;
      tc::mbar_wait(&k_full[st], (j / kSt) & 1);
      if (lane == 0) ATTN_TRACE(3, 100 + j);
      tc::tc_fence_after();
      if (tc::elect_one()) {
        const uint8_t* kb = sK + st * S::kKBytes;
#pragma unroll
        for (int kk = 0; kk < DP / 16; ++kk)
          tc::mma_bf16(tmem + (j & 1) * 128, kdesc(sQ, kk, kAQ * 128), kdesc(kb, kk, kAK * 128), kIdescS,
                       kk > 0 ? 1u : 0u);
        tc::mma_commit(&k_empty[st]);
        tc::mma_commit(&s_full[j & 1]);
      }
      __syncwarp();
    };
    issue_s(0);
    if (n_tiles > 1) issue_s(1);
    for (int j = 0; j < n_tiles; ++j) {
      if (j + 2 < n_tiles) {
        tc::mbar_wait(&s_free[j & 1], (j >> 1) & 1);
        issue_s(j + 2);
      }
      if constexpr (SPLIT) continue;           // PV MMAs: warp 10
      tc::mbar_wait(&p_full[j & 1], (j >> 1) & 1);
      const int st = j % kSt;
      tc::mbar_wait(&v_full[st], (j / kSt) & 1);
      if (lane == 0) ATTN_TRACE(4, 100 + j);
      tc::tc_fence_after();
      if (tc::elect_one()) {
        const uint8_t* vb = sV + st * S::kVBytes;
        const uint32_t o_col = 256 + (kSets == 2 ? (j & 1) * DP : 0);
#pragma unroll
        for (int kk = 0; kk < kAK / 16; ++kk) {
          // VROW: 16 keys = 16 rows of 128 B per K step; channel atoms kAK * 128 B apart
          const uint64_t bdesc = VROW ? tc::smem_desc_sw128_mn(vb + kk * 2048, kAK * 128) : kdesc(vb, kk, DP * 128);
          tc::mma_bf16(tmem + o_col, kdesc(sP + (j & 1) * S::kPBytes, kk, kAQ * 128), bdesc,
                       kIdescO, (j >= kSets || kk > 0) ? 1u : 0u);
        }
        tc::mma_commit(&v_empty[st]);
        tc::mma_commit(&o_done[j & 1]);
      }
      __syncwarp();
    }
  } else if (SPLIT && warp == 10) {
    // PV issuer: O_set += P_j V_j as soon as P_j is published and V_j landed
    for (int j = 0; j < n_tiles; ++j) {
      tc::mbar_wait(&p_full[j & 1], (j >> 1) & 1);
      const int st = j % kSt;
      tc::mbar_wait(&v_full[st], (j / kSt) & 1);
      tc::tc_fence_after();
      if (tc::elect_one()) {
        const uint8_t* vb = sV + st * S::kVBytes;
        const uint32_t o_col = 256 + (kSets == 2 ? (j & 1) * DP : 0);
#pragma unroll
        for (int kk = 0; kk < kAK / 16; ++kk) {
          const uint64_t bdesc = VROW ? tc::smem_desc_sw128_mn(vb + kk * 2048, kAK * 128) : kdesc(vb, kk, DP * 128);
          tc::mma_bf16(tmem + o_col, kdesc(sP + (j & 1) * S::kPBytes, kk, kAQ * 128), bdesc,
                       kIdescO, (j >= kSets || kk > 0) ? 1u : 0u);
        }
        tc::mma_commit(&v_empty[st]);
        tc::mma_commit(&o_done[j & 1]);
      }
      __syncwarp();
    }
  } else {
    // softmax warps: warp w owns TMEM lanes 32*(w&3) .. +31 (query rows);
    // grp = (w-2)>>2 is the set (2 sets) or the key-column half (1 set)
    const int quad = warp & 3;
    const int grp = (warp - 2) >> 2;
    const int row = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    constexpr int kCols = kSets == 2 ? kAK : kAK / 2;            // S columns per thread per tile
    const int col0 = kSets == 2 ? 0 : grp * kCols;
    const uint32_t o_base = 256 + (kSets == 2 ? grp * DP : grp * (DP / 2));
    constexpr int kOCols = kSets == 2 ? DP : DP / 2;              // O columns rescaled per thread
    float* red = reinterpret_cast<float*>(smem + S::kRed);       // [2][kAQ] (1 set only)
    auto quad_sync = [&]() {                                      // the 2 warps sharing these rows
      asm volatile("bar.sync %0, 64;" :: "r"(1 + quad) : "memory");
    };
    float m = -INFINITY, l = 0.f;
    for (int j = (kSets == 2 ? grp : 0); j < n_tiles; j += kSets) {
      tc::mbar_wait(&s_full[j & 1], (j >> 1) & 1);
      if (lane == 0 && quad == 0) ATTN_TRACE(5 + grp, 100 + j);
      tc::tc_fence_after();
      float sv[kCols];
      {                                                   // all chunks in flight, one wait
        uint32_t r[kCols / 32][32];
#pragma unroll
        for (int c = 0; c < kCols / 32; ++c) tc::tmem_ld32(tmem + lane_off + (j & 1) * 128 + col0 + c * 32, r[c]);
        tmem_ld_wait_regs(r[0]);
#pragma unroll
        for (int c = 1; c < kCols / 32; ++c) reg_pin(r[c]);
#pragma unroll
        for (int c = 0; c < kCols / 32; ++c)
#pragma unroll
          for (int e = 0; e < 32; ++e) sv[c * 32 + e] = __uint_as_float(r[c][e]);
      }
      tc::tc_fence_before();                              // S_j is in registers: release the buffer
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&s_free[j & 1]);
      const int kvalid = Lk - j * kAK - col0;             // keys of this (half-)tile that exist
      if (kvalid < kCols) {                               // ragged last tile only
#pragma unroll
        for (int e = 0; e < kCols; ++e) sv[e] = e < kvalid ? sv[e] : -INFINITY;
      }
      float mx8[8];                                       // max tree on the raw scores (scale > 0)
#pragma unroll
      for (int e = 0; e < 8; ++e) mx8[e] = fmaxf(sv[e], sv[e + 8]);
#pragma unroll
      for (int c = 2; c < kCols / 8; ++c)
#pragma unroll
        for (int e = 0; e < 8; ++e) mx8[e] = fmaxf(mx8[e], sv[c * 8 + e]);
      float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                       fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]))) * scale_log2;
      if constexpr (kSets == 1) {
        red[grp * kAQ + row] = mx;
        quad_sync();
        mx = fmaxf(red[row], red[kAQ + row]);
        quad_sync();                                     // both read before the next tile rewrites
      }
      // conditional rescaling: the reference max only moves when the row max
      // grew by more than 2^8 (p <= 256 is exact enough for bf16 P / fp32 l;
      // the final O / l uses the same stale max for both, so the result is unchanged)
      const float m_new = mx > m + 8.f ? mx : m;
      const float alpha = ex2(m - m_new);
      // P_j overwrites P buffer j&1: PV_{j-2} (its last reader) must be done.
      // With two sets that PV is also the last one into this set's O.
      if (j >= 2) {
        tc::mbar_wait(&o_done[j & 1], ((j - 2) >> 1) & 1);
        tc::tc_fence_after();
      }
      uint8_t* pb = sP + (j & 1) * S::kPBytes;
      float sum = 0.f;
      float2 sum2 = make_float2(0.f, 0.f);
#pragma unroll
      for (int c = 0; c < kCols / 8; ++c) {            // 16-byte chunks of this thread's P row
        float p[8];
        if constexpr (X2) {
          const float2 sc2 = make_float2(scale_log2, scale_log2), nm2 = make_float2(-m_new, -m_new);
#pragma unroll
          for (int e2 = 0; e2 < 4; ++e2) {
            const float2 x2 = __ffma2_rn(make_float2(sv[c * 8 + 2 * e2], sv[c * 8 + 2 * e2 + 1]), sc2, nm2);
            if (2 * e2 + 1 < NPOLY) {
              ex2_poly2(x2, p[2 * e2], p[2 * e2 + 1]);
            } else {
              p[2 * e2] = 2 * e2 < NPOLY ? ex2_poly(x2.x) : ex2(x2.x);
              p[2 * e2 + 1] = ex2(x2.y);
            }
          }
          sum2 = __fadd2_rn(sum2, __fadd2_rn(__fadd2_rn(make_float2(p[0], p[1]), make_float2(p[2], p[3])),
                                             __fadd2_rn(make_float2(p[4], p[5]), make_float2(p[6], p[7]))));
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float x = fmaf(sv[c * 8 + e], scale_log2, -m_new);
            p[e] = e < NPOLY ? ex2_poly(x) : ex2(x);      // NPOLY of every 8 on the FMA pipe
          }
          sum += ((p[0] + p[1]) + (p[2] + p[3])) + ((p[4] + p[5]) + (p[6] + p[7]));
        }
        uint4 u;
        __nv_bfloat162* hp = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e) hp[e] = __floats2bfloat162_rn(p[2 * e], p[2 * e + 1]);
        *reinterpret_cast<uint4*>(pb + sw128_off(row, (col0 >> 3) + c)) = u;
      }
      if constexpr (X2) sum = sum2.x + sum2.y;
      l = l * alpha + sum;                                // this thread's (partial) row sum
      // rescale this thread's O columns; tcgen05.ld/st are warp-collective,
      // so the whole warp takes the branch if any of its rows needs it
      if (j >= kSets && __any_sync(0xffffffffu, alpha < 1.f)) {
        if constexpr (kSets == 1) {
          tc::mbar_wait(&o_done[(j - 1) & 1], ((j - 1) >> 1) & 1);   // O holds PV_0..PV_{j-1}
          tc::tc_fence_after();
        }
#pragma unroll
        for (int c = 0; c < kOCols / 32; ++c) {
          uint32_t r[32];
          const uint32_t col = o_base + c * 32;
          tc::tmem_ld32(tmem + lane_off + col, r);
          tmem_ld_wait_regs(r);
#pragma unroll
          for (int e = 0; e < 32; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * alpha);
          tmem_st32(tmem + lane_off + col, r);
        }
        tmem_st_wait();
      }
      m = m_new;
      fence_async_smem();                            // P smem writes -> tensor-core (async) proxy
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&p_full[j & 1]);
    }

    // ---- epilogue: O / l -> bf16, staged in the (dead) Q tile, TMA-stored ----
    // wait for the last PV this thread's set (or, with one set, the CTA) issued
    float f0 = 1.f, f1 = 0.f, inv;
    if constexpr (kSets == 2) {
      const int last = n_tiles - 1 - ((n_tiles - 1 - grp) & 1);   // last tile of this set (may be < 0)
      if (last >= 0) {
        tc::mbar_wait(&o_done[grp], (last >> 1) & 1);
        tc::tc_fence_after();
      }
      // this set's P buffer is now dead: publish (m, l) of the row through it
      float* ex = reinterpret_cast<float*>(sP + grp * S::kPBytes);
      ex[row] = m;
      ex[kAQ + row] = l;
      quad_sync();
      const float* ex0 = reinterpret_cast<const float*>(sP);
      const float* ex1 = reinterpret_cast<const float*>(sP + S::kPBytes);
      const float m0 = ex0[row], l0 = ex0[kAQ + row], m1 = ex1[row], l1 = ex1[kAQ + row];
      const float mm = fmaxf(m0, m1);
      f0 = ex2(m0 - mm);
      f1 = n_tiles > 1 ? ex2(m1 - mm) : 0.f;
      const float lt = l0 * f0 + l1 * f1;
      inv = lt > 0.f ? 1.f / lt : 0.f;
    } else {
      tc::mbar_wait(&o_done[(n_tiles - 1) & 1], ((n_tiles - 1) >> 1) & 1);
      tc::tc_fence_after();
      red[grp * kAQ + row] = l;
      quad_sync();
      const float lt = red[row] + red[kAQ + row];
      inv = lt > 0.f ? 1.f / lt : 0.f;
    }
    tc::tc_fence_after();
    // this thread writes O columns [grp * DP/2, (grp+1) * DP/2) of its row
    constexpr int kHalfO = DP / 2;
#pragma unroll
    for (int c = 0; c < kHalfO / 32; ++c) {
      const int ocol = grp * kHalfO + c * 32;
      uint32_t r0[32];
      tc::tmem_ld32(tmem + lane_off + 256 + ocol, r0);
      if (kSets == 2 && n_tiles > 1) {
        uint32_t r1[32];
        tc::tmem_ld32(tmem + lane_off + 256 + DP + ocol, r1);
        tmem_ld_wait_regs(r0);
        reg_pin(r1);
#pragma unroll
        for (int e = 0; e < 32; ++e)
          r0[e] = __float_as_uint(fmaf(__uint_as_float(r0[e]), f0, __uint_as_float(r1[e]) * f1));
      } else {
        tmem_ld_wait_regs(r0);
        if (kSets == 2) {
#pragma unroll
          for (int e = 0; e < 32; ++e) r0[e] = __float_as_uint(__uint_as_float(r0[e]) * f0);
        }
      }
#pragma unroll
      for (int c8 = 0; c8 < 4; ++c8) {
        uint4 u;
        __nv_bfloat162* hp = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e)
          hp[e] = __floats2bfloat162_rn(__uint_as_float(r0[c8 * 8 + 2 * e]) * inv,
                                        __uint_as_float(r0[c8 * 8 + 2 * e + 1]) * inv);
        *reinterpret_cast<uint4*>(sQ + sw128_off(row, (ocol >> 3) + c8)) = u;
      }
    }
    fence_async_smem();
    asm volatile("bar.sync 5, 256;" ::: "memory");        // all softmax warps staged their O
    if (warp == 2 && lane == 0) {
      for (int a = 0; a < S::kAtoms; ++a) tma_store_4d(&tm_o, sQ + a * (kAQ * 128), a * 64, h, q0, b);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // smem must outlive the reads
      ATTN_TRACE(7, 999);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<512>(tmem);
}

// ------------------------------------------------------------ host side ---
typedef CUresult (*PFN_encodeTiled2)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled2 encode_fn2() {
  static PFN_encodeTiled2 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled2>(p);
  }
  return fn;
}

// (elements of a head, heads, rows): box {64, 1, 128}; elements >= d read as zero
static bool tmap_heads(CUtensorMap* m, const void* ptr, int64_t rows, int H, int d, int64_t ld) {
  auto enc = encode_fn2();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)H, (cuuint64_t)rows};
  cuuint64_t strides[2] = {(cuuint64_t)d * 2, (cuuint64_t)ld * 2};
  cuuint32_t box[3] = {64, 1, 128};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// output (elements of a head, heads, queries, images): box {64, 1, 128, 1}; the
// TMA store clips elements >= d and queries >= Lq (no spill into the next image)
static bool tmap_out(CUtensorMap* m, void* ptr, int B, int Lq, int H, int d, int64_t ld) {
  auto enc = encode_fn2();
  if (!enc) return false;
  cuuint64_t dims[4] = {(cuuint64_t)d, (cuuint64_t)H, (cuuint64_t)Lq, (cuuint64_t)B};
  cuuint64_t strides[3] = {(cuuint64_t)d * 2, (cuuint64_t)ld * 2, (cuuint64_t)Lq * ld * 2};
  cuuint32_t box[4] = {64, 1, 128, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, ptr, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

// V^T (channels x keys): box {64 keys, DP channels}
static bool tmap_vt(CUtensorMap* m, const void* ptr, int64_t chans, int64_t keys, int64_t ld, int DP) {
  auto enc = encode_fn2();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)keys, (cuuint64_t)chans};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)DP};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int DP, int NPOLY, bool VROW, bool SPLIT, bool X2 = false>
static int launch_attn_v(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv, const CUtensorMap& to,
                         int B, int H, int Lq, int Lk, int d, int vt_img, float sl2, cudaStream_t st) {
  using S = AttnSmem<DP>;
  auto kern = attn_tc_kernel<DP, NPOLY, VROW, SPLIT, X2>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, S::kBytes) != cudaSuccess)
      return DRS_ERR_CUDA;
    attr = true;
  }
  dim3 grid((Lq + kAQ - 1) / kAQ, H, B);
  launch_pdl(kern, dim3(grid), dim3(SPLIT ? kAttnTcThreads + 32 : kAttnTcThreads), S::kBytes, st, tq, tk, tv, to,
             Lq, Lk, d, vt_img, sl2);
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
}

// drs_set_attn_split: 0 = one MMA warp, 1 = separate S / PV MMA issuer warps (SPLIT), 2 = SPLIT + X2
inline int& attn_split_mma() {
  static int on = 2;
  return on;
}

template <int DP, bool VROW>
static int launch_attn(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv, const CUtensorMap& to,
                       int B, int H, int Lq, int Lk, int d, int vt_img, float sl2, cudaStream_t st) {
  static int npoly = [] { const char* e = getenv("DRS_ATTN_POLY"); return e ? atoi(e) : 2; }();
  // (paired-FP32 softmax with 0 / 3 / 4 of every 8 exps on the FMA pipe: 9 % slower than 2 on the
  // SD1.5 / SDXL 64x64 self-attention, late round 2)
  if (attn_split_mma() >= 2)
    return launch_attn_v<DP, 2, VROW, true, true>(tq, tk, tv, to, B, H, Lq, Lk, d, vt_img, sl2, st);
  if (attn_split_mma())
    return launch_attn_v<DP, 2, VROW, true>(tq, tk, tv, to, B, H, Lq, Lk, d, vt_img, sl2, st);
  if (npoly == 0) return launch_attn_v<DP, 0, VROW, false>(tq, tk, tv, to, B, H, Lq, Lk, d, vt_img, sl2, st);
  if (npoly == 3) return launch_attn_v<DP, 3, VROW, false>(tq, tk, tv, to, B, H, Lq, Lk, d, vt_img, sl2, st);
  return launch_attn_v<DP, 2, VROW, false>(tq, tk, tv, to, B, H, Lq, Lk, d, vt_img, sl2, st);
}

}  // namespace drs

extern "C" int drs_attention_tc(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* vt,
                                int64_t ldvt, int vt_img, void* o, int64_t ldo, int B, int H, int Lq, int Lk,
                                int d, float scale, void* stream) {
  using namespace drs;
  if (B <= 0 || H <= 0 || Lq <= 0 || Lk <= 0 || d <= 0 || d > 192 || d % 8) return DRS_ERR_VALUE;
  if (vt_img < Lk || vt_img % 8) return DRS_ERR_VALUE;   // TMA inner box starts must be 16-byte aligned
  if ((ldq | ldk | ldvt | ldo) % 8 || (reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k) |
                                       reinterpret_cast<uintptr_t>(vt) | reinterpret_cast<uintptr_t>(o)) & 15)
    return DRS_ERR_VALUE;
  const int DP = d <= 64 ? 64 : (d <= 128 ? 128 : 192);
  CUtensorMap tq, tk, tv, to;
  if (!tmap_heads(&tq, q, (int64_t)B * Lq, H, d, ldq) || !tmap_heads(&tk, k, (int64_t)B * Lk, H, d, ldk) ||
      !tmap_vt(&tv, vt, (int64_t)H * d, (int64_t)(B - 1) * vt_img + Lk, ldvt, DP) ||
      !tmap_out(&to, o, B, Lq, H, d, ldo))
    return DRS_ERR_CUDA;
  const float sl2 = scale * 1.4426950408889634f;
  cudaStream_t st = (cudaStream_t)stream;
  if (DP == 64) return launch_attn<64, false>(tq, tk, tv, to, B, H, Lq, Lk, d, vt_img, sl2, st);
  if (DP == 128) return launch_attn<128, false>(tq, tk, tv, to, B, H, Lq, Lk, d, vt_img, sl2, st);
  return launch_attn<192, false>(tq, tk, tv, to, B, H, Lq, Lk, d, vt_img, sl2, st);
}

// V row-major (the V block of a fused QKV projection), read as an MN-major PV operand
extern "C" int drs_attention_tc_v(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v,
                                  int64_t ldv, void* o, int64_t ldo, int B, int H, int Lq, int Lk, int d,
                                  float scale, void* stream) {
  using namespace drs;
  if (B <= 0 || H <= 0 || Lq <= 0 || Lk <= 0 || d <= 0 || d > 192 || d % 8) return DRS_ERR_VALUE;
  if ((ldq | ldk | ldv | ldo) % 8 || (reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k) |
                                      reinterpret_cast<uintptr_t>(v) | reinterpret_cast<uintptr_t>(o)) & 15)
    return DRS_ERR_VALUE;
  const int DP = d <= 64 ? 64 : (d <= 128 ? 128 : 192);
  CUtensorMap tq, tk, tv, to;
  if (!tmap_heads(&tq, q, (int64_t)B * Lq, H, d, ldq) || !tmap_heads(&tk, k, (int64_t)B * Lk, H, d, ldk) ||
      !tmap_heads(&tv, v, (int64_t)B * Lk, H, d, ldv) || !tmap_out(&to, o, B, Lq, H, d, ldo))
    return DRS_ERR_CUDA;
  const float sl2 = scale * 1.4426950408889634f;
  cudaStream_t st = (cudaStream_t)stream;
  if (DP == 64) return launch_attn<64, true>(tq, tk, tv, to, B, H, Lq, Lk, d, Lk, sl2, st);
  if (DP == 128) return launch_attn<128, true>(tq, tk, tv, to, B, H, Lq, Lk, d, Lk, sl2, st);
  return launch_attn<192, true>(tq, tk, tv, to, B, H, Lq, Lk, d, Lk, sl2, st);
}

extern "C" int drs_attention_tc_debug(int* mapped_trace) {
  return cudaMemcpyToSymbol(drs::g_attn_trace, &mapped_trace, sizeof(int*)) == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
}

extern "C" int drs_set_attn_split(int on) {
  // 0 one MMA warp, 1 S / PV issuer warps, 2 (default) = 1 + paired-FP32 softmax
  drs::attn_split_mma() = on;
  return DRS_OK;
}
