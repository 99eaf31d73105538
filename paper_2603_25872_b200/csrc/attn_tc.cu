// K6: fused attention forward on the 5th-gen tensor cores (non-causal).
//
//   O[b, q, h, :] = softmax_k( Q[b, q, h, :] . K[b, k, h, :] * scale ) V[b, k, h, :]
//
// One CTA per (128-query tile, head, batch).  Warp roles (192 threads):
//   warp 0      TMA producer: Q once, then K / V^T tiles of 128 keys into a
//               kStages ring (mbarrier full/empty)
//   warp 1      TMEM allocator + MMA issuer:  S_j = Q K_j^T   (M=128, N=128, K=DP)
//               into one of two TMEM S buffers, then O += P_j V_j (M=128, N=DP,
//               K=128) into the TMEM O accumulator
//   warps 2..9  softmax, two warps per TMEM lane quadrant: a query row (TMEM
//               lane) is shared by two threads that each own 64 of the 128 key
//               columns (and half of the O columns): tcgen05.ld their half of S,
//               exchange the row max through shared memory, exp2 / partial sums,
//               rescale their half of the O row only when the running max moved,
//               write their half of P (bf16) in the UMMA SWIZZLE_128B K-major
//               layout; the partial row sums are combined once, in the epilogue.
// Operands: Q and K through 3-D tensor maps (elem, head, row) so head dims that
// are not multiples of 64 are zero-filled by TMA up to DP; V is consumed as V^T
// (channels x keys, keys contiguous -- produced directly by a swapped-operand
// GEMM), so every UMMA operand is K-major with the same descriptors as K4.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
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
  static constexpr int kStages = DP <= 128 ? 2 : 1;
  static constexpr int kAtoms = DP / 64;                   // 64-element K atoms of Q / K rows
  static constexpr int kQBytes = kAQ * DP * 2;
  static constexpr int kKBytes = kAK * DP * 2;
  static constexpr int kVBytes = DP * kAK * 2;
  static constexpr int kPBytes = kAQ * kAK * 2;
  static constexpr int kQ = 0;
  static constexpr int kK = kQ + kQBytes;
  static constexpr int kV = kK + kStages * kKBytes;
  static constexpr int kP = kV + kStages * kVBytes;
  static constexpr int kRed = kP + kPBytes;                // [2 halves][128 rows] float row maxima / sums
  static constexpr int kBar = kRed + 2 * kAQ * 4;
  // >= 116 KB so two CTAs never share an SM: each allocates all 512 TMEM columns
  static constexpr int kRaw = kBar + 16 * 8 + 16 + 1024;
  static constexpr int kBytes = kRaw < 116 * 1024 ? 116 * 1024 : kRaw;
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
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
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

template <int DP>
__global__ void __launch_bounds__(kAttnTcThreads, 1)
attn_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
               const __grid_constant__ CUtensorMap tm_vt, __nv_bfloat16* __restrict__ o, int64_t ldo,
               int Lq, int Lk, int d, int vt_img, float scale_log2) {
  using S = AttnSmem<DP>;
  constexpr int kSt = S::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::kBar);
  uint64_t* q_full = bars;                 // 1
  uint64_t* kv_full = bars + 1;            // kSt
  uint64_t* kv_empty = bars + 3;           // kSt
  uint64_t* s_full = bars + 5;             // 2 (per S buffer)
  uint64_t* p_full = bars + 7;             // 1 (count 8: softmax warps)
  uint64_t* o_done = bars + 8;             // 1
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 10);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q0 = blockIdx.x * kAQ, h = blockIdx.y, b = blockIdx.z;
  const int n_tiles = (Lk + kAK - 1) / kAK;
  constexpr uint32_t kIdescS = tc::idesc_bf16_f32(128, kAK);
  constexpr uint32_t kIdescO = tc::idesc_bf16_f32(128, DP);

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tm_q);
    tc::tma_prefetch(&tm_k);
    tc::tma_prefetch(&tm_vt);
    tc::mbar_init(q_full, 1);
    for (int s = 0; s < kSt; ++s) { tc::mbar_init(&kv_full[s], 1); tc::mbar_init(&kv_empty[s], 1); }
    tc::mbar_init(&s_full[0], 1);
    tc::mbar_init(&s_full[1], 1);
    tc::mbar_init(p_full, 8);
    tc::mbar_init(o_done, 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc<512>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  pdl_wait();       // everything above is data-independent setup (PDL overlap)
  pdl_trigger();
  const uint32_t tmem = *tmem_slot;         // S0 at col 0, S1 at col 128, O at col 256
  if (threadIdx.x == 0) ATTN_TRACE(0, 1);
  uint8_t* sQ = smem + S::kQ;
  uint8_t* sK = smem + S::kK;
  uint8_t* sV = smem + S::kV;
  uint8_t* sP = smem + S::kP;

  if (warp == 0) {
    if (tc::elect_one()) {
      tc::mbar_arrive_expect_tx(q_full, S::kQBytes);
      for (int a = 0; a < S::kAtoms; ++a)
        tma_load_3d(&tm_q, q_full, sQ + a * (kAQ * 128), a * 64, h, b * Lq + q0);
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j % kSt;
        const uint32_t ph = (j / kSt) & 1;
        tc::mbar_wait(&kv_empty[st], ph ^ 1);
        ATTN_TRACE(1, 100 + j);
        tc::mbar_arrive_expect_tx(&kv_full[st], S::kKBytes + S::kVBytes);
        uint8_t* k_dst = sK + st * S::kKBytes;
        uint8_t* v_dst = sV + st * S::kVBytes;
        for (int a = 0; a < S::kAtoms; ++a)
          tma_load_3d(&tm_k, &kv_full[st], k_dst + a * (kAK * 128), a * 64, h, b * Lk + j * kAK);
        for (int a = 0; a < kAK / 64; ++a)
          tc::tma_load_2d(&tm_vt, &kv_full[st], v_dst + a * (DP * 128), b * vt_img + j * kAK + a * 64, h * d);
      }
    }
  } else if (warp == 1) {
    // S_j = Q K_j^T into TMEM buffer j&1; O += P_j V_j after the softmax publishes P_j.
    if (lane == 0) ATTN_TRACE(2, 5);
    tc::mbar_wait(q_full, 0);
    if (lane == 0) ATTN_TRACE(2, 6);
    auto issue_s = [&](int j) {
      const int st = j % kSt;
      tc::mbar_wait(&kv_full[st], (j / kSt) & 1);
      if (lane == 0) ATTN_TRACE(3, 100 + j);
      tc::tc_fence_after();
      if (tc::elect_one()) {
        const uint8_t* kb = sK + st * S::kKBytes;
#pragma unroll
        for (int kk = 0; kk < DP / 16; ++kk)
          tc::mma_bf16(tmem + (j & 1) * 128, kdesc(sQ, kk, kAQ * 128), kdesc(kb, kk, kAK * 128), kIdescS,
                       kk > 0 ? 1u : 0u);
        tc::mma_commit(&s_full[j & 1]);
      }
      __syncwarp();
    };
    issue_s(0);
    for (int j = 0; j < n_tiles; ++j) {
      // with a 2-deep K/V ring S_{j+1} overlaps the softmax of tile j; with one
      // stage it must wait until PV_j has released the ring slot
      if (kSt > 1 && j + 1 < n_tiles) issue_s(j + 1);
      tc::mbar_wait(p_full, j & 1);
      if (lane == 0) ATTN_TRACE(4, 100 + j);
      tc::tc_fence_after();
      if (tc::elect_one()) {
        const int st = j % kSt;
        const uint8_t* vb = sV + st * S::kVBytes;
#pragma unroll
        for (int kk = 0; kk < kAK / 16; ++kk)
          tc::mma_bf16(tmem + 256, kdesc(sP, kk, kAQ * 128), kdesc(vb, kk, DP * 128), kIdescO,
                       (j > 0 || kk > 0) ? 1u : 0u);
        tc::mma_commit(&kv_empty[st]);
        tc::mma_commit(o_done);
      }
      __syncwarp();
      if (kSt == 1 && j + 1 < n_tiles) issue_s(j + 1);
    }
  } else {
    // softmax warps: warp w owns TMEM lanes 32*(w&3) .. +31 (query rows) and
    // the half (w-2)>>2 of the key columns / O columns of those rows
    const int quad = warp & 3;
    const int half = (warp - 2) >> 2;
    const int row = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    float* red = reinterpret_cast<float*>(smem + S::kRed);      // [2][kAQ]
    constexpr int kHalfK = kAK / 2;                              // 64 key columns per thread
    constexpr int kHalfO = DP / 2;                               // O columns per thread
    auto quad_sync = [&]() {                                      // the 2 warps sharing these rows
      asm volatile("bar.sync %0, 64;" :: "r"(1 + quad) : "memory");
    };
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < n_tiles; ++j) {
      tc::mbar_wait(&s_full[j & 1], (j >> 1) & 1);
      if (lane == 0 && quad == 0 && half == 0) ATTN_TRACE(5, 100 + j);
      tc::tc_fence_after();
      float sv[kHalfK];
#pragma unroll
      for (int c = 0; c < kHalfK / 32; ++c) {
        uint32_t r[32];
        tc::tmem_ld32(tmem + lane_off + (j & 1) * 128 + half * kHalfK + c * 32, r);
        tc::tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) sv[c * 32 + e] = __uint_as_float(r[e]);
      }
      const int kvalid = Lk - j * kAK - half * kHalfK;   // keys of this half-tile that exist
      float mx = -INFINITY;
#pragma unroll
      for (int e = 0; e < kHalfK; ++e) {
        sv[e] = e < kvalid ? sv[e] * scale_log2 : -INFINITY;
        mx = fmaxf(mx, sv[e]);
      }
      red[half * kAQ + row] = mx;
      quad_sync();
      mx = fmaxf(red[row], red[kAQ + row]);
      quad_sync();                                       // both read before the next tile rewrites
      const float m_new = fmaxf(m, mx);
      const float alpha = exp2f(m - m_new);
      float sum = 0.f;
      // P_j overwrites the P buffer and O may be rescaled: PV_{j-1} must be done
      if (j > 0) {
        tc::mbar_wait(o_done, (j - 1) & 1);
        tc::tc_fence_after();
      }
      if (lane == 0 && quad == 0 && half == 0) ATTN_TRACE(6, 100 + j);
#pragma unroll
      for (int c = 0; c < kHalfK / 8; ++c) {            // 16-byte chunks of this half of the P row
        float p[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          p[e] = exp2f(sv[c * 8 + e] - m_new);
          sum += p[e];
        }
        uint4 u;
        __nv_bfloat162* hp = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e) hp[e] = __floats2bfloat162_rn(p[2 * e], p[2 * e + 1]);
        // this half is atom column `half` of the K-major P tile
        uint8_t* dst = sP + half * (kAQ * 128) + (row >> 3) * 1024 + (row & 7) * 128 + ((c ^ (row & 7)) << 4);
        *reinterpret_cast<uint4*>(dst) = u;
      }
      l = l * alpha + sum;                                // partial (this half's keys) row sum
      // rescale this thread's half of the O row; tcgen05.ld/st are warp-collective,
      // so the whole warp takes the branch if any of its rows needs it
      if (j > 0 && __any_sync(0xffffffffu, alpha < 1.f)) {
#pragma unroll
        for (int c = 0; c < kHalfO / 32; ++c) {
          uint32_t r[32];
          const uint32_t col = 256 + half * kHalfO + c * 32;
          tc::tmem_ld32(tmem + lane_off + col, r);
          tc::tmem_ld_wait();
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
      if (lane == 0) tc::mbar_arrive(p_full);
    }
    red[half * kAQ + row] = l;
    quad_sync();
    const float lt = red[row] + red[kAQ + row];
    tc::mbar_wait(o_done, (n_tiles - 1) & 1);
    if (lane == 0 && quad == 0 && half == 0) ATTN_TRACE(7, 999);
    tc::tc_fence_after();
    const float inv = lt > 0.f ? 1.f / lt : 0.f;
    const int qrow = q0 + row;
    __nv_bfloat16* orow = o + ((int64_t)b * Lq + qrow) * ldo + (int64_t)h * d;
#pragma unroll
    for (int c = 0; c < kHalfO / 32; ++c) {
      uint32_t r[32];
      tc::tmem_ld32(tmem + lane_off + 256 + half * kHalfO + c * 32, r);
      tc::tmem_ld_wait();
      if (qrow < Lq) {
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          const int col = half * kHalfO + c * 32 + e;
          if (col < d)
            *reinterpret_cast<__nv_bfloat162*>(orow + col) =
                __floats2bfloat162_rn(__uint_as_float(r[e]) * inv, __uint_as_float(r[e + 1]) * inv);
        }
      }
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

template <int DP>
static int launch_attn(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv, void* o, int64_t ldo,
                       int B, int H, int Lq, int Lk, int d, int vt_img, float sl2, cudaStream_t st) {
  using S = AttnSmem<DP>;
  auto kern = attn_tc_kernel<DP>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, S::kBytes) != cudaSuccess)
      return DRS_ERR_CUDA;
    attr = true;
  }
  dim3 grid((Lq + kAQ - 1) / kAQ, H, B);
  launch_pdl(kern, dim3(grid), dim3(kAttnTcThreads), S::kBytes, st, tq, tk, tv, static_cast<__nv_bfloat16*>(o), ldo, Lq, Lk, d, vt_img,
                                                sl2);
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
}

}  // namespace drs

extern "C" int drs_attention_tc(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* vt,
                                int64_t ldvt, int vt_img, void* o, int64_t ldo, int B, int H, int Lq, int Lk,
                                int d, float scale, void* stream) {
  using namespace drs;
  if (B <= 0 || H <= 0 || Lq <= 0 || Lk <= 0 || d <= 0 || d > 192 || d % 8) return DRS_ERR_VALUE;
  if (vt_img < Lk || vt_img % 8) return DRS_ERR_VALUE;   // TMA inner box starts must be 16-byte aligned
  if ((ldq | ldk | ldvt) % 8 || (reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k) |
                                 reinterpret_cast<uintptr_t>(vt)) & 15)
    return DRS_ERR_VALUE;
  const int DP = d <= 64 ? 64 : (d <= 128 ? 128 : 192);
  CUtensorMap tq, tk, tv;
  if (!tmap_heads(&tq, q, (int64_t)B * Lq, H, d, ldq) || !tmap_heads(&tk, k, (int64_t)B * Lk, H, d, ldk) ||
      !tmap_vt(&tv, vt, (int64_t)H * d, (int64_t)(B - 1) * vt_img + Lk, ldvt, DP))
    return DRS_ERR_CUDA;
  const float sl2 = scale * 1.4426950408889634f;
  cudaStream_t st = (cudaStream_t)stream;
  if (DP == 64) return launch_attn<64>(tq, tk, tv, o, ldo, B, H, Lq, Lk, d, vt_img, sl2, st);
  if (DP == 128) return launch_attn<128>(tq, tk, tv, o, ldo, B, H, Lq, Lk, d, vt_img, sl2, st);
  return launch_attn<192>(tq, tk, tv, o, ldo, B, H, Lq, Lk, d, vt_img, sl2, st);
}

extern "C" int drs_attention_tc_debug(int* mapped_trace) {
  return cudaMemcpyToSymbol(drs::g_attn_trace, &mapped_trace, sizeof(int*)) == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
}
