/* drs_net.h -- C ABI of the denoiser-network kernels in libdrs.so (sm_100a).
 *
 * The reference has no networks: its eps is an analytic oracle
 * (skipdiff denoiser.py:85-145).  BASELINE configs C3-C5 put random-init
 * SD1.5-UNet / DiT-XL/2 / SDXL-UNet shaped networks behind the same
 * `evaluate(d, s, x, t)` boundary (paper_2603_25872_b200/denoiser.py
 * NetworkEps); these are their hot ops.  Same conventions as drs.h: plain
 * device pointers, a cudaStream_t as void*, int status (DRS_OK = 0).
 */
#ifndef DRS_NET_H_
#define DRS_NET_H_
#include <stdint.h>
#include <stddef.h>
#include "drs.h"

#ifdef __cplusplus
extern "C" {
#endif

#define DRS_ACT_NONE 0
#define DRS_ACT_GELU_TANH 1   /* DiT MLP (GELU(approximate="tanh"))                      */
#define DRS_ACT_SILU 2
#define DRS_ACT_GELU_ERF 3
#define DRS_ACT_GEGLU 4       /* weight rows interleaved (value, gate): out[n/2] = v * gelu(g) */
#define DRS_ACT_HEADSOFTMAX 5 /* scores -> probabilities: every 96-column block (one attention head)
                               * is softmax-normalised over its first hs_valid columns (exp2 of
                               * the raw accumulator: fold scale * log2(e) into B), zeros after;
                               * bf16 out, bn = 192, split = 1, one CTA per tile                */

/* C[M,N] = act(alpha * A[M,K] . B[N,K]^T + bias[N]) (+ residual[M,N]).
 * A, B bf16 K-major (lda/ldb in elements, multiples of 8, 16-byte aligned),
 * C bf16 (out_f32 = 0) or fp32, residual bf16 or NULL, bias fp32 or NULL.
 * tcgen05.mma (M=128, N=bn in {64,128,256}) with TMA-fed SWIZZLE_128B smem
 * ring and a double-buffered TMEM accumulator; split in 2..8 = deterministic
 * split-K over a thread-block cluster (partials reduced through DSMEM in a
 * fixed order); `workspace` is unused (kept for ABI stability, may be NULL). */
int drs_gemm_bf16(const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                  int M, int N, int K, const float* bias, const void* residual, int64_t ldr,
                  int act, int out_f32, float alpha, int bn, int split, float* workspace, void* stream);

/* Full-epilogue form:
 *   C = act(alpha*A.B^T + bias[n] + rowbias[(m / rb_group)*rb_ld + n]) * colscale + residual
 * residual fp32 (res_f32 = 1, a transformer residual stream) or bf16;
 * colscale (adaLN-Zero gate) indexed [(m / cs_group)*cs_ld + n] if cs_group > 0
 * else [n]; rowbias = per-image bias (UNet time-embedding injection). */
typedef struct drs_gemm_args {
  const void* A; int64_t lda;
  const void* B; int64_t ldb;
  void* C; int64_t ldc;
  int M, N, K;
  int act, out_f32;
  float alpha;
  const float* bias;
  const void* residual; int64_t ldr; int res_f32;
  const float* colscale; int cs_group; int64_t cs_ld;
  const float* rowbias; int rb_group; int64_t rb_ld;
  int bn, split;
  float* workspace;
  /* implicit 3x3 conv (stride 1, pad 1): conv_C > 0 makes A the NHWC bf16
   * input [conv_N, conv_H, conv_W, conv_C] (M = N*H*W, K = 9*C, weights
   * (Cout, ky, kx, C)); C % 64 == 0, W a power of two <= 128. */
  int conv_N, conv_H, conv_W, conv_C;
  /* 1: run the tile on a CTA PAIR (tcgen05.mma.cta_group::2, M = 256 per pair,
   * each CTA loads its 128 A rows and half of the B tile -> (128 + bn/2) x 128 B
   * of operand ingest per SM per k-block instead of (128 + bn) x 128 B).
   * Needs M >= 256 and split == 1; otherwise ignored.  0: one CTA per tile. */
  int cta_pair;
  /* Per-image B operand (CFG: unconditional / conditional context): when
   * b_img_rows > 0, rows [m, m+128) of A with (m / b_img_rows) odd use B rows
   * offset by b_img_off (B holds N + b_img_off rows).  b_img_rows % 128 == 0
   * (% 256 for CTA pairs, else the pair flag is ignored). */
  int b_img_rows, b_img_off;
  /* DRS_ACT_HEADSOFTMAX: valid columns per 96-column head block (<= 96). */
  int hs_valid;
  /* Optional bf16 copy of an fp32 output (act none, no row bias / column gate):
   * out2[m, n] = bf16(C[m, n]), row stride ldo2 (the transformer's residual stream
   * and the bf16 input of the projection that follows, in one epilogue). */
  void* out2; int64_t ldo2;
  /* implicit conv stride: 0 / 1, or 2 (conv_H / conv_W are then the OUTPUT grid of
   * a stride-2, pad-1 3x3 conv over a 2H x 2W input; the A box is loaded with TMA
   * element stride 2 -- downsamplers without an im2col copy). */
  int conv_stride;
  /* k-blocks (of 64) per TMA box: 0 = library default (drs_set_gemm_kb2), 1 or 2
   * (3-D [K/64][rows][64] tensor maps, K % 64 == 0; 4 is accepted and runs as 2). */
  int kbox;
} drs_gemm_args;
int drs_gemm(const drs_gemm_args* args, void* stream);

/* Tile width / split-K the library picks when drs_gemm gets bn == 0 and/or
 * split == 0 (in/out: nonzero inputs are kept).  Cost model calibrated on
 * B200 (per-SM operand streaming rate, MMA rate, launch and cluster-reduce
 * latency, cluster co-residency from cudaOccupancyMaxActiveClusters). */
int drs_gemm_pick(int M, int N, int K, int* bn, int* split);
/* The model's time for one configuration, in ns (-1 on bad arguments). */
int drs_gemm_cost_us(int M, int N, int K, int bn, int split);

/* out[m, :] = LN(x[m, :]) (*gamma + beta) (*(1 + scale) + shift) -> bf16.
 * x fp32 (x_f32 = 1) or bf16; gamma/beta fp32 [C] (16-byte aligned) or NULL; shift/scale fp32
 * or NULL, indexed [(m / mod_group) * mod_ld + c] when mod_group > 0 (per-sample
 * adaLN modulation of a token batch), else [c].  C <= 2048. */
int drs_layernorm(const void* x, int64_t ldx, int x_f32, int M, int C, const float* gamma, const float* beta,
                  const float* shift, const float* scale, int mod_group, int64_t mod_ld, float eps, void* out,
                  int64_t ldo, void* stream);

/* O = softmax(Q K^T * scale) V per (batch b, head h): Q rows b*Lq.., K/V rows
 * b*Lk.., head h at column h*d of each row (strides in elements).  bf16 in/out,
 * fp32 softmax; mma.sync m16n8k16, 64 queries per CTA.  d % 8 == 0, d <= 160. */
int drs_attention(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v, int64_t ldv,
                  void* o, int64_t ldo, int B, int H, int Lq, int Lk, int d, float scale, void* stream);

/* Same on the 5th-gen tensor cores (tcgen05.mma S = Q K^T and O += P V with TMEM
 * accumulators, TMA-fed Q / K / V^T tiles, 128 queries per CTA).  V is given
 * TRANSPOSED: vt[(h*d + j), b*vt_img + key] (row stride ldvt), as produced by a
 * swapped-operand GEMM; vt_img >= Lk, multiple of 8.  d % 8 == 0, d <= 192. */
int drs_attention_tc(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* vt, int64_t ldvt,
                     int vt_img, void* o, int64_t ldo, int B, int H, int Lq, int Lk, int d, float scale,
                     void* stream);

/* Same with V row-major -- v[b*Lk + key, h*d + j] (row stride ldv), e.g. the V block
 * of one fused QKV projection -- loaded like K and read by the PV MMA as an
 * MN-major B operand (no V^T GEMM).  d % 8 == 0, d <= 192. */
int drs_attention_tc_v(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v, int64_t ldv,
                       void* o, int64_t ldo, int B, int H, int Lq, int Lk, int d, float scale, void* stream);

/* GEMV for M <= 4 rows: out[m, n] = act(x[m, :] . w[n, :] + bias[n]) (+ res[m, n]),
 * act DRS_ACT_NONE / DRS_ACT_SILU, bf16 x / w (K % 8 == 0, w 16-byte aligned),
 * fp32 or bf16 residual / output.  HBM-bound weight stream on the CUDA cores
 * (the conditioning MLPs of the denoisers: timestep and adaLN embeddings). */
int drs_gemv(const void* x, int64_t ldx, const void* w, int64_t ldw, const float* bias, const void* res,
             int64_t ldr, int res_f32, void* out, int64_t ldo, int out_f32, int M, int N, int K, int act,
             int ctas_per_sm /* 0: 4 per SM; 1: leaves room for co-resident GEMM CTAs */, void* stream);

/* Measurement switch: 0 = attention with one MMA warp, 1 = separate S and PV MMA issuer warps,
 * 2 (default) = 1 + the softmax on the paired FP32 pipe (FFMA2 / FADD2). */
int drs_set_attn_split(int on);

/* DiT helpers */
int drs_timestep_embedding(const float* t, int n, int dim, float max_period, void* out_bf16, void* stream);
int drs_patchify(const void* x, int x_f64, int C, int H, int W, int p, void* out_bf16, void* stream);
int drs_unpatchify(const float* tok, int Cout, int Ckeep, int H, int W, int p, float* out, void* stream);
int drs_silu_cast(const float* x, int64_t n, void* out_bf16, void* stream);
int drs_cast_f32_bf16(const float* x, int64_t n, void* out_bf16, void* stream);

/* UNet helpers (NHWC bf16 activations) */
/* A[(n,oy,ox), (ky,kx,c)] for a ks x ks conv over the channel concat [x1 | x2],
 * stride/pad, nearest-upsampled input when up = 2.  C1, C2 multiples of 8. */
int drs_im2col(const void* x1, int C1, const void* x2, int C2, int N, int H, int W, int ks, int stride,
               int pad, int up, void* out, void* stream);
/* GroupNorm(G) + affine (+ SiLU) over NHWC -> bf16, bit-reproducible (fixed
 * reduction order, no atomics).  C % 8 == 0, C/G >= 8, G <= 32, input
 * <= 12 MB, 16-byte aligned x/out: one launch of thread-block clusters (per image x group chunk;
 * partial sums exchanged over DSMEM, input slice kept in shared memory);
 * workspace unused (may be NULL).  Otherwise two kernels (HW % 16 == 0) with
 * drs_groupnorm_workspace_bytes(N, G) bytes of workspace. */
/* GroupNorm implementation switch (measurement): 0 auto (default), 1 one CTA per
 * (image, group) with two L2 sweeps, 2 the cluster / two-kernel paths only. */
int drs_set_gn_mode(int mode);
int drs_groupnorm(const void* x, int x_f32, int N, int HW, int C, int G, const float* gamma, const float* beta,
                  float eps, int silu, void* out, void* workspace, void* stream);
size_t drs_groupnorm_workspace_bytes(int N, int G);
int drs_latent_to_nhwc(const void* x, int x_f64, int C, int HW, int Cpad, void* out, void* stream);
/* eps (C,H,W) fp32 = u + g (c - u) from NHWC fp32 rows [uncond | cond] (pair = 1) */
int drs_cfg_combine(const float* y, int64_t ld, int HW, int C, float g, int pair, float* eps, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DRS_NET_H_ */
