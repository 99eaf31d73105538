/* drs.h -- C ABI of libdrs.so, the B200 (sm_100a) kernels behind the
 * DRiffusion draft-and-refine sampler (package paper_2603_25872_b200).
 *
 * Every entry point takes plain pointers/sizes and a cudaStream_t (passed as
 * void*), launches asynchronously on that stream, never allocates, never
 * synchronises, and returns an int status (DRS_OK or one of the codes below).
 * Argument validation happens on the host before any launch, so a non-zero
 * status means nothing was enqueued.  Device-side failures that can only be
 * detected while running (a ziggurat tail needing more lookahead than the
 * window holds) are reported through the caller's `err` word, which the host
 * wrapper inspects after the run (see paper_2603_25872_b200/_lib.py).
 *
 * The reference (skipdiff, /root/reference/pkg/src/skipdiff) has no FFI: its
 * boundary is Python.  Each function below replaces one reference routine;
 * the citation says which.  The ctypes binding a skipdiff maintainer would add
 * is in INTEGRATION.md.
 */
#ifndef DRS_H_
#define DRS_H_
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: 1:1 with skipdiff/errors.py (+ ValueError/TypeError) -- */
#define DRS_OK                       0
#define DRS_ERR_VALUE                1  /* ValueError (bad argument, z missing)        */
#define DRS_ERR_TIMESTEP_OUT_OF_RANGE 2 /* errors.py:12  TimestepOutOfRange           */
#define DRS_ERR_INVALID_SKIP         3  /* errors.py:24  InvalidSkip                  */
#define DRS_ERR_VARIANCE_TOO_LARGE   4  /* errors.py:28  VarianceTooLarge             */
#define DRS_ERR_DIMENSION_MISMATCH   5  /* errors.py:16  DimensionMismatch            */
#define DRS_ERR_INVALID_PLAN         6  /* errors.py:40  InvalidPlanParams            */
#define DRS_ERR_CUDA                 7  /* launch failure (cudaGetLastError != 0)     */
#define DRS_ERR_NOISE_WINDOW         8  /* device: ziggurat tail exceeded lookahead   */

/* ---- noise generators ---------------------------------------------------- */
#define DRS_GEN_PCG64 0  /* numpy PCG64 (XSL-RR 128/64): skipdiff rng.py:32        */
#define DRS_GEN_SFC64 1  /* numpy SFC64 seeded by the same SeedSequence key        */

/* One counter-based stream key = the entropy tuple numpy's SeedSequence sees.
 *   skipdiff rng.py:32      -> (0x7A9C, seed & 0xFFFFFFFFFFFF, t, role)
 *   skipdiff denoiser.py:144 -> (0x51DE, seed & 0xFFFFFFFF, t)
 * vals[0..n_vals) are non-negative integers (each becomes 1..2 little-endian
 * uint32 words, 0 -> [0]).  If seed_slot >= 0, vals[1] is replaced on device
 * by seeds[seed_slot] & seed_mask, so a captured CUDA graph can be replayed
 * for a new seed by rewriting one device word. */
typedef struct drs_key {
  int64_t vals[4];
  int32_t n_vals;
  int32_t seed_slot;
  uint64_t seed_mask;
} drs_key;

/* Fill out[s*ld + 0..n) with the first n standard normals of stream keys[s],
 * bit-identical to numpy `Generator(BitGen(SeedSequence(key))).standard_normal(n)`
 * (numpy random_standard_normal ziggurat; glibc log1p/exp on the slow paths).
 * keys and seeds are DEVICE pointers.  Replaces rng.py:27-33 derive_noise and
 * denoiser.py:139-145 state_independent_eps.  One CTA per stream. */
int drs_noise_fill(int gen, const drs_key* keys, int n_streams, const uint64_t* seeds,
                   int64_t n, double* out, int64_t ld, int* err, void* stream);
/* Measurement switch: 1 (default) = parallel chain resolve (slow-attempt list),
 * 0 = the serial one-warp resolve.  Same output bits either way. */
int drs_set_noise_resolve(int mode);

/* ---- skip transitions (K2/K3) -------------------------------------------- */
#define DRS_FAMILY_DDIM 0     /* ddim_skip                                   */
#define DRS_FAMILY_DDPM 1     /* ddpm_skip_sample(.., predicted_x0(eps), z)  */
#define DRS_FAMILY_DDPM_X0 2  /* ddpm_skip_sample with x0_hat given in eps   */
#define DRS_FAMILY_PRED_X0 3  /* predicted_x0: (x - c0 eps)/c1               */
#define DRS_FAMILY_EULER 4    /* euler_skip: x + c0 v   (transitions.py:188) */
#define DRS_SRC_X   0   /* op input = op.x (a state vector in HBM)             */
#define DRS_SRC_CUR 1   /* op input = result of the previous op (register)    */
#define DRS_SRC_ANCHOR 2 /* op input = result saved by the last SAVE_ANCHOR op */
#define DRS_OP_SAVE_ANCHOR 1

/* One elementwise skip update x_{t-k} = F(x_t, eps[, z]) with host-computed
 * fp64 coefficients (expression order of the reference, no FMA contraction):
 *  DDIM (transitions.py:155-179):
 *    c = {sqrt(1-ab_t), sqrt(ab_t), sqrt(ab_s), sqrt(1-ab_s-sigma**2), sigma, -}
 *    x0 = (x - c0*eps)/c1 ; out = c2*x0 + c3*eps ; if noisy: out = out + c4*z
 *  DDPM (sequential.py:51-54 + transitions.py:105-134):
 *    c = {sqrt(1-ab_t), sqrt(ab_t), sqrt(r)*(1-ab_s), sqrt(ab_s)*(1-r), 1-ab_t, sqrt(var)}
 *    x0 = (x - c0*eps)/c1 ; out = (c2*x + c3*x0)/c4 ; if noisy: out = out + c5*z
 * eps is fp64 (eps_f32 == 0) or fp32 (eps_f32 == 1, upcast exactly). */
typedef struct drs_op {
  double c[6];
  int32_t family;
  int32_t noisy;
  int32_t src;
  int32_t flags;
  int32_t eps_f32;
  int32_t pad;
  const double* x;
  const void* eps;
  const double* z;
  double* out;
  double* out2;
} drs_op;

/* Run ops[0..n_ops) (a DEVICE array) in order for every element j < D.
 * Intermediate states stay in registers; each op writes out/out2 if set.
 * Replaces ddim_skip / ddpm_skip_sample calls of parallel.py:256-306 and
 * sequential.py:68-74,106-111: a draft fan-out, a refine chain, or a refine
 * chain fused with the next block's drafts, in one launch. n_ops <= 64. */
int drs_skip_chain(const drs_op* ops, int n_ops, int64_t D, void* stream);
/* Measurement switch: 1 (default) = 16-byte vector kernel for HBM-sized even D, 0 = scalar kernel. */
int drs_set_chain_vec(int on);

/* ---- toy eps oracle (K9) ------------------------------------------------- */
#define DRS_GM_MAX_COMP 1920   /* mixture components per launch (shared-memory bound) */
/* Gaussian-mixture eps (denoiser.py:73-107) for rows r < n_rows:
 *   x = xs[r] (fp64, D), t = ts[r] (DEVICE int32), abar = alpha_bar[t]
 *   eps[r] = -sqrt(1-abar) * sum_i resp_i(x) (sqrt(abar) m_i - x)/s_i,
 *   s_i = abar v_i + 1-abar.  means: n_comp x D fp64, logw/var: n_comp fp64.
 * xs / out are DEVICE arrays of n_rows pointers.  1 <= n_comp <= 1920 (DRS_GM_MAX_COMP). */
int drs_gm_eps(const double* const* xs, const int32_t* ts, int n_rows, int64_t D,
               const double* alpha_bar, int T, const double* means, const double* log_w,
               const double* var, int n_comp, double* const* out, int* err, void* stream);

/* Euler family (next-row scope): VE-mixture ODE velocity (denoiser.py:124-136,
 * replaces velocity_oracle at parallel.py:343-344 / sequential.py:125) for
 * rows r < n_rows: x = xs[r], sigma = sigmas[idx[r]] (idx DEVICE int32 in
 * 0..N), s_i = v_i + sigma**2, gain_i = v_i / s_i,
 *   x0_hat = sum_i resp_i(x) (m_i + gain_i (x - m_i)),  v[r] = (x - x0_hat) / sigma.
 * *err |= 2 for an index outside 0..N, |= 4 for sigma <= 0 (NonPositiveSigma). */
int drs_gm_velocity(const double* const* xs, const int32_t* idx, int n_rows, int64_t D,
                    const double* sigmas, int N, const double* means, const double* log_w,
                    const double* var, int n_comp, double* const* out, int* err, void* stream);

/* E[x0 | x_t = x] of the VP-noised mixture (x0_posterior_mean, denoiser.py:110-121)
 * at one abar in (0, 1] (abar: DEVICE fp64 scalar; zeros: DEVICE int32[n_rows] of 0):
 *   centers sqrt(abar) m_i, s_i = abar v_i + 1-abar, gain_i = sqrt(abar) v_i / s_i,
 *   out[r] = sum_i resp_i(x) (m_i + gain_i (x - sqrt(abar) m_i)). */
int drs_gm_x0_mean(const double* const* xs, const int32_t* zeros, int n_rows, int64_t D,
                   const double* abar, const double* means, const double* log_w, const double* var,
                   int n_comp, double* const* out, int* err, void* stream);

/* ---- Perturbed-denoiser ablation (next-row scope) ----------------------------- */
/* keys[r] = the noise key of denoiser.py:224-231's perturbation of state xs[r]
 * (fp64, D) at timestep ts[r] (DEVICE int32): BLAKE2b-64(b"perturb" || t ||
 * round(x / quantum) as int64) as a one-value drs_key, consumed by
 * drs_noise_fill to draw the perturbation (default_rng(digest).standard_normal).
 * quantum = 1e-8 in the reference.  xs: DEVICE array of n_rows pointers. */
int drs_perturb_keys(const double* const* xs, const int32_t* ts, int n_rows, int64_t D, double quantum,
                     drs_key* keys, void* stream);

/* ---- quality metrics (K10, next-row scope: metrics.py:42-89) ---------------- */
/* out[i] = |X[i,:]|^2 for a row-major (n, dim) fp64 matrix (squared row norms). */
int drs_row_sqnorm(const double* X, int n, int dim, double* out, void* stream);
/* Gaussian-kernel MMD partial sums (mmd_gaussian, metrics.py:72-89) without the
 * n x m kernel matrix: partial[by * gx + bx] = sum over the 64 x 64 pair tile
 * (bx, by) of exp(-gamma * max(na[i] + nb[j] - 2 A_i . B_j, 0)), pairs i == j
 * skipped when same != 0 (A == B).  gx = ceil(m/64), gy = ceil(n/64) <= 65535;
 * the caller sums the gx*gy partials in index order (bit-reproducible). */
int drs_mmd_partials(const double* A, const double* na, int n, const double* B, const double* nb, int m,
                     int dim, double gamma, int same, double* partial, void* stream);

/* Copy rows: out[r][0..D) = src[r][0..D) (DEVICE pointer arrays). */
int drs_copy_rows(const double* const* src, double* const* out, int n_rows, int64_t D,
                  void* stream);

/* Busy-wait `n_ctas` CTAs for `us` microseconds each (concurrently): the
 * device analogue of the Latency wrapper's sleep (denoiser.py:204-209,258-263). */
int drs_spin(double us, int n_ctas, void* stream);

/* Host-side ports used by the device kernels, exported for the CPU tests. */
double drs_host_log1p(double x);
double drs_host_exp(double x);
/* Host restatement of SeedSequence(key).generate_state(n_words32, uint32). */
int drs_host_seedseq(const drs_key* key, uint64_t seed, uint32_t* out, int n_words32);

int drs_version(void);
/* 1: launch every kernel with programmatic dependent launch so its prologue
 * overlaps the predecessor's tail; 0 (default): plain stream ordering. */
int drs_set_pdl(int on);
/* 1 (default): GEMM producers request their first weight (B) tiles before the
 * PDL wait, overlapping the cold weight stream with the predecessor kernel. */
int drs_set_early_weights(int on);
/* Default k-blocks per GEMM TMA box for calls whose drs_gemm_args.kbox is 0: 0 -> 1 (default),
 * otherwise 2 (separate kernel instantiations with 3-D tensor maps, K % 64 == 0).  Fewer, larger
 * TMA operations: the per-op issue cost bounds the operand stream of small tiles. */
int drs_set_gemm_kb2(int on);

#ifdef __cplusplus
}
#endif
#endif /* DRS_H_ */
