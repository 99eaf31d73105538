// Perturbed-denoiser keys on device (SURVEY 8f row 4 ablation; skipdiff
// denoiser.py:191-201,224-231):
//
//   q      = round_half_even(x / 1e-8) as int64                 (numpy np.round)
//   digest = BLAKE2b-64(b"perturb" || int64le(t) || q[0..D) as int64le)
//   noise  = default_rng(int.from_bytes(digest, "little")).standard_normal(D)
//
// This kernel hashes one state row per warp and writes the digest as a drs_key
// (one 64-bit entropy value -> two SeedSequence words, as numpy coerces a
// Python int), so the existing K1 noise kernel draws the perturbation from the
// key in HBM -- no host round trip, capturable in the sampler's CUDA graph.
// BLAKE2b follows RFC 7693 (unkeyed, digest length 8).  The 15-byte prefix
// shifts every q word across two message words: with Q[0] = t, Q[j] = q[j-1],
// message word w >= 1 is (Q[w-1] >> 8) | (Q[w] << 56) (zero past the end).
#include <cuda_runtime.h>
#include <stdint.h>
#include "drs.h"
#include "pdl.cuh"

namespace drs {

__constant__ uint64_t kB2bIv[8] = {0x6a09e667f3bcc908ull, 0xbb67ae8584caa73bull, 0x3c6ef372fe94f82bull,
                                   0xa54ff53a5f1d36f1ull, 0x510e527fade682d1ull, 0x9b05688c2b3e6c1full,
                                   0x1f83d9abfb41bd6bull, 0x5be0cd19137e2179ull};
// message schedule (RFC 7693 section 2.7); constexpr so the fully unrolled
// rounds index m[] with constants (registers, no local-memory array)
__host__ __device__ constexpr int b2b_sigma(int r, int i) {
  constexpr uint8_t S[12][16] = {
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
    {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4}, {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
    {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13}, {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
    {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11}, {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
    {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5}, {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0},
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3}};
  return S[r][i];
}

__device__ __forceinline__ uint64_t rotr64(uint64_t x, int n) { return (x >> n) | (x << (64 - n)); }

__device__ __forceinline__ void b2b_g(uint64_t* v, int a, int b, int c, int d, uint64_t x, uint64_t y) {
  v[a] = v[a] + v[b] + x;
  v[d] = rotr64(v[d] ^ v[a], 32);
  v[c] = v[c] + v[d];
  v[b] = rotr64(v[b] ^ v[c], 24);
  v[a] = v[a] + v[b] + y;
  v[d] = rotr64(v[d] ^ v[a], 16);
  v[c] = v[c] + v[d];
  v[b] = rotr64(v[b] ^ v[c], 63);
}

__device__ void b2b_compress(uint64_t* h, const uint64_t* m, uint64_t t_lo, bool last) {
  uint64_t v[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) { v[i] = h[i]; v[i + 8] = kB2bIv[i]; }
  v[12] ^= t_lo;                        // message length < 2^64 bytes: high counter word is 0
  if (last) v[14] = ~v[14];
#pragma unroll
  for (int r = 0; r < 12; ++r) {                        // unrolled: every m index is a constant
    b2b_g(v, 0, 4, 8, 12, m[b2b_sigma(r, 0)], m[b2b_sigma(r, 1)]);
    b2b_g(v, 1, 5, 9, 13, m[b2b_sigma(r, 2)], m[b2b_sigma(r, 3)]);
    b2b_g(v, 2, 6, 10, 14, m[b2b_sigma(r, 4)], m[b2b_sigma(r, 5)]);
    b2b_g(v, 3, 7, 11, 15, m[b2b_sigma(r, 6)], m[b2b_sigma(r, 7)]);
    b2b_g(v, 0, 5, 10, 15, m[b2b_sigma(r, 8)], m[b2b_sigma(r, 9)]);
    b2b_g(v, 1, 6, 11, 12, m[b2b_sigma(r, 10)], m[b2b_sigma(r, 11)]);
    b2b_g(v, 2, 7, 8, 13, m[b2b_sigma(r, 12)], m[b2b_sigma(r, 13)]);
    b2b_g(v, 3, 4, 9, 14, m[b2b_sigma(r, 14)], m[b2b_sigma(r, 15)]);
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) h[i] ^= v[i] ^ v[i + 8];
}

// Q[j]: j = 0 -> t; 1 <= j <= D -> q[j-1]; beyond -> 0
__device__ __forceinline__ uint64_t perturb_q(const double* __restrict__ x, int64_t D, int64_t t, int64_t j,
                                              double quantum) {
  if (j == 0) return (uint64_t)t;
  if (j > D) return 0;
  return (uint64_t)(long long)rint(x[j - 1] / quantum);
}

__global__ void __launch_bounds__(32)
perturb_keys_kernel(const double* const* __restrict__ xs, const int32_t* __restrict__ ts, int64_t D,
                    double quantum, uint64_t salt7, drs_key* __restrict__ keys) {
  pdl_wait();
  pdl_trigger();
  const int row = blockIdx.x, lane = threadIdx.x;
  const double* x = xs[row];
  const int64_t t = ts[row];
  const int64_t len = 15 + 8 * D;                     // message bytes
  const int64_t n_words = (len + 7) / 8;
  const int64_t n_blocks = (len + 127) / 128;
  uint64_t h[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) h[i] = kB2bIv[i];
  h[0] ^= 0x01010000ull ^ 8ull;                       // digest length 8, no key, fanout = depth = 1
  for (int64_t blk = 0; blk < n_blocks; ++blk) {
    // lanes 0..15 assemble message word w = 16 blk + lane
    uint64_t word = 0;
    if (lane < 16) {
      const int64_t w = blk * 16 + lane;
      if (w == 0) {
        word = salt7 | ((uint64_t)(t & 0xff) << 56);
      } else if (w < n_words) {
        word = (perturb_q(x, D, t, w - 1, quantum) >> 8) | (perturb_q(x, D, t, w, quantum) << 56);
      }
    }
    uint64_t m[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) m[i] = __shfl_sync(0xffffffffu, word, i);
    const bool last = blk == n_blocks - 1;
    const uint64_t counter = last ? (uint64_t)len : (uint64_t)(blk + 1) * 128;
    b2b_compress(h, m, counter, last);               // every lane, identical result
  }
  if (lane == 0) {
    drs_key k;
    k.vals[0] = (int64_t)h[0];                        // digest = first 8 bytes of h, little-endian
    k.vals[1] = k.vals[2] = k.vals[3] = 0;
    k.n_vals = 1;
    k.seed_slot = -1;
    k.seed_mask = ~0ull;
    keys[row] = k;
  }
}

}  // namespace drs

extern "C" int drs_perturb_keys(const double* const* xs, const int32_t* ts, int n_rows, int64_t D,
                                double quantum, drs_key* keys, void* stream) {
  if (n_rows < 0 || D < 0 || !(quantum > 0.0)) return DRS_ERR_VALUE;
  if (n_rows == 0) return DRS_OK;
  if (!xs || !ts || !keys) return DRS_ERR_VALUE;
  const uint64_t salt7 = 0x0062727574726570ull;       // int.from_bytes(b"perturb", "little") (denoiser.py:23)
  drs::launch_pdl(drs::perturb_keys_kernel, dim3(n_rows), dim3(32), 0, (cudaStream_t)stream, xs, ts, D, quantum,
                  salt7, keys);
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
}
