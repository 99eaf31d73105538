// K1/K1b: bit-exact counter-based normal streams on sm_100a.
//
// Replaces skipdiff rng.py:27-33 (derive_noise) and denoiser.py:139-145
// (state_independent_eps): numpy Generator.standard_normal over PCG64 (or the
// SFC64 variant) seeded by SeedSequence(key).  numpy's ziggurat
// (random_standard_normal, 256 layers) consumes a VARIABLE number of 64-bit
// words per normal: 1 on the fast path (98.5%), 2 on a wedge test (which may
// reject and restart), 1+2m on the tail.  Output j therefore depends on how
// many words normals 0..j-1 consumed; the decode is a chain over word
// positions.  One CTA owns one stream and walks it in tiles of W positions:
//
//   1. generate: words[tile_base .. tile_base+W+MARGIN) into shared memory.
//      PCG64: every thread jumps (affine LCG map) to its own 9-word chunk.
//      SFC64: no jump-ahead -> one thread generates sequentially.
//   2. classify (all threads, independent per position p): the attempt that
//      would START at p -> (step = words consumed, accept, value).  Wedge and
//      tail attempts read their extra words from the lookahead margin.
//   3. resolve (warp 0): the chain visits p iff no earlier visited attempt
//      covers it.  Per 32-position window: ballot the slow lanes, jump over
//      covered lanes with __ffs, rank the visited+accepted lanes with popc,
//      and store their values to out[] coalesced.  A cover that runs past the
//      window/tile is carried in a register.
//
// Arithmetic is IEEE double with contraction disabled (--fmad=false), in the
// operation order of numpy's C code (no FMA in libnpyrandom), with glibc's
// FMA-variant log1p/exp ported in glibc_math.cuh.
#include <cuda_runtime.h>
#include "drs.h"
#include "pdl.cuh"
#include "bitgen.cuh"
#include "glibc_math.cuh"

namespace drs {

// 0: serial one-warp resolve; 1 (default): parallel resolve over the slow list
__device__ int g_resolve_mode = 1;
__device__ __forceinline__ int resolve_mode() { return g_resolve_mode; }

__device__ const uint64_t kZigKi[256] = DRS_ZIG_KI;
__device__ const double kZigWi[256] = DRS_ZIG_WI;
__device__ const double kZigFi[256] = DRS_ZIG_FI;

constexpr int kThreads = 256;
constexpr int kPer = 9;                       // words generated per thread per tile
constexpr int kWords = kThreads * kPer;       // 2304 words in smem per tile
constexpr int kMargin = 64;                   // lookahead for wedge/tail attempts
constexpr int kW = kWords - kMargin;          // 2240 positions classified per tile
static_assert(kW % 32 == 0, "tile must be whole warps");

constexpr double kZigR = 3.6541528853610088;
constexpr double kZigInvR = 0.27366123732975828;

__device__ __forceinline__ double next_double_of(uint64_t w) {
  return (double)(w >> 11) * (1.0 / 9007199254740992.0);
}

// Classify positions p = p0, p0+stride, ... < W of one tile: the ziggurat
// attempt starting at p -> (value, words consumed, accept).  words[] holds
// W + kMarginWords valid entries.
__device__ __forceinline__ void classify(const uint64_t* __restrict__ words, int n_words,
                                         double* __restrict__ vals, uint8_t* __restrict__ steps,
                                         int W, int p0, int stride, int& local_err) {
  for (int p = p0; p < W; p += stride) {
    const uint64_t w = words[p];
    const int idx = (int)(w & 0xff);
    const uint64_t r = w >> 8;
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
    double x = (double)rabs * kZigWi[idx];
    if (r & 1) x = -x;
    int step = 1, acc = 1;
    if (rabs >= kZigKi[idx]) {
      if (idx == 0) {                      // tail: 2 doubles per iteration
        int q = p + 1;
        double xx;
        for (;;) {
          if (q + 1 >= n_words) { local_err = 1; xx = 0.0; break; }
          xx = -kZigInvR * log1p_glibc(-next_double_of(words[q]));
          const double yy = -log1p_glibc(-next_double_of(words[q + 1]));
          q += 2;
          if (yy + yy > xx * xx) break;
        }
        x = ((rabs >> 8) & 1) ? -(kZigR + xx) : kZigR + xx;
        step = q - p;
        if (step > 127) { local_err = 1; step = 127; }
      } else {                             // wedge: 1 double, may reject
        const double u = next_double_of(words[p + 1]);
        const double lhs = (kZigFi[idx - 1] - kZigFi[idx]) * u + kZigFi[idx];
        acc = lhs < exp_glibc(-0.5 * x * x) ? 1 : 0;
        step = 2;
      }
    }
    vals[p] = x;
    steps[p] = (uint8_t)(step | (acc << 7));
  }
}

// Resolve the visit chain over one classified tile and store the accepted
// values (called by one full warp).  count / cover carry across tiles.
__device__ __forceinline__ void resolve(const double* __restrict__ vals, const uint8_t* __restrict__ steps,
                                        int W, double* __restrict__ o, int64_t n, int64_t& count,
                                        int& cover, int lane) {
  for (int base = 0; base < W && count < n; base += 32) {
    const uint8_t sv = steps[base + lane];
    const int my_step = sv & 0x7f;
    const unsigned slow = __ballot_sync(0xffffffffu, my_step != 1);
    const unsigned accm = __ballot_sync(0xffffffffu, (sv >> 7) & 1);
    unsigned vis = 0;
    if (cover >= 32) {
      cover -= 32;
    } else {
      int pos = cover;
      while (pos < 32) {
        const unsigned ahead = slow & (0xffffffffu << pos);
        if (ahead == 0) { vis |= 0xffffffffu << pos; pos = 32; break; }
        const int s = __ffs(ahead) - 1;
        const unsigned upto = (s == 31) ? 0xffffffffu : ((1u << (s + 1)) - 1u);
        vis |= upto & (0xffffffffu << pos);
        pos = s + __shfl_sync(0xffffffffu, my_step, s);
      }
      cover = pos - 32;
    }
    const unsigned va = vis & accm;
    if ((va >> lane) & 1u) {
      const int64_t oi = count + __popc(va & ((1u << lane) - 1u));
      if (oi < n) o[oi] = vals[base + lane];
    }
    count += __popc(va);
  }
}

// ---- parallel resolve (all worker threads) ---------------------------------
// The visit chain only branches at SLOW attempts (step > 1: wedge tests and
// tails, ~1.5 % of positions): a position is visited iff it is >= the entry
// cover and not strictly inside the span [s, s + step_s) of a VISITED slow
// attempt s, and a slow attempt is visited iff it is not inside an earlier
// visited span.  So: (1) the tile's slow positions are listed in order
// (per-window ballots + a window prefix), (2) one thread walks only that short
// list, (3) every worker marks the visited spans in a bitmap and (4) writes the
// accepted values of visited positions at their prefix-sum output index.  Same
// chain as `resolve` (bit-identical output), without 70 serial windows.
template <int W>
struct ResolveScratch {
  static constexpr int kWin = W / 32;
  uint16_t slow[W];             // slow positions, in order
  int win_cnt[kWin];            // slow count, then accepted count, per window
  int win_off[kWin];
  uint32_t covered[kWin];       // bit p%32 of word p/32: inside a visited slow span
  int n_slow;
  int cover_out;
  int64_t count_out;
};

__device__ __forceinline__ void wsync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" :: "r"(id), "r"(nthreads) : "memory");
}

// Exclusive prefix over kWin window counts (kWin <= 96), done by warp 0 of the workers.
template <int kWin>
__device__ __forceinline__ void window_scan(const int* cnt, int* off, int lane, int& total) {
  int carry = 0;
#pragma unroll
  for (int b = 0; b < kWin; b += 32) {
    const int v = b + lane < kWin ? cnt[b + lane] : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (b + lane < kWin) off[b + lane] = carry + x - v;
    carry += __shfl_sync(0xffffffffu, x, 31);
  }
  total = carry;
}

template <int W>
__device__ __forceinline__ void resolve_parallel(const double* __restrict__ vals, const uint8_t* __restrict__ steps,
                                                 ResolveScratch<W>& sc, double* __restrict__ o, int64_t n,
                                                 int64_t& count, int& cover, int tid, int nthreads, int bar_id) {
  constexpr int kWin = W / 32;
  const int lane = tid & 31, warp = tid >> 5, nwarps = nthreads >> 5;
  // (1) slow positions per window
  for (int w = warp; w < kWin; w += nwarps) {
    const unsigned slow = __ballot_sync(0xffffffffu, (steps[w * 32 + lane] & 0x7f) != 1);
    if (lane == 0) { sc.win_cnt[w] = __popc(slow); sc.covered[w] = 0u; }
  }
  wsync(bar_id, nthreads);
  if (warp == 0) {
    int total;
    window_scan<kWin>(sc.win_cnt, sc.win_off, lane, total);
    if (lane == 0) sc.n_slow = total;
  }
  wsync(bar_id, nthreads);
  for (int w = warp; w < kWin; w += nwarps) {
    const bool sl = (steps[w * 32 + lane] & 0x7f) != 1;
    const unsigned slow = __ballot_sync(0xffffffffu, sl);
    if (sl) sc.slow[sc.win_off[w] + __popc(slow & ((1u << lane) - 1u))] = (uint16_t)(w * 32 + lane);
  }
  wsync(bar_id, nthreads);
  // (2) walk the slow attempts in order (one thread; ~35 per 2240 positions);
  //     a visited one is flagged by setting bit 15 of its list entry
  if (tid == 0) {
    int cov = cover;                              // first position not covered
    const int ns = sc.n_slow;
    for (int i = 0; i < ns; ++i) {
      const int sp = sc.slow[i];
      if (sp >= cov) {
        cov = sp + (steps[sp] & 0x7f);
        sc.slow[i] = (uint16_t)(sp | 0x8000);
      }
    }
    sc.cover_out = cov > W ? cov - W : 0;
  }
  wsync(bar_id, nthreads);
  // (3) mark the interiors of visited spans (and the entry cover) as covered
  for (int i = tid; i < sc.n_slow; i += nthreads) {
    const int e = sc.slow[i];
    if (e & 0x8000) {
      const int sp = e & 0x7fff;
      const int end = min(W, sp + (steps[sp] & 0x7f));
      for (int q = sp + 1; q < end; ++q) atomicOr(&sc.covered[q >> 5], 1u << (q & 31));
    }
  }
  for (int q = tid; q < min(cover, W); q += nthreads) atomicOr(&sc.covered[q >> 5], 1u << (q & 31));
  wsync(bar_id, nthreads);
  // (4) accepted & visited -> output index (window prefix), coalesced stores
  for (int w = warp; w < kWin; w += nwarps) {
    const bool vis = !((sc.covered[w] >> lane) & 1u);
    const bool acc = vis && ((steps[w * 32 + lane] >> 7) & 1);
    const unsigned am = __ballot_sync(0xffffffffu, acc);
    if (lane == 0) sc.win_cnt[w] = __popc(am);
  }
  wsync(bar_id, nthreads);
  if (warp == 0) {
    int total;
    window_scan<kWin>(sc.win_cnt, sc.win_off, lane, total);
    if (lane == 0) sc.count_out = count + total;
  }
  wsync(bar_id, nthreads);
  for (int w = warp; w < kWin; w += nwarps) {
    const bool vis = !((sc.covered[w] >> lane) & 1u);
    const bool acc = vis && ((steps[w * 32 + lane] >> 7) & 1);
    const unsigned am = __ballot_sync(0xffffffffu, acc);
    if (acc) {
      const int64_t oi = count + sc.win_off[w] + __popc(am & ((1u << lane) - 1u));
      if (oi < n) o[oi] = vals[w * 32 + lane];
    }
  }
  count = sc.count_out;
  cover = sc.cover_out;
}

__device__ __forceinline__ void load_key(const drs_key* keys, const uint64_t* seeds, int sidx,
                                         uint32_t* ent, int& ne) {
  const drs_key k = keys[sidx];
  const uint64_t seed = k.seed_slot >= 0 ? seeds[k.seed_slot] : 0ull;
  ne = key_words(k, seed, ent);
}

// ------------------------------------------------------------- PCG64 -------
// Every thread jumps to its own 9-word chunk of the tile (affine LCG map).
__global__ void __launch_bounds__(kThreads)
noise_pcg64_kernel(const drs_key* __restrict__ keys, const uint64_t* __restrict__ seeds,
                   int64_t n, double* __restrict__ out, int64_t ld, int* __restrict__ err) {
  pdl_wait();
  pdl_trigger();
  __shared__ uint64_t words[kWords];
  __shared__ double vals[kW];
  __shared__ uint8_t steps[kW];               // bit7 = accept, bits0..6 = words consumed
  __shared__ u128 s_state, s_inc;
  __shared__ int64_t s_count;
  __shared__ ResolveScratch<kW> sc;
  const int tid = threadIdx.x, lane = tid & 31;
  double* const o = out + (int64_t)blockIdx.x * ld;
  if (tid == 0) {
    uint32_t ent[8];
    int ne;
    load_key(keys, seeds, blockIdx.x, ent, ne);
    Pcg64 g; g.seed(ent, ne);
    s_state = g.state; s_inc = g.inc;
    s_count = 0;
  }
  __syncthreads();
  const u128 inc = s_inc;
  u128 st, tile_m, tile_p;
  {
    u128 am, ap;
    Pcg64::jump(inc, (uint64_t)tid * kPer, am, ap);
    st = am * s_state + ap;                    // state after tid*kPer steps
    Pcg64::jump(inc, (uint64_t)kW, tile_m, tile_p);
  }
  int64_t count = 0;
  int cover = 0, local_err = 0;
  for (;;) {
    u128 s = st;
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      s = s * pcg_mult() + inc;
      words[tid * kPer + j] = Pcg64::output(s);
    }
    st = tile_m * st + tile_p;
    __syncthreads();
    classify(words, kWords, vals, steps, kW, tid, kThreads, local_err);
    __syncthreads();
    if (resolve_mode() == 0) {
      if (tid < 32) {
        resolve(vals, steps, kW, o, n, count, cover, lane);
        if (lane == 0) s_count = count;
      }
    } else {
      resolve_parallel<kW>(vals, steps, sc, o, n, count, cover, tid, kThreads, 0);
      if (tid == 0) s_count = count;
    }
    __syncthreads();
    if (s_count >= n) break;
  }
  if (local_err) atomicOr(err, 1);
}

// ------------------------------------------------------------- SFC64 -------
// No jump-ahead: one generator lane (warp kSfcGenWarp) produces tile i+1 into
// the other half of a double buffer while warps 0..kSfcGenWarp-1 classify
// and resolve tile i, so the serial recurrence is the only critical path.
constexpr int kSfcW = 512;                        // positions per tile (less speculative waste)
constexpr int kSfcWords = kSfcW + kMargin;        // words generated per tile
constexpr int kSfcGenWarp = kThreads / 32 - 1;    // last warp generates
constexpr int kSfcWorkers = kThreads - 32;

__global__ void __launch_bounds__(kThreads)
noise_sfc64_kernel(const drs_key* __restrict__ keys, const uint64_t* __restrict__ seeds,
                   int64_t n, double* __restrict__ out, int64_t ld, int* __restrict__ err) {
  pdl_wait();
  pdl_trigger();
  __shared__ uint64_t words[2][kSfcWords];
  __shared__ double vals[kSfcW];
  __shared__ uint8_t steps[kSfcW];
  __shared__ int64_t s_count;
  __shared__ ResolveScratch<kSfcW> sc;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* const o = out + (int64_t)blockIdx.x * ld;
  const bool gen_lane = warp == kSfcGenWarp && lane == 0;
  Sfc64 g;
  if (gen_lane) {
    uint32_t ent[8];
    int ne;
    load_key(keys, seeds, blockIdx.x, ent, ne);
    g.seed(ent, ne);
    Sfc64 h = g;                                   // tile 0
    for (int j = 0; j < kSfcWords; ++j) {
      words[0][j] = h.next();
      if (j == kSfcW - 1) g = h;                  // tile 1 starts kSfcW words in
    }
  }
  if (tid == 0) s_count = 0;
  __syncthreads();
  int64_t count = 0;
  int cover = 0, local_err = 0;
  for (int tile = 0;; ++tile) {
    const int cur = tile & 1;
    if (warp == kSfcGenWarp) {
      if (lane == 0) {                             // speculatively generate the next tile
        Sfc64 h = g;
        uint64_t* dst = words[cur ^ 1];
#pragma unroll 4
        for (int j = 0; j < kSfcWords; ++j) {
          dst[j] = h.next();
          if (j == kSfcW - 1) g = h;
        }
      }
    } else {
      classify(words[cur], kSfcWords, vals, steps, kSfcW, tid, kSfcWorkers, local_err);
      asm volatile("bar.sync 1, %0;" :: "n"(kSfcWorkers));
      if (resolve_mode() == 0) {
        if (warp == 0) {
          resolve(vals, steps, kSfcW, o, n, count, cover, lane);
          if (lane == 0) s_count = count;
        }
      } else {
        resolve_parallel<kSfcW>(vals, steps, sc, o, n, count, cover, tid, kSfcWorkers, 1);
        if (tid == 0) s_count = count;
      }
    }
    __syncthreads();
    if (s_count >= n) break;
  }
  if (local_err) atomicOr(err, 1);
}

}  // namespace drs

extern "C" int drs_noise_fill(int gen, const drs_key* keys, int n_streams, const uint64_t* seeds,
                              int64_t n, double* out, int64_t ld, int* err, void* stream) {
  if (n_streams < 0 || n < 0 || (n_streams > 0 && ld < n)) return DRS_ERR_VALUE;
  if (n_streams == 0 || n == 0) return DRS_OK;
  if (!keys || !out || !err) return DRS_ERR_VALUE;
  cudaStream_t s = (cudaStream_t)stream;
  if (gen == DRS_GEN_PCG64)
    drs::launch_pdl(drs::noise_pcg64_kernel, dim3(n_streams), dim3(drs::kThreads), 0, s, keys, seeds, n, out, ld, err);
  else if (gen == DRS_GEN_SFC64)
    drs::launch_pdl(drs::noise_sfc64_kernel, dim3(n_streams), dim3(drs::kThreads), 0, s, keys, seeds, n, out, ld, err);
  else
    return DRS_ERR_VALUE;
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
}

extern "C" int drs_set_noise_resolve(int mode) {
  if (mode < 0 || mode > 1) return DRS_ERR_VALUE;
  return cudaMemcpyToSymbol(drs::g_resolve_mode, &mode, sizeof(int)) == cudaSuccess ? DRS_OK : DRS_ERR_CUDA;
}
