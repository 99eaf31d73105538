// Counter-based bit generators of the reference's noise streams, host+device.
//
// skipdiff rng.py:32 seeds `np.random.default_rng((0x7A9C, seed48, t, role))`,
// i.e. numpy PCG64 seeded through SeedSequence; denoiser.py:144 does the same
// with (0x51DE, seed32, t).  numpy 2.3.5 (bit_generator.pyx SeedSequence,
// pcg64.h, sfc64.h) is the third-party dependency that holds the algorithm;
// this header restates it:
//   SeedSequence: 4-word uint32 pool, hashmix/mix (constants below), then
//                 generate_state(n) with the INIT_B/MULT_B hash.
//   PCG64:  state/inc from generate_state(4, uint64); 128-bit LCG,
//           output XSL-RR (rotr64(hi ^ lo, state >> 122)); step THEN output.
//   SFC64:  a,b,c from generate_state(3, uint64), w = 1, 12 discarded draws.
// PCG64 is an affine map s -> M s + inc, so any position of the stream is
// reachable in O(log n) (pcg_advance): that is what lets every thread of the
// noise kernel start at its own word.  SFC64 has no jump-ahead.
#pragma once
#include <stdint.h>
#include "drs.h"

#ifdef __CUDACC__
#define DRS_HD __host__ __device__ __forceinline__
#else
#define DRS_HD static inline
#endif

namespace drs {

typedef unsigned __int128 u128;

// ------------------------------------------------------------ SeedSequence --
struct SeedSeq {
  static constexpr uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u;
  static constexpr uint32_t INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
  static constexpr uint32_t MIX_L = 0xca01f9ddu, MIX_R = 0x4973f715u;
  uint32_t pool[4];

  // ent: assembled entropy words (numpy _coerce_to_uint32_array of the key)
  DRS_HD void init(const uint32_t* ent, int n_ent) {
    uint32_t hc = INIT_A;
    auto hashmix = [&hc](uint32_t v) {
      v ^= hc; hc *= MULT_A; v *= hc; v ^= v >> 16; return v;
    };
    auto mix = [](uint32_t x, uint32_t y) {
      uint32_t r = MIX_L * x - MIX_R * y; r ^= r >> 16; return r;
    };
    for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < n_ent ? ent[i] : 0u);
    for (int s = 0; s < 4; ++s)
      for (int d = 0; d < 4; ++d)
        if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
    for (int s = 4; s < n_ent; ++s)
      for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(ent[s]));
  }
  DRS_HD void generate(uint32_t* out, int n) const {
    uint32_t hb = INIT_B;
    for (int i = 0; i < n; ++i) {
      uint32_t v = pool[i & 3];
      v ^= hb; hb *= MULT_B; v *= hb; v ^= v >> 16;
      out[i] = v;
    }
  }
};

// Turn a drs_key into SeedSequence entropy words (int -> little-endian uint32
// words, 0 -> [0]); returns the word count (<= 8).
DRS_HD int key_words(const drs_key& k, uint64_t seed, uint32_t* w) {
  int n = 0;
  for (int i = 0; i < k.n_vals && i < 4; ++i) {
    uint64_t v = (uint64_t)k.vals[i];
    if (i == 1 && k.seed_slot >= 0) v = seed & k.seed_mask;
    if (v == 0) { w[n++] = 0u; continue; }
    while (v) { w[n++] = (uint32_t)v; v >>= 32; }
  }
  return n;
}

// ------------------------------------------------------------------ PCG64 --
DRS_HD u128 pcg_mult() {
  return ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
}
struct Pcg64 {
  u128 state, inc;
  DRS_HD void seed(const uint32_t* ent, int n_ent) {
    SeedSeq ss; ss.init(ent, n_ent);
    uint32_t w[8]; ss.generate(w, 8);
    uint64_t v[4];
    for (int i = 0; i < 4; ++i) v[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
    const u128 initstate = ((u128)v[0] << 64) | v[1];
    const u128 initseq = ((u128)v[2] << 64) | v[3];
    inc = (initseq << 1) | 1u;
    state = 0;
    state = state * pcg_mult() + inc;
    state += initstate;
    state = state * pcg_mult() + inc;
  }
  DRS_HD static uint64_t output(u128 s) {
    const uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
    const unsigned rot = (unsigned)(s >> 122);
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
  DRS_HD uint64_t next() { state = state * pcg_mult() + inc; return output(state); }
  // affine map of `delta` steps: s -> am * s + ap
  DRS_HD static void jump(u128 inc, uint64_t delta, u128& am, u128& ap) {
    u128 acc_m = 1, acc_p = 0, cur_m = pcg_mult(), cur_p = inc;
    while (delta) {
      if (delta & 1) { acc_m *= cur_m; acc_p = acc_p * cur_m + cur_p; }
      cur_p = (cur_m + 1) * cur_p;
      cur_m *= cur_m;
      delta >>= 1;
    }
    am = acc_m; ap = acc_p;
  }
};

// ------------------------------------------------------------------ SFC64 --
struct Sfc64 {
  uint64_t a, b, c, w;
  DRS_HD void seed(const uint32_t* ent, int n_ent) {
    SeedSeq ss; ss.init(ent, n_ent);
    uint32_t x[6]; ss.generate(x, 6);
    a = (uint64_t)x[0] | ((uint64_t)x[1] << 32);
    b = (uint64_t)x[2] | ((uint64_t)x[3] << 32);
    c = (uint64_t)x[4] | ((uint64_t)x[5] << 32);
    w = 1;
    for (int i = 0; i < 12; ++i) next();
  }
  DRS_HD uint64_t next() {
    const uint64_t tmp = a + b + w++;
    a = b ^ (b >> 11);
    b = c + (c << 3);
    c = ((c << 24) | (c >> 40)) + tmp;
    return tmp;
  }
};

}  // namespace drs
