// Bit-exact ports of the two libm routines numpy's ziggurat calls on its slow
// paths (numpy random_standard_normal: wedge test uses exp(), tail uses
// npy_log1p()).  The reference's noise (skipdiff rng.py:32-33) therefore
// depends on the host libm; the golden vectors were produced on glibc 2.39
// (Ubuntu 2.39-0ubuntu8.5) on an FMA/AVX2 host, where both functions resolve
// through IFUNC to their `-mfma -mavx2` builds:
//   log1p -> __log1p_fma  (fdlibm s_log1p.c, GCC contracted a*b+c into FMA)
//   exp   -> __exp_fma    (ARM optimized-routines exp, N=128, poly order 5)
// Every fma() below sits exactly where the disassembly of those builds has a
// vfmadd/vfnmadd/vfmsub; every other operation is a separately rounded IEEE
// op.  The translation unit MUST be compiled with contraction disabled
// (nvcc --fmad=false, host -ffp-contract=off) so no further fusing happens.
// tests/test_glibc_math.py checks both against the host libm bit-for-bit.
#pragma once
#include <stdint.h>
#include <math.h>

#ifdef __CUDACC__
#define DRS_HD __host__ __device__ __forceinline__
#else
#define DRS_HD static inline
#endif

#include "gen_tables.h"

namespace drs {

DRS_HD uint64_t asu64(double x) {
#ifdef __CUDA_ARCH__
  return (uint64_t)__double_as_longlong(x);
#else
  union { double d; uint64_t u; } v; v.d = x; return v.u;
#endif
}
DRS_HD double asf64(uint64_t u) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)u);
#else
  union { double d; uint64_t u; } v; v.u = u; return v.d;
#endif
}
DRS_HD double dfma(double a, double b, double c) {
#ifdef __CUDA_ARCH__
  return __fma_rn(a, b, c);
#else
  return fma(a, b, c);
#endif
}

// ---------------------------------------------------------------- log1p ----
DRS_HD double log1p_glibc(double x) {
  const double ln2_hi = 6.93147180369123816490e-01;  // 3fe62e42 fee00000
  const double ln2_lo = 1.90821492927058770002e-10;  // 3dea39ef 35793c76
  const double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01,
               Lp3 = 2.857142874366239149e-01, Lp4 = 2.222219843214978396e-01,
               Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
               Lp7 = 1.479819860511658591e-01;
  const uint64_t bits = asu64(x);
  const int32_t hx = (int32_t)(bits >> 32);
  const int32_t ax = hx & 0x7fffffff;
  int32_t k = 1, hu = 0;
  double f = 0.0, c = 0.0;
  if (hx < 0x3FDA827A) {                 // x < 0.41422
    if (ax >= 0x3ff00000) {              // x <= -1.0
      if (x == -1.0) return -INFINITY;
      return NAN;
    }
    if (ax < 0x3e200000) {               // |x| < 2**-29
      if (ax < 0x3c900000) return x;     // |x| < 2**-54
      return dfma(-(x * x), 0.5, x);     // vfnmadd231sd
    }
    if (hx > 0 || hx <= (int32_t)0xbfd2bec3) { k = 0; f = x; hu = 1; }  // -0.2929<x<0.41422
  } else if (hx >= 0x7ff00000) {
    return x + x;
  }
  if (k != 0) {
    double u;
    if (hx < 0x43400000) {
      u = 1.0 + x;
      hu = (int32_t)(asu64(u) >> 32);
      k = (hu >> 20) - 1023;
      c = (k > 0) ? 1.0 - (u - x) : x - (u - 1.0);
      c = c / u;
    } else {
      u = x;
      hu = (int32_t)(asu64(u) >> 32);
      k = (hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffff;
    const uint64_t lo = asu64(u) & 0xffffffffull;
    if (hu < 0x6a09e) {
      u = asf64(((uint64_t)(uint32_t)(hu | 0x3ff00000) << 32) | lo);
    } else {
      k += 1;
      u = asf64(((uint64_t)(uint32_t)(hu | 0x3fe00000) << 32) | lo);
      hu = (0x00100000 - hu) >> 2;
    }
    f = u - 1.0;
  }
  const double hfsq = (0.5 * f) * f;
  if (hu == 0) {                          // |f| < 2**-20
    if (f == 0.0) {
      if (k == 0) return 0.0;
      const double dk = (double)k;
      c = dfma(dk, ln2_lo, c);
      return dfma(dk, ln2_hi, c);
    }
    const double R = dfma(-f, 0.66666666666666666, 1.0) * hfsq;
    if (k == 0) return f - R;
    const double dk = (double)k;
    return dfma(dk, ln2_hi, -((R - dfma(dk, ln2_lo, c)) - f));
  }
  const double s = f / (2.0 + f);
  const double z = s * s;
  const double R2 = dfma(z, Lp3, Lp2);
  const double R3 = dfma(z, Lp5, Lp4);
  const double R4 = dfma(z, Lp7, Lp6);
  const double z2 = z * z;
  const double z4 = z2 * z2;
  const double z6 = z2 * z4;
  double R = dfma(z, Lp1, z2 * R2);
  R = dfma(z4, R3, R);
  R = dfma(z6, R4, R);
  const double t = s * (hfsq + R);
  if (k == 0) return f - (hfsq - t);
  const double dk = (double)k;
  const double cc = dfma(dk, ln2_lo, c);
  return dfma(dk, ln2_hi, -((hfsq - (cc + t)) - f));
}

// ------------------------------------------------------------------ exp ----
#ifdef __CUDACC__
__device__ const uint64_t kExpTab[256] = DRS_EXP_TAB;
#endif
static const uint64_t kExpTabHost[256] = DRS_EXP_TAB;
#ifdef __CUDA_ARCH__
#define DRS_EXPTAB kExpTab
#else
#define DRS_EXPTAB kExpTabHost
#endif

DRS_HD double exp_specialcase(double tmp, uint64_t sbits, uint64_t ki) {
  if ((ki & 0x80000000ull) == 0) {        // k > 0: exponent of scale might have overflowed by <= 460
    sbits -= 1009ull << 52;
    const double scale = asf64(sbits);
    return 0x1p1009 * dfma(scale, tmp, scale);
  }
  sbits += 1022ull << 52;                 // k < 0: need special care in the subnormal range
  const double scale = asf64(sbits);
  double y = scale + scale * tmp;
  if (y < 1.0) {
    double lo = scale - y + scale * tmp;
    const double hi = 1.0 + y;
    lo = 1.0 - hi + y + lo;
    y = (hi + lo) - 1.0;
    if (y == 0.0) y = 0.0;
  }
  return 0x1p-1022 * y;
}

DRS_HD double exp_glibc(double x) {
  const double InvLn2N = 0x1.71547652b82fep7, Shift = 0x1.8p52;
  const double NegLn2hiN = -0x1.62e42fefa0000p-8, NegLn2loN = -0x1.cf79abc9e3b3ap-47;
  const double C2 = 0x1.ffffffffffdbdp-2, C3 = 0x1.555555555543cp-3,
               C4 = 0x1.55555cf172b91p-5, C5 = 0x1.1111167a4d017p-7;
  const uint64_t ix = asu64(x);
  uint32_t abstop = (uint32_t)(ix >> 52) & 0x7ff;
  if (abstop - 0x3c9u > 0x3eu) {
    if ((int32_t)(abstop - 0x3c9u) < 0) return 1.0 + x;   // tiny x
    if (abstop >= 0x409u) {
      if (ix == 0xfff0000000000000ull) return 0.0;
      if (abstop >= 0x7ffu) return 1.0 + x;
      return (ix >> 63) ? 0.0 : INFINITY;
    }
    abstop = 0;                                           // large x: special-cased below
  }
  double kd = dfma(x, InvLn2N, Shift);
  const uint64_t ki = asu64(kd);
  kd = kd - Shift;
  double r = dfma(kd, NegLn2hiN, x);
  r = dfma(kd, NegLn2loN, r);
  const uint64_t idx = 2 * (ki & 127);
  const uint64_t top = ki << 45;
  const double tail = asf64(DRS_EXPTAB[idx]);
  const uint64_t sbits = DRS_EXPTAB[idx + 1] + top;
  const double r2 = r * r;
  const double p23 = dfma(r, C3, C2);
  const double p45 = dfma(r, C5, C4);
  double tmp = dfma(p23, r2, tail + r);
  tmp = dfma(r2 * r2, p45, tmp);
  if (abstop == 0) return exp_specialcase(tmp, sbits, ki);
  const double scale = asf64(sbits);
  return dfma(scale, tmp, scale);
}

}  // namespace drs
