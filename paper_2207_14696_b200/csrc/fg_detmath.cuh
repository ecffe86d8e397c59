// Deterministic float64 elementary functions for the synthetic generators.
//
// The generators (fg_data.cu) must produce bit-identical graphs and features
// on the device and in the C restatement that builds the CPU reference arm's
// world (oracle/fgoracle.c, SURVEY.md §8d "row-addressable generator").  CUDA's
// pow/log/cos and their fast intrinsics are not correctly rounded, so they
// differ from glibc in the last ulp -- enough to move a truncated power-law
// rank once in ~10^8 edges.  These functions use only IEEE-rounded add / mul
// / fma / div / sqrt, written with explicit-rounding intrinsics so nvcc never
// contracts or reorders them; the C side performs the same operations in the
// same order (fma() and -ffp-contract=off), so both produce the same bits.
// Accuracy is ~1e-15 relative, which is all a generator needs.
#pragma once

#include <stdint.h>

namespace fg {
namespace det {

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double fma(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }

// log2(x) for finite x > 0 (normal range): x = m 2^e with m in [sqrt(1/2),
// sqrt(2)], ln m = 2 atanh(s), s = (m - 1) / (m + 1), |s| <= 0.1716.
__device__ __forceinline__ double log2(double x) {
  const uint64_t b = (uint64_t)__double_as_longlong(x);
  int e = (int)((b >> 52) & 0x7FF) - 1023;
  double m = __longlong_as_double((long long)((b & 0xFFFFFFFFFFFFFull) | (1023ull << 52)));
  if (m > 0x1.6a09e667f3bcdp+0) {  // sqrt(2)
    m = mul(m, 0.5);
    e += 1;
  }
  const double s = div(sub(m, 1.0), add(m, 1.0));
  const double s2 = mul(s, s);
  double p = 0x1.47ae147ae147bp-5;  // 1/25
  p = fma(p, s2, 0x1.642c8590b2164p-5);
  p = fma(p, s2, 0x1.8618618618618p-5);
  p = fma(p, s2, 0x1.af286bca1af28p-5);
  p = fma(p, s2, 0x1.e1e1e1e1e1e1ep-5);
  p = fma(p, s2, 0x1.1111111111111p-4);
  p = fma(p, s2, 0x1.3b13b13b13b14p-4);
  p = fma(p, s2, 0x1.745d1745d1746p-4);
  p = fma(p, s2, 0x1.c71c71c71c71cp-4);
  p = fma(p, s2, 0x1.2492492492492p-3);
  p = fma(p, s2, 0x1.999999999999ap-3);
  p = fma(p, s2, 0x1.5555555555555p-2);
  p = fma(p, s2, 1.0);
  const double ln_m = mul(mul(2.0, s), p);
  return fma(ln_m, 0x1.71547652b82fep+0, (double)e);  // ln_m / ln 2 + e
}

// 2^y for |y| < 1000: y = k + f, |f| <= 1/2, 2^f = e^(f ln 2) by Taylor.
__device__ __forceinline__ double exp2(double y) {
  const double k = floor(add(y, 0.5));
  const double t = mul(sub(y, k), 0x1.62e42fefa39efp-1);
  double p = 0x1.93974a8c07c9dp-37;  // 1/14!
  p = fma(p, t, 0x1.6124613a86d09p-33);
  p = fma(p, t, 0x1.1eed8eff8d898p-29);
  p = fma(p, t, 0x1.ae64567f544e4p-26);
  p = fma(p, t, 0x1.27e4fb7789f5cp-22);
  p = fma(p, t, 0x1.71de3a556c734p-19);
  p = fma(p, t, 0x1.a01a01a01a01ap-16);
  p = fma(p, t, 0x1.a01a01a01a01ap-13);
  p = fma(p, t, 0x1.6c16c16c16c17p-10);
  p = fma(p, t, 0x1.1111111111111p-7);
  p = fma(p, t, 0x1.5555555555555p-5);
  p = fma(p, t, 0x1.5555555555555p-3);
  p = fma(p, t, 0.5);
  p = fma(p, t, 1.0);
  p = fma(p, t, 1.0);
  const double scale = __longlong_as_double((long long)((uint64_t)((int64_t)k + 1023) << 52));
  return mul(p, scale);
}

// base^e for base >= 1 (the generator's only use)
__device__ __forceinline__ double pow(double base, double e) { return exp2(mul(e, log2(base))); }

// cos(2 pi t) for t in [0, 1): quadrant q = floor(4t), theta = 2 pi (t - q/4)
// in [0, pi/2), then the Taylor series of cos / sin.
__device__ __forceinline__ double cos_turns(double t) {
  const double q = floor(mul(t, 4.0));
  const double th = mul(sub(t, mul(q, 0.25)), 0x1.921fb54442d18p+2);
  const double t2 = mul(th, th);
  double c = 0x1.0ce396db7f853p-70;  // 1/22!
  c = fma(c, -t2, 0x1.e542ba4020225p-62);
  c = fma(c, -t2, 0x1.6827863b97d97p-53);
  c = fma(c, -t2, 0x1.ae7f3e733b81fp-45);
  c = fma(c, -t2, 0x1.93974a8c07c9dp-37);
  c = fma(c, -t2, 0x1.1eed8eff8d898p-29);
  c = fma(c, -t2, 0x1.27e4fb7789f5cp-22);
  c = fma(c, -t2, 0x1.a01a01a01a01ap-16);
  c = fma(c, -t2, 0x1.6c16c16c16c17p-10);
  c = fma(c, -t2, 0x1.5555555555555p-5);
  c = fma(c, -t2, 0.5);
  c = fma(c, -t2, 1.0);
  double s = 0x1.71b8ef6dcf572p-66;  // 1/21!
  s = fma(s, -t2, 0x1.2f49b46814157p-57);
  s = fma(s, -t2, 0x1.952c77030ad4ap-49);
  s = fma(s, -t2, 0x1.ae7f3e733b81fp-41);
  s = fma(s, -t2, 0x1.6124613a86d09p-33);
  s = fma(s, -t2, 0x1.ae64567f544e4p-26);
  s = fma(s, -t2, 0x1.71de3a556c734p-19);
  s = fma(s, -t2, 0x1.a01a01a01a01ap-13);
  s = fma(s, -t2, 0x1.1111111111111p-7);
  s = fma(s, -t2, 0x1.5555555555555p-3);
  s = fma(s, -t2, 1.0);
  s = mul(s, th);
  const int qi = (int)q;
  return qi == 0 ? c : qi == 1 ? -s : qi == 2 ? -c : s;
}

}  // namespace det
}  // namespace fg
