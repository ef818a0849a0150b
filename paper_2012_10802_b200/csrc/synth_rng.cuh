// synth_rng.cuh — the random streams of the reference scene generator
// (synth.cpp:16-149), restated so that the device reproduces libstdc++'s
// std::mt19937 / uniform_real_distribution / normal_distribution bit for bit.
//
// Host + device: tests/cpp/synth_rng_check.cpp compiles this header with g++
// and checks every function against <random> (the CPU suite), the kernels in
// abi_synth.cu use it on sm_100a.  All double arithmetic is plain IEEE
// (the library is built with --fmad=false), fma() appears only inside the
// exact error-free transforms.
#pragma once

#include <cmath>
#include <cstdint>

#ifdef __CUDACC__
#define RPD_HD __host__ __device__ __forceinline__
#else
#define RPD_HD inline
#endif
#ifdef __CUDA_ARCH__
#define RPD_UNROLL _Pragma("unroll")
#else
#define RPD_UNROLL
#endif

namespace rpd_synth {

// ---- std::mt19937 (N = 624, M = 397) ---------------------------------------
// As a sequence: x[0..623] is the seeded state and, for n >= 624,
//   x[n] = x[n-227] ^ t[n-624],   t[m] = twist(x[m], x[m+1]);
// the k-th output is temper(x[624 + k]).
constexpr int kMtN = 624;
constexpr uint32_t kMtMatrixA = 0x9908b0dfu;

RPD_HD uint32_t mt_seed_next(uint32_t prev, uint32_t i) {
  return 1812433253u * (prev ^ (prev >> 30)) + i;
}

RPD_HD uint32_t mt_twist(uint32_t xm, uint32_t xm1) {
  const uint32_t y = (xm & 0x80000000u) | (xm1 & 0x7fffffffu);
  return (y >> 1) ^ ((y & 1u) ? kMtMatrixA : 0u);
}

// Word n >= 624 from words at least kMtRound back: the x[n-227] link unrolled
// twice, so a block computes kMtRound = 620 consecutive words at once (the
// nearest in-round dependency is x[n-623] through t[n-624]; 620 keeps rounds
// aligned to the 4 draws of a polar attempt).  x(i) / t(i) read the history.
constexpr int kMtRound = 620;
template <class I, class XF, class TF>
RPD_HD uint32_t mt_word(I n, XF x, TF t) {
  if (n < 851) return x(n - 227) ^ t(n - 624);
  if (n < 1078) return x(n - 454) ^ t(n - 851) ^ t(n - 624);
  return x(n - 681) ^ t(n - 1078) ^ t(n - 851) ^ t(n - 624);
}

RPD_HD uint32_t mt_temper(uint32_t y) {
  y ^= y >> 11;
  y ^= (y << 7) & 0x9d2c5680u;
  y ^= (y << 15) & 0xefc60000u;
  y ^= y >> 18;
  return y;
}

// ---- libstdc++ generate_canonical -------------------------------------------
// float (24 bits): one 32-bit draw, float(o) / 2^32, clamped below 1.
RPD_HD float canonical_f32(uint32_t o) {
  const float r = static_cast<float>(o) * 2.3283064365386963e-10f;  // exact: / 2^32
  return r >= 1.0f ? 0.99999994f : r;                                 // nextafter(1, 0)
}
// double (53 bits): two draws, (o0 + o1 * 2^32) / 2^64, clamped below 1.
RPD_HD double canonical_f64(uint32_t o0, uint32_t o1) {
  const double s = static_cast<double>(o0) + static_cast<double>(o1) * 4294967296.0;
  const double r = s * 5.421010862427522e-20;  // exact: / 2^64
  return r >= 1.0 ? 0.99999999999999989 : r;
}

// normal_distribution<double> (Marsaglia polar): an attempt takes four draws,
// x = 2 u(o0,o1) - 1, y = 2 u(o2,o3) - 1, accepted when 0 < x^2 + y^2 <= 1.
// An accepted pair returns y * m first, then x * m, m = sqrt(-2 ln r2 / r2).
RPD_HD bool polar_attempt(uint32_t o0, uint32_t o1, uint32_t o2, uint32_t o3, double& x,
                          double& y) {
  x = 2.0 * canonical_f64(o0, o1) - 1.0;
  y = 2.0 * canonical_f64(o2, o3) - 1.0;
  const double r2 = x * x + y * y;
  return !(r2 > 1.0 || r2 == 0.0);
}

// ---- log(r2), r2 in (0, 1], in double-double, rounded once ----------------
// Correctly rounded with overwhelming probability, so it equals glibc's log
// (itself within 0.52 ulp) except in astronomically rare hard cases.
struct Dd {
  double hi, lo;
};
RPD_HD Dd dd_two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
RPD_HD Dd dd_fast_two_sum(double a, double b) {
  const double s = a + b;
  return {s, b - (s - a)};
}
RPD_HD Dd dd_add(Dd a, Dd b) {
  Dd s = dd_two_sum(a.hi, b.hi);
  const Dd t = dd_two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = dd_fast_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return dd_fast_two_sum(s.hi, s.lo);
}
RPD_HD Dd dd_mul(Dd a, Dd b) {
  const double p = a.hi * b.hi;
  double e = fma(a.hi, b.hi, -p);
  e += a.hi * b.lo + a.lo * b.hi;
  return dd_fast_two_sum(p, e);
}
RPD_HD Dd dd_div(Dd a, Dd b) {
  const double q1 = a.hi / b.hi;
  // r = a - q1 * b
  const double p = q1 * b.hi;
  const double pe = fma(q1, b.hi, -p);
  Dd r = dd_two_sum(a.hi, -p);
  r.lo += a.lo - pe - q1 * b.lo;
  r = dd_fast_two_sum(r.hi, r.lo);
  const double q2 = r.hi / b.hi;
  return dd_fast_two_sum(q1, q2);
}
RPD_HD double log_dd(double r2) {
  // r2 = m 2^e with m in [sqrt(1/2), sqrt(2))
  int e = 0;
  double m = frexp(r2, &e);  // m in [0.5, 1)
  if (m < 0.70710678118654752) {
    m *= 2.0;
    e -= 1;
  }
  // log m = 2 atanh(s), s = (m - 1) / (m + 1)
  const Dd num = {m - 1.0, 0.0};  // exact (Sterbenz)
  const Dd den = dd_two_sum(m, 1.0);
  const Dd s = dd_div(num, den);
  const Dd s2 = dd_mul(s, s);
  // P(s2) = sum_k s2^k / (2k+1): tail k = 22..6 in double, head k = 5..0 in
  // double-double (coefficients: 1/(2k+1) correctly rounded, plus the residual)
  const double tail_c[17] = {
      0.022222222222222223, 0.023255813953488372, 0.024390243902439025, 0.02564102564102564,
      0.02702702702702703, 0.02857142857142857, 0.030303030303030304, 0.03225806451612903,
      0.034482758620689655, 0.037037037037037035, 0.04, 0.043478260869565216,
      0.047619047619047616, 0.05263157894736842, 0.058823529411764705, 0.06666666666666667,
      0.07692307692307693};
  double tail = tail_c[0];
RPD_UNROLL
  for (int k = 1; k < 17; ++k) tail = tail * s2.hi + tail_c[k];
  const Dd head_c[6] = {
      {0.09090909090909091, -2.523234146875356e-18},
      {0.1111111111111111, 6.1679056923619804e-18},
      {0.14285714285714285, 7.93016446160826e-18},
      {0.2, -1.1102230246251566e-17},
      {0.3333333333333333, 1.850371707708594e-17},
      {1.0, 0.0}};
  Dd p = {tail, 0.0};
RPD_UNROLL
  for (int k = 0; k < 6; ++k) p = dd_add(dd_mul(p, s2), head_c[k]);
  Dd lm = dd_mul(s, p);
  lm.hi *= 2.0;
  lm.lo *= 2.0;
  // + e ln 2
  const double ln2_hi = 0.69314718055994529, ln2_lo = 2.3190468138462996e-17;
  const double ed = static_cast<double>(e);
  const double eh = ed * ln2_hi;
  const Dd el = {eh, fma(ed, ln2_hi, -eh) + ed * ln2_lo};
  const Dd r = dd_add(el, lm);
  return r.hi;
}

// One normal pair of the polar method: (first, second) = (y m, x m).
RPD_HD void polar_pair(double x, double y, double& first, double& second) {
  const double r2 = x * x + y * y;
  const double mult = sqrt(-2 * log_dd(r2) / r2);
  first = y * mult;
  second = x * mult;
}

}  // namespace rpd_synth
