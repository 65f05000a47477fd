// fastmath.cuh -- branch-free FP64 exp(-s), log and |d|^p for the correlation kernels.
//
// correlation.hpp:29-34 and :193-221 evaluate |d|^p = std::exp(p * std::log|d|) and
// R_ij = std::exp(-s) with glibc. libdevice exp()/log() are accurate but each call is its own
// branch region (slow paths for extreme arguments) and loads every coefficient through two
// uniform moves, so kernels could not interleave the transcendentals of several candidates or
// dimensions. These versions are straight-line code, and they carry the leading terms in
// double-double so the single final rounding lands on glibc's result in ~98% of cases
// (tools/fastmath_sim.py: exact-FMA emulation vs glibc; never more than 1 ulp from it for
// exp / log, and the composed |d|^p has no multi-ulp tail).
#pragma once

namespace gpemu_dev {

// 1/j! for j = 2..13: e^r = 1 + r + r^2 P(r), truncation < 5e-18 on |r| <= ln2/2.
static __constant__ double kExpP[12] = {
    0.5,
    0.16666666666666666,
    0.041666666666666664,
    0.008333333333333333,
    0.001388888888888889,
    0.0001984126984126984,
    2.48015873015873e-05,
    2.7557319223985893e-06,
    2.755731922398589e-07,
    2.505210838544172e-08,
    2.08767569878681e-09,
    1.6059043836821613e-10,
};

// fdlibm split of ln2: k * kLn2Hi is exact for |k| < 2^21.
constexpr double kLn2Hi = 6.93147180369123816490e-01;
constexpr double kLn2Lo = 1.90821492927058770002e-10;

// exp(-s) for any s except NaN, which maps to 0 (callers test s: correlation.hpp:58-61).
//   x = clamp(-s, -1000, 1000) (exp(-1000) underflows to 0 and exp(1000) overflows to inf,
//   as the unclamped values do); k = rint(x log2 e); r_hi = x - k ln2_hi (exact),
//   r_lo = -k ln2_lo; e^r = (1 + r_hi) [Fast2Sum] + (r^2 P(r) + r_lo);
//   result = (e^r 2^(k>>1)) 2^(k - (k>>1)): both scale factors are normal, so subnormal
//   results are rounded once.
template <bool kClampHigh>
__device__ __forceinline__ double exp_core(double x) {
  x = fmax(x, -1000.0);
  if (kClampHigh) x = fmin(x, 1000.0);
  const double kd = fma(x, 1.4426950408889634, 6755399441055744.0);  // 1.5 * 2^52: rint
  const int k = __double2loint(kd);
  const double kf = kd - 6755399441055744.0;
  const double rh = fma(kf, -kLn2Hi, x);
  const double rl = __dmul_rn(kf, -kLn2Lo);
  const double r = __dadd_rn(rh, rl);
  double P = kExpP[11];
#pragma unroll
  for (int j = 10; j >= 0; --j) P = fma(P, r, kExpP[j]);
  const double t = fma(__dmul_rn(r, r), P, rl);
  const double hi = __dadd_rn(1.0, rh);
  const double lo = __dadd_rn(__dsub_rn(1.0, hi), rh);
  const double e = __dadd_rn(hi, __dadd_rn(lo, t));
  const int k1 = k >> 1, k2 = k - k1;  // |k| <= 1443: both halves are normal exponents
  return (e * __hiloint2double((k1 + 1023) << 20, 0)) * __hiloint2double((k2 + 1023) << 20, 0);
}

__device__ __forceinline__ double exp_neg(double s) { return exp_core<true>(-s); }

// Fast2Sum: s + err == a + b exactly when |a| >= |b| (or a == 0).
__device__ __forceinline__ double fast_two_sum(double a, double b, double& err) {
  const double s = __dadd_rn(a, b);
  err = __dsub_rn(b, __dsub_rn(s, a));
  return s;
}

// log(a) for finite a > 0 (subnormals included): fdlibm e_log.c reduction and minimax
// coefficients Lg1..Lg7, a = 2^k m, m in [sqrt(2)/2, sqrt(2)), f = m - 1, s = f / (2 + f),
// log m = (f - f^2/2) + (s (f^2/2 + R(s^2)) - lo(f^2/2)); f - f^2/2 and k ln2_hi + (f - f^2/2)
// are exact Fast2Sums (|f^2/2| <= 0.21 |f|; |k ln2_hi| >= 0.69 > |log m| or k = 0) so only
// the last addition rounds. The division is an rcp.approx seed +
// two FMA Newton steps (2 + f lies in [1.29, 2.42]: no special cases).
__device__ __forceinline__ double log_pos(double a) {
  const bool sub = a < 2.2250738585072014e-308;
  const double a2 = sub ? a * 18014398509481984.0 : a;  // 2^54
  int hx = __double2hiint(a2);
  int k = (hx >> 20) - 1023 - (sub ? 54 : 0);
  hx &= 0x000fffff;
  const int i = (hx + 0x95f64) & 0x100000;  // m >= sqrt(2): halve it
  const double m = __hiloint2double(hx | (i ^ 0x3ff00000), __double2loint(a2));
  k += i >> 20;
  const double f = __dsub_rn(m, 1.0);
  const double den = __dadd_rn(2.0, f);
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(den));
  r = fma(r, fma(-den, r, 1.0), r);
  r = fma(r, fma(-den, r, 1.0), r);
  const double s = __dmul_rn(f, r);
  const double hf = __dmul_rn(0.5, f);
  const double hfsq = __dmul_rn(hf, f);
  const double hfsq_lo = fma(hf, f, -hfsq);
  const double z = __dmul_rn(s, s), w = __dmul_rn(z, z);
  const double t1 = __dmul_rn(w, fma(w, fma(w, 1.531383769920937332e-01, 2.222219843214978396e-01),
                                     3.999999999940941908e-01));
  const double t2 = __dmul_rn(z, fma(w, fma(w, fma(w, 1.479819860511658591e-01, 1.818357216161805012e-01),
                                            2.857142874366239149e-01),
                                     6.666666666666735130e-01));
  const double c = fma(s, __dadd_rn(hfsq, __dadd_rn(t2, t1)), -hfsq_lo);
  double dl, rl;
  const double dh = fast_two_sum(f, -hfsq, dl);
  const double dk = (double)k;
  const double rh = fast_two_sum(__dmul_rn(dk, kLn2Hi), dh, rl);
  return __dadd_rn(rh, __dadd_rn(rl, __dadd_rn(dl, fma(dk, kLn2Lo, c))));
}

// detail::pow_abs (correlation.hpp:29-34): |delta|^p = exp(p log|delta|), 0 -> 0, branch-free.
__device__ __forceinline__ double pow_abs_fast(double delta, double p) {
  // p log a <= p log(1 + 2e-12): no upper clamp needed; log_pos(0) is finite (-746.5, via the
  // subnormal path) and its result is discarded by the select.
  const double a = fabs(delta);
  const double v = exp_core<false>(__dmul_rn(p, log_pos(a)));
  return a == 0.0 ? 0.0 : v;
}

}  // namespace gpemu_dev
