// fastmath.cuh -- branch-free FP64 exp(-s) for the correlation kernels.
//
// correlation.hpp:193-221 evaluates R_ij = std::exp(-s) (glibc). libdevice exp() is
// accurate but each call is its own branch region (a slow path for |x| >= 708) and loads
// every coefficient through two uniform moves, so the kernels could not interleave the
// exps of several candidates. exp_neg(s) = exp(-s) for any s except NaN, which maps to 0
// (callers test s itself: correlation.hpp:58-61 flags a non-finite value):
//   x = clamp(-s, -1000, 1000); k = rint(x log2 e); r = x - k ln2 (two-constant split, FMA);
//   e^r by degree-13 Taylor on |r| <= ln2/2 (truncation 4e-18); result = (p 2^(k>>1)) 2^(k-(k>>1)),
// the split scale keeps both factors normal so subnormal results are rounded once.
// Accuracy: <= 1 ulp from glibc exp over [0, 745] (tools/expsim.py, exact-FMA emulation;
// 95% of samples bit-equal), the same bound libdevice exp gives.
#pragma once

namespace gpemu_dev {

static __constant__ double kExpTaylor[14] = {
    1.0,
    1.0,
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

__device__ __forceinline__ double exp_neg(double s) {
  // exp(-1000) underflows to 0 like exp(-s) for s > 745.2; exp(1000) overflows to +inf
  const double x = fmin(fmax(-s, -1000.0), 1000.0);
  const double kd = fma(x, 1.4426950408889634, 6755399441055744.0);  // 1.5 * 2^52: rint
  const int k = __double2loint(kd);
  const double kf = kd - 6755399441055744.0;
  double r = fma(kf, -0.6931471805599453, x);  // ln2 = 0.6931471805599453 + 2.319e-17
  r = fma(kf, -2.3190468138462996e-17, r);
  double p = kExpTaylor[13];
#pragma unroll
  for (int j = 12; j >= 0; --j) p = fma(p, r, kExpTaylor[j]);
  const int k1 = k >> 1, k2 = k - k1;  // |k| <= 1443: both halves are normal exponents
  const double e1 = __hiloint2double((k1 + 1023) << 20, 0);
  const double e2 = __hiloint2double((k2 + 1023) << 20, 0);
  return (p * e1) * e2;
}

}  // namespace gpemu_dev
