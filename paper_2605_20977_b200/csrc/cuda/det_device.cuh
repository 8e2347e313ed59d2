// fp64 restatement of the reference's deterministic transcendentals
// (proj/src/det_math.cpp:49-153) for device code. Every translation unit that
// includes this must be compiled with -fmad=false so that each add / mul
// rounds on its own, exactly as the host build (-ffp-contract=off) does:
// results are then bit-identical to the host (test_cdf_tables_bitexact,
// test_tensor_api).
#pragma once
#include <cstdint>

namespace pswa_dev {

__device__ inline double d_pow2i(int k) {
  if (k > 1023) return __longlong_as_double(0x7FF0000000000000LL);
  if (k < -1074) return 0.0;
  if (k >= -1022) return __longlong_as_double(static_cast<long long>(k + 1023) << 52);
  return __longlong_as_double(1LL << (k + 1074));
}
__device__ inline double d_exp(double x) {
  if (x != x) return x;
  if (x > 709.782712893384) return __longlong_as_double(0x7FF0000000000000LL);
  if (x < -745.1332191019412) return 0.0;
  const double t = x * 1.44269504088896338700e+00;
  const int n = static_cast<int>(t >= 0.0 ? t + 0.5 : t - 0.5);
  const double nd = n;
  const double r = (x - nd * 6.93147180369123816490e-01) - nd * 1.90821492927058770002e-10;
  const double c[11] = {1.0 / 6227020800.0, 1.0 / 479001600.0, 1.0 / 39916800.0,
                        1.0 / 3628800.0,    1.0 / 362880.0,    1.0 / 40320.0,
                        1.0 / 5040.0,       1.0 / 720.0,       1.0 / 120.0,
                        1.0 / 24.0,         1.0 / 6.0};
  double p = c[0];
#pragma unroll
  for (int i = 1; i < 11; ++i) p = p * r + c[i];
  const double rr = r * r;
  return (1.0 + r + 0.5 * rr + rr * r * p) * d_pow2i(n);
}
__device__ inline double d_log(double x) {
  long long b = __double_as_longlong(x);
  int e = 0;
  if (b < (1LL << 52)) {
    x *= 18014398509481984.0;  // 2^54
    e = -54;
    b = __double_as_longlong(x);
  }
  e += static_cast<int>((b >> 52) & 0x7FF) - 1023;
  double m = __longlong_as_double((b & ((1LL << 52) - 1)) | (1023LL << 52));
  if (m > 1.4142135623730951) {
    m *= 0.5;
    e += 1;
  }
  const double f = m - 1.0, s = f / (2.0 + f), z = s * s, w = z * z;
  const double t1 = w * (3.999999999940941908e-01 +
                         w * (2.222219843214978396e-01 + w * 1.531383769920937332e-01));
  const double t2 = z * (6.666666666666735130e-01 +
                         w * (2.857142874366239149e-01 +
                              w * (1.818357216161805012e-01 + w * 1.479819860511658591e-01)));
  const double hf = 0.5 * f * f, R = t2 + t1, ed = e;
  return ed * 6.93147180369123816490e-01 -
         ((hf - (s * (hf + R) + ed * 1.90821492927058770002e-10)) - f);
}
__device__ inline double d_erf(double x) {
  const double a = x < 0.0 ? -x : x;
  const double t = 1.0 / (1.0 + 0.3275911 * a);
  const double poly =
      t * (0.254829592 +
           t * (-0.284496736 + t * (1.421413741 + t * (-1.453152027 + t * 1.061405429))));
  const double y = 1.0 - poly * d_exp(-a * a);
  return x < 0.0 ? -y : y;
}

// det::exp_f32 / silu_f32 (det_math.cpp:132-137)
__device__ inline float d_exp_f32(float x) { return static_cast<float>(d_exp(static_cast<double>(x))); }
__device__ inline float d_silu_f32(float x) {
  const double xd = x;
  return static_cast<float>(xd / (1.0 + d_exp(-xd)));
}

}  // namespace pswa_dev
