// Host implementation of pswa/det_math.h (the reference contract of
// proj/src/det_math.cpp:49-153): Cody-Waite exp with a degree-13 Taylor
// core, fdlibm log, A&S 7.1.26 erf. Built with -ffp-contract=off.
#include "pswa/det_math.h"

#include <bit>
#include <cstdint>
#include <limits>

namespace pswa::det {

namespace {
constexpr double kInf = std::numeric_limits<double>::infinity();

double exact_pow2(int k) {
  if (k > 1023) return kInf;
  if (k < -1074) return 0.0;
  const uint64_t bits = k >= -1022 ? static_cast<uint64_t>(k + 1023) << 52
                                   : uint64_t{1} << (k + 1074);
  return std::bit_cast<double>(bits);
}
}  // namespace

double exp(double x) {
  if (x != x) return x;
  if (x > 709.782712893384) return kInf;
  if (x < -745.1332191019412) return 0.0;
  const double t = x * 1.44269504088896338700e+00;
  const int k = static_cast<int>(t >= 0.0 ? t + 0.5 : t - 0.5);
  const double kd = k;
  const double r = (x - kd * 6.93147180369123816490e-01) - kd * 1.90821492927058770002e-10;
  static constexpr double kInvFact[11] = {
      1.0 / 6227020800.0, 1.0 / 479001600.0, 1.0 / 39916800.0, 1.0 / 3628800.0,
      1.0 / 362880.0,     1.0 / 40320.0,     1.0 / 5040.0,     1.0 / 720.0,
      1.0 / 120.0,        1.0 / 24.0,        1.0 / 6.0};
  double p = kInvFact[0];
  for (int i = 1; i < 11; ++i) p = p * r + kInvFact[i];
  const double r2 = r * r;
  return (1.0 + r + 0.5 * r2 + r2 * r * p) * exact_pow2(k);
}

double log(double x) {
  if (x != x) return x;
  if (x < 0.0) return std::numeric_limits<double>::quiet_NaN();
  if (x == 0.0) return -kInf;
  if (x == kInf) return x;
  uint64_t b = std::bit_cast<uint64_t>(x);
  int e = 0;
  if (b < (uint64_t{1} << 52)) {
    x *= 0x1p54;
    e = -54;
    b = std::bit_cast<uint64_t>(x);
  }
  e += static_cast<int>((b >> 52) & 0x7FF) - 1023;
  double m = std::bit_cast<double>((b & 0x000FFFFFFFFFFFFFULL) | (uint64_t{1023} << 52));
  if (m > 1.4142135623730951) {
    m *= 0.5;
    ++e;
  }
  const double f = m - 1.0, s = f / (2.0 + f), z = s * s, w = z * z;
  const double t1 = w * (3.999999999940941908e-01 +
                         w * (2.222219843214978396e-01 + w * 1.531383769920937332e-01));
  const double t2 = z * (6.666666666666735130e-01 +
                         w * (2.857142874366239149e-01 +
                              w * (1.818357216161805012e-01 + w * 1.479819860511658591e-01)));
  const double hf = 0.5 * f * f, ed = e;
  return ed * 6.93147180369123816490e-01 -
         ((hf - (s * (hf + (t2 + t1)) + ed * 1.90821492927058770002e-10)) - f);
}

double erf(double x) {
  const double a = x < 0.0 ? -x : x;
  const double t = 1.0 / (1.0 + 0.3275911 * a);
  const double poly =
      t * (0.254829592 +
           t * (-0.284496736 + t * (1.421413741 + t * (-1.453152027 + t * 1.061405429))));
  const double y = 1.0 - poly * det::exp(-a * a);
  return x < 0.0 ? -y : y;
}

double normal_cdf(double x) { return 0.5 * (1.0 + det::erf(x * 0.7071067811865475244)); }
float exp_f32(float x) { return static_cast<float>(det::exp(x)); }
float silu_f32(float x) {
  const double v = x;
  return static_cast<float>(v / (1.0 + det::exp(-v)));
}
float tanh_f32(float x) {
  const double v = x, a = v < 0.0 ? -v : v;
  if (a > 20.0) return x < 0.0f ? -1.0f : 1.0f;
  const double y = 1.0 - 2.0 / (det::exp(2.0 * a) + 1.0);
  return static_cast<float>(v < 0.0 ? -y : y);
}
float softplus_f32(float x) {
  const double v = x;
  if (v > 30.0) return x;
  if (v < -30.0) return static_cast<float>(det::exp(v));
  return static_cast<float>(det::log(1.0 + det::exp(v)));
}

}  // namespace pswa::det
