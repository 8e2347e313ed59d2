// pswa/det_math.h — platform-bit-identical transcendentals (drop-in for the
// reference's proj/include/pswa/det_math.h:25-36; same names). Implemented
// with IEEE add/mul/div only; the device copy used to build the CDF tables
// lives in csrc/cuda/coder.cu and is compiled with -fmad=false.
#ifndef PSWA_DET_MATH_H_
#define PSWA_DET_MATH_H_

namespace pswa::det {

double exp(double x);
double log(double x);
double erf(double x);  // Abramowitz & Stegun 7.1.26
double normal_cdf(double x);
float exp_f32(float x);
float silu_f32(float x);
float tanh_f32(float x);
float softplus_f32(float x);

}  // namespace pswa::det

#endif  // PSWA_DET_MATH_H_
