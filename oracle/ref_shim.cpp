// ORACLE — C shim over the reference's own numerics (compiled unmodified from
// /root/reference/proj/src/{det_math,tensor,threading}.cpp) so tests can
// compare the restatement against the reference bit for bit.
#include "pswa/det_math.h"
#include "pswa/rng.h"
#include "pswa/tensor.h"
#include "pswa/threading.h"

extern "C" {

void ref_set_workers(int n) { pswa::set_workers(n); }

void ref_matmul(const float* a, const float* b, float* c, int m, int k, int p) {
  pswa::Tensor A({m, k}), B({k, p});
  std::copy(a, a + static_cast<long>(m) * k, A.data.begin());
  std::copy(b, b + static_cast<long>(k) * p, B.data.begin());
  const pswa::Tensor C = pswa::matmul(A, B);
  std::copy(C.data.begin(), C.data.end(), c);
}

void ref_softmax_rows(const float* x, float* y, int m, int k) {
  pswa::Tensor X({m, k});
  std::copy(x, x + static_cast<long>(m) * k, X.data.begin());
  const pswa::Tensor Y = pswa::softmax_rows(X);
  std::copy(Y.data.begin(), Y.data.end(), y);
}

void ref_rmsnorm(const float* x, const float* g, int d, float* out) { pswa::rmsnorm(x, g, d, out); }

int ref_ffn_hidden_dim(int d) { return pswa::ffn_hidden_dim(d); }

void ref_swiglu_ffn(const float* x, const float* wg, const float* wu, const float* wd, int d, int f,
                    float* out) {
  pswa::Tensor G({d, f}), U({d, f}), D({f, d});
  std::copy(wg, wg + static_cast<long>(d) * f, G.data.begin());
  std::copy(wu, wu + static_cast<long>(d) * f, U.data.begin());
  std::copy(wd, wd + static_cast<long>(f) * d, D.data.begin());
  pswa::swiglu_ffn(x, G, U, D, d, f, out);
}

void ref_conv2d(const float* x, int c, int h, int w, const float* k, int o, int kh, int kw,
                int stride, int pad, float* y, int* oh, int* ow) {
  pswa::Tensor X({c, h, w}), K({o, c, kh, kw});
  std::copy(x, x + static_cast<long>(c) * h * w, X.data.begin());
  std::copy(k, k + static_cast<long>(o) * c * kh * kw, K.data.begin());
  const pswa::Tensor Y = pswa::conv2d(X, K, stride, pad);
  *oh = Y.dim(1);
  *ow = Y.dim(2);
  std::copy(Y.data.begin(), Y.data.end(), y);
}

void ref_upsample2(const float* x, int c, int h, int w, float* y) {
  pswa::Tensor X({c, h, w});
  std::copy(x, x + static_cast<long>(c) * h * w, X.data.begin());
  const pswa::Tensor Y = pswa::upsample_nearest2(X);
  std::copy(Y.data.begin(), Y.data.end(), y);
}

double ref_det(int fn, double x) {
  switch (fn) {
    case 0: return pswa::det::exp(x);
    case 1: return pswa::det::log(x);
    case 2: return pswa::det::erf(x);
    case 3: return pswa::det::normal_cdf(x);
    default: return 0.0;
  }
}

float ref_det_f32(int fn, float x) {
  switch (fn) {
    case 0: return pswa::det::exp_f32(x);
    case 1: return pswa::det::silu_f32(x);
    case 2: return pswa::det::tanh_f32(x);
    case 3: return pswa::det::softplus_f32(x);
    default: return 0.0f;
  }
}

void ref_rng(unsigned long long seed, int n, unsigned long long* u64_out, float* uniform_out,
             float* normal_out) {
  pswa::Rng a(seed), b(seed), c(seed);
  for (int i = 0; i < n; ++i) {
    if (u64_out) u64_out[i] = a.next_u64();
    if (uniform_out) uniform_out[i] = b.next_uniform();
    if (normal_out) normal_out[i] = c.next_normal();
  }
}

unsigned long long ref_fnv1a(const void* p, unsigned long n) { return pswa::fnv1a64(p, n); }

void ref_init_tensor(unsigned long long seed, float* dst, int n, int kind, int fan_in) {
  pswa::Rng r(seed);
  const pswa::InitScheme s = kind == 1   ? pswa::InitScheme::kZeros
                             : kind == 2 ? pswa::InitScheme::kOnes
                                         : pswa::InitScheme::kScaledNormal;
  const pswa::Tensor t = pswa::init_tensor(r, {n}, s, fan_in);
  std::copy(t.data.begin(), t.data.end(), dst);
}

}  // extern "C"
