// pswa/tensor.h on the device (see the header; kernels in
// csrc/cuda/tensor_ops.cu). Shape checks and error types follow
// proj/src/tensor.cpp:42-162; the copies in and out are synchronous, like
// the reference's by-value results.
#include "pswa/tensor.h"

#include <cuda_runtime.h>

#include <cfloat>
#include <cmath>
#include <cstring>
#include <stdexcept>

#include "../cuda/check.h"
#include "../cuda/kernels.h"
#include "abi_util.h"

namespace pswa {
namespace {

// A device copy of host floats (or scratch), freed at scope exit.
class Dev {
 public:
  explicit Dev(size_t n, const float* src = nullptr) : n_(n) {
    PSWA_CUDA(cudaMalloc(&p_, sizeof(float) * (n ? n : 1)));
    if (src && n) PSWA_CUDA(cudaMemcpy(p_, src, sizeof(float) * n, cudaMemcpyHostToDevice));
  }
  ~Dev() { cudaFree(p_); }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  float* p() const { return p_; }
  void to_host(float* dst) const {
    if (n_) PSWA_CUDA(cudaMemcpy(dst, p_, sizeof(float) * n_, cudaMemcpyDeviceToHost));
  }

 private:
  float* p_ = nullptr;
  size_t n_;
};

void sync() {
  PSWA_CUDA(cudaGetLastError());
  PSWA_CUDA(cudaDeviceSynchronize());
}

}  // namespace

bool Tensor::all_finite() const {
  for (float v : data)
    if (!std::isfinite(v)) return false;
  return true;
}

bool Tensor::same_bytes(const Tensor& o) const {
  return shape == o.shape && data.size() == o.data.size() &&
         (data.empty() || std::memcmp(data.data(), o.data.data(), data.size() * sizeof(float)) == 0);
}

float mask_sentinel() { return -FLT_MAX; }

Tensor matmul(const Tensor& a, const Tensor& b) {
  if (a.rank() != 2 || b.rank() != 2 || a.dim(1) != b.dim(0))
    throw std::invalid_argument("matmul: shape mismatch");
  const int m = a.dim(0), k = a.dim(1), p = b.dim(1);
  Tensor c({m, p});
  Dev da(a.data.size(), a.data.data()), db(b.data.size(), b.data.data()), dc(c.data.size());
  pswa_dev::matmul_exact(da.p(), db.p(), dc.p(), m, k, p, nullptr);
  sync();
  dc.to_host(c.data.data());
  return c;
}

Tensor softmax_rows(const Tensor& x) {
  if (x.rank() != 2) throw std::invalid_argument("softmax_rows: rank != 2");
  const int m = x.dim(0), k = x.dim(1);
  Tensor y({m, k});
  Dev dx(x.data.size(), x.data.data()), dy(y.data.size());
  pswa_dev::softmax_rows_exact(dx.p(), dy.p(), m, k, nullptr);
  sync();
  dy.to_host(y.data.data());
  return y;
}

void rmsnorm(const float* x, const float* gain, int d, float* out) {
  if (d <= 0) return;
  Dev dx(d, x), dg(d, gain), dout(d);
  pswa_dev::rmsnorm_exact(dx.p(), dg.p(), d, dout.p(), 1, nullptr);
  sync();
  dout.to_host(out);
}

int ffn_hidden_dim(int d) {
  const int units = static_cast<int>(std::lround(static_cast<double>(d) / 3.0));
  return 8 * (units < 1 ? 1 : units);
}

void swiglu_ffn(const float* x, const Tensor& w_gate, const Tensor& w_up, const Tensor& w_down, int d,
                int f, float* out) {
  if (w_gate.rank() != 2 || w_up.rank() != 2 || w_down.rank() != 2 || w_gate.dim(0) != d ||
      w_gate.dim(1) != f || w_up.dim(0) != d || w_up.dim(1) != f || w_down.dim(0) != f ||
      w_down.dim(1) != d)
    throw std::invalid_argument("swiglu_ffn: shape mismatch");
  Dev dx(d, x), dg(w_gate.data.size(), w_gate.data.data()), du(w_up.data.size(), w_up.data.data()),
      dd(w_down.data.size(), w_down.data.data()), h(f), dout(d);
  pswa_dev::swiglu_exact(dx.p(), dg.p(), du.p(), dd.p(), d, f, h.p(), dout.p(), nullptr);
  sync();
  dout.to_host(out);
}

Tensor conv2d(const Tensor& x, const Tensor& k, int stride, int pad) {
  if (x.rank() != 3 || k.rank() != 4 || k.dim(1) != x.dim(0))
    throw std::invalid_argument("conv2d: shape mismatch");
  const int c = x.dim(0), h = x.dim(1), w = x.dim(2), o = k.dim(0), kh = k.dim(2), kw = k.dim(3);
  if (kh % 2 == 0 || kw % 2 == 0) throw std::invalid_argument("conv2d: kernel extents must be odd");
  if (stride < 1) throw std::invalid_argument("conv2d: stride < 1");
  const int oh = (h + 2 * pad - kh) / stride + 1, ow = (w + 2 * pad - kw) / stride + 1;
  Tensor y({o, oh, ow});
  Dev dx(x.data.size(), x.data.data()), dk(k.data.size(), k.data.data()), dy(y.data.size());
  pswa_dev::conv2d_exact(dx.p(), c, h, w, dk.p(), o, kh, kw, stride, pad, dy.p(), nullptr);
  sync();
  dy.to_host(y.data.data());
  return y;
}

Tensor upsample_nearest2(const Tensor& x) {
  if (x.rank() != 3) throw std::invalid_argument("upsample: rank != 3");
  const int c = x.dim(0), h = x.dim(1), w = x.dim(2);
  Tensor y({c, 2 * h, 2 * w});
  Dev dx(x.data.size(), x.data.data()), dy(y.data.size());
  pswa_dev::upsample2_chw(dx.p(), c, h, w, dy.p(), nullptr);
  sync();
  dy.to_host(y.data.data());
  return y;
}

Tensor init_tensor(Rng& rng, std::vector<int> shape, InitScheme scheme, int fan_in) {
  Tensor t(std::move(shape));
  if (scheme == InitScheme::kOnes) {
    for (float& v : t.data) v = 1.0f;
  } else if (scheme == InitScheme::kScaledNormal) {
    const float sd = 1.0f / std::sqrt(static_cast<float>(fan_in < 1 ? 1 : fan_in));
    for (float& v : t.data) v = rng.next_normal() * sd;
  }
  return t;
}

}  // namespace pswa

// ---- C ABI over pswa/tensor.h (ctypes / cgo bindings, parity tests) --------
extern "C" {

int pswa_tensor_matmul(const float* a, const float* b, float* c, int m, int k, int p) {
  return pswa_abi::guard([&] {
    pswa::Tensor A({m, k}), B({k, p});
    std::memcpy(A.data.data(), a, sizeof(float) * A.data.size());
    std::memcpy(B.data.data(), b, sizeof(float) * B.data.size());
    const pswa::Tensor Cm = pswa::matmul(A, B);
    std::memcpy(c, Cm.data.data(), sizeof(float) * Cm.data.size());
  });
}

int pswa_tensor_softmax_rows(const float* x, float* y, int m, int k) {
  return pswa_abi::guard([&] {
    pswa::Tensor X({m, k});
    std::memcpy(X.data.data(), x, sizeof(float) * X.data.size());
    const pswa::Tensor Y = pswa::softmax_rows(X);
    std::memcpy(y, Y.data.data(), sizeof(float) * Y.data.size());
  });
}

int pswa_tensor_rmsnorm(const float* x, const float* g, int d, float* out) {
  return pswa_abi::guard([&] { pswa::rmsnorm(x, g, d, out); });
}

int pswa_tensor_swiglu_ffn(const float* x, const float* wg, const float* wu, const float* wd, int d,
                           int f, float* out) {
  return pswa_abi::guard([&] {
    pswa::Tensor G({d, f}), U({d, f}), D({f, d});
    std::memcpy(G.data.data(), wg, sizeof(float) * G.data.size());
    std::memcpy(U.data.data(), wu, sizeof(float) * U.data.size());
    std::memcpy(D.data.data(), wd, sizeof(float) * D.data.size());
    pswa::swiglu_ffn(x, G, U, D, d, f, out);
  });
}

int pswa_tensor_conv2d(const float* x, int c, int h, int w, const float* k, int o, int kh, int kw,
                       int stride, int pad, float* y) {
  return pswa_abi::guard([&] {
    pswa::Tensor X({c, h, w}), K({o, c, kh, kw});
    std::memcpy(X.data.data(), x, sizeof(float) * X.data.size());
    std::memcpy(K.data.data(), k, sizeof(float) * K.data.size());
    const pswa::Tensor Y = pswa::conv2d(X, K, stride, pad);
    std::memcpy(y, Y.data.data(), sizeof(float) * Y.data.size());
  });
}

int pswa_tensor_upsample2(const float* x, int c, int h, int w, float* y) {
  return pswa_abi::guard([&] {
    pswa::Tensor X({c, h, w});
    std::memcpy(X.data.data(), x, sizeof(float) * X.data.size());
    const pswa::Tensor Y = pswa::upsample_nearest2(X);
    std::memcpy(y, Y.data.data(), sizeof(float) * Y.data.size());
  });
}

int pswa_tensor_ffn_hidden_dim(int d) { return pswa::ffn_hidden_dim(d); }

}  // extern "C"
