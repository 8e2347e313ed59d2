// The reference's fp32 operator API (proj/include/pswa/tensor.h) on the
// device, bit-exact: every output element is reduced by one thread in the
// reference's order (ascending k / channel / tap) with IEEE round-to-nearest
// adds and multiplies kept apart (this file is compiled with -fmad=false, the
// intrinsics make the rounding explicit), and the transcendentals are the
// fp64 restatement of det_math.cpp (det_device.cuh). The parallelism the
// reference gets from parallel_for (threading.h:30) comes from independent
// output elements, which is why the bytes do not depend on it.
//
// These kernels back pswa::matmul / softmax_rows / rmsnorm / swiglu_ffn /
// conv2d / upsample_nearest2 for callers of the reference API; the frame
// programs use the fp16 tensor-core kernels instead (gemm.cu, attention_mma.cu).
#include <cfloat>

#include "check.h"
#include "det_device.cuh"
#include "kernels.h"

namespace pswa_dev {
namespace {

// c[i][j] = sum_t a[i][t] * b[t][j] (tensor.cpp:42-58): thread per (i, j),
// threads of a block along j (coalesced b rows, a[i][t] broadcast).
__global__ void matmul_exact_kernel(const float* __restrict__ a, const float* __restrict__ b,
                                    float* __restrict__ c, int m, int k, int p) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x, i = blockIdx.y;
  if (j >= p || i >= m) return;
  const float* ar = a + static_cast<size_t>(i) * k;
  float acc = 0.0f;
  for (int t = 0; t < k; ++t) acc = __fadd_rn(acc, __fmul_rn(__ldg(ar + t), __ldg(b + static_cast<size_t>(t) * p + j)));
  c[static_cast<size_t>(i) * p + j] = acc;
}

// tensor.cpp:60-79: a row per thread (the sum is sequential by definition).
__global__ void softmax_rows_exact_kernel(const float* __restrict__ x, float* __restrict__ y, int m,
                                          int k) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const float* in = x + static_cast<size_t>(i) * k;
  float* out = y + static_cast<size_t>(i) * k;
  const float sentinel = -FLT_MAX;
  float mx = sentinel;
  for (int j = 0; j < k; ++j) mx = in[j] > mx ? in[j] : mx;
  if (mx == sentinel) {  // fully masked row: zeros
    for (int j = 0; j < k; ++j) out[j] = 0.0f;
    return;
  }
  float sum = 0.0f;
  for (int j = 0; j < k; ++j) {
    out[j] = d_exp_f32(__fsub_rn(in[j], mx));
    sum = __fadd_rn(sum, out[j]);
  }
  for (int j = 0; j < k; ++j) out[j] = __fdiv_rn(out[j], sum);
}

// tensor.cpp:81-86, one vector per block (rows = several calls batched).
__global__ void rmsnorm_exact_kernel(const float* __restrict__ x, const float* __restrict__ g, int d,
                                     float* __restrict__ out, int rows) {
  const int r = blockIdx.x;
  if (r >= rows) return;
  const float* xr = x + static_cast<size_t>(r) * d;
  __shared__ float inv;
  if (threadIdx.x == 0) {
    float ss = 0.0f;
    for (int i = 0; i < d; ++i) ss = __fadd_rn(ss, __fmul_rn(xr[i], xr[i]));
    inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(ss, static_cast<float>(d)), 1e-5f)));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < d; i += blockDim.x)
    out[static_cast<size_t>(r) * d + i] = __fmul_rn(__fmul_rn(g[i], xr[i]), inv);
}

// tensor.cpp:88-116, gate/up half: h[j] = silu(sum_i x_i wg[i][j]) * sum_i x_i wu[i][j]
__global__ void swiglu_hidden_kernel(const float* __restrict__ x, const float* __restrict__ wg,
                                     const float* __restrict__ wu, int d, int f, float* __restrict__ h) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= f) return;
  float g = 0.0f, u = 0.0f;
  for (int i = 0; i < d; ++i) {
    const float xi = x[i];
    g = __fadd_rn(g, __fmul_rn(xi, __ldg(wg + static_cast<size_t>(i) * f + j)));
    u = __fadd_rn(u, __fmul_rn(xi, __ldg(wu + static_cast<size_t>(i) * f + j)));
  }
  h[j] = __fmul_rn(d_silu_f32(g), u);
}

// down half: out[i] = sum_j h[j] wd[j][i]
__global__ void swiglu_down_kernel(const float* __restrict__ h, const float* __restrict__ wd, int d,
                                   int f, float* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d) return;
  float acc = 0.0f;
  for (int j = 0; j < f; ++j) acc = __fadd_rn(acc, __fmul_rn(h[j], __ldg(wd + static_cast<size_t>(j) * d + i)));
  out[i] = acc;
}

// tensor.cpp:118-150: thread per output element, ascending (c, ky, kx),
// out-of-bounds taps skipped (zero padding contributes no add).
__global__ void conv2d_exact_kernel(const float* __restrict__ x, int c, int h, int w,
                                    const float* __restrict__ k, int o, int kh, int kw, int stride,
                                    int pad, int oh, int ow, float* __restrict__ y) {
  const long idx = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<long>(o) * oh * ow) return;
  const int ox = static_cast<int>(idx % ow), oy = static_cast<int>((idx / ow) % oh),
            oc = static_cast<int>(idx / (static_cast<long>(ow) * oh));
  float acc = 0.0f;
  for (int ic = 0; ic < c; ++ic)
    for (int ky = 0; ky < kh; ++ky) {
      const int iy = oy * stride - pad + ky;
      if (iy < 0 || iy >= h) continue;
      for (int kx = 0; kx < kw; ++kx) {
        const int ix = ox * stride - pad + kx;
        if (ix < 0 || ix >= w) continue;
        acc = __fadd_rn(acc, __fmul_rn(__ldg(x + (static_cast<size_t>(ic) * h + iy) * w + ix),
                                       __ldg(k + ((static_cast<size_t>(oc) * c + ic) * kh + ky) * kw + kx)));
      }
    }
  y[idx] = acc;
}

__global__ void upsample2_chw_kernel(const float* __restrict__ x, int c, int h, int w, float* __restrict__ y) {
  const long idx = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int W2 = 2 * w, H2 = 2 * h;
  if (idx >= static_cast<long>(c) * H2 * W2) return;
  const int ix = static_cast<int>(idx % W2), iy = static_cast<int>((idx / W2) % H2),
            ic = static_cast<int>(idx / (static_cast<long>(W2) * H2));
  y[idx] = x[(static_cast<size_t>(ic) * h + iy / 2) * w + ix / 2];
}

inline int nblk(long n, int t) { return static_cast<int>((n + t - 1) / t); }

}  // namespace

void matmul_exact(const float* a, const float* b, float* c, int m, int k, int p, cudaStream_t st) {
  if (m <= 0 || p <= 0) return;
  matmul_exact_kernel<<<dim3(nblk(p, 128), m), 128, 0, st>>>(a, b, c, m, k, p);
  PSWA_LAUNCH_CHECK();
}

void softmax_rows_exact(const float* x, float* y, int m, int k, cudaStream_t st) {
  if (m <= 0) return;
  softmax_rows_exact_kernel<<<nblk(m, 128), 128, 0, st>>>(x, y, m, k);
  PSWA_LAUNCH_CHECK();
}

void rmsnorm_exact(const float* x, const float* g, int d, float* out, int rows, cudaStream_t st) {
  if (rows <= 0) return;
  rmsnorm_exact_kernel<<<rows, 128, 0, st>>>(x, g, d, out, rows);
  PSWA_LAUNCH_CHECK();
}

void swiglu_exact(const float* x, const float* wg, const float* wu, const float* wd, int d, int f,
                  float* h_scratch, float* out, cudaStream_t st) {
  swiglu_hidden_kernel<<<nblk(f, 128), 128, 0, st>>>(x, wg, wu, d, f, h_scratch);
  PSWA_LAUNCH_CHECK();
  swiglu_down_kernel<<<nblk(d, 128), 128, 0, st>>>(h_scratch, wd, d, f, out);
  PSWA_LAUNCH_CHECK();
}

void conv2d_exact(const float* x, int c, int h, int w, const float* k, int o, int kh, int kw, int stride,
                  int pad, float* y, cudaStream_t st) {
  const int oh = (h + 2 * pad - kh) / stride + 1, ow = (w + 2 * pad - kw) / stride + 1;
  const long n = static_cast<long>(o) * oh * ow;
  if (n <= 0) return;
  conv2d_exact_kernel<<<nblk(n, 128), 128, 0, st>>>(x, c, h, w, k, o, kh, kw, stride, pad, oh, ow, y);
  PSWA_LAUNCH_CHECK();
}

void upsample2_chw(const float* x, int c, int h, int w, float* y, cudaStream_t st) {
  const long n = 4L * c * h * w;
  if (n <= 0) return;
  upsample2_chw_kernel<<<nblk(n, 256), 256, 0, st>>>(x, c, h, w, y);
  PSWA_LAUNCH_CHECK();
}

}  // namespace pswa_dev
