// Hyperprior convolution support: implicit 3x3 im2col (zero padding 1,
// stride 1 or 2, optional nearest-x2 folded into the addressing) feeding the
// tcgen05 GEMM, plus the NHWC resampling / rounding helpers. Replaces
// conv2d / upsample_nearest2 (tensor.cpp:118-162) on the hyper path
// (SPEC.md:338-346). Patch column order is (ky, kx, c) to match the packed
// conv weights.
#include "check.h"
#include "kernels.h"
#include "launch.cuh"

namespace pswa_dev {

namespace {

__global__ void im2col3x3_kernel(const float* __restrict__ x, int h, int w, int c, int stride,
                                 int up2, int oh, int ow, __half* __restrict__ out, int kcols) {
  pdl_wait();
  pdl_trigger();
  const size_t total = static_cast<size_t>(oh) * ow * kcols;
  const int ih = up2 ? 2 * h : h, iw = up2 ? 2 * w : w;  // logical input grid
  for (size_t idx = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int col = static_cast<int>(idx % kcols);
    const size_t pix = idx / kcols;
    float v = 0.0f;
    if (col < 9 * c) {
      const int tap = col / c, ci = col % c;
      const int oy = static_cast<int>(pix / ow), ox = static_cast<int>(pix % ow);
      const int iy = oy * stride - 1 + tap / 3, ix = ox * stride - 1 + tap % 3;
      if (iy >= 0 && iy < ih && ix >= 0 && ix < iw) {
        const int sy = up2 ? iy >> 1 : iy, sx = up2 ? ix >> 1 : ix;
        v = x[(static_cast<size_t>(sy) * w + sx) * c + ci];
      }
    }
    out[idx] = __float2half_rn(v);
  }
}

// 8 patch columns per thread (one tap, 8 consecutive channels: c % 8 == 0):
// two 16 B loads of the NHWC input and one 16 B store of the fp16 patch row
// segment, 32-bit index math -- the element-per-thread form above ran at
// ~0.5 TB/s on the 1080p hyper grid.
__global__ void im2col3x3_v8_kernel(const float* __restrict__ x, int h, int w, int c, int stride, int up2,
                                    int oh, int ow, __half* __restrict__ out, int kcols) {
  pdl_wait();
  pdl_trigger();
  const int g8 = kcols >> 3, ngrp = 9 * c >> 3;
  const unsigned total = static_cast<unsigned>(oh) * ow * g8;
  const int ih = up2 ? 2 * h : h, iw = up2 ? 2 * w : w;
  for (unsigned idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
    const unsigned pix = idx / g8;
    const int grp = static_cast<int>(idx - pix * g8);
    uint4 o = make_uint4(0u, 0u, 0u, 0u);
    if (grp < ngrp) {
      const int col = grp << 3, tap = col / c, ci = col - tap * c;
      const int oy = static_cast<int>(pix / ow), ox = static_cast<int>(pix - static_cast<unsigned>(oy) * ow);
      const int iy = oy * stride - 1 + tap / 3, ix = ox * stride - 1 + tap % 3;
      if (iy >= 0 && iy < ih && ix >= 0 && ix < iw) {
        const int sy = up2 ? iy >> 1 : iy, sx = up2 ? ix >> 1 : ix;
        const float4* src = reinterpret_cast<const float4*>(x + (static_cast<size_t>(sy) * w + sx) * c + ci);
        const float4 a = __ldg(src), b = __ldg(src + 1);
        __half2 h0 = __floats2half2_rn(a.x, a.y), h1 = __floats2half2_rn(a.z, a.w);
        __half2 h2 = __floats2half2_rn(b.x, b.y), h3 = __floats2half2_rn(b.z, b.w);
        o = make_uint4(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1),
                       *reinterpret_cast<uint32_t*>(&h2), *reinterpret_cast<uint32_t*>(&h3));
      }
    }
    reinterpret_cast<uint4*>(out)[idx] = o;
  }
}

__global__ void resample_kernel(const float* __restrict__ x, int h, int w, int c, int up,
                                float* __restrict__ out, __half* __restrict__ out16) {
  pdl_wait();
  pdl_trigger();
  const int oh = up ? 2 * h : h / 2, ow = up ? 2 * w : w / 2;
  const size_t total = static_cast<size_t>(oh) * ow * c;
  for (size_t idx = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int ci = static_cast<int>(idx % c);
    const size_t pix = idx / c;
    const int oy = static_cast<int>(pix / ow), ox = static_cast<int>(pix % ow);
    const int sy = up ? oy >> 1 : 2 * oy, sx = up ? ox >> 1 : 2 * ox;
    const float v = x[(static_cast<size_t>(sy) * w + sx) * c + ci];
    out[idx] = v;
    if (out16) out16[idx] = __float2half_rn(v);  // the implicit-GEMM conv's operand
  }
}

__global__ void zhat_nhwc_kernel(const int32_t* __restrict__ z, int c, int hw, float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const size_t total = static_cast<size_t>(c) * hw;
  for (size_t idx = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int ci = static_cast<int>(idx % c);
    const size_t p = idx / c;
    out[idx] = static_cast<float>(z[static_cast<size_t>(ci) * hw + p]);
  }
}

__global__ void round_zhat_kernel(const float* __restrict__ x, int c, int hw, int32_t* __restrict__ z) {
  pdl_wait();
  pdl_trigger();
  const size_t total = static_cast<size_t>(c) * hw;
  for (size_t idx = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int ci = static_cast<int>(idx % c);
    const size_t p = idx / c;
    z[static_cast<size_t>(ci) * hw + p] = __float2int_rn(x[idx]);  // half-to-even
  }
}

inline int grid_for(size_t n) {
  const size_t b = (n + 255) / 256;
  return static_cast<int>(b < 148 * 16 ? (b < 1 ? 1 : b) : 148 * 16);
}

}  // namespace

void im2col3x3(const float* x, int h, int w, int c, int stride, int up2, __half* out, int kcols,
               cudaStream_t st) {
  const int ih = up2 ? 2 * h : h, iw = up2 ? 2 * w : w;
  const int oh = (ih + 2 - 3) / stride + 1, ow = (iw + 2 - 3) / stride + 1;
  const bool v8 = c % 8 == 0 && kcols % 8 == 0 && reinterpret_cast<uintptr_t>(x) % 16 == 0 &&
                  reinterpret_cast<uintptr_t>(out) % 16 == 0 &&
                  static_cast<size_t>(oh) * ow * (kcols / 8) < (size_t{1} << 31);
  if (v8)
    launch_k(im2col3x3_v8_kernel, dim3(grid_for(static_cast<size_t>(oh) * ow * (kcols / 8))), dim3(256), 0, st, x,
             h, w, c, stride, up2, oh, ow, out, kcols);
  else
    launch_k(im2col3x3_kernel, dim3(grid_for(static_cast<size_t>(oh) * ow * kcols)), dim3(256), 0, st, x, h, w, c,
             stride, up2, oh, ow, out, kcols);
  PSWA_LAUNCH_CHECK();
}

void upsample2_nhwc(const float* x, int h, int w, int c, float* out, cudaStream_t st, __half* out16) {
  launch_k(resample_kernel, dim3(grid_for(static_cast<size_t>(4) * h * w * c)), dim3(256), 0, st, x, h, w, c, 1, out,
           out16);
  PSWA_LAUNCH_CHECK();
}

void subsample2_nhwc(const float* x, int h, int w, int c, float* out, cudaStream_t st) {
  launch_k(resample_kernel, dim3(grid_for(static_cast<size_t>(h) * w * c / 4 + 1)), dim3(256), 0, st, x, h, w, c, 0,
           out, static_cast<__half*>(nullptr));
  PSWA_LAUNCH_CHECK();
}

void zhat_to_nhwc(const int32_t* z, int c, int hw, float* out, cudaStream_t st) {
  launch_k(zhat_nhwc_kernel, dim3(grid_for(static_cast<size_t>(c) * hw)), dim3(256), 0, st, z, c, hw, out);
  PSWA_LAUNCH_CHECK();
}

void round_to_zhat(const float* x, int c, int hw, int32_t* z, cudaStream_t st) {
  launch_k(round_zhat_kernel, dim3(grid_for(static_cast<size_t>(c) * hw)), dim3(256), 0, st, x, c, hw, z);
  PSWA_LAUNCH_CHECK();
}

}  // namespace pswa_dev
