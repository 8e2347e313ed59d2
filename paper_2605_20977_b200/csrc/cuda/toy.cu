// Toy transform: the fixed, invertible stand-in for the
// learned analysis / synthesis transforms, so frames run end to end.
//   analysis : per 8x8 patch and colour plane, orthonormal 2D DCT-II of the
//              pixels centred at 128, channels in zigzag-major order
//              (channel = 3 * zigzag + colour; group 0 = lowest frequencies),
//              divided by q[rate] = {8, 5, 3, 2};
//   synthesis: inverse DCT of y_rec * q[rate], + 128, clamp [0, 255], round.
// One thread per (patch, channel): the 64 basis products are tiny, and the
// transform runs once per frame outside the entropy path.
#include "check.h"
#include "kernels.h"
#include "launch.cuh"

namespace pswa_dev {

namespace {

__constant__ float kQ[4] = {8.0f, 5.0f, 3.0f, 2.0f};
// zigzag index -> (row, col) of the 8x8 coefficient block (JPEG order)
__constant__ unsigned char kZig[64] = {
    0,  1,  8,  16, 9,  2,  3,  10, 17, 24, 32, 25, 18, 11, 4,  5,  12, 19, 26, 33, 40, 48,
    41, 34, 27, 20, 13, 6,  7,  14, 21, 28, 35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23,
    30, 37, 44, 51, 58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63};

__device__ __forceinline__ float dct_basis(int k, int n) {  // orthonormal DCT-II basis
  const float a = k == 0 ? 0.35355339059327373f : 0.5f;     // sqrt(1/8), sqrt(2/8)
  return a * cospif((2.0f * n + 1.0f) * k / 16.0f);
}

__global__ void analysis_kernel(const uint8_t* __restrict__ rgb, int Hpx, int Wpx, int rate,
                                float* __restrict__ y) {
  const int h = Hpx / 8, w = Wpx / 8;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;  // (channel, patch)
  if (i >= 192 * h * w) return;
  const int ch = i / (h * w), p = i % (h * w), py = p / w, px = p % w;
  const int z = ch / 3, col = ch % 3, u = kZig[z] / 8, v = kZig[z] % 8;
  float acc = 0.0f;
  for (int r = 0; r < 8; ++r) {
    const float bu = dct_basis(u, r);
    for (int c = 0; c < 8; ++c) {
      const float pix = static_cast<float>(rgb[((py * 8 + r) * Wpx + px * 8 + c) * 3 + col]) - 128.0f;
      acc = fmaf(bu * dct_basis(v, c), pix, acc);
    }
  }
  y[i] = acc / kQ[rate];
}

__global__ void synthesis_kernel(const float* __restrict__ y, int Hpx, int Wpx, int rate,
                                 uint8_t* __restrict__ rgb) {
  const int h = Hpx / 8, w = Wpx / 8;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;  // (pixel, colour)
  if (i >= Hpx * Wpx * 3) return;
  const int col = i % 3, pix = i / 3, yy = pix / Wpx, xx = pix % Wpx;
  const int py = yy / 8, px = xx / 8, r = yy % 8, c = xx % 8;
  const float q = kQ[rate];
  float acc = 0.0f;
  for (int z = 0; z < 64; ++z) {
    const int u = kZig[z] / 8, v = kZig[z] % 8;
    acc = fmaf(dct_basis(u, r) * dct_basis(v, c), y[((z * 3 + col) * h + py) * w + px] * q, acc);
  }
  const float o = fminf(fmaxf(rintf(acc + 128.0f), 0.0f), 255.0f);
  rgb[i] = static_cast<uint8_t>(o);
}

}  // namespace

void toy_analysis(const uint8_t* rgb, int Hpx, int Wpx, int rate, float* y, cudaStream_t st) {
  if (Hpx % 8 || Wpx % 8 || rate < 0 || rate > 3) throw std::invalid_argument("toy_analysis: shape / rate");
  const int n = 192 * (Hpx / 8) * (Wpx / 8);
  analysis_kernel<<<(n + 255) / 256, 256, 0, st>>>(rgb, Hpx, Wpx, rate, y);
  PSWA_LAUNCH_CHECK();
}

void toy_synthesis(const float* y, int Hpx, int Wpx, int rate, uint8_t* rgb, cudaStream_t st) {
  if (Hpx % 8 || Wpx % 8 || rate < 0 || rate > 3) throw std::invalid_argument("toy_synthesis: shape / rate");
  const int n = Hpx * Wpx * 3;
  synthesis_kernel<<<(n + 255) / 256, 256, 0, st>>>(y, Hpx, Wpx, rate, rgb);
  PSWA_LAUNCH_CHECK();
}

}  // namespace pswa_dev
