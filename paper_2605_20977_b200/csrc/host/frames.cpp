// Frame I/O for end-to-end coding (SPEC.md:663-670 read_ppm / write_ppm,
// :499-548 toy transform): binary P6 PPM, replicate-edge padding to
// multiples of 8, and host entry points of the device toy transform.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../cuda/check.h"
#include "../cuda/kernels.h"
#include "abi_util.h"
#include "pswa/pswa_cuda.h"

using pswa_abi::guard;

namespace {

struct File {
  FILE* f;
  explicit File(const char* p, const char* m) : f(std::fopen(p, m)) {
    if (!f) throw std::invalid_argument(std::string("cannot open ") + p);
  }
  ~File() { std::fclose(f); }
};

// next header token of a P6 file (skips whitespace and # comments)
long token(FILE* f) {
  int c = std::fgetc(f);
  while (c == '#' || c == ' ' || c == '\t' || c == '\n' || c == '\r') {
    if (c == '#')
      while (c != '\n' && c != EOF) c = std::fgetc(f);
    c = std::fgetc(f);
  }
  if (c < '0' || c > '9') throw std::invalid_argument("PPM: malformed header");
  long v = 0;
  while (c >= '0' && c <= '9') {
    v = v * 10 + (c - '0');
    if (v > (1 << 20)) throw std::invalid_argument("PPM: dimension too large");
    c = std::fgetc(f);
  }
  return v;  // the single whitespace after the token is consumed
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  explicit DevBuf(size_t n) { PSWA_CUDA(cudaMalloc(&p, n * sizeof(T))); }
  ~DevBuf() { cudaFree(p); }
};

}  // namespace

extern "C" {

int pswa_read_ppm(const char* path, uint8_t* rgb, size_t cap, int* width, int* height) {
  return guard([&] {
    File f(path, "rb");
    char m[2];
    if (std::fread(m, 1, 2, f.f) != 2 || m[0] != 'P') throw std::invalid_argument("PPM: not a PPM file");
    if (m[1] != '6') throw std::invalid_argument("PPM: only binary P6 is supported (P3 / others rejected)");
    const long w = token(f.f), h = token(f.f), maxv = token(f.f);
    if (w <= 0 || h <= 0) throw std::invalid_argument("PPM: empty image");
    if (maxv != 255) throw std::invalid_argument("PPM: maxval must be 255");
    *width = static_cast<int>(w);
    *height = static_cast<int>(h);
    if (!rgb) return;
    const size_t n = static_cast<size_t>(w) * h * 3;
    if (cap < n) throw std::invalid_argument("PPM: buffer too small");
    if (std::fread(rgb, 1, n, f.f) != n) throw pswa_abi::TruncatedError("PPM: truncated pixel data");
  });
}

int pswa_write_ppm(const char* path, const uint8_t* rgb, int width, int height) {
  return guard([&] {
    if (width <= 0 || height <= 0) throw std::invalid_argument("PPM: empty image");
    File f(path, "wb");
    std::fprintf(f.f, "P6\n%d %d\n255\n", width, height);
    const size_t n = static_cast<size_t>(width) * height * 3;
    if (std::fwrite(rgb, 1, n, f.f) != n) throw std::runtime_error("PPM: write failed");
  });
}

int pswa_pad8(const uint8_t* rgb, int height, int width, uint8_t* out, int* h8, int* w8) {
  return guard([&] {
    if (width <= 0 || height <= 0) throw std::invalid_argument("pad8: empty image");
    const int H = (height + 7) / 8 * 8, W = (width + 7) / 8 * 8;
    *h8 = H;
    *w8 = W;
    if (!out) return;
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x)
        std::memcpy(out + (static_cast<size_t>(y) * W + x) * 3,
                    rgb + (static_cast<size_t>(std::min(y, height - 1)) * width + std::min(x, width - 1)) * 3, 3);
  });
}

int pswa_toy_analysis(const uint8_t* rgb, int h_px, int w_px, int rate_idx, float* y_out) {
  return guard([&] {
    const size_t np = static_cast<size_t>(h_px) * w_px * 3, ny = static_cast<size_t>(192) * (h_px / 8) * (w_px / 8);
    DevBuf<uint8_t> d_rgb(np);
    DevBuf<float> d_y(ny);
    PSWA_CUDA(cudaMemcpy(d_rgb.p, rgb, np, cudaMemcpyHostToDevice));
    pswa_dev::toy_analysis(d_rgb.p, h_px, w_px, rate_idx, d_y.p, nullptr);
    PSWA_CUDA(cudaMemcpy(y_out, d_y.p, ny * sizeof(float), cudaMemcpyDeviceToHost));
  });
}

int pswa_toy_synthesis(const float* y, int h_px, int w_px, int rate_idx, uint8_t* rgb_out) {
  return guard([&] {
    const size_t np = static_cast<size_t>(h_px) * w_px * 3, ny = static_cast<size_t>(192) * (h_px / 8) * (w_px / 8);
    DevBuf<uint8_t> d_rgb(np);
    DevBuf<float> d_y(ny);
    PSWA_CUDA(cudaMemcpy(d_y.p, y, ny * sizeof(float), cudaMemcpyHostToDevice));
    pswa_dev::toy_synthesis(d_y.p, h_px, w_px, rate_idx, d_rgb.p, nullptr);
    PSWA_CUDA(cudaMemcpy(rgb_out, d_rgb.p, np, cudaMemcpyDeviceToHost));
  });
}

}  // extern "C"
