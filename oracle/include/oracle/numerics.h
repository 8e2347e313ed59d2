// ORACLE — test infrastructure only. Never linked into the product path.
//
// CPU restatement of the reference's deterministic numerics floor:
//   det::*        proj/include/pswa/det_math.h:25-36, proj/src/det_math.cpp:49-153
//   Rng / fnv1a   proj/include/pswa/rng.h:24-78
//   tensor ops    proj/include/pswa/tensor.h:58-93, proj/src/tensor.cpp:40-180
//   parallel_for  proj/include/pswa/threading.h:24-31, proj/src/threading.cpp:38-72
// Every function reproduces the reference's operation order so results are
// bit-identical (pinned against oracle/_ref, the reference sources compiled
// unmodified; see tests/test_oracle_ref.py).
#pragma once
#include <cstddef>
#include <cstdint>
#include <functional>
#include <string_view>
#include <vector>

namespace oracle {

// ---- det_math (fp64 transcendentals with fixed polynomials) -------------
namespace det {
double exp(double x);
double log(double x);
double erf(double x);
double normal_cdf(double x);
float exp_f32(float x);
float silu_f32(float x);
float tanh_f32(float x);
float softplus_f32(float x);
}  // namespace det

// ---- SplitMix64 + FNV-1a (rng.h) -----------------------------------------
struct Rng {
  uint64_t s;
  explicit Rng(uint64_t seed) : s(seed) {}
  uint64_t u64();
  float uniform();  // 24-bit, [0,1)
  float normal();   // Irwin-Hall(12) - 6
};
uint64_t fnv1a(std::string_view s);
uint64_t fnv1a(const void* p, size_t n);
inline Rng param_rng(uint64_t seed, std::string_view name) { return Rng(seed ^ fnv1a(name)); }

// ---- threading (index-partitioned, byte-identical for any worker count) --
void set_threads(int n);
int threads();
void pfor(int64_t n, const std::function<void(int64_t)>& fn);

// ---- tensor ops ----------------------------------------------------------
float sentinel();  // most negative finite f32
// c[m][p] = sum_k a[m][k]*b[k][p], ascending k, f32 accumulator.
void matmul(const float* a, const float* b, float* c, int m, int k, int p);
// In-place softmax of one row, reference semantics (fully masked -> zeros).
void softmax_row(float* row, int k);
void rmsnorm(const float* x, const float* gain, int d, float* out);
constexpr float kEps = 1e-5f;
int ffn_hidden(int d);
// Cross-correlation on (C,H,W) with (O,C,kh,kw), zero padding, ascending
// (c, ky, kx); out-of-bounds taps are skipped.
void conv2d(const float* x, int c, int h, int w, const float* k, int o, int kh, int kw,
            int stride, int pad, float* y, int* oh, int* ow);
void upsample2(const float* x, int c, int h, int w, float* y);
// init_tensor: kind 0 scaled-normal(1/sqrt(fan_in)), 1 zeros, 2 ones
void init_values(Rng& r, float* dst, size_t n, int kind, int fan_in);

}  // namespace oracle
