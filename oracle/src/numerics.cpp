// ORACLE — test infrastructure only (see numerics.h for the reference map).
#include "oracle/numerics.h"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <thread>

namespace oracle {

// ============================================================ det_math ====
namespace {

double from_bits(uint64_t b) {
  double d;
  std::memcpy(&d, &b, sizeof d);
  return d;
}
uint64_t to_bits(double d) {
  uint64_t b;
  std::memcpy(&b, &d, sizeof b);
  return b;
}

// Exact power of two 2^k (subnormals included) — det_math.cpp:29-43.
double two_to(int k) {
  if (k > 1023) return std::numeric_limits<double>::infinity();
  if (k < -1074) return 0.0;
  if (k >= -1022) return from_bits(static_cast<uint64_t>(k + 1023) << 52);
  return from_bits(uint64_t{1} << (k + 1074));
}

// Cody-Waite split of ln2 and 1/ln2 (det_math.cpp:45-47).
constexpr double LN2_HI = 6.93147180369123816490e-01;
constexpr double LN2_LO = 1.90821492927058770002e-10;
constexpr double INV_LN2 = 1.44269504088896338700e+00;

// Taylor tail 1/13! .. 1/3!, evaluated Horner-wise from the top
// (det_math.cpp:60-71).
constexpr double kTaylor[11] = {
    1.0 / 6227020800.0, 1.0 / 479001600.0, 1.0 / 39916800.0, 1.0 / 3628800.0,
    1.0 / 362880.0,     1.0 / 40320.0,     1.0 / 5040.0,     1.0 / 720.0,
    1.0 / 120.0,        1.0 / 24.0,        1.0 / 6.0};

// fdlibm log polynomial (det_math.cpp:98-106).
constexpr double kLg[7] = {6.666666666666735130e-01, 3.999999999940941908e-01,
                           2.857142874366239149e-01, 2.222219843214978396e-01,
                           1.818357216161805012e-01, 1.531383769920937332e-01,
                           1.479819860511658591e-01};

// Abramowitz & Stegun 7.1.26 (det_math.cpp:115-126).
constexpr double kAsP = 0.3275911;
constexpr double kAs[5] = {0.254829592, -0.284496736, 1.421413741, -1.453152027, 1.061405429};

}  // namespace

namespace det {

double exp(double x) {
  if (std::isnan(x)) return x;
  if (x > 709.782712893384) return std::numeric_limits<double>::infinity();
  if (x < -745.1332191019412) return 0.0;
  const double t = x * INV_LN2;
  const int n = static_cast<int>(t >= 0.0 ? t + 0.5 : t - 0.5);
  const double nd = n;
  const double r = (x - nd * LN2_HI) - nd * LN2_LO;
  double poly = kTaylor[0];
  for (int i = 1; i < 11; ++i) poly = poly * r + kTaylor[i];
  const double rr = r * r;
  const double e_r = 1.0 + r + 0.5 * rr + rr * r * poly;
  return e_r * two_to(n);
}

double log(double x) {
  if (std::isnan(x)) return x;
  if (x < 0.0) return std::numeric_limits<double>::quiet_NaN();
  if (x == 0.0) return -std::numeric_limits<double>::infinity();
  if (std::isinf(x)) return x;
  int ex = 0;
  uint64_t b = to_bits(x);
  if (b < (uint64_t{1} << 52)) {  // subnormal
    x *= 0x1p54;
    ex = -54;
    b = to_bits(x);
  }
  ex += static_cast<int>((b >> 52) & 0x7FF) - 1023;
  double m = from_bits((b & ((uint64_t{1} << 52) - 1)) | (uint64_t{1023} << 52));
  if (m > 1.4142135623730951) {
    m *= 0.5;
    ex += 1;
  }
  const double f = m - 1.0;
  const double s = f / (2.0 + f);
  const double z = s * s;
  const double w = z * z;
  // odd / even halves of the polynomial in w
  const double odd = w * (kLg[1] + w * (kLg[3] + w * kLg[5]));
  const double even = z * (kLg[0] + w * (kLg[2] + w * (kLg[4] + w * kLg[6])));
  const double half_f2 = 0.5 * f * f;
  const double R = even + odd;
  const double e = ex;
  return e * LN2_HI - ((half_f2 - (s * (half_f2 + R) + e * LN2_LO)) - f);
}

double erf(double x) {
  const double a = x < 0.0 ? -x : x;
  const double t = 1.0 / (1.0 + kAsP * a);
  double poly = kAs[4];
  for (int i = 3; i >= 0; --i) poly = kAs[i] + t * poly;
  poly = t * poly;
  const double y = 1.0 - poly * det::exp(-a * a);
  return x < 0.0 ? -y : y;
}

double normal_cdf(double x) { return 0.5 * (1.0 + det::erf(x * 0.7071067811865475244)); }

float exp_f32(float x) { return static_cast<float>(det::exp(static_cast<double>(x))); }

float silu_f32(float x) {
  const double v = x;
  return static_cast<float>(v / (1.0 + det::exp(-v)));
}

float tanh_f32(float x) {
  const double v = x;
  const double a = v < 0.0 ? -v : v;
  if (a > 20.0) return x < 0.0f ? -1.0f : 1.0f;
  const double q = 1.0 - 2.0 / (det::exp(2.0 * a) + 1.0);
  return static_cast<float>(v < 0.0 ? -q : q);
}

float softplus_f32(float x) {
  const double v = x;
  if (v > 30.0) return x;
  if (v < -30.0) return static_cast<float>(det::exp(v));
  return static_cast<float>(det::log(1.0 + det::exp(v)));
}

}  // namespace det

// ================================================================= rng ====
uint64_t Rng::u64() {
  s += 0x9E3779B97F4A7C15ULL;
  uint64_t z = s;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
float Rng::uniform() { return static_cast<float>(u64() >> 40) * 0x1p-24f; }
float Rng::normal() {
  float acc = 0.0f;
  for (int i = 0; i < 12; ++i) acc += uniform();
  return acc - 6.0f;
}
uint64_t fnv1a(const void* p, size_t n) {
  const auto* c = static_cast<const unsigned char*>(p);
  uint64_t h = 0xCBF29CE484222325ULL;
  for (size_t i = 0; i < n; ++i) h = (h ^ c[i]) * 0x100000001B3ULL;
  return h;
}
uint64_t fnv1a(std::string_view s) { return fnv1a(s.data(), s.size()); }

// =========================================================== threading ====
namespace {
int g_threads = 0;
}
void set_threads(int n) { g_threads = n < 1 ? 1 : n; }
int threads() {
  if (g_threads == 0) {
    const char* e = std::getenv("PSWA_THREADS");
    const int v = e ? std::atoi(e) : 0;
    g_threads = v >= 1 ? v : 1;
  }
  return g_threads;
}
void pfor(int64_t n, const std::function<void(int64_t)>& fn) {
  if (n <= 0) return;
  int w = threads();
  if (w <= 1 || n == 1) {
    for (int64_t i = 0; i < n; ++i) fn(i);
    return;
  }
  if (w > n) w = static_cast<int>(n);
  std::atomic<int64_t> next{0};
  const int64_t chunk = std::max<int64_t>(1, n / (int64_t{w} * 8));
  auto worker = [&] {
    for (;;) {
      const int64_t lo = next.fetch_add(chunk);
      if (lo >= n) break;
      const int64_t hi = std::min(n, lo + chunk);
      for (int64_t i = lo; i < hi; ++i) fn(i);
    }
  };
  std::vector<std::thread> pool;
  for (int i = 1; i < w; ++i) pool.emplace_back(worker);
  worker();
  for (auto& t : pool) t.join();
}

// =========================================================== tensor ops ===
float sentinel() { return std::numeric_limits<float>::lowest(); }

// Row-blocked i-k-j loop. Every c[m][p] still receives a[m][0]*b[0][p],
// a[m][1]*b[1][p], ... added in ascending k into an f32 accumulator that
// starts at 0, exactly like tensor.cpp:49-55, so the bits are identical; only
// the traversal (and hence the speed) differs.
void matmul(const float* a, const float* b, float* c, int m, int k, int p) {
  constexpr int RB = 16;   // rows per task
  constexpr int CB = 512;  // columns per chunk
  const int64_t row_blocks = (m + RB - 1) / RB;
  pfor(row_blocks, [&](int64_t rb) {
    const int r0 = static_cast<int>(rb) * RB;
    const int r1 = std::min(m, r0 + RB);
    std::vector<float> acc(static_cast<size_t>(RB) * CB);
    for (int c0 = 0; c0 < p; c0 += CB) {
      const int cw = std::min(CB, p - c0);
      std::fill(acc.begin(), acc.end(), 0.0f);
      for (int t = 0; t < k; ++t) {
        const float* brow = b + static_cast<size_t>(t) * p + c0;
        for (int r = r0; r < r1; ++r) {
          const float av = a[static_cast<size_t>(r) * k + t];
          float* ar = acc.data() + static_cast<size_t>(r - r0) * CB;
          for (int j = 0; j < cw; ++j) ar[j] += av * brow[j];
        }
      }
      for (int r = r0; r < r1; ++r)
        std::memcpy(c + static_cast<size_t>(r) * p + c0,
                    acc.data() + static_cast<size_t>(r - r0) * CB, sizeof(float) * cw);
    }
  });
}

void softmax_row(float* row, int k) {
  const float s = sentinel();
  float mx = s;
  for (int j = 0; j < k; ++j) mx = row[j] > mx ? row[j] : mx;
  if (mx == s) {
    for (int j = 0; j < k; ++j) row[j] = 0.0f;
    return;
  }
  float sum = 0.0f;
  for (int j = 0; j < k; ++j) {
    row[j] = det::exp_f32(row[j] - mx);
    sum += row[j];
  }
  for (int j = 0; j < k; ++j) row[j] /= sum;
}

void rmsnorm(const float* x, const float* gain, int d, float* out) {
  float ss = 0.0f;
  for (int i = 0; i < d; ++i) ss += x[i] * x[i];
  const float inv = 1.0f / std::sqrt(ss / static_cast<float>(d) + kEps);
  for (int i = 0; i < d; ++i) out[i] = gain[i] * x[i] * inv;
}

int ffn_hidden(int d) {
  const long u = std::lround(static_cast<double>(d) / 3.0);
  return 8 * static_cast<int>(u < 1 ? 1 : u);
}

void conv2d(const float* x, int c, int h, int w, const float* k, int o, int kh, int kw,
            int stride, int pad, float* y, int* oh_out, int* ow_out) {
  const int oh = (h + 2 * pad - kh) / stride + 1;
  const int ow = (w + 2 * pad - kw) / stride + 1;
  *oh_out = oh;
  *ow_out = ow;
  pfor(static_cast<int64_t>(o) * oh, [&](int64_t idx) {
    const int oc = static_cast<int>(idx / oh);
    const int oy = static_cast<int>(idx % oh);
    for (int ox = 0; ox < ow; ++ox) {
      float acc = 0.0f;
      for (int ic = 0; ic < c; ++ic) {
        for (int ky = 0; ky < kh; ++ky) {
          const int iy = oy * stride - pad + ky;
          if (iy < 0 || iy >= h) continue;
          const float* xr = x + (static_cast<size_t>(ic) * h + iy) * w;
          const float* kr = k + ((static_cast<size_t>(oc) * c + ic) * kh + ky) * kw;
          for (int kx = 0; kx < kw; ++kx) {
            const int ix = ox * stride - pad + kx;
            if (ix < 0 || ix >= w) continue;
            acc += xr[ix] * kr[kx];
          }
        }
      }
      y[(static_cast<size_t>(oc) * oh + oy) * ow + ox] = acc;
    }
  });
}

void upsample2(const float* x, int c, int h, int w, float* y) {
  for (int ic = 0; ic < c; ++ic)
    for (int yy = 0; yy < 2 * h; ++yy)
      for (int xx = 0; xx < 2 * w; ++xx)
        y[(static_cast<size_t>(ic) * 2 * h + yy) * 2 * w + xx] =
            x[(static_cast<size_t>(ic) * h + yy / 2) * w + xx / 2];
}

void init_values(Rng& r, float* dst, size_t n, int kind, int fan_in) {
  if (kind == 1) {
    std::fill(dst, dst + n, 0.0f);
  } else if (kind == 2) {
    std::fill(dst, dst + n, 1.0f);
  } else {
    const float sd = 1.0f / std::sqrt(static_cast<float>(fan_in < 1 ? 1 : fan_in));
    for (size_t i = 0; i < n; ++i) dst[i] = r.normal() * sd;
  }
}

}  // namespace oracle
