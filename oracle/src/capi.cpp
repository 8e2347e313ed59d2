// ORACLE — test infrastructure only: C entry points for tests/ (ctypes) and
// bench.py's cpu_baseline leg. Config is passed as the 22 ints of pswa_cfg.
#include <cmath>
#include <cstring>
#include <vector>
#include <exception>
#include <stdexcept>
#include <string>

#include "oracle/model.h"

using namespace oracle;

namespace {
thread_local std::string g_err;

Config to_cfg(const int* a) {
  Config c;
  c.d = a[0];
  c.heads = a[1];
  c.ctx_blocks = a[2];
  c.s1_blocks = a[3];
  c.s2_blocks = a[4];
  c.d_ch = a[5];
  c.ch_blocks = a[6];
  c.hyper_ch = a[7];
  c.C = a[8];
  c.s = a[9];
  c.N = a[10];
  c.wh = a[11];
  c.ww = a[12];
  c.wt = a[13];
  c.T = a[14];
  c.rates = a[15];
  c.H = a[16];
  c.W = a[17];
  c.lanes = a[18];
  c.hyper_lanes = a[19];
  c.prior = a[20];
  c.lrp_blocks = a[21];
  return c;
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

std::vector<const int32_t*> past_list(const int32_t* const* past, int npast) {
  std::vector<const int32_t*> v;
  for (int i = 0; i < npast; ++i) v.push_back(past[i]);
  return v;
}

int copy_out(const std::vector<uint8_t>& src, uint8_t* dst, size_t cap, size_t* len) {
  *len = src.size();
  if (!dst) return 0;
  if (cap < src.size()) {
    g_err = "buffer too small";
    return 1;
  }
  std::memcpy(dst, src.data(), src.size());
  return 0;
}
}  // namespace

extern "C" {

const char* oracle_last_error() { return g_err.c_str(); }
void oracle_set_threads(int n) { set_threads(n); }
int oracle_threads() { return threads(); }

// ---- numerics floor ------------------------------------------------------
void oracle_matmul(const float* a, const float* b, float* c, int m, int k, int p) {
  matmul(a, b, c, m, k, p);
}
void oracle_softmax_row(float* row, int k) { softmax_row(row, k); }
void oracle_rmsnorm(const float* x, const float* g, int d, float* out) { rmsnorm(x, g, d, out); }
int oracle_ffn_hidden(int d) { return ffn_hidden(d); }
void oracle_conv2d(const float* x, int c, int h, int w, const float* k, int o, int kh, int kw,
                   int stride, int pad, float* y, int* oh, int* ow) {
  conv2d(x, c, h, w, k, o, kh, kw, stride, pad, y, oh, ow);
}
void oracle_upsample2(const float* x, int c, int h, int w, float* y) { upsample2(x, c, h, w, y); }
double oracle_det(int fn, double x) {
  switch (fn) {
    case 0: return det::exp(x);
    case 1: return det::log(x);
    case 2: return det::erf(x);
    case 3: return det::normal_cdf(x);
    default: return 0.0;
  }
}
float oracle_det_f32(int fn, float x) {
  switch (fn) {
    case 0: return det::exp_f32(x);
    case 1: return det::silu_f32(x);
    case 2: return det::tanh_f32(x);
    case 3: return det::softplus_f32(x);
    default: return 0.0f;
  }
}
void oracle_rng(uint64_t seed, int n, uint64_t* u64_out, float* uniform_out, float* normal_out) {
  Rng a(seed), b(seed), c(seed);
  for (int i = 0; i < n; ++i) {
    if (u64_out) u64_out[i] = a.u64();
    if (uniform_out) uniform_out[i] = b.uniform();
    if (normal_out) normal_out[i] = c.normal();
  }
}
uint64_t oracle_fnv1a(const void* p, size_t n) { return fnv1a(p, n); }
void oracle_init_values(uint64_t seed, float* dst, size_t n, int kind, int fan_in) {
  Rng r(seed);
  init_values(r, dst, n, kind, fan_in);
}

// ---- wavefront -------------------------------------------------------------
int oracle_positions_of_step(int H, int W, int s, int t, int* out) {
  const auto v = positions_of_step(H, W, s, t);
  if (out) std::memcpy(out, v.data(), v.size() * sizeof(int));
  return static_cast<int>(v.size());
}
void oracle_channel_mask(int N, int dg, uint8_t* out) {
  const auto v = channel_mask(N, dg);
  std::memcpy(out, v.data(), v.size());
}
int oracle_validate_schedule(int H, int W, int s, int wh, int ww, int N, int* steps) {
  const Schedule r = validate_schedule(H, W, s, wh, ww, N);
  *steps = r.steps;
  return r.ok ? 1 : 0;
}

// ---- coder -----------------------------------------------------------------
void oracle_scale_table(float* out) { std::memcpy(out, tables().scale, sizeof(float) * kScales); }
void oracle_cdf_tables(uint32_t* out) { std::memcpy(out, tables().cdf, sizeof(tables().cdf) / 2); }
void oracle_cdf_tables_family(int laplace, uint32_t* out) {
  std::memcpy(out, tables().cdf[laplace ? kScales : 0], sizeof(tables().cdf) / 2);
}
int oracle_scale_index(float s) { return scale_index(s); }
int oracle_encode_lanes(const int32_t* v, const int32_t* idx, size_t n, int lanes, uint8_t* out,
                        size_t cap, size_t* len) {
  return guard([&] {
    std::vector<CodedSym> s(n);
    for (size_t i = 0; i < n; ++i) s[i] = {v[i], idx[i]};
    if (copy_out(encode_lanes(s, lanes), out, cap, len)) throw std::runtime_error(g_err);
  });
}
// returns 0 ok, 2 corrupt/truncated
int oracle_decode_lanes(const uint8_t* data, size_t n, const int32_t* idx, size_t count,
                        int32_t* v_out) {
  LaneDecoder d;
  if (!d.init(data, n) || d.count != count) return 2;
  for (size_t i = 0; i < count; ++i) v_out[i] = d.decode(i, idx[i]);
  return d.error ? 2 : 0;
}
double oracle_bits(const int32_t* v, const int32_t* idx, size_t n) {
  double b = 0;
  for (size_t i = 0; i < n; ++i) b += bits_of({v[i], idx[i]});
  return b;
}

// ---- model -------------------------------------------------------------------
int oracle_gen_weights(const int* cfg, uint64_t seed, uint8_t* buf, size_t cap, size_t* len) {
  return guard([&] {
    const Config c = to_cfg(cfg);
    if (copy_out(to_psww(c, gen_weights(c, seed)), buf, cap, len)) throw std::runtime_error(g_err);
  });
}
int64_t oracle_param_count(const int* cfg) {
  int64_t n = 0;
  for (const auto& s : param_specs(to_cfg(cfg))) {
    int64_t k = 1;
    for (int e : s.shape) k *= e;
    n += k;
  }
  return n;
}
void* oracle_model_create(const int* cfg, const uint8_t* blob, size_t n) {
  try {
    const Config c = to_cfg(cfg);
    return new Model(c, from_psww(c, blob, n));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
void oracle_model_destroy(void* h) { delete static_cast<Model*>(h); }

int oracle_forward(void* h, const int32_t* yhat, const int32_t* zhat_or_null, int rate,
                   const int32_t* const* past, int npast, float* mu, float* sigma,
                   int32_t* zhat_out, float* s2_out) {
  return guard([&] {
    const Model& m = *static_cast<Model*>(h);
    const Forward f = forward(m, yhat, zhat_or_null, rate, past_list(past, npast));
    std::memcpy(mu, f.mu.data(), f.mu.size() * sizeof(float));
    std::memcpy(sigma, f.sigma.data(), f.sigma.size() * sizeof(float));
    if (zhat_out) std::memcpy(zhat_out, f.zhat.data(), f.zhat.size() * sizeof(int32_t));
    if (s2_out) std::memcpy(s2_out, f.s2.data(), f.s2.size() * sizeof(float));
  });
}

int oracle_lrp(void* h, const int32_t* yhat, const int32_t* zhat, int rate,
               const int32_t* const* past, int npast, float* eps) {
  return guard([&] {
    const Model& m = *static_cast<Model*>(h);
    if (m.c.lrp_blocks <= 0) throw std::invalid_argument("oracle_lrp: lrp_blocks == 0");
    const Forward f = forward(m, yhat, zhat, rate, past_list(past, npast));
    std::memcpy(eps, f.eps.data(), f.eps.size() * sizeof(float));
  });
}

int oracle_forward_debug(void* h, const int32_t* yhat, const int32_t* zhat, int rate,
                         const int32_t* const* past, int npast, float* ctx, float* s1, float* hq,
                         float* a, float* s2) {
  return guard([&] {
    const Model& m = *static_cast<Model*>(h);
    const Forward f = forward(m, yhat, zhat, rate, past_list(past, npast));
    const size_t n = f.ctx.size() * sizeof(float);
    std::memcpy(ctx, f.ctx.data(), n);
    std::memcpy(s1, f.s1.data(), n);
    std::memcpy(hq, f.hq.data(), n);
    std::memcpy(a, f.a.data(), n);
    std::memcpy(s2, f.s2.data(), n);
  });
}

int oracle_encode(void* h, const int32_t* yhat, int rate, int fidx, const int32_t* const* past,
                  int npast, const int32_t* zhat_override, uint8_t* hyper, size_t hcap,
                  size_t* hlen, uint8_t* main, size_t mcap, size_t* mlen, double* bits,
                  int32_t* zhat_out) {
  return guard([&] {
    const Model& m = *static_cast<Model*>(h);
    const Payload p = encode_frame(m, yhat, rate, fidx, past_list(past, npast), zhat_override);
    if (copy_out(p.hyper, hyper, hcap, hlen) || copy_out(p.main, main, mcap, mlen))
      throw std::runtime_error(g_err);
    if (bits) {
      bits[0] = p.hyper_bits;
      bits[1] = p.main_bits;
    }
    if (zhat_out) std::memcpy(zhat_out, p.zhat.data(), p.zhat.size() * sizeof(int32_t));
  });
}

// mode 0: wavefront, 1: serial. Returns 0 ok, 1 error, 2 corrupt stream.
int oracle_decode(void* h, int mode, const uint8_t* hyper, size_t hlen, const uint8_t* main,
                  size_t mlen, int rate, int fidx, const int32_t* const* past, int npast,
                  int32_t* yhat_out, double* bits, int* phases) {
  int rc = 0;
  const int g = guard([&] {
    const Model& m = *static_cast<Model*>(h);
    Payload p;
    p.hyper.assign(hyper, hyper + hlen);
    p.main.assign(main, main + mlen);
    const Decoded d = mode == 0 ? decode_wavefront(m, p, rate, fidx, past_list(past, npast))
                                : decode_serial(m, p, rate, fidx, past_list(past, npast));
    if (!d.ok) {
      rc = 2;
      return;
    }
    std::memcpy(yhat_out, d.yhat.data(), d.yhat.size() * sizeof(int32_t));
    if (bits) {
      bits[0] = d.hyper_bits;
      bits[1] = d.main_bits;
    }
    if (phases) *phases = d.phases;
  });
  return g ? 1 : rc;
}

}  // extern "C"

// ---- synthetic latents ------------------------------------------
// Independent restatement of the bench input generator, so the reference arm
// of bench.py builds its inputs without the product library:
//   y[c,p] ~ Laplace(0, b_g), b_g = 8 / 2^g for channel group g (inverse CDF
//   with det::log on a 24-bit uniform in (0,1)); P-frames add Laplace(0, b_g/4)
//   to the previous frame; frame seed 1000 + 100 gop + frame; y_hat =
//   round-half-even(y); 1 in 10^4 positions forced to +-300.
// Writes frames [0, n_frames) of GOP `gop`: out[f][C][H][W].
extern "C" int oracle_synth_gop(const int* cfg, int gop, int n_frames, int32_t* out) {
  return guard([&] {
    const Config c = to_cfg(cfg);
    const int C = c.C, HW = c.H * c.W, Cg = C / c.N;
    std::vector<float> y(static_cast<size_t>(C) * HW, 0.0f);
    auto lap = [](Rng& r, double b) {
      const double u = (static_cast<double>(r.u64() >> 40) + 0.5) / 16777216.0;
      return u < 0.5 ? b * det::log(2.0 * u) : -b * det::log(2.0 * (1.0 - u));
    };
    for (int f = 0; f < n_frames; ++f) {
      const uint64_t seed = 1000ull + 100ull * static_cast<uint64_t>(gop) + static_cast<uint64_t>(f);
      Rng r(seed);
      for (int ch = 0; ch < C; ++ch) {
        const int g = ch / Cg;
        const double b = 8.0 / static_cast<double>(1 << (g < 30 ? g : 30));
        float* row = y.data() + static_cast<size_t>(ch) * HW;
        for (int p = 0; p < HW; ++p)
          row[p] = f == 0 ? static_cast<float>(lap(r, b)) : row[p] + static_cast<float>(lap(r, b / 4.0));
      }
      int32_t* o = out + static_cast<size_t>(f) * C * HW;
      for (size_t i = 0; i < y.size(); ++i) o[i] = static_cast<int32_t>(std::nearbyint(y[i]));
      Rng e(seed ^ 0x5EEDE5CA9Eull);
      for (int p = 0; p < HW; ++p)
        if (e.u64() % 10000 == 0) {
          const int ch = static_cast<int>(e.u64() % static_cast<uint64_t>(C));
          o[static_cast<size_t>(ch) * HW + p] = (e.u64() & 1) ? 300 : -300;
        }
    }
  });
}
