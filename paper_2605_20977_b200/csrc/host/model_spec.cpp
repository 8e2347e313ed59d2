#include "model_spec.h"

#include <cmath>
#include <cstring>
#include <sstream>
#include <stdexcept>
#include <algorithm>
#include <atomic>
#include <thread>

#include "pswa/det_math.h"
#include "pswa/rng.h"

namespace pswa_host {

namespace {
int up64(int v) { return (v + 63) / 64 * 64; }
}  // namespace

int ffn_hidden_dim(int d) {
  const long units = std::lround(static_cast<double>(d) / 3.0);
  return 8 * static_cast<int>(units < 1 ? 1 : units);
}

Dims::Dims(const pswa_cfg& cfg) : c(cfg) {
  d = c.d_spatial;
  heads = c.heads;
  hd = d / heads;
  f = ffn_hidden_dim(d);
  fp = up64(f);
  dch = c.d_channel;
  N = c.n_groups;
  slot = dch / N;
  sp = up64(slot);
  fg = ffn_hidden_dim(slot);
  fgp = up64(fg);
  C = c.latent_ch;
  Cg = C / N;
  Cgp = up64(Cg);
  hc = c.hyper_ch;
  hcp = up64(hc);
  kconv = up64(9 * hc);
  H = c.height;
  W = c.width;
  HW = H * W;
  Hp = (H + 3) / 4 * 4;
  Wp = (W + 3) / 4 * 4;
  zh = Hp / 4;
  zw = Wp / 4;
  T = c.ctx_slots;
  taps2 = c.win_h * c.win_w;
  taps3 = c.win_t * taps2;
}

void validate_cfg(const pswa_cfg& c) {
  auto req = [](bool ok, const char* what) {
    if (!ok) throw std::invalid_argument(std::string("pswa_cfg: ") + what);
  };
  req(c.d_spatial > 0 && c.heads > 0 && c.d_spatial % c.heads == 0, "d % heads");
  req(c.d_spatial % 64 == 0, "d_spatial must be a multiple of 64");
  req(c.n_groups > 0 && c.latent_ch % c.n_groups == 0, "C % N");
  req(c.latent_ch % 64 == 0, "latent_ch must be a multiple of 64");
  req(c.d_channel % c.n_groups == 0, "d_channel % N");
  req(c.win_h % 2 == 1 && c.win_w % 2 == 1 && c.win_t >= 1, "window extents must be odd");
  req(c.height > 0 && c.width > 0 && c.height < 4096 && c.width < 4096, "grid");
  req(c.s >= 1 && c.ctx_slots >= 1 && c.ctx_slots < 64 && c.rate_points >= 1, "s / T / R");
  req(c.lanes >= 1 && c.hyper_lanes >= 1, "lanes");
  req(c.prior == 0 || c.prior == 1, "prior must be 0 (Gaussian) or 1 (Laplace)");
  req(c.lrp_blocks >= 0 && c.lrp_blocks <= 16, "lrp_blocks in [0, 16]");
  req(c.win_t * c.win_h * c.win_w <= 256, "window taps <= 256");
  const int hd = c.d_spatial / c.heads;
  req(hd == 4 || hd == 8 || hd == 16 || hd == 32 || hd == 64, "head_dim in {4..64}");
}

std::string canonical_cfg(const pswa_cfg& c) {
  std::ostringstream o;
  o << "pswa-v1;d=" << c.d_spatial << ";h=" << c.heads << ";ctx=" << c.ctx_blocks
    << ";s1=" << c.s1_blocks << ";s2=" << c.s2_blocks << ";dch=" << c.d_channel
    << ";chb=" << c.ch_blocks << ";hc=" << c.hyper_ch << ";C=" << c.latent_ch << ";s=" << c.s
    << ";N=" << c.n_groups << ";wh=" << c.win_h << ";ww=" << c.win_w << ";wt=" << c.win_t
    << ";T=" << c.ctx_slots << ";R=" << c.rate_points;
  if (c.lrp_blocks > 0) o << ";lrp=" << c.lrp_blocks;
  return o.str();
}

std::vector<ParamDecl> param_inventory(const pswa_cfg& c) {
  const Dims D(c);
  const int R = c.rate_points;
  std::vector<ParamDecl> v;
  auto P = [&](std::string n, std::vector<int> s, Init i, int fan = 1) {
    v.push_back({std::move(n), std::move(s), i, fan});
  };
  auto linear = [&](const std::string& n, int in, int out) { P(n, {in, out}, Init::kScaledNormal, in); };
  auto gain = [&](const std::string& n, int w) { P(n, {w}, Init::kOnes); };
  auto zeros = [&](const std::string& n, int w) { P(n, {w}, Init::kZeros); };

  linear("embed.w", D.C, D.d);
  zeros("embed.b", D.d);
  P("rate.in", {R, D.d}, Init::kOnes);
  P("rate.hyper", {R, D.d}, Init::kOnes);
  P("rate.out", {R, D.C}, Init::kOnes);
  P("pad", {D.d}, Init::kScaledNormal, D.d);

  // context transformer (3D SWA), spatial modules 1 and 2 (2D, self/cross)
  const struct {
    const char* tag;
    int blocks, taps;
  } stacks[] = {{"ctx", c.ctx_blocks, D.taps3}, {"s1", c.s1_blocks, D.taps2}, {"s2", c.s2_blocks, D.taps2}};
  for (const auto& st : stacks) {
    for (int b = 0; b < st.blocks; ++b) {
      const std::string p = std::string(st.tag) + ".b" + std::to_string(b);
      gain(p + ".norm1.g", D.d);
      for (const char* w : {".wq", ".wk", ".wv", ".wo"}) linear(p + w, D.d, D.d);
      P(p + ".pos", {D.heads, st.taps}, Init::kScaledNormal, st.taps);
      gain(p + ".norm2.g", D.d);
      linear(p + ".ffn.wg", D.d, D.f);
      linear(p + ".ffn.wu", D.d, D.f);
      linear(p + ".ffn.wd", D.f, D.d);
    }
    gain(std::string(st.tag) + ".norm_out.g", D.d);
  }
  // hyperprior decoder / encoder (RB-up / RB-down residual blocks)
  auto rb = [&](const std::string& p) {
    for (const char* cv : {".c1", ".c2"}) {
      P(p + cv + ".w", {D.hc, D.hc, 3, 3}, Init::kScaledNormal, D.hc * 9);
      zeros(p + cv + ".b", D.hc);
    }
  };
  rb("hd.rb0");
  rb("hd.rb1");
  P("hd.out.w", {D.d, D.hc, 1, 1}, Init::kScaledNormal, D.hc);
  zeros("hd.out.b", D.d);
  P("he.in.w", {D.hc, D.d, 1, 1}, Init::kScaledNormal, D.d);
  zeros("he.in.b", D.hc);
  rb("he.rb0");
  rb("he.rb1");
  P("hyper.loc", {R, 5, D.hc}, Init::kZeros);
  P("hyper.scale", {R, 5, D.hc}, Init::kTwo);
  // accumulator
  gain("acc.normq.g", D.d);
  for (const char* w : {"acc.wq", "acc.wk", "acc.wv", "acc.wo"}) linear(w, D.d, D.d);
  P("acc.pos", {D.heads, D.taps2}, Init::kScaledNormal, D.taps2);
  // channel transformer
  for (int g = 0; g < D.N; ++g) linear("ch.proj" + std::to_string(g) + ".w", D.d, D.slot);
  for (int g = 1; g < D.N; ++g) linear("ch.emb" + std::to_string(g) + ".w", D.Cg, D.slot);
  for (int b = 0; b < c.ch_blocks; ++b) {
    const std::string p = "ch.b" + std::to_string(b);
    gain(p + ".norm1.g", D.dch);
    linear(p + ".mix.w", D.dch, D.dch);
    gain(p + ".norm2.g", D.dch);
    for (int g = 0; g < D.N; ++g) {
      const std::string q = p + ".ffn" + std::to_string(g);
      linear(q + ".wg", D.slot, D.fg);
      linear(q + ".wu", D.slot, D.fg);
      linear(q + ".wd", D.fg, D.slot);
    }
  }
  gain("ch.norm_out.g", D.dch);
  // grouped two-layer heads for mu and sigma
  for (int g = 0; g < D.N; ++g)
    for (const char* h : {"mu", "sg"}) {
      const std::string p = std::string("head.") + h + std::to_string(g);
      linear(p + ".w1", D.slot, D.slot);
      zeros(p + ".b1", D.slot);
      linear(p + ".w2", D.slot, D.Cg);
      zeros(p + ".b2", D.Cg);
    }
  // LRP transformer (A8)
  if (c.lrp_blocks > 0) {
    linear("lrp.in.w", D.dch + D.C, D.d);
    zeros("lrp.in.b", D.d);
    for (int b = 0; b < c.lrp_blocks; ++b) {
      const std::string p = "lrp.b" + std::to_string(b);
      gain(p + ".norm1.g", D.d);
      for (const char* w : {".wq", ".wk", ".wv", ".wo"}) linear(p + w, D.d, D.d);
      P(p + ".pos", {D.heads, D.taps3}, Init::kScaledNormal, D.taps3);
      gain(p + ".norm2.g", D.d);
      linear(p + ".ffn.wg", D.d, D.f);
      linear(p + ".ffn.wu", D.d, D.f);
      linear(p + ".ffn.wd", D.f, D.d);
    }
    gain("lrp.norm_out.g", D.d);
    linear("lrp.head.w", D.d, D.C);
    zeros("lrp.head.b", D.C);
  }
  return v;
}

namespace {
struct Writer {
  std::vector<uint8_t> b;
  void u32(uint32_t x) {
    for (int k = 0; k < 4; ++k) b.push_back(static_cast<uint8_t>(x >> (8 * k)));
  }
  void u64(uint64_t x) {
    u32(static_cast<uint32_t>(x));
    u32(static_cast<uint32_t>(x >> 32));
  }
};
}  // namespace

std::vector<uint8_t> gen_weights_psww(const pswa_cfg& c, uint64_t seed) {
  validate_cfg(c);
  const auto inv = param_inventory(c);
  Writer w;
  w.b = {'P', 'S', 'W', 'W'};
  w.u32(1);
  w.u64(pswa::fnv1a64(canonical_cfg(c)));
  w.u32(static_cast<uint32_t>(inv.size()));
  // layout pass: headers written now, data offsets recorded
  std::vector<size_t> off(inv.size()), cnt(inv.size());
  for (size_t k = 0; k < inv.size(); ++k) {
    const ParamDecl& p = inv[k];
    w.u32(static_cast<uint32_t>(p.name.size()));
    w.b.insert(w.b.end(), p.name.begin(), p.name.end());
    w.u32(static_cast<uint32_t>(p.shape.size()));
    size_t n = 1;
    for (int e : p.shape) {
      w.u32(static_cast<uint32_t>(e));
      n *= static_cast<size_t>(e);
    }
    off[k] = w.b.size();
    cnt[k] = n;
    w.b.resize(w.b.size() + 4 * n);
  }
  // value pass: one independent stream per parameter, so parameters can be
  // generated concurrently without changing a single byte
  auto fill = [&](size_t k) {
    const ParamDecl& p = inv[k];
    pswa::Rng r = pswa::rng_for_parameter(seed, p.name);
    const float sd = 1.0f / std::sqrt(static_cast<float>(p.fan_in < 1 ? 1 : p.fan_in));
    uint8_t* dst = w.b.data() + off[k];
    for (size_t i = 0; i < cnt[k]; ++i) {
      float x = 0.0f;
      switch (p.init) {
        case Init::kScaledNormal: x = r.next_normal() * sd; break;
        case Init::kZeros: x = 0.0f; break;
        case Init::kOnes: x = 1.0f; break;
        case Init::kTwo: x = 1.0f * 2.0f; break;
      }
      std::memcpy(dst + 4 * i, &x, 4);  // little-endian host
    }
  };
  const unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  std::vector<std::thread> pool;
  std::atomic<size_t> next{0};
  for (unsigned t = 0; t < nt; ++t)
    pool.emplace_back([&] {
      for (size_t k; (k = next.fetch_add(1)) < inv.size();) fill(k);
    });
  for (auto& th : pool) th.join();
  return w.b;
}

WeightMap parse_psww(const pswa_cfg& c, const void* blob, size_t n) {
  const auto* p = static_cast<const uint8_t*>(blob);
  size_t at = 0;
  auto need = [&](size_t k) {
    if (at + k > n) throw std::invalid_argument("PSWW: truncated");
  };
  auto u32 = [&]() {
    need(4);
    uint32_t x = 0;
    for (int k = 0; k < 4; ++k) x |= static_cast<uint32_t>(p[at + k]) << (8 * k);
    at += 4;
    return x;
  };
  need(4);
  if (std::memcmp(p, "PSWW", 4) != 0) throw std::invalid_argument("PSWW: bad magic");
  at = 4;
  if (u32() != 1) throw std::invalid_argument("PSWW: unsupported version");
  const uint64_t lo = u32(), hi = u32();
  if ((lo | (hi << 32)) != pswa::fnv1a64(canonical_cfg(c)))
    throw std::invalid_argument("PSWW: config hash mismatch");
  const uint32_t count = u32();
  WeightMap m;
  for (uint32_t e = 0; e < count; ++e) {
    const uint32_t ln = u32();
    need(ln);
    std::string name(reinterpret_cast<const char*>(p + at), ln);
    at += ln;
    HostTensor t;
    const uint32_t rank = u32();
    size_t numel = 1;
    for (uint32_t k = 0; k < rank; ++k) {
      t.shape.push_back(static_cast<int>(u32()));
      numel *= static_cast<size_t>(t.shape.back());
    }
    need(numel * 4);
    t.v.resize(numel);
    std::memcpy(t.v.data(), p + at, numel * 4);
    at += numel * 4;
    if (!m.emplace(name, std::move(t)).second) throw std::invalid_argument("PSWW: duplicate " + name);
  }
  const auto inv = param_inventory(c);
  for (const ParamDecl& d : inv) {
    auto it = m.find(d.name);
    if (it == m.end()) throw std::invalid_argument("PSWW: missing tensor " + d.name);
    if (it->second.shape != d.shape) throw std::invalid_argument("PSWW: shape mismatch " + d.name);
  }
  if (m.size() != inv.size()) throw std::invalid_argument("PSWW: unexpected extra tensors");
  return m;
}

// Frames [f_from, f_to] of GOP `gop` (the y random walk is regenerated from
// frame 0); frame f lands at out[(f - f_from) * C * HW].
static void synth_frames(const pswa_cfg& c, int gop, int f_from, int f_to, int32_t* out) {
  const int C = c.latent_ch, HW = c.height * c.width, Cg = C / c.n_groups;
  std::vector<float> y(static_cast<size_t>(C) * HW, 0.0f);
  auto laplace = [](pswa::Rng& r, double b) {
    const double u = (static_cast<double>(r.next_u64() >> 40) + 0.5) * 0x1p-24;  // (0,1)
    return u < 0.5 ? b * pswa::det::log(2.0 * u) : -b * pswa::det::log(2.0 * (1.0 - u));
  };
  for (int f = 0; f <= f_to; ++f) {
    pswa::Rng r(1000ull + 100ull * static_cast<uint64_t>(gop) + static_cast<uint64_t>(f));
    for (int ch = 0; ch < C; ++ch) {
      const double b = 8.0 / static_cast<double>(1 << (ch / Cg < 30 ? ch / Cg : 30));
      for (int p = 0; p < HW; ++p) {
        float& v = y[static_cast<size_t>(ch) * HW + p];
        v = f == 0 ? static_cast<float>(laplace(r, b)) : v + static_cast<float>(laplace(r, b / 4.0));
      }
    }
    if (f < f_from) continue;
    int32_t* yhat = out + static_cast<size_t>(f - f_from) * C * HW;
    for (size_t i = 0; i < y.size(); ++i) yhat[i] = static_cast<int32_t>(std::nearbyint(y[i]));
    pswa::Rng e((1000ull + 100ull * static_cast<uint64_t>(gop) + static_cast<uint64_t>(f)) ^ 0x5EEDE5CA9Eull);
    for (int p = 0; p < HW; ++p)
      if (e.next_u64() % 10000 == 0) {
        const int ch = static_cast<int>(e.next_u64() % static_cast<uint64_t>(C));
        yhat[static_cast<size_t>(ch) * HW + p] = (e.next_u64() & 1) ? 300 : -300;
      }
  }
}

void synth_latent(const pswa_cfg& c, int gop, int frame_idx, int32_t* yhat) {
  synth_frames(c, gop, frame_idx, frame_idx, yhat);
}

void synth_gop(const pswa_cfg& c, int gop, int n_frames, int32_t* out) {
  if (n_frames > 0) synth_frames(c, gop, 0, n_frames - 1, out);
}

}  // namespace pswa_host
