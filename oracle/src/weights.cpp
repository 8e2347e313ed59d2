// ORACLE — test infrastructure only.
// Config presets, wavefront schedule (wavefront.h:29-66),
// deterministic weights and the PSWW container.
#include <cstring>
#include <sstream>
#include <stdexcept>

#include "oracle/model.h"

namespace oracle {

std::string Config::canonical() const {
  std::ostringstream o;
  o << "pswa-v1;d=" << d << ";h=" << heads << ";ctx=" << ctx_blocks << ";s1=" << s1_blocks
    << ";s2=" << s2_blocks << ";dch=" << d_ch << ";chb=" << ch_blocks << ";hc=" << hyper_ch
    << ";C=" << C << ";s=" << s << ";N=" << N << ";wh=" << wh << ";ww=" << ww << ";wt=" << wt
    << ";T=" << T << ";R=" << rates;
  if (lrp_blocks > 0) o << ";lrp=" << lrp_blocks;
  return o.str();
}

Config preset(int paper, int H, int W) {
  Config c;
  if (paper) {
    c.d = 512;
    c.ctx_blocks = c.s1_blocks = c.s2_blocks = 8;
    c.d_ch = 1024;
    c.hyper_ch = 128;
  }
  c.H = H;
  c.W = W;
  return c;
}

// ------------------------------------------------------------ wavefront ---
std::vector<int> positions_of_step(int H, int W, int s, int t) {
  std::vector<int> out;
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x)
      if (step_of(y, x, s) == t) out.push_back(y * W + x);
  return out;
}

std::vector<uint8_t> channel_mask(int N, int dg) {
  const int n = N * dg;
  std::vector<uint8_t> m(static_cast<size_t>(n) * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) m[static_cast<size_t>(i) * n + j] = (i / dg) >= (j / dg);
  return m;
}

// Enumerates every direct dependency edge of the model's symbol graph and
// checks (a) accumulator edges strictly backward in step, (b) spatial-self
// edges never forward, (c) canonical order (t, g, raster) is topological,
// (d) the number of sequential phases is s*N.
Schedule validate_schedule(int H, int W, int s, int wh, int ww, int N) {
  Schedule r;
  auto rank = [&](int y, int x, int g) {
    // canonical decode rank: step-major, group-minor, raster within step
    return (static_cast<int64_t>(step_of(y, x, s)) * N + g) * H * W + y * W + x;
  };
  const int ry = wh / 2, rx = ww / 2;
  for (int y = 0; y < H && r.ok; ++y)
    for (int x = 0; x < W && r.ok; ++x) {
      const int qs = step_of(y, x, s);
      for (int dy = -ry; dy <= ry && r.ok; ++dy)
        for (int dx = -rx; dx <= rx && r.ok; ++dx) {
          const int ky = y + dy, kx = x + dx;
          if (ky < 0 || ky >= H || kx < 0 || kx >= W) continue;
          const int ks = step_of(ky, kx, s);
          if (mask_allows(kAccLt, qs, ks) && !(ks < qs)) {
            r.ok = false;
            r.violation = "accumulator edge not strictly backward";
          }
          if (mask_allows(kSelfLe, qs, ks) && ks > qs) {
            r.ok = false;
            r.violation = "spatial_self edge goes forward";
          }
          // symbol edges: (k, g') -> (q, g) through S1 -> accumulator
          if (mask_allows(kAccLt, qs, ks))
            for (int g = 0; g < N && r.ok; ++g)
              for (int g2 = 0; g2 < N; ++g2)
                if (rank(ky, kx, g2) >= rank(y, x, g)) {
                  r.ok = false;
                  r.violation = "decode order not topological";
                  break;
                }
        }
      // channel edges at the same position: (q, g') -> (q, g), g' < g
      for (int g = 0; g < N && r.ok; ++g)
        for (int g2 = 0; g2 < g; ++g2)
          if (rank(y, x, g2) >= rank(y, x, g)) {
            r.ok = false;
            r.violation = "channel order not topological";
          }
    }
  r.steps = s * N;
  return r;
}

// ------------------------------------------------------------- weights ----
std::vector<ParamSpec> param_specs(const Config& c) {
  std::vector<ParamSpec> v;
  const int d = c.d, h = c.heads, f = c.f(), hc = c.hyper_ch, R = c.rates;
  const int sl = c.slot(), fg = c.fg(), Cg = c.Cg(), dch = c.d_ch;
  auto add = [&](std::string n, std::vector<int> s, int kind, int fan) {
    v.push_back({std::move(n), std::move(s), kind, fan});
  };
  add("embed.w", {c.C, d}, 0, c.C);
  add("embed.b", {d}, 1, 1);
  add("rate.in", {R, d}, 2, 1);
  add("rate.hyper", {R, d}, 2, 1);
  add("rate.out", {R, c.C}, 2, 1);
  add("pad", {d}, 0, d);
  struct Mod {
    const char* name;
    int blocks;
    int taps;
  };
  const Mod mods[3] = {{"ctx", c.ctx_blocks, c.taps3()},
                       {"s1", c.s1_blocks, c.taps2()},
                       {"s2", c.s2_blocks, c.taps2()}};
  for (const Mod& md : mods) {
    for (int i = 0; i < md.blocks; ++i) {
      const std::string P = std::string(md.name) + ".b" + std::to_string(i);
      add(P + ".norm1.g", {d}, 2, 1);
      add(P + ".wq", {d, d}, 0, d);
      add(P + ".wk", {d, d}, 0, d);
      add(P + ".wv", {d, d}, 0, d);
      add(P + ".wo", {d, d}, 0, d);
      add(P + ".pos", {h, md.taps}, 0, md.taps);
      add(P + ".norm2.g", {d}, 2, 1);
      add(P + ".ffn.wg", {d, f}, 0, d);
      add(P + ".ffn.wu", {d, f}, 0, d);
      add(P + ".ffn.wd", {f, d}, 0, f);
    }
    add(std::string(md.name) + ".norm_out.g", {d}, 2, 1);
  }
  for (int j = 0; j < 2; ++j) {
    const std::string P = "hd.rb" + std::to_string(j);
    add(P + ".c1.w", {hc, hc, 3, 3}, 0, hc * 9);
    add(P + ".c1.b", {hc}, 1, 1);
    add(P + ".c2.w", {hc, hc, 3, 3}, 0, hc * 9);
    add(P + ".c2.b", {hc}, 1, 1);
  }
  add("hd.out.w", {d, hc, 1, 1}, 0, hc);
  add("hd.out.b", {d}, 1, 1);
  add("he.in.w", {hc, d, 1, 1}, 0, d);
  add("he.in.b", {hc}, 1, 1);
  for (int j = 0; j < 2; ++j) {
    const std::string P = "he.rb" + std::to_string(j);
    add(P + ".c1.w", {hc, hc, 3, 3}, 0, hc * 9);
    add(P + ".c1.b", {hc}, 1, 1);
    add(P + ".c2.w", {hc, hc, 3, 3}, 0, hc * 9);
    add(P + ".c2.b", {hc}, 1, 1);
  }
  add("hyper.loc", {R, 5, hc}, 1, 1);
  add("hyper.scale", {R, 5, hc}, 3, 1);
  add("acc.normq.g", {d}, 2, 1);
  add("acc.wq", {d, d}, 0, d);
  add("acc.wk", {d, d}, 0, d);
  add("acc.wv", {d, d}, 0, d);
  add("acc.wo", {d, d}, 0, d);
  add("acc.pos", {h, c.taps2()}, 0, c.taps2());
  for (int g = 0; g < c.N; ++g) add("ch.proj" + std::to_string(g) + ".w", {d, sl}, 0, d);
  for (int g = 1; g < c.N; ++g) add("ch.emb" + std::to_string(g) + ".w", {Cg, sl}, 0, Cg);
  for (int b = 0; b < c.ch_blocks; ++b) {
    const std::string P = "ch.b" + std::to_string(b);
    add(P + ".norm1.g", {dch}, 2, 1);
    add(P + ".mix.w", {dch, dch}, 0, dch);
    add(P + ".norm2.g", {dch}, 2, 1);
    for (int g = 0; g < c.N; ++g) {
      const std::string F = P + ".ffn" + std::to_string(g);
      add(F + ".wg", {sl, fg}, 0, sl);
      add(F + ".wu", {sl, fg}, 0, sl);
      add(F + ".wd", {fg, sl}, 0, fg);
    }
  }
  add("ch.norm_out.g", {dch}, 2, 1);
  for (int g = 0; g < c.N; ++g)
    for (const char* hn : {"mu", "sg"}) {
      const std::string P = std::string("head.") + hn + std::to_string(g);
      add(P + ".w1", {sl, sl}, 0, sl);
      add(P + ".b1", {sl}, 1, 1);
      add(P + ".w2", {sl, Cg}, 0, sl);
      add(P + ".b2", {Cg}, 1, 1);
    }
  if (c.lrp_blocks > 0) {  // LRP transformer (A8)
    add("lrp.in.w", {dch + c.C, d}, 0, dch + c.C);
    add("lrp.in.b", {d}, 1, 1);
    for (int i = 0; i < c.lrp_blocks; ++i) {
      const std::string P = "lrp.b" + std::to_string(i);
      add(P + ".norm1.g", {d}, 2, 1);
      add(P + ".wq", {d, d}, 0, d);
      add(P + ".wk", {d, d}, 0, d);
      add(P + ".wv", {d, d}, 0, d);
      add(P + ".wo", {d, d}, 0, d);
      add(P + ".pos", {h, c.taps3()}, 0, c.taps3());
      add(P + ".norm2.g", {d}, 2, 1);
      add(P + ".ffn.wg", {d, f}, 0, d);
      add(P + ".ffn.wu", {d, f}, 0, d);
      add(P + ".ffn.wd", {f, d}, 0, f);
    }
    add("lrp.norm_out.g", {d}, 2, 1);
    add("lrp.head.w", {d, c.C}, 0, d);
    add("lrp.head.b", {c.C}, 1, 1);
  }
  return v;
}

const Param& Weights::at(const std::string& n) const {
  auto it = p.find(n);
  if (it == p.end()) throw std::invalid_argument("missing weight: " + n);
  return it->second;
}
const float* Weights::operator[](const std::string& n) const { return at(n).v.data(); }

Weights gen_weights(const Config& c, uint64_t seed) {
  Weights w;
  for (const ParamSpec& s : param_specs(c)) {
    size_t n = 1;
    for (int e : s.shape) n *= static_cast<size_t>(e);
    Param prm;
    prm.shape = s.shape;
    prm.v.resize(n);
    Rng r = param_rng(seed, s.name);
    if (s.kind == 3) {
      init_values(r, prm.v.data(), n, 2, 1);
      for (float& x : prm.v) x *= 2.0f;
    } else {
      init_values(r, prm.v.data(), n, s.kind, s.fan_in);
    }
    w.order.push_back(s.name);
    w.p.emplace(s.name, std::move(prm));
  }
  return w;
}

namespace {
void put32(std::vector<uint8_t>& b, uint32_t v) {
  for (int i = 0; i < 4; ++i) b.push_back(static_cast<uint8_t>(v >> (8 * i)));
}
void put64(std::vector<uint8_t>& b, uint64_t v) {
  for (int i = 0; i < 8; ++i) b.push_back(static_cast<uint8_t>(v >> (8 * i)));
}
struct Reader {
  const uint8_t* p;
  const uint8_t* e;
  uint32_t u32() {
    if (e - p < 4) throw std::invalid_argument("PSWW truncated");
    uint32_t v = 0;
    for (int i = 0; i < 4; ++i) v |= static_cast<uint32_t>(p[i]) << (8 * i);
    p += 4;
    return v;
  }
  uint64_t u64() {
    const uint64_t lo = u32();
    return lo | (static_cast<uint64_t>(u32()) << 32);
  }
};
}  // namespace

std::vector<uint8_t> to_psww(const Config& c, const Weights& w) {
  std::vector<uint8_t> b = {'P', 'S', 'W', 'W'};
  put32(b, 1);
  put64(b, fnv1a(c.canonical()));
  put32(b, static_cast<uint32_t>(w.order.size()));
  for (const std::string& n : w.order) {
    const Param& p = w.at(n);
    put32(b, static_cast<uint32_t>(n.size()));
    b.insert(b.end(), n.begin(), n.end());
    put32(b, static_cast<uint32_t>(p.shape.size()));
    for (int e : p.shape) put32(b, static_cast<uint32_t>(e));
    const size_t off = b.size();
    b.resize(off + p.v.size() * 4);
    std::memcpy(b.data() + off, p.v.data(), p.v.size() * 4);  // x86: LE
  }
  return b;
}

Weights from_psww(const Config& c, const uint8_t* data, size_t n) {
  Reader r{data, data + n};
  if (n < 4 || std::memcmp(data, "PSWW", 4) != 0) throw std::invalid_argument("PSWW magic");
  r.p += 4;
  if (r.u32() != 1) throw std::invalid_argument("PSWW version");
  if (r.u64() != fnv1a(c.canonical())) throw std::invalid_argument("PSWW config hash mismatch");
  const uint32_t count = r.u32();
  Weights w;
  for (uint32_t i = 0; i < count; ++i) {
    const uint32_t ln = r.u32();
    if (static_cast<size_t>(r.e - r.p) < ln) throw std::invalid_argument("PSWW truncated");
    std::string name(reinterpret_cast<const char*>(r.p), ln);
    r.p += ln;
    Param p;
    const uint32_t rank = r.u32();
    size_t numel = 1;
    for (uint32_t k = 0; k < rank; ++k) {
      p.shape.push_back(static_cast<int>(r.u32()));
      numel *= static_cast<size_t>(p.shape.back());
    }
    if (static_cast<size_t>(r.e - r.p) < numel * 4) throw std::invalid_argument("PSWW truncated");
    p.v.resize(numel);
    std::memcpy(p.v.data(), r.p, numel * 4);
    r.p += numel * 4;
    if (w.p.count(name)) throw std::invalid_argument("PSWW duplicate name " + name);
    w.order.push_back(name);
    w.p.emplace(name, std::move(p));
  }
  for (const ParamSpec& s : param_specs(c)) {
    auto it = w.p.find(s.name);
    if (it == w.p.end()) throw std::invalid_argument("PSWW missing " + s.name);
    if (it->second.shape != s.shape) throw std::invalid_argument("PSWW shape " + s.name);
  }
  if (w.p.size() != param_specs(c).size()) throw std::invalid_argument("PSWW extra tensors");
  return w;
}

}  // namespace oracle
