// ORACLE — test infrastructure only.
// The P-SWA entropy model on the reference numerics. Token
// tensors are [positions][width]; attention follows SPEC.md:221-256 with the
// out-of-bounds-masked window, raster key order and the zero-key contract.
#include <cmath>
#include <cstring>
#include <stdexcept>

#include "oracle/model.h"

namespace oracle {

Model::Model(const Config& cfg, Weights wts) : c(cfg), w(std::move(wts)) {
  if (c.d % c.heads || c.C % c.N || c.d_ch % c.N || c.H < 1 || c.W < 1)
    throw std::invalid_argument("oracle: bad config");
}

namespace {

// rows x [n][din] times W [din][dout]
Tok mm(const Tok& x, int n, int din, const float* w, int dout) {
  Tok y(static_cast<size_t>(n) * dout);
  matmul(x.data(), w, y.data(), n, din, dout);
  return y;
}

Tok norm_rows(const Tok& x, int n, int d, const float* g, int group) {
  Tok y(x.size());
  pfor(n, [&](int64_t i) {
    for (int o = 0; o < d; o += group)
      rmsnorm(x.data() + i * d + o, g + o, group, y.data() + i * d + o);
  });
  return y;
}

void add_into(Tok& x, const Tok& dlt) {
  for (size_t i = 0; i < x.size(); ++i) x[i] = x[i] + dlt[i];
}

Tok swiglu_rows(const Tok& xn, int n, int d, int f, const float* wg, const float* wu,
                const float* wd) {
  Tok g = mm(xn, n, d, wg, f);
  const Tok u = mm(xn, n, d, wu, f);
  for (size_t i = 0; i < g.size(); ++i) g[i] = det::silu_f32(g[i]) * u[i];
  return mm(g, n, f, wd, d);
}

// Windowed attention. Queries: positions qpos (raster) at slot qslot; keys:
// slots [qslot - wt + 1, qslot] (clipped at 0) of K/V ([slots][HW][d]) within
// the wh x ww window, filtered by bounds and the step mask. Softmax over the
// allowed keys in (slot, dy, dx) raster order.
void window_attention(const Config& c, int nq, const float* q, const int* qpos, const int* qslot,
                      const float* K, const float* V, int three_d, int mask, const float* bias,
                      float* out) {
  const int d = c.d, hd = c.hd(), H = c.H, W = c.W, ry = c.wh / 2, rx = c.ww / 2;
  const int taps = three_d ? c.taps3() : c.taps2();
  const float scale = 1.0f / std::sqrt(static_cast<float>(hd));
  pfor(nq, [&](int64_t i) {
    const int p = qpos[i], y = p / W, x = p % W, qs = step_of(y, x, c.s);
    const int sl = qslot ? qslot[i] : 0;
    const int j0 = three_d ? std::max(0, sl - c.wt + 1) : sl;
    std::vector<int> key_row, key_tap;
    for (int j = j0; j <= sl; ++j)
      for (int dy = -ry; dy <= ry; ++dy)
        for (int dx = -rx; dx <= rx; ++dx) {
          const int ky = y + dy, kx = x + dx;
          if (ky < 0 || ky >= H || kx < 0 || kx >= W) continue;
          if (!mask_allows(mask, qs, step_of(ky, kx, c.s))) continue;
          key_row.push_back(j * H * W + ky * W + kx);
          const int t2 = (dy + ry) * c.ww + (dx + rx);
          key_tap.push_back(three_d ? (j - sl + c.wt - 1) * c.taps2() + t2 : t2);
        }
    const int nk = static_cast<int>(key_row.size());
    std::vector<float> sc(static_cast<size_t>(nk));
    float* o = out + i * d;
    for (int h = 0; h < c.heads; ++h) {
      const float* qh = q + i * d + h * hd;
      for (int k = 0; k < nk; ++k) {
        const float* kh = K + static_cast<size_t>(key_row[k]) * d + h * hd;
        float dot = 0.0f;
        for (int e = 0; e < hd; ++e) dot += qh[e] * kh[e];
        sc[k] = dot * scale + bias[h * taps + key_tap[k]];
      }
      if (nk > 0) softmax_row(sc.data(), nk);
      for (int e = 0; e < hd; ++e) {
        float acc = 0.0f;
        for (int k = 0; k < nk; ++k) acc += sc[k] * V[static_cast<size_t>(key_row[k]) * d + h * hd + e];
        o[h * hd + e] = acc;
      }
    }
  });
}

std::vector<int> iota(int n) {
  std::vector<int> v(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) v[i] = i;
  return v;
}

// Rows of x for the given position set.
Tok gather(const Tok& x, int width, const std::vector<int>& pos) {
  Tok y(pos.size() * static_cast<size_t>(width));
  for (size_t i = 0; i < pos.size(); ++i)
    std::memcpy(y.data() + i * width, x.data() + static_cast<size_t>(pos[i]) * width,
                sizeof(float) * width);
  return y;
}

// (C,H,W) <-> tokens [HW][C]
Tok chw_to_tok(const float* x, int ch, int hw) {
  Tok t(static_cast<size_t>(ch) * hw);
  for (int c = 0; c < ch; ++c)
    for (int p = 0; p < hw; ++p) t[static_cast<size_t>(p) * ch + c] = x[static_cast<size_t>(c) * hw + p];
  return t;
}
std::vector<float> tok_to_chw(const Tok& t, int ch, int hw) {
  std::vector<float> x(static_cast<size_t>(ch) * hw);
  for (int c = 0; c < ch; ++c)
    for (int p = 0; p < hw; ++p) x[static_cast<size_t>(c) * hw + p] = t[static_cast<size_t>(p) * ch + c];
  return x;
}

std::vector<float> conv_bias(const std::vector<float>& x, int ci, int h, int w, const float* k,
                             const float* b, int co, int ks, int stride, int& oh, int& ow) {
  std::vector<float> y(static_cast<size_t>(co) * ((h + stride - 1) / stride + 2) *
                       ((w + stride - 1) / stride + 2));
  conv2d(x.data(), ci, h, w, k, co, ks, ks, stride, ks / 2, y.data(), &oh, &ow);
  y.resize(static_cast<size_t>(co) * oh * ow);
  for (int c = 0; c < co; ++c)
    for (int i = 0; i < oh * ow; ++i) y[static_cast<size_t>(c) * oh * ow + i] += b[c];
  return y;
}

}  // namespace

Tok embed(const Model& m, const int32_t* yhat, int rate) {
  const Config& c = m.c;
  const int hw = c.HW();
  Tok yt(static_cast<size_t>(hw) * c.C);
  for (int ch = 0; ch < c.C; ++ch)
    for (int p = 0; p < hw; ++p)
      yt[static_cast<size_t>(p) * c.C + ch] = static_cast<float>(yhat[static_cast<size_t>(ch) * hw + p]);
  Tok e = mm(yt, hw, c.C, m.w["embed.w"], c.d);
  const float* rs = m.w["rate.in"] + static_cast<size_t>(rate) * c.d;
  const float* b = m.w["embed.b"];
  for (int p = 0; p < hw; ++p)
    for (int j = 0; j < c.d; ++j) {
      float& v = e[static_cast<size_t>(p) * c.d + j];
      v = rs[j] * v + b[j];
    }
  return e;
}

Tok context_forward(const Model& m, const std::vector<const float*>& slots) {
  const Config& c = m.c;
  const int hw = c.HW(), d = c.d, T = c.T;
  Tok x(static_cast<size_t>(T) * hw * d);
  const float* pad = m.w["pad"];
  for (int t = 0; t < T; ++t)
    for (int p = 0; p < hw; ++p)
      std::memcpy(x.data() + (static_cast<size_t>(t) * hw + p) * d,
                  slots[t] ? slots[t] + static_cast<size_t>(p) * d : pad, sizeof(float) * d);
  const std::vector<int> all_pos = [&] {
    std::vector<int> v;
    for (int t = 0; t < T; ++t)
      for (int p = 0; p < hw; ++p) v.push_back(p);
    return v;
  }();
  for (int b = 0; b < c.ctx_blocks; ++b) {
    const std::string P = "ctx.b" + std::to_string(b);
    const bool last = b == c.ctx_blocks - 1;
    const int n = T * hw;
    const Tok xn = norm_rows(x, n, d, m.w[P + ".norm1.g"], d);
    const Tok K = mm(xn, n, d, m.w[P + ".wk"], d);
    const Tok V = mm(xn, n, d, m.w[P + ".wv"], d);
    // queries: every slot, or only the last slot in the final block
    const int q0 = last ? (T - 1) * hw : 0;
    const int nq = n - q0;
    Tok xq(xn.begin() + static_cast<size_t>(q0) * d, xn.end());
    const Tok Q = mm(xq, nq, d, m.w[P + ".wq"], d);
    std::vector<int> qpos(all_pos.begin() + q0, all_pos.end()), qslot(static_cast<size_t>(nq));
    for (int i = 0; i < nq; ++i) qslot[i] = (q0 + i) / hw;
    Tok att(static_cast<size_t>(nq) * d);
    window_attention(c, nq, Q.data(), qpos.data(), qslot.data(), K.data(), V.data(), 1, kNone,
                     m.w[P + ".pos"], att.data());
    const Tok o = mm(att, nq, d, m.w[P + ".wo"], d);
    Tok xs(x.begin() + static_cast<size_t>(q0) * d, x.end());
    add_into(xs, o);
    const Tok xn2 = norm_rows(xs, nq, d, m.w[P + ".norm2.g"], d);
    add_into(xs, swiglu_rows(xn2, nq, d, c.f(), m.w[P + ".ffn.wg"], m.w[P + ".ffn.wu"],
                             m.w[P + ".ffn.wd"]));
    std::memcpy(x.data() + static_cast<size_t>(q0) * d, xs.data(), xs.size() * sizeof(float));
  }
  Tok last(x.begin() + static_cast<size_t>(T - 1) * hw * d, x.end());
  return norm_rows(last, hw, d, m.w["ctx.norm_out.g"], d);
}

Tok spatial_forward(const Model& m, const std::string& prefix, int blocks, Tok x, const Tok& ctx) {
  const Config& c = m.c;
  const int hw = c.HW(), d = c.d;
  const std::vector<int> pos = iota(hw);
  for (int b = 0; b < blocks; ++b) {
    const std::string P = prefix + ".b" + std::to_string(b);
    const bool cross = (b % 2) == 1;  // strict alternation, self first
    const Tok xn = norm_rows(x, hw, d, m.w[P + ".norm1.g"], d);
    const Tok Q = mm(xn, hw, d, m.w[P + ".wq"], d);
    const Tok& kvsrc = cross ? ctx : xn;
    const Tok K = mm(kvsrc, hw, d, m.w[P + ".wk"], d);
    const Tok V = mm(kvsrc, hw, d, m.w[P + ".wv"], d);
    Tok att(static_cast<size_t>(hw) * d);
    window_attention(c, hw, Q.data(), pos.data(), nullptr, K.data(), V.data(), 0,
                     cross ? kNone : kSelfLe, m.w[P + ".pos"], att.data());
    add_into(x, mm(att, hw, d, m.w[P + ".wo"], d));
    const Tok xn2 = norm_rows(x, hw, d, m.w[P + ".norm2.g"], d);
    add_into(x, swiglu_rows(xn2, hw, d, c.f(), m.w[P + ".ffn.wg"], m.w[P + ".ffn.wu"],
                            m.w[P + ".ffn.wd"]));
  }
  return norm_rows(x, hw, d, m.w[prefix + ".norm_out.g"], d);
}

std::vector<int32_t> hyper_encode(const Model& m, const Tok& s1) {
  const Config& c = m.c;
  const int hc = c.hyper_ch;
  int h = c.Hp(), w = c.Wp(), oh, ow;
  // zero-padded to the hyper grid; pad positions are never coded
  std::vector<float> x(static_cast<size_t>(c.d) * h * w, 0.0f);
  for (int p = 0; p < c.HW(); ++p)
    for (int ch = 0; ch < c.d; ++ch)
      x[(static_cast<size_t>(ch) * h + p / c.W) * w + p % c.W] = s1[static_cast<size_t>(p) * c.d + ch];
  x = conv_bias(x, c.d, h, w, m.w["he.in.w"], m.w["he.in.b"], hc, 1, 1, oh, ow);
  for (int j = 0; j < 2; ++j) {
    const std::string P = "he.rb" + std::to_string(j);
    std::vector<float> h1 = conv_bias(x, hc, h, w, m.w[P + ".c1.w"], m.w[P + ".c1.b"], hc, 3, 2, oh, ow);
    for (float& v : h1) v = det::silu_f32(v);
    const int h2h = oh, h2w = ow;
    std::vector<float> h2 = conv_bias(h1, hc, h2h, h2w, m.w[P + ".c2.w"], m.w[P + ".c2.b"], hc, 3, 1, oh, ow);
    std::vector<float> out(static_cast<size_t>(hc) * oh * ow);
    for (int ch = 0; ch < hc; ++ch)
      for (int yy = 0; yy < oh; ++yy)
        for (int xx = 0; xx < ow; ++xx) {
          const float skip = x[(static_cast<size_t>(ch) * h + 2 * yy) * w + 2 * xx];
          out[(static_cast<size_t>(ch) * oh + yy) * ow + xx] =
              skip + h2[(static_cast<size_t>(ch) * oh + yy) * ow + xx];
        }
    x = std::move(out);
    h = oh;
    w = ow;
  }
  std::vector<int32_t> z(x.size());
  for (size_t i = 0; i < x.size(); ++i) z[i] = static_cast<int32_t>(std::nearbyint(x[i]));
  return z;
}

Tok hyper_decode(const Model& m, const int32_t* zhat, int rate) {
  const Config& c = m.c;
  const int hc = c.hyper_ch;
  int h = c.Hp() / 4, w = c.Wp() / 4, oh, ow;
  std::vector<float> x(static_cast<size_t>(hc) * h * w);
  for (size_t i = 0; i < x.size(); ++i) x[i] = static_cast<float>(zhat[i]);
  for (int j = 0; j < 2; ++j) {
    const std::string P = "hd.rb" + std::to_string(j);
    std::vector<float> u(static_cast<size_t>(hc) * 4 * h * w);
    upsample2(x.data(), hc, h, w, u.data());
    h *= 2;
    w *= 2;
    std::vector<float> h1 = conv_bias(u, hc, h, w, m.w[P + ".c1.w"], m.w[P + ".c1.b"], hc, 3, 1, oh, ow);
    for (float& v : h1) v = det::silu_f32(v);
    std::vector<float> h2 = conv_bias(h1, hc, h, w, m.w[P + ".c2.w"], m.w[P + ".c2.b"], hc, 3, 1, oh, ow);
    for (size_t i = 0; i < u.size(); ++i) u[i] = u[i] + h2[i];
    x = std::move(u);
  }
  std::vector<float> y = conv_bias(x, hc, h, w, m.w["hd.out.w"], m.w["hd.out.b"], c.d, 1, 1, oh, ow);
  const float* rs = m.w["rate.hyper"] + static_cast<size_t>(rate) * c.d;
  for (int ch = 0; ch < c.d; ++ch)
    for (int i = 0; i < h * w; ++i) {
      float& v = y[static_cast<size_t>(ch) * h * w + i];
      v = v * rs[ch];
    }
  // crop the padded hyper grid back to the latent grid
  Tok t(static_cast<size_t>(c.HW()) * c.d);
  for (int p = 0; p < c.HW(); ++p)
    for (int ch = 0; ch < c.d; ++ch)
      t[static_cast<size_t>(p) * c.d + ch] = y[(static_cast<size_t>(ch) * h + p / c.W) * w + p % c.W];
  return t;
}

Tok accumulate(const Model& m, const Tok& hq, const Tok& s1) {
  const Config& c = m.c;
  const int hw = c.HW(), d = c.d;
  const Tok qn = norm_rows(hq, hw, d, m.w["acc.normq.g"], d);
  const Tok Q = mm(qn, hw, d, m.w["acc.wq"], d);
  const Tok K = mm(s1, hw, d, m.w["acc.wk"], d);
  const Tok V = mm(s1, hw, d, m.w["acc.wv"], d);
  const std::vector<int> pos = iota(hw);
  Tok att(static_cast<size_t>(hw) * d);
  window_attention(c, hw, Q.data(), pos.data(), nullptr, K.data(), V.data(), 0, kAccLt,
                   m.w["acc.pos"], att.data());
  Tok a = hq;
  add_into(a, mm(att, hw, d, m.w["acc.wo"], d));
  return a;
}

void channel_heads(const Model& m, const Tok& s2, const int32_t* yhat, const std::vector<int>& pos,
                   int rate, int n_out, float* mu, float* sigma, Tok* final_rep) {
  const Config& c = m.c;
  const int n = static_cast<int>(pos.size()), d = c.d, sl = c.slot(), Cg = c.Cg(), hw = c.HW();
  const int dch = c.d_ch;
  if (n == 0) return;
  const Tok s2p = gather(s2, d, pos);
  Tok x(static_cast<size_t>(n) * dch, 0.0f);
  auto put_slot = [&](Tok& dst, int g, const Tok& src) {
    for (int i = 0; i < n; ++i)
      std::memcpy(dst.data() + static_cast<size_t>(i) * dch + g * sl, src.data() + static_cast<size_t>(i) * sl,
                  sizeof(float) * sl);
  };
  auto get_cols = [&](const Tok& src, int c0, int width) {
    Tok out(static_cast<size_t>(n) * width);
    for (int i = 0; i < n; ++i)
      std::memcpy(out.data() + static_cast<size_t>(i) * width, src.data() + static_cast<size_t>(i) * dch + c0,
                  sizeof(float) * width);
    return out;
  };
  for (int g = 0; g < n_out; ++g) {
    Tok xs = mm(s2p, n, d, m.w["ch.proj" + std::to_string(g) + ".w"], sl);
    if (g >= 1) {  // channel shift: slot g sees y_hat group g-1
      Tok yg(static_cast<size_t>(n) * Cg);
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < Cg; ++j)
          yg[static_cast<size_t>(i) * Cg + j] =
              static_cast<float>(yhat[static_cast<size_t>((g - 1) * Cg + j) * hw + pos[i]]);
      add_into(xs, mm(yg, n, Cg, m.w["ch.emb" + std::to_string(g) + ".w"], sl));
    }
    put_slot(x, g, xs);
  }
  const int act = n_out * sl;  // live width: slots >= n_out never read
  for (int b = 0; b < c.ch_blocks; ++b) {
    const std::string P = "ch.b" + std::to_string(b);
    const Tok xn = norm_rows(x, n, dch, m.w[P + ".norm1.g"], sl);
    const float* wm = m.w[P + ".mix.w"];
    for (int g = 0; g < n_out; ++g) {
      // masked mixing: output slot g reads input slots <= g only
      const int kin = (g + 1) * sl;
      std::vector<float> wsub(static_cast<size_t>(kin) * sl);
      for (int k = 0; k < kin; ++k)
        std::memcpy(wsub.data() + static_cast<size_t>(k) * sl, wm + static_cast<size_t>(k) * dch + g * sl,
                    sizeof(float) * sl);
      const Tok xin = get_cols(xn, 0, kin);
      const Tok mg = mm(xin, n, kin, wsub.data(), sl);
      Tok xs = get_cols(x, g * sl, sl);
      add_into(xs, mg);
      put_slot(x, g, xs);
    }
    const Tok xn2 = norm_rows(x, n, dch, m.w[P + ".norm2.g"], sl);
    for (int g = 0; g < n_out; ++g) {
      const std::string F = P + ".ffn" + std::to_string(g);
      const Tok xg = get_cols(xn2, g * sl, sl);
      Tok xs = get_cols(x, g * sl, sl);
      add_into(xs, swiglu_rows(xg, n, sl, c.fg(), m.w[F + ".wg"], m.w[F + ".wu"], m.w[F + ".wd"]));
      put_slot(x, g, xs);
    }
  }
  (void)act;
  const Tok fo = norm_rows(x, n, dch, m.w["ch.norm_out.g"], sl);
  if (final_rep) *final_rep = fo;
  const float* rso = m.w["rate.out"] + static_cast<size_t>(rate) * c.C;
  for (int g = 0; g < n_out; ++g) {
    const Tok fg = get_cols(fo, g * sl, sl);
    for (int which = 0; which < 2; ++which) {
      const std::string P = std::string("head.") + (which ? "sg" : "mu") + std::to_string(g);
      Tok h1 = mm(fg, n, sl, m.w[P + ".w1"], sl);
      const float* b1 = m.w[P + ".b1"];
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < sl; ++j) {
          float& v = h1[static_cast<size_t>(i) * sl + j];
          v = det::silu_f32(v + b1[j]);
        }
      const Tok o = mm(h1, n, sl, m.w[P + ".w2"], Cg);
      const float* b2 = m.w[P + ".b2"];
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < Cg; ++j) {
          const float v = o[static_cast<size_t>(i) * Cg + j] + b2[j];
          const int ch = g * Cg + j;
          if (which == 0)
            mu[static_cast<size_t>(i) * c.C + ch] = v * rso[ch];
          else
            sigma[static_cast<size_t>(i) * c.C + ch] = 0.11f + det::softplus_f32(v);
        }
    }
  }
}

Forward forward(const Model& m, const int32_t* yhat, const int32_t* zhat_or_null, int rate,
                const std::vector<const int32_t*>& past) {
  const Config& c = m.c;
  const int hw = c.HW();
  Forward f;
  std::vector<Tok> past_emb;
  std::vector<const float*> slots(static_cast<size_t>(c.T), nullptr);
  const int np = static_cast<int>(past.size());
  for (int i = 0; i < c.T; ++i) {
    const int k = np - c.T + i;
    if (k >= 0) past_emb.push_back(embed(m, past[k], rate));
  }
  for (int i = 0, e = 0; i < c.T; ++i)
    if (np - c.T + i >= 0) slots[i] = past_emb[e++].data();
  f.ctx = context_forward(m, slots);
  f.s1 = spatial_forward(m, "s1", c.s1_blocks, embed(m, yhat, rate), f.ctx);
  f.zhat = zhat_or_null
               ? std::vector<int32_t>(zhat_or_null, zhat_or_null + c.zcount())
               : hyper_encode(m, f.s1);
  f.hq = hyper_decode(m, f.zhat.data(), rate);
  f.a = accumulate(m, f.hq, f.s1);
  f.s2 = spatial_forward(m, "s2", c.s2_blocks, f.a, f.ctx);
  std::vector<float> mu_t(static_cast<size_t>(hw) * c.C), sg_t(mu_t.size());
  channel_heads(m, f.s2, yhat, iota(hw), rate, c.N, mu_t.data(), sg_t.data(), &f.final_rep);
  f.mu = tok_to_chw(mu_t, c.C, hw);
  f.sigma = tok_to_chw(sg_t, c.C, hw);
  if (c.lrp_blocks > 0) f.eps = lrp_forward(m, f.final_rep, yhat, slots);
  return f;
}

std::vector<float> lrp_forward(const Model& m, const Tok& final_rep, const int32_t* yhat,
                               const std::vector<const float*>& slots) {
  const Config& c = m.c;
  const int hw = c.HW(), d = c.d, T = c.T, S = T + 1, dch = c.d_ch, kin = dch + c.C;
  // current slot: in_proj(concat(final_rep, y_hat)) + bias
  Tok cat(static_cast<size_t>(hw) * kin);
  for (int p = 0; p < hw; ++p) {
    std::memcpy(cat.data() + static_cast<size_t>(p) * kin, final_rep.data() + static_cast<size_t>(p) * dch,
                sizeof(float) * dch);
    for (int ch = 0; ch < c.C; ++ch)
      cat[static_cast<size_t>(p) * kin + dch + ch] = static_cast<float>(yhat[static_cast<size_t>(ch) * hw + p]);
  }
  Tok cur = mm(cat, hw, kin, m.w["lrp.in.w"], d);
  const float* bin = m.w["lrp.in.b"];
  for (int p = 0; p < hw; ++p)
    for (int j = 0; j < d; ++j) cur[static_cast<size_t>(p) * d + j] += bin[j];
  // slots 0..T-1: the context transformer's inputs; slot T: the current frame
  Tok x(static_cast<size_t>(S) * hw * d);
  const float* pad = m.w["pad"];
  for (int t = 0; t < T; ++t)
    for (int p = 0; p < hw; ++p)
      std::memcpy(x.data() + (static_cast<size_t>(t) * hw + p) * d,
                  slots[t] ? slots[t] + static_cast<size_t>(p) * d : pad, sizeof(float) * d);
  std::memcpy(x.data() + static_cast<size_t>(T) * hw * d, cur.data(), cur.size() * sizeof(float));
  std::vector<int> all_pos;
  for (int t = 0; t < S; ++t)
    for (int p = 0; p < hw; ++p) all_pos.push_back(p);
  for (int b = 0; b < c.lrp_blocks; ++b) {
    const std::string P = "lrp.b" + std::to_string(b);
    const bool last = b == c.lrp_blocks - 1;
    const int n = S * hw;
    const Tok xn = norm_rows(x, n, d, m.w[P + ".norm1.g"], d);
    const Tok K = mm(xn, n, d, m.w[P + ".wk"], d);
    const Tok V = mm(xn, n, d, m.w[P + ".wv"], d);
    const int q0 = last ? T * hw : 0;  // last block: the current slot's queries only
    const int nq = n - q0;
    Tok xq(xn.begin() + static_cast<size_t>(q0) * d, xn.end());
    const Tok Q = mm(xq, nq, d, m.w[P + ".wq"], d);
    std::vector<int> qpos(all_pos.begin() + q0, all_pos.end()), qslot(static_cast<size_t>(nq));
    for (int i = 0; i < nq; ++i) qslot[i] = (q0 + i) / hw;
    Tok att(static_cast<size_t>(nq) * d);
    window_attention(c, nq, Q.data(), qpos.data(), qslot.data(), K.data(), V.data(), 1, kNone,
                     m.w[P + ".pos"], att.data());
    const Tok o = mm(att, nq, d, m.w[P + ".wo"], d);
    Tok xs(x.begin() + static_cast<size_t>(q0) * d, x.end());
    add_into(xs, o);
    const Tok xn2 = norm_rows(xs, nq, d, m.w[P + ".norm2.g"], d);
    add_into(xs, swiglu_rows(xn2, nq, d, c.f(), m.w[P + ".ffn.wg"], m.w[P + ".ffn.wu"],
                             m.w[P + ".ffn.wd"]));
    std::memcpy(x.data() + static_cast<size_t>(q0) * d, xs.data(), xs.size() * sizeof(float));
  }
  Tok xc(x.begin() + static_cast<size_t>(T) * hw * d, x.end());
  const Tok xo = norm_rows(xc, hw, d, m.w["lrp.norm_out.g"], d);
  Tok e = mm(xo, hw, d, m.w["lrp.head.w"], c.C);
  const float* hb = m.w["lrp.head.b"];
  for (int p = 0; p < hw; ++p)
    for (int ch = 0; ch < c.C; ++ch) {
      float& v = e[static_cast<size_t>(p) * c.C + ch];
      v = 0.5f * det::tanh_f32(v + hb[ch]);
    }
  return tok_to_chw(e, c.C, hw);
}

}  // namespace oracle
