// ORACLE — test infrastructure only.
// Codec pipeline: teacher-forced encoder, the SPEC-literal
// wavefront decoder (S1/A/S2 recomputed over the frame each step)
// and the serial reference decoder (one (position, group) per recompute).
#include <cmath>
#include <stdexcept>

#include "oracle/model.h"

namespace oracle {

namespace {
int32_t rint_i(float v) { return static_cast<int32_t>(std::nearbyint(v)); }

const float* prior(const Model& m, const char* what, int rate, int fidx) {
  const int slot = fidx < 4 ? fidx : 4;  // select_prior
  return m.w[std::string("hyper.") + what] + (static_cast<size_t>(rate) * 5 + slot) * m.c.hyper_ch;
}

std::vector<int32_t> decode_hyper(const Model& m, const std::vector<uint8_t>& pl, int rate,
                                  int fidx, double* bits, bool* ok) {
  const Config& c = m.c;
  const int n = c.zcount(), per = c.zper();
  std::vector<int32_t> z(static_cast<size_t>(n));
  LaneDecoder dec;
  if (!dec.init(pl.data(), pl.size()) || dec.count != static_cast<uint32_t>(n)) {
    *ok = false;
    return z;
  }
  const float* loc = prior(m, "loc", rate, fidx);
  const float* sc = prior(m, "scale", rate, fidx);
  for (int i = 0; i < n; ++i) {
    const int ch = i / per;
    const int idx = scale_index(sc[ch]);
    const int32_t v = dec.decode(static_cast<uint64_t>(i), idx);
    z[i] = v + rint_i(loc[ch]);
    *bits += bits_of({v, idx});
  }
  if (dec.error) *ok = false;
  return z;
}
}  // namespace

std::vector<CodedSym> main_symbols(const Model& m, const int32_t* yhat, const float* mu,
                                   const float* sigma) {
  const Config& c = m.c;
  const int hw = c.HW(), Cg = c.Cg();
  std::vector<CodedSym> out;
  out.reserve(static_cast<size_t>(hw) * c.C);
  for (int t = 0; t < c.s; ++t) {
    const std::vector<int> pos = positions_of_step(c.H, c.W, c.s, t);
    for (int g = 0; g < c.N; ++g)
      for (int p : pos)
        for (int j = 0; j < Cg; ++j) {
          const size_t e = static_cast<size_t>(g * Cg + j) * hw + p;
          out.push_back({yhat[e] - rint_i(mu[e]), main_index(c, sigma[e])});
        }
  }
  return out;
}

std::vector<CodedSym> hyper_symbols(const Model& m, const int32_t* zhat, int rate, int fidx) {
  const Config& c = m.c;
  const int per = c.zper(), n = c.zcount();
  const float* loc = prior(m, "loc", rate, fidx);
  const float* sc = prior(m, "scale", rate, fidx);
  std::vector<CodedSym> out(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) out[i] = {zhat[i] - rint_i(loc[i / per]), scale_index(sc[i / per])};
  return out;
}

Payload encode_frame(const Model& m, const int32_t* yhat, int rate, int fidx,
                     const std::vector<const int32_t*>& past, const int32_t* zhat_override) {
  Forward f = forward(m, yhat, zhat_override, rate, past);
  Payload pl;
  pl.zhat = f.zhat;
  const auto hs = hyper_symbols(m, f.zhat.data(), rate, fidx);
  const auto ms = main_symbols(m, yhat, f.mu.data(), f.sigma.data());
  for (const auto& s : hs) pl.hyper_bits += bits_of(s);
  for (const auto& s : ms) pl.main_bits += bits_of(s);
  pl.hyper = encode_lanes(hs, m.c.hyper_lanes);
  pl.main = encode_lanes(ms, m.c.lanes);
  return pl;
}

namespace {
struct DecodeCommon {
  const Model& m;
  int rate;
  Tok ctx, hq;
  std::vector<const float*> slots;
  std::vector<Tok> past_emb;
  DecodeCommon(const Model& mm, int r, const std::vector<const int32_t*>& past, const int32_t* z)
      : m(mm), rate(r) {
    const Config& c = m.c;
    const int np = static_cast<int>(past.size());
    slots.assign(static_cast<size_t>(c.T), nullptr);
    for (int i = 0; i < c.T; ++i)
      if (np - c.T + i >= 0) past_emb.push_back(embed(m, past[np - c.T + i], rate));
    for (int i = 0, e = 0; i < c.T; ++i)
      if (np - c.T + i >= 0) slots[i] = past_emb[e++].data();
    ctx = context_forward(m, slots);
    hq = hyper_decode(m, z, rate);
  }
  // S1 -> accumulator -> S2 over the whole frame from the partial y_hat.
  Tok s2_from(const std::vector<int32_t>& yhat) const {
    const Tok s1 = spatial_forward(m, "s1", m.c.s1_blocks, embed(m, yhat.data(), rate), ctx);
    return spatial_forward(m, "s2", m.c.s2_blocks, accumulate(m, hq, s1), ctx);
  }
};
}  // namespace

Decoded decode_wavefront(const Model& m, const Payload& pl, int rate, int fidx,
                         const std::vector<const int32_t*>& past) {
  const Config& c = m.c;
  const int hw = c.HW(), Cg = c.Cg();
  Decoded out;
  const std::vector<int32_t> z = decode_hyper(m, pl.hyper, rate, fidx, &out.hyper_bits, &out.ok);
  if (!out.ok) return out;
  DecodeCommon dc(m, rate, past, z.data());
  LaneDecoder dec;
  if (!dec.init(pl.main.data(), pl.main.size()) ||
      dec.count != static_cast<uint32_t>(hw * c.C)) {
    out.ok = false;
    return out;
  }
  out.yhat.assign(static_cast<size_t>(hw) * c.C, 0);  // undecoded placeholder = 0
  uint64_t ordinal = 0;
  for (int t = 0; t < c.s; ++t) {
    const std::vector<int> pos = positions_of_step(c.H, c.W, c.s, t);
    const Tok s2 = dc.s2_from(out.yhat);
    std::vector<float> mu(pos.size() * c.C), sg(mu.size());
    for (int g = 0; g < c.N; ++g) {
      channel_heads(m, s2, out.yhat.data(), pos, rate, g + 1, mu.data(), sg.data());
      for (size_t k = 0; k < pos.size(); ++k)
        for (int j = 0; j < Cg; ++j) {
          const int ch = g * Cg + j;
          const float mv = mu[k * c.C + ch];
          const int idx = main_index(c, sg[k * c.C + ch]);
          const int32_t v = dec.decode(ordinal++, idx);
          out.yhat[static_cast<size_t>(ch) * hw + pos[k]] = v + rint_i(mv);
          out.main_bits += bits_of({v, idx});
        }
      ++out.phases;
    }
  }
  if (dec.error) out.ok = false;
  return out;
}

Decoded decode_serial(const Model& m, const Payload& pl, int rate, int fidx,
                      const std::vector<const int32_t*>& past) {
  const Config& c = m.c;
  const int hw = c.HW(), Cg = c.Cg();
  Decoded out;
  const std::vector<int32_t> z = decode_hyper(m, pl.hyper, rate, fidx, &out.hyper_bits, &out.ok);
  if (!out.ok) return out;
  DecodeCommon dc(m, rate, past, z.data());
  LaneDecoder dec;
  if (!dec.init(pl.main.data(), pl.main.size()) ||
      dec.count != static_cast<uint32_t>(hw * c.C)) {
    out.ok = false;
    return out;
  }
  out.yhat.assign(static_cast<size_t>(hw) * c.C, 0);
  uint64_t ordinal = 0;
  float mu[1024], sg[1024];
  for (int t = 0; t < c.s; ++t) {
    const std::vector<int> pos = positions_of_step(c.H, c.W, c.s, t);
    for (int g = 0; g < c.N; ++g)
      for (int p : pos) {
        // one (position, group) per full recompute of the network
        const Tok s2 = dc.s2_from(out.yhat);
        channel_heads(m, s2, out.yhat.data(), {p}, rate, g + 1, mu, sg);
        for (int j = 0; j < Cg; ++j) {
          const int ch = g * Cg + j;
          const int idx = main_index(c, sg[ch]);
          const int32_t v = dec.decode(ordinal++, idx);
          out.yhat[static_cast<size_t>(ch) * hw + p] = v + rint_i(mu[ch]);
          out.main_bits += bits_of({v, idx});
        }
        ++out.phases;
      }
  }
  if (dec.error) out.ok = false;
  return out;
}

}  // namespace oracle
