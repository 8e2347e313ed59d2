// ORACLE — test infrastructure only. Never linked into the product path.
//
// CPU restatement of the P-SWA entropy model and codec pipeline, following
// SPEC.md module by module (wavefront :114-201, swa_attention :203-281,
// entropy_model :283-429, range_coder :431-497, codec_pipeline :550-635,
// io_formats :637-662) on the numerics of numerics.h. The architecture
// decisions the SPEC leaves open are frozen in DESIGN.md §3 and implemented
// identically here and on the GPU.
#pragma once
#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "oracle/numerics.h"

namespace oracle {

// ModelConfig + grid + coder lanes.
struct Config {
  int d = 64, heads = 16, ctx_blocks = 2, s1_blocks = 2, s2_blocks = 2;
  int d_ch = 128, ch_blocks = 2, hyper_ch = 32, C = 192, s = 4, N = 4;
  int wh = 7, ww = 7, wt = 5, T = 4, rates = 4;
  int H = 16, W = 16;
  int lanes = 1, hyper_lanes = 1;
  int prior = 0;  // main-latent head: 0 Gaussian, 1 Laplace (tables offset kScales)
  int lrp_blocks = 0;  // LRP transformer blocks (0: no LRP, eps = 0)
  int hd() const { return d / heads; }
  int f() const { return ffn_hidden(d); }
  int slot() const { return d_ch / N; }
  int fg() const { return ffn_hidden(d_ch / N); }
  int Cg() const { return C / N; }
  int taps2() const { return wh * ww; }
  int taps3() const { return wt * wh * ww; }
  int HW() const { return H * W; }
  // hyperprior grid: latent padded up to multiples of 4
  int Hp() const { return (H + 3) / 4 * 4; }
  int Wp() const { return (W + 3) / 4 * 4; }
  int zper() const { return Hp() / 4 * (Wp() / 4); }
  int zcount() const { return hyper_ch * zper(); }
  std::string canonical() const;  // hashed into PSWW
};
Config preset(int paper, int H, int W);

// ---- wavefront module (wavefront.h:29-66) --------------
inline int step_of(int y, int x, int s) { return (y + x) % s; }
enum Mask { kNone = 0, kSelfLe = 1, kAccLt = 2 };
inline bool mask_allows(int mask, int q_step, int k_step) {
  if (mask == kSelfLe) return k_step <= q_step;
  if (mask == kAccLt) return k_step < q_step;
  return true;
}
std::vector<int> positions_of_step(int H, int W, int s, int t);  // raster idx
std::vector<uint8_t> channel_mask(int N, int dg);
struct Schedule {
  bool ok = true;
  int steps = 0;
  std::string violation;
};
Schedule validate_schedule(int H, int W, int s, int wh, int ww, int N);

// ---- weights (gen_weights / PSWW) ----------------------
struct Param {
  std::vector<int> shape;
  std::vector<float> v;
};
struct Weights {
  std::vector<std::string> order;
  std::map<std::string, Param> p;
  const float* operator[](const std::string& n) const;
  const Param& at(const std::string& n) const;
};
struct ParamSpec {
  std::string name;
  std::vector<int> shape;
  int kind;    // 0 scaled-normal, 1 zeros, 2 ones, 3 constant two
  int fan_in;
};
std::vector<ParamSpec> param_specs(const Config& c);
Weights gen_weights(const Config& c, uint64_t seed);
std::vector<uint8_t> to_psww(const Config& c, const Weights& w);
Weights from_psww(const Config& c, const uint8_t* data, size_t n);

// ---- range coder ---------------------------------------
constexpr int kScales = 64;
constexpr int kSupport = 127;          // v in [-127, 127]
constexpr int kSyms = 2 * kSupport + 3;  // 255 in-range + 2 escapes = 257
// Tables: [0, 64) discretised Gaussian, [64, 128) the
// Laplace family of the prior = 1 head (scale b = the table sigma).
struct Tables {
  float scale[kScales];
  uint32_t cdf[2 * kScales][kSyms + 1];  // cumulative, c[0]=0, c[257]=65536
};
const Tables& tables();
int scale_index(float sigma);  // smallest i with scale[i] >= sigma, else 63
// Table of a main-latent symbol: the sigma index in the head's family.
inline int main_index(const Config& c, float sigma) {
  return scale_index(sigma) + (c.prior ? kScales : 0);
}
void build_cdf(int idx, uint32_t* cum /* kSyms+1 */);  // idx >= kScales: Laplace

struct CodedSym {  // one latent symbol ready for the coder
  int32_t v;        // y_hat - round(mu)  (escape when |v| > 127)
  int32_t idx;      // scale-table index
};
// Multi-lane payload: symbol ordinal o goes to lane o % L.
std::vector<uint8_t> encode_lanes(const std::vector<CodedSym>& syms, int lanes);
// Decodes `count` symbols; idx_of(o) supplies the table index of ordinal o
// (in the pipeline it depends on previously decoded symbols).
struct LaneDecoder {
  struct Lane {
    uint64_t code = 0, range = (uint64_t{1} << 48) - 1;
    const uint8_t* p = nullptr;
    const uint8_t* end = nullptr;
  };
  std::vector<Lane> lanes;
  uint32_t count = 0;
  bool error = false;
  bool init(const uint8_t* data, size_t n);
  int32_t decode(uint64_t ordinal, int idx);  // returns v
};
double bits_of(const CodedSym& s);  // -log2(freq/65536) + escape bits

// ---- model -----------------------------------------------------------------
struct Model {
  Config c;
  Weights w;
  std::vector<float> mix_masked[8];  // per channel block: W_mix * channel_mask
  Model(const Config& cfg, Weights wts);
};

// token tensors are [H*W][width] row-major (raster position-major)
using Tok = std::vector<float>;

Tok embed(const Model& m, const int32_t* yhat /*C,H,W*/, int rate);
// Context transformer over T slots (nullptr slot -> learned pad); returns
// ctx = rmsnorm of the last slot's final features.
Tok context_forward(const Model& m, const std::vector<const float*>& slots);
// Spatial modules on the full frame with step masks; `prefix` = "s1" / "s2".
Tok spatial_forward(const Model& m, const std::string& prefix, int blocks, Tok x, const Tok& ctx);
std::vector<int32_t> hyper_encode(const Model& m, const Tok& s1);  // [hc][H/4][W/4]
Tok hyper_decode(const Model& m, const int32_t* zhat, int rate);
Tok accumulate(const Model& m, const Tok& hq, const Tok& s1);
// Channel transformer + heads for a set of positions. s2: [HW][d];
// yhat [C][H][W]; writes mu/sigma [npos][C] for groups < n_groups_out.
void channel_heads(const Model& m, const Tok& s2, const int32_t* yhat, const std::vector<int>& pos,
                   int rate, int n_groups_out, float* mu, float* sigma, Tok* final_rep = nullptr);

// LRP transformer (A8): eps [C][H][W] =
// 0.5 tanh(head(rmsnorm(x))) of the current slot after lrp_blocks of 3D SWA
// over T + 1 slots: the T past slots carry the context transformer's inputs
// (embedded past y_hat or the learned pad), the current slot
// in_proj(concat(final channel representation, y_hat)).
std::vector<float> lrp_forward(const Model& m, const Tok& final_rep /*[HW][d_ch]*/,
                               const int32_t* yhat, const std::vector<const float*>& slots);

// Full teacher-forced forward (encoder side): mu/sigma [C][H][W].
struct Forward {
  Tok ctx, s1, hq, a, s2;
  std::vector<int32_t> zhat;
  std::vector<float> mu, sigma;
  Tok final_rep;             // [HW][d_ch] normalised channel output (LRP input)
  std::vector<float> eps;    // [C][H][W] (empty when lrp_blocks == 0)
};
// past: up to T previous y_hat frames, oldest first (empty -> I-frame).
Forward forward(const Model& m, const int32_t* yhat, const int32_t* zhat_or_null, int rate,
                const std::vector<const int32_t*>& past);

// ---- pipeline -----------------------------------------
struct Payload {
  std::vector<uint8_t> hyper, main;
  double hyper_bits = 0, main_bits = 0;
  std::vector<int32_t> zhat;
};
Payload encode_frame(const Model& m, const int32_t* yhat, int rate, int frame_idx_in_gop,
                     const std::vector<const int32_t*>& past,
                     const int32_t* zhat_override = nullptr);
struct Decoded {
  std::vector<int32_t> yhat;
  double hyper_bits = 0, main_bits = 0;
  int phases = 0;
  bool ok = true;
};
Decoded decode_wavefront(const Model& m, const Payload& pl, int rate, int frame_idx_in_gop,
                         const std::vector<const int32_t*>& past);
Decoded decode_serial(const Model& m, const Payload& pl, int rate, int frame_idx_in_gop,
                      const std::vector<const int32_t*>& past);

// symbols of the main payload in canonical order, from a known frame
std::vector<CodedSym> main_symbols(const Model& m, const int32_t* yhat, const float* mu,
                                   const float* sigma);
std::vector<CodedSym> hyper_symbols(const Model& m, const int32_t* zhat, int rate,
                                    int frame_idx_in_gop);

}  // namespace oracle
