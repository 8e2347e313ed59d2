// Model configuration, parameter inventory, PSWW weight container and the
// synthetic-input generator of the product host layer.
//
// The parameter inventory is the architecture frozen in DESIGN.md §3 (SPEC.md
// :283-429 plus the decisions the SPEC leaves open); init follows
// gen_weights / init_tensor (tensor.cpp:164-180) on
// pswa/rng.h streams keyed by parameter name.
#pragma once
#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "pswa/pswa_cuda.h"

namespace pswa_host {

struct Dims {
  pswa_cfg c;
  int d, heads, hd, f, fp;        // spatial width, FFN hidden and its 64-padded width
  int dch, N, slot, sp, fg, fgp;  // channel transformer: slot width, padded slot, FFN
  int C, Cg, Cgp;                 // latent channels, per group, padded
  int hc, hcp, kconv;             // hyper channels, padded, 9*hc padded to 64
  int H, W, HW, Hp, Wp, zh, zw, T;
  int taps2, taps3;
  explicit Dims(const pswa_cfg& cfg);
};

int ffn_hidden_dim(int d);
void validate_cfg(const pswa_cfg& c);
std::string canonical_cfg(const pswa_cfg& c);  // hashed into PSWW headers

enum class Init { kScaledNormal, kZeros, kOnes, kTwo };
struct ParamDecl {
  std::string name;
  std::vector<int> shape;
  Init init;
  int fan_in;
};
std::vector<ParamDecl> param_inventory(const pswa_cfg& c);

struct HostTensor {
  std::vector<int> shape;
  std::vector<float> v;
};
using WeightMap = std::map<std::string, HostTensor>;

std::vector<uint8_t> gen_weights_psww(const pswa_cfg& c, uint64_t seed);
// Validates magic, version, config hash, names and shapes.
WeightMap parse_psww(const pswa_cfg& c, const void* blob, size_t n);

// Synthetic latent frame: Laplace(0, b_g) per channel group,
// b_g = 8 / 2^g, drifting by Laplace(0, b_g/4) per P-frame, 1 in 10^4
// positions forced to +-300 (escape path), y_hat = round-half-even(y).
void synth_latent(const pswa_cfg& c, int gop, int frame_idx, int32_t* yhat_chw);
// frames 0..n_frames-1 of GOP `gop` in one pass: out[f][C][H][W]
void synth_gop(const pswa_cfg& c, int gop, int n_frames, int32_t* out);

}  // namespace pswa_host
