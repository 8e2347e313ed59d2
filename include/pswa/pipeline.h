// pswa/pipeline.h — C++ host API over the C ABI (header-only).
//
// The reference declares its codec pipeline in pipeline.h (missing from the
// shipped tree; proj/CMakeLists.txt:29 lists src/pipeline.cpp) with the SPEC
// signatures
//   encode_frame(y, state, weights, cfg, rate_idx) -> (payloads, ŷ, ε, BitStats)
//                                                                SPEC.md:567-575
//   decode_frame_wavefront(payloads, state, weights, cfg, workers) -> (ŷ, ε)
//                                                                SPEC.md:585-593
// Here `state` (the FrameState ring) and `weights` live on
// the device inside a handle; `workers` has no meaning on the device and the
// result is independent of it, as SPEC.md:593 requires. ε is the LRP output
// (all zero when the handle has no LRP transformer). Errors
// are rethrown as the reference does: std::invalid_argument for shape /
// argument errors (tensor.h:63 convention), std::runtime_error for stream /
// CUDA errors.
#ifndef PSWA_PIPELINE_H_
#define PSWA_PIPELINE_H_

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "pswa/pswa_cuda.h"

namespace pswa {

struct Payloads {
  std::vector<uint8_t> hyper;  // z-hat lanes (decoded first)
  std::vector<uint8_t> main;   // y-hat lanes
};

struct FrameBits {
  double hyper = 0.0, main = 0.0;  // estimate_bits
};

// BitStats: per-position, per-group estimated bits
// [N][H][W] (group g of position (y, x) at g*H*W + y*W + x) and the frame
// totals {hyper, main}; the per-position entries sum to `main`.
struct BitStats {
  int n_groups = 0, height = 0, width = 0;
  std::vector<double> per_position_group;
  FrameBits totals;
  double at(int g, int y, int x) const {
    return per_position_group[(static_cast<size_t>(g) * height + y) * width + x];
  }
};

inline void throw_on(int rc) {
  if (rc == PSWA_OK) return;
  const std::string msg = pswa_gpu_last_error();
  if (rc == PSWA_E_ARG || rc == PSWA_E_HASH) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

// One device-resident codec state machine (one stream). Encoder and decoder
// sides keep their own temporal rings; handles on different devices run
// concurrently (GOP sharding).
class GpuCodec {
 public:
  GpuCodec(int device, const pswa_cfg& cfg, const std::vector<uint8_t>& psww) : cfg_(cfg) {
    throw_on(pswa_gpu_create(device, &cfg_, psww.data(), psww.size(), &h_));
  }
  ~GpuCodec() { pswa_gpu_destroy(h_); }
  GpuCodec(const GpuCodec&) = delete;
  GpuCodec& operator=(const GpuCodec&) = delete;

  const pswa_cfg& cfg() const { return cfg_; }
  pswa_gpu* handle() { return h_; }
  size_t latent_count() const {
    return static_cast<size_t>(cfg_.latent_ch) * cfg_.height * cfg_.width;
  }
  void reset_gop() { throw_on(pswa_gpu_reset_gop(h_)); }
  // BitStats for every later frame call (off by default: the taps cost one
  // 8-byte store per symbol and a reduction per frame).
  void set_stats(bool on) { throw_on(pswa_gpu_set_stats(h_, on ? 1 : 0)); }
  BitStats last_bitstats(const FrameBits& totals) {
    BitStats s;
    s.n_groups = cfg_.n_groups;
    s.height = cfg_.height;
    s.width = cfg_.width;
    s.per_position_group.resize(static_cast<size_t>(s.n_groups) * s.height * s.width);
    throw_on(pswa_gpu_last_bitstats(h_, s.per_position_group.data()));
    s.totals = totals;
    return s;
  }
  std::vector<float> last_eps() {
    std::vector<float> e(latent_count(), 0.0f);
    if (cfg_.lrp_blocks > 0) throw_on(pswa_gpu_last_eps(h_, e.data()));
    return e;
  }

 private:
  pswa_cfg cfg_;
  pswa_gpu* h_ = nullptr;
};

struct EncodedFrame {
  Payloads payloads;
  std::vector<int32_t> yhat;  // the quantised latents coded (== the input)
  std::vector<float> eps;     // LRP output for the reconstruction ŷ + ε
  BitStats stats;             // per-position bits when the codec has stats on
};

struct DecodedFrame {
  std::vector<int32_t> yhat;  // [C][H][W], bit-exact to the encoder's
  std::vector<float> eps;     // [C][H][W]
  FrameBits bits;
};

// encode_frame: y_hat [C][H][W] -> payloads; advances the
// encoder's temporal ring. `stats` is filled when enc.set_stats(true).
inline EncodedFrame encode_frame(GpuCodec& enc, const std::vector<int32_t>& yhat, int rate_idx,
                                 int frame_idx_in_gop, bool with_stats = false) {
  if (yhat.size() != enc.latent_count()) throw std::invalid_argument("encode_frame: y_hat shape");
  const size_t cap = 20 * yhat.size() + (1u << 20);
  EncodedFrame out;
  Payloads& p = out.payloads;
  p.hyper.resize(cap);
  p.main.resize(cap);
  size_t hl = 0, ml = 0;
  double b[2] = {0, 0};
  if (with_stats) enc.set_stats(true);
  throw_on(pswa_gpu_encode_frame(enc.handle(), yhat.data(), rate_idx, frame_idx_in_gop,
                                 p.hyper.data(), cap, &hl, p.main.data(), cap, &ml, b));
  p.hyper.resize(hl);
  p.main.resize(ml);
  out.yhat = yhat;
  out.eps = enc.last_eps();
  if (with_stats) out.stats = enc.last_bitstats({b[0], b[1]});
  else out.stats.totals = {b[0], b[1]};
  return out;
}

// decode_frame_wavefront: s*N phases on the device, y_hat
// [C][H][W] bit-exact to the encoder's, and ε; advances the decoder's ring.
inline DecodedFrame decode_frame_wavefront(GpuCodec& dec, const Payloads& p, int rate_idx,
                                           int frame_idx_in_gop, int /*workers*/ = 1) {
  DecodedFrame out;
  out.yhat.resize(dec.latent_count());
  double b[2] = {0, 0};
  throw_on(pswa_gpu_decode_frame(dec.handle(), p.hyper.data(), p.hyper.size(), p.main.data(),
                                 p.main.size(), rate_idx, frame_idx_in_gop, 1, out.yhat.data(),
                                 nullptr, nullptr, b));
  out.bits = {b[0], b[1]};
  out.eps = dec.last_eps();
  return out;
}

}  // namespace pswa

#endif  // PSWA_PIPELINE_H_
