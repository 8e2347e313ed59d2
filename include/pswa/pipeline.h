// pswa/pipeline.h — C++ host API over the C ABI (header-only).
//
// The reference declares its codec pipeline in pipeline.h (missing from the
// shipped tree; proj/CMakeLists.txt:29 lists src/pipeline.cpp) with the SPEC
// signatures
//   encode_frame(y, state, weights, cfg, rate_idx)
//   decode_frame_wavefront(payloads, state, weights, cfg, workers) SPEC.md:585-593
// Here `state` (the FrameState ring) and `weights` live on
// the device inside a handle; `workers` has no meaning on the device and the
// result is independent of it, as SPEC.md:593 requires. Errors are rethrown
// as the reference does: std::invalid_argument for shape/argument errors
// (tensor.h:63 convention), std::runtime_error for stream / CUDA errors.
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

 private:
  pswa_cfg cfg_;
  pswa_gpu* h_ = nullptr;
};

// encode_frame: y_hat [C][H][W] -> payloads; advances the
// encoder's temporal ring.
inline Payloads encode_frame(GpuCodec& enc, const std::vector<int32_t>& yhat, int rate_idx,
                             int frame_idx_in_gop, FrameBits* bits = nullptr) {
  if (yhat.size() != enc.latent_count()) throw std::invalid_argument("encode_frame: y_hat shape");
  const size_t cap = 20 * yhat.size() + (1u << 20);
  Payloads p;
  p.hyper.resize(cap);
  p.main.resize(cap);
  size_t hl = 0, ml = 0;
  double b[2] = {0, 0};
  throw_on(pswa_gpu_encode_frame(enc.handle(), yhat.data(), rate_idx, frame_idx_in_gop,
                                 p.hyper.data(), cap, &hl, p.main.data(), cap, &ml, b));
  p.hyper.resize(hl);
  p.main.resize(ml);
  if (bits) *bits = {b[0], b[1]};
  return p;
}

// decode_frame_wavefront: s*N phases on the device, y_hat
// [C][H][W] bit-exact to the encoder's; advances the decoder's ring.
inline std::vector<int32_t> decode_frame_wavefront(GpuCodec& dec, const Payloads& p, int rate_idx,
                                                   int frame_idx_in_gop, int /*workers*/ = 1,
                                                   FrameBits* bits = nullptr) {
  std::vector<int32_t> y(dec.latent_count());
  double b[2] = {0, 0};
  throw_on(pswa_gpu_decode_frame(dec.handle(), p.hyper.data(), p.hyper.size(), p.main.data(),
                                 p.main.size(), rate_idx, frame_idx_in_gop, 1, y.data(), b));
  if (bits) *bits = {b[0], b[1]};
  return y;
}

}  // namespace pswa

#endif  // PSWA_PIPELINE_H_
