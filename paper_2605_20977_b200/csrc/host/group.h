// BandGroup: one frame decoded as N row bands (BASELINE config
// 5), one Engine per band, on N devices or stacked on one device.
//
// Every band runs the same per-frame program, split into segments at halo
// exchanges: a segment ends with the band pushing the K/V rows its
// neighbours need straight into their caches (halo_push, P2P stores when the
// neighbour is on another GPU). Segment k of band b starts once segment k-1
// of both neighbours has completed (CUDA events, no host round trip), so the
// bands advance in a wavefront of their own and the result is bitwise the
// single-GPU decode: every kernel sees the same inputs at the same tile
// anchors.
#pragma once
#include <array>
#include <memory>
#include <vector>

#include "engine.h"

namespace pswa_host {

// Banded main payload: "PSWB" | u32 n | u64 len[n] | band payloads (lane format)
std::vector<uint8_t> pack_banded(const std::vector<std::vector<uint8_t>>& bands);
// Returns (offset, length) of each band payload; throws TruncatedError.
std::vector<std::pair<size_t, size_t>> parse_banded(const uint8_t* p, size_t len, int n);

class BandGroup {
 public:
  BandGroup(const std::vector<int>& devices, const pswa_cfg& cfg, const void* blob, size_t len);
  ~BandGroup();
  BandGroup(const BandGroup&) = delete;
  BandGroup& operator=(const BandGroup&) = delete;

  int size() const { return static_cast<int>(bands_.size()); }
  Engine& band(int b) { return *bands_[b]; }
  int last_launches() const { return last_launches_; }

  void reset_gop();
  void push_frame(const int32_t* yhat, int rate);
  // Full-frame host buffers ([C][H][W]); main_out receives the banded container.
  FrameResult encode(const int32_t* yhat, int rate, int fidx, const int32_t* zhat_in, float* mu_out,
                     float* sigma_out, uint8_t* hyper_out, size_t hyper_cap, uint8_t* main_out,
                     size_t main_cap, bool advance);
  FrameResult decode(const uint8_t* hyper, size_t hyper_len, const uint8_t* main_pl, size_t main_len,
                     int rate, int fidx, bool advance, int32_t* yhat_out);

 private:
  void run(const std::string& key);
  std::vector<std::unique_ptr<Engine>> bands_;
  std::vector<std::array<cudaEvent_t, 2>> ev_;
  int last_launches_ = 0;
};

}  // namespace pswa_host
