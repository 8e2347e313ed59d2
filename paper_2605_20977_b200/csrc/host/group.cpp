// BandGroup: segment orchestration of banded frames (see group.h).
#include "group.h"

#include <cstdlib>
#include <cstring>
#include <stdexcept>

#include "../cuda/check.h"
#include "abi_util.h"

namespace pswa_host {

std::vector<uint8_t> pack_banded(const std::vector<std::vector<uint8_t>>& bands) {
  std::vector<uint8_t> out = {'P', 'S', 'W', 'B'};
  auto put = [&](uint64_t v, int bytes) {
    for (int i = 0; i < bytes; ++i) out.push_back(static_cast<uint8_t>(v >> (8 * i)));
  };
  put(bands.size(), 4);
  for (const auto& b : bands) put(b.size(), 8);
  for (const auto& b : bands) out.insert(out.end(), b.begin(), b.end());
  return out;
}

std::vector<std::pair<size_t, size_t>> parse_banded(const uint8_t* p, size_t len, int n) {
  const size_t hdr = 8 + 8 * static_cast<size_t>(n);
  if (len < hdr || std::memcmp(p, "PSWB", 4) != 0)
    throw pswa_abi::TruncatedError("banded payload: bad header");
  uint32_t nb = 0;
  std::memcpy(&nb, p + 4, 4);
  if (static_cast<int>(nb) != n) throw std::invalid_argument("banded payload: band count differs from the group");
  std::vector<std::pair<size_t, size_t>> r;
  size_t off = hdr;
  for (int b = 0; b < n; ++b) {
    uint64_t l = 0;
    std::memcpy(&l, p + 8 + 8 * b, 8);
    if (l > len - off) throw pswa_abi::TruncatedError("banded payload: truncated band");
    r.emplace_back(off, static_cast<size_t>(l));
    off += l;
  }
  return r;
}

BandGroup::BandGroup(const std::vector<int>& devices, const pswa_cfg& cfg, const void* blob,
                     size_t len) {
  const int n = static_cast<int>(devices.size());
  if (n < 1) throw std::invalid_argument("BandGroup: no devices");
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      // neighbours push halos; every band writes its S1 rows to band 0 (encoder)
      if (i == j || devices[i] == devices[j]) continue;
      int ok = 0;
      PSWA_CUDA(cudaDeviceCanAccessPeer(&ok, devices[i], devices[j]));
      if (!ok) throw std::invalid_argument("BandGroup: no peer access between the band devices");
      PSWA_CUDA(cudaSetDevice(devices[i]));
      const cudaError_t e = cudaDeviceEnablePeerAccess(devices[j], 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else PSWA_CUDA(e);
    }
  for (int b = 0; b < n; ++b)
    bands_.push_back(std::make_unique<Engine>(devices[b], cfg, blob, len, b, n));
  for (int b = 0; b < n; ++b) {
    PSWA_CUDA(cudaSetDevice(devices[b]));
    if (n > 1)
      bands_[b]->link(b > 0 ? bands_[b - 1].get() : nullptr, b + 1 < n ? bands_[b + 1].get() : nullptr,
                      bands_[0].get());
    std::array<cudaEvent_t, 2> e{};
    for (auto& x : e) PSWA_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
    ev_.push_back(e);
  }
}

BandGroup::~BandGroup() {
  for (size_t b = 0; b < ev_.size(); ++b) {
    cudaSetDevice(bands_[b]->device());
    for (auto x : ev_[b]) cudaEventDestroy(x);
  }
}

// Segment k of band b waits for segment k-1 of its neighbours (of every band
// after a global cut). Two events per band alternate by segment parity, so a
// wait enqueued in round k always sees the neighbour's round k-1 record.
void BandGroup::run(const std::string& key) {
  const int n = size();
  std::vector<Program*> P(n);
  for (int b = 0; b < n; ++b) {
    // building a program allocates tables and launches on the band's stream
    PSWA_CUDA(cudaSetDevice(bands_[b]->device()));
    P[b] = &bands_[b]->program(key);
  }
  const int S = bands_[0]->segments(*P[0]);
  last_launches_ = 0;
  for (int b = 0; b < n; ++b) {
    if (bands_[b]->segments(*P[b]) != S) throw std::logic_error("band programs differ in segments");
    last_launches_ += P[b]->launches;
  }
  for (int k = 0; k < S; ++k)
    for (int b = 0; b < n; ++b) {
      Engine& e = *bands_[b];
      PSWA_CUDA(cudaSetDevice(e.device()));
      if (k > 0) {
        const bool global = e.cut_global(*P[b], k - 1);
        for (int o = 0; o < n; ++o)
          if (o != b && (global || std::abs(o - b) == 1))
            PSWA_CUDA(cudaStreamWaitEvent(e.stream(), ev_[o][(k - 1) & 1], 0));
      }
      e.launch_segment(*P[b], k);
      PSWA_CUDA(cudaEventRecord(ev_[b][k & 1], e.stream()));
    }
}

void BandGroup::reset_gop() {  // host-side ring indices only
  for (auto& e : bands_) e->reset_gop();
}

void BandGroup::push_frame(const int32_t* yhat, int rate) {
  for (auto& e : bands_) {
    PSWA_CUDA(cudaSetDevice(e->device()));
    e->push_frame(yhat, rate);
  }
}

FrameResult BandGroup::encode(const int32_t* yhat, int rate, int fidx, const int32_t* zhat_in,
                              float* mu_out, float* sigma_out, uint8_t* hyper_out, size_t hyper_cap,
                              uint8_t* main_out, size_t main_cap, bool advance) {
  const int n = size();
  for (auto& e : bands_) {
    PSWA_CUDA(cudaSetDevice(e->device()));
    e->prep_encode(yhat, rate, fidx, zhat_in);
    e->set_want_musig(mu_out != nullptr);
  }
  run(bands_[0]->encode_key(zhat_in != nullptr, mu_out != nullptr));
  FrameResult r;
  std::vector<std::vector<uint8_t>> mains(n);
  for (int b = 0; b < n; ++b) {
    Engine& e = *bands_[b];
    PSWA_CUDA(cudaSetDevice(e.device()));
    const FrameResult rb = e.finish_encode(mu_out, sigma_out, nullptr, 0, nullptr, 0, advance);
    mains[b].resize(rb.main_len);
    e.fetch_payloads(b == 0 ? hyper_out : nullptr, b == 0 ? hyper_cap : 0, rb, mains[b].data());
    if (b == 0) {
      r.hyper_len = rb.hyper_len;
      r.bits[0] = rb.bits[0];
    }
    r.bits[1] += rb.bits[1];
  }
  const auto packed = pack_banded(mains);
  r.main_len = packed.size();
  if (main_out) {
    if (main_cap < packed.size()) throw std::invalid_argument("main output buffer too small");
    std::memcpy(main_out, packed.data(), packed.size());
  }
  return r;
}

FrameResult BandGroup::decode(const uint8_t* hyper, size_t hyper_len, const uint8_t* main_pl,
                              size_t main_len, int rate, int fidx, bool advance, int32_t* yhat_out) {
  const int n = size();
  const auto parts = parse_banded(main_pl, main_len, n);
  for (int b = 0; b < n; ++b) {
    Engine& e = *bands_[b];
    PSWA_CUDA(cudaSetDevice(e.device()));
    e.prep_decode(hyper, hyper_len, main_pl + parts[b].first, parts[b].second, rate, fidx, false);
  }
  run("decode");
  FrameResult r;
  for (int b = 0; b < n; ++b) {
    Engine& e = *bands_[b];
    PSWA_CUDA(cudaSetDevice(e.device()));
    const FrameResult rb = e.finish_decode(advance, yhat_out, false);
    if (b == 0) r.bits[0] = rb.bits[0];
    r.bits[1] += rb.bits[1];
  }
  return r;
}

}  // namespace pswa_host
