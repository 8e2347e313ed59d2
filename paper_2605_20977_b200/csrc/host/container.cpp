// Sequence container reader / writer (see container.h, FORMAT.md).
#include "container.h"

#include <string>

#include <cstring>
#include <stdexcept>

#include "abi_util.h"
#include "model_spec.h"
#include "pswa/rng.h"

namespace pswa_host {

namespace {
void put(std::vector<uint8_t>& o, uint64_t v, int bytes) {
  for (int i = 0; i < bytes; ++i) o.push_back(static_cast<uint8_t>(v >> (8 * i)));
}
uint64_t get(const uint8_t* p, int bytes) {
  uint64_t v = 0;
  for (int i = 0; i < bytes; ++i) v |= static_cast<uint64_t>(p[i]) << (8 * i);
  return v;
}
}  // namespace

uint64_t stream_cfg_hash(const pswa_cfg& c, int n_bands) {
  const std::string s = canonical_cfg(c) + ";H=" + std::to_string(c.height) + ";W=" +
                        std::to_string(c.width) + ";L=" + std::to_string(c.lanes) + ";Lz=" +
                        std::to_string(c.hyper_lanes) + ";prior=" + std::to_string(c.prior) +
                        ";bands=" + std::to_string(n_bands);
  return pswa::fnv1a64(s);
}

void write_header(std::vector<uint8_t>& o, const ContainerHeader& h) {
  o.insert(o.end(), {'P', 'S', 'W', 'A'});
  put(o, kContainerVersion, 2);
  put(o, kContainerHeader, 2);
  for (uint32_t v : {h.w_px, h.h_px, h.frames, h.gop, h.rate, h.s, h.N}) put(o, v, 4);
  put(o, h.cfg_hash, 8);
  put(o, h.weights_hash, 8);
  put(o, h.prior, 4);
  put(o, h.n_bands, 4);
  put(o, 0, 4);  // reserved
}

void append_frame(std::vector<uint8_t>& o, const uint8_t* hyper, size_t hl, const uint8_t* main,
                  size_t ml) {
  put(o, hl, 4);
  o.insert(o.end(), hyper, hyper + hl);
  put(o, ml, 4);
  o.insert(o.end(), main, main + ml);
}

ContainerHeader parse_container(const uint8_t* p, size_t len, std::vector<FrameRef>* frames) {
  if (len < kContainerHeader || std::memcmp(p, "PSWA", 4) != 0)
    throw pswa_abi::TruncatedError("container: not a PSWA stream");
  if (get(p + 4, 2) != kContainerVersion || get(p + 6, 2) != kContainerHeader)
    throw std::invalid_argument("container: unsupported version " + std::to_string(get(p + 4, 2)) +
                                " (this decoder reads version " + std::to_string(kContainerVersion) +
                                "; other versions were coded under other model numerics)");
  ContainerHeader h;
  uint32_t* f[7] = {&h.w_px, &h.h_px, &h.frames, &h.gop, &h.rate, &h.s, &h.N};
  for (int i = 0; i < 7; ++i) *f[i] = static_cast<uint32_t>(get(p + 8 + 4 * i, 4));
  h.cfg_hash = get(p + 36, 8);
  h.weights_hash = get(p + 44, 8);
  h.prior = static_cast<uint32_t>(get(p + 52, 4));
  h.n_bands = static_cast<uint32_t>(get(p + 56, 4));
  if (h.gop == 0) throw std::invalid_argument("container: gop_size 0");
  if (frames) {
    frames->clear();
    size_t off = kContainerHeader;
    for (uint32_t k = 0; k < h.frames; ++k) {
      if (len - off < 4) break;
      const size_t hl = get(p + off, 4);
      if (len - off - 4 < hl + 4) break;
      const size_t ml = get(p + off + 4 + hl, 4);
      if (len - off - 8 - hl < ml) break;
      frames->push_back({off + 4, hl, off + 8 + hl, ml});
      off += 8 + hl + ml;
    }
  }
  return h;
}

}  // namespace pswa_host
