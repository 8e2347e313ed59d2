// ORACLE — test infrastructure only.
// Discretised-Gaussian CDF tables and the multi-lane range coder
// (lane format DESIGN.md "Bitstream").
#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <stdexcept>

#include "oracle/model.h"

namespace oracle {

namespace {
constexpr int kEscLo = 2 * kSupport + 1;  // 255: v < -127
constexpr int kEscHi = 2 * kSupport + 2;  // 256: v >  127

int sym_of(int32_t v) {
  if (v < -kSupport) return kEscLo;
  if (v > kSupport) return kEscHi;
  return v + kSupport;
}
}  // namespace

void build_cdf(int idx, uint32_t* cum) {
  // scale table: 64 log-spaced sigmas in [0.11, 64]
  const bool laplace = idx >= kScales;
  if (laplace) idx -= kScales;
  const double ratio = det::log(64.0 / 0.11);
  const double sigma = static_cast<float>(0.11 * det::exp(ratio * idx / 63.0));
  const double inv = 1.0 / (sigma * 1.4142135623730951);
  uint32_t freq[kSyms];
  auto q = [](double p) {
    if (p < 0.0) p = 0.0;
    return 1u + static_cast<uint32_t>(std::floor(p * 65279.0));
  };
  if (!laplace) {
    freq[kSupport] = q(det::erf(0.5 * inv));
    for (int v = 1; v <= kSupport; ++v) {
      const double p = 0.5 * (det::erf((v + 0.5) * inv) - det::erf((v - 0.5) * inv));
      freq[kSupport + v] = freq[kSupport - v] = q(p);
    }
    freq[kEscLo] = freq[kEscHi] = q(0.5 * (1.0 - det::erf((kSupport + 0.5) * inv)));
  } else {
    // discretised Laplace with scale b = sigma: F(x) = 1 - exp(-x / b) / 2,
    // x >= 0, so p(0) = 1 - exp(-1/(2b)), p(v) = (exp(-(v-1/2)/b) -
    // exp(-(v+1/2)/b)) / 2, tail = exp(-(127+1/2)/b) / 2
    const double ib = 1.0 / sigma;
    freq[kSupport] = q(1.0 - det::exp(-0.5 * ib));
    for (int v = 1; v <= kSupport; ++v) {
      const double p = 0.5 * (det::exp(-(v - 0.5) * ib) - det::exp(-(v + 0.5) * ib));
      freq[kSupport + v] = freq[kSupport - v] = q(p);
    }
    freq[kEscLo] = freq[kEscHi] = q(0.5 * det::exp(-(kSupport + 0.5) * ib));
  }
  uint32_t sum = 0;
  for (int k = 0; k < kSyms; ++k) sum += freq[k];
  freq[kSupport] += 65536u - sum;  // deficit to the mode keeps symmetry
  cum[0] = 0;
  for (int k = 0; k < kSyms; ++k) cum[k + 1] = cum[k] + freq[k];
}

const Tables& tables() {
  static Tables t;
  static std::once_flag once;
  std::call_once(once, [] {
    const double ratio = det::log(64.0 / 0.11);
    for (int i = 0; i < kScales; ++i) {
      t.scale[i] = static_cast<float>(0.11 * det::exp(ratio * i / 63.0));
      build_cdf(i, t.cdf[i]);
      build_cdf(kScales + i, t.cdf[kScales + i]);
    }
  });
  return t;
}

int scale_index(float sigma) {
  const Tables& t = tables();
  for (int i = 0; i < kScales; ++i)
    if (t.scale[i] >= sigma) return i;
  return kScales - 1;
}

double bits_of(const CodedSym& s) {
  const uint32_t* c = tables().cdf[s.idx];
  const int k = sym_of(s.v);
  double b = 16.0 - std::log2(static_cast<double>(c[k + 1] - c[k]));
  if (k >= kEscLo) {
    const uint64_t x = static_cast<uint64_t>(std::abs(static_cast<int64_t>(s.v)) - 128) + 1;
    int nb = 0;
    while ((x >> (nb + 1)) != 0) ++nb;
    b += 2 * nb + 1;
  }
  return b;
}

// ------------------------------------------------------------ encoder ----
// 64-bit-state range coder with a 48-bit window: range in [2^40, 2^48), byte
// renormalisation (big-endian), carry propagated into written bytes, 4-byte
// flush. r = range >> 16 >= 2^24 keeps the truncation loss below
// 2^-24 relative per symbol, so the coded length stays within the +32-bit
// bound of SPEC.md:478.
namespace {
constexpr uint64_t kWin = (uint64_t{1} << 48) - 1;
constexpr uint64_t kBot = uint64_t{1} << 40;

struct LaneEnc {
  uint64_t low = 0;
  uint64_t range = kWin;
  std::vector<uint8_t> out;
  void carry() {
    for (size_t i = out.size(); i-- > 0;)
      if (++out[i] != 0) break;
  }
  void put(uint32_t cum, uint32_t freq) {
    const uint64_t r = range >> 16;
    low += r * cum;
    range = r * freq;
    if (low > kWin) {
      low &= kWin;
      carry();
    }
    while (range < kBot) {
      out.push_back(static_cast<uint8_t>(low >> 40));
      low = (low << 8) & kWin;
      range <<= 8;
    }
  }
  void bit(int b) { put(b ? 32768u : 0u, 32768u); }
  void finish() {
    uint64_t v = (low + 0xFFFF) & ~uint64_t{0xFFFF};  // in [low, low + range)
    if (v > kWin) {
      v &= kWin;
      carry();
    }
    for (int sh = 40; sh >= 16; sh -= 8) out.push_back(static_cast<uint8_t>(v >> sh));
  }
};
void put32le(std::vector<uint8_t>& b, uint32_t v) {
  for (int i = 0; i < 4; ++i) b.push_back(static_cast<uint8_t>(v >> (8 * i)));
}
uint32_t get32le(const uint8_t* p) {
  return p[0] | (p[1] << 8) | (p[2] << 16) | (static_cast<uint32_t>(p[3]) << 24);
}
}  // namespace

std::vector<uint8_t> encode_lanes(const std::vector<CodedSym>& syms, int lanes) {
  if (lanes < 1) throw std::invalid_argument("lanes < 1");
  std::vector<LaneEnc> L(static_cast<size_t>(lanes));
  const Tables& t = tables();
  for (size_t o = 0; o < syms.size(); ++o) {
    LaneEnc& e = L[o % lanes];
    const CodedSym& s = syms[o];
    const int k = sym_of(s.v);
    const uint32_t* c = t.cdf[s.idx];
    e.put(c[k], c[k + 1] - c[k]);
    if (k >= kEscLo) {  // Exp-Golomb(0) of |v| - 128, raw equiprobable bits
      const uint64_t x = static_cast<uint64_t>(std::abs(static_cast<int64_t>(s.v)) - 128) + 1;
      int nb = 0;
      while ((x >> (nb + 1)) != 0) ++nb;
      for (int i = 0; i < nb; ++i) e.bit(0);
      for (int i = nb; i >= 0; --i) e.bit(static_cast<int>((x >> i) & 1));
    }
  }
  // header: lanes, symbol count, width of the length entries (2 when every
  // lane is shorter than 64 KiB, else 4), then the lane lengths
  size_t longest = 0;
  for (auto& e : L) {
    e.finish();
    longest = std::max(longest, e.out.size());
  }
  const uint32_t w = longest < 65536 ? 2u : 4u;
  std::vector<uint8_t> out;
  put32le(out, static_cast<uint32_t>(lanes));
  put32le(out, static_cast<uint32_t>(syms.size()));
  put32le(out, w);
  for (auto& e : L) {
    const uint32_t n = static_cast<uint32_t>(e.out.size());
    for (uint32_t b = 0; b < w; ++b) out.push_back(static_cast<uint8_t>(n >> (8 * b)));
  }
  for (auto& e : L) out.insert(out.end(), e.out.begin(), e.out.end());
  return out;
}

// ------------------------------------------------------------ decoder ----
namespace {
// Next stream byte; up to 2 implicit zero bytes past the end are part of the
// format (the flush carries window bits 47..16), anything further is a
// truncated stream.
uint32_t next_byte(LaneDecoder::Lane& l, bool& err) {
  if (l.p < l.end) return *l.p++;
  if (l.p < l.end + 2) {
    ++l.p;
    return 0;
  }
  err = true;
  return 0;
}
}  // namespace

bool LaneDecoder::init(const uint8_t* data, size_t n) {
  error = false;
  lanes.clear();
  if (n < 12) return !(error = true);
  const uint32_t L = get32le(data);
  count = get32le(data + 4);
  const uint32_t w = get32le(data + 8);
  if (L == 0 || (w != 2 && w != 4) || n < 12 + static_cast<uint64_t>(w) * L) return !(error = true);
  size_t off = 12 + static_cast<size_t>(w) * L;
  lanes.resize(L);
  for (uint32_t i = 0; i < L; ++i) {
    const uint8_t* lp = data + 12 + static_cast<size_t>(w) * i;
    const uint32_t len = w == 2 ? static_cast<uint32_t>(lp[0] | (lp[1] << 8)) : get32le(lp);
    if (len < 4 || off + len > n) return !(error = true);
    Lane& l = lanes[i];
    l.p = data + off;
    l.end = data + off + len;
    l.code = 0;
    for (int b = 0; b < 6; ++b) l.code = (l.code << 8) | next_byte(l, error);
    off += len;
  }
  return !error;
}

namespace {
// Decodes one symbol of cumulative table `cum` (nsym+1 entries): the largest
// k with r*cum[k] <= code (no division needed).
int lane_get(LaneDecoder::Lane& l, const uint32_t* cum, int nsym, bool& err) {
  const uint64_t r = l.range >> 16;
  if (l.code >= r * 65536u) {
    err = true;
    l.code = r * 65536u - 1;
  }
  int lo = 0, hi = nsym;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (r * cum[mid] <= l.code)
      lo = mid;
    else
      hi = mid;
  }
  l.code -= r * cum[lo];
  l.range = r * (cum[lo + 1] - cum[lo]);
  while (l.range < kBot) {
    l.code = (l.code << 8) | next_byte(l, err);
    l.range <<= 8;
  }
  return lo;
}
const uint32_t kBitCum[3] = {0, 32768, 65536};
}  // namespace

int32_t LaneDecoder::decode(uint64_t ordinal, int idx) {
  Lane& l = lanes[ordinal % lanes.size()];
  const int k = lane_get(l, tables().cdf[idx], kSyms, error);
  if (k < kEscLo) return k - kSupport;
  int nb = 0;
  while (lane_get(l, kBitCum, 2, error) == 0) {
    if (++nb > 31 || error) {
      error = true;
      return 0;
    }
  }
  uint64_t x = 1;
  for (int i = 0; i < nb; ++i) x = (x << 1) | static_cast<uint64_t>(lane_get(l, kBitCum, 2, error));
  const int64_t m = static_cast<int64_t>(x) - 1 + 128;
  return static_cast<int32_t>(k == kEscLo ? -m : m);
}

}  // namespace oracle
