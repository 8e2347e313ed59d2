// pswa/rng.h — deterministic random streams (drop-in for the reference's
// proj/include/pswa/rng.h:24-78, same names and semantics).
//
//   Rng                 SplitMix64; next_uniform() has 24-bit resolution
//                       (exact in f32); next_normal() is Irwin-Hall(12) - 6
//   fnv1a64             64-bit FNV-1a over a string or a byte range
//   rng_for_parameter   one stream per named parameter: seed ^ fnv1a64(name)
//
// Used on the host for the synthetic weights (gen_weights) and inputs that
// the CPU oracle and the sm_100a path share.
#ifndef PSWA_RNG_H_
#define PSWA_RNG_H_

#include <cstddef>
#include <cstdint>
#include <string_view>

namespace pswa {

class Rng {
 public:
  explicit Rng(uint64_t seed) : s_(seed) {}

  uint64_t next_u64() {
    s_ += kGamma;
    return mix(s_);
  }
  float next_uniform() { return static_cast<float>(next_u64() >> 40) * 0x1p-24f; }
  float next_normal() {
    float acc = 0.0f;
    for (int k = 0; k < 12; ++k) acc += next_uniform();
    return acc - 6.0f;
  }

 private:
  static constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ULL;
  static uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
  uint64_t s_;
};

inline uint64_t fnv1a64(const void* data, size_t n) {
  constexpr uint64_t kPrime = 0x100000001B3ULL;
  uint64_t h = 0xCBF29CE484222325ULL;
  const auto* b = static_cast<const unsigned char*>(data);
  for (size_t k = 0; k < n; ++k) h = (h ^ b[k]) * kPrime;
  return h;
}
inline uint64_t fnv1a64(std::string_view s) { return fnv1a64(s.data(), s.size()); }

inline Rng rng_for_parameter(uint64_t global_seed, std::string_view name) {
  return Rng(global_seed ^ fnv1a64(name));
}

}  // namespace pswa

#endif  // PSWA_RNG_H_
