// rnnwave/rng.hpp -- SplitMix64 (Steele, Lea, Flood) and its derived streams, identical in
// output to the reference generator (proj/include/rnnwave/rng.hpp:13-48): every weight and
// synthetic input of the facade is reproducible from one 64-bit seed.
#pragma once

#include <cstdint>

namespace rnnwave {

inline std::uint64_t splitmix64_mix(std::uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

class SplitMix64 {
 public:
  explicit SplitMix64(std::uint64_t seed) : s_(seed) {}
  std::uint64_t next_u64() { return splitmix64_mix(s_ += 0x9E3779B97F4A7C15ull); }
  double next_unit() { return double(next_u64() >> 11) * 0x1.0p-53; }
  float next_symmetric(double range) { return float((2.0 * next_unit() - 1.0) * range); }

 private:
  std::uint64_t s_;
};

inline SplitMix64 split_stream(std::uint64_t seed, std::uint64_t k) {
  return SplitMix64(splitmix64_mix(seed + k * 0x9E3779B97F4A7C15ull));
}

}  // namespace rnnwave
