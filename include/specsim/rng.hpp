// Seed derivation and the deterministic RNG of the drop-in API; draws are
// identical to the reference's rng.hpp:11-68 (SplitMix64 finaliser, 4-way
// mix_seed, std::mt19937_64 with hand-rolled distributions).
#pragma once

#include <cstdint>
#include <random>

namespace specsim {

std::uint64_t splitmix64(std::uint64_t x);
std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t a, std::uint64_t b = 0, std::uint64_t c = 0);

// Stream tags (the reference's four plus the B200 prompt stream).
enum : std::uint64_t {
  kStreamWorkload = 0x01,
  kStreamPolicy = 0x02,
  kStreamOutcome = 0x03,
  kStreamToyAttention = 0x04,
  kStreamPrompt = 0x05,  // synthetic prompt tokens of the B200 backend
};

class Rng {
 public:
  explicit Rng(std::uint64_t seed) : engine_(seed) {}
  std::uint64_t next() { return engine_(); }
  double unit();                                // [0, 1), 53 random bits
  double uniform(double lo, double hi);         // lo + (hi - lo) * unit()
  bool bernoulli(double p) { return unit() < p; }
  long long uniform_int(long long lo, long long hi);  // inclusive, rejection sampled

 private:
  std::mt19937_64 engine_;
};

}  // namespace specsim
