// rng.cpp — the reference's seeded generator on the host side of libmlra
// (include/mlra.h, mlra_gaussian_fill / mlra_mix_seed), so init_adapter and
// seeded inputs reproduce the reference's values bit-for-bit:
//   Rng (rng.hpp:15-48): std::mt19937_64 with the reference's own mappings —
//   uniform = (x >> 11) * 2^-53 (:24-26), gaussian = Box-Muller cosine branch,
//   no cached spare (:30-35); mix_seed = splitmix64 finalizer (:52-57);
//   DenseMatrix::gaussian (matrix.cpp:62-67) fills row-major as mean + std·g.
#include <cmath>
#include <cstdint>

#include "../../include/mlra.h"

namespace {

class Mt64 {  // std::mt19937_64, written out so the stream is platform-pinned
 public:
  explicit Mt64(uint64_t seed) {
    mt_[0] = seed;
    for (int i = 1; i < kN; ++i)
      mt_[i] = 6364136223846793005ULL * (mt_[i - 1] ^ (mt_[i - 1] >> 62)) + static_cast<uint64_t>(i);
    idx_ = kN;
  }
  uint64_t next() {
    if (idx_ >= kN) twist();
    uint64_t x = mt_[idx_++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
  }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double gaussian() {
    const double u1 = 1.0 - uniform();
    const double u2 = uniform();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.14159265358979323846 * u2);
  }

 private:
  static constexpr int kN = 312;
  void twist() {
    const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
    for (int i = 0; i < kN; ++i) {
      const uint64_t x = (mt_[i] & upper) | (mt_[(i + 1) % kN] & lower);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      mt_[i] = mt_[(i + 156) % kN] ^ xa;
    }
    idx_ = 0;
  }
  uint64_t mt_[kN];
  int idx_;
};

}  // namespace

extern "C" {

uint64_t mlra_mix_seed(uint64_t seed, uint64_t salt) {
  uint64_t z = seed + 0x9E3779B97F4A7C15ULL * (salt + 1);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

void mlra_gaussian_fill(uint64_t seed, double* out, uint64_t n, double mean, double stddev) {
  if (!out) return;
  Mt64 r(seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = mean + stddev * r.gaussian();
}

}  // extern "C"
