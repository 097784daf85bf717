// Host-side parameter realisation with the reference's own seeded generator.
//
// The reference draws every diagonal on the host from mt19937_64 seeded through
// splitmix64 (proj/include/spinners/common.hpp:51-92) in a fixed order
// (proj/src/spinner.cpp:137-151, draw_tail :92-106, stacking :248-256).  These
// functions reproduce that order bit for bit (std::mt19937_64 is fully specified
// by the C++ standard; Box-Muller uses the same libm calls), so the uploaded
// diagonals equal the reference's realised ones exactly.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <vector>

namespace spn {

inline uint64_t mix_seed(uint64_t base, uint64_t stream) {  // common.hpp:51-56
  uint64_t z = base + 0x9e3779b97f4a7c15ULL * (stream + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

class HostRng {  // common.hpp:61-92
 public:
  explicit HostRng(uint64_t seed) : eng_(seed) {}
  uint64_t next_u64() { return eng_(); }
  double uniform01() { return (static_cast<double>(eng_() >> 11) + 1.0) * 0x1p-53; }
  double gaussian() {
    if (have_spare_) {
      have_spare_ = false;
      return spare_;
    }
    const double u = uniform01();
    const double v = uniform01();
    const double rad = std::sqrt(-2.0 * std::log(u));
    const double ang = 2.0 * M_PI * v;
    spare_ = rad * std::sin(ang);
    have_spare_ = true;
    return rad * std::cos(ang);
  }
  double rademacher() { return (eng_() & 1) ? 1.0 : -1.0; }

 private:
  std::mt19937_64 eng_;
  bool have_spare_ = false;
  double spare_ = 0.0;
};

enum Variant : int { V_HD3 = 0, V_HDG = 1, V_GAUSS3 = 100 };

// One block (spec seed = mix_seed(stacked_seed, b)): D1, D2 from the front stream,
// D3 (Rademacher) or g (Gaussian) from the tail stream.  V_GAUSS3 is the
// builder-defined all-Gaussian variant of BASELINE config 5 (same streams).
inline void realize_block(int variant, int64_t n, uint64_t spec_seed, double* d1, double* d2,
                          double* d3) {
  HostRng front(mix_seed(spec_seed, 1));
  HostRng tail(mix_seed(spec_seed, 2));
  if (variant == V_GAUSS3) {
    for (int64_t i = 0; i < n; ++i) d1[i] = front.gaussian();
    for (int64_t i = 0; i < n; ++i) d2[i] = front.gaussian();
    for (int64_t i = 0; i < n; ++i) d3[i] = tail.gaussian();
    return;
  }
  for (int64_t i = 0; i < n; ++i) d1[i] = front.rademacher();
  for (int64_t i = 0; i < n; ++i) d2[i] = front.rademacher();
  if (variant == V_HDG)
    for (int64_t i = 0; i < n; ++i) d3[i] = tail.gaussian();
  else
    for (int64_t i = 0; i < n; ++i) d3[i] = tail.rademacher();
}

// Builder-defined coordinate sampler (BASELINE config 4): partial
// Fisher-Yates over [0, N) with unbiased rejection, Rng(mix_seed(seed, 0x5a3b)).
inline std::vector<int64_t> sample_rows(int64_t N, int64_t m, uint64_t seed) {
  std::vector<int64_t> idx(static_cast<size_t>(N));
  for (int64_t i = 0; i < N; ++i) idx[static_cast<size_t>(i)] = i;
  HostRng r(mix_seed(seed, 0x5a3b));
  for (int64_t i = 0; i < m; ++i) {
    const uint64_t range = static_cast<uint64_t>(N - i);
    const uint64_t threshold = (0 - range) % range;
    uint64_t u;
    do {
      u = r.next_u64();
    } while (u < threshold);
    std::swap(idx[static_cast<size_t>(i)], idx[static_cast<size_t>(i + static_cast<int64_t>(u % range))]);
  }
  idx.resize(static_cast<size_t>(m));
  std::sort(idx.begin(), idx.end());
  return idx;
}

}  // namespace spn
