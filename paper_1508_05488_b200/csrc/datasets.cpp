// Synthetic point sets, bit-identical to the reference generator
// (datasets.hpp:13-35, datasets.cpp:17-106): std::mt19937_64 seeded with
// the spec seed, unit doubles from the top 53 bits of each draw, libm for
// the disk/circle/gaussian shapes (the GPU box runs the same image, hence
// the same glibc). Used for the benchmark and the parity fixtures' inputs;
// tests/test_oracle.py pins every distribution against hashes of the
// reference's own output.
//
// chgpu_generate_range writes points [begin, begin + count) of the n-point
// set: every distribution consumes a fixed number of draws per point (the
// circle one draw in all), so a slice starts after discarding the draws of
// the points before it. That is how each rank of the sharded run builds
// its contiguous shard of the 1B-point set without the whole set.

#include <cmath>
#include <cstdint>
#include <random>

#include "chgpu.h"

namespace {

constexpr double kTwoPi = 2.0 * 3.141592653589793;

inline double draw01(std::mt19937_64& g) { return static_cast<double>(g() >> 11) * 0x1.0p-53; }

// Generator draws consumed per point (0: the circle draws once per set).
int draws_per_point(int dist) {
  switch (dist) {
    case 0: case 1: case 3: case 5: return 2;
    case 4: return 1;
    case 2: return 0;
    default: return -1;
  }
}

void one_point(int dist, std::mt19937_64& g, double* p) {
  switch (dist) {
    case 0:  // uniform_square
      p[0] = draw01(g);
      p[1] = draw01(g);
      break;
    case 1: {  // uniform_disk: r = sqrt(u), theta = 2*pi*u
      const double r = std::sqrt(draw01(g));
      const double th = kTwoPi * draw01(g);
      p[0] = r * std::cos(th);
      p[1] = r * std::sin(th);
      break;
    }
    case 3: {  // gaussian: Box-Muller, two draws per point
      const double u1 = 1.0 - draw01(g);
      const double u2 = draw01(g);
      const double mag = std::sqrt(-2.0 * std::log(u1));
      p[0] = mag * std::cos(kTwoPi * u2);
      p[1] = mag * std::sin(kTwoPi * u2);
      break;
    }
    case 4:  // collinear: (u, u)
      p[0] = p[1] = draw01(g);
      break;
    default: {  // 5 duplicates_heavy: 9x9 lattice (x drawn first)
      const double x = static_cast<double>(g() % 9) / 8.0;
      p[0] = x;
      p[1] = static_cast<double>(g() % 9) / 8.0;
      break;
    }
  }
}

}  // namespace

extern "C" int chgpu_generate_range(int dist, size_t n, uint64_t seed, size_t begin, size_t count,
                                    double* out) {
  const int dpp = draws_per_point(dist);
  if (dpp < 0 || n == 0 || begin > n || count > n - begin) return CHGPU_INVALID_ARG;
  std::mt19937_64 g(seed);
  if (dist == 2) {  // circle: n evenly spaced angles after one phase draw
    const double phase = kTwoPi * draw01(g);
    for (size_t j = 0; j < count; ++j) {
      const double th =
          phase + kTwoPi * static_cast<double>(begin + j) / static_cast<double>(n);
      out[2 * j] = std::cos(th);
      out[2 * j + 1] = std::sin(th);
    }
    return CHGPU_OK;
  }
  g.discard(static_cast<unsigned long long>(begin) * static_cast<unsigned long long>(dpp));
  for (size_t j = 0; j < count; ++j) one_point(dist, g, out + 2 * j);
  return CHGPU_OK;
}

extern "C" int chgpu_generate(int dist, size_t n, uint64_t seed, double* out) {
  return chgpu_generate_range(dist, n, seed, 0, n, out);
}
