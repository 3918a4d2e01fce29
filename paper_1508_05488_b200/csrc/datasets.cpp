// Synthetic point sets, bit-identical to the reference generator
// (datasets.hpp:13-35, datasets.cpp:17-106): std::mt19937_64 seeded with
// the spec seed, unit doubles from the top 53 bits of each draw, libm for
// the disk/circle/gaussian shapes (the GPU box runs the same image, hence
// the same glibc). Used for the benchmark and the parity fixtures' inputs;
// tests/test_golden.py pins every distribution against hashes of the
// reference's own output.

#include <cmath>
#include <cstdint>
#include <random>

#include "chgpu.h"

namespace {

constexpr double kTwoPi = 2.0 * 3.141592653589793;

inline double draw01(std::mt19937_64& g) { return static_cast<double>(g() >> 11) * 0x1.0p-53; }

}  // namespace

extern "C" int chgpu_generate(int dist, size_t n, uint64_t seed, double* out) {
  if (n == 0) return CHGPU_INVALID_ARG;
  std::mt19937_64 g(seed);
  switch (dist) {
    case 0:  // uniform_square
      for (size_t i = 0; i < n; ++i) {
        out[2 * i] = draw01(g);
        out[2 * i + 1] = draw01(g);
      }
      return CHGPU_OK;
    case 1:  // uniform_disk: r = sqrt(u), theta = 2*pi*u
      for (size_t i = 0; i < n; ++i) {
        const double r = std::sqrt(draw01(g));
        const double th = kTwoPi * draw01(g);
        out[2 * i] = r * std::cos(th);
        out[2 * i + 1] = r * std::sin(th);
      }
      return CHGPU_OK;
    case 2: {  // circle: n evenly spaced angles with a random phase
      const double phase = kTwoPi * draw01(g);
      for (size_t i = 0; i < n; ++i) {
        const double th = phase + kTwoPi * static_cast<double>(i) / static_cast<double>(n);
        out[2 * i] = std::cos(th);
        out[2 * i + 1] = std::sin(th);
      }
      return CHGPU_OK;
    }
    case 3:  // gaussian: Box-Muller, two draws per point
      for (size_t i = 0; i < n; ++i) {
        const double u1 = 1.0 - draw01(g);
        const double u2 = draw01(g);
        const double mag = std::sqrt(-2.0 * std::log(u1));
        out[2 * i] = mag * std::cos(kTwoPi * u2);
        out[2 * i + 1] = mag * std::sin(kTwoPi * u2);
      }
      return CHGPU_OK;
    case 4:  // collinear: (u, u)
      for (size_t i = 0; i < n; ++i) out[2 * i] = out[2 * i + 1] = draw01(g);
      return CHGPU_OK;
    case 5:  // duplicates_heavy: 9x9 lattice
      for (size_t i = 0; i < n; ++i) {
        out[2 * i] = static_cast<double>(g() % 9) / 8.0;
        out[2 * i + 1] = static_cast<double>(g() % 9) / 8.0;
      }
      return CHGPU_OK;
    default:
      return CHGPU_INVALID_ARG;
  }
}
