// qt_rng.cpp — seeded synthetic inputs for the T-product (host side).
//
// QT_DIST_UNIFORM_SYM is bitwise the reference's gen_random_tensor
// (/root/reference/proj/src/rng.cpp:21-33, Rng::sym at rng.hpp:24-26):
// mt19937_64(seed), u = (x >> 11) * 2^-53, sym = 2u - 1, drawn per entry in
// file order (slice, row, column) as w, x, y, z; t1 = w + x i, t2 = y + z i
// (the Cayley-Dickson split of algebra.hpp:61-68).
// The other two distributions are this repo's convention for BASELINE configs
// 2 and 4: Box-Muller over consecutive top-53 uniforms
// (u1 -> 1-u1 in (0,1], one normal per pair) and the pure-quaternion RGB
// tensor (w = 0, x, y, z uniform in [0,1)).
#include <cmath>
#include <cstdint>
#include <random>

#include "../../include/qtensor_b200.h"

namespace {

inline double top53(std::mt19937_64& g) { return static_cast<double>(g() >> 11) * 0x1.0p-53; }

inline double normal(std::mt19937_64& g) {
  const double u1 = 1.0 - top53(g);  // (0, 1]
  const double u2 = top53(g);        // [0, 1)
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925286766559 * u2);
}

inline uint64_t splitmix64(uint64_t& state) {  // rng.cpp:7-12
  uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

}  // namespace

extern "C" {

uint64_t qt_derive_seed(uint64_t base, uint64_t stream) {  // rng.cpp:15-19
  uint64_t state = base, out = 0;
  for (uint64_t k = 0; k <= stream; ++k) out = splitmix64(state);
  return out;
}

int qt_gen_tensor_f64(int dist, uint64_t m, uint64_t n, uint64_t p, uint64_t seed, double scale, double* t1,
                      double* t2) {
  if (m == 0 || n == 0 || p == 0) return QT_EINVAL;  // rng.cpp:23-24
  if (!t1 || !t2) return QT_EINVAL;
  std::mt19937_64 g(seed);
  const uint64_t count = m * n * p;
  switch (dist) {
    case QT_DIST_UNIFORM_SYM:
      for (uint64_t k = 0; k < count; ++k) {
        const double w = 2.0 * top53(g) - 1.0, x = 2.0 * top53(g) - 1.0;
        const double y = 2.0 * top53(g) - 1.0, z = 2.0 * top53(g) - 1.0;
        t1[2 * k] = w; t1[2 * k + 1] = x;
        t2[2 * k] = y; t2[2 * k + 1] = z;
      }
      return QT_OK;
    case QT_DIST_NORMAL:
      for (uint64_t k = 0; k < count; ++k) {
        const double w = normal(g), x = normal(g), y = normal(g), z = normal(g);
        t1[2 * k] = scale * w; t1[2 * k + 1] = scale * x;
        t2[2 * k] = scale * y; t2[2 * k + 1] = scale * z;
      }
      return QT_OK;
    case QT_DIST_PURE_UNIT:
      for (uint64_t k = 0; k < count; ++k) {
        const double x = top53(g), y = top53(g), z = top53(g);
        t1[2 * k] = 0.0; t1[2 * k + 1] = x;
        t2[2 * k] = y; t2[2 * k + 1] = z;
      }
      return QT_OK;
    default:
      return QT_EINVAL;
  }
}

}  // extern "C"
