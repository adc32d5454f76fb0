// FP8 E4M3 ("e4m3fn": bias 7, no infinities, max finite 448, 0x7F / 0xFF NaN)
// KV storage (the paper evaluates at FP4).
//
// encode: round-to-nearest-even from a double, saturating to +-448 (the
// semantics of cvt.rn.satfinite.e4m3x2 and of oracle round_e4m3); identical on
// host and device, so the hash fill, the host-side grow_random draws and the
// QKV epilogue's appended rows all round exactly as the oracle does.
// decode: every e4m3 value is exactly representable in f16 (and float).
#pragma once

#include <stdint.h>

#ifdef __CUDACC__
#define HX_HD __host__ __device__ __forceinline__
#else
#define HX_HD inline
#endif

namespace hx {

HX_HD uint8_t e4m3_from_double(double x) {
  if (x != x) return 0x7F;
  const uint8_t sign = x < 0.0 ? 0x80 : 0x00;
  const double a = x < 0.0 ? -x : x;
  if (a >= 464.0) return sign | 0x7E;  // beyond the 448 / 480 midpoint: saturate
  // binade of a: a in [2^e, 2^(e+1)); subnormals share the 2^-6 binade's quantum
  int e = -6;
  double p = 0x1.0p-6;  // 2^e
  if (a >= p) {
    while (a >= 2.0 * p) {
      p *= 2.0;
      ++e;
    }
  }
  const double q = p * 0.125;                  // quantum: 3 mantissa bits
  const double t = a / q;                      // exact (power-of-two scale)
  double r = static_cast<double>(static_cast<long long>(t));
  const double frac = t - r;
  if (frac > 0.5 || (frac == 0.5 && (static_cast<long long>(r) & 1))) r += 1.0;  // RNE
  long long m = static_cast<long long>(r);     // a ~= m * q, m in [0, 16]
  if (e == -6 && m < 8) return sign | static_cast<uint8_t>(m);  // subnormal (or zero)
  if (m == 16) {                               // carried into the next binade
    m = 8;
    ++e;
  }
  const int ef = e + 7;
  if (ef > 15 || (ef == 15 && m - 8 == 7)) return sign | 0x7E;
  return sign | static_cast<uint8_t>(ef << 3) | static_cast<uint8_t>(m - 8);
}

HX_HD float e4m3_to_float(uint8_t v) {
  const int ef = (v >> 3) & 15, m = v & 7;
  float r;
  if (ef == 0) {
    r = static_cast<float>(m) * 0x1.0p-9f;
  } else if (ef == 15 && m == 7) {
    r = 0.0f / 0.0f;
  } else {
    r = (1.0f + static_cast<float>(m) * 0.125f);
    int k = ef - 7;
    while (k > 0) {
      r *= 2.0f;
      --k;
    }
    while (k < 0) {
      r *= 0.5f;
      ++k;
    }
  }
  return (v & 0x80) ? -r : r;
}

}  // namespace hx
