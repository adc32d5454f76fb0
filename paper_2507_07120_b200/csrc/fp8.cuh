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
#define HX_F8HD __host__ __device__ __forceinline__
#else
#define HX_F8HD inline
#endif

namespace hx {

HX_F8HD uint8_t e4m3_from_double(double x) {
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

HX_F8HD float e4m3_to_float(uint8_t v) {
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

// ---------------------------------------------------------------------------
// FP4 E2M1 KV storage (PAPER.md:158 evaluates Helix at FP4): MX-style blocks of
// 32 elements -- one (token, KV head, 32-dim group) of K or of V -- share a
// power-of-two scale 2^e, e = the smallest exponent with 6 * 2^e >= max |x|
// (clamped to [-14, 13], so 2^e is a normal f16 and every stored value grid * 2^e
// is exact in f16);
// each element is the e2m1 code of x / 2^e rounded to nearest-even on the grid
// {0, 0.5, 1, 1.5, 2, 3, 4, 6} (saturating at 6). Identical on host, device and
// in the oracle (round_e2m1_block), always from the value the writer holds
// (double for grown / hash-filled rows, fp32 for projected rows).
namespace hx {

constexpr int kE2m1MinExp = -14, kE2m1MaxExp = 13;  // 2^e normal in f16: the kernel builds it by a shift

HX_F8HD int e2m1_block_exp(double amax) {
  if (!(amax > 0.0)) return 0;
  // smallest e with 6 * 2^e >= amax: amax / 6 = m * 2^k, m in [0.5, 1)
  const double r = amax / 6.0;
  int k = 0;
  double m = r;
  while (m >= 1.0) {
    m *= 0.5;
    ++k;
  }
  while (m < 0.5) {
    m *= 2.0;
    --k;
  }
  int e = (m == 0.5) ? k - 1 : k;
  if (e < kE2m1MinExp) e = kE2m1MinExp;
  if (e > kE2m1MaxExp) e = kE2m1MaxExp;
  return e;
}

HX_F8HD double pow2i(int e) {
  double s = 1.0;
  for (; e > 0; --e) s *= 2.0;
  for (; e < 0; ++e) s *= 0.5;
  return s;
}

// e2m1 code (sign << 3 | magnitude code) of x / 2^e, round to nearest even.
HX_F8HD uint8_t e2m1_from_double(double x, int e) {
  const uint8_t sign = x < 0.0 ? 8 : 0;
  const double t = (x < 0.0 ? -x : x) / pow2i(e);  // exact: power-of-two scale
  // grid 0 0.5 1 1.5 2 3 4 6 (codes 0..7); midpoints go to the even code
  uint8_t c;
  if (t < 0.25) c = 0;
  else if (t == 0.25) c = 0;
  else if (t < 0.75) c = 1;
  else if (t == 0.75) c = 2;
  else if (t < 1.25) c = 2;
  else if (t == 1.25) c = 2;
  else if (t < 1.75) c = 3;
  else if (t == 1.75) c = 4;
  else if (t < 2.5) c = 4;
  else if (t == 2.5) c = 4;
  else if (t < 3.5) c = 5;
  else if (t == 3.5) c = 6;
  else if (t < 5.0) c = 6;
  else if (t == 5.0) c = 6;
  else c = 7;
  return sign | c;
}

HX_F8HD float e2m1_to_float(uint8_t code, int e) {
  const float grid[8] = {0.f, 0.5f, 1.f, 1.5f, 2.f, 3.f, 4.f, 6.f};
  const float v = grid[code & 7] * static_cast<float>(pow2i(e));
  return (code & 8) ? -v : v;
}

}  // namespace hx
