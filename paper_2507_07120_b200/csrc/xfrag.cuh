// Activation fragments ("xf"): the B x K activation matrix pre-split into bf16
// terms in the exact register image of the GEMV's mma.sync B operand, written
// ONCE by whoever produces the activation (embedding, residual epilogues,
// SwiGLU epilogue, the attention merge) and streamed by the GEMV next to its
// weights with the TMA bulk engine.
//
// Layout: [k-step ks][term t < 3][batch group bg < NB8][lane][2 x u32]
//   lane (g = lane/4, c = lane%4), batch b = 8*bg + g:
//   u32 0 = (x[b][16ks+2c], x[b][16ks+2c+1]), u32 1 = (x[b][16ks+2c+8], x[b][16ks+2c+9])
//   terms: hi = bf16(x), mid = bf16(x - hi), lo = bf16(x - hi - mid); a GEMV
//   that needs ~16-bit activations reads hi+mid, the QKV projection all three.
//   FP8-weight models (xf16 = 1) store two f16 terms instead (hi = f16(x),
//   lo = f16(x - hi): 22 significant bits, absolute floor 2^-25; term 2 zero)
//   for the f16 MMA that multiplies the widened e4m3 weights.
//
// Batches above 16 (nb8 >= 4) run the tcgen05 GEMV (gemv_tc.cu), whose B
// operand is K-major in canonical core matrices: layout
//   [k-step][term][batch group bg][k-half][batch row g][8 k] bf16
// -- per k-step the terms' batch groups are consecutive 256-byte pairs of core
// matrices (UMMA descriptor LBO = 128 B along K, SBO = 256 B per 8 rows), so
// one MMA with N = 2 * 8 * nb8 multiplies the hi and mid terms at once.
#pragma once

#include "common.cuh"
#include "kernels.h"  // xf_nb8

namespace hx {

constexpr int kXfTerms = 3;

__host__ __device__ __forceinline__ size_t xf_step_bytes(int nb8) {
  return static_cast<size_t>(kXfTerms) * nb8 * 32 * 8;
}

// Write activation value v of (batch b, column k) into the fragment buffer.
HX_DEV void xf_write(uint8_t* xf, int nb8, int b, int k, float v, int xf16 = 0) {
  const int ks = k >> 4, r = k & 15;
  const int half = r >> 3, c = (r & 7) >> 1, elem = r & 1;
  const int g = b & 7, bg = b >> 3;
  const int lane = g * 4 + c;
  float t[3];
  if (xf16) {
    split2h(v, t[0], t[1]);
    t[2] = 0.f;
  } else {
    split3(v, t[0], t[1], t[2]);
  }
  const bool tc = nb8 >= 4;
#pragma unroll
  for (int term = 0; term < kXfTerms; ++term) {
    const size_t blk = ((static_cast<size_t>(ks) * kXfTerms + term) * nb8 + bg) * 32 * 8;
    const size_t off = tc ? blk + half * 128 + g * 16 + (r & 7) * 2 : blk + lane * 8 + half * 4 + elem * 2;
    if (xf16)
      *reinterpret_cast<__half*>(xf + off) = __float2half_rn(t[term]);
    else
      *reinterpret_cast<__nv_bfloat16*>(xf + off) = __float2bfloat16_rn(t[term]);
  }
}

}  // namespace hx
