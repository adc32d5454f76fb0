// Device helpers shared by the sm_100a kernels: bf16 packing and hi/mid/lo
// splits, the legacy-HMMA m16n8k16 wrapper, mbarrier + cp.async.bulk (TMA
// bulk-copy engine) PTX, and the counter-based RNG that mirrors
// oracle/layer_oracle.hpp::hash_unit bit for bit.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define HX_DEV __device__ __forceinline__

namespace hx {

// ---------------------------------------------------------------- numerics
HX_DEV uint32_t pack_bf16(float lo, float hi) {
  // low 16 bits = first element (k / column index 2c), high = second
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
HX_DEV float bf16_to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
HX_DEV float round_bf16f(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

// x = hi + mid + lo with each term exactly representable in bf16; the sum
// reproduces x to ~24 significant bits (fp32 level).
HX_DEV void split3(float x, float& hi, float& mid, float& lo) {
  hi = round_bf16f(x);
  const float r1 = x - hi;
  mid = round_bf16f(r1);
  lo = round_bf16f(r1 - mid);
}
HX_DEV void split2(float x, float& hi, float& lo) {
  hi = round_bf16f(x);
  lo = round_bf16f(x - hi);
}

HX_DEV float fast_exp2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// D(16x8, f32) += A(16x16, bf16, row) * B(16x8, bf16, col). Legacy HMMA path:
// the GQA/GEMV operands here are 8-16 rows wide, far from a dense tcgen05
// M=128 tile, and the kernels are HBM-bound.
// f16 variants (FP8 KV pages widen to f16: every e4m3 value is exact in f16)
HX_DEV uint32_t pack_f16(float lo, float hi) {
  __half2 v = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
HX_DEV float round_f16f(float x) { return __half2float(__float2half_rn(x)); }
HX_DEV void split3h(float x, float& hi, float& mid, float& lo) {
  hi = round_f16f(x);
  const float r1 = x - hi;
  mid = round_f16f(r1);
  lo = round_f16f(r1 - mid);
}
HX_DEV void split2h(float x, float& hi, float& lo) {
  hi = round_f16f(x);
  lo = round_f16f(x - hi);
}
// four e4m3 bytes (byte i = element i) -> two f16x2 (elements 0,1 and 2,3; low half first)
HX_DEV void e4m3x4_to_f16x2x2(uint32_t four, uint32_t& lo, uint32_t& hi) {
  asm("{\n .reg .b16 a, b;\n mov.b32 {a, b}, %2;\n cvt.rn.f16x2.e4m3x2 %0, a;\n cvt.rn.f16x2.e4m3x2 %1, b;\n}"
      : "=r"(lo), "=r"(hi)
      : "r"(four));
}
// x = hi + lo with both halves f16 (22 significant bits), packed per pair
HX_DEV void split2h_pack(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(x0, x1);
  const float2 hf = __half22float2(h);
  const __half2 l = __floats2half2_rn(x0 - hf.x, x1 - hf.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}
HX_DEV void mma_f16_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                          uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 "
      "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
HX_DEV void mma_bf16_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                           uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 "
      "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// ---------------------------------------------------------------- loads
HX_DEV uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
HX_DEV uint4 ldg_stream(const void* p, uint64_t pol) {
  // streamed once: do not allocate in L1, evict-first in L2
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol));
  return v;
}
HX_DEV uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr));
  return v;
}
HX_DEV uint2 lds64(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}
HX_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- mbarrier / TMA bulk copy
HX_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
HX_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
HX_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
HX_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n.reg .b64 st;\nmbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(smem_u32(bar))
               : "memory");
}
HX_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "{\n.reg .b64 st;\nmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}" ::"r"(
          smem_u32(bar)),
      "r"(bytes)
      : "memory");
}
HX_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Bulk global->shared copy on the TMA engine, completion via mbarrier tx bytes.
HX_DEV void bulk_g2s(void* smem_dst, const void* gmem_src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---------------------------------------------------------------- programmatic dependent launch
// A kernel launched with programmatic stream serialization may start while the
// previous kernel drains; it must griddep_wait() before touching anything the
// previous kernel writes. No-ops for ordinary launches.
HX_DEV void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
HX_DEV void griddep_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---------------------------------------------------------------- RNG (== layer_oracle.hpp)
HX_DEV uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
HX_DEV double hash_unit(uint64_t seed, uint64_t stream, uint64_t index) {
  const uint64_t z = splitmix64(splitmix64(seed ^ (stream * 0xD1B54A32D192ED03ull)) + index);
  return 2.0 * (static_cast<double>(z >> 11) * 0x1.0p-53) - 1.0;
}
// Round-to-nearest-even of a double to bf16 (same values as oracle round_bf16).
HX_DEV __nv_bfloat16 double_to_bf16_rne(double x) {
  uint64_t b = static_cast<uint64_t>(__double_as_longlong(x));
  const uint64_t lsb = (b >> 45) & 1ull;
  b += 0x0FFFFFFFFFFFull + lsb;  // 2^44 - 1 + lsb
  b &= ~0x1FFFFFFFFFFFull;       // clear the low 45 bits
  return __float2bfloat16_rn(static_cast<float>(__longlong_as_double(static_cast<long long>(b))));
}

}  // namespace hx
