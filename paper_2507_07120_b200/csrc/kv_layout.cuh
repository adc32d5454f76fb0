// KV page layout in HBM (one page = 16 tokens of one KV head, K then V).
//
// Pages are stored "fragment-major": the byte image of a page is exactly the
// register image the decode kernel's mma.sync B-operands need, so a consumer
// warp reads its page with conflict-free 16-byte shared-memory loads (each
// warp instruction touches 512 contiguous bytes) after one bulk TMA copy.
//
//   K region [0, 32*DP):   for nt in {0,1} (tokens 8nt..8nt+7), kp in [0, DP/32),
//                          lane (g = lane/4, c = lane%4): 16 B =
//                            ks = 2kp   : (K[8nt+g][16ks+2c], +1), (K[..][16ks+2c+8], +9)
//                            ks = 2kp+1 : same two pairs
//   V region [32*DP, 64*DP): for nd2 in [0, DP/16), lane: 16 B =
//                            nd = 2nd2  : (V[2c][8nd+g], V[2c+1][8nd+g]), (V[2c+8][..], V[2c+9][..])
//                            nd = 2nd2+1: same two pairs
// bf16 pairs are packed low half = first element. DP is the head size padded
// to a multiple of 32; padded dims hold zeros.
#pragma once

#include <stdint.h>

#include "fp8.cuh"

namespace hx {

__host__ __device__ __forceinline__ uint32_t page_bytes(int dp) { return 64u * static_cast<uint32_t>(dp); }

// Byte offset of K[t][d] inside a page (t in [0,16), d in [0,DP)).
__host__ __device__ __forceinline__ uint32_t k_offset(int dp, int t, int d) {
  const int nt = t >> 3, g = t & 7;
  const int ks = d >> 4, r = d & 15;
  const int half = r >> 3, c = (r & 7) >> 1, elem = r & 1;
  const int kp = ks >> 1, sub = ks & 1;
  const int lane = g * 4 + c;
  return static_cast<uint32_t>(((nt * (dp / 32) + kp) * 32 + lane) * 16 + (sub * 2 + half) * 4 + elem * 2);
}

// Byte offset of V[t][d] inside a page.
__host__ __device__ __forceinline__ uint32_t v_offset(int dp, int t, int d) {
  const int nd = d >> 3, g = d & 7;
  const int nd2 = nd >> 1, sub = nd & 1;
  const int tt = t & 15;
  const int half = tt >> 3, c = (tt & 7) >> 1, elem = tt & 1;
  const int lane = g * 4 + c;
  return static_cast<uint32_t>(32 * dp + (nd2 * 32 + lane) * 16 + (sub * 2 + half) * 4 + elem * 2);
}

// FP8 (e4m3, fp8.cuh) pages: the same fragment order with 1-byte elements --
// every lane's 16-byte bf16 chunk becomes an 8-byte chunk, so each offset is
// exactly half of its bf16 offset and a page is 32*DP bytes. A consumer lane
// reads its 8 bytes and widens them (cvt e4m3x2 -> f16x2) into the register
// image the f16 mma.sync B-operands need.
__host__ __device__ __forceinline__ uint32_t page_bytes_kv(int dp, bool fp8) {
  return (fp8 ? 32u : 64u) * static_cast<uint32_t>(dp);
}
// FP8 pages in the tensor-core layout (fp8 mode 2; DP = 128, the tcgen05 GQA
// kernel, attention_tc.cu): two 8-token halves of 2 KB, each
//   K [dim/16 : 8][token : 8][16 dims]   -- the K-major UMMA core matrices
//                                           (8 rows x 16 B) of kind::f8f6f4, so
//                                           a 128-token tile of 8 pages is the A
//                                           operand of S^T = K . Q^T as loaded
//                                           (LBO 128 B, SBO 2 KB), no conversion
//   V [dim : 128][token : 8]             -- a converter thread (= dim) reads its
//                                           8 tokens as one 8-byte word
__host__ __device__ __forceinline__ uint32_t kv8tc_offset(int t, int d, bool is_v) {
  const uint32_t half = static_cast<uint32_t>(t >> 3) * 2048u, r = static_cast<uint32_t>(t & 7);
  return is_v ? half + 1024u + static_cast<uint32_t>(d) * 8u + r
              : half + static_cast<uint32_t>(d >> 4) * 128u + r * 16u + static_cast<uint32_t>(d & 15);
}
// fp8: 0 bf16 pages, 1 FP8 fragment-major pages, 2 FP8 tensor-core layout
__host__ __device__ __forceinline__ uint32_t kv_offset(int dp, int t, int d, bool is_v, int fp8) {
  if (fp8 == 2) return kv8tc_offset(t, d, is_v);
  const uint32_t off = is_v ? v_offset(dp, t, d) : k_offset(dp, t, d);
  return fp8 ? off >> 1 : off;
}

// FP4 (e2m1, fp8.cuh) pages: the same fragment order with 4-bit elements (a
// lane's 16-byte bf16 chunk becomes 4 bytes; element 2r of the chunk in the low
// nibble of byte r), K data [0, 8*DP), V data [8*DP, 16*DP), then the block
// scales 2^e (one per token and 32-dim group): K as exponent bytes e + 15,
// [16][DP/32] at 16*DP; V as ready-made f16 values, [DP/32][16 tokens] x 2 B
// at 16*DP + DP/2 -- so the V converters of the tcgen05 kernel load the f16x2
// scale of tokens (2c, 2c+1) as one word (attention_tc.cu). The f16 of 2^e is
// (e + 15) << 10: low byte 0, high byte (e + 15) << 2. A page is 17.5*DP bytes.
__host__ __device__ __forceinline__ uint32_t page_bytes_kv4(int dp) { return 35u * static_cast<uint32_t>(dp) / 2u; }
// byte offset of element (t, d) and whether it is the high nibble
__host__ __device__ __forceinline__ uint32_t kv4_offset(int dp, int t, int d, bool is_v, bool* high) {
  const uint32_t off = is_v ? v_offset(dp, t, d) - 32u * static_cast<uint32_t>(dp) : k_offset(dp, t, d);
  *high = ((off >> 1) & 1u) != 0;
  return (is_v ? 8u * static_cast<uint32_t>(dp) : 0u) + (off >> 2);
}
// the byte that carries the block scale of (t, d): K its exponent byte, V the
// high byte of its f16 (the low byte stays 0)
__host__ __device__ __forceinline__ uint32_t kv4_scale_offset(int dp, int t, int d, bool is_v) {
  return 16u * static_cast<uint32_t>(dp) +
         (is_v ? static_cast<uint32_t>(dp) / 2u + static_cast<uint32_t>((d / 32) * 32 + 2 * t + 1)
               : static_cast<uint32_t>(t * (dp / 32) + d / 32));
}
constexpr int kE2m1ExpBias = 15;  // K: stored exponent byte = e + 15
__host__ __device__ __forceinline__ uint8_t kv4_scale_byte(int e, bool is_v) {
  return static_cast<uint8_t>(is_v ? (e + kE2m1ExpBias) << 2 : e + kE2m1ExpBias);
}
__host__ __device__ __forceinline__ int kv4_scale_exp(uint8_t byte, bool is_v) {
  return (is_v ? byte >> 2 : byte) - kE2m1ExpBias;
}
// page bytes for a KV storage type: 0 bf16, 1 fp8, 2 fp4
__host__ __device__ __forceinline__ uint32_t page_bytes_kvt(int dp, int kvt) {
  return kvt == 2 ? page_bytes_kv4(dp) : page_bytes_kv(dp, kvt == 1);
}

// Round-robin placement (attention.hpp:262-282 in closed form): global token
// g of a cache grown only by append_round_robin with chunk c over kvp ranks.
__host__ __device__ __forceinline__ int rr_rank(long long g, int chunk, int kvp) {
  return static_cast<int>((g / chunk) % kvp);
}
__host__ __device__ __forceinline__ long long rr_row(long long g, int chunk, int kvp) {
  return (g / (static_cast<long long>(chunk) * kvp)) * chunk + g % chunk;
}
// Tokens held by rank r after `total` round-robin appends.
__host__ __device__ __forceinline__ long long rr_count(long long total, int r, int chunk, int kvp) {
  const long long cyc = static_cast<long long>(chunk) * kvp;
  const long long full = total / cyc, rem = total % cyc;
  long long extra = rem - static_cast<long long>(r) * chunk;
  extra = extra < 0 ? 0 : (extra > chunk ? chunk : extra);
  return full * chunk + extra;
}

}  // namespace hx

// ---------------------------------------------------------------------------
// MLA latent pages (types.hpp:37-49: one latent "KV head" of width W = 576 per
// token; keys = the whole latent, values = its first DV = 512 dims).
// One page = 128 local rows of one (rank shard, request). Layout = UMMA
// canonical no-swizzle core matrices, d-group major:
//   [dg = d/8 : 72][tg = row/8 : 16][row%8 : 8][d%8 : 8] bf16
// so 64 consecutive latent dims of all 128 rows are one contiguous 16 KB
// block: a K-major B operand (rows = tokens) for S = Q . C^T and, read with
// the other stride pair, an MN-major B operand (rows = tokens, N = dims) for
// O = P . V -- the same bytes, no transpose.
constexpr int kMlaW = 576;
constexpr int kMlaDV = 512;
constexpr int kMlaPageRows = 128;
constexpr int kMlaHeads = 128;  // UMMA M: query heads per CTA (zero-padded)
__host__ __device__ __forceinline__ uint32_t mla_page_bytes(bool f8 = false) {
  return kMlaPageRows * kMlaW * (f8 ? 1 : 2);
}
__host__ __device__ __forceinline__ uint32_t mla_kv_offset(int r, int d) {
  return static_cast<uint32_t>((((d >> 3) * (kMlaPageRows / 8) + (r >> 3)) * 64 + (r & 7) * 8 + (d & 7)) * 2);
}
// FP8 (e4m3) latent pages (kv_dtype = HX_KV_FP8_E4M3): the same core-matrix
// order with 16-byte rows of 16 dims --
//   [dg = d/16 : 36][tg = row/8 : 16][row%8 : 8][d%16 : 16] e4m3
// (a page = 36 rows of 2 KB): K-major A operand of S^T (kind::f8f6f4, K = 32
// per MMA = two dim groups), and MN-major A operand of O^T (tokens along K).
__host__ __device__ __forceinline__ uint32_t mla_kv_offset8(int r, int d) {
  return static_cast<uint32_t>((((d >> 4) * (kMlaPageRows / 8) + (r >> 3)) * 8 + (r & 7)) * 16 + (d & 15));
}
// Per-request absorbed-query image, split in two head halves (one per CTA of
// the MLA pair): [head/64 : 2][dg : 72][(head%64)/8 : 8][head%8][d%8] bf16 --
// each half is the K-major B operand (N = 64 heads) of S^T = C . Q^T and one
// contiguous 73,728-byte block. Written by the QKV epilogue.
__host__ __device__ __forceinline__ uint32_t mla_q_bytes(bool f8 = false) {
  return f8 ? kMlaW * kMlaHeads + kMlaHeads * 4 : kMlaW * kMlaHeads * 2;
}
// FP8 query image (FP8 latents): [head/64 : 2][dg = d/16 : 36][(head%64)/8 : 8][head%8][d%16]
// e4m3 of q * 2^e_h (per head, the largest power of two keeping max |q_h| <= 448),
// then float 2^-e_h per head at offset kMlaW * kMlaHeads.
__host__ __device__ __forceinline__ uint32_t mla_q_offset8(int head, int d) {
  return static_cast<uint32_t>(((((head >> 6) * 36 + (d >> 4)) * 8 + ((head & 63) >> 3)) * 8 + (head & 7)) * 16 +
                               (d & 15));
}
__host__ __device__ __forceinline__ uint32_t mla_q_offset(int head, int d) {
  return static_cast<uint32_t>(((((head >> 6) * 72 + (d >> 3)) * 8 + ((head & 63) >> 3)) * 8 + (head & 7)) * 16 +
                               (d & 7) * 2);
}
