// Small kernels around the decode step: fragment merge for the attention-only
// harness output, embedding gather, greedy-token finish, KV scatter/fill into
// the round-robin page pool, and hash-RNG weight init directly into the
// fragment-major layout (values identical to oracle/layer_oracle.hpp).
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "kv_layout.cuh"
#include "xfrag.cuh"
#include "merge.cuh"

namespace hx {

// ---------------------------------------------------------------- merge (harness output)
// out[b][head][d] = canonical LSE merge over kvp rank fragments
// (merge_fragments / merge_head_fragments, attention.hpp:118-175).
template <int MAXK>
__global__ void merge_out_kernel(const float* frag_o, const float* frag_lse, int batch,
                                 int q_heads, int q_per_slot, int kvp, int head_dim, int dp,
                                 float* out, float* out_lse, int* bump_total) {
  griddep_wait();
  griddep_launch_dependents();
  const int gi = blockIdx.x * blockDim.x + threadIdx.x;
  if (bump_total && gi < batch) bump_total[gi] += 1;  // attend-then-append: the new token now counts
  const int warp = gi >> 5, lane = threadIdx.x & 31;
  if (warp >= batch * q_heads) return;
  const int b = warp / q_heads, head = warp - b * q_heads;
  const int grp = head / q_per_slot, qi = head - grp * q_per_slot;
  float lse[MAXK], o[MAXK];
  for (int r = 0; r < kvp; ++r)
    lse[r] = frag_lse[(static_cast<size_t>(grp * kvp + r) * batch + b) * q_per_slot + qi];
  for (int d = lane; d < head_dim; d += 32) {
    for (int r = 0; r < kvp; ++r)
      o[r] = frag_o[((static_cast<size_t>(grp * kvp + r) * batch + b) * q_per_slot + qi) * dp + d];
    out[(static_cast<size_t>(b) * q_heads + head) * head_dim + d] = merge_sources<MAXK>(lse, o, kvp);
  }
  if (lane == 0 && out_lse) {
    // lse = m + ln(sum of weights); the weights' sum does not depend on how lse ties are ordered
    float m = -INFINITY;
    for (int r = 0; r < kvp; ++r) m = fmaxf(m, lse[r]);
    float z = 0.f;
    if (m != -INFINITY) {
      // same descending-lse order as merge_sources
      int ord[MAXK];
      for (int r = 0; r < kvp; ++r) ord[r] = r;
      for (int i = 1; i < kvp; ++i) {
        const int v = ord[i];
        int j = i - 1;
        while (j >= 0 && merge_before(lse[v], 0.f, v, lse[ord[j]], 0.f, ord[j])) {
          ord[j + 1] = ord[j];
          --j;
        }
        ord[j + 1] = v;
      }
      for (int i = 0; i < kvp; ++i)
        if (lse[ord[i]] != -INFINITY) z += __expf(lse[ord[i]] - m);
    }
    out_lse[b * q_heads + head] = m == -INFINITY ? m : m + logf(z);
  }
}

cudaError_t launch_merge_out(const float* frag_o, const float* frag_lse, int batch, int q_heads,
                             int q_per_slot, int kvp, int head_dim, int dp, float* out,
                             float* out_lse, int* bump_total, cudaStream_t stream) {
  if (kvp > kMaxKvp) return cudaErrorInvalidValue;
  const int warps = batch * q_heads;
  auto k = kvp <= 8 ? merge_out_kernel<8> : merge_out_kernel<kMaxKvp>;
  return launch_k(k, dim3((warps * 32 + 255) / 256), dim3(256), 0, stream, frag_o, frag_lse,
                  batch, q_heads, q_per_slot, kvp, head_dim, dp, out, out_lse, bump_total);
}

// ---------------------------------------------------------------- embedding
// x[b][:] = E[token_b][:] (bf16 -> fp32) with its x-fragments; one CTA per
// (128-column block, request), ss_part[blk][b] = sum of x^2 over the block --
// the same RMSNorm partials the residual epilogues write.
__global__ void embed_kernel(const __nv_bfloat16* emb, const int* tokens, int batch, int hidden,
                             float* x, float* ss_part, uint8_t* xf, int xf16) {
  griddep_wait();
  griddep_launch_dependents();
  const int nb = blockIdx.x, b = blockIdx.y;
  const int col = nb * 128 + threadIdx.x;
  float v = 0.f;
  if (col < hidden) {
    v = __bfloat162float(emb[static_cast<size_t>(tokens[b]) * hidden + col]);
    x[static_cast<size_t>(b) * hidden + col] = v;
    xf_write(xf, xf_nb8(batch), b, col, v, xf16);
  }
  float s = v * v;
  __shared__ float red[4];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) ss_part[static_cast<size_t>(nb) * batch + b] = (red[0] + red[1]) + (red[2] + red[3]);
}

cudaError_t launch_embed(const uint16_t* emb, const int* tokens, int batch, int hidden, float* x,
                         float* ss_part, uint8_t* xf, cudaStream_t stream, int xf16) {
  return launch_k(embed_kernel, dim3((hidden + 127) / 128, batch), dim3(128), 0, stream,
                  reinterpret_cast<const __nv_bfloat16*>(emb), tokens, batch, hidden, x, ss_part, xf, xf16);
}

__global__ void argmax_finish_kernel(const unsigned long long* best, int batch, int* tokens_out,
                                     unsigned long long* best_reset) {
  griddep_wait();
  griddep_launch_dependents();
  const int b = threadIdx.x;
  if (b < batch) {
    const unsigned long long k = best[b];
    tokens_out[b] = static_cast<int>(0xFFFFFFFFu - static_cast<unsigned>(k & 0xFFFFFFFFull));
    if (best_reset) best_reset[b] = 0ull;
  }
}

cudaError_t launch_argmax_finish(const unsigned long long* best, int batch, int* tokens_out,
                                 unsigned long long* best_reset, cudaStream_t stream) {
  return launch_k(argmax_finish_kernel, dim3(1), dim3(64), 0, stream, best, batch, tokens_out, best_reset);
}

// ---------------------------------------------------------------- KV scatter / fill
__device__ __forceinline__ uint8_t* kv_elem_ptr(uint8_t* kv, long long g, int b, int h, int d,
                                                int is_v, int batch, int kvh_per_slot, int kvp,
                                                int chunk, int dp, int page_cap, int slot_base,
                                                int n_local_slots, int fp8) {
  const int rank = rr_rank(g, chunk, kvp);
  const long long row = rr_row(g, chunk, kvp);
  const int grp = h / kvh_per_slot, kvh = h - grp * kvh_per_slot;
  const int slot_local = grp * kvp + rank - slot_base;
  if (slot_local < 0 || slot_local >= n_local_slots) return nullptr;
  const size_t page =
      ((static_cast<size_t>(slot_local) * batch + b) * kvh_per_slot + kvh) * page_cap +
      static_cast<size_t>(row >> 4);
  return kv + page * page_bytes_kv(dp, fp8) + kv_offset(dp, static_cast<int>(row & 15), d, is_v != 0, fp8);
}

// k_rows / v_rows: bf16 bits (2 bytes per element) or e4m3 codes (fp8 pages, 1 byte)
__global__ void kv_append_rows_kernel(uint8_t* kv, const void* k_rows, const void* v_rows,
                                      int n, int b, const int* total, int batch, int kv_heads,
                                      int kvh_per_slot, int kvp, int chunk, int head_dim, int dp,
                                      int page_cap, int slot_base, int n_local_slots, int fp8) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long per_tok = static_cast<long long>(kv_heads) * head_dim;
  if (idx >= n * per_tok) return;
  const int i = static_cast<int>(idx / per_tok);
  const int hd = static_cast<int>(idx - i * per_tok);
  const int h = hd / head_dim, d = hd - h * head_dim;
  const long long g = static_cast<long long>(total[b]) + i;
  uint8_t* pk = kv_elem_ptr(kv, g, b, h, d, 0, batch, kvh_per_slot, kvp, chunk, dp, page_cap,
                            slot_base, n_local_slots, fp8);
  if (!pk) return;
  uint8_t* pv = kv_elem_ptr(kv, g, b, h, d, 1, batch, kvh_per_slot, kvp, chunk, dp, page_cap,
                            slot_base, n_local_slots, fp8);
  if (fp8) {
    *pk = static_cast<const uint8_t*>(k_rows)[idx];
    *pv = static_cast<const uint8_t*>(v_rows)[idx];
  } else {
    *reinterpret_cast<uint16_t*>(pk) = static_cast<const uint16_t*>(k_rows)[idx];
    *reinterpret_cast<uint16_t*>(pv) = static_cast<const uint16_t*>(v_rows)[idx];
  }
}

__global__ void add_total_kernel(int* total, int b, int n) { total[b] += n; }

cudaError_t launch_kv_append_rows(uint8_t* kv, const void* k_rows, const void* v_rows,
                                  int n, int b, int* total, int batch, int kv_heads,
                                  int kvh_per_slot, int kvp, int chunk, int head_dim, int dp,
                                  int page_cap, int slot_base, int n_local_slots, int fp8,
                                  cudaStream_t stream) {
  const long long work = static_cast<long long>(n) * kv_heads * head_dim;
  if (work > 0) {
    kv_append_rows_kernel<<<static_cast<unsigned>((work + 255) / 256), 256, 0, stream>>>(
        kv, k_rows, v_rows, n, b, total, batch, kv_heads, kvh_per_slot, kvp, chunk, head_dim, dp,
        page_cap, slot_base, n_local_slots, fp8);
  }
  add_total_kernel<<<1, 1, 0, stream>>>(total, b, n);
  return cudaGetLastError();
}

// Hash fill: element (b, h, g, d) = hash_unit(seed, stream, ((b*K + h) << 32 + g) * Hsz + d)
// (layer_oracle.hpp ModelOracle::grow_hash). One warp per page of one stream
// (slot, request, kv head); each lane writes whole 16-byte chunks of the
// fragment-major page image (coalesced 512 B per warp store). Rows outside the
// new token range keep their old contents (read-modify-write on edge pages).
__device__ __forceinline__ long long rr_global_of_row(long long row, int rank, int chunk, int kvp) {
  return (row / chunk) * static_cast<long long>(chunk) * kvp + static_cast<long long>(rank) * chunk + row % chunk;
}

__device__ __forceinline__ double hash_kv_unit(uint64_t sseed, uint64_t index) {
  const uint64_t z = splitmix64(sseed + index);
  return 2.0 * (static_cast<double>(z >> 11) * 0x1.0p-53) - 1.0;
}
__device__ __forceinline__ uint16_t hash_bf16_bits(uint64_t sseed, uint64_t index) {
  const __nv_bfloat16 h = double_to_bf16_rne(hash_kv_unit(sseed, index));
  return *reinterpret_cast<const uint16_t*>(&h);
}

__global__ void kv_fill_hash_kernel(uint8_t* kv, const int* total, int batch, int kv_heads,
                                    int kvh_per_slot, int kvp, int chunk, int head_dim, int dp,
                                    int page_cap, int slot_base, int n_local_slots, long long n,
                                    uint64_t seed, uint64_t stream_k, uint64_t stream_v, int fp8) {
  const long long warp = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const long long streams = static_cast<long long>(n_local_slots) * batch * kvh_per_slot;
  if (warp >= streams * page_cap) return;
  const int page = static_cast<int>(warp % page_cap);
  const long long stream_idx = warp / page_cap;  // ((slot_local*B + b)*kvh_per_slot + kvh)
  long long st = stream_idx;
  const int kvh = static_cast<int>(st % kvh_per_slot);
  st /= kvh_per_slot;
  const int b = static_cast<int>(st % batch);
  const int slot = static_cast<int>(st / batch) + slot_base;
  const int rank = slot % kvp, grp = slot / kvp;
  const int h = grp * kvh_per_slot + kvh;
  const long long t0 = total[b], t1 = t0 + n;
  const long long gmin = rr_global_of_row(16ll * page, rank, chunk, kvp);
  const long long gmax = rr_global_of_row(16ll * page + 15, rank, chunk, kvp);
  if (gmax < t0 || gmin >= t1) return;
  const bool full = gmin >= t0 && gmax < t1;
  const uint64_t kseed = splitmix64(seed ^ (stream_k * 0xD1B54A32D192ED03ull));
  const uint64_t vseed = splitmix64(seed ^ (stream_v * 0xD1B54A32D192ED03ull));
  const uint64_t base = static_cast<uint64_t>(b * kv_heads + h) << 32;
  uint8_t* pg = kv + (static_cast<size_t>(stream_idx) * page_cap + page) * page_bytes_kv(dp, fp8);
  const int chunks = 64 * dp / 16;  // 8-element lane chunks per page (16 B bf16, 8 B fp8)
  for (int ci = lane; ci < chunks; ci += 32) {
    uint4* dst = reinterpret_cast<uint4*>(pg + ci * 16);
    uint2* dst8 = reinterpret_cast<uint2*>(pg + ci * 8);
    uint4 old = full ? make_uint4(0, 0, 0, 0) : (fp8 ? make_uint4(dst8->x, dst8->y, 0, 0) : *dst);
    uint16_t* ov = reinterpret_cast<uint16_t*>(&old);
    uint8_t* ov8 = reinterpret_cast<uint8_t*>(&old);
    // tensor-core FP8 layout (fp8 == 2, kv_layout.cuh kv8tc_offset): a chunk is
    // 8 dims of one token (K) or 8 tokens of one dim (V)
    const int tco = ci * 8 & 2047, tch = ci * 8 >> 11;
    const int is_v = fp8 == 2 ? tco >= 1024 : ci >= chunks / 2;
    const int cl = is_v ? ci - chunks / 2 : ci;
    const int ln = cl & 31, grpi = cl >> 5;
    const int g = ln >> 2, c = ln & 3;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      // e = sub*4 + half*2 + elem  (see kv_layout.cuh)
      const int sub = e >> 2, half = (e >> 1) & 1, elem = e & 1;
      int t, d;
      if (fp8 == 2) {
        if (!is_v) {
          t = tch * 8 + ((tco & 127) >> 4);
          d = (tco >> 7) * 16 + (tco & 15) + e;
        } else {
          t = tch * 8 + e;
          d = (tco - 1024) >> 3;
        }
      } else if (!is_v) {  // grpi = nt*(dp/32) + kp
        const int nt = grpi / (dp / 32), kp = grpi % (dp / 32);
        t = nt * 8 + g;
        d = (2 * kp + sub) * 16 + half * 8 + 2 * c + elem;
      } else {      // grpi = nd2
        const int nd = 2 * grpi + sub;
        d = nd * 8 + g;
        t = half * 8 + 2 * c + elem;
      }
      const long long gtok = rr_global_of_row(16ll * page + t, rank, chunk, kvp);
      if (gtok < t0 || gtok >= t1) continue;
      if (d >= head_dim) {
        if (fp8)
          ov8[e] = 0;
        else
          ov[e] = 0;
        continue;
      }
      const uint64_t index = (base + static_cast<uint64_t>(gtok)) * static_cast<uint64_t>(head_dim) +
                             static_cast<uint64_t>(d);
      if (fp8)
        ov8[e] = e4m3_from_double(hash_kv_unit(is_v ? vseed : kseed, index));
      else
        ov[e] = hash_bf16_bits(is_v ? vseed : kseed, index);
    }
    if (fp8)
      *dst8 = make_uint2(old.x, old.y);
    else
      *dst = old;
  }
}

__global__ void add_total_all_kernel(int* total, int batch, int n);

// FP4 pages (kv_layout.cuh kv4_*): one thread per (stream, page row t, K or V,
// 32-dim group) -- the e2m1 block. Values are the same hash doubles as the bf16
// fill, block-rounded exactly as the oracle (round_e2m1_block). K blocks own 16
// contiguous bytes (plain stores); a V byte pairs tokens t and t^1 (atomicOr:
// pages start zeroed and every position is written once).
__global__ void kv4_fill_hash_kernel(uint8_t* kv, const int* total, int batch, int kv_heads, int kvh_per_slot,
                                     int kvp, int chunk, int head_dim, int dp, int page_cap, int slot_base,
                                     int n_local_slots, long long n, uint64_t seed, uint64_t stream_k,
                                     uint64_t stream_v) {
  const int groups = dp / 32;
  long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long streams = static_cast<long long>(n_local_slots) * batch * kvh_per_slot;
  if (i >= streams * page_cap * 16 * 2 * groups) return;
  const int grp = static_cast<int>(i % groups);
  i /= groups;
  const int is_v = static_cast<int>(i % 2);
  i /= 2;
  const int t = static_cast<int>(i % 16);
  i /= 16;
  const int page = static_cast<int>(i % page_cap);
  const long long stream_idx = i / page_cap;
  long long st = stream_idx;
  const int kvh = static_cast<int>(st % kvh_per_slot);
  st /= kvh_per_slot;
  const int b = static_cast<int>(st % batch);
  const int slot = static_cast<int>(st / batch) + slot_base;
  const int rank = slot % kvp, grpi = slot / kvp;
  const int h = grpi * kvh_per_slot + kvh;
  const long long t0 = total[b];
  const long long gtok = rr_global_of_row(16ll * page + t, rank, chunk, kvp);
  if (gtok < t0 || gtok >= t0 + n) return;
  const uint64_t sseed = splitmix64(seed ^ ((is_v ? stream_v : stream_k) * 0xD1B54A32D192ED03ull));
  const uint64_t base = ((static_cast<uint64_t>(b * kv_heads + h) << 32) + static_cast<uint64_t>(gtok)) *
                        static_cast<uint64_t>(head_dim);
  double v[32];
  double am = 0.0;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const int d = grp * 32 + j;
    v[j] = d < head_dim ? hash_kv_unit(sseed, base + static_cast<uint64_t>(d)) : 0.0;
    am = fmax(am, fabs(v[j]));
  }
  const int ex = e2m1_block_exp(am);
  uint8_t* pg = kv + (static_cast<size_t>(stream_idx) * page_cap + page) * page_bytes_kv4(dp);
  uint32_t words[4] = {0u, 0u, 0u, 0u};
  uint32_t kbase = 0;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const int d = grp * 32 + j;
    bool high = false;
    const uint32_t off = kv4_offset(dp, t, d, is_v != 0, &high);
    const uint32_t nib = static_cast<uint32_t>(e2m1_from_double(v[j], ex)) << ((off & 3u) * 8u + (high ? 4u : 0u));
    if (is_v) {
      atomicOr(reinterpret_cast<unsigned*>(pg + (off & ~3u)), nib);
    } else {  // the block's 16 bytes are contiguous: 4 lane chunks of 4 bytes
      if (j == 0) kbase = off & ~15u;
      words[((off & ~3u) - kbase) >> 2] |= nib;
    }
  }
  if (!is_v) *reinterpret_cast<uint4*>(pg + kbase) = make_uint4(words[0], words[1], words[2], words[3]);
  pg[kv4_scale_offset(dp, t, grp * 32, is_v != 0)] = kv4_scale_byte(ex, is_v != 0);
}

cudaError_t launch_kv4_fill_hash(uint8_t* kv, int* total, int batch, int kv_heads, int kvh_per_slot, int kvp,
                                 int chunk, int head_dim, int dp, int page_cap, int slot_base, int n_local_slots,
                                 long long n, uint64_t seed, uint64_t stream_k, uint64_t stream_v,
                                 cudaStream_t stream) {
  const long long work = static_cast<long long>(n_local_slots) * batch * kvh_per_slot * page_cap * 16 * 2 * (dp / 32);
  if (n > 0)
    kv4_fill_hash_kernel<<<static_cast<unsigned>((work + 255) / 256), 256, 0, stream>>>(
        kv, total, batch, kv_heads, kvh_per_slot, kvp, chunk, head_dim, dp, page_cap, slot_base, n_local_slots, n,
        seed, stream_k, stream_v);
  add_total_all_kernel<<<1, 64, 0, stream>>>(total, batch, static_cast<int>(n));
  return cudaGetLastError();
}

// Host-quantized FP4 rows (codes [n][kv_heads][head_dim], block exponents
// [n][kv_heads][head_dim / 32] for K and V) into the pages of request b, tokens
// total[b] ..: one thread per (token, head, K/V, group).
__global__ void kv4_append_rows_kernel(uint8_t* kv, const uint8_t* codes_k, const uint8_t* codes_v,
                                       const int8_t* exp_k, const int8_t* exp_v, int n, int b, const int* total,
                                       int batch, int kv_heads, int kvh_per_slot, int kvp, int chunk, int head_dim,
                                       int dp, int page_cap, int slot_base, int n_local_slots) {
  const int groups = head_dim / 32;
  long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<long long>(n) * kv_heads * 2 * groups) return;
  const int grp = static_cast<int>(i % groups);
  i /= groups;
  const int is_v = static_cast<int>(i % 2);
  i /= 2;
  const int h = static_cast<int>(i % kv_heads);
  const int tok = static_cast<int>(i / kv_heads);
  const long long g = static_cast<long long>(total[b]) + tok;
  const int rank = rr_rank(g, chunk, kvp);
  const long long row = rr_row(g, chunk, kvp);
  const int grpi = h / kvh_per_slot, kvh = h - grpi * kvh_per_slot;
  const int slot_local = grpi * kvp + rank - slot_base;
  if (slot_local < 0 || slot_local >= n_local_slots) return;
  uint8_t* pg = kv + (((static_cast<size_t>(slot_local) * batch + b) * kvh_per_slot + kvh) * page_cap +
                      static_cast<size_t>(row >> 4)) * page_bytes_kv4(dp);
  const int t = static_cast<int>(row & 15);
  const uint8_t* codes = (is_v ? codes_v : codes_k) + (static_cast<size_t>(tok) * kv_heads + h) * head_dim;
  for (int j = 0; j < 32; ++j) {
    const int d = grp * 32 + j;
    bool high = false;
    const uint32_t off = kv4_offset(dp, t, d, is_v != 0, &high);
    atomicOr(reinterpret_cast<unsigned*>(pg + (off & ~3u)),
             static_cast<uint32_t>(codes[d]) << ((off & 3u) * 8u + (high ? 4u : 0u)));
  }
  const int8_t ex = (is_v ? exp_v : exp_k)[(static_cast<size_t>(tok) * kv_heads + h) * groups + grp];
  pg[kv4_scale_offset(dp, t, grp * 32, is_v != 0)] = kv4_scale_byte(ex, is_v != 0);
}

cudaError_t launch_kv4_append_rows(uint8_t* kv, const uint8_t* codes_k, const uint8_t* codes_v, const int8_t* exp_k,
                                   const int8_t* exp_v, int n, int b, int* total, int batch, int kv_heads,
                                   int kvh_per_slot, int kvp, int chunk, int head_dim, int dp, int page_cap,
                                   int slot_base, int n_local_slots, cudaStream_t stream) {
  const long long work = static_cast<long long>(n) * kv_heads * 2 * (head_dim / 32);
  if (work > 0)
    kv4_append_rows_kernel<<<static_cast<unsigned>((work + 255) / 256), 256, 0, stream>>>(
        kv, codes_k, codes_v, exp_k, exp_v, n, b, total, batch, kv_heads, kvh_per_slot, kvp, chunk, head_dim, dp,
        page_cap, slot_base, n_local_slots);
  add_total_kernel<<<1, 1, 0, stream>>>(total, b, n);
  return cudaGetLastError();
}

__global__ void add_total_all_kernel(int* total, int batch, int n) {
  for (int b = threadIdx.x; b < batch; b += blockDim.x) total[b] += n;
}

cudaError_t launch_kv_fill_hash(uint8_t* kv, int* total, int batch, int kv_heads,
                                int kvh_per_slot, int kvp, int chunk, int head_dim, int dp,
                                int page_cap, int slot_base, int n_local_slots, long long n,
                                uint64_t seed, uint64_t stream_k, uint64_t stream_v, int fp8,
                                cudaStream_t stream) {
  const long long work = static_cast<long long>(n_local_slots) * batch * kvh_per_slot * page_cap * 32;
  if (n > 0)
    kv_fill_hash_kernel<<<static_cast<unsigned>((work + 255) / 256), 256, 0, stream>>>(
        kv, total, batch, kv_heads, kvh_per_slot, kvp, chunk, head_dim, dp, page_cap, slot_base,
        n_local_slots, n, seed, stream_k, stream_v, fp8);
  add_total_all_kernel<<<1, 64, 0, stream>>>(total, batch, static_cast<int>(n));
  return cudaGetLastError();
}

// ---------------------------------------------------------------- weight init
// Element (n, k) of the combined [Npad x K] GEMV matrix (row n = output feature)
// at its fragment-major byte offset (see gemv.cu).
__host__ __device__ __forceinline__ size_t wfrag_offset(int n, int k, int kst) {
  const int nt = n >> 4, rn = n & 15, ks = k >> 4, rk = k & 15;
  const int g = rn & 7, rowhalf = rn >> 3;
  const int c = (rk & 7) >> 1, khalf = rk >> 3, elem = rk & 1;
  const int reg = khalf * 2 + rowhalf;
  const int lane = g * 4 + c;
  return ((static_cast<size_t>(nt) * kst + ks) * 32 + lane) * 16 + reg * 4 + elem * 2;
}

__device__ double wseg_value(const WSeg* segs, int nseg, int n, int k, uint64_t seed) {
  for (int s = 0; s < nseg; ++s) {
    const WSeg sg = segs[s];
    if (n < sg.rows_begin || n >= sg.rows_end) continue;
    int col;
    if (sg.interleave == 0) {
      col = sg.col_offset + (n - sg.rows_begin);
    } else {
      // SwiGLU: per 128-row block, rows [0,64) gate features, [64,128) up features
      const int blk = n >> 7, r = n & 127;
      if ((sg.interleave == 1) != (r < 64)) continue;
      col = sg.col_offset + blk * 64 + (r & 63);
      if (col >= sg.col_limit) return 0.0;
    }
    const uint64_t index = static_cast<uint64_t>(k + sg.k_offset) * static_cast<uint64_t>(sg.cols_total) +
                           static_cast<uint64_t>(col);
    return hash_unit(seed, sg.stream, index) * sg.scale;
  }
  return 0.0;
}

// One thread per 16-byte chunk (n-tile, k-step, lane) of the fragment-major image;
// tc: the tcgen05 GEMV's image instead -- per (row block, k-step) 4 KB of
// canonical K-major core matrices [row group 16][k-half 2][row 8][8 k] (gemv_tc.cu).
__global__ void weight_init_hash_kernel(uint4* w, int Npad, int K, const WSeg* segs, int nseg,
                                        uint64_t seed, int tc) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int kst = K >> 4;
  if (idx >= static_cast<long long>(Npad / 16) * kst * 32) return;
  // chunk index = ((nb * kst + ks) * 8 + ntl) * 32 + lane  (CTA-tile-major, see gemv.cu)
  const int lane = static_cast<int>(idx & 31);
  long long t = idx >> 5;
  const int ntl = static_cast<int>(t & 7);
  t >>= 3;
  const int ks = static_cast<int>(t % kst), nb = static_cast<int>(t / kst);
  const int nt = nb * 8 + ntl;
  const int g = lane >> 2, c = lane & 3;
  uint4 out;
  uint16_t* o = reinterpret_cast<uint16_t*>(&out);
  if (tc) {
    const int j = static_cast<int>(idx & 255);  // chunk within the (row block, k-step) 4 KB block
    const int n = nb * 128 + (j >> 4) * 8 + (j & 7);
    const int k0 = ks * 16 + ((j >> 3) & 1) * 8;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const __nv_bfloat16 h = double_to_bf16_rne(wseg_value(segs, nseg, n, k0 + e, seed));
      o[e] = *reinterpret_cast<const uint16_t*>(&h);
    }
    w[idx] = out;
    return;
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int reg = e >> 1, elem = e & 1;          // reg = khalf*2 + rowhalf
    const int rowhalf = reg & 1, khalf = reg >> 1;
    const int n = nt * 16 + rowhalf * 8 + g;
    const int k = ks * 16 + khalf * 8 + 2 * c + elem;
    const __nv_bfloat16 h = double_to_bf16_rne(wseg_value(segs, nseg, n, k, seed));
    o[e] = *reinterpret_cast<const uint16_t*>(&h);
  }
  w[idx] = out;
}

// FP8 weights: the same chunk order with 8 e4m3 bytes per chunk, value / scale[n].
__global__ void weight_init_hash_w8_kernel(uint2* w, int Npad, int K, const WSeg* segs, int nseg, uint64_t seed,
                                           const float* scale) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int kst = K >> 4;
  if (idx >= static_cast<long long>(Npad / 16) * kst * 32) return;
  const int lane = static_cast<int>(idx & 31);
  long long t = idx >> 5;
  const int ntl = static_cast<int>(t & 7);
  t >>= 3;
  const int ks = static_cast<int>(t % kst), nb = static_cast<int>(t / kst);
  const int nt = nb * 8 + ntl;
  const int g = lane >> 2, c = lane & 3;
  uint2 out;
  uint8_t* o = reinterpret_cast<uint8_t*>(&out);
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int reg = e >> 1, elem = e & 1;
    const int rowhalf = reg & 1, khalf = reg >> 1;
    const int n = nt * 16 + rowhalf * 8 + g;
    const int k = ks * 16 + khalf * 8 + 2 * c + elem;
    o[e] = e4m3_from_double(wseg_value(segs, nseg, n, k, seed) / static_cast<double>(scale[n]));
  }
  w[idx] = out;
}

// scale[n] = the smallest power of two >= max over the FULL input range of
// |W[k][n]| / 448 (oracle fp8_pow2_scale; k in [-k_offset, k_full - k_offset)
// of a tensor-parallel input shard), 1 for an all-zero row. One warp per row.
__global__ void weight_scale_hash_kernel(float* scale, int Npad, int k_full, const WSeg* segs, int nseg,
                                         uint64_t seed) {
  const int n = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (n >= Npad) return;
  int koff = 0;
  for (int s = 0; s < nseg; ++s)
    if (n >= segs[s].rows_begin && n < segs[s].rows_end) koff = segs[s].k_offset;
  double mx = 0.0;
  for (int k = lane; k < k_full; k += 32) mx = fmax(mx, fabs(wseg_value(segs, nseg, n, k - koff, seed)));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) {
    double sc = 1.0;
    if (mx > 0.0) {
      int e;
      const double f = frexp(mx / 448.0, &e);
      sc = ldexp(1.0, f == 0.5 ? e - 1 : e);
    }
    scale[n] = static_cast<float>(sc);
  }
}

cudaError_t launch_weight_init_hash_w8(uint8_t* w, float* scale, int Npad, int K, int k_full, const WSeg* segs,
                                       int nseg, uint64_t seed, cudaStream_t stream) {
  weight_scale_hash_kernel<<<static_cast<unsigned>((Npad + 7) / 8), 256, 0, stream>>>(scale, Npad, k_full, segs,
                                                                                     nseg, seed);
  const long long work = static_cast<long long>(Npad / 16) * (K / 16) * 32;
  weight_init_hash_w8_kernel<<<static_cast<unsigned>((work + 255) / 256), 256, 0, stream>>>(
      reinterpret_cast<uint2*>(w), Npad, K, segs, nseg, seed, scale);
  return cudaGetLastError();
}

// FP4 weights: one thread per (output row n, 32-input block): the block's 32
// values, its power-of-two scale (e2m1_block_exp: the oracle's round_e2m1_block)
// and 16 code bytes at their fragment positions (a byte holds elements k, k+1
// of one row: both nibbles from this thread) + the exponent byte.
__global__ void weight_init_hash_w4_kernel(uint8_t* w, int Npad, int K, const WSeg* segs, int nseg, uint64_t seed) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int kblocks = K >> 5;
  if (idx >= static_cast<long long>(Npad) * kblocks) return;
  const int n = static_cast<int>(idx % Npad), kb = static_cast<int>(idx / Npad);
  double v[32];
  double am = 0.0;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    v[i] = wseg_value(segs, nseg, n, kb * 32 + i, seed);
    am = fmax(am, fabs(v[i]));
  }
  const int ex = e2m1_block_exp(am);
  const int nb = n >> 7, r = n & 127, warp = r >> 4, rr = r & 15, g = rr & 7, rowhalf = rr >> 3;
  uint8_t* blk = w + (static_cast<size_t>(nb) * kblocks + kb) * 2176;
#pragma unroll
  for (int i = 0; i < 32; i += 2) {  // k = 32 kb + i: (k-step half, khalf, c) ; elements i, i+1 share a byte
    const int sub = i >> 4, kk = i & 15, khalf = kk >> 3, c = (kk & 7) >> 1;
    const int lane = g * 4 + c, reg = khalf * 2 + rowhalf;
    blk[sub * 1024 + warp * 128 + lane * 4 + reg] =
        static_cast<uint8_t>(e2m1_from_double(v[i], ex) | (e2m1_from_double(v[i + 1], ex) << 4));
  }
  blk[2048 + r] = static_cast<uint8_t>(ex + 15);
}

cudaError_t launch_weight_init_hash_w4(uint8_t* w, int Npad, int K, const WSeg* segs, int nseg, uint64_t seed,
                                       cudaStream_t stream) {
  const long long work = static_cast<long long>(Npad) * (K / 32);
  weight_init_hash_w4_kernel<<<static_cast<unsigned>((work + 255) / 256), 256, 0, stream>>>(w, Npad, K, segs, nseg,
                                                                                           seed);
  return cudaGetLastError();
}

cudaError_t launch_weight_init_hash(uint4* w, int Npad, int K, const WSeg* segs, int nseg,
                                    uint64_t seed, cudaStream_t stream, int tc) {
  const long long work = static_cast<long long>(Npad / 16) * (K / 16) * 32;
  weight_init_hash_kernel<<<static_cast<unsigned>((work + 255) / 256), 256, 0, stream>>>(
      w, Npad, K, segs, nseg, seed, tc);
  return cudaGetLastError();
}

// Plain row-major bf16 array: w[i] = bf16(hash_unit(seed, stream, idx0 + i) * scale).
__global__ void plain_init_hash_kernel(__nv_bfloat16* w, long long n, uint64_t seed, uint64_t stream_id,
                                       long long idx0, double scale) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= n) return;
  w[idx] = double_to_bf16_rne(hash_unit(seed, stream_id, static_cast<uint64_t>(idx0 + idx)) * scale);
}

cudaError_t launch_plain_init_hash(uint16_t* w, long long n, uint64_t seed, uint64_t stream_id, long long idx0,
                                   double scale, cudaStream_t stream) {
  plain_init_hash_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(
      reinterpret_cast<__nv_bfloat16*>(w), n, seed, stream_id, idx0, scale);
  return cudaGetLastError();
}

cudaError_t launch_emb_init_hash(uint16_t* emb, int vocab, int hidden, uint64_t seed,
                                 uint64_t stream_id, cudaStream_t stream) {
  return launch_plain_init_hash(emb, static_cast<long long>(vocab) * hidden, seed, stream_id, 0, 1.0, stream);
}

cudaError_t launch_fill_zero(void* p, size_t bytes, cudaStream_t stream) {
  return cudaMemsetAsync(p, 0, bytes, stream);
}

}  // namespace hx

// ---------------------------------------------------------------- loopback reductions (comm.h)
namespace hx {
__global__ void sum_buffers_kernel(const float* const* srcs, int n, float* dst, size_t count) {
  const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= count) return;
  float s = 0.f;
  for (int r = 0; r < n; ++r) s += srcs[r][i];  // rank order: deterministic, identical on every rank
  dst[i] = s;
}
__global__ void max_u64_buffers_kernel(const unsigned long long* const* srcs, int n, unsigned long long* dst,
                                       size_t count) {
  const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= count) return;
  unsigned long long m = 0;
  for (int r = 0; r < n; ++r) m = srcs[r][i] > m ? srcs[r][i] : m;
  dst[i] = m;
}
cudaError_t launch_sum_buffers(const float* const* srcs, int n, float* dst, size_t count, cudaStream_t s) {
  sum_buffers_kernel<<<static_cast<unsigned>((count + 255) / 256), 256, 0, s>>>(srcs, n, dst, count);
  return cudaGetLastError();
}
cudaError_t launch_max_u64_buffers(const unsigned long long* const* srcs, int n, unsigned long long* dst,
                                   size_t count, cudaStream_t s) {
  max_u64_buffers_kernel<<<static_cast<unsigned>((count + 255) / 256), 256, 0, s>>>(srcs, n, dst, count);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- Helix fragment exchange (pack side)
// send[p][b][0:slice]           = this rank's fragment elements [p*slice, (p+1)*slice) of its
//                                 group's flattened (heads x head_dim) output (attention.hpp:495-502)
// send[p][b][slice:slice+nh_p]  = lse of the heads that slice touches
__global__ void pack_exchange_kernel(const float* frag_o, const float* frag_lse, int b_begin, int b_count,
                                     int batch, int q_per_slot, int head_dim, int dp, int kvp, int slice,
                                     int chunk, float* send) {
  griddep_wait();
  griddep_launch_dependents();
  const int per_req = slice + (chunk - slice);
  const long long total = static_cast<long long>(kvp) * b_count * per_req;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int e = static_cast<int>(i % per_req);
    const long long t = i / per_req;
    const int bl = static_cast<int>(t % b_count), p = static_cast<int>(t / b_count);
    const int b = b_begin + bl;
    const int first_head = (p * slice) / head_dim;
    const int last_head = ((p + 1) * slice - 1) / head_dim;
    float v = 0.f;
    if (e < slice) {
      const int flat = p * slice + e;
      const int head = flat / head_dim, d = flat - head * head_dim;
      v = frag_o[(static_cast<size_t>(b) * q_per_slot + head) * dp + d];
    } else if (e - slice <= last_head - first_head) {
      v = frag_lse[static_cast<size_t>(b) * q_per_slot + first_head + (e - slice)];
    }
    send[(static_cast<size_t>(p) * batch + b) * chunk + e] = v;
  }
}
cudaError_t launch_pack_exchange(const float* frag_o, const float* frag_lse, int b_begin, int b_count, int batch,
                                 int q_per_slot, int head_dim, int dp, int kvp, int slice, int chunk, float* send,
                                 cudaStream_t s) {
  const long long total = static_cast<long long>(kvp) * b_count * chunk;
  const int blocks = static_cast<int>(std::min<long long>((total + 255) / 256, 1024));
  return launch_k(pack_exchange_kernel, dim3(blocks), dim3(256), 0, s, frag_o, frag_lse, b_begin, b_count, batch,
                  q_per_slot, head_dim, dp, kvp, slice, chunk, send);
}

// Receive side of the device-initiated exchange: one CTA waits until every
// peer's attention kernel has raised its flag (system-scope acquire), then
// lowers it for the next layer. The merge that follows reads the pushed slices.
__global__ void wait_flags_kernel(unsigned* flags, int n, long long max_spin) {
  griddep_wait();  // after this rank's own attention: never holds an SM the attention needs
  griddep_launch_dependents();
  const int i = threadIdx.x;
  if (i >= n) return;
  unsigned v = 0;
  for (long long it = 0;; ++it) {
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + i) : "memory");
    if (v) break;
    if (max_spin > 0 && it == max_spin)  // HX_DEBUG_WAIT: report a long wait (keeps waiting)
      printf("wait_flags: flag %d of %d (%p) not raised after %lld polls\n", i, n, flags + i, it);
    __nanosleep(64);
  }
  flags[i] = 0u;
}
cudaError_t launch_wait_flags(unsigned* flags, int n, cudaStream_t s) {
  static const long long max_spin = std::getenv("HX_DEBUG_WAIT") ? std::atoll(std::getenv("HX_DEBUG_WAIT")) : 0;
  return launch_k(wait_flags_kernel, dim3(1), dim3(32 * ((n + 31) / 32)), 0, s, flags, n, max_spin);
}

// x[b][n] += part[b][n]; ss_part[blk][b] = sum over the 128-column block of x^2 (deterministic).
__global__ void residual_add_kernel(float* x, const float* part, int batch, int hidden, float* ss_part,
                                    uint8_t* xf, int xf16) {
  griddep_wait();
  griddep_launch_dependents();
  const int blk = blockIdx.x, b = blockIdx.y;
  const int n = blk * 128 + threadIdx.x;
  float v = 0.f;
  if (n < hidden) {
    v = x[static_cast<size_t>(b) * hidden + n] + part[static_cast<size_t>(b) * hidden + n];
    x[static_cast<size_t>(b) * hidden + n] = v;
    xf_write(xf, xf_nb8(batch), b, n, v, xf16);
  }
  float s = v * v;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ float red[4];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) ss_part[static_cast<size_t>(blk) * batch + b] = (red[0] + red[1]) + (red[2] + red[3]);
}
cudaError_t launch_residual_add(float* x, const float* part, int batch, int hidden, float* ss_part,
                                uint8_t* xf, cudaStream_t s, int xf16) {
  return launch_k(residual_add_kernel, dim3((hidden + 127) / 128, batch), dim3(128), 0, s, x, part, batch, hidden,
                  ss_part, xf, xf16);
}
}  // namespace hx

// ---------------------------------------------------------------- x-fragment producers
namespace hx {
__global__ void xprep_plain_kernel(const float* x, int batch, int K, int x_stride, uint8_t* xf, int xf16) {
  griddep_wait();
  griddep_launch_dependents();
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<long long>(batch) * K) return;
  const int b = static_cast<int>(i / K), k = static_cast<int>(i % K);
  xf_write(xf, xf_nb8(batch), b, k, x[static_cast<size_t>(b) * x_stride + k], xf16);
}
cudaError_t launch_xprep_plain(const float* x, int batch, int K, int x_stride, uint8_t* xf, cudaStream_t s,
                               int xf16) {
  const long long n = static_cast<long long>(batch) * K;
  return launch_k(xprep_plain_kernel, dim3(static_cast<unsigned>((n + 255) / 256)), dim3(256), 0, s, x, batch, K,
                  x_stride, xf, xf16);
}


template <int MAXK>
__global__ void xprep_merge_local_kernel(const float* frag_o, const float* frag_lse, int batch, int q_per_slot,
                                         int kvp, int head_dim, int dp, int K, uint8_t* xf, int* bump_total,
                                         float* plain, int xf16) {
  griddep_wait();
  griddep_launch_dependents();
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  // the attention of this layer has read its token totals: the appended token now counts
  if (bump_total && i < batch) bump_total[i] += 1;
  if (i >= static_cast<long long>(batch) * K) return;
  const int b = static_cast<int>(i / K), k = static_cast<int>(i % K);
  const int head = k / head_dim, d = k - head * head_dim;
  const int grp = head / q_per_slot, qi = head - grp * q_per_slot;
  float lse[MAXK], o[MAXK];
#pragma unroll
  for (int r = 0; r < MAXK; ++r) {
    if (r < kvp) {
      const size_t f = (static_cast<size_t>(grp * kvp + r) * batch + b) * q_per_slot + qi;
      lse[r] = frag_lse[f];
      o[r] = frag_o[f * dp + d];
    }
  }
  const float v = merge_sources<MAXK>(lse, o, kvp);
  if (plain)
    plain[i] = v;
  else
    xf_write(xf, xf_nb8(batch), b, k, v, xf16);
}
cudaError_t launch_xprep_merge_local(const float* frag_o, const float* frag_lse, int batch, int q_per_slot,
                                     int kvp, int head_dim, int dp, int K, uint8_t* xf, int* bump_total,
                                     cudaStream_t s, float* plain, int xf16) {
  if (kvp > kMaxKvp) return cudaErrorInvalidValue;
  const long long n = static_cast<long long>(batch) * K;
  return launch_k(kvp <= 8 ? xprep_merge_local_kernel<8> : xprep_merge_local_kernel<kMaxKvp>, dim3(static_cast<unsigned>((n + 255) / 256)), dim3(256), 0, s, frag_o,
                  frag_lse, batch, q_per_slot, kvp, head_dim, dp, K, xf, bump_total, plain, xf16);
}

template <int MAXK>
__global__ void xprep_merge_recv_kernel(const float* recv, int batch, int kvp, int chunk, int slice, int exch_rank,
                                        int head_dim, uint8_t* xf, int* bump_total, float* plain, int xf16) {
  griddep_wait();
  griddep_launch_dependents();
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (bump_total && i < batch) bump_total[i] += 1;
  if (i >= static_cast<long long>(batch) * slice) return;
  const int b = static_cast<int>(i / slice), k = static_cast<int>(i % slice);
  const int first = (exch_rank * slice) / head_dim;
  const int head = (exch_rank * slice + k) / head_dim;
  float lse[MAXK], o[MAXK];
#pragma unroll
  for (int r = 0; r < MAXK; ++r) {
    if (r < kvp) {
      const float* src = recv + (static_cast<size_t>(r) * batch + b) * chunk;
      lse[r] = src[slice + head - first];
      o[r] = src[k];
    }
  }
  const float v = merge_sources<MAXK>(lse, o, kvp);
  if (plain)
    plain[i] = v;
  else
    xf_write(xf, xf_nb8(batch), b, k, v, xf16);
}
cudaError_t launch_xprep_merge_recv(const float* recv, int batch, int kvp, int chunk, int slice, int exch_rank,
                                    int head_dim, uint8_t* xf, int* bump_total, cudaStream_t s, float* plain,
                                    int xf16) {
  if (kvp > kMaxKvp) return cudaErrorInvalidValue;
  const long long n = static_cast<long long>(batch) * slice;
  return launch_k(kvp <= 8 ? xprep_merge_recv_kernel<8> : xprep_merge_recv_kernel<kMaxKvp>, dim3(static_cast<unsigned>((n + 255) / 256)), dim3(256), 0, s, recv,
                  batch, kvp, chunk, slice, exch_rank, head_dim, xf, bump_total, plain, xf16);
}
}  // namespace hx

// ---------------------------------------------------------------- MoE routing
namespace hx {
// One warp per request: its logits live in registers (lane holds experts
// lane, lane+32, ...; E <= 32 * kRouteSlots), k rounds of warp argmax (ties: lower
// index) knock the winner out in place; softmax over the selected; then warp 0
// compacts the ascending list of active local experts with ballots.
constexpr int kRouteSlots = 16;
__global__ void moe_route_kernel(const float* logits, int batch, int n_experts, int top_k, int e_begin, int e_end,
                                 float* route_w, int* group_ids, int* group_count) {
  griddep_wait();
  griddep_launch_dependents();
  extern __shared__ int s_flag[];  // [n_experts]
  for (int i = threadIdx.x; i < n_experts; i += blockDim.x) s_flag[i] = 0;
  for (int i = threadIdx.x; i < batch * n_experts; i += blockDim.x) route_w[i] = 0.f;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int b = warp; b < batch; b += nw) {
    const float* r = logits + static_cast<size_t>(b) * n_experts;
    float v[kRouteSlots];
#pragma unroll
    for (int i = 0; i < kRouteSlots; ++i) {
      const int e = lane + 32 * i;
      v[i] = e < n_experts ? r[e] : -INFINITY;
    }
    float sel_v = 0.f, top = 0.f, z = 0.f;
    int sel_i = 0;
    for (int k = 0; k < top_k; ++k) {
      float bv = -INFINITY;
      int bi = 0x7fffffff;
#pragma unroll
      for (int i = 0; i < kRouteSlots; ++i) {
        const int e = lane + 32 * i;
        if (e < n_experts && (v[i] > bv || (v[i] == bv && e < bi))) {
          bv = v[i];
          bi = e;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      if ((bi & 31) == lane) {  // knock the winner out (its owning lane, static slot index)
#pragma unroll
        for (int i = 0; i < kRouteSlots; ++i)
          if (i == (bi >> 5)) v[i] = -INFINITY;
      }
      if (k == 0) top = bv;
      z += expf(bv - top);  // same order as the oracle's sum over the selected
      if (lane == k) {      // lane k keeps the k-th selection
        sel_v = bv;
        sel_i = bi;
      }
    }
    if (lane < top_k) {
      route_w[static_cast<size_t>(b) * n_experts + sel_i] = expf(sel_v - top) / z;
      s_flag[sel_i] = 1;
    }
  }
  __syncthreads();
  if (warp == 0) {  // ascending list of active local experts
    int c = 0;
    for (int e0 = e_begin; e0 < e_end; e0 += 32) {
      const int e = e0 + lane;
      const bool on = e < e_end && s_flag[e];
      const unsigned m = __ballot_sync(0xffffffffu, on);
      if (on) group_ids[c + __popc(m & ((1u << lane) - 1u))] = e;
      c += __popc(m);
    }
    if (lane == 0) *group_count = c;
  }
}
cudaError_t launch_moe_route(const float* logits, int batch, int n_experts, int top_k, int e_begin, int e_end,
                             float* route_w, int* group_ids, int* group_count, cudaStream_t s) {
  if (top_k > 16 || n_experts > 32 * kRouteSlots) return cudaErrorInvalidValue;
  return launch_k(moe_route_kernel, dim3(1), dim3(512), static_cast<size_t>(n_experts) * sizeof(int), s, logits,
                  batch, n_experts, top_k, e_begin, e_end, route_w, group_ids, group_count);
}
}  // namespace hx
