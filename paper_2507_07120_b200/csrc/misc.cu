// Small kernels around the decode step: fragment merge for the attention-only
// harness output, embedding gather, greedy-token finish, KV scatter/fill into
// the round-robin page pool, and hash-RNG weight init directly into the
// fragment-major layout (values identical to oracle/layer_oracle.hpp).
#include "common.cuh"
#include "kernels.h"
#include "kv_layout.cuh"

namespace hx {

// ---------------------------------------------------------------- merge (harness output)
// out[b][head][d] = canonical LSE merge over kvp rank fragments
// (merge_fragments / merge_head_fragments, attention.hpp:118-175).
__global__ void merge_out_kernel(const float* frag_o, const float* frag_lse, int batch,
                                 int q_heads, int q_per_slot, int kvp, int head_dim, int dp,
                                 float* out, float* out_lse) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= batch * q_heads) return;
  const int b = warp / q_heads, head = warp - b * q_heads;
  const int grp = head / q_per_slot, qi = head - grp * q_per_slot;
  float lse[8];
  int ord[8];
  for (int r = 0; r < kvp; ++r) {
    lse[r] = frag_lse[(static_cast<size_t>(grp * kvp + r) * batch + b) * q_per_slot + qi];
    ord[r] = r;
  }
  for (int i = 1; i < kvp; ++i) {
    const int o = ord[i];
    int j = i - 1;
    while (j >= 0 && lse[ord[j]] < lse[o]) {
      ord[j + 1] = ord[j];
      --j;
    }
    ord[j + 1] = o;
  }
  const float m = lse[ord[0]];
  float z = 0.f;
  for (int i = 0; i < kvp; ++i)
    if (lse[ord[i]] != -INFINITY) z += expf(lse[ord[i]] - m);
  for (int d = lane; d < head_dim; d += 32) {
    float acc = 0.f;
    for (int i = 0; i < kvp; ++i) {
      const int r = ord[i];
      if (lse[r] == -INFINITY) continue;
      const float w = expf(lse[r] - m);
      acc += w * frag_o[((static_cast<size_t>(grp * kvp + r) * batch + b) * q_per_slot + qi) * dp + d];
    }
    out[(static_cast<size_t>(b) * q_heads + head) * head_dim + d] = m == -INFINITY ? 0.f : acc / z;
  }
  if (lane == 0 && out_lse) out_lse[b * q_heads + head] = m == -INFINITY ? m : m + logf(z);
}

cudaError_t launch_merge_out(const float* frag_o, const float* frag_lse, int batch, int q_heads,
                             int q_per_slot, int kvp, int head_dim, int dp, float* out,
                             float* out_lse, cudaStream_t stream) {
  const int warps = batch * q_heads;
  merge_out_kernel<<<(warps * 32 + 255) / 256, 256, 0, stream>>>(
      frag_o, frag_lse, batch, q_heads, q_per_slot, kvp, head_dim, dp, out, out_lse);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- embedding
// x[b][:] = E[token_b][:] (bf16 -> fp32); ss_part[0][b] = sum x^2.
__global__ void embed_kernel(const __nv_bfloat16* emb, const int* tokens, int batch, int hidden,
                             float* x, float* ss_part) {
  const int b = blockIdx.x;
  const int tok = tokens[b];
  float s = 0.f;
  for (int i = threadIdx.x; i < hidden; i += blockDim.x) {
    const float v = __bfloat162float(emb[static_cast<size_t>(tok) * hidden + i]);
    x[static_cast<size_t>(b) * hidden + i] = v;
    s += v * v;
  }
  __shared__ float red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) ss_part[b] = s;
  }
}

cudaError_t launch_embed(const uint16_t* emb, const int* tokens, int batch, int hidden, float* x,
                         float* ss_part, cudaStream_t stream) {
  embed_kernel<<<batch, 256, 0, stream>>>(reinterpret_cast<const __nv_bfloat16*>(emb), tokens,
                                          batch, hidden, x, ss_part);
  return cudaGetLastError();
}

__global__ void argmax_finish_kernel(const unsigned long long* best, int batch, int* tokens_out,
                                     unsigned long long* best_reset) {
  const int b = threadIdx.x;
  if (b < batch) {
    const unsigned long long k = best[b];
    tokens_out[b] = static_cast<int>(0xFFFFFFFFu - static_cast<unsigned>(k & 0xFFFFFFFFull));
    if (best_reset) best_reset[b] = 0ull;
  }
}

cudaError_t launch_argmax_finish(const unsigned long long* best, int batch, int* tokens_out,
                                 unsigned long long* best_reset, cudaStream_t stream) {
  argmax_finish_kernel<<<1, 32, 0, stream>>>(best, batch, tokens_out, best_reset);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- KV scatter / fill
__device__ __forceinline__ uint8_t* kv_elem_ptr(uint8_t* kv, long long g, int b, int h, int d,
                                                int is_v, int batch, int kvh_per_slot, int kvp,
                                                int chunk, int dp, int page_cap, int slot_base,
                                                int n_local_slots) {
  const int rank = rr_rank(g, chunk, kvp);
  const long long row = rr_row(g, chunk, kvp);
  const int grp = h / kvh_per_slot, kvh = h - grp * kvh_per_slot;
  const int slot_local = grp * kvp + rank - slot_base;
  if (slot_local < 0 || slot_local >= n_local_slots) return nullptr;
  const size_t page =
      ((static_cast<size_t>(slot_local) * batch + b) * kvh_per_slot + kvh) * page_cap +
      static_cast<size_t>(row >> 4);
  const uint32_t off = is_v ? v_offset(dp, static_cast<int>(row & 15), d)
                            : k_offset(dp, static_cast<int>(row & 15), d);
  return kv + page * page_bytes(dp) + off;
}

__global__ void kv_append_rows_kernel(uint8_t* kv, const uint16_t* k_rows, const uint16_t* v_rows,
                                      int n, int b, const int* total, int batch, int kv_heads,
                                      int kvh_per_slot, int kvp, int chunk, int head_dim, int dp,
                                      int page_cap, int slot_base, int n_local_slots) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long per_tok = static_cast<long long>(kv_heads) * head_dim;
  if (idx >= n * per_tok) return;
  const int i = static_cast<int>(idx / per_tok);
  const int hd = static_cast<int>(idx - i * per_tok);
  const int h = hd / head_dim, d = hd - h * head_dim;
  const long long g = static_cast<long long>(total[b]) + i;
  uint8_t* pk = kv_elem_ptr(kv, g, b, h, d, 0, batch, kvh_per_slot, kvp, chunk, dp, page_cap,
                            slot_base, n_local_slots);
  if (!pk) return;
  uint8_t* pv = kv_elem_ptr(kv, g, b, h, d, 1, batch, kvh_per_slot, kvp, chunk, dp, page_cap,
                            slot_base, n_local_slots);
  *reinterpret_cast<uint16_t*>(pk) = k_rows[idx];
  *reinterpret_cast<uint16_t*>(pv) = v_rows[idx];
}

__global__ void add_total_kernel(int* total, int b, int n) { total[b] += n; }

cudaError_t launch_kv_append_rows(uint8_t* kv, const uint16_t* k_rows, const uint16_t* v_rows,
                                  int n, int b, int* total, int batch, int kv_heads,
                                  int kvh_per_slot, int kvp, int chunk, int head_dim, int dp,
                                  int page_cap, int slot_base, int n_local_slots,
                                  cudaStream_t stream) {
  const long long work = static_cast<long long>(n) * kv_heads * head_dim;
  if (work > 0) {
    kv_append_rows_kernel<<<static_cast<unsigned>((work + 255) / 256), 256, 0, stream>>>(
        kv, k_rows, v_rows, n, b, total, batch, kv_heads, kvh_per_slot, kvp, chunk, head_dim, dp,
        page_cap, slot_base, n_local_slots);
  }
  add_total_kernel<<<1, 1, 0, stream>>>(total, b, n);
  return cudaGetLastError();
}

// Hash fill: element (b, h, g, d) = hash_unit(seed, stream, ((b*K + h) << 32 + g) * Hsz + d)
// (layer_oracle.hpp ModelOracle::grow_hash). One thread per (b, h, g, 8 dims).
__global__ void kv_fill_hash_kernel(uint8_t* kv, const int* total, int batch, int kv_heads,
                                    int kvh_per_slot, int kvp, int chunk, int head_dim, int dp,
                                    int page_cap, int slot_base, int n_local_slots, long long n,
                                    uint64_t seed, uint64_t stream_k, uint64_t stream_v) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int dgroups = (head_dim + 7) / 8;
  const long long per_b = static_cast<long long>(kv_heads) * n * dgroups;
  if (idx >= per_b * batch) return;
  const int b = static_cast<int>(idx / per_b);
  long long r = idx - b * per_b;
  const int h = static_cast<int>(r / (n * dgroups));
  r -= static_cast<long long>(h) * n * dgroups;
  const long long i = r / dgroups;
  const int dg = static_cast<int>(r - i * dgroups);
  const long long g = static_cast<long long>(total[b]) + i;
  const uint64_t kseed = splitmix64(seed ^ (stream_k * 0xD1B54A32D192ED03ull));
  const uint64_t vseed = splitmix64(seed ^ (stream_v * 0xD1B54A32D192ED03ull));
  for (int d = dg * 8; d < min(head_dim, dg * 8 + 8); ++d) {
    const uint64_t index =
        ((static_cast<uint64_t>(b * kv_heads + h) << 32) + static_cast<uint64_t>(g)) *
            static_cast<uint64_t>(head_dim) + static_cast<uint64_t>(d);
    const uint64_t zk = splitmix64(kseed + index);
    const uint64_t zv = splitmix64(vseed + index);
    const double uk = 2.0 * (static_cast<double>(zk >> 11) * 0x1.0p-53) - 1.0;
    const double uv = 2.0 * (static_cast<double>(zv >> 11) * 0x1.0p-53) - 1.0;
    uint8_t* pk = kv_elem_ptr(kv, g, b, h, d, 0, batch, kvh_per_slot, kvp, chunk, dp, page_cap,
                              slot_base, n_local_slots);
    if (!pk) continue;
    uint8_t* pv = kv_elem_ptr(kv, g, b, h, d, 1, batch, kvh_per_slot, kvp, chunk, dp, page_cap,
                              slot_base, n_local_slots);
    *reinterpret_cast<__nv_bfloat16*>(pk) = double_to_bf16_rne(uk);
    *reinterpret_cast<__nv_bfloat16*>(pv) = double_to_bf16_rne(uv);
  }
}

__global__ void add_total_all_kernel(int* total, int batch, int n) {
  const int b = threadIdx.x;
  if (b < batch) total[b] += n;
}

cudaError_t launch_kv_fill_hash(uint8_t* kv, int* total, int batch, int kv_heads,
                                int kvh_per_slot, int kvp, int chunk, int head_dim, int dp,
                                int page_cap, int slot_base, int n_local_slots, long long n,
                                uint64_t seed, uint64_t stream_k, uint64_t stream_v,
                                cudaStream_t stream) {
  const long long work = static_cast<long long>(batch) * kv_heads * n * ((head_dim + 7) / 8);
  if (work > 0)
    kv_fill_hash_kernel<<<static_cast<unsigned>((work + 255) / 256), 256, 0, stream>>>(
        kv, total, batch, kv_heads, kvh_per_slot, kvp, chunk, head_dim, dp, page_cap, slot_base,
        n_local_slots, n, seed, stream_k, stream_v);
  add_total_all_kernel<<<1, 32, 0, stream>>>(total, batch, static_cast<int>(n));
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

__global__ void weight_init_hash_kernel(uint8_t* w, int Npad, int K, const WSeg* segs, int nseg,
                                        uint64_t seed) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<long long>(Npad) * K) return;
  const int n = static_cast<int>(idx / K), k = static_cast<int>(idx - static_cast<long long>(n) * K);
  double v = 0.0;
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
      col = blk * 64 + (r & 63);
      if (col >= sg.cols_total) continue;
    }
    const uint64_t index = static_cast<uint64_t>(k) * static_cast<uint64_t>(sg.cols_total) +
                           static_cast<uint64_t>(col);
    v = hash_unit(seed, sg.stream, index) * sg.scale;
    break;
  }
  *reinterpret_cast<__nv_bfloat16*>(w + wfrag_offset(n, k, K >> 4)) = double_to_bf16_rne(v);
}

cudaError_t launch_weight_init_hash(uint4* w, int Npad, int K, const WSeg* segs, int nseg,
                                    uint64_t seed, cudaStream_t stream) {
  const long long work = static_cast<long long>(Npad) * K;
  weight_init_hash_kernel<<<static_cast<unsigned>((work + 255) / 256), 256, 0, stream>>>(
      reinterpret_cast<uint8_t*>(w), Npad, K, segs, nseg, seed);
  return cudaGetLastError();
}

__global__ void emb_init_hash_kernel(__nv_bfloat16* emb, int vocab, int hidden, uint64_t seed,
                                     uint64_t stream_id) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<long long>(vocab) * hidden) return;
  emb[idx] = double_to_bf16_rne(hash_unit(seed, stream_id, static_cast<uint64_t>(idx)));
}

cudaError_t launch_emb_init_hash(uint16_t* emb, int vocab, int hidden, uint64_t seed,
                                 uint64_t stream_id, cudaStream_t stream) {
  const long long work = static_cast<long long>(vocab) * hidden;
  emb_init_hash_kernel<<<static_cast<unsigned>((work + 255) / 256), 256, 0, stream>>>(
      reinterpret_cast<__nv_bfloat16*>(emb), vocab, hidden, seed, stream_id);
  return cudaGetLastError();
}

cudaError_t launch_fill_zero(void* p, size_t bytes, cudaStream_t stream) {
  return cudaMemsetAsync(p, 0, bytes, stream);
}

}  // namespace hx
