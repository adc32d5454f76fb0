// Exact (fp64) harness path: the reference's DecodeHarness<double> /
// free-function numerics (attention.hpp:35-175, 375-396, 460-539) on the GPU
// in double precision, for the drop-in C++ API (include/helixsim/exact_b200.hpp)
// whose callers hold the reference's 1e-10 / 1e-12 tolerances. This is the
// numerics-preserving mirror of the harness, not the decode hot path (that is
// attention.cu / mla.cu on bf16 pages); it keeps the KV cache device-resident
// in plain row-major fp64 shards: [slot][request][kv head][row][width].
#include <cmath>

#include "common.cuh"
#include "kernels.h"
#include "kv_layout.cuh"

namespace hx {

namespace {

constexpr int kF64Warps = 8;
constexpr int kF64MaxPerLane = kF64MaxWidth / 32;

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Online softmax state of one warp: lanes hold dims lane, lane+32, ...
struct F64State {
  double m, z;
  double acc[kF64MaxPerLane];
};

// Stream rows [0, n) of one K/V segment (row-major, `w` wide) through warp
// `warp` of `nwarps` (rows warp, warp+nwarps, ...). sq: the query in shared
// memory; logit = (K_t . q) * scale (attention.hpp:49-50).
__device__ __forceinline__ void f64_rows(const double* sq, int w, const double* K, const double* V, long long n,
                                         double scale, int warp, int nwarps, F64State& st) {
  const int lane = threadIdx.x & 31;
  for (long long t = warp; t < n; t += nwarps) {
    const double* kr = K + t * w;
    const double* vr = V + t * w;
    double d = 0.0;
    for (int i = lane; i < w; i += 32) d += kr[i] * sq[i];
    const double logit = warp_sum_d(d) * scale;
    double r, p;
    if (logit > st.m) {  // new running max: rescale what we have
      r = exp(st.m - logit);
      p = 1.0;
      st.m = logit;
    } else {
      r = 1.0;
      p = exp(logit - st.m);
    }
    st.z = st.z * r + p;
#pragma unroll
    for (int j = 0; j < kF64MaxPerLane; ++j) {
      const int i = lane + 32 * j;
      if (i < w) st.acc[j] = st.acc[j] * r + p * vr[i];
    }
  }
}

// Combine the CTA's warps in warp order (deterministic) and store the
// normalised output and natural-log lse; no rows at all -> (0, -inf)
// (attention.hpp:69-70).
__device__ __forceinline__ void f64_finish(F64State& st, int w, double* out, double* lse) {
  __shared__ double s_m[kF64Warps], s_z[kF64Warps];
  __shared__ double s_acc[kF64Warps][kF64MaxWidth];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    s_m[warp] = st.m;
    s_z[warp] = st.z;
  }
#pragma unroll
  for (int j = 0; j < kF64MaxPerLane; ++j) {
    const int i = lane + 32 * j;
    if (i < w) s_acc[warp][i] = st.acc[j];
  }
  __syncthreads();
  double M = -INFINITY;
  for (int k = 0; k < kF64Warps; ++k) M = fmax(M, s_m[k]);
  if (M == -INFINITY) {
    for (int i = threadIdx.x; i < w; i += blockDim.x) out[i] = 0.0;
    if (threadIdx.x == 0 && lse) *lse = -INFINITY;
    return;
  }
  double Z = 0.0;
  for (int k = 0; k < kF64Warps; ++k)
    if (s_m[k] != -INFINITY) Z += s_z[k] * exp(s_m[k] - M);
  for (int i = threadIdx.x; i < w; i += blockDim.x) {
    double a = 0.0;
    for (int k = 0; k < kF64Warps; ++k)
      if (s_m[k] != -INFINITY) a += s_acc[k][i] * exp(s_m[k] - M);
    out[i] = a / Z;
  }
  if (threadIdx.x == 0 && lse) *lse = M + log(Z);
}

__device__ __forceinline__ void f64_init(F64State& st) {
  st.m = -INFINITY;
  st.z = 0.0;
#pragma unroll
  for (int j = 0; j < kF64MaxPerLane; ++j) st.acc[j] = 0.0;
}

// ---- free functions: nq queries over one caller-supplied K/V [n][w]
__global__ void __launch_bounds__(kF64Warps * 32) attn_f64_plain_kernel(const double* q, const double* K,
                                                                       const double* V, long long n, int w,
                                                                       double scale, double* out, double* lse) {
  __shared__ double sq[kF64MaxWidth];
  const int qi = blockIdx.x;
  for (int i = threadIdx.x; i < w; i += blockDim.x) sq[i] = q[static_cast<size_t>(qi) * w + i];
  __syncthreads();
  F64State st;
  f64_init(st);
  f64_rows(sq, w, K, V, n, scale, threadIdx.x >> 5, kF64Warps, st);
  f64_finish(st, w, out + static_cast<size_t>(qi) * w, lse ? lse + qi : nullptr);
}

// ---- the harness: one CTA per (slot, request, query head of the slot)
// partial (mono = 0): fragment of one KVP rank (shard_attention, :375-396);
// monolithic (mono = 1): one softmax over every rank of the TPA group
// (DecodeHarness::reference, :514-529). q: [B][qkv_stride] projections,
// head h at column h*w.
__global__ void __launch_bounds__(kF64Warps * 32) attn_f64_harness_kernel(F64HarnessParams p, int mono,
                                                                         double* frag_o, double* frag_lse) {
  __shared__ double sq[kF64MaxWidth];
  int t = blockIdx.x;
  const int qi = t % p.q_per_slot;
  t /= p.q_per_slot;
  const int b = t % p.batch;
  const int s = t / p.batch;  // slot (partial) or TPA group (monolithic)
  const int grp = mono ? s : s / p.kvp;
  const int head = grp * p.q_per_slot + qi;
  const int kvh = qi / p.group;
  const int w = p.w;
  for (int i = threadIdx.x; i < w; i += blockDim.x)
    sq[i] = p.qkv[static_cast<size_t>(b) * p.qkv_stride + static_cast<size_t>(head) * w + i];
  __syncthreads();
  F64State st;
  f64_init(st);
  const int r0 = mono ? 0 : s % p.kvp, r1 = mono ? p.kvp : r0 + 1;
  for (int r = r0; r < r1; ++r) {
    const int slot = grp * p.kvp + r;
    const long long n = rr_count(p.total[b], r, p.chunk, p.kvp);
    const size_t base = ((static_cast<size_t>(slot) * p.batch + b) * p.kvh_per_slot + kvh) * p.rows_cap * w;
    f64_rows(sq, w, p.k + base, p.v + base, n, p.scale, threadIdx.x >> 5, kF64Warps, st);
  }
  const size_t f = static_cast<size_t>(blockIdx.x);  // [slot or grp][b][qi]
  f64_finish(st, w, frag_o + f * w, frag_lse + f);
}

// Canonical merge (attention.hpp:90-137): thread 0 orders the fragments by
// descending lse, ties by the first differing coefficient (ascending) -- the
// reference's exact order, so the result is bitwise invariant to fragment
// order -- then every thread folds its coefficients in that order.
__device__ void f64_merge(const double* outs, size_t out_stride, const double* lses, size_t lse_stride, int nf,
                          int w, double* out, double* lse, int* ord) {
  if (threadIdx.x == 0) {
    for (int i = 0; i < nf; ++i) ord[i] = i;
    auto before = [&](int a, int c) {
      const double la = lses[a * lse_stride], lc = lses[c * lse_stride];
      if (la != lc) return la > lc;
      for (int i = 0; i < w; ++i) {
        const double oa = outs[a * out_stride + i], oc = outs[c * out_stride + i];
        if (oa != oc) return oa < oc;
      }
      return false;
    };
    for (int i = 1; i < nf; ++i) {
      const int v = ord[i];
      int j = i - 1;
      while (j >= 0 && before(v, ord[j])) {
        ord[j + 1] = ord[j];
        --j;
      }
      ord[j + 1] = v;
    }
  }
  __syncthreads();
  const double m = lses[ord[0] * lse_stride];
  double z = 0.0;
  for (int k = 0; k < nf; ++k) {
    const double l = lses[ord[k] * lse_stride];
    if (l != -INFINITY) z += exp(l - m);
  }
  for (int i = threadIdx.x; i < w; i += blockDim.x) {
    double a = 0.0;
    for (int k = 0; k < nf; ++k) {
      const double l = lses[ord[k] * lse_stride];
      if (l == -INFINITY) continue;
      a += exp(l - m) * outs[ord[k] * out_stride + i];
    }
    out[i] = a / z;
  }
  if (threadIdx.x == 0 && lse) *lse = m + log(z);
}

__global__ void merge_f64_plain_kernel(const double* outs, const double* lses, int nf, int w, double* out,
                                       double* lse) {
  extern __shared__ int s_ord[];
  f64_merge(outs, static_cast<size_t>(w), lses, 1, nf, w, out, lse, s_ord);
}

// harness: one CTA per (request, head): fragments [slot][b][qi] of the head's group
__global__ void merge_f64_harness_kernel(F64HarnessParams p, const double* frag_o, const double* frag_lse,
                                         double* out, double* lse) {
  extern __shared__ int s_ord[];
  const int q_heads = p.q_per_slot * p.tpa;
  const int b = blockIdx.x / q_heads, head = blockIdx.x % q_heads;
  const int grp = head / p.q_per_slot, qi = head % p.q_per_slot;
  const size_t f0 = (static_cast<size_t>(grp * p.kvp) * p.batch + b) * p.q_per_slot + qi;
  const size_t fstride = static_cast<size_t>(p.batch) * p.q_per_slot;  // next rank's fragment
  f64_merge(frag_o + f0 * p.w, fstride * p.w, frag_lse + f0, fstride, p.kvp, p.w,
            out + (static_cast<size_t>(b) * q_heads + head) * p.w, lse ? lse + b * q_heads + head : nullptr, s_ord);
}

// y[b][n] = sum_k x[b][k] W[k][n] (row-major W [K x N]), k in order
__global__ void gemv_f64_kernel(const double* x, const double* W, int K, int N, double* y) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x, b = blockIdx.y;
  if (n >= N) return;
  const double* xb = x + static_cast<size_t>(b) * K;
  double acc = 0.0;
  for (int k = 0; k < K; ++k) acc += xb[k] * W[static_cast<size_t>(k) * N + n];
  y[static_cast<size_t>(b) * N + n] = acc;
}

// Round-robin append (attention.hpp:262-282) of rows [n][kv_heads][w] for one
// request (src_stride: per-token stride; from the projection: the k/v columns of
// qkv), tokens total[b] .. total[b]+n-1; bump the total afterwards (separate kernel).
__global__ void append_f64_kernel(F64HarnessParams p, const double* ksrc, const double* vsrc, size_t src_stride,
                                  int b, long long n, int kv_heads) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long per = static_cast<long long>(kv_heads) * p.w;
  if (i >= n * per) return;
  const long long tok = i / per;
  const int h = static_cast<int>((i % per) / p.w), d = static_cast<int>(i % p.w);
  const long long g = p.total[b] + tok;
  const int rank = rr_rank(g, p.chunk, p.kvp);
  const long long row = rr_row(g, p.chunk, p.kvp);
  const int grp = h / p.kvh_per_slot, kvh = h % p.kvh_per_slot;
  const int slot = grp * p.kvp + rank;
  const size_t dst = (((static_cast<size_t>(slot) * p.batch + b) * p.kvh_per_slot + kvh) * p.rows_cap + row) * p.w + d;
  p.k[dst] = ksrc[tok * src_stride + static_cast<size_t>(h) * p.w + d];
  p.v[dst] = vsrc[tok * src_stride + static_cast<size_t>(h) * p.w + d];
}

__global__ void bump_total_kernel(int* total, int b0, int nb, long long n) {
  const int i = threadIdx.x;
  if (i < nb) total[b0 + i] += static_cast<int>(n);
}

// Rows of (slot, request, kv head) back to the host (ShardedKVCache::context)
__global__ void read_f64_kernel(F64HarnessParams p, int slot, int b, int kvh, long long n, double* k, double* v) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n * p.w) return;
  const size_t src = ((static_cast<size_t>(slot) * p.batch + b) * p.kvh_per_slot + kvh) * p.rows_cap * p.w + i;
  k[i] = p.k[src];
  v[i] = p.v[src];
}

}  // namespace

cudaError_t launch_attn_f64_plain(const double* q, int nq, const double* K, const double* V, long long n, int w,
                                  double* out, double* lse, cudaStream_t s) {
  if (w < 1 || w > kF64MaxWidth || nq < 1) return cudaErrorInvalidValue;
  attn_f64_plain_kernel<<<nq, kF64Warps * 32, 0, s>>>(q, K, V, n, w, 1.0 / std::sqrt(static_cast<double>(w)), out,
                                                      lse);
  return cudaGetLastError();
}

cudaError_t launch_merge_f64_plain(const double* outs, const double* lses, int nf, int w, double* out, double* lse,
                                   cudaStream_t s) {
  if (w < 0 || nf < 1) return cudaErrorInvalidValue;
  merge_f64_plain_kernel<<<1, 256, nf * sizeof(int), s>>>(outs, lses, nf, w, out, lse);
  return cudaGetLastError();
}

cudaError_t launch_gemv_f64(const double* x, int B, const double* W, int K, int N, double* y, cudaStream_t s) {
  gemv_f64_kernel<<<dim3((N + 127) / 128, B), 128, 0, s>>>(x, W, K, N, y);
  return cudaGetLastError();
}

cudaError_t launch_attn_f64_harness(const F64HarnessParams& p, int mono, double* frag_o, double* frag_lse,
                                    cudaStream_t s) {
  if (p.w > kF64MaxWidth) return cudaErrorInvalidValue;
  const int ctas = (mono ? p.tpa : p.tpa * p.kvp) * p.batch * p.q_per_slot;
  attn_f64_harness_kernel<<<ctas, kF64Warps * 32, 0, s>>>(p, mono, frag_o, frag_lse);
  return cudaGetLastError();
}

cudaError_t launch_merge_f64_harness(const F64HarnessParams& p, const double* frag_o, const double* frag_lse,
                                     double* out, double* lse, cudaStream_t s) {
  merge_f64_harness_kernel<<<p.batch * p.q_per_slot * p.tpa, 128, p.kvp * sizeof(int), s>>>(p, frag_o, frag_lse,
                                                                                            out, lse);
  return cudaGetLastError();
}

cudaError_t launch_append_f64(const F64HarnessParams& p, const double* ksrc, const double* vsrc, size_t src_stride,
                              int b, long long n, int kv_heads, cudaStream_t s) {
  const long long cnt = n * kv_heads * p.w;
  if (cnt == 0) return cudaSuccess;
  append_f64_kernel<<<static_cast<unsigned>((cnt + 255) / 256), 256, 0, s>>>(p, ksrc, vsrc, src_stride, b, n,
                                                                             kv_heads);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  bump_total_kernel<<<1, 64, 0, s>>>(p.total, b, 1, n);
  return cudaGetLastError();
}

cudaError_t launch_read_f64(const F64HarnessParams& p, int slot, int b, int kvh, long long n, double* k, double* v,
                            cudaStream_t s) {
  const long long cnt = n * p.w;
  if (cnt == 0) return cudaSuccess;
  read_f64_kernel<<<static_cast<unsigned>((cnt + 255) / 256), 256, 0, s>>>(p, slot, b, kvh, n, k, v);
  return cudaGetLastError();
}

}  // namespace hx
