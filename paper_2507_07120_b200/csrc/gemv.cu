// Weight-streaming GEMV / skinny GEMM for the decode step (B <= 16 rows).
//
// y[b][n] = sum_k x[b][k] * W[k][n] with W stored fragment-major bf16 in
// CTA-tile-major order [128-row block][k-step][8 n-tiles][512 B] (one 16x16
// A tile = 512 contiguous bytes = one 16-byte shared load per lane), so each
// CTA's weights are ONE contiguous range: a producer warp streams it through
// a 4-stage shared-memory ring with cp.async.bulk (TMA bulk engine), 8
// consumer warps run HMMA m16n8k16 against x fragments staged in shared
// memory as bf16 hi+lo (or hi+mid+lo) terms, fp32 accumulation.
//
// Split-K over gridDim.y with a deterministic last-CTA reduction (partials
// summed in split order), followed by a fused epilogue:
//   E_QKV    q -> [B][head][DP]; K/V -> appended into the round-robin page
//            pool at the cursor position (attention.hpp:531-539, :262-282)
//   E_RESID  residual add (+ per-block sum of squares for the next RMSNorm)
//   E_SWIGLU silu(gate) * up for interleaved gate/up row blocks
//   E_LOGITS LM-head logits + greedy argmax (lowest index on ties)
//   E_STORE  plain store (+ sum of squares)
// x sources: X_PLAIN, X_NORM (RMSNorm from the producer's partial sums of
// squares), X_MERGE (the LSE-rescale combine of KVP fragments, fused into
// the O-projection prologue; canonical order of attention.hpp:90-102).
#include "common.cuh"
#include "kernels.h"
#include "kv_layout.cuh"

namespace hx {

namespace {

constexpr int kRows = 128;        // rows (output features) per CTA: 8 consumer warps x 16
constexpr int kThreads = 256;     // consumer threads (+1 producer warp)
constexpr int kStageSteps = 2;    // k-steps per ring stage (2 x 4 KB)
constexpr int kStages = 4;        // ring depth: 32 KB in flight per CTA, 4 CTAs per SM

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ unsigned long long logit_key(float v, int n) {
  unsigned u = __float_as_uint(v);
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return (static_cast<unsigned long long>(u) << 32) | (0xFFFFFFFFu - static_cast<unsigned>(n));
}

// KVP fragment combine (attention.hpp:118-137) for the O-projection prologue,
// in two phases so each is one latency round trip:
//  merge_weights: per (request, head) covered by this CTA's k-range, the
//    canonical order (descending lse, ties by rank; attention.hpp:90-102),
//    w_r = exp(lse_r - m) and z = sum w_r, into shared memory;
//  merge_elem: (sum_r w_r * o_r in that order) / z.
constexpr int kMaxKr = 32;          // k-steps per CTA (engine plan guarantees)
constexpr int kMaxMergePairs = 256; // (request, head) pairs per CTA (engine plan guarantees)
struct MergeSmem {
  float w[kMaxMergePairs][8];
  float z[kMaxMergePairs];
  int ord[kMaxMergePairs][8];
};

// Flattened index of column k inside the merged attention output:
// X_MERGE: k is a global hidden index; X_RECV: k is an offset into this rank's
// exchanged slice r*slice .. of its group's flattened (heads x head_dim) block.
template <int XM>
__device__ __forceinline__ int merge_flat(const GemvParams& p, int k) {
  return XM == X_RECV ? p.exch_rank * p.slice + k : k;
}
template <int XM>
__device__ __forceinline__ int merge_nh(const GemvParams& p, int ks0, int nks) {
  return merge_flat<XM>(p, (ks0 + nks) * 16 - 1) / p.head_dim - merge_flat<XM>(p, ks0 * 16) / p.head_dim + 1;
}
template <int XM>
__device__ __forceinline__ float merge_lse(const GemvParams& p, int r, int b, int head) {
  if (XM == X_RECV) {
    const int first = (p.exch_rank * p.slice) / p.head_dim;
    return p.recv[(static_cast<size_t>(r) * p.batch + b) * p.chunk + p.slice + head - first];
  }
  const int grp = head / p.q_per_slot, qi = head - grp * p.q_per_slot;
  return p.frag_lse[(static_cast<size_t>(grp * p.kvp + r) * p.batch + b) * p.q_per_slot + qi];
}
template <int XM>
__device__ __forceinline__ float merge_o(const GemvParams& p, int r, int b, int k, int head, int d) {
  if (XM == X_RECV) return p.recv[(static_cast<size_t>(r) * p.batch + b) * p.chunk + k];
  const int grp = head / p.q_per_slot, qi = head - grp * p.q_per_slot;
  return p.frag_o[((static_cast<size_t>(grp * p.kvp + r) * p.batch + b) * p.q_per_slot + qi) * p.dp + d];
}

template <int XM>
__device__ void merge_weights(const GemvParams& p, int ks0, int nks, MergeSmem* ms) {
  const int h0 = merge_flat<XM>(p, ks0 * 16) / p.head_dim;
  const int nh = merge_nh<XM>(p, ks0, nks);
  for (int pr = threadIdx.x; pr < nh * p.batch; pr += 256) {
    const int b = pr / nh, head = h0 + pr % nh;
    float lse[8];
    int ord[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      lse[r] = r < p.kvp ? merge_lse<XM>(p, r, b, head) : -INFINITY;
      ord[r] = r;
    }
    for (int i = 1; i < p.kvp; ++i) {  // insertion sort: lse desc, rank asc
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
    for (int i = 0; i < 8; ++i) {
      const int r = ord[i];
      const float w = (i < p.kvp && m != -INFINITY && lse[r] != -INFINITY) ? __expf(lse[r] - m) : 0.f;
      ms->ord[pr][i] = r;
      ms->w[pr][i] = w;
      z += w;
    }
    ms->z[pr] = z;
  }
}

template <int XM>
__device__ __forceinline__ float merge_elem(const GemvParams& p, int b, int k, int ks0, int nks,
                                            const MergeSmem* ms) {
  const int flat = merge_flat<XM>(p, k);
  const int head = flat / p.head_dim, d = flat - head * p.head_dim;
  const int pr = b * merge_nh<XM>(p, ks0, nks) + head - merge_flat<XM>(p, ks0 * 16) / p.head_dim;
  const float z = ms->z[pr];
  if (z == 0.f) return 0.f;
  float acc = 0.f;
  for (int i = 0; i < p.kvp; ++i) {
    const int r = ms->ord[pr][i];
    acc += ms->w[pr][i] * merge_o<XM>(p, r, b, k, head, d);
  }
  return acc / z;
}

}  // namespace

__host__ __device__ __forceinline__ size_t xs_bytes(const GemvParams& p, int nb8, int xs_terms) {
  return static_cast<size_t>(p.kr_steps) * nb8 * xs_terms * 32 * 8;
}

template <int NB8, int XM, int EM, int XS>
__global__ void __launch_bounds__(kThreads + 32) gemv_kernel(const GemvParams p) {
  // Shared memory: [ring: kStages x kStageSteps x 4 KB][xs fragments][mbarriers]
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* ring = smem;
  uint2* xs = reinterpret_cast<uint2*>(smem + kStages * kStageSteps * 4096);
  __shared__ float s_inv[16];
  __shared__ int s_last;
  __shared__ unsigned long long s_best[16];
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nblk = blockIdx.x, ksp = blockIdx.y;
  const int KST = p.K >> 4;
  const int ks0 = ksp * p.kr_steps;
  const int ks1 = min(ks0 + p.kr_steps, KST);
  const int nks = ks1 - ks0;
  const int nst = (nks + kStageSteps - 1) / kStageSteps;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 8);
    }
    fence_mbar_init();
  }
  __syncthreads();
  griddep_launch_dependents();

  if (warp == 8) {
    // ------------------------------------------------------------ producer: TMA bulk weight stream
    // the CTA's weights [nblk][ks0..ks1][8 n-tiles][512 B] are one contiguous range
    if (lane == 0) {
      const uint8_t* src = reinterpret_cast<const uint8_t*>(p.w) + (static_cast<size_t>(nblk) * KST + ks0) * 4096;
      for (int st = 0; st < nst; ++st) {
        const int s = st % kStages;
        if (st >= kStages) mbar_wait(&empty[s], ((st / kStages) & 1) ^ 1);
        const int steps = min(kStageSteps, nks - st * kStageSteps);
        const uint32_t bytes = static_cast<uint32_t>(steps) * 4096u;
        mbar_arrive_expect_tx(&full[s], bytes);
        bulk_g2s(ring + s * kStageSteps * 4096, src + static_cast<size_t>(st) * kStageSteps * 4096, bytes, &full[s]);
      }
    }
    return;  // exited threads do not block later CTA barriers
  }
  // weights are constant: the producer streams them while the previous kernel
  // drains; everything below reads activations it produced.
  griddep_wait();

  // ---------------------------------------------------------------- prologue (overlaps the stream)
  // Every global load below is issued before any of its results is consumed
  // (one latency round trip per phase, not one per element).
  if (XM == X_NORM) {
    for (int b = warp; b < p.batch; b += 8) {
      float ss = 0.f;
      for (int i = lane; i < p.n_ss; i += 32) ss += p.ss_part[i * p.batch + b];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if (lane == 0) s_inv[b] = rsqrtf(ss / static_cast<float>(p.K) + p.eps);
    }
  }
  MergeSmem* ms = reinterpret_cast<MergeSmem*>(smem + kStages * kStageSteps * 4096 + xs_bytes(p, NB8, XS));
  if (XM == X_MERGE || XM == X_RECV) merge_weights<XM>(p, ks0, nks, ms);
  if (XM != X_PLAIN) named_bar_sync(1, kThreads);
  {
    constexpr int MAXE = (kMaxKr * NB8 * 32) / kThreads;  // entries per thread (kr <= kMaxKr)
    float v[MAXE][4];
#pragma unroll
    for (int j = 0; j < MAXE; ++j) {
      const int e = threadIdx.x + j * kThreads;
      const int ln = e & 31, t = e >> 5;
      const int bg = t % NB8, ksl = t / NB8;
      const int b = bg * 8 + (ln >> 2);
      const int k = (ks0 + ksl) * 16 + 2 * (ln & 3);
      const bool ok = ksl < nks && b < p.batch;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int kk = k + (i & 1) + (i >> 1) * 8;
        v[j][i] = ok ? ((XM == X_MERGE || XM == X_RECV) ? merge_elem<XM>(p, b, kk, ks0, nks, ms)
                                                        : p.x[static_cast<size_t>(b) * p.x_stride + kk])
                     : 0.f;
      }
    }
#pragma unroll
    for (int j = 0; j < MAXE; ++j) {
      const int e = threadIdx.x + j * kThreads;
      const int ln = e & 31, t = e >> 5;
      const int bg = t % NB8, ksl = t / NB8;
      if (ksl >= nks) continue;
      const int b = bg * 8 + (ln >> 2);
      if (XM == X_NORM && b < p.batch)
#pragma unroll
        for (int i = 0; i < 4; ++i) v[j][i] *= s_inv[b];
      if (XS == 2) {
        float hi[4], lo[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) split2(v[j][i], hi[i], lo[i]);
        xs[(ksl * 2 * NB8 + bg) * 32 + ln] = make_uint2(pack_bf16(hi[0], hi[1]), pack_bf16(hi[2], hi[3]));
        xs[(ksl * 2 * NB8 + NB8 + bg) * 32 + ln] = make_uint2(pack_bf16(lo[0], lo[1]), pack_bf16(lo[2], lo[3]));
      } else {
        float hi[4], mid[4], lo[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) split3(v[j][i], hi[i], mid[i], lo[i]);
        xs[(ksl * 3 * NB8 + bg) * 32 + ln] = make_uint2(pack_bf16(hi[0], hi[1]), pack_bf16(hi[2], hi[3]));
        xs[(ksl * 3 * NB8 + NB8 + bg) * 32 + ln] = make_uint2(pack_bf16(mid[0], mid[1]), pack_bf16(mid[2], mid[3]));
        xs[(ksl * 3 * NB8 + 2 * NB8 + bg) * 32 + ln] = make_uint2(pack_bf16(lo[0], lo[1]), pack_bf16(lo[2], lo[3]));
      }
    }
  }
  named_bar_sync(1, kThreads);

  // ---------------------------------------------------------------- consume the weight ring
  const int ntile = nblk * 8 + warp;
  float acc[XS * NB8][4];
#pragma unroll
  for (int j = 0; j < XS * NB8; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
  const uint32_t xs_base = smem_u32(xs) + lane * 8;
  const uint32_t ring_base = smem_u32(ring) + warp * 512 + lane * 16;
  for (int st = 0; st < nst; ++st) {
    const int s = st % kStages;
    mbar_wait(&full[s], (st / kStages) & 1);
    const int steps = min(kStageSteps, nks - st * kStageSteps);
#pragma unroll
    for (int kk = 0; kk < kStageSteps; ++kk) {
      if (kk < steps) {
        const uint4 wa = lds128(ring_base + (s * kStageSteps + kk) * 4096);
        const uint32_t xa = xs_base + ((st * kStageSteps + kk) * XS * NB8) * 256;
#pragma unroll
        for (int j = 0; j < XS * NB8; ++j) {
          const uint2 bx = lds64(xa + j * 256);
          mma_bf16_16816(acc[j], wa.x, wa.y, wa.z, wa.w, bx.x, bx.y);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  // partials: rows ntile*16 + g (+8), batches bg*8 + 2c (+1)
  {
    const int g = lane >> 2, c = lane & 3;
    const int n0 = ntile * 16 + g;
#pragma unroll
    for (int bg = 0; bg < NB8; ++bg) {
      float y[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        y[i] = acc[bg][i] + acc[(XS - 1) * NB8 + bg][i];
        if (XS == 3) y[i] += acc[NB8 + bg][i];
      }
      const int b0 = bg * 8 + 2 * c;
      float* yp = p.ypart + static_cast<size_t>(ksp) * p.batch * p.Npad;
      if (b0 < p.batch) {
        yp[static_cast<size_t>(b0) * p.Npad + n0] = y[0];
        yp[static_cast<size_t>(b0) * p.Npad + n0 + 8] = y[2];
      }
      if (b0 + 1 < p.batch) {
        yp[static_cast<size_t>(b0 + 1) * p.Npad + n0] = y[1];
        yp[static_cast<size_t>(b0 + 1) * p.Npad + n0 + 8] = y[3];
      }
    }
  }
  __threadfence();  // every writer publishes its partials device-wide
  named_bar_sync(1, kThreads);
  if (threadIdx.x == 0) {
    const int prev = atomicAdd(&p.counters[nblk], 1);
    s_last = prev == p.ksplit - 1;
  }
  named_bar_sync(1, kThreads);
  if (!s_last) return;
  __threadfence();

  // ---------------------------------------------------------------- epilogue (last CTA of the n-block)
  float* vt = reinterpret_cast<float*>(smem);  // [16][kRows] staged results (reuses the ring)
  if (EM == E_LOGITS) {
    if (threadIdx.x < 16) s_best[threadIdx.x] = 0ull;
    named_bar_sync(1, kThreads);
  }
  const int rows_here = EM == E_SWIGLU ? kRows / 2 : kRows;
  for (int e = threadIdx.x; e < rows_here * p.batch; e += kThreads) {
    const int r = e % rows_here, b = e / rows_here;
    auto ysum = [&](int rr) {
      // all split partials are loaded before summing (in split order: deterministic)
      const int n = nblk * kRows + rr;
      const float* base = p.ypart + static_cast<size_t>(b) * p.Npad + n;
      const size_t stride = static_cast<size_t>(p.batch) * p.Npad;
      float y = 0.f;
      for (int s0 = 0; s0 < p.ksplit; s0 += 16) {
        float v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = s0 + j < p.ksplit ? __ldcg(base + (s0 + j) * stride) : 0.f;
#pragma unroll
        for (int j = 0; j < 16; ++j) y += v[j];
      }
      return y;
    };
    if (EM == E_SWIGLU) {
      const float gt = ysum(r), up = ysum(r + kRows / 2);
      const int f = nblk * (kRows / 2) + r;
      const float m = gt / (1.f + __expf(-gt)) * up;
      if (f < p.N / 2) p.out[static_cast<size_t>(b) * p.out_stride + f] = m;
      continue;
    }
    const float y = ysum(r);
    const int n = nblk * kRows + r;
    float keep = 0.f;
    if (n < p.N) {
      if (EM == E_STORE) {
        p.out[static_cast<size_t>(b) * p.out_stride + n] = y;
        keep = y;
      } else if (EM == E_RESID) {
        float* o = p.out + static_cast<size_t>(b) * p.out_stride + n;
        keep = *o + y;
        *o = keep;
      } else if (EM == E_LOGITS) {
        if (p.out) p.out[static_cast<size_t>(b) * p.out_stride + n] = y;
        atomicMax(&s_best[b], logit_key(y, n + p.n_offset));
      } else if (EM == E_QKV) {
        if (n < p.nq) {
          const int head = n / p.head_dim, d = n - head * p.head_dim;
          const int q_heads = p.nq / p.head_dim;
          p.q_out[(static_cast<size_t>(b) * q_heads + head) * p.dp + d] = y;
        } else {
          const int kvn = n - p.nq;
          const int is_v = kvn >= p.nk;
          const int kn = is_v ? kvn - p.nk : kvn;
          const int hl = kn / p.head_dim, d = kn - hl * p.head_dim;
          const int h = p.kv_head_base + hl;
          if (p.kv_dbg)
            p.kv_dbg[((static_cast<size_t>(b) * 2 + is_v) * p.kv_heads + hl) * p.head_dim + d] = y;
          if (p.append) {
            const long long g = p.total[b];
            const int rank = rr_rank(g, p.rr_chunk, p.kvp);
            const long long row = rr_row(g, p.rr_chunk, p.kvp);
            const int grp = h / p.kvh_per_slot, kvh = h - grp * p.kvh_per_slot;
            const int slot_local = grp * p.kvp + rank - p.slot_base;
            if (slot_local >= 0 && slot_local < p.n_local_slots) {
              const size_t page =
                  ((static_cast<size_t>(slot_local) * p.batch + b) * p.kvh_per_slot + kvh) * p.page_cap +
                  static_cast<size_t>(row >> 4);
              const uint32_t off = is_v ? v_offset(p.dp, static_cast<int>(row & 15), d)
                                        : k_offset(p.dp, static_cast<int>(row & 15), d);
              *reinterpret_cast<__nv_bfloat16*>(p.kv + page * page_bytes(p.dp) + off) =
                  __float2bfloat16_rn(y);
            }
          }
        }
      }
    }
    if (EM == E_STORE || EM == E_RESID) vt[b * kRows + r] = keep * keep;
  }
  if (EM == E_STORE || EM == E_RESID) {
    if (p.ss_out) {
      named_bar_sync(1, kThreads);
      for (int b = warp; b < p.batch; b += kThreads / 32) {
        float s = 0.f;
        for (int r = lane; r < kRows; r += 32) s += vt[b * kRows + r];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) p.ss_out[static_cast<size_t>(nblk) * p.batch + b] = s;
      }
    }
  }
  if (EM == E_LOGITS) {
    named_bar_sync(1, kThreads);
    if (threadIdx.x < p.batch) atomicMax(&p.best[threadIdx.x], s_best[threadIdx.x]);
  }
  if (threadIdx.x == 0) p.counters[nblk] = 0;  // self-reset for the next launch
}

size_t gemv_smem_bytes(const GemvParams& p, int xs_terms, bool merge) {
  const int nb8 = (p.batch + 7) / 8;
  // epilogue staging reuses the ring
  return static_cast<size_t>(kStages) * kStageSteps * 4096 + xs_bytes(p, nb8, xs_terms) +
         (merge ? sizeof(MergeSmem) : 0);
}

template <int NB8, int XM, int EM>
static cudaError_t launch_t(const GemvParams& p, cudaStream_t stream) {
  // QKV feeds exp(q.k) with |logits| up to ~1e3 under the reference's unscaled
  // weights: carry x at fp32 precision there (3 bf16 terms), 2 terms elsewhere.
  constexpr int XS = EM == E_QKV ? 3 : 2;
  const size_t smem = gemv_smem_bytes(p, XS, XM == X_MERGE || XM == X_RECV);
  static size_t configured = 0;  // opt in once per instantiation (static smem adds to the 48 KB default)
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(gemv_kernel<NB8, XM, EM, XS>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  dim3 grid(p.Npad / kRows, p.ksplit);
  return launch_k(gemv_kernel<NB8, XM, EM, XS>, grid, dim3(kThreads + 32), smem, stream, p);
}

template <int NB8>
static cudaError_t dispatch_nb(const GemvParams& p, int xm, int em, cudaStream_t s) {
#define HX_CASE(X, E) \
  if (xm == X && em == E) return launch_t<NB8, X, E>(p, s);
  HX_CASE(X_PLAIN, E_QKV)
  HX_CASE(X_NORM, E_QKV)
  HX_CASE(X_MERGE, E_RESID)
  HX_CASE(X_MERGE, E_STORE)
  HX_CASE(X_RECV, E_STORE)
  HX_CASE(X_NORM, E_SWIGLU)
  HX_CASE(X_PLAIN, E_RESID)
  HX_CASE(X_PLAIN, E_STORE)
  HX_CASE(X_NORM, E_LOGITS)
  HX_CASE(X_NORM, E_STORE)
#undef HX_CASE
  return cudaErrorInvalidValue;
}

cudaError_t launch_gemv(const GemvParams& p, int xmode, int emode, cudaStream_t stream) {
  if (p.batch < 1 || p.batch > 16 || (p.K & 15) || (p.Npad % kRows)) return cudaErrorInvalidValue;
  if (p.batch <= 8) return dispatch_nb<1>(p, xmode, emode, stream);
  return dispatch_nb<2>(p, xmode, emode, stream);
}

}  // namespace hx
