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
constexpr int kStageSteps = 4;    // k-steps per ring stage (4 x 4 KB)
constexpr int kStages = 4;        // ring depth: 64 KB of weights in flight per CTA

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ unsigned long long logit_key(float v, int n) {
  unsigned u = __float_as_uint(v);
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return (static_cast<unsigned long long>(u) << 32) | (0xFFFFFFFFu - static_cast<unsigned>(n));
}

// Merged attention output element (KVP fragment combine, attention.hpp:118-137):
// canonical order = descending lse, ties broken by source rank.
__device__ float merge_elem(const GemvParams& p, int b, int k) {
  const int head = k / p.head_dim, d = k - head * p.head_dim;
  const int grp = head / p.q_per_slot, qi = head - grp * p.q_per_slot;
  float lse[8];
  int ord[8];
  const int kvp = p.kvp;
  for (int r = 0; r < kvp; ++r) {
    const int slot = grp * kvp + r;
    lse[r] = p.frag_lse[(static_cast<size_t>(slot) * p.batch + b) * p.q_per_slot + qi];
    ord[r] = r;
  }
  for (int i = 1; i < kvp; ++i) {  // insertion sort: lse desc, rank asc
    const int o = ord[i];
    int j = i - 1;
    while (j >= 0 && lse[ord[j]] < lse[o]) {
      ord[j + 1] = ord[j];
      --j;
    }
    ord[j + 1] = o;
  }
  const float m = lse[ord[0]];
  if (m == -INFINITY) return 0.f;
  float acc = 0.f, z = 0.f;
  for (int i = 0; i < kvp; ++i) {
    const int r = ord[i];
    if (lse[r] == -INFINITY) continue;
    const float w = __expf(lse[r] - m);
    const int slot = grp * kvp + r;
    acc += w * p.frag_o[((static_cast<size_t>(slot) * p.batch + b) * p.q_per_slot + qi) * p.dp + d];
    z += w;
  }
  return acc / z;
}

template <int XM>
__device__ __forceinline__ float x_value(const GemvParams& p, const float* s_inv, int b, int k) {
  if (XM == X_MERGE) return merge_elem(p, b, k);
  const float v = p.x[static_cast<size_t>(b) * p.x_stride + k];
  return XM == X_NORM ? v * s_inv[b] : v;
}

}  // namespace

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

  // ---------------------------------------------------------------- prologue (overlaps the stream)
  if (XM == X_NORM) {
    if (threadIdx.x < p.batch) {
      float s = 0.f;
      for (int i = 0; i < p.n_ss; ++i) s += p.ss_part[i * p.batch + threadIdx.x];
      s_inv[threadIdx.x] = rsqrtf(s / static_cast<float>(p.K) + p.eps);
    }
    named_bar_sync(1, kThreads);
  }
  for (int e = threadIdx.x; e < nks * NB8 * 32; e += kThreads) {
    const int ln = e & 31;
    const int t = e >> 5;
    const int bg = t % NB8, ksl = t / NB8;
    const int g = ln >> 2, c = ln & 3;
    const int b = bg * 8 + g;
    const int k = (ks0 + ksl) * 16 + 2 * c;
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    if (b < p.batch) {
      v[0] = x_value<XM>(p, s_inv, b, k);
      v[1] = x_value<XM>(p, s_inv, b, k + 1);
      v[2] = x_value<XM>(p, s_inv, b, k + 8);
      v[3] = x_value<XM>(p, s_inv, b, k + 9);
    }
    if (XS == 2) {
      float hi[4], lo[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) split2(v[i], hi[i], lo[i]);
      xs[(ksl * 2 * NB8 + bg) * 32 + ln] = make_uint2(pack_bf16(hi[0], hi[1]), pack_bf16(hi[2], hi[3]));
      xs[(ksl * 2 * NB8 + NB8 + bg) * 32 + ln] = make_uint2(pack_bf16(lo[0], lo[1]), pack_bf16(lo[2], lo[3]));
    } else {
      float hi[4], mid[4], lo[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) split3(v[i], hi[i], mid[i], lo[i]);
      xs[(ksl * 3 * NB8 + bg) * 32 + ln] = make_uint2(pack_bf16(hi[0], hi[1]), pack_bf16(hi[2], hi[3]));
      xs[(ksl * 3 * NB8 + NB8 + bg) * 32 + ln] = make_uint2(pack_bf16(mid[0], mid[1]), pack_bf16(mid[2], mid[3]));
      xs[(ksl * 3 * NB8 + 2 * NB8 + bg) * 32 + ln] = make_uint2(pack_bf16(lo[0], lo[1]), pack_bf16(lo[2], lo[3]));
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
      float y = 0.f;
      const int n = nblk * kRows + rr;
      for (int s = 0; s < p.ksplit; ++s)
        y += __ldcg(p.ypart + (static_cast<size_t>(s) * p.batch + b) * p.Npad + n);
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
        atomicMax(&s_best[b], logit_key(y, n));
      } else if (EM == E_QKV) {
        if (n < p.nq) {
          const int head = n / p.head_dim, d = n - head * p.head_dim;
          const int q_heads = p.nq / p.head_dim;
          p.q_out[(static_cast<size_t>(b) * q_heads + head) * p.dp + d] = y;
        } else {
          const int kvn = n - p.nq;
          const int is_v = kvn >= p.nk;
          const int kn = is_v ? kvn - p.nk : kvn;
          const int h = kn / p.head_dim, d = kn - h * p.head_dim;
          if (p.kv_dbg)
            p.kv_dbg[((static_cast<size_t>(b) * 2 + is_v) * p.kv_heads + h) * p.head_dim + d] = y;
          if (p.append) {
            const long long g = p.total[b];
            const int rank = rr_rank(g, p.chunk, p.kvp);
            const long long row = rr_row(g, p.chunk, p.kvp);
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

size_t gemv_smem_bytes(const GemvParams& p, int xs_terms) {
  const int nb8 = (p.batch + 7) / 8;
  const size_t xs = static_cast<size_t>(p.kr_steps) * nb8 * xs_terms * 32 * 8;
  return static_cast<size_t>(kStages) * kStageSteps * 4096 + xs;  // epilogue staging reuses the ring
}

template <int NB8, int XM, int EM>
static cudaError_t launch_t(const GemvParams& p, cudaStream_t stream) {
  // QKV feeds exp(q.k) with |logits| up to ~1e3 under the reference's unscaled
  // weights: carry x at fp32 precision there (3 bf16 terms), 2 terms elsewhere.
  constexpr int XS = EM == E_QKV ? 3 : 2;
  const size_t smem = gemv_smem_bytes(p, XS);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(gemv_kernel<NB8, XM, EM, XS>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  dim3 grid(p.Npad / kRows, p.ksplit);
  gemv_kernel<NB8, XM, EM, XS><<<grid, kThreads + 32, smem, stream>>>(p);
  return cudaGetLastError();
}

template <int NB8>
static cudaError_t dispatch_nb(const GemvParams& p, int xm, int em, cudaStream_t s) {
#define HX_CASE(X, E) \
  if (xm == X && em == E) return launch_t<NB8, X, E>(p, s);
  HX_CASE(X_PLAIN, E_QKV)
  HX_CASE(X_NORM, E_QKV)
  HX_CASE(X_MERGE, E_RESID)
  HX_CASE(X_MERGE, E_STORE)
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
