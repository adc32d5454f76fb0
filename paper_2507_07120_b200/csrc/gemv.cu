// Weight-streaming GEMV / skinny GEMM for the decode step (B <= 64 rows).
//
// y[b][n] = sum_k x[b][k] * W[k][n]. W is bf16, fragment-major in CTA-tile
// order [128-row block][k-step][8 n-tiles][512 B] (one 16x16 HMMA A tile = 512
// contiguous bytes = one 16-byte shared load per lane). x arrives pre-split
// into bf16 terms in the HMMA B-operand image (xfrag.cuh), written once by its
// producer. The kernel is PERSISTENT (one CTA per SM) like the attention
// kernel: a producer warp pulls tiles (128-row block, k-chunk) from a
// self-resetting queue and streams each tile's weights and x slice through a
// 4-stage shared-memory ring with cp.async.bulk (TMA bulk engine); 8 consumer
// warps run HMMA m16n8k16 (fp32 accumulate). Split-K tiles publish partials;
// the last tile of a row block runs the fused epilogue while the producer
// keeps streaming:
//   E_QKV    q -> [B][head][DP]; K/V -> appended into the round-robin page
//            pool at the cursor position (attention.hpp:531-539, :262-282)
//   E_RESID  residual add, per-block sums of squares (next RMSNorm) and the
//            new residual's x-fragments
//   E_SWIGLU silu(gate) * up for interleaved gate/up rows -> x-fragments of m
//   E_LOGITS LM-head logits + greedy argmax (lowest index on ties)
//   E_STORE  plain store (tensor-parallel partial products before AllReduce)
// RMSNorm without a weight is a per-row scalar: (x * s) W = s * (x W), so
// normalised consumers multiply y by s = rsqrt(mean(x^2) + eps) in the epilogue.
//
// FP8 weights (W8, hx_runtime_config.w_dtype = HX_W_FP8_E4M3): the same tile
// order with 8 e4m3 bytes per lane (256 B per 16x16 tile, 2 KB per 128-row
// k-step), widened exactly to f16 by cvt.rn.f16x2.e4m3x2 and multiplied by the
// activation's two f16 terms (xfrag.cuh, xf16) on the f16 MMA; the per-output
// power-of-two scale s_n is applied in the epilogue after the split-K sum
// (exact: y_n = s_n * sum_k x_k q_kn).
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "kv_layout.cuh"
#include "merge.cuh"
#include "xfrag.cuh"

namespace hx {

namespace {

constexpr int kRows = 128;        // rows (output features) per tile: 8 consumer warps x 16
constexpr int kThreads = 256;     // consumer threads (+1 producer warp)
constexpr int kStages = 4;        // ring depth (~150 KB in flight per SM)
// k-steps per ring stage: 32 KB of weights (+ x slice) for B <= 16; fewer
// k-steps when the x slice grows with the batch (B <= 64) so 4 stages fit.
// WQ: weight storage 0 bf16, 1 e4m3 (FP8), 2 e2m1 blocks (FP4; stages of whole 32-input pairs)
template <int NB8, int WQ = 0>
constexpr int stage_steps() { return WQ ? (NB8 == 1 ? 8 : 4) : (NB8 <= 2 ? 8 : (NB8 <= 4 ? 4 : 2)); }
// weight bytes per k-step and 128 rows (FP4: 2176 B per pair of k-steps)
__host__ __device__ constexpr uint32_t weight_step_bytes(int wq) { return wq == 2 ? 1088u : (wq ? 2048u : 4096u); }
constexpr int kDone = -1;

struct TileMeta {
  int tile, nb, ks0, nks;  // stage covers k-steps [ks0, ks0 + nks) of row block nb
  int last;                // last stage of its tile
  int kc, gi;              // k-chunk and group (expert slot) of the tile
  int pad;
};

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ void cp_async4(float* smem_dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(smem_dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ unsigned long long logit_key(float v, int n) {
  unsigned u = __float_as_uint(v);
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return (static_cast<unsigned long long>(u) << 32) | (0xFFFFFFFFu - static_cast<unsigned>(n));
}

__host__ __device__ __forceinline__ int stage_steps_rt(int nb8, int wq) {
  return wq ? (nb8 == 1 ? 8 : 4) : (nb8 <= 2 ? 8 : (nb8 <= 4 ? 4 : 2));
}
__host__ __device__ __forceinline__ size_t stage_bytes(int nb8, int wq) {
  return static_cast<size_t>(stage_steps_rt(nb8, wq)) * (weight_step_bytes(wq) + xf_step_bytes(nb8));
}
// four e2m1 pairs (bytes 0..3 of w) -> f16x2 each, low nibble = first element
__device__ __forceinline__ void e2m1x8_to_f16x2x4_w(uint32_t w, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                                     uint32_t& r3) {
  asm("{\n .reg .b8 b0, b1, b2, b3;\n mov.b32 {b0, b1, b2, b3}, %4;\n"
      " cvt.rn.f16x2.e2m1x2 %0, b0;\n cvt.rn.f16x2.e2m1x2 %1, b1;\n"
      " cvt.rn.f16x2.e2m1x2 %2, b2;\n cvt.rn.f16x2.e2m1x2 %3, b3;\n}"
      : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
      : "r"(w));
}
__device__ __forceinline__ int ld_acquire_gpu_i(const int* ptr) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(ptr) : "memory");
  return v;
}

// Fused LSE combine (GemvParams::merge): the KVP fragments of each input element
// merged in the reference's canonical order (merge.cuh merge_sources,
// attention.hpp:90-137) -- the work xprep_merge_recv / xprep_merge_local do as a
// separate kernel -- by the 256 consumer threads of every CTA, grid-strided,
// written into p.xf; then a gpu-scope release of this CTA's share.
template <int MAXK>
__device__ __forceinline__ void merge_elems(const GemvParams& p) {
  const long long n = static_cast<long long>(p.batch) * p.K;
  uint8_t* xf = const_cast<uint8_t*>(p.xf);
  for (long long i = static_cast<long long>(blockIdx.x) * kThreads + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * kThreads) {
    const int b = static_cast<int>(i / p.K), k = static_cast<int>(i % p.K);
    float lse[MAXK], o[MAXK];
    if ((p.merge & 3) == 1) {  // received slices [src][b][chunk]: values, then the lse of every head the slice touches
      const int first = (p.m_rank * p.m_slice) / p.m_head_dim;
      const int head = (p.m_rank * p.m_slice + k) / p.m_head_dim;
#pragma unroll
      for (int r = 0; r < MAXK; ++r)
        if (r < p.m_kvp) {
          const float* src = p.m_recv + (static_cast<size_t>(r) * p.batch + b) * p.m_chunk;
          lse[r] = src[p.m_slice + head - first];
          o[r] = src[k];
        }
    } else {  // local fragments [grp * kvp + r][b][q][dp]
      const int head = k / p.m_head_dim, d = k - head * p.m_head_dim;
      const int grp = head / p.m_q_per_slot, qi = head - grp * p.m_q_per_slot;
#pragma unroll
      for (int r = 0; r < MAXK; ++r)
        if (r < p.m_kvp) {
          const size_t f = (static_cast<size_t>(grp * p.m_kvp + r) * p.batch + b) * p.m_q_per_slot + qi;
          lse[r] = p.m_frag_lse[f];
          o[r] = p.m_frag_o[f * p.m_dp + d];
        }
    }
    xf_write(xf, xf_nb8(p.batch), b, k, merge_sources<MAXK>(lse, o, p.m_kvp), p.xf16);
  }
}
__device__ void merge_prologue(const GemvParams& p) {
  griddep_wait();  // the fragments / received slices come from the previous kernels
  if (p.merge & 8) {
  } else if (p.m_kvp <= 8)
    merge_elems<8>(p);
  else
    merge_elems<kMaxKvp>(p);
  // generic-proxy stores of p.xf -> the producers' bulk (async-proxy) reads, then the release
  asm volatile("fence.proxy.async.global;" ::: "memory");
  __threadfence();
  asm volatile("bar.sync 1, %0;" ::"r"(kThreads) : "memory");
  if (threadIdx.x == 0) atomicAdd(p.merge_ctr, 1);
}

__device__ __forceinline__ uint32_t lds32_w(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint32_t hmul2_w(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

}  // namespace

template <int NB8, int EM, int XS, bool NORM, int WQ>
__global__ void __launch_bounds__(kThreads + 32, 1) gemv_kernel(const GemvParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr bool W8 = WQ != 0;  // e4m3 or e2m1: f16 MMAs on the widened weights
  constexpr int kStageSteps = stage_steps<NB8, WQ>();
  constexpr uint32_t WB = weight_step_bytes(WQ);              // weight bytes per k-step (128 rows)
  constexpr size_t SW = kStageSteps * WB;                     // weight bytes per stage
  constexpr size_t SX = kStageSteps * kXfTerms * NB8 * 256;   // x-fragment bytes per stage
  constexpr size_t SB = SW + SX;
  uint8_t* ring = smem;
  TileMeta* meta = reinterpret_cast<TileMeta*>(smem + kStages * SB);
  uint64_t* full = reinterpret_cast<uint64_t*>(meta + kStages);
  uint64_t* empty = full + kStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KST = p.K >> 4;

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
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      int st = 0;
      bool waited = false;  // x fragments come from the previous kernel; weights are constant
      // Before griddepcontrol.wait the producer fills the WHOLE ring with weights
      // (the x copies of those stages are deferred until the previous kernel has
      // completed): with PDL this CTA streams ~kStages stages of weights while the
      // previous GEMV's epilogue still runs.
      const uint8_t* pend_src[kStages];
      uint32_t pend_bytes[kStages];
      int pend_stage[kStages];
      int npend = 0;
      auto flush_x = [&]() {
        griddep_wait();
        waited = true;
        if (p.merge && !(p.merge & 4))  // every CTA's share of the fused LSE combine is in p.xf (see the consumers)
          while (ld_acquire_gpu_i(p.merge_ctr) < static_cast<int>(gridDim.x)) __nanosleep(32);
        for (int i = 0; i < npend; ++i)
          bulk_g2s(ring + pend_stage[i] * SB + SW, pend_src[i], pend_bytes[i], &full[pend_stage[i]]);
        npend = 0;
      };
      int n_tiles = p.n_tiles;
      if (p.group_count) {  // the active-expert list is produced by the routing kernel
        griddep_wait();
        waited = true;
        n_tiles = *p.group_count * p.tiles_per_group;
      }
      for (;;) {
        const int tile = atomicAdd(p.work_counter, 1);
        const bool done = tile >= n_tiles;
        const int gi = (done || !p.group_count) ? 0 : tile / p.tiles_per_group;
        const int rem = done ? 0 : tile - gi * p.tiles_per_group;
        const int nb = rem / p.ksplit;  // row-block-major: a block's k-chunks finish together
        const int kc = rem - nb * p.ksplit;
        const int k0 = kc * p.kr_steps;
        const int k1 = min(k0 + p.kr_steps, KST);
        const int nstage = done ? 1 : (k1 - k0 + kStageSteps - 1) / kStageSteps;
        const uint8_t* wg = reinterpret_cast<const uint8_t*>(p.w);
        const uint8_t* xg = p.xf;
        if (!done && p.group_count) {
          wg += static_cast<size_t>(p.group_ids[gi] - p.group_base) * p.w_group_stride;
          xg += static_cast<size_t>(gi) * p.xf_group_stride;
        }
        for (int si = 0; si < nstage; ++si, ++st) {
          const int s = st % kStages;
          if (st >= kStages) mbar_wait(&empty[s], ((st / kStages) & 1) ^ 1);
          TileMeta& m = meta[s];
          if (done) {
            if (!waited) flush_x();
            m.tile = kDone;
            mbar_arrive(&full[s]);
            break;
          }
          const int a = k0 + si * kStageSteps;
          const int n = min(kStageSteps, k1 - a);
          m.tile = tile;
          m.nb = nb;
          m.ks0 = a;
          m.nks = n;
          m.last = si == nstage - 1;
          m.kc = kc;
          m.gi = gi;
          uint8_t* dst = ring + s * SB;
          mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(n) * (WB + kXfTerms * NB8 * 256u));
          bulk_g2s(dst, wg + (static_cast<size_t>(nb) * KST + a) * WB, static_cast<uint32_t>(n) * WB, &full[s]);
          const uint8_t* xsrc = xg + static_cast<size_t>(a) * kXfTerms * NB8 * 256;
          const uint32_t xbytes = static_cast<uint32_t>(n) * kXfTerms * NB8 * 256u;
          if (waited) {
            bulk_g2s(dst + SW, xsrc, xbytes, &full[s]);
          } else {  // st < kStages here: no empty-slot wait can precede the flush
            pend_src[npend] = xsrc;
            pend_bytes[npend] = xbytes;
            pend_stage[npend] = s;
            if (++npend == min(max(p.prefetch_stages, 1), kStages)) flush_x();
          }
        }
        if (done) break;
      }
    }
  } else {
    // ------------------------------------------------------------ consumers
    if (p.merge) merge_prologue(p);  // fused LSE combine -> this GEMV's input fragments
    float acc[XS * NB8][4];
#pragma unroll
    for (int j = 0; j < XS * NB8; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
    const uint32_t ring_base = smem_u32(ring);
    for (int st = 0;; ++st) {
      const int s = st % kStages;
      mbar_wait(&full[s], (st / kStages) & 1);
      const TileMeta m = meta[s];
      if (m.tile == kDone) break;
      const uint32_t wbase = ring_base + s * SB + warp * (WB / 8) + lane * (WB / 256);
      const uint32_t xbase = ring_base + s * SB + SW + lane * 8;
#pragma unroll
      for (int kk = 0; kk < kStageSteps; ++kk) {
        if (WQ == 2 && kk < m.nks) {
          // FP4: the lane's 8 codes (rows g / g+8, inputs 2c, 2c+1, 2c+8, 2c+9 -- the bf16
          // chunk's order) widen exactly to f16 and take their block's 2^e (rows g, g+8)
          const uint32_t pb = ring_base + s * SB + (kk >> 1) * 2176;
          const uint32_t wv = lds32_w(pb + (kk & 1) * 1024 + warp * 128 + lane * 4);
          const uint8_t* sc = ring + s * SB + (kk >> 1) * 2176 + 2048 + warp * 16 + (lane >> 2);
          const uint32_t eg = sc[0], eg8 = sc[8];
          const uint32_t sg = (eg << 10) | (eg << 26), sg8 = (eg8 << 10) | (eg8 << 26);
          uint32_t a0, a1, a2, a3;
          e2m1x8_to_f16x2x4_w(wv, a0, a1, a2, a3);
          a0 = hmul2_w(a0, sg);
          a1 = hmul2_w(a1, sg8);
          a2 = hmul2_w(a2, sg);
          a3 = hmul2_w(a3, sg8);
#pragma unroll
          for (int t = 0; t < XS; ++t)
#pragma unroll
            for (int bg = 0; bg < NB8; ++bg) {
              const uint2 bx = lds64(xbase + ((kk * kXfTerms + t) * NB8 + bg) * 256);
              mma_f16_16816(acc[t * NB8 + bg], a0, a1, a2, a3, bx.x, bx.y);
            }
        } else if (W8 && kk < m.nks) {
          const uint2 w8 = lds64(wbase + kk * WB);
          uint32_t a0, a1, a2, a3;
          e4m3x4_to_f16x2x2(w8.x, a0, a1);
          e4m3x4_to_f16x2x2(w8.y, a2, a3);
#pragma unroll
          for (int t = 0; t < XS; ++t)
#pragma unroll
            for (int bg = 0; bg < NB8; ++bg) {
              const uint2 bx = lds64(xbase + ((kk * kXfTerms + t) * NB8 + bg) * 256);
              mma_f16_16816(acc[t * NB8 + bg], a0, a1, a2, a3, bx.x, bx.y);
            }
        } else if (kk < m.nks) {
          const uint4 wa = lds128(wbase + kk * 4096);
#pragma unroll
          for (int t = 0; t < XS; ++t)
#pragma unroll
            for (int bg = 0; bg < NB8; ++bg) {
              const uint2 bx = lds64(xbase + ((kk * kXfTerms + t) * NB8 + bg) * 256);
              mma_bf16_16816(acc[t * NB8 + bg], wa.x, wa.y, wa.z, wa.w, bx.x, bx.y);
            }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (!m.last) continue;

      // ---- tile complete: store the split-K partial of rows nb*128 + warp*16 + g (+8).
      // Plain stores: the epilogue kernel (next in stream order) reduces them.
      const int g = lane >> 2, c = lane & 3;
      const int n0 = m.nb * kRows + warp * 16 + g;
      float* yp = p.ypart + static_cast<size_t>(m.gi) * p.part_group_stride +
                  static_cast<size_t>(m.kc) * p.batch * p.Npad;
#pragma unroll
      for (int bg = 0; bg < NB8; ++bg) {
        float y[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          float v = 0.f;
#pragma unroll
          for (int t = 0; t < XS; ++t) v += acc[t * NB8 + bg][i];
          y[i] = v;
        }
        const int b0 = bg * 8 + 2 * c;
        if (b0 < p.batch) {
          yp[static_cast<size_t>(b0) * p.Npad + n0] = y[0];
          yp[static_cast<size_t>(b0) * p.Npad + n0 + 8] = y[2];
        }
        if (b0 + 1 < p.batch) {
          yp[static_cast<size_t>(b0 + 1) * p.Npad + n0] = y[1];
          yp[static_cast<size_t>(b0 + 1) * p.Npad + n0 + 8] = y[3];
        }
      }
#pragma unroll
      for (int j = 0; j < XS * NB8; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(p.work_counter + 1, 1) == static_cast<int>(gridDim.x) - 1) {
      p.work_counter[0] = 0;  // every CTA drained the queue: reset for the next launch
      p.work_counter[1] = 0;
      if (p.merge) *p.merge_ctr = 0;
      __threadfence();
    }
  }
}


// ---------------------------------------------------------------------------
// Epilogue: one CTA per 128-row block reduces the split-K partials in split
// order (deterministic) and applies the fused epilogue.
template <int NB8, int EM, bool NORM>
__global__ void __launch_bounds__(1024) gemv_epilogue_kernel(const GemvParams p) {
  // One thread per (row, request) element of a 128-row block; every global load
  // an element needs (its split partials, the old residual) is issued before use.
  extern __shared__ float stage[];  // [NP * 16][blockDim] split partials in flight
  __shared__ float s_inv[64];
  __shared__ float vt[64][kRows];
  __shared__ unsigned long long s_best[64];
  __shared__ long long s_pos[64][2];  // E_QKV: append (rank, local row) per request
  griddep_wait();
  griddep_launch_dependents();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const int nb = blockIdx.x;
  // batches above 8: one grid layer per 8 requests (more CTAs in flight; every
  // per-request reduction below stays inside its layer)
  const int bz0 = static_cast<int>(blockIdx.z) * 8, bz1 = min(p.batch, bz0 + (gridDim.z > 1 ? 8 : p.batch));
  const int rows_here = EM == E_SWIGLU ? kRows / 2 : kRows;
  const size_t stride = static_cast<size_t>(p.batch) * p.Npad;
  constexpr int NP = 2;  // partial streams per element (SwiGLU: gate + up)
  const int np = EM == E_SWIGLU ? 2 : 1;
  // grouped SwiGLU: one grid row per active expert slot
  const int gi_epi = (p.group_count && EM == E_SWIGLU) ? static_cast<int>(blockIdx.y) : 0;
  const bool combine = p.group_count && EM != E_SWIGLU;  // MoE combine (possibly of zero experts)
  // One element per thread and one staging batch: issue the split copies FIRST,
  // so their L2 round trip overlaps the RMSNorm / append-position loads below.
  const bool pre = !combine && p.ksplit > 4 && p.ksplit <= 16 && rows_here * (bz1 - bz0) <= static_cast<int>(blockDim.x);
  if (pre && static_cast<int>(threadIdx.x) < rows_here * (bz1 - bz0)) {
    const int r = threadIdx.x % rows_here, b = bz0 + threadIdx.x / rows_here;
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      if (q >= np) continue;
      const float* base = p.ypart + static_cast<size_t>(gi_epi) * p.part_group_stride +
                          static_cast<size_t>(b) * p.Npad + nb * kRows + r + q * (kRows / 2);
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < p.ksplit) cp_async4(stage + threadIdx.x + (q * 16 + j) * blockDim.x, base + j * stride);
    }
  }
  if (NORM) {
    for (int b = bz0 + warp; b < bz1; b += nwarps) {
      float ss = 0.f;
      for (int i = lane; i < p.n_ss; i += 32) ss += p.ss_part[i * p.batch + b];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if (lane == 0) s_inv[b] = rsqrtf(ss / static_cast<float>(p.K) + p.eps);
    }
  }
  if (EM == E_QKV && bz0 + static_cast<int>(threadIdx.x) < bz1) {
    const int b = bz0 + threadIdx.x;
    const long long g = p.total[b];
    s_pos[b][0] = rr_rank(g, p.rr_chunk, p.kvp);
    s_pos[b][1] = rr_row(g, p.rr_chunk, p.kvp);
  }
  if (EM == E_LOGITS && threadIdx.x < 64) s_best[threadIdx.x] = 0ull;
  // one-source pools: the attention's appended token counts from here on (the
  // merge kernel that bumped it is skipped; nothing reads the totals in between)
  if (p.bump_total && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && static_cast<int>(threadIdx.x) < p.batch)
    p.bump_total[threadIdx.x] += 1;
  if (EM == E_STORE || EM == E_RESID)
    for (int i = threadIdx.x; i < 64 * kRows; i += blockDim.x) vt[i / kRows][i % kRows] = 0.f;
  __syncthreads();
  if (p.group_count && EM == E_SWIGLU && gi_epi >= *p.group_count) {
    cp_async_wait_all();  // no copies left in flight into this CTA's shared memory
    return;
  }
  const int n_comb = combine ? *p.group_count : 0;
  uint8_t* xf_out = p.xf_out + static_cast<size_t>(gi_epi) * p.xf_out_group_stride;
  for (int e = threadIdx.x; e < rows_here * (bz1 - bz0); e += blockDim.x) {
    const int r = e % rows_here, b = bz0 + e / rows_here;
    float y[NP] = {0.f, 0.f};
    float old = 0.f;
    const int n = nb * kRows + r;
    if (EM == E_RESID && n < p.N) old = p.out[static_cast<size_t>(b) * p.out_stride + n];
    const int ngrp = combine ? n_comb : 1;
    for (int gq = 0; gq < ngrp; ++gq) {
      const int gsl = combine ? gq : gi_epi;
      float yg[NP] = {0.f, 0.f};
      // The split partials are staged through shared memory with cp.async: ptxas
      // interleaved register loads with the adds that consume them (one L2 round
      // trip per split; ncu: ~10 us for the O-proj epilogue's 16 splits), while
      // cp.async has no destination register, so all of a thread's copies are in
      // flight together. Slot (q, j) of thread t: stage[(q * 16 + j) * blockDim + t].
      float* st = stage + threadIdx.x;
      if (p.ksplit <= 4) {  // a few splits: direct loads (no staging round trip)
#pragma unroll
        for (int q = 0; q < NP; ++q) {
          if (q >= np) continue;
          const float* base = p.ypart + static_cast<size_t>(gsl) * p.part_group_stride +
                              static_cast<size_t>(b) * p.Npad + nb * kRows + r + q * (kRows / 2);
          float v[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) v[j] = j < p.ksplit ? __ldcg(base + j * stride) : 0.f;
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (j < p.ksplit) yg[q] += v[j];  // split order: deterministic
        }
      }
      if (pre) {  // copies issued at kernel entry
        cp_async_wait_all();
#pragma unroll
        for (int q = 0; q < NP; ++q) {
          if (q >= np) continue;
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (j < p.ksplit) yg[q] += st[(q * 16 + j) * blockDim.x];  // split order: deterministic
        }
      }
      for (int s0 = 0; !pre && p.ksplit > 4 && s0 < p.ksplit; s0 += 16) {
        const int nj = min(16, p.ksplit - s0);
#pragma unroll
        for (int q = 0; q < NP; ++q) {
          if (q >= np) continue;
          const float* base = p.ypart + static_cast<size_t>(gsl) * p.part_group_stride +
                              static_cast<size_t>(b) * p.Npad + nb * kRows + r + q * (kRows / 2);
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (j < nj) cp_async4(st + (q * 16 + j) * blockDim.x, base + (s0 + j) * stride);
        }
        cp_async_wait_all();
#pragma unroll
        for (int q = 0; q < NP; ++q) {
          if (q >= np) continue;
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (j < nj) yg[q] += st[(q * 16 + j) * blockDim.x];  // split order: deterministic
        }
      }
      if (p.wscale) {  // FP8 weights: this weight block's per-output power-of-two scale (exact)
        const float* ws = p.wscale + (p.group_count ? static_cast<size_t>(p.group_ids[gsl] - p.group_base) * p.Npad : 0);
        yg[0] *= ws[nb * kRows + r];
        if (EM == E_SWIGLU) yg[1] *= ws[nb * kRows + r + kRows / 2];
      }
      if (combine) {  // MoE combine in ascending expert order (deterministic)
        const float w = p.route_w[static_cast<size_t>(b) * p.n_experts + p.group_ids[gq]];
        y[0] += w * yg[0];
      } else {
        y[0] = yg[0];
        y[1] = yg[1];
      }
    }
    if (NORM) {
      y[0] *= s_inv[b];
      y[1] *= s_inv[b];
    }
    if (EM == E_SWIGLU) {
      const int f = nb * (kRows / 2) + r;
      if (f < p.N / 2) xf_write(xf_out, NB8, b, f, y[0] / (1.f + __expf(-y[0])) * y[1], p.xf16);
      continue;
    }
    if (EM == E_LOGITS) {
      // argmax: one shared atomic per warp (a warp's 32 rows share the request b;
      // 128 contending atomics per request made this epilogue ~30 us)
      unsigned long long key = 0ull;
      if (n < p.N) {
        if (p.out) p.out[static_cast<size_t>(b) * p.out_stride + n] = y[0];
        key = logit_key(y[0], n + p.n_offset);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
        key = other > key ? other : key;
      }
      if (lane == 0 && key) atomicMax(&s_best[b], key);
      continue;
    }
    if (n >= p.N) continue;
    if (p.addend) y[0] += p.addend[static_cast<size_t>(b) * p.out_stride + n];
    if (EM == E_STORE) {
      p.out[static_cast<size_t>(b) * p.out_stride + n] = y[0];
      vt[b][r] = y[0] * y[0];
    } else if (EM == E_RESID) {
      const float keep = old + y[0];
      p.out[static_cast<size_t>(b) * p.out_stride + n] = keep;
      xf_write(p.xf_out, NB8, b, n, keep, p.xf16);
      vt[b][r] = keep * keep;
    } else if (EM == E_QKV && p.mla && n >= p.nq) {
      // MLA latent row -> its round-robin page (q heads: the GQA branch below,
      // then mla_absorb_q_kernel builds the tcgen05 query image)
      {
        const int d = n - p.nq;
        if (p.kv_dbg) p.kv_dbg[static_cast<size_t>(b) * 2 * kMlaW + d] = y[0];
        if (p.append) {
          const int slot_local = static_cast<int>(s_pos[b][0]) - p.slot_base;
          const long long row = s_pos[b][1];
          if (slot_local >= 0 && slot_local < p.n_local_slots) {
            const size_t page = (static_cast<size_t>(slot_local) * p.batch + b) * p.page_cap +
                                static_cast<size_t>(row / kMlaPageRows);
            if (p.kv8)  // FP8 latents: e4m3 RNE of the fp32 row (oracle: round_e4m3)
              p.kv[page * mla_page_bytes(true) + mla_kv_offset8(static_cast<int>(row % kMlaPageRows), d)] =
                  e4m3_from_double(static_cast<double>(y[0]));
            else
              *reinterpret_cast<__nv_bfloat16*>(p.kv + page * mla_page_bytes() +
                                                mla_kv_offset(static_cast<int>(row % kMlaPageRows), d)) =
                  __float2bfloat16_rn(y[0]);
          }
        }
      }
    } else if (EM == E_QKV) {
      if (n < p.nq) {
        const int head = n / p.head_dim, d = n - head * p.head_dim;
        const int q_heads = p.nq / p.head_dim;
        p.q_out[(static_cast<size_t>(b) * q_heads + head) * p.dp + d] = y[0];
      } else {
        const int kvn = n - p.nq;
        const int is_v = kvn >= p.nk;
        const int kn = is_v ? kvn - p.nk : kvn;
        const int hl = kn / p.head_dim, d = kn - hl * p.head_dim;
        const int h = p.kv_head_base + hl;
        if (p.kv_dbg)
          p.kv_dbg[((static_cast<size_t>(b) * 2 + is_v) * p.kv_heads + hl) * p.head_dim + d] = y[0];
        if (p.append) {
          const int rank = static_cast<int>(s_pos[b][0]);
          const long long row = s_pos[b][1];
          const int grp = h / p.kvh_per_slot, kvh = h - grp * p.kvh_per_slot;
          const int slot_local = grp * p.kvp + rank - p.slot_base;
          if (slot_local >= 0 && slot_local < p.n_local_slots) {
            const size_t page =
                ((static_cast<size_t>(slot_local) * p.batch + b) * p.kvh_per_slot + kvh) * p.page_cap +
                static_cast<size_t>(row >> 4);
            if (p.kv4) {
              // FP4 block = 32 dims of this token's K or V row of one head: the warp's 32
              // lanes (32 consecutive output features, head_dim % 32 == 0) -- amax by shuffles
              float am = fabsf(y[0]);
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, o));
              const int ex = e2m1_block_exp(static_cast<double>(am));
              uint8_t* pg = p.kv + page * page_bytes_kv4(p.dp);
              bool high = false;
              const uint32_t off = kv4_offset(p.dp, static_cast<int>(row & 15), d, is_v != 0, &high);
              const uint32_t code = e2m1_from_double(static_cast<double>(y[0]), ex);
              atomicOr(reinterpret_cast<unsigned*>(pg + (off & ~3u)), code << ((off & 3u) * 8u + (high ? 4u : 0u)));
              if ((d & 31) == 0) pg[kv4_scale_offset(p.dp, static_cast<int>(row & 15), d, is_v != 0)] = kv4_scale_byte(ex, is_v != 0);
            } else {
              uint8_t* dst = p.kv + page * page_bytes_kv(p.dp, p.kv8 != 0) +
                             kv_offset(p.dp, static_cast<int>(row & 15), d, is_v != 0, p.kv8);
              if (p.kv8)
                *dst = e4m3_from_double(static_cast<double>(y[0]));
              else
                *reinterpret_cast<__nv_bfloat16*>(dst) = __float2bfloat16_rn(y[0]);
            }
          }
        }
      }
    }
  }
  if ((EM == E_STORE || EM == E_RESID) && p.ss_out) {
    __syncthreads();
    for (int b = bz0 + warp; b < bz1; b += nwarps) {
      float s = 0.f;
      for (int r = lane; r < kRows; r += 32) s += vt[b][r];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) p.ss_out[static_cast<size_t>(nb) * p.batch + b] = s;
    }
  }
  if (EM == E_LOGITS) {
    __syncthreads();
    if (bz0 + static_cast<int>(threadIdx.x) < bz1)
      atomicMax(&p.best[bz0 + threadIdx.x], s_best[bz0 + threadIdx.x]);
  }
}

size_t gemv_smem_bytes(const GemvParams& p) {
  const int nb8 = xf_nb8(p.batch);
  return static_cast<size_t>(kStages) * stage_bytes(nb8, p.w8) + kStages * sizeof(TileMeta) +
         2 * kStages * 8 + 64;
}

template <int NB8, int EM, int XS, bool NORM, int W8 = 0>
static cudaError_t launch_t(const GemvParams& p, int grid, cudaStream_t stream) {
  const size_t smem = gemv_smem_bytes(p);
  if (!p.tc) {
    cudaError_t e = smem_optin<gemv_kernel<NB8, EM, XS, NORM, W8>>(smem);
    if (e != cudaSuccess) return e;
  }
  // FP8 / FP4 weights: the consumer's per-k-step chain (widening (+ block scale)
  // + 2 MMAs) is latency-bound at 8 warps per SM, so two (e4m3) or three (e2m1,
  // smaller stages) CTAs per SM: FP4 step -3.8% vs two, FP8 best at two
  // (tools/time_step.py across processes, HX_W8_CTAS)
  static const int w8_ctas = std::getenv("HX_W8_CTAS") ? std::atoi(std::getenv("HX_W8_CTAS")) : 0;
  const int g = W8 ? grid * (w8_ctas > 0 ? w8_ctas : (W8 == 2 ? 3 : 2)) : grid;
  if (p.merge && p.tc) return cudaErrorInvalidValue;  // the tcgen05 GEMV has no merge prologue
  if (p.merge) {
    // the fused combine needs every CTA of the grid resident at once (CTAs wait
    // for each other's share): refuse a grid that cannot be
    int per_sm = 0, dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gemv_kernel<NB8, EM, XS, NORM, W8>, kThreads + 32, smem);
    if (per_sm * sms < g) return cudaErrorCooperativeLaunchTooLarge;
  }
  cudaError_t e = p.tc ? launch_gemv_tc(p, NB8, XS, grid, stream)
                       : launch_k(gemv_kernel<NB8, EM, XS, NORM, W8>, dim3(g), dim3(kThreads + 32), smem, stream, p);
  if (e != cudaSuccess) return e;
  const int rows_here = EM == E_SWIGLU ? kRows / 2 : kRows;
  const int gz = p.batch > 8 ? (p.batch + 7) / 8 : 1;  // one grid layer per 8 requests
  const int per = p.batch > 8 ? 8 : p.batch;
  const int threads = std::min(1024, (rows_here * per + 31) / 32 * 32);
  const int gy = (p.group_count && EM == E_SWIGLU) ? p.n_groups_max : 1;
  const size_t epi_smem = p.ksplit <= 4 ? 0 : static_cast<size_t>(EM == E_SWIGLU ? 2 : 1) * 16 * threads * sizeof(float);
  if (epi_smem > 0) {
    e = smem_optin<gemv_epilogue_kernel<NB8, EM, NORM>>(epi_smem);
    if (e != cudaSuccess) return e;
  }
  return launch_k(gemv_epilogue_kernel<NB8, EM, NORM>, dim3(p.Npad / kRows, gy, gz), dim3(threads), epi_smem,
                  stream, p);
}

template <int NB8>
static cudaError_t dispatch_nb(const GemvParams& p, int norm, int em, int grid, cudaStream_t s) {
  if constexpr (NB8 <= 2) {
    if (p.w8) {  // FP8 / FP4 weights: two f16 activation terms (22 bits) serve every projection
#define HX_CASE8(E, NORMV)                                                                       \
  if (em == E && (norm != 0) == NORMV)                                                           \
    return p.w8 == 2 ? launch_t<NB8, E, 2, NORMV, 2>(p, grid, s) : launch_t<NB8, E, 2, NORMV, 1>(p, grid, s);
      HX_CASE8(E_QKV, true)
      HX_CASE8(E_QKV, false)
      HX_CASE8(E_RESID, false)
      HX_CASE8(E_STORE, false)
      HX_CASE8(E_STORE, true)  // MoE router (f16 terms: 22 bits, like 3 bf16 terms' ~24)
      HX_CASE8(E_SWIGLU, true)
      HX_CASE8(E_LOGITS, true)
#undef HX_CASE8
      return cudaErrorInvalidValue;
    }
  }
  // QKV feeds exp(q.k) with |logits| up to ~1e3 under the reference's unscaled
  // weights: carry x at fp32 precision there (3 bf16 terms), 2 terms elsewhere.
#define HX_CASE(E, XS, NORMV) \
  if (em == E && (norm != 0) == NORMV) return launch_t<NB8, E, XS, NORMV>(p, grid, s);
  HX_CASE(E_QKV, 3, true)
  HX_CASE(E_QKV, 3, false)
  HX_CASE(E_RESID, 2, false)
  HX_CASE(E_STORE, 2, false)
  HX_CASE(E_STORE, 3, true)  // MoE router: fp32-accurate logits keep top-k ties rare
  HX_CASE(E_SWIGLU, 2, true)
  HX_CASE(E_LOGITS, 2, true)
#undef HX_CASE
  return cudaErrorInvalidValue;
}

cudaError_t launch_gemv(const GemvParams& p, int norm, int emode, int grid, cudaStream_t stream) {
  if (p.batch < 1 || p.batch > 64 || (p.K & 15) || (p.Npad % kRows)) return cudaErrorInvalidValue;
  if (p.tc && p.batch <= 16) return cudaErrorInvalidValue;  // tcgen05 path: N = 32 or 64 batch rows
  if (p.w8 && (p.tc || p.batch > 16 || (p.w8 == 1 && !p.wscale) || (p.w8 == 2 && (p.K & 31))))
    return cudaErrorInvalidValue;
  if (p.batch <= 8) return dispatch_nb<1>(p, norm, emode, grid, stream);
  if (p.batch <= 16) return dispatch_nb<2>(p, norm, emode, grid, stream);
  if (p.batch <= 32) return dispatch_nb<4>(p, norm, emode, grid, stream);
  return dispatch_nb<8>(p, norm, emode, grid, stream);
}

}  // namespace hx
