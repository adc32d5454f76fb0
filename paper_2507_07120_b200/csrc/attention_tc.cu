// K1-TC: GQA flash-decode partial attention over QUANTISED KV pages (FP8 e4m3,
// FP4 e2m1 blocks) on the 5th-generation tensor cores (tcgen05 + TMEM).
//
// Same contract as attn_decode_kernel (attention.cu): per work item (stream =
// (rank slot, request, KV head), split = page range) the locally normalised
// partial output and log2-sum-exp of every query head of the GQA group --
// HeadFragment of partial_head_attention (reference attention.hpp:56-78,
// :375-396) -- so the split reduce / merge / exchange path is unchanged.
//
// Why a second kernel: the legacy-HMMA kernel widens every KV element into
// mma.sync operands on the consumer warps, and with 16 query rows (405B-like
// G = 16) or 4-bit pages the widen + MMA issue chain, not HBM, bounds it
// (FP8 G16 66%, FP4 33-47% of the copy bandwidth; K1-FP4).
// Here the tensor core does all the MACs and each KV byte is widened once:
//
//   tile = 128 tokens (8 pages), transposed formulation (token = TMEM lane):
//   S^T [128 tok x NC] = K [128 tok x 128 dim] . Q^T        (A = K f16 in TMEM)
//   O^T [128 dim x NC] += V^T [128 dim x 128 tok] . P^T     (A = V^T f16 in TMEM)
//   NC = 2 * NQ columns: (term, query) -- q and P each split into f16 hi + lo
//   (22 significant bits), so as in the legacy kernel the only rounding is the
//   KV storage itself (e4m3 / e2m1 x 2^e values are exact in f16).
//
// One CTA per SM, two ITEM SLOTS whose tiles alternate through the shared converters:
//   warps 0-3 / 4-7   softmax of slot 0 / 1 (thread = token lane of S^T, = dim
//                     lane of O^T): lazy online softmax (rescale only when a
//                     query's max grows by > 8 in log2 units, found with one
//                     barrier.red.or), P^T hi/lo into shared memory, the rare
//                     O^T rescale in TMEM, the item's partial at its end
//   warps 8-11        K converters: thread = token t; K's 128 dims (FP8 8-byte /
//                     FP4 4-byte fragment chunks of the page) widen to f16 and go
//                     to TMEM lane t (tcgen05.st) (+ the item's query image)
//   warps 12-15       V converters: thread = dim d; d's 16 tokens per page -> lane d
//   warp 16           producer: cp.async.bulk of each tile's 8 pages (+ the
//                     item's query rows) into a shared-memory ring
//   warp 17           MMA issue (elected lane of the converged warp): S(i+1), PV(i)
// (18 warps: the sub-partitions holding 5 cap registers at 96 per thread)
// MMAs are issued from converged warps by one elected lane (descriptors stay
// warp-uniform: ~21 cycles per tcgen05.mma, tools/tc_issue_probe.cu).
// Work is statically assigned (item = unit + n * units, unit = 2 CTA + slot):
// every role walks the same deterministic tile sequence, so only mbarrier
// phases pass between roles.
#include <cstdio>

#include "common.cuh"
#include "kernels.h"
#include "kv_layout.cuh"
#include "tc05.cuh"

namespace hx {

namespace {

constexpr int kTcDP = 128;  // head dim (padded) this kernel serves
constexpr int kTcThreads = 576;
constexpr int kWarpKConv = 8, kWarpVConv = 12, kWarpProd = 16, kWarpMma = 17;

template <int NQ, int KVF, int NST>
struct TcCfg {
  static constexpr int NC = 2 * NQ;                                   // MMA N
  static constexpr int NV = NC == 32 ? 3 : 4;                         // V buffers in TMEM
  static constexpr uint32_t PAGE = KVF == 2 ? 35u * kTcDP / 2u : 32u * kTcDP;
  static constexpr uint32_t STAGE = 8 * PAGE;                          // 8 pages = 128 tokens
  static constexpr uint32_t QRAW = NQ * kTcDP * 4;                    // fp32 query rows
  static constexpr uint32_t QIMG = NC * kTcDP * 2;                    // Q^T f16, K-major core matrices
  static constexpr uint32_t PBUF = 128 * NC * 2;                      // P^T f16, MN-major core matrices
  static constexpr uint32_t OFF_QIMG = NST * STAGE;                   // (STAGE % 128 == 0)
  static constexpr uint32_t OFF_PBUF = OFF_QIMG + 2 * QIMG;           // [slot][2]
  static constexpr uint32_t OFF_QRAW = OFF_PBUF + 4 * PBUF;           // [slot]
  static constexpr uint32_t OFF_RED = OFF_QRAW + 2 * QRAW;            // float [slot][4 warps][NQ]
  static constexpr uint32_t OFF_BAR = OFF_RED + 2 * 4 * NQ * 4;
  static constexpr int NBAR = 2 * NST + 2 * NV + 28;
  static constexpr uint32_t SMEM = OFF_BAR + NBAR * 8 + 16;
  // TMEM columns: K x2 | V x NV | S [slot][2] | O [slot]
  static constexpr uint32_t COL_K = 0, COL_V = 128, COL_S = 128 + 64 * NV, COL_O = COL_S + 4 * NC;
  static_assert(COL_O + 2 * NC <= 512, "TMEM columns");
  // instruction descriptors (kind::f16, f16 x f16 -> f32): S^T (B = Q^T K-major), O^T (B = P^T MN-major)
  static constexpr uint32_t IDESC_S = (1u << 4) | (static_cast<uint32_t>(NC >> 3) << 17) | (128u >> 4 << 24);
  static constexpr uint32_t IDESC_O = IDESC_S | (1u << 16);
};

// barrier indices
template <int NST, int NV>
struct TcBars {
  static constexpr int RAW_FULL = 0, RAW_EMPTY = NST;
  static constexpr int KFULL = 2 * NST, KFREE = KFULL + 2, VFULL = KFREE + 2, VFREE = VFULL + NV;
  static constexpr int SFULL = VFREE + NV, SFREE = SFULL + 4;  // [slot][buffer]
  static constexpr int PFULL = SFREE + 4, ODONE = PFULL + 4;   // [slot][P buffer]
  static constexpr int QFREE = ODONE + 4, QRAWFREE = QFREE + 2;  // [slot]
};

struct TcTile {
  int slot, item, np, ntok, rows, first, last;
  int tok0;           // first token (within the stream's shard) of the tile
  const uint8_t* kv;  // the tile's first page
  const float* q;     // the item's query rows
};

// Deterministic tile sequence of this CTA (every role runs one): two item
// slots, tiles alternate between them while both have work. Slot state lives in
// two named members (no runtime-indexed arrays: with ~200 KB of shared memory
// the L1 left for a local-memory stack is tiny, and a stack round trip to L2
// per tile costs ~0.3 us).
struct TcSlot {
  int kord, item, tile, ntiles, pg0, pg1, ntok, rows;
  const uint8_t* kvs;
  const float* q;
  bool act;
};
struct TcSeq {
  const AttnParams* p;
  int units, unit0, last;
  uint32_t page_bytes;
  TcSlot s0, s1;

  __device__ void load(TcSlot& S, int g) {
    for (;;) {
      const long long it = static_cast<long long>(S.kord++) * units + unit0 + g;
      if (it >= p->n_items) {
        S.act = false;
        return;
      }
      const int iti = static_cast<int>(it);
      // split-major (the tcgen05 kernel never runs the HOP-B order: attn_tc_supported)
      const int split = iti / p->n_streams;
      const int stream = iti - split * p->n_streams;
      int t = stream;
      const int qc = t % p->q_chunks;
      t /= p->q_chunks;
      const int kvh = t % p->kvh_per_slot;
      t /= p->kvh_per_slot;
      const int bl = t % p->stream_batch;
      const int sl = t / p->stream_batch;
      const int b = bl + p->b_begin;
      const int slot = sl + p->slot_base;
      const int rank = slot % p->kvp;
      const int nt = static_cast<int>(rr_count(p->total[b], rank, p->chunk, p->kvp));
      const int pages = (nt + 15) >> 4;
      const int a = static_cast<int>((static_cast<long long>(split) * pages) / p->splits);
      const int e = static_cast<int>((static_cast<long long>(split + 1) * pages) / p->splits);
      if (e <= a) continue;  // empty split: nothing to emit (the split reduce skips it)
      S.item = iti;
      S.tile = 0;
      S.ntiles = (e - a + 7) >> 3;
      S.pg0 = a;
      S.pg1 = e;
      S.ntok = nt;
      const int g_rows = p->group - qc * p->qrows;
      S.rows = g_rows < p->qrows ? g_rows : p->qrows;
      const size_t pool_stream = (static_cast<size_t>(sl) * p->batch + b) * p->kvh_per_slot + kvh;
      S.kvs = p->kv + pool_stream * p->page_cap * static_cast<size_t>(page_bytes);
      const int grp = slot / p->kvp;
      const int head0 = ((grp - p->q_grp_base) * p->kvh_per_slot + kvh) * p->group + qc * p->qrows;
      S.q = p->q + (static_cast<size_t>(b) * p->q_heads + head0) * kTcDP;
      S.act = true;
      return;
    }
  }
  __device__ void init(const AttnParams& pp, uint32_t pb) {
    p = &pp;
    page_bytes = pb;
    units = 2 * gridDim.x;
    unit0 = 2 * blockIdx.x;
    s0.kord = s1.kord = 0;
    last = 1;
    load(s0, 0);
    load(s1, 1);
  }
  __device__ void emit(TcSlot& S, int g, TcTile& t) {
    last = g;
    t.slot = g;
    t.item = S.item;
    const int a = S.pg0 + 8 * S.tile;
    t.np = min(8, S.pg1 - a);
    t.ntok = S.ntok;
    t.rows = S.rows;
    t.first = S.tile == 0;
    t.last = S.tile == S.ntiles - 1;
    t.tok0 = a * 16;
    t.kv = S.kvs + static_cast<size_t>(a) * page_bytes;
    t.q = S.q;
    if (++S.tile == S.ntiles) load(S, g);
  }
  __device__ bool next(TcTile& t) {
    const bool want1 = last == 0;  // alternate
    if (want1 ? s1.act : !s0.act) {
      if (!s1.act) return false;
      emit(s1, 1, t);
    } else {
      if (!s0.act) return false;
      emit(s0, 0, t);
    }
    return true;
  }
};

HX_DEV uint32_t tm_lane(uint32_t tbase, int warp) { return tbase + (static_cast<uint32_t>((warp & 3) * 32) << 16); }

HX_DEV void tmem_st32u(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
HX_DEV void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
template <int N>
HX_DEV void tmem_ldn(uint32_t taddr, float (&v)[N]) {
  if constexpr (N == 32) {
    tmem_ld32(taddr, v);
  } else {
    tmem_ld16(taddr, v);
  }
}
template <int N>
HX_DEV void tmem_stn(uint32_t taddr, float (&v)[N]) {
  if constexpr (N == 32) {
    tmem_st32(taddr, v);
  } else {
    uint32_t r[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(v[i]);
    tmem_st16(taddr, r);
  }
}

HX_DEV uint32_t lds32_(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
HX_DEV void e2m1x4_to_f16x2x2(uint32_t two_bytes, uint32_t& lo, uint32_t& hi) {
  asm("{\n .reg .b8 b0, b1, b2, b3;\n mov.b32 {b0, b1, b2, b3}, %2;\n"
      " cvt.rn.f16x2.e2m1x2 %0, b0;\n cvt.rn.f16x2.e2m1x2 %1, b1;\n}"
      : "=r"(lo), "=r"(hi)
      : "r"(two_bytes));
}
HX_DEV uint32_t hmul2_(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
HX_DEV uint32_t pack_f16x2(float lo, float hi) {
  uint32_t d;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}
HX_DEV float2 unpack_f16x2(uint32_t v) {
  const __half2 h = *reinterpret_cast<const __half2*>(&v);
  return __half22float2(h);
}


#ifdef HX_TC_TRACE
__device__ unsigned long long g_tc_trace[64][8];
__device__ unsigned long long g_tc_v[64][4];
__device__ unsigned long long g_tc_k[64][6];
HX_DEV unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TC_TRACE(i, ev) \
  do { if (blockIdx.x == 0 && (i) < 64 && (threadIdx.x & 31) == 0) g_tc_trace[i][ev] = gtime(); } while (0)
#else
#define TC_TRACE(i, ev) do {} while (0)
#endif
}  // namespace

template <int NQ, int KVF, int NST>
__global__ void __launch_bounds__(kTcThreads, 1) attn_tc_kernel(const __grid_constant__ AttnParams p) {
  using C = TcCfg<NQ, KVF, NST>;
  constexpr int NV = C::NV;
  using Bn = TcBars<NST, NV>;
  constexpr int NC = C::NC;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + C::OFF_BAR + C::NBAR * 8);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&bars[Bn::RAW_FULL + s], 1);
      mbar_init(&bars[Bn::RAW_EMPTY + s], 8);  // 4 K + 4 V converter warps
    }
    for (int v = 0; v < NV; ++v) {
      mbar_init(&bars[Bn::VFULL + v], 4);
      mbar_init(&bars[Bn::VFREE + v], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars[Bn::KFULL + i], 4);
      mbar_init(&bars[Bn::KFREE + i], 1);
      mbar_init(&bars[Bn::QFREE + i], 1);
      mbar_init(&bars[Bn::QRAWFREE + i], 4);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&bars[Bn::SFULL + i], 1);
      mbar_init(&bars[Bn::SFREE + i], 4);
      mbar_init(&bars[Bn::PFULL + i], 4);
      mbar_init(&bars[Bn::ODONE + i], 1);
    }
    fence_mbar_init();
  }
  if (warp == kWarpMma) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  griddep_launch_dependents();
  const uint32_t tbase = *tslot;
  const uint32_t sbase = smem_u32(smem);

  TcSeq seq;
  seq.init(p, C::PAGE);
  TcTile t;

  if (warp >= kWarpKConv && warp < kWarpVConv) {
    // ---------------------------------------------------------------- K converters (thread = token) + S issue
    const int tl = threadIdx.x - kWarpKConv * 32;
    const int page = tl >> 4, r = tl & 15, nt = r >> 3, g8 = r & 7;
    const uint32_t lane_addr = tm_lane(tbase, warp);
    int nitem0 = 0, nitem1 = 0;
    for (int i = 0; seq.next(t); ++i) {
      const int s = i % NST, kb = i & 1, g = t.slot;
#ifdef HX_TC_TRACE
      if (blockIdx.x == 0 && i < 64 && threadIdx.x == kWarpKConv * 32) g_tc_k[i][0] = gtime();
#endif
      mbar_wait(&bars[Bn::RAW_FULL + s], (i / NST) & 1);
#ifdef HX_TC_TRACE
      if (blockIdx.x == 0 && i < 64 && threadIdx.x == kWarpKConv * 32) g_tc_k[i][1] = gtime();
#endif
      if (t.first) {
        // the slot's query image: previous item's S MMAs done, then this item's rows
        const int ni = g ? nitem1++ : nitem0++;
        if (ni > 0) mbar_wait(&bars[Bn::QFREE + g], (ni - 1) & 1);
        const float* qs = reinterpret_cast<const float*>(smem + C::OFF_QRAW + g * C::QRAW);
        uint8_t* qi = smem + C::OFF_QIMG + g * C::QIMG;
        for (int u = tl; u < NQ * 16; u += 128) {
          const int q = u % NQ, dg = u / NQ;
          uint32_t h[4], l[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float x0 = q < t.rows ? qs[q * kTcDP + dg * 8 + 2 * e] * p.qscale : 0.f;
            const float x1 = q < t.rows ? qs[q * kTcDP + dg * 8 + 2 * e + 1] * p.qscale : 0.f;
            h[e] = pack_f16x2(x0, x1);
            const float2 hf = unpack_f16x2(h[e]);
            l[e] = pack_f16x2(x0 - hf.x, x1 - hf.y);
          }
          // [dg][cg][c%8][d%8]: hi term in column q, lo term in column NQ + q
          *reinterpret_cast<uint4*>(qi + (dg * (NC / 8) + (q >> 3)) * 128 + (q & 7) * 16) =
              make_uint4(h[0], h[1], h[2], h[3]);
          *reinterpret_cast<uint4*>(qi + (dg * (NC / 8) + ((NQ + q) >> 3)) * 128 + (q & 7) * 16) =
              make_uint4(l[0], l[1], l[2], l[3]);
        }
        fence_proxy_async();  // generic-proxy image writes -> the tensor core's async proxy
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[Bn::QRAWFREE + g]);
      }
      if (i >= 2) mbar_wait(&bars[Bn::KFREE + kb], ((i >> 1) - 1) & 1);
      tc_fence_after();
      TC_TRACE(i, 1);
      // this token's K row: every load issued first (rows of pages past np hold
      // stale bytes; their logits are masked by the softmax, so no zeroing)
      const uint32_t pbase = sbase + s * C::STAGE + page * C::PAGE;
      uint4 kv[8];
      uint32_t ex = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if constexpr (KVF == 1) {
          kv[j] = lds128(pbase + (((nt * 4 + (j >> 1)) * 32 + g8 * 4 + 2 * (j & 1)) * 8));  // kp = j/2, chunks 2(j%2)..+1
        } else if (j < 4) {
          kv[j] = lds128(pbase + (((nt * 4 + j) * 32 + g8 * 4) * 4));  // kp = j: chunks c = 0..3
        }
      }
      if constexpr (KVF == 2) ex = lds32_(pbase + 16 * kTcDP + r * 4);  // this token's 4 block exponents
#pragma unroll
      for (int half = 0; half < 2; ++half) {  // dims [64 half, 64 half + 64) -> columns [32 half, +32)
        uint32_t w[32];
#pragma unroll
        for (int kq = 0; kq < 2; ++kq) {
          const int kp = 2 * half + kq;
          if constexpr (KVF == 1) {
#pragma unroll
            for (int c2 = 0; c2 < 2; ++c2) {  // chunks c = 2 c2, 2 c2 + 1
              const uint4 v = kv[2 * kp + c2];
              const uint32_t wd[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
              for (int cc = 0; cc < 2; ++cc) {
                const int c = 2 * c2 + cc;
                uint32_t a0, a1, a2, a3;
                e4m3x4_to_f16x2x2(wd[2 * cc], a0, a1);
                e4m3x4_to_f16x2x2(wd[2 * cc + 1], a2, a3);
                w[16 * kq + c] = a0;       // dims 32kp + 2c, +1
                w[16 * kq + 4 + c] = a1;   // +8, +9
                w[16 * kq + 8 + c] = a2;   // +16, +17
                w[16 * kq + 12 + c] = a3;  // +24, +25
              }
            }
          } else {
            const uint32_t sc = ((ex >> (8 * kp)) & 0xFFu) << 10;
            const uint32_t ss = sc | (sc << 16);
            const uint4 v = kv[kp];
            const uint32_t wd[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              uint32_t a0, a1, a2, a3;
              e2m1x4_to_f16x2x2(wd[c] & 0xFFFFu, a0, a1);
              e2m1x4_to_f16x2x2(wd[c] >> 16, a2, a3);
              w[16 * kq + c] = hmul2_(a0, ss);
              w[16 * kq + 4 + c] = hmul2_(a1, ss);
              w[16 * kq + 8 + c] = hmul2_(a2, ss);
              w[16 * kq + 12 + c] = hmul2_(a3, ss);
            }
          }
        }
        tmem_st32u(lane_addr + C::COL_K + kb * 64 + 32 * half, w);
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      TC_TRACE(i, 2);
      if (lane == 0) {
        mbar_arrive(&bars[Bn::KFULL + kb]);
        mbar_arrive(&bars[Bn::RAW_EMPTY + s]);
      }
    }
  } else if (warp == kWarpMma) {
    // ---------------------------------------------------------------- MMA issue: S(i+1) before PV(i)
    // The whole warp walks the sequence and waits (converged, so descriptors stay
    // warp-uniform); one elected lane issues each batch (a lone-lane issue loop
    // costs ~145 cycles per tcgen05.mma in R2UR / waterfall code; converged, 8
    // unrolled MMAs issue at ~21 cycles each: tools/tc_issue_probe.cu).
    const uint64_t qdesc0 = umma_desc(sbase + C::OFF_QIMG, (NC / 8) * 128, 128);
    const uint64_t pdesc0 = umma_desc(sbase + C::OFF_PBUF, 128, 16 * 128);
    int jslot0 = 0, jslot1 = 0;
    bool pend = false;
    int pi = 0, pg = 0, pj = 0, pfirst = 0;
    auto issue_pv = [&](int i, int g, int j, int first) {
      const int vb = i % NV, pb = j & 1;
      mbar_wait(&bars[Bn::VFULL + vb], (i / NV) & 1);
      mbar_wait(&bars[Bn::PFULL + 2 * g + pb], (j >> 1) & 1);
      tc_fence_after();
      const uint32_t acol = tbase + C::COL_V + vb * 64, dcol = tbase + C::COL_O + g * NC;
      const uint64_t pdesc = pdesc0 + static_cast<uint64_t>(((2 * g + pb) * C::PBUF) >> 4);
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          umma_ts(dcol, acol + k * 8, pdesc + static_cast<uint64_t>((k * 256) >> 4), C::IDESC_O,
                  (first && k == 0) ? 0u : 1u);
        umma_commit(&bars[Bn::VFREE + vb]);
        umma_commit(&bars[Bn::ODONE + 2 * g + pb]);
      }
      __syncwarp();
    };
    for (int i = 0; seq.next(t); ++i) {
      const int kb = i & 1, g = t.slot, j = g ? jslot1++ : jslot0++, sb = j & 1;
      mbar_wait(&bars[Bn::KFULL + kb], (i >> 1) & 1);
      if (j >= 2) mbar_wait(&bars[Bn::SFREE + 2 * g + sb], ((j >> 1) - 1) & 1);
      tc_fence_after();
      const uint32_t dcol = tbase + C::COL_S + (2 * g + sb) * NC, acol = tbase + C::COL_K + kb * 64;
      const uint64_t qdesc = qdesc0 + static_cast<uint64_t>((g * C::QIMG) >> 4);
      const bool lst = t.last;
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          umma_ts(dcol, acol + k * 8, qdesc + static_cast<uint64_t>((k * NC * 32) >> 4), C::IDESC_S,
                  k > 0 ? 1u : 0u);
        umma_commit(&bars[Bn::SFULL + 2 * g + sb]);
        umma_commit(&bars[Bn::KFREE + kb]);
        if (lst) umma_commit(&bars[Bn::QFREE + g]);
      }
      __syncwarp();
      TC_TRACE(i, 5);
      if (pend) issue_pv(pi, pg, pj, pfirst);
      pend = true;
      pi = i;
      pg = g;
      pj = j;
      pfirst = t.first;
    }
    if (pend) issue_pv(pi, pg, pj, pfirst);
  } else if (warp == kWarpProd) {
    // ---------------------------------------------------------------- producer (one lane; a bulk-copy
    // issue blocks its warp ~0.3 us, so it has a warp of its own)
    if (lane == 0) {
      bool waited = false;
      int nitem0 = 0, nitem1 = 0;
      for (int i = 0; seq.next(t); ++i) {
        const int s = i % NST;
        if (i >= NST) mbar_wait(&bars[Bn::RAW_EMPTY + s], ((i / NST) - 1) & 1);
        const uint32_t bytes = t.np * C::PAGE;
        const uint32_t qbytes = t.first ? static_cast<uint32_t>(t.rows) * kTcDP * 4 : 0u;
        if (t.first) {
          const int ni = t.slot ? nitem1++ : nitem0++;
          if (ni > 0) mbar_wait(&bars[Bn::QRAWFREE + t.slot], (ni - 1) & 1);  // the slot's previous rows consumed
        }
        TC_TRACE(i, 0);
        mbar_arrive_expect_tx(&bars[Bn::RAW_FULL + s], bytes + qbytes);
        bulk_g2s(smem + s * C::STAGE, t.kv, bytes, &bars[Bn::RAW_FULL + s]);  // KV: no dependency
        if (!waited) {
          griddep_wait();  // query rows come from the QKV kernel
          waited = true;
        }
        if (qbytes) bulk_g2s(smem + C::OFF_QRAW + t.slot * C::QRAW, t.q, qbytes, &bars[Bn::RAW_FULL + s]);
      }
      if (!waited) griddep_wait();
    }
  } else if (warp >= kWarpVConv) {
    // ---------------------------------------------------------------- V converters (thread = dim)
    const int d = threadIdx.x - kWarpVConv * 32;
    const int vnd = d >> 3, vg8 = d & 7, nd2 = vnd >> 1, sub = vnd & 1;
    const uint32_t lane_addr = tm_lane(tbase, warp);
    for (int i = 0; seq.next(t); ++i) {
      const int s = i % NST, vb = i % NV;
#ifdef HX_TC_TRACE
      if (blockIdx.x == 0 && i < 64 && threadIdx.x == kWarpVConv * 32) g_tc_v[i][0] = gtime();
#endif
      mbar_wait(&bars[Bn::RAW_FULL + s], (i / NST) & 1);
#ifdef HX_TC_TRACE
      if (blockIdx.x == 0 && i < 64 && threadIdx.x == kWarpVConv * 32) g_tc_v[i][1] = gtime();
#endif
      if (i >= NV) mbar_wait(&bars[Bn::VFREE + vb], ((i / NV) - 1) & 1);
      tc_fence_after();
      TC_TRACE(i, 3);
      const uint32_t stage = sbase + s * C::STAGE;
#pragma unroll
      for (int half = 0; half < 2; ++half) {  // pages [4 half, 4 half + 4) -> columns [32 half, +32)
        // all of the half's shared-memory loads first (pages past np read stale
        // bytes and are zeroed below), then the widening
        uint4 v0[4], v1[4], v2[4];
#pragma unroll
        for (int pq = 0; pq < 4; ++pq) {
          const uint32_t pbase = stage + (4 * half + pq) * C::PAGE;
          if constexpr (KVF == 1) {
            // chunks c = 0..3 of (nd2, g8): 32 contiguous bytes; this dim's 4 bytes of each
            const uint32_t cb = pbase + 16 * kTcDP + (nd2 * 32 + vg8 * 4) * 8;
            v0[pq] = lds128(cb);
            v1[pq] = lds128(cb + 16);
          } else {
            v0[pq] = lds128(pbase + 8 * kTcDP + (nd2 * 32 + vg8 * 4) * 4);
            v1[pq] = lds128(pbase + 16 * kTcDP + kTcDP / 2 + (d >> 5) * 32);  // f16x2 scales, tokens 0..7
            v2[pq] = lds128(pbase + 16 * kTcDP + kTcDP / 2 + (d >> 5) * 32 + 16);  // tokens 8..15
          }
        }
        uint32_t w[32];
#pragma unroll
        for (int pq = 0; pq < 4; ++pq) {
          const bool have = 4 * half + pq < t.np;
          if constexpr (KVF == 1) {
            const uint32_t wd[4] = {sub ? v0[pq].y : v0[pq].x, sub ? v0[pq].w : v0[pq].z, sub ? v1[pq].y : v1[pq].x,
                                    sub ? v1[pq].w : v1[pq].z};
#pragma unroll
            for (int c = 0; c < 4; ++c) {  // tokens (2c, 2c+1) and (2c+8, 2c+9)
              uint32_t lo, hi;
              e4m3x4_to_f16x2x2(have ? wd[c] : 0u, lo, hi);
              w[8 * pq + c] = lo;
              w[8 * pq + 4 + c] = hi;
            }
          } else {
            const uint32_t wd[4] = {v0[pq].x, v0[pq].y, v0[pq].z, v0[pq].w};
            const uint32_t s0w[4] = {v1[pq].x, v1[pq].y, v1[pq].z, v1[pq].w};  // (2^e_2c, 2^e_2c+1)
            const uint32_t s1w[4] = {v2[pq].x, v2[pq].y, v2[pq].z, v2[pq].w};  // tokens 2c+8, 2c+9
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              uint32_t a0, a1;
              e2m1x4_to_f16x2x2(__byte_perm(wd[c], 0u, sub ? 0x3232u : 0x1010u), a0, a1);
              // pages past np: stale bytes (a stale scale may be inf / nan) -> exact zeros
              w[8 * pq + c] = have ? hmul2_(a0, s0w[c]) : 0u;
              w[8 * pq + 4 + c] = have ? hmul2_(a1, s1w[c]) : 0u;
            }
          }
        }
        tmem_st32u(lane_addr + C::COL_V + vb * 64 + 32 * half, w);
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      TC_TRACE(i, 4);
      if (lane == 0) {
        mbar_arrive(&bars[Bn::VFULL + vb]);
        mbar_arrive(&bars[Bn::RAW_EMPTY + s]);
      }
#ifdef HX_TC_TRACE
      if (blockIdx.x == 0 && i < 64 && threadIdx.x == kWarpVConv * 32) g_tc_v[i][2] = gtime();
#endif
    }
  } else {
    // ---------------------------------------------------------------- softmax + PV (slot g)
    const int g = warp >> 2, wq = warp & 3;
    const int tl = threadIdx.x - g * 128;  // token lane of S^T, dim lane of O^T
    const uint32_t lane_addr = tm_lane(tbase, warp);
    const int barid = 1 + g;
    float* red = reinterpret_cast<float*>(smem + C::OFF_RED) + g * 4 * NQ;
    const uint32_t prow = sbase + C::OFF_PBUF + (2 * g) * C::PBUF + (tl >> 3) * 128 + (tl & 7) * 16;
    const uint64_t pdesc0 = umma_desc(sbase + C::OFF_PBUF + (2 * g) * C::PBUF, 128, 16 * 128);
    float m[NQ], l[NQ];
    int j = 0;
    for (int i = 0; seq.next(t); ++i) {
      if (t.slot != g) continue;
      const int sb = j & 1;
      mbar_wait(&bars[Bn::SFULL + 2 * g + sb], (j >> 1) & 1);
      tc_fence_after();
      TC_TRACE(i, 6);
      float sv[NC];
      tmem_ldn<NC>(lane_addr + C::COL_S + (2 * g + sb) * NC, sv);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[Bn::SFREE + 2 * g + sb]);
      if (t.first) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          m[q] = -INFINITY;
          l[q] = 0.f;
        }
      }
      const bool valid = tl < t.np * 16 && t.tok0 + tl < t.ntok;
      float s[NQ];
      bool grow = false;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        s[q] = valid ? sv[q] + sv[NQ + q] : -INFINITY;
        grow |= s[q] > m[q] + 8.f;
      }
      bool rescale = false;
      float alpha[NQ];
      if (bar_red_or(barid, 128, grow)) {
        // tile maxima per query over the 128 token lanes
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const float mx = redux_max_f32(s[q]);
          if (lane == 0) red[wq * NQ + q] = mx;
        }
        named_bar(barid, 128);
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const float tm = fmaxf(fmaxf(red[q], red[NQ + q]), fmaxf(red[2 * NQ + q], red[3 * NQ + q]));
          const float mn = tm > m[q] + 8.f ? tm : m[q];
          alpha[q] = fast_exp2(m[q] - mn);  // 0 when m = -inf
          rescale |= mn != m[q];
          l[q] *= alpha[q];
          m[q] = mn;
        }
        rescale = rescale && !t.first;  // a new item's first PV overwrites O^T
      }
      // P^T buffer sb of this slot: PV(j-2) done
      if (j >= 2) mbar_wait(&bars[Bn::ODONE + 2 * g + sb], ((j >> 1) - 1) & 1);
      {
        uint32_t ph[NQ / 2], pl[NQ / 2];
#pragma unroll
        for (int q2 = 0; q2 < NQ / 2; ++q2) {
          const float p0 = fast_exp2(s[2 * q2] - m[2 * q2]), p1 = fast_exp2(s[2 * q2 + 1] - m[2 * q2 + 1]);
          l[2 * q2] += p0;
          l[2 * q2 + 1] += p1;
          ph[q2] = pack_f16x2(p0, p1);
          const float2 hf = unpack_f16x2(ph[q2]);
          pl[q2] = pack_f16x2(p0 - hf.x, p1 - hf.y);
        }
        // hi terms in columns [0, NQ), lo terms in [NQ, 2 NQ); [cg][tg][t%8][c%8]
        const uint32_t pr = prow + sb * C::PBUF;
#pragma unroll
        for (int cg = 0; cg < NQ / 8; ++cg) {
          sts128(pr + cg * 2048, make_uint4(ph[4 * cg], ph[4 * cg + 1], ph[4 * cg + 2], ph[4 * cg + 3]));
          sts128(pr + (NQ / 8 + cg) * 2048, make_uint4(pl[4 * cg], pl[4 * cg + 1], pl[4 * cg + 2], pl[4 * cg + 3]));
        }
      }
      if (rescale) {  // rare: some query's max grew by > 8 (log2): wait for PV(j-1), rescale O^T
        mbar_wait(&bars[Bn::ODONE + 2 * g + (sb ^ 1)], ((j - 1) >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int h = 0; h < NC / 16; ++h) {  // columns [16h, 16h + 16): query (16h + c) % NQ
          float ov[16];
          const uint32_t col = lane_addr + C::COL_O + g * NC + 16 * h;
          tmem_ld16(col, ov);
          uint32_t rr[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) rr[c] = __float_as_uint(ov[c] * alpha[(16 * h + c) % NQ]);
          tmem_st16(col, rr);
        }
        tmem_wait_st();
      }
      fence_proxy_async();
      tc_fence_before();
      __syncwarp();
      TC_TRACE(i, 7);
      if (lane == 0) mbar_arrive(&bars[Bn::PFULL + 2 * g + sb]);
      if (t.last) {
        // ---- the item's partial: O^T (lane = dim) / l, lse2 = m + log2 l
        // l: sum over the 128 token lanes -- warp transpose-reduce (each step
        // halves the values a lane keeps), then the 4 warps through shared memory
        float v[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) v[q] = l[q];
        int qi = 0;
#pragma unroll
        for (int step = 0, cnt = NQ, off = 16; step < 5; ++step, off >>= 1) {
          if (cnt > 1) {
            const int half = cnt / 2;
            const bool upper = (lane & off) != 0;
#pragma unroll
            for (int e = 0; e < NQ / 2; ++e) {
              if (e < half) {
                const float send = upper ? v[e] : v[e + half];
                const float keep = upper ? v[e + half] : v[e];
                v[e] = keep + __shfl_xor_sync(0xffffffffu, send, off);
              }
            }
            qi = qi * 2 + (upper ? 1 : 0);
            cnt = half;
          } else {
            v[0] += __shfl_xor_sync(0xffffffffu, v[0], off);
          }
        }
        named_bar(barid, 128);  // red free: every grow-path reader is past it
        if ((lane & (32 / NQ - 1)) == 0) red[wq * NQ + qi] = v[0];
        mbar_wait(&bars[Bn::ODONE + 2 * g + sb], (j >> 1) & 1);  // this item's last PV
        tc_fence_after();
        float ov[NC];
        tmem_ldn<NC>(lane_addr + C::COL_O + g * NC, ov);
        tc_fence_before();
        named_bar(barid, 128);
        const size_t obase = static_cast<size_t>(t.item) * p.qrows;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          if (q < t.rows) {
            const float L = red[q] + red[NQ + q] + red[2 * NQ + q] + red[3 * NQ + q];
            p.part_o[(obase + q) * kTcDP + tl] = (ov[q] + ov[NQ + q]) / L;
            if (tl == q) p.part_lse2[obase + q] = m[q] + __log2f(L);
          }
        }
        named_bar(barid, 128);  // red reads done before the next item's grow path
      }
      ++j;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kWarpMma) {
    tc_fence_after();
    tmem_dealloc(tbase, 512);
  }
#ifdef HX_TC_TRACE
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const unsigned long long t0 = g_tc_trace[0][0];
    for (int i = 0; i < 40; ++i)
      printf("tile %2d tma %6llu  k %6llu-%6llu S %6llu  v %6llu-%6llu  sm %6llu-%6llu\n", i, g_tc_trace[i][0] - t0,
             g_tc_trace[i][1] - t0, g_tc_trace[i][2] - t0, g_tc_trace[i][5] - t0, g_tc_trace[i][3] - t0,
             g_tc_trace[i][4] - t0, g_tc_trace[i][6] - t0, g_tc_trace[i][7] - t0);
    for (int i = 10; i < 24; ++i)
      printf("k %2d top %6llu rawfull %6llu | kfull %6llu sfree %6llu\n", i, g_tc_k[i][0] - t0, g_tc_k[i][1] - t0,
             g_tc_k[i][2] - t0, g_tc_k[i][3] - t0);
    for (int i = 0; i < 30; ++i)
      printf("v %2d top %6llu rawfull %6llu produced %6llu\n", i, g_tc_v[i][0] - t0, g_tc_v[i][1] - t0, g_tc_v[i][2] - t0);
  }
#endif
}

template <int NQ, int KVF, int NST>
static cudaError_t launch_tc_t(const AttnParams& p, int grid, cudaStream_t stream) {
  using C = TcCfg<NQ, KVF, NST>;
  const cudaError_t e = smem_optin<attn_tc_kernel<NQ, KVF, NST>>(C::SMEM);
  if (e != cudaSuccess) return e;
  return launch_k(attn_tc_kernel<NQ, KVF, NST>, dim3(grid), dim3(kTcThreads), C::SMEM, stream, p);
}

bool attn_tc_supported(const AttnParams& p) {
  return (p.kv8 || p.kv4) && p.dp == kTcDP && p.q_chunks == 1 && (p.qrows == 8 || p.qrows == 16) && !p.fused;
}

// grid: CTAs; two item slots each, items statically assigned (item = unit + n *
// 2 grid for unit = 2 CTA + slot)
cudaError_t launch_attn_tc(const AttnParams& p, int grid, cudaStream_t stream) {
  if (!attn_tc_supported(p)) return cudaErrorInvalidValue;
  if (p.kv4) return p.qrows == 16 ? launch_tc_t<16, 2, 9>(p, grid, stream) : launch_tc_t<8, 2, 11>(p, grid, stream);
  return p.qrows == 16 ? launch_tc_t<16, 1, 4>(p, grid, stream) : launch_tc_t<8, 1, 5>(p, grid, stream);
}

}  // namespace hx
