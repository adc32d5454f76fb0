// K1-TC: GQA flash-decode partial attention over FP8 (e4m3) KV pages on the
// 5th-generation tensor cores (tcgen05 + TMEM). Opt-in (HX_ATTN_TC=1): the
// engine then stores its FP8 pages in the tensor-core layout
// (kv_layout.cuh kv8tc_offset), which only this kernel reads.
//
// Same contract as attn_decode_kernel (attention.cu): per work item (stream =
// (rank slot, request, KV head), split = page range) the locally normalised
// partial output and log2-sum-exp of every query head of the GQA group --
// HeadFragment of partial_head_attention (reference attention.hpp:56-78,
// :375-396) -- so the split reduce / merge / exchange path is unchanged.
//
// Why: the legacy-HMMA kernel widens every e4m3 element into mma.sync operands
// on the consumer warps, and with 16 query rows (405B-like G = 16) that widen
// + MMA chain, not HBM, bounds it (66% of the copy bandwidth). Here
//
//   tile = 128 tokens (8 pages), transposed formulation (token = TMEM lane):
//   S^T [128 tok x NS] = K [128 tok x 128 dim] . Q8^T   kind::f8f6f4: K is the
//       A operand STRAIGHT FROM THE PAGES (e4m3, K-major core matrices), Q8 the
//       query split into T = 4 e4m3 terms, q ~ s0 * sum_j 16^-j * c_j (s0 a
//       power of two per query), so the only rounding is K's storage (~2^-16
//       relative in q; S = s0 * sum_j 16^-j S_j in the softmax)
//   O^T [128 dim x NC] += V^T [128 dim x 128 tok] . P^T  kind::f16: V widened to
//       f16 into TMEM by converter warps (one cvt per 2 elements), P split into
//       f16 hi + lo (22 bits); NC = 2 * NQ
//
// Roles (448 threads = 14 warps: <= 4 per SM sub-partition, 128 registers):
//   warps 0-3 / 4-7  softmax of item slot 0 / 1 (thread = token lane of S^T,
//                    = dim lane of O^T): lazy online softmax (rescale only when
//                    a query's max grows by > 8 in log2 units, found with one
//                    barrier.red.or), P^T hi/lo into shared memory, the rare O^T
//                    rescale in TMEM, the item's partial at its end
//   warps 8-11       V converters (thread = dim d: d's 8-token words of the
//                    page -> f16 pairs -> TMEM lane d) + the item's e4m3 query
//                    image
//   warp 12          producer: cp.async.bulk of each tile's 8 pages (+ the
//                    item's query rows) into a shared-memory ring
//   warp 13          MMA issue (one elected lane of the converged warp): S(i+1)
//                    before PV(i)
// Two item slots per CTA: their tiles alternate through the shared converters
// and tensor core, so one slot's softmax overlaps the other's MMAs. Work is
// statically assigned (item = unit + n * units, unit = 2 CTA + slot): every
// role walks the same deterministic tile sequence; only mbarrier phases pass
// between roles.
#include <cstdio>

#include "common.cuh"
#include "kernels.h"
#include "kv_layout.cuh"
#include "tc05.cuh"

namespace hx {

namespace {

constexpr int kTcDP = 128;  // head dim (padded) this kernel serves
constexpr int kTcThreads = 448;
constexpr int kWarpVConv = 8, kWarpProd = 12, kWarpMma = 13;
constexpr int kQTerms = 4;  // e4m3 terms of the query
// Lazy online softmax: the reference max of a query moves only when a logit
// exceeds it by more than this (log2 units); P <= 2^14 keeps its f16 hi term
// finite. A group-wide max update costs a barrier + shared-memory exchange and
// an O^T rescale in TMEM, so the threshold is set as high as f16 allows (the
// legacy kernel's per-warp update uses 8).
constexpr float kGrow = 14.f;

template <int NQ, int NST>
struct TcCfg {
  static constexpr int NC = 2 * NQ;                                   // PV MMA N: P hi/lo x query
  static constexpr int NS = kQTerms * NQ;                             // S MMA N: term x query
  // TMEM budget (512 columns): NQ = 16 keeps one S buffer per slot to afford 5 V
  // buffers (the converters run further ahead of the PV MMAs); NQ = 8 double-buffers S
  static constexpr int SB = NS == 64 ? 1 : 2;                         // S buffers per slot
  static constexpr int NV = NS == 64 ? 5 : 4;                         // V buffers in TMEM
  static constexpr uint32_t PAGE = 32u * kTcDP;                       // FP8 page, tensor-core layout
  static constexpr uint32_t STAGE = 8 * PAGE;                          // 8 pages = 128 tokens
  static constexpr uint32_t QRAW = NQ * kTcDP * 4;                    // fp32 query rows
  static constexpr uint32_t QIMG = NS * kTcDP;                        // Q8^T e4m3, K-major core matrices
  static constexpr uint32_t PBUF = 128 * NC * 2;                      // P^T f16, MN-major core matrices
  static constexpr uint32_t OFF_QIMG = NST * STAGE;
  static constexpr uint32_t OFF_PBUF = OFF_QIMG + 2 * QIMG;           // [slot][2]
  static constexpr uint32_t OFF_QRAW = OFF_PBUF + 4 * PBUF;           // [slot]
  static constexpr uint32_t OFF_QS0 = OFF_QRAW + 2 * QRAW;            // float [slot][NQ]: q term-0 scales
  static constexpr uint32_t OFF_RED = OFF_QS0 + 2 * NQ * 4;           // float [slot][4 warps][NQ]
  static constexpr uint32_t OFF_BAR = OFF_RED + 2 * 4 * NQ * 4;
  static constexpr int NBAR = 2 * NST + 2 * NV + 30;
  static constexpr uint32_t SMEM = OFF_BAR + NBAR * 8 + 16;
  // TMEM columns: V x NV | S [slot][2] | O [slot]
  static constexpr uint32_t COL_V = 0, COL_S = 64 * NV, COL_O = COL_S + 2 * SB * NS;
  static_assert(COL_O + 2 * NC <= 512, "TMEM columns");
  // S^T: kind::f8f6f4, e4m3 x e4m3 -> f32, both K-major
  static constexpr uint32_t IDESC_S = (1u << 4) | (static_cast<uint32_t>(NS >> 3) << 17) | (128u >> 4 << 24);
  // O^T: kind::f16, f16 x f16 -> f32, B (P^T) MN-major
  static constexpr uint32_t IDESC_O =
      (1u << 4) | (1u << 16) | (static_cast<uint32_t>(NC >> 3) << 17) | (128u >> 4 << 24);
};

// barrier indices
template <int NST, int NV>
struct TcBars {
  static constexpr int RAW_FULL = 0, RAW_EMPTY = NST;
  static constexpr int VFULL = 2 * NST, VFREE = VFULL + NV;
  static constexpr int SFULL = VFREE + NV, SFREE = SFULL + 4;  // [slot][buffer]
  static constexpr int PFULL = SFREE + 4, ODONE = PFULL + 4;   // [slot][P buffer]
  static constexpr int QFULL = ODONE + 4, QFREE = QFULL + 2, QRAWFREE = QFREE + 2;  // [slot]
};

struct TcTile {
  int slot, item, stream, np, ntok, rows, first, last;
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
  int kord, item, stream, tile, ntiles, pg0, pg1, ntok, rows;
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
      S.stream = stream;
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
    t.stream = S.stream;
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

HX_DEV uint32_t pack_f16x2(float lo, float hi) {
  uint32_t d;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}
HX_DEV float2 unpack_f16x2(uint32_t v) {
  const __half2 h = *reinterpret_cast<const __half2*>(&v);
  return __half22float2(h);
}


HX_DEV uint32_t e4m3x2_from_f32(float lo, float hi) {  // RNE, saturating (cvt.rn.satfinite)
  uint16_t r;
  asm("{\n.reg .b16 t;\ncvt.rn.satfinite.e4m3x2.f32 t, %1, %2;\nmov.b16 %0, t;\n}" : "=h"(r) : "f"(hi), "f"(lo));
  return r;
}
HX_DEV float2 f32x2_from_e4m3x2(uint32_t two) {
  uint32_t h;
  asm("{\n.reg .b16 t;\ncvt.u16.u32 t, %1;\ncvt.rn.f16x2.e4m3x2 %0, t;\n}" : "=r"(h) : "r"(two));
  return unpack_f16x2(h);
}
// smallest power of two >= x (x > 0, normal)
HX_DEV float pow2_ceil(float x) {
  const uint32_t b = __float_as_uint(x);
  return (b & 0x007FFFFFu) ? __uint_as_float((b & 0x7F800000u) + 0x00800000u) : x;
}
#ifdef HX_TC_TRACE
__device__ unsigned long long g_tc_trace[64][8];
__device__ unsigned long long g_tc_sm[64][4];
__device__ unsigned long long g_tc_mma[64][6];
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
#ifdef HX_TC_TRACE
#define TC_SM(i, ev) do { if (blockIdx.x == 0 && (i) < 64 && threadIdx.x == 0) g_tc_sm[i][ev] = gtime(); } while (0)
#else
#define TC_SM(i, ev) do {} while (0)
#endif
#ifdef HX_TC_TRACE
#define TC_M(i, ev) do { if (blockIdx.x == 0 && (i) < 64 && lane == 0) g_tc_mma[i][ev] = gtime(); } while (0)
#else
#define TC_M(i, ev) do {} while (0)
#endif
}  // namespace

template <int NQ, int NST>
__global__ void __launch_bounds__(kTcThreads, 1) attn_tc_kernel(const __grid_constant__ AttnParams p) {
  using C = TcCfg<NQ, NST>;
  constexpr int NV = C::NV, NS = C::NS, NC = C::NC;
  using Bn = TcBars<NST, NV>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + C::OFF_BAR + C::NBAR * 8);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&bars[Bn::RAW_FULL + s], 1);
      mbar_init(&bars[Bn::RAW_EMPTY + s], 5);  // 4 V converter warps + the S MMAs (they read K in place)
    }
    for (int v = 0; v < NV; ++v) {
      mbar_init(&bars[Bn::VFULL + v], 4);
      mbar_init(&bars[Bn::VFREE + v], 1);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&bars[Bn::SFULL + i], 1);
      mbar_init(&bars[Bn::SFREE + i], 4);
      mbar_init(&bars[Bn::PFULL + i], 4);
      mbar_init(&bars[Bn::ODONE + i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars[Bn::QFULL + i], 4);
      mbar_init(&bars[Bn::QFREE + i], 1);
      mbar_init(&bars[Bn::QRAWFREE + i], 4);
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

  if (warp == kWarpMma) {
    // ---------------------------------------------------------------- MMA issue: S(i+1) before PV(i)
    // The whole warp walks the sequence and waits (converged, so descriptors stay
    // warp-uniform); one elected lane issues each batch (tc05.cuh elect_one).
    const uint64_t qdesc0 = umma_desc(sbase + C::OFF_QIMG, (NS / 8) * 128, 128);
    const uint64_t pdesc0 = umma_desc(sbase + C::OFF_PBUF, 128, 16 * 128);
    // K of a 128-token tile, as landed: core matrices (8 tokens x 16 dims) 128 B
    // apart along the dims, 2 KB apart along the tokens (kv_layout.cuh kv8tc_offset)
    const uint64_t kdesc0 = umma_desc(sbase, 128, 2048);
    int jslot0 = 0, jslot1 = 0, nit0 = 0, nit1 = 0;
    // PV lags S by two tiles (S(i), then PV(i-2)): S runs ahead of the softmax
    // instead of queueing behind the previous tile's P, and the raw stages
    // holding K are released early
    int npend = 0;  // pending PVs (scalars, not arrays: no local memory)
    int ai = 0, ag = 0, aj = 0, af = 0, bi = 0, bg = 0, bj = 0, bf = 0;
    auto issue_pv = [&](int i, int g, int j, int first) {
      const int vb = i % NV, pb = j & 1;
      TC_M(i, 3);
      mbar_wait(&bars[Bn::VFULL + vb], (i / NV) & 1);
      TC_M(i, 4);
      mbar_wait(&bars[Bn::PFULL + 2 * g + pb], (j >> 1) & 1);
      TC_M(i, 5);
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
      const int s = i % NST, g = t.slot, j = g ? jslot1++ : jslot0++, sb = C::SB == 2 ? (j & 1) : 0;
      TC_M(i, 0);
      mbar_wait(&bars[Bn::RAW_FULL + s], (i / NST) & 1);
      TC_M(i, 1);
      if (t.first) {
        const int ni = g ? nit1++ : nit0++;
        mbar_wait(&bars[Bn::QFULL + g], ni & 1);  // this item's query image
      }
      if (j >= C::SB) mbar_wait(&bars[Bn::SFREE + 2 * g + sb], ((j / C::SB) - 1) & 1);
      TC_M(i, 2);
      tc_fence_after();
      const uint32_t dcol = tbase + C::COL_S + (C::SB * g + sb) * NS;
      const uint64_t kdesc = kdesc0 + static_cast<uint64_t>((s * C::STAGE) >> 4);
      const uint64_t qdesc = qdesc0 + static_cast<uint64_t>((g * C::QIMG) >> 4);
      const bool lst = t.last;
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < 4; ++k)  // K = 32 dims per MMA: two core matrices along the dims
          umma_ss_f8(dcol, kdesc + static_cast<uint64_t>((k * 256) >> 4),
                     qdesc + static_cast<uint64_t>((k * 2 * (NS / 8) * 128) >> 4), C::IDESC_S, k > 0 ? 1u : 0u);
        umma_commit(&bars[Bn::SFULL + 2 * g + sb]);
        umma_commit(&bars[Bn::RAW_EMPTY + s]);  // K read: the stage may refill once V is converted too
        if (lst) umma_commit(&bars[Bn::QFREE + g]);
      }
      __syncwarp();
      TC_TRACE(i, 5);
      if (npend == 2) {
        issue_pv(ai, ag, aj, af);
        ai = bi;
        ag = bg;
        aj = bj;
        af = bf;
        npend = 1;
      }
      if (npend == 0) {
        ai = i;
        ag = g;
        aj = j;
        af = t.first;
      } else {
        bi = i;
        bg = g;
        bj = j;
        bf = t.first;
      }
      ++npend;
    }
    if (npend >= 1) issue_pv(ai, ag, aj, af);
    if (npend == 2) issue_pv(bi, bg, bj, bf);
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
    // ---------------------------------------------------------------- V converters (thread = dim) + query image
    const int d = threadIdx.x - kWarpVConv * 32, vw = warp - kWarpVConv;
    const uint32_t lane_addr = tm_lane(tbase, warp);
    int nitem0 = 0, nitem1 = 0;
    for (int i = 0; seq.next(t); ++i) {
      const int s = i % NST, vb = i % NV, g = t.slot;
      mbar_wait(&bars[Bn::RAW_FULL + s], (i / NST) & 1);
      if (t.first) {
        // The item's query as T e4m3 terms: q * qscale = s0 * sum_j 16^-j c_j, s0 the
        // smallest power of two with max|q| <= 448 s0 (per query; every scaling exact).
        // Image: Q8^T K-major core matrices [dim/16][row/8][row%8][16 dims], row = j NQ + q.
        const int ni = g ? nitem1++ : nitem0++;
        if (ni > 0) mbar_wait(&bars[Bn::QFREE + g], (ni - 1) & 1);  // previous item's S MMAs done
        const float* qs = reinterpret_cast<const float*>(smem + C::OFF_QRAW + g * C::QRAW);
        uint8_t* qi = smem + C::OFF_QIMG + g * C::QIMG;
        float* qs0 = reinterpret_cast<float*>(smem + C::OFF_QS0) + g * NQ;
        for (int q = vw; q < NQ; q += 4) {
          float x[4];
          float am = 0.f;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            x[e] = q < t.rows ? qs[q * kTcDP + 4 * lane + e] * p.qscale : 0.f;
            am = fmaxf(am, fabsf(x[e]));
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, o));
          const float s0 = am > 0.f ? pow2_ceil(am / 448.f) : 1.f;
#pragma unroll
          for (int e = 0; e < 4; ++e) x[e] /= s0;  // exact
          float sc = 1.f;
#pragma unroll
          for (int jt = 0; jt < kQTerms; ++jt, sc *= 16.f) {
            const uint32_t c01 = e4m3x2_from_f32(x[0] * sc, x[1] * sc), c23 = e4m3x2_from_f32(x[2] * sc, x[3] * sc);
            const float2 d01 = f32x2_from_e4m3x2(c01), d23 = f32x2_from_e4m3x2(c23);
            x[0] -= d01.x / sc;
            x[1] -= d01.y / sc;
            x[2] -= d23.x / sc;
            x[3] -= d23.y / sc;
            const int row = jt * NQ + q;
            *reinterpret_cast<uint32_t*>(qi + ((lane >> 2) * (NS / 8) + (row >> 3)) * 128 + (row & 7) * 16 +
                                         4 * (lane & 3)) = c01 | (c23 << 16);
          }
          if (lane == 0) qs0[q] = s0;
        }
        fence_proxy_async();  // generic-proxy image writes -> the tensor core's async proxy
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&bars[Bn::QRAWFREE + g]);
          mbar_arrive(&bars[Bn::QFULL + g]);
        }
      }
      if (i >= NV) mbar_wait(&bars[Bn::VFREE + vb], ((i / NV) - 1) & 1);
      tc_fence_after();
      TC_TRACE(i, 3);
      const uint32_t vbase = sbase + s * C::STAGE + 1024 + d * 8;  // this dim's 8-token word, first half
#pragma unroll
      for (int half = 0; half < 2; ++half) {  // pages [4 half, 4 half + 4) -> columns [32 half, +32)
        uint2 w[4][2];
#pragma unroll
        for (int pq = 0; pq < 4; ++pq) {
          const uint32_t pb = vbase + (4 * half + pq) * C::PAGE;
          w[pq][0] = lds64(pb);         // tokens 0..7
          w[pq][1] = lds64(pb + 2048);  // tokens 8..15
        }
        uint32_t r[32];
#pragma unroll
        for (int pq = 0; pq < 4; ++pq) {
          const bool have = 4 * half + pq < t.np;  // pages past np: stale bytes (maybe nan) -> zeros
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            e4m3x4_to_f16x2x2(have ? w[pq][hh].x : 0u, r[8 * pq + 4 * hh], r[8 * pq + 4 * hh + 1]);
            e4m3x4_to_f16x2x2(have ? w[pq][hh].y : 0u, r[8 * pq + 4 * hh + 2], r[8 * pq + 4 * hh + 3]);
          }
        }
        tmem_st32u(lane_addr + C::COL_V + vb * 64 + 32 * half, r);
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      TC_TRACE(i, 4);
      if (lane == 0) {
        mbar_arrive(&bars[Bn::VFULL + vb]);
        mbar_arrive(&bars[Bn::RAW_EMPTY + s]);
      }
    }
  } else {
    // ---------------------------------------------------------------- softmax (slot g)
    const int g = warp >> 2, wq = warp & 3;
    const int tl = threadIdx.x - g * 128;  // token lane of S^T, dim lane of O^T
    const uint32_t lane_addr = tm_lane(tbase, warp);
    const int barid = 1 + g;
    float* red = reinterpret_cast<float*>(smem + C::OFF_RED) + g * 4 * NQ;
    const float* qs0 = reinterpret_cast<const float*>(smem + C::OFF_QS0) + g * NQ;
    const uint32_t prow = sbase + C::OFF_PBUF + (2 * g) * C::PBUF + (tl >> 3) * 128 + (tl & 7) * 16;
    float m[NQ], l[NQ];
    int j = 0;
    for (int i = 0; seq.next(t); ++i) {
      if (t.slot != g) continue;
      const int sb = j & 1;                               // P^T buffer
      const int ss = C::SB == 2 ? sb : 0;                 // S buffer
      mbar_wait(&bars[Bn::SFULL + 2 * g + ss], (j / C::SB) & 1);
      tc_fence_after();
      TC_TRACE(i, 6);
      // S = s0 * (S_0 + S_1 / 16 + S_2 / 256 + S_3 / 4096), columns jt * NQ + q
      float part[NQ];
      {
        const uint32_t scol = lane_addr + C::COL_S + (C::SB * g + ss) * NS;
        float sv[32];
        tmem_ld32(scol, sv);  // NQ = 8: all four terms; NQ = 16: terms 0, 1
        if constexpr (NQ == 8) {
#pragma unroll
          for (int q = 0; q < 8; ++q)
            part[q] = ((sv[24 + q] * (1.f / 16.f) + sv[16 + q]) * (1.f / 16.f) + sv[8 + q]) * (1.f / 16.f) + sv[q];
        } else {
#pragma unroll
          for (int q = 0; q < 16; ++q) part[q] = sv[16 + q] * (1.f / 16.f) + sv[q];
          tmem_ld32(scol + 32, sv);  // terms 2, 3
#pragma unroll
          for (int q = 0; q < 16; ++q)
            part[q] += (sv[16 + q] * (1.f / 16.f) + sv[q]) * (1.f / 256.f);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[Bn::SFREE + 2 * g + ss]);
      TC_SM(i, 0);
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
        s[q] = valid ? qs0[q] * part[q] : -INFINITY;
        grow |= s[q] > m[q] + kGrow;
      }
      bool rescale = false;
      float alpha[NQ];
      const bool any_grow = bar_red_or(barid, 128, grow);
      TC_SM(i, 1);
      if (any_grow) {
        // tile maxima per query over the 128 token lanes
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const float mx = redux_max_f32(s[q]);
          if (lane == 0) red[wq * NQ + q] = mx;
        }
        named_bar(barid, 128);
        float tmx[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) tmx[q] = -INFINITY;
#pragma unroll
        for (int w4 = 0; w4 < 4; ++w4)
#pragma unroll
          for (int q4 = 0; q4 < NQ / 4; ++q4) {
            const float4 v4 = *reinterpret_cast<const float4*>(red + w4 * NQ + 4 * q4);
            tmx[4 * q4] = fmaxf(tmx[4 * q4], v4.x);
            tmx[4 * q4 + 1] = fmaxf(tmx[4 * q4 + 1], v4.y);
            tmx[4 * q4 + 2] = fmaxf(tmx[4 * q4 + 2], v4.z);
            tmx[4 * q4 + 3] = fmaxf(tmx[4 * q4 + 3], v4.w);
          }
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const float tm = tmx[q];
          const float mn = tm > m[q] + kGrow ? tm : m[q];
          alpha[q] = fast_exp2(m[q] - mn);  // 0 when m = -inf
          rescale |= mn != m[q];
          l[q] *= alpha[q];
          m[q] = mn;
        }
        rescale = rescale && !t.first;  // a new item's first PV overwrites O^T
      }
      // P^T buffer sb of this slot: PV(j-2) done
      if (j >= 2) mbar_wait(&bars[Bn::ODONE + 2 * g + sb], ((j >> 1) - 1) & 1);
      TC_SM(i, 2);
      if (rescale) {  // rare: some query's max grew by > kGrow (log2): wait for PV(j-1), rescale O^T
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
        named_bar(barid, 128);  // red reads and the partial's stores done
        // HOP-B stream reducer (fused == 2): publish the finished split (cumulative
        // gpu-scope release of the whole group's stores, ordered by the barrier)
        if (p.fused == 2 && tl == 0)
          asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(p.stream_done + t.stream) : "memory");
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
      printf("tile %2d tma %6llu  v %6llu-%6llu  S %6llu  sm %6llu ld %6llu vote %6llu odone %6llu end %6llu\n", i,
             g_tc_trace[i][0] - t0, g_tc_trace[i][3] - t0, g_tc_trace[i][4] - t0, g_tc_trace[i][5] - t0,
             g_tc_trace[i][6] - t0, g_tc_sm[i][0] - t0, g_tc_sm[i][1] - t0, g_tc_sm[i][2] - t0, g_tc_trace[i][7] - t0);
    for (int i = 14; i < 26; ++i)
      printf("mma %2d top %6llu rawfull %6llu sfree %6llu | pv top %6llu vfull %6llu pfull %6llu\n", i,
             g_tc_mma[i][0] - t0, g_tc_mma[i][1] - t0, g_tc_mma[i][2] - t0, g_tc_mma[i][3] - t0, g_tc_mma[i][4] - t0,
             g_tc_mma[i][5] - t0);
  }
#endif
}

template <int NQ, int NST>
static cudaError_t launch_tc_t(const AttnParams& p, int grid, cudaStream_t stream) {
  using C = TcCfg<NQ, NST>;
  const cudaError_t e = smem_optin<attn_tc_kernel<NQ, NST>>(C::SMEM);
  if (e != cudaSuccess) return e;
  return launch_k(attn_tc_kernel<NQ, NST>, dim3(grid), dim3(kTcThreads), C::SMEM, stream, p);
}

bool attn_tc_supported(const AttnParams& p) {
  return p.kv8 && !p.kv4 && p.dp == kTcDP && p.q_chunks == 1 && (p.qrows == 8 || p.qrows == 16) &&
         (p.fused == 0 || p.fused == 2);
}

// grid: CTAs; two item slots each, items statically assigned (item = unit + n *
// 2 grid for unit = 2 CTA + slot)
cudaError_t launch_attn_tc(const AttnParams& p, int grid, cudaStream_t stream) {
  if (!attn_tc_supported(p)) return cudaErrorInvalidValue;
  return p.qrows == 16 ? launch_tc_t<16, 5>(p, grid, stream) : launch_tc_t<8, 6>(p, grid, stream);
}

}  // namespace hx
