// K1: KV-parallel GQA flash-decode partial attention for sm_100a.
//
// Replaces the per-(rank, kv head, query head) Eigen GEMVs of
// shard_attention / partial_head_attention (reference attention.hpp:65-78,
// :375-396): one pass over a rank's KV shard serves every query head of the
// GQA group, emitting a locally normalised partial output plus its
// log-sum-exp per query head -- exactly the (partial_out, lse) pair of
// HeadFragment (:56-59), computed per contiguous page range ("split").
//
// Structure (persistent, one CTA per SM, warp specialised):
//   * producer warp: grabs work items (stream, split) from a global counter,
//     streams the split's contiguous 16-token pages into a shared-memory ring
//     with cp.async.bulk (TMA bulk engine), completion via mbarrier tx-bytes;
//     the item's query rows ride along in the first stage.
//   * NWC consumer warps: one page each per stage (QC = 2 query chunks of
//     8 rows per item when the GQA group exceeds 8: warp w takes chunk w % QC
//     and pages w / QC + k * NWC / QC, so each KV page is read from HBM once
//     and from shared memory QC times); S = Q K^T and O += P V on
//     legacy HMMA m16n8k16 (bf16 in, fp32 accumulate). The fp32 query is
//     split hi+mid+lo into three bf16 terms (rows 0-7 / 8-15 of M-tile 0 and
//     rows 0-7 of M-tile 1) and P into hi+lo (rows 0-7 / 8-15), so the only
//     rounding is the bf16 KV storage itself.
//   * per item, consumers combine their per-warp (m, l, O) through shared
//     memory and write the split's normalised O and log2-sum-exp.
// The KV stream is the roofline: 64*DP bytes per page, no re-reads.

#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kv_layout.cuh"
#include "xfrag.cuh"
#include "merge.cuh"
#include "kernels.h"

namespace hx {

namespace {

constexpr int kItemDone = -1;

struct StageMeta {
  int item;         // work item id, or kItemDone
  int stream;       // stream index
  int page0;        // first page (within the stream) of this stage
  int npages;       // pages in this stage (<= NWC)
  int ntok;         // tokens on this rank for the stream
  int first;        // first stage of the item (q rows staged)
  int last;         // last stage of the item
  int rows;         // valid query rows in this stream (<= 8 * QC)
};

template <int DP, int KVF>
struct AttnCfg {
  static constexpr int KS = DP / 16;     // k-steps over the head dim
  static constexpr int ND = DP / 8;      // PV n-tiles
  // kv_layout.cuh: bf16 64*DP, fp8 32*DP, fp4 17.5*DP bytes per page
  static constexpr uint32_t PAGE = KVF == 2 ? 35u * DP / 2u : (KVF == 1 ? 32u : 64u) * DP;
};

// KVF = 1: FP8 e4m3 pages; each lane's 8-byte chunk widens to the f16 register
// image of the bf16 path's 16-byte chunk. KVF = 2: FP4 e2m1 pages; each lane's
// 4-byte chunk widens (cvt e2m1x2 -> f16x2) and is scaled by its block's 2^e in
// f16 (exact, fp8.cuh). Either way the MMAs run in f16 (q and P split into f16
// terms); the only rounding is the storage itself.
__device__ __forceinline__ void e2m1x8_to_f16x2x4(uint32_t w, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm("{\n .reg .b8 b0, b1, b2, b3;\n mov.b32 {b0, b1, b2, b3}, %4;\n"
      " cvt.rn.f16x2.e2m1x2 %0, b0;\n cvt.rn.f16x2.e2m1x2 %1, b1;\n"
      " cvt.rn.f16x2.e2m1x2 %2, b2;\n cvt.rn.f16x2.e2m1x2 %3, b3;\n}"
      : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
      : "r"(w));
}
// f16 bits of 2^e from the stored exponent byte e + 15 (e in [-14, 13]: normal)
__device__ __forceinline__ uint32_t f16_pow2(uint32_t ebyte) { return ebyte << 10; }
__device__ __forceinline__ uint32_t lds16(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint32_t hmul2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t lds8(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

// Lane chunk ci of the page's K region (tokens 8 nt + g, 32-dim group kp):
// the register image of the bf16 chunk (kv_layout.cuh).
template <int DP, int KVF>
__device__ __forceinline__ uint4 load_k(uint32_t pbase, int ci) {
  if constexpr (KVF == 0) {
    return lds128(pbase + ci * 16);
  } else if constexpr (KVF == 1) {
    const uint2 b = lds64(pbase + ci * 8);
    uint4 r;
    e4m3x4_to_f16x2x2(b.x, r.x, r.y);
    e4m3x4_to_f16x2x2(b.y, r.z, r.w);
    return r;
  } else {
    uint4 r;
    e2m1x8_to_f16x2x4(lds32(pbase + ci * 4), r.x, r.y, r.z, r.w);
    const int grp = ci >> 5, kp = grp % (DP / 32), nt = grp / (DP / 32);
    const int t = nt * 8 + ((ci & 31) >> 2);
    const uint32_t s = f16_pow2(lds8(pbase + 16 * DP + t * (DP / 32) + kp));
    const uint32_t ss = s | (s << 16);
    r.x = hmul2(r.x, ss);
    r.y = hmul2(r.y, ss);
    r.z = hmul2(r.z, ss);
    r.w = hmul2(r.w, ss);
    return r;
  }
}
// Lane chunk ci of the page's V region (dims 16 nd2 + g, 16 nd2 + 8 + g; tokens
// 2c, 2c+1 in .x/.z and 2c+8, 2c+9 in .y/.w).
template <int DP, int KVF>
__device__ __forceinline__ uint4 load_v(uint32_t pbase, int ci) {
  if constexpr (KVF == 0) {
    return lds128(pbase + 32 * DP + ci * 16);
  } else if constexpr (KVF == 1) {
    const uint2 b = lds64(pbase + 16 * DP + ci * 8);
    uint4 r;
    e4m3x4_to_f16x2x2(b.x, r.x, r.y);
    e4m3x4_to_f16x2x2(b.y, r.z, r.w);
    return r;
  } else {
    uint4 r;
    e2m1x8_to_f16x2x4(lds32(pbase + 8 * DP + ci * 4), r.x, r.y, r.z, r.w);
    const int c = ci & 3, grp = (ci >> 5) >> 1;
    const uint32_t sb = pbase + 16 * DP + DP / 2 + grp * 32;  // V scales, f16 [DP/32][16 tokens]
    const uint32_t lo = lds32(sb + 4 * c), hi = lds32(sb + 4 * c + 16);  // tokens (2c, 2c+1), (2c+8, 2c+9)
    r.x = hmul2(r.x, lo);
    r.y = hmul2(r.y, hi);
    r.z = hmul2(r.z, lo);
    r.w = hmul2(r.w, hi);
    return r;
  }
}
template <bool KV8>
__device__ __forceinline__ void mma_kv(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                       uint32_t b0, uint32_t b1) {
  if constexpr (KV8)
    mma_f16_16816(d, a0, a1, a2, a3, b0, b1);
  else
    mma_bf16_16816(d, a0, a1, a2, a3, b0, b1);
}
template <bool KV8>
__device__ __forceinline__ uint32_t pack_kv(float lo, float hi) {
  if constexpr (KV8)
    return pack_f16(lo, hi);
  else
    return pack_bf16(lo, hi);
}

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Work item of (stream, split): split-major (every stream advances together --
// the faster order for one batched launch), or in groups of stream_major
// consecutive streams, split-major inside a group and the groups in order
// (1 = stream-major): streams, hence requests, complete group by group (HOP-B).
__device__ __forceinline__ size_t attn_item(const AttnParams& p, int stream, int split) {
  if (!p.stream_major) return static_cast<size_t>(split) * p.n_streams + stream;
  const int G = p.stream_major, g0 = (stream / G) * G;
  const int gs = min(G, p.n_streams - g0);  // streams in this (possibly short, last) group
  return static_cast<size_t>(g0) * p.splits + static_cast<size_t>(split) * gs + (stream - g0);
}
__device__ __forceinline__ void attn_item_decode(const AttnParams& p, int item, int& stream, int& split) {
  if (!p.stream_major) {
    split = item / p.n_streams;
    stream = item - split * p.n_streams;
    return;
  }
  const int G = p.stream_major, per_group = G * p.splits;
  const int g0 = (item / per_group) * G;
  const int gs = min(G, p.n_streams - g0);
  const int r = item - g0 * p.splits;
  split = r / gs;
  stream = g0 + (r - split * gs);
}

}  // namespace

// ------------------------------------------------------------------------
// Fused split reduce + device-initiated exchange (AttnParams::fused / push)

// Stream `stream`'s split partials -> the rank's fragment rows (HeadFragment,
// attention.hpp:56-59), splits merged in order. Warp `warp` of `nwarps` takes
// rows warp, warp + nwarps, ...; lanes hold dims lane + 32 i, and each batch of
// 16 splits issues all its loads before using any (the partials are L2-resident:
// other CTAs wrote them in this launch, so ld.cg). nwarps = 0: a single thread
// (the producer, for an empty stream: the identity fragment).
// Device-initiated exchange (AttnParams::push): element d of query head qg of
// this rank's group output for request b goes to peer e / slice at offset
// e % slice of its [this rank][b] chunk, e = qg * hd + d; the head's lse rides
// in the lse slots of every slice that touches the head (attention.hpp:495-502).
__device__ __forceinline__ void push_value(const AttnParams& p, int b, int qg, int d, float o) {
  const int e = qg * p.hd + d;
  const int dst = e / p.xslice;
  p.peer_recv[dst][(static_cast<size_t>(p.xrank) * p.batch + b) * p.xchunk + (e - dst * p.xslice)] = o;
}
__device__ __forceinline__ void push_lse(const AttnParams& p, int b, int qg, float lse) {
  const size_t row = (static_cast<size_t>(p.xrank) * p.batch + b) * p.xchunk;
  const int p0 = (qg * p.hd) / p.xslice, p1 = ((qg + 1) * p.hd - 1) / p.xslice;
  for (int pd = p0; pd <= p1; ++pd) p.peer_recv[pd][row + p.xslice + (qg - (pd * p.xslice) / p.hd)] = lse;
}
// One more unit (stream / reduce CTA) is out; the `total`-th raises this
// rank's flag in every peer (system-scope release after a system fence).
__device__ __forceinline__ void signal_pushed(const AttnParams& p, int total) {
  __threadfence_system();  // this unit's peer stores before the count
  const int cnt = atomicAdd(p.pushed, 1);
#ifdef HX_DEBUG_PUSH
  printf("push rank %d unit %d/%d\n", p.xrank, cnt, total);
#endif
  if (cnt == total - 1) {
    __threadfence_system();
    for (int r = 0; r < p.kvp; ++r) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p.peer_flag[r]), "r"(1u)
                                                 : "memory");
    *p.pushed = 0;
  }
}

constexpr int kRedBatch = 16;  // splits whose loads are in flight together
template <int DP>
__device__ void reduce_stream(const AttnParams& p, int stream, int rows, int warp, int nwarps, int q_begin = 0,
                              int q_end = 1 << 30) {
  constexpr int PER = DP / 32;
  int t = stream;
  const int qc = t % p.q_chunks;
  t /= p.q_chunks;
  const int kvh = t % p.kvh_per_slot;
  t /= p.kvh_per_slot;
  const int b = t % p.stream_batch + p.b_begin;
  const int sl = t / p.stream_batch;
  const int slot = sl + p.slot_base;
  const int rank = slot % p.kvp;
  const int QR = p.qrows;
  const int pages = (static_cast<int>(rr_count(p.total[b], rank, p.chunk, p.kvp)) + 15) >> 4;
  const int q0 = kvh * p.group + qc * QR;  // first query row of the stream within the slot's group
  const size_t fbase = (static_cast<size_t>(sl) * p.batch + b) * p.q_per_slot + q0;
  const bool single = nwarps == 0;
  const int lane = single ? 0 : (threadIdx.x & 31);
  const bool all_full = pages >= p.splits;  // every split holds >= 1 page (the usual case)
  auto nonempty = [&](int s) {
    return all_full ||
           (static_cast<long long>(s + 1) * pages) / p.splits > (static_cast<long long>(s) * pages) / p.splits;
  };
  if (q_end > rows) q_end = rows;
  for (int q = q_begin + (single ? 0 : warp); q < q_end; q += single ? 1 : nwarps) {
    float M = -INFINITY;
    if (!single) {
      for (int s = lane; s < p.splits; s += 32)
        if (nonempty(s)) M = fmaxf(M, __ldcg(p.part_lse2 + attn_item(p, stream, s) * QR + q));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    }
    float L = 0.f, acc[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) acc[i] = 0.f;
    if (M != -INFINITY) {
      for (int s0 = 0; s0 < p.splits; s0 += kRedBatch) {
        float e[kRedBatch], v[kRedBatch][PER];
#pragma unroll
        for (int j = 0; j < kRedBatch; ++j) {
          const int s = s0 + j;
          const bool ok = s < p.splits && nonempty(s);
          const size_t it = attn_item(p, stream, ok ? s : 0);
          e[j] = ok ? __ldcg(p.part_lse2 + it * QR + q) : -INFINITY;
          const float* po = p.part_o + (it * QR + q) * DP + lane;
#pragma unroll
          for (int i = 0; i < PER; ++i) v[j][i] = ok ? __ldcg(po + 32 * i) : 0.f;
        }
#pragma unroll
        for (int j = 0; j < kRedBatch; ++j) {
          const float w = e[j] == -INFINITY ? 0.f : fast_exp2(e[j] - M);
          L += w;
#pragma unroll
          for (int i = 0; i < PER; ++i) acc[i] += v[j][i] * w;
        }
      }
    }
    const float lse = L > 0.f ? (M + __log2f(L)) * 0.69314718055994530942f : -INFINITY;
    const int qg = q0 + q;  // query head within the slot's group
    for (int i = 0; i < (single ? DP : PER); ++i) {
      const int d = single ? i : lane + 32 * i;
      const float o = single ? 0.f : (L > 0.f ? acc[i] / L : 0.f);  // single: empty stream
      p.frag_o[(fbase + q) * DP + d] = o;
      if (d >= p.hd) continue;
      if (p.xf_out)  // one-source pool: this fragment IS the merged output
        xf_write(p.xf_out, xf_nb8(p.batch), b, (slot / p.kvp) * p.q_per_slot * p.hd + qg * p.hd + d, o, p.xf16);
      if (p.push) push_value(p, b, qg, d, o);
    }
    if (lane == 0) {
      p.frag_lse[fbase + q] = lse;
      if (p.push) push_lse(p, b, qg, lse);
    }
  }
}

// Consumer warps after an item's partial is stored: count the stream's
// completed splits; the CTA completing the last one reduces (and pushes) it
// (fused == 1), or -- fused == 2 -- only the count is published and the
// co-resident stream reducer (attn_stream_reduce_kernel) does the rest.
template <int DP, int NWC>
__device__ __forceinline__ void fused_stream_done(const AttnParams& p, int stream, int rows, int ntok) {
  __shared__ int s_last;
  if (p.fused == 3) return;  // timing experiment only (no count; the reducer does not wait)
  if (p.fused == 2) {
    // the item's partial (every consumer thread's stores, ordered before this by
    // the named barrier) released with the count: a cumulative gpu-scope release
    // instead of a full fence + atomic
    if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(p.stream_done + stream) : "memory");
    return;
  }
  if (threadIdx.x == 0) {
    __threadfence();  // the item's partial (all consumer threads, ordered by the barrier) before the count
    const int pages = (ntok + 15) >> 4;
    const int need = pages < p.splits ? pages : p.splits;  // non-empty splits of the stream
    s_last = atomicAdd(p.stream_done + stream, 1) == need - 1;
    if (s_last) __threadfence();
  }
  named_bar_sync(1, NWC * 32);
  if (!s_last) return;
  reduce_stream<DP>(p, stream, rows, threadIdx.x >> 5, NWC);
  named_bar_sync(1, NWC * 32);
  if (threadIdx.x == 0) {
    p.stream_done[stream] = 0;  // for the next launch / graph replay
    if (p.push) signal_pushed(p, p.n_streams);
  }
}

// W16 (bf16 pages, 9-16 query heads per KV head): every consumer warp takes
// one page per stage for ALL 16 query rows. The three bf16 terms of the query
// (hi/mid/lo) are three 16-row M-tiles accumulated into ONE S fragment (rows =
// queries), and P's hi/lo tiles into one O fragment, so a page costs
// 3·2·KS + 2·ND MMAs (80 at Hsz 128) instead of two 8-row passes (96); the
// per-item query fragment image (3 terms x KS k-steps x 32 lanes x 16 B) lives
// in shared memory, keeping registers at the 8-row path's level.
template <int DP, int NWC, int NSTAGE, int QC, int KVF, bool W16>
__global__ void __launch_bounds__((NWC + 1) * 32, 1) attn_decode_kernel(const AttnParams p) {
  using Cfg = AttnCfg<DP, KVF>;
  constexpr bool KV8 = KVF != 0;  // f16 MMAs on the widened FP8 / FP4 operands
  static_assert(NWC % QC == 0, "query chunks must divide the consumer warps");
  static_assert(!W16 || QC == 2, "W16: 16 query rows per warp");
  constexpr int QR = 8 * QC;           // query rows per item
  constexpr int WPC = NWC / QC;        // warps (pages per stage slot) per query chunk
  constexpr int SR = W16 ? 16 : 8;     // query rows per warp
  constexpr uint32_t STAGE_KV = NWC * Cfg::PAGE;
  constexpr uint32_t Q_BYTES = QR * DP * 4;
  constexpr uint32_t STAGE_BYTES = STAGE_KV + Q_BYTES;
  constexpr int WS = SR * DP + 2 * SR; // per-warp combine scratch (floats): O rows, m, l
  // FP4 pages, 8 query rows: the query fragments live in shared memory (one image per
  // query chunk) instead of 32 registers per thread, so more consumer warps fit
  constexpr bool QSM = KVF == 2 && !W16;
  constexpr uint32_t QIMG_BYTES = W16 ? 3u * Cfg::KS * 32u * 16u : (QSM ? QC * Cfg::KS * 32u * 16u : 0u);

  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* stages = smem;                                                     // NSTAGE * STAGE_BYTES
  float* scratch = reinterpret_cast<float*>(smem + NSTAGE * STAGE_BYTES);     // NWC * WS
  uint4* qimg = reinterpret_cast<uint4*>(scratch + NWC * WS);                 // W16: [3][KS][32]
  StageMeta* meta = reinterpret_cast<StageMeta*>(reinterpret_cast<uint8_t*>(qimg) + QIMG_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(meta + NSTAGE);
  uint64_t* empty = full + NSTAGE;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NWC);
    }
    fence_mbar_init();
  }
  __syncthreads();
  griddep_launch_dependents();

  if (warp == NWC) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      int st = 0;
      bool waited = false;  // q rows come from the QKV kernel: wait before staging them
      for (;;) {
        const int item = atomicAdd(p.work_counter, 1);
        const bool done = item >= p.n_items;
        int stream = 0, pg0 = 0, pg1 = 0, ntok = 0, rows = 0;
        const uint8_t* kv_base = nullptr;
        const float* q_src = nullptr;
        if (!done) {
          // decode the item once: (stream, split) (attn_item), then
          // stream -> (slot, request, kv head, query chunk)
          int split;
          attn_item_decode(p, item, stream, split);
          int t = stream;
          const int qc = t % p.q_chunks;
          t /= p.q_chunks;
          const int kvh = t % p.kvh_per_slot;
          t /= p.kvh_per_slot;
          const int bl = t % p.stream_batch;
          const int sl = t / p.stream_batch;
          const int b = bl + p.b_begin;
          const int slot = sl + p.slot_base;
          const int rank = slot % p.kvp;
          ntok = static_cast<int>(rr_count(p.total[b], rank, p.chunk, p.kvp));
          const int pages = (ntok + 15) >> 4;
          pg0 = static_cast<int>((static_cast<long long>(split) * pages) / p.splits);
          pg1 = static_cast<int>((static_cast<long long>(split + 1) * pages) / p.splits);
          const int g_rows = p.group - qc * QR;
          rows = g_rows < QR ? g_rows : QR;
          if (pg1 <= pg0) {  // empty split: nothing to emit
            if (p.fused == 1 && pages == 0 && split == 0) {
              // no tokens on this rank for the stream: its fragment is the identity (0, -inf)
              // (attention.hpp:69-70); the producer thread writes / pushes it
              if (!waited) {
                griddep_wait();
                waited = true;
              }
              reduce_stream<DP>(p, stream, rows, 0, 0);
              if (p.push) signal_pushed(p, p.n_streams);
            }
            continue;
          }
          const size_t pool_stream = (static_cast<size_t>(sl) * p.batch + b) * p.kvh_per_slot + kvh;
          kv_base = p.kv + pool_stream * p.page_cap * static_cast<size_t>(Cfg::PAGE);
          const int grp = slot / p.kvp;
          const int head0 = ((grp - p.q_grp_base) * p.kvh_per_slot + kvh) * p.group + qc * QR;
          q_src = p.q + (static_cast<size_t>(b) * p.q_heads + head0) * DP;
        }
        const int nchunks = done ? 1 : (pg1 - pg0 + NWC - 1) / NWC;
        for (int ch = 0; ch < nchunks; ++ch, ++st) {
          const int s = st % NSTAGE;
          if (st >= NSTAGE) mbar_wait(&empty[s], ((st / NSTAGE) & 1) ^ 1);
          StageMeta& m = meta[s];
          if (done) {
            if (!waited) {
              griddep_wait();
              waited = true;
            }
            m.item = kItemDone;
            mbar_arrive(&full[s]);
            break;
          }
          const int a = pg0 + ch * NWC;
          const int np = min(NWC, pg1 - a);
          m.item = item;
          m.stream = stream;
          m.page0 = a;
          m.npages = np;
          m.ntok = ntok;
          m.first = ch == 0;
          m.last = ch == nchunks - 1;
          m.rows = rows;
          uint8_t* dst = stages + s * STAGE_BYTES;
          const uint32_t bytes = np * Cfg::PAGE;
          const uint32_t qbytes = ch == 0 ? static_cast<uint32_t>(rows) * DP * 4 : 0u;
          mbar_arrive_expect_tx(&full[s], bytes + qbytes);
          bulk_g2s(dst, kv_base + static_cast<size_t>(a) * Cfg::PAGE, bytes, &full[s]);  // KV: no dependency
          if (!waited) {
            griddep_wait();
            waited = true;
          }
          if (qbytes) bulk_g2s(dst + STAGE_KV, q_src, qbytes, &full[s]);
        }
        if (done) break;
      }
    }
  } else if constexpr (W16) {
    // ------------------------------------------------------------ consumers, 16 query rows per warp
    constexpr int kQTerms = KV8 ? 2 : 3;
    const int g = lane >> 2, c = lane & 3;
    float acc[Cfg::ND][4];           // rows g (query g) and g+8 (query g+8)
    float m_ref[2] = {-INFINITY, -INFINITY}, l_sum[2] = {0.f, 0.f};
    const uint32_t stage_base = smem_u32(stages);
    const uint32_t qimg_base = smem_u32(qimg);
    for (int st = 0;; ++st) {
      const int s = st % NSTAGE;
      mbar_wait(&full[s], (st / NSTAGE) & 1);
      const StageMeta m = meta[s];
      if (m.item == kItemDone) break;
      const uint32_t sbase = stage_base + s * STAGE_BYTES;
      if (m.first) {
        // query fragment image: warp w builds k-steps w, w + NWC, ... of every term
        // (bf16 pages: hi/mid/lo bf16; FP8 pages: hi/lo f16, 22 significant bits)
        const float* qs = reinterpret_cast<const float*>(stages + s * STAGE_BYTES + STAGE_KV);
        for (int ks = warp; ks < Cfg::KS; ks += NWC) {
          float t[3][2][4];  // [term][row g / g+8][d0, d0+1, d0+8, d0+9]
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            const int row = g + 8 * r;
            const bool valid = row < m.rows;
            const int d0 = ks * 16 + 2 * c;
            const int dd[4] = {d0, d0 + 1, d0 + 8, d0 + 9};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float v = valid ? qs[row * DP + dd[i]] * p.qscale : 0.f;
              if constexpr (KV8) {
                split2h(v, t[0][r][i], t[1][r][i]);
                t[2][r][i] = 0.f;
              } else {
                split3(v, t[0][r][i], t[1][r][i], t[2][r][i]);
              }
            }
          }
#pragma unroll
          for (int term = 0; term < kQTerms; ++term)
            qimg[(term * Cfg::KS + ks) * 32 + lane] =
                make_uint4(pack_kv<KV8>(t[term][0][0], t[term][0][1]), pack_kv<KV8>(t[term][1][0], t[term][1][1]),
                           pack_kv<KV8>(t[term][0][2], t[term][0][3]), pack_kv<KV8>(t[term][1][2], t[term][1][3]));
        }
        named_bar_sync(1, NWC * 32);  // image complete before any warp's first page
#pragma unroll
        for (int nd = 0; nd < Cfg::ND; ++nd) acc[nd][0] = acc[nd][1] = acc[nd][2] = acc[nd][3] = 0.f;
        m_ref[0] = m_ref[1] = -INFINITY;
        l_sum[0] = l_sum[1] = 0.f;
      }
      if (warp < m.npages) {
        const uint32_t pbase = sbase + warp * Cfg::PAGE;
        const int tok0 = (m.page0 + warp) * 16;
        const int valid_tok = m.ntok - tok0;  // >= 1
        // ---- S = Q K^T: three query terms accumulate into one fragment
        float sacc[2][4];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) sacc[nt][0] = sacc[nt][1] = sacc[nt][2] = sacc[nt][3] = 0.f;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
          for (int kp = 0; kp < Cfg::KS / 2; ++kp) {
            const int ci = (nt * (Cfg::KS / 2) + kp) * 32 + lane;
            const uint4 kf = load_k<DP, KVF>(pbase, ci);
#pragma unroll
            for (int term = 0; term < kQTerms; ++term) {
              const uint4 qa = lds128(qimg_base + ((term * Cfg::KS + 2 * kp) * 32 + lane) * 16);
              mma_kv<KV8>(sacc[nt], qa.x, qa.y, qa.z, qa.w, kf.x, kf.y);
              const uint4 qb = lds128(qimg_base + ((term * Cfg::KS + 2 * kp + 1) * 32 + lane) * 16);
              mma_kv<KV8>(sacc[nt], qb.x, qb.y, qb.z, qb.w, kf.z, kf.w);
            }
          }
        }
        // logits (log2 units): query g -> sacc[nt][0..1], query g+8 -> sacc[nt][2..3];
        // tokens 2c, 2c+1 (nt 0) and 8+2c, 9+2c (nt 1)
        float sv[2][4];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          sv[r][0] = sacc[0][2 * r];
          sv[r][1] = sacc[0][2 * r + 1];
          sv[r][2] = sacc[1][2 * r];
          sv[r][3] = sacc[1][2 * r + 1];
          if (valid_tok < 16) {
            if (2 * c >= valid_tok) sv[r][0] = -INFINITY;
            if (2 * c + 1 >= valid_tok) sv[r][1] = -INFINITY;
            if (8 + 2 * c >= valid_tok) sv[r][2] = -INFINITY;
            if (9 + 2 * c >= valid_tok) sv[r][3] = -INFINITY;
          }
        }
        float mx[2];
        bool grow[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          mx[r] = fmaxf(fmaxf(sv[r][0], sv[r][1]), fmaxf(sv[r][2], sv[r][3]));
          mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
          mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
          grow[r] = mx[r] > m_ref[r] + 8.f;  // lazy rescale, as the 8-row path
        }
        if (__any_sync(0xffffffffu, grow[0] || grow[1])) {
          float alpha[2];
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            const float m_new = grow[r] ? mx[r] : m_ref[r];
            alpha[r] = fast_exp2(m_ref[r] - m_new);  // 0 when m_ref = -inf
            l_sum[r] *= alpha[r];
            m_ref[r] = m_new;
          }
#pragma unroll
          for (int nd = 0; nd < Cfg::ND; ++nd) {
            acc[nd][0] *= alpha[0];
            acc[nd][1] *= alpha[0];
            acc[nd][2] *= alpha[1];
            acc[nd][3] *= alpha[1];
          }
        }
        float ph[2][4], pl[2][4];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float pv = fast_exp2(sv[r][i] - m_ref[r]);
            if constexpr (KV8) {
              // quantised pages: P as ONE f16 term (11 significant bits) -- the row sum
              // takes the same rounded weights, so the output stays an exact weighted
              // mean of V; half the P.V MMAs of the hi/lo split
              ph[r][i] = __half2float(__float2half_rn(pv));
              pl[r][i] = 0.f;
              l_sum[r] += ph[r][i];
            } else {
              l_sum[r] += pv;
              split2(pv, ph[r][i], pl[r][i]);
            }
          }
        }
        // P A-fragments (rows = queries g, g+8; k = tokens): hi tile and lo tile
        const uint32_t h0 = pack_kv<KV8>(ph[0][0], ph[0][1]), h1 = pack_kv<KV8>(ph[1][0], ph[1][1]);
        const uint32_t h2 = pack_kv<KV8>(ph[0][2], ph[0][3]), h3 = pack_kv<KV8>(ph[1][2], ph[1][3]);
        const uint32_t q0 = pack_kv<KV8>(pl[0][0], pl[0][1]), q1 = pack_kv<KV8>(pl[1][0], pl[1][1]);
        const uint32_t q2 = pack_kv<KV8>(pl[0][2], pl[0][3]), q3 = pack_kv<KV8>(pl[1][2], pl[1][3]);
        // ---- O += P V
#pragma unroll
        for (int nd2 = 0; nd2 < Cfg::ND / 2; ++nd2) {
          const int ci = nd2 * 32 + lane;
          const uint4 vf = load_v<DP, KVF>(pbase, ci);
          mma_kv<KV8>(acc[2 * nd2], h0, h1, h2, h3, vf.x, vf.y);
          if constexpr (!KV8) mma_kv<KV8>(acc[2 * nd2], q0, q1, q2, q3, vf.x, vf.y);
          mma_kv<KV8>(acc[2 * nd2 + 1], h0, h1, h2, h3, vf.z, vf.w);
          if constexpr (!KV8) mma_kv<KV8>(acc[2 * nd2 + 1], q0, q1, q2, q3, vf.z, vf.w);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);

      if (m.last) {
        // ---- combine the NWC warps' (m, l, O) for the item's 16 rows
        float* ws = scratch + warp * WS;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          float l_tot = l_sum[r];
          l_tot += __shfl_xor_sync(0xffffffffu, l_tot, 1);
          l_tot += __shfl_xor_sync(0xffffffffu, l_tot, 2);
          if (c == 0) {
            ws[SR * DP + g + 8 * r] = m_ref[r];  // -inf for warps that saw no page
            ws[SR * DP + SR + g + 8 * r] = l_tot;
          }
        }
#pragma unroll
        for (int nd = 0; nd < Cfg::ND; ++nd) {
          const int d = nd * 8 + 2 * c;
          ws[g * DP + d] = acc[nd][0];
          ws[g * DP + d + 1] = acc[nd][1];
          ws[(g + 8) * DP + d] = acc[nd][2];
          ws[(g + 8) * DP + d + 1] = acc[nd][3];
        }
        named_bar_sync(1, NWC * 32);
        const int rows = m.rows;
        const size_t obase = static_cast<size_t>(m.item) * QR * DP;
        for (int idx = threadIdx.x; idx < rows * DP; idx += NWC * 32) {
          const int q = idx / DP, d = idx - q * DP;
          float M = -INFINITY;
#pragma unroll
          for (int w = 0; w < NWC; ++w) M = fmaxf(M, scratch[w * WS + SR * DP + q]);
          float L = 0.f, O = 0.f;
#pragma unroll
          for (int w = 0; w < NWC; ++w) {
            const float* wsw = scratch + w * WS;
            const float mw = wsw[SR * DP + q];
            const float e = mw == -INFINITY ? 0.f : fast_exp2(mw - M);
            L += wsw[SR * DP + SR + q] * e;
            O += wsw[q * DP + d] * e;
          }
          p.part_o[obase + idx] = O / L;
          if (d == 0) p.part_lse2[static_cast<size_t>(m.item) * QR + q] = M + __log2f(L);
        }
        named_bar_sync(1, NWC * 32);
        if (p.fused) fused_stream_done<DP, NWC>(p, m.stream, m.rows, m.ntok);
        m_ref[0] = m_ref[1] = -INFINITY;
        l_sum[0] = l_sum[1] = 0.f;
#pragma unroll
        for (int nd = 0; nd < Cfg::ND; ++nd) acc[nd][0] = acc[nd][1] = acc[nd][2] = acc[nd][3] = 0.f;
      }
    }
  } else {
    // ------------------------------------------------------------ consumers
    const int g = lane >> 2, c = lane & 3;
    const int qch = warp % QC;   // this warp's query chunk (rows qch*8 .. qch*8+7 of the item)
    const int wpg = warp / QC;   // its page slot within the chunk's share of a stage
    uint32_t qa[Cfg::KS][4];  // M-tile 0: hi (rows 0-7), mid (rows 8-15)
    uint32_t qb[Cfg::KS][2];  // M-tile 1: lo (rows 0-7); rows 8-15 are zero
    float acc[Cfg::ND][4];
    float m_ref = -INFINITY, l_sum = 0.f;
    int st = 0;
    const uint32_t stage_base = smem_u32(stages);
    for (;; ++st) {
      const int s = st % NSTAGE;
      mbar_wait(&full[s], (st / NSTAGE) & 1);
      const StageMeta m = meta[s];
      if (m.item == kItemDone) break;
      const uint32_t sbase = stage_base + s * STAGE_BYTES;
      if (m.first) {
        // stage the item's query rows as hi/mid/lo bf16 fragments
        const float* qs = reinterpret_cast<const float*>(stages + s * STAGE_BYTES + STAGE_KV) + qch * 8 * DP;
        const bool valid = qch * 8 + g < m.rows;
#pragma unroll
        for (int ks = 0; ks < Cfg::KS; ++ks) {
          float v[4];
          const int d0 = ks * 16 + 2 * c;
          v[0] = valid ? qs[g * DP + d0] * p.qscale : 0.f;
          v[1] = valid ? qs[g * DP + d0 + 1] * p.qscale : 0.f;
          v[2] = valid ? qs[g * DP + d0 + 8] * p.qscale : 0.f;
          v[3] = valid ? qs[g * DP + d0 + 9] * p.qscale : 0.f;
          float hi[4], mid[4], lo[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            if constexpr (KV8) {
              // f16 hi + lo carries 22 significant bits (~fp32): one M-tile [hi; lo]
              split2h(v[i], hi[i], mid[i]);
              lo[i] = 0.f;
            } else {
              split3(v[i], hi[i], mid[i], lo[i]);
            }
          }
          if constexpr (QSM) {
            if (ks % WPC == wpg)  // the chunk's warps split the k-steps of its image
              qimg[(qch * Cfg::KS + ks) * 32 + lane] =
                  make_uint4(pack_kv<KV8>(hi[0], hi[1]), pack_kv<KV8>(mid[0], mid[1]), pack_kv<KV8>(hi[2], hi[3]),
                             pack_kv<KV8>(mid[2], mid[3]));
          } else {
            qa[ks][0] = pack_kv<KV8>(hi[0], hi[1]);
            qa[ks][1] = pack_kv<KV8>(mid[0], mid[1]);
            qa[ks][2] = pack_kv<KV8>(hi[2], hi[3]);
            qa[ks][3] = pack_kv<KV8>(mid[2], mid[3]);
            qb[ks][0] = pack_kv<KV8>(lo[0], lo[1]);
            qb[ks][1] = pack_kv<KV8>(lo[2], lo[3]);
          }
        }
        // (every warp finished the previous item: its combine ended with a barrier)
        if constexpr (QSM) named_bar_sync(1, NWC * 32);
#pragma unroll
        for (int nd = 0; nd < Cfg::ND; ++nd) acc[nd][0] = acc[nd][1] = acc[nd][2] = acc[nd][3] = 0.f;
        m_ref = -INFINITY;
        l_sum = 0.f;
      }
#pragma unroll
      for (int kq = 0; kq < QC; ++kq) {
        const int pj = QC == 1 ? warp : wpg + kq * WPC;
        if (pj >= m.npages) break;
        const uint32_t pbase = sbase + pj * Cfg::PAGE;
        const int tok0 = (m.page0 + pj) * 16;
        const int valid_tok = m.ntok - tok0;  // >= 1
        // ---- S = Q K^T over the 16 tokens of this page
        float s0[2][4], s1[2][4];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int i = 0; i < 4; ++i) s0[nt][i] = s1[nt][i] = 0.f;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
          for (int kp = 0; kp < Cfg::KS / 2; ++kp) {
            const int ci = (nt * (Cfg::KS / 2) + kp) * 32 + lane;
            const uint4 kf = load_k<DP, KVF>(pbase, ci);
            const int k0 = 2 * kp, k1 = 2 * kp + 1;
            if constexpr (QSM) {
              const uint32_t qb0 = smem_u32(qimg) + ((qch * Cfg::KS + k0) * 32 + lane) * 16;
              const uint4 a0 = lds128(qb0), a1 = lds128(qb0 + 32 * 16);
              mma_kv<KV8>(s0[nt], a0.x, a0.y, a0.z, a0.w, kf.x, kf.y);
              mma_kv<KV8>(s0[nt], a1.x, a1.y, a1.z, a1.w, kf.z, kf.w);
            } else {
              mma_kv<KV8>(s0[nt], qa[k0][0], qa[k0][1], qa[k0][2], qa[k0][3], kf.x, kf.y);
              if constexpr (!KV8) mma_kv<KV8>(s1[nt], qb[k0][0], 0u, qb[k0][1], 0u, kf.x, kf.y);
              mma_kv<KV8>(s0[nt], qa[k1][0], qa[k1][1], qa[k1][2], qa[k1][3], kf.z, kf.w);
              if constexpr (!KV8) mma_kv<KV8>(s1[nt], qb[k1][0], 0u, qb[k1][1], 0u, kf.z, kf.w);
            }
          }
        }
        // logits (log2 units) for query row g, tokens 2c, 2c+1, 8+2c, 9+2c
        float sv[4];
        sv[0] = s0[0][0] + s0[0][2] + s1[0][0];
        sv[1] = s0[0][1] + s0[0][3] + s1[0][1];
        sv[2] = s0[1][0] + s0[1][2] + s1[1][0];
        sv[3] = s0[1][1] + s0[1][3] + s1[1][1];
        if (valid_tok < 16) {
          if (2 * c >= valid_tok) sv[0] = -INFINITY;
          if (2 * c + 1 >= valid_tok) sv[1] = -INFINITY;
          if (8 + 2 * c >= valid_tok) sv[2] = -INFINITY;
          if (9 + 2 * c >= valid_tok) sv[3] = -INFINITY;
        }
        float mx = fmaxf(fmaxf(sv[0], sv[1]), fmaxf(sv[2], sv[3]));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        // Lazy rescale: keep the reference max unless it grows by > 8 (log2),
        // exact in real arithmetic; bounds p by 2^8.
        const bool grow = mx > m_ref + 8.f;
        if (__any_sync(0xffffffffu, grow)) {
          const float m_new = grow ? mx : m_ref;
          const float alpha = fast_exp2(m_ref - m_new);  // 0 when m_ref = -inf
          l_sum *= alpha;
#pragma unroll
          for (int nd = 0; nd < Cfg::ND; ++nd)
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[nd][i] *= alpha;
          m_ref = m_new;
        }
        float pv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) pv[i] = fast_exp2(sv[i] - m_ref);
        l_sum += (pv[0] + pv[1]) + (pv[2] + pv[3]);
        uint32_t a0, a1, a2, a3;
        if constexpr (KV8) {
          split2h_pack(pv[0], pv[1], a0, a1);
          split2h_pack(pv[2], pv[3], a2, a3);
        } else {
          float ph[4], pl[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) split2(pv[i], ph[i], pl[i]);
          a0 = pack_bf16(ph[0], ph[1]);
          a1 = pack_bf16(pl[0], pl[1]);
          a2 = pack_bf16(ph[2], ph[3]);
          a3 = pack_bf16(pl[2], pl[3]);
        }
        // ---- O += P V
#pragma unroll
        for (int nd2 = 0; nd2 < Cfg::ND / 2; ++nd2) {
          const int ci = nd2 * 32 + lane;
          const uint4 vf = load_v<DP, KVF>(pbase, ci);
          mma_kv<KV8>(acc[2 * nd2], a0, a1, a2, a3, vf.x, vf.y);
          mma_kv<KV8>(acc[2 * nd2 + 1], a0, a1, a2, a3, vf.z, vf.w);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);

      if (m.last) {
        // ---- combine the NWC warps' (m, l, O) for this item
        float* ws = scratch + warp * WS;
        float l_tot = l_sum;
        l_tot += __shfl_xor_sync(0xffffffffu, l_tot, 1);
        l_tot += __shfl_xor_sync(0xffffffffu, l_tot, 2);
        if (c == 0) {
          ws[8 * DP + g] = m_ref;      // -inf for warps that saw no page
          ws[8 * DP + 8 + g] = l_tot;
        }
#pragma unroll
        for (int nd = 0; nd < Cfg::ND; ++nd) {
          const int d = nd * 8 + 2 * c;
          ws[g * DP + d] = acc[nd][0] + acc[nd][2];
          ws[g * DP + d + 1] = acc[nd][1] + acc[nd][3];
        }
        named_bar_sync(1, NWC * 32);
        const int rows = m.rows;
        const size_t obase = static_cast<size_t>(m.item) * QR * DP;
        for (int idx = threadIdx.x; idx < rows * DP; idx += NWC * 32) {
          const int qi = idx / DP, d = idx - qi * DP;
          const int qc = qi >> 3, q = qi & 7;  // chunk qc is combined over warps qc, qc + QC, ...
          float M = -INFINITY;
#pragma unroll
          for (int w = qc; w < NWC; w += QC) M = fmaxf(M, scratch[w * WS + 8 * DP + q]);
          float L = 0.f, O = 0.f;
#pragma unroll
          for (int w = qc; w < NWC; w += QC) {
            const float* wsw = scratch + w * WS;
            const float mw = wsw[8 * DP + q];
            const float e = mw == -INFINITY ? 0.f : fast_exp2(mw - M);
            L += wsw[8 * DP + 8 + q] * e;
            O += wsw[q * DP + d] * e;
          }
          p.part_o[obase + idx] = O / L;
          if (d == 0) p.part_lse2[static_cast<size_t>(m.item) * QR + qi] = M + __log2f(L);
        }
        named_bar_sync(1, NWC * 32);
        if (p.fused) fused_stream_done<DP, NWC>(p, m.stream, m.rows, m.ntok);
        // the next item re-initialises state on its first stage
        m_ref = -INFINITY;
        l_sum = 0.f;
#pragma unroll
        for (int nd = 0; nd < Cfg::ND; ++nd) acc[nd][0] = acc[nd][1] = acc[nd][2] = acc[nd][3] = 0.f;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(p.done_counter, 1) == static_cast<int>(gridDim.x) - 1) {
      // every CTA has drained the work queue: reset for the next launch / graph replay
      *p.work_counter = 0;
      *p.done_counter = 0;
      __threadfence();
    }
  }
}

// ------------------------------------------------------------------------
// Split reduce: merge a stream's split partials into the rank's fragment for
// each query head, natural-log lse (HeadFragment, attention.hpp:56-59; empty
// shard -> (0, -inf) as at :69-70). One CTA per (stream, query row): warp w
// takes splits w, w+8, ... in order (all its loads in flight together), the 8
// warp partials are combined in warp order -- deterministic, one load round.
constexpr int kSrWarps = 8;
template <int DP>
__global__ void __launch_bounds__(kSrWarps * 32) attn_split_reduce_kernel(const AttnParams p, float* frag_o,
                                                                          float* frag_lse) {
  griddep_wait();
  griddep_launch_dependents();
  __shared__ float s_m[kSrWarps], s_l[kSrWarps];
  __shared__ float s_o[kSrWarps][DP];
  const int QR = p.qrows;  // query rows per stream: 8 or 16
  const int row = blockIdx.x % QR;
  const int stream = blockIdx.x / QR;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int t = stream;
  const int qc = t % p.q_chunks; t /= p.q_chunks;
  const int kvh = t % p.kvh_per_slot; t /= p.kvh_per_slot;
  const int b = t % p.stream_batch + p.b_begin;
  const int slot_local = t / p.stream_batch;
  const int slot = slot_local + p.slot_base;
  const int rank = slot % p.kvp;
  const int qrow = qc * QR + row;
  if (qrow >= p.group) {  // whole CTA: nothing to reduce, still one unit of the exchange count
    if (p.push && threadIdx.x == 0) signal_pushed(p, gridDim.x);
    return;
  }
  const int ntok = static_cast<int>(rr_count(p.total[b], rank, p.chunk, p.kvp));
  const int pages = (ntok + 15) >> 4;
  constexpr int PER = DP / 32;
  auto valid = [&](int s) {
    const int pg0 = static_cast<int>((static_cast<long long>(s) * pages) / p.splits);
    const int pg1 = static_cast<int>((static_cast<long long>(s + 1) * pages) / p.splits);
    return pg1 > pg0;
  };
  // pass 1: max lse over the non-empty splits
  float M = -INFINITY;
  for (int s = warp * 32 + lane; s < p.splits; s += kSrWarps * 32)
    if (valid(s)) M = fmaxf(M, p.part_lse2[attn_item(p, stream, s) * QR + row]);
#pragma unroll
  for (int o2 = 16; o2 > 0; o2 >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o2));
  if (lane == 0) s_m[warp] = M;
  __syncthreads();
  M = s_m[0];
#pragma unroll
  for (int w = 1; w < kSrWarps; ++w) M = fmaxf(M, s_m[w]);
  // pass 2: this warp's splits in order, 4 at a time with every load issued first
  float o[PER], L = 0.f;
#pragma unroll
  for (int i = 0; i < PER; ++i) o[i] = 0.f;
  for (int s0 = warp; s0 < p.splits; s0 += 4 * kSrWarps) {
    float w4[4], v[4][PER];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int s = s0 + j * kSrWarps;
      const bool ok = s < p.splits && valid(s);
      const size_t item = attn_item(p, stream, ok ? s : 0);
      w4[j] = ok ? p.part_lse2[item * QR + row] : -INFINITY;
#pragma unroll
      for (int i = 0; i < PER; ++i) v[j][i] = ok ? p.part_o[(item * QR + row) * DP + lane + 32 * i] : 0.f;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float e = w4[j] == -INFINITY ? 0.f : exp2f(w4[j] - M);
#pragma unroll
      for (int i = 0; i < PER; ++i) o[i] += v[j][i] * e;
      L += e;
    }
  }
#pragma unroll
  for (int i = 0; i < PER; ++i) s_o[warp][lane + 32 * i] = o[i];
  if (lane == 0) s_l[warp] = L;
  __syncthreads();
  if (warp == 0) {
    float Lt = 0.f, ot[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) ot[i] = 0.f;
#pragma unroll
    for (int w = 0; w < kSrWarps; ++w) {
      Lt += s_l[w];
#pragma unroll
      for (int i = 0; i < PER; ++i) ot[i] += s_o[w][lane + 32 * i];
    }
    // fragment layout: [slot_local][b][q_in_group][DP]
    const int q_in_group = kvh * p.group + qrow;
    const size_t fo = ((static_cast<size_t>(slot_local) * p.batch + b) * p.q_per_slot + q_in_group);
#pragma unroll
    for (int i = 0; i < PER; ++i) frag_o[fo * DP + lane + 32 * i] = Lt > 0.f ? ot[i] / Lt : 0.f;
    if (lane == 0) frag_lse[fo] = Lt > 0.f ? (M + log2f(Lt)) * 0.69314718055994530942f : -INFINITY;
    if (p.xf_out) {  // one-source pool: the merged attention output IS this fragment
      const int head = ((slot_local + p.slot_base) / p.kvp) * p.q_per_slot + q_in_group;
#pragma unroll
      for (int i = 0; i < PER; ++i)
        if (lane + 32 * i < p.hd)
          xf_write(p.xf_out, xf_nb8(p.batch), b, head * p.hd + lane + 32 * i, Lt > 0.f ? ot[i] / Lt : 0.f, p.xf16);
    }
    if (p.push) {  // device-initiated exchange straight from the reduce (no pack, no collective)
#pragma unroll
      for (int i = 0; i < PER; ++i)
        if (lane + 32 * i < p.hd) push_value(p, b, q_in_group, lane + 32 * i, Lt > 0.f ? ot[i] / Lt : 0.f);
      if (lane == 0) push_lse(p, b, q_in_group, Lt > 0.f ? (M + log2f(Lt)) * 0.69314718055994530942f : -INFINITY);
    }
  }
  if (p.push) {
    __syncthreads();
    if (threadIdx.x == 0) signal_pushed(p, gridDim.x);
  }
}

// Few splits (<= 8, e.g. large batches): one WARP per (stream, query row),
// lanes across the head dim, splits merged in order with all loads issued
// first -- the 8-warp CTA above would idle most of its warps.
template <int DP>
__global__ void __launch_bounds__(256) attn_split_reduce_small_kernel(const AttnParams p, float* frag_o,
                                                                      float* frag_lse) {
  griddep_wait();
  griddep_launch_dependents();
  const int QR = p.qrows;
  const int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int row = wg % QR, stream = wg / QR;
  if (stream < p.n_streams && (stream % p.q_chunks) * QR + row < p.group) {
  int t = stream;
  const int qc = t % p.q_chunks; t /= p.q_chunks;
  const int kvh = t % p.kvh_per_slot; t /= p.kvh_per_slot;
  const int b = t % p.stream_batch + p.b_begin;
  const int slot_local = t / p.stream_batch;
  const int rank = (slot_local + p.slot_base) % p.kvp;
  const int qrow = qc * QR + row;
  const int ntok = static_cast<int>(rr_count(p.total[b], rank, p.chunk, p.kvp));
  const int pages = (ntok + 15) >> 4;
  constexpr int PER = DP / 32;
  float w[8], v[8][PER];
  float M = -INFINITY;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int pg0 = static_cast<int>((static_cast<long long>(j) * pages) / p.splits);
    const int pg1 = static_cast<int>((static_cast<long long>(j + 1) * pages) / p.splits);
    const bool ok = j < p.splits && pg1 > pg0;
    const size_t item = attn_item(p, stream, ok ? j : 0);
    w[j] = ok ? p.part_lse2[item * QR + row] : -INFINITY;
#pragma unroll
    for (int i = 0; i < PER; ++i) v[j][i] = ok ? p.part_o[(item * QR + row) * DP + lane + 32 * i] : 0.f;
    M = fmaxf(M, w[j]);
  }
  float o[PER], L = 0.f;
#pragma unroll
  for (int i = 0; i < PER; ++i) o[i] = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float e = w[j] == -INFINITY ? 0.f : exp2f(w[j] - M);
#pragma unroll
    for (int i = 0; i < PER; ++i) o[i] += v[j][i] * e;
    L += e;
  }
  const int q_in_group = kvh * p.group + qrow;
  const size_t fo = ((static_cast<size_t>(slot_local) * p.batch + b) * p.q_per_slot + q_in_group);
#pragma unroll
  for (int i = 0; i < PER; ++i) frag_o[fo * DP + lane + 32 * i] = L > 0.f ? o[i] / L : 0.f;
  if (lane == 0) frag_lse[fo] = L > 0.f ? (M + log2f(L)) * 0.69314718055994530942f : -INFINITY;
  if (p.xf_out) {  // one-source pool: the merged attention output IS this fragment
    const int head = ((slot_local + p.slot_base) / p.kvp) * p.q_per_slot + q_in_group;
#pragma unroll
    for (int i = 0; i < PER; ++i)
      if (lane + 32 * i < p.hd)
        xf_write(p.xf_out, xf_nb8(p.batch), b, head * p.hd + lane + 32 * i, L > 0.f ? o[i] / L : 0.f, p.xf16);
  }
  if (p.push) {  // device-initiated exchange straight from the reduce
#pragma unroll
    for (int i = 0; i < PER; ++i)
      if (lane + 32 * i < p.hd) push_value(p, b, q_in_group, lane + 32 * i, L > 0.f ? o[i] / L : 0.f);
    if (lane == 0) push_lse(p, b, q_in_group, L > 0.f ? (M + log2f(L)) * 0.69314718055994530942f : -INFINITY);
  }
  }  // active warp
  if (p.push) {
    __syncthreads();
    if (threadIdx.x == 0) signal_pushed(p, gridDim.x);
  }
}

// HOP-B without stalling the KV stream (AttnParams::fused == 2, overlap.hpp:37-69
// at stream granularity): the attention kernel only publishes each stream's
// finished-split count; this kernel, launched right behind it with
// programmatic dependent launch and small enough (128 threads, no shared
// memory) to sit next to the attention CTAs on their SMs, reduces and pushes
// every stream as soon as its last split has landed -- request b's slices
// travel while the requests after it are still streaming KV, and no attention
// CTA ever pauses its stream for a reduce. Streams in request order (the
// attention's work order is stream-major under HOP-B).
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
constexpr int kSrRowsPerCta = 4;  // one warp per query row
template <int DP>
__global__ void __launch_bounds__(128) attn_stream_reduce_kernel(const AttnParams p) {
  const int warp = threadIdx.x >> 5;
#ifdef HX_SR_SERIAL
  griddep_wait();
#endif
  const int chunks = (p.qrows + kSrRowsPerCta - 1) / kSrRowsPerCta;
  // CTA = (stream, chunk of 4 query rows), dispatched in stream (= completion) order
  {
    const int stream = blockIdx.x / chunks, q0 = (blockIdx.x % chunks) * kSrRowsPerCta;
    int t = stream;
    const int qc = t % p.q_chunks;
    t /= p.q_chunks;
    t /= p.kvh_per_slot;
    const int b = t % p.stream_batch + p.b_begin;
    const int rank = (t / p.stream_batch + p.slot_base) % p.kvp;
    const int pages = (static_cast<int>(rr_count(p.total[b], rank, p.chunk, p.kvp)) + 15) >> 4;
    const int need = p.fused == 3 ? 0 : (pages < p.splits ? pages : p.splits);  // non-empty splits of the stream
    const int g_rows = p.group - qc * p.qrows;
    const int rows = g_rows < p.qrows ? g_rows : p.qrows;
    if (threadIdx.x == 0) {
      while (ld_acquire_gpu(p.stream_done + stream) < need) __nanosleep(512);  // light polling: L2 stays with the KV stream
    }
    __syncthreads();
    if (need == 0) {
      if (threadIdx.x == 0) reduce_stream<DP>(p, stream, rows, 0, 0, q0, q0 + kSrRowsPerCta);  // identity (0, -inf)
    } else {
      reduce_stream<DP>(p, stream, rows, warp, 4, q0, q0 + kSrRowsPerCta);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      // the stream's counter is reset by its last chunk (the others have read it)
      if (atomicAdd(p.stream_done + p.n_streams + stream, 1) == chunks - 1) {
        p.stream_done[stream] = 0;  // for the next launch / graph replay
        p.stream_done[p.n_streams + stream] = 0;
      }
      if (p.push) signal_pushed(p, gridDim.x);
    }
  }
  // completion of this grid implies the attention grid's (the next kernel's
  // griddepcontrol.wait sees only this one)
  griddep_wait();
  griddep_launch_dependents();
}

cudaError_t launch_attn_stream_reduce(const AttnParams& p, cudaStream_t stream) {
  const int grid = p.n_streams * ((p.qrows + kSrRowsPerCta - 1) / kSrRowsPerCta);
  switch (p.dp) {
    case 32: return launch_k(attn_stream_reduce_kernel<32>, dim3(grid), dim3(128), 0, stream, p);
    case 64: return launch_k(attn_stream_reduce_kernel<64>, dim3(grid), dim3(128), 0, stream, p);
    case 128: return launch_k(attn_stream_reduce_kernel<128>, dim3(grid), dim3(128), 0, stream, p);
    default: return cudaErrorInvalidValue;
  }
}

__global__ void bump_totals_kernel(int* total, int n) {
  griddep_wait();
  griddep_launch_dependents();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) total[i] += 1;
}

// ------------------------------------------------------------------------
// host launchers
template <int DP, int NWC, int NSTAGE, int QC, int KVF, bool W16>
static size_t attn_smem_bytes() {
  constexpr int SR = W16 ? 16 : 8;
  return NSTAGE * (NWC * AttnCfg<DP, KVF>::PAGE + QC * 8 * DP * 4) + NWC * (SR * DP + 2 * SR) * 4 +
         (W16 ? 3 * (DP / 16) * 32 * 16 : (KVF == 2 ? QC * (DP / 16) * 32 * 16 : 0)) + NSTAGE * sizeof(StageMeta) +
         2 * NSTAGE * 8 + 64;
}

template <int DP, int NWC, int NSTAGE, int QC, int KVF, bool W16>
static cudaError_t launch_attn_t(const AttnParams& p, int grid, cudaStream_t stream) {
  const size_t smem = attn_smem_bytes<DP, NWC, NSTAGE, QC, KVF, W16>();
  const cudaError_t e = smem_optin<attn_decode_kernel<DP, NWC, NSTAGE, QC, KVF, W16>>(smem);
  if (e != cudaSuccess) return e;
  return launch_k(attn_decode_kernel<DP, NWC, NSTAGE, QC, KVF, W16>, dim3(grid), dim3((NWC + 1) * 32), smem, stream,
                  p);
}

// bf16 pages: 2-4 stages of 8 pages; FP8 pages are half the bytes, so twice the
// stages in flight. 9-16 query rows of bf16 pages take the W16 consumers.
template <int QC, int KVF>
static cudaError_t launch_attn_dp(const AttnParams& p, int grid, cudaStream_t stream) {
  constexpr bool W16 = QC == 2;  // 9-16 query rows: every warp takes 16 rows
  constexpr bool KV8 = KVF != 0;
  switch (p.dp) {
    case 32: return launch_attn_t<32, 8, KV8 ? 8 : 4, QC, KVF, W16>(p, grid, stream);
    case 64: return launch_attn_t<64, 8, KV8 ? 6 : 3, QC, KVF, W16>(p, grid, stream);
    case 128:
      // FP4 pages (2240 B each): the widening + scaling dominates the consumer work --
      // as many consumer warps as registers allow: with the query fragments in shared
      // memory (QSM) 12 warps x 4 stages at 128 registers (configs[1] FP4 KV, 8 layers:
      // 3.43 ms vs 3.56 at 10 x 6, 3.46 at 12 x 5, 3.48 at 14 x 4; registers-held
      // query at 10 x 6: 3.66 ms)
      if constexpr (KVF == 2 && QC == 1) return launch_attn_t<128, 12, 4, QC, KVF, W16>(p, grid, stream);
      // 16-row (W16) FP4 consumers, single-term P (128 registers): 12 warps x 3 stages,
      // 405B-like FP4 slice 0.406 ms vs 0.463 at 8 x 4, 0.444 at 10 x 4, 0.419 at 14 x 2
      // (14 x 3 and 12 x 4 exceed the shared memory)
      else if constexpr (KVF == 2) return launch_attn_t<128, 12, 3, QC, KVF, W16>(p, grid, stream);
      else {
      // FP8 pages: 10 consumer warps x 4 stages (217 KB of shared memory) -- the
      // e4m3 widening doubles the per-byte consumer work, so more pages in flight
      // per SM: 0.366 -> 0.339 ms per configs[1] launch vs 8 x 4 (12 x 3: 0.351)
      if constexpr (KV8 && QC == 1) return launch_attn_t<128, 10, 4, QC, KVF, W16>(p, grid, stream);
      // 16 rows per warp (W16) of FP8 pages: 12 warps x 2 stages next to the 16-row
      // scratch (224 KB; 405B-like FP8 slice 0.430 ms vs 0.450 at 8 x 3, 0.479 at 10 x 2)
      if constexpr (KV8) return launch_attn_t<128, 12, 2, QC, KVF, W16>(p, grid, stream);
      // bf16 pages, 8 query rows: 7 consumer warps x 3 stages (168 KB of KV in flight):
      // configs[1] launch 0.606 -> 0.591 ms (7.27 TB/s) vs 8 x 2; 6 x 3 0.597, 5 x 4 0.603, 4 x 5 0.599
      if constexpr (!KV8 && QC == 1) return launch_attn_t<128, 7, 3, QC, KVF, W16>(p, grid, stream);
      return launch_attn_t<128, 8, 2, QC, KVF, W16>(p, grid, stream);
      }
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_attn_decode(const AttnParams& p, int grid, cudaStream_t stream) {
  if (p.qrows != 8 && p.qrows != 16) return cudaErrorInvalidValue;
  if (p.kv4) return p.qrows == 16 ? launch_attn_dp<2, 2>(p, grid, stream) : launch_attn_dp<1, 2>(p, grid, stream);
  if (p.kv8) return p.qrows == 16 ? launch_attn_dp<2, 1>(p, grid, stream) : launch_attn_dp<1, 1>(p, grid, stream);
  return p.qrows == 16 ? launch_attn_dp<2, 0>(p, grid, stream) : launch_attn_dp<1, 0>(p, grid, stream);
}

cudaError_t launch_attn_split_reduce(const AttnParams& p, float* frag_o, float* frag_lse,
                                     cudaStream_t stream) {
  if (p.splits <= 8) {  // one warp per (stream, query row)
    const int blocks = (p.n_streams * p.qrows + 7) / 8;
    switch (p.dp) {
      case 32: return launch_k(attn_split_reduce_small_kernel<32>, dim3(blocks), dim3(256), 0, stream, p, frag_o, frag_lse);
      case 64: return launch_k(attn_split_reduce_small_kernel<64>, dim3(blocks), dim3(256), 0, stream, p, frag_o, frag_lse);
      case 128: return launch_k(attn_split_reduce_small_kernel<128>, dim3(blocks), dim3(256), 0, stream, p, frag_o, frag_lse);
      default: return cudaErrorInvalidValue;
    }
  }
  const int blocks = p.n_streams * p.qrows;  // one CTA per (stream, query row)
  const int threads = kSrWarps * 32;
  switch (p.dp) {
    case 32: return launch_k(attn_split_reduce_kernel<32>, dim3(blocks), dim3(threads), 0, stream, p, frag_o, frag_lse);
    case 64: return launch_k(attn_split_reduce_kernel<64>, dim3(blocks), dim3(threads), 0, stream, p, frag_o, frag_lse);
    case 128: return launch_k(attn_split_reduce_kernel<128>, dim3(blocks), dim3(threads), 0, stream, p, frag_o, frag_lse);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_bump_totals(int* total, int n, cudaStream_t stream) {
  return launch_k(bump_totals_kernel, dim3((n + 127) / 128), dim3(128), 0, stream, total, n);
}

static bool g_pdl = true;
void set_pdl(bool on) { g_pdl = on; }
bool pdl_enabled() { return g_pdl; }

size_t attn_decode_smem_bytes(int dp) {
  switch (dp) {  // the larger (two query chunks) variant
    case 32: return attn_smem_bytes<32, 8, 4, 2, 0, true>();
    case 64: return attn_smem_bytes<64, 8, 3, 2, 0, true>();
    case 128: return attn_smem_bytes<128, 8, 2, 2, 0, true>();
    default: return 0;
  }
}

}  // namespace hx
