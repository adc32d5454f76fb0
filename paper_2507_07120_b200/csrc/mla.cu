// MLA decode attention on the 5th-generation tensor cores (tcgen05 + TMEM),
// one CTA PAIR (cluster of 2, cta_group::2) per work item.
//
// Per (rank shard, request): 128 query heads share one latent KV "head" of
// width W = 576 (keys = the latent, values = its first 512 dims):
//   S = Q . C^T / sqrt(W),  P = exp(S - m),  O = P . C[:, :512]
// -- partial_head_attention (attention.hpp:65-78) for every head of the rank
// with each head's LSE (HeadFragment), so the fragments merge exactly as
// merge_head_fragments (:118-137). ~242 FLOP per KV byte: at the B200 ridge.
//
// Transposed, paired formulation (exact FLOPs, each latent byte staged once
// per pair):
//   S^T = C . Q^T   UMMA M = 256 tokens (128 per CTA: each CTA stages ONLY its
//                   own 128-row page), N = 128 heads (the B operand is split by
//                   N: each CTA holds HALF the query image, 73.7 KB), K = 576
//   softmax per head = per COLUMN of S^T: warp redux.max over token lanes,
//                   4 warps through shared memory, the pair through DSMEM
//   O^T += V^T . P^T  M = 256 value dims (128 per CTA, two blocks cover 512),
//                   N = 128 heads (each CTA holds P^T for its 64 heads; every
//                   thread writes its token's P to both CTAs), K = 256 tokens
// The fp32 O^T [512 dims x 128 heads] is split across the pair's TMEM (256
// columns each); per-head row sums are kept per thread and reduced at the end.
//
// TMEM (per CTA, 512 columns x 128 lanes):
//   S^T buffer 0 [0,128)   S^T buffer 1 [128,256)   O^T block 0 [256,384)   block 1 [384,512)
// Shared memory (per CTA, same offsets in both): Q^T half 73,728 B | S ring
// 3 x 16 KB (64 dims x 128 own rows) | V ring 2 x 32 KB (128 dims x 128 rows)
// | P^T 32 KB [tokens 256 x this CTA's 64 heads] | exchange arrays + barriers.
// Roles (352 threads per CTA):
//   warps 0-7  softmax / correction: two warpgroups on the same TMEM lanes
//              (thread = token lane of S^T, = dim lane of O^T), warpgroup k
//              owns heads [64k, 64k+64) -- exactly the heads whose P^T lives
//              in CTA k, so one warpgroup writes locally, the other remotely
//   warps 8,11 S producers: cp.async.bulk of the Q^T half (warp 8) and the S
//              chunks (even / odd chunks: a warp issues ~1 bulk copy per 300 ns,
//              so two issuers double the per-SM ingest of 16 KB chunks)
//   warp 10    V producer: cp.async.bulk of the V blocks (own ring, runs ahead)
//   warp 9     TMEM alloc (pair); leader CTA: MMA issue (one thread), in the
//              order S(0) S(1) V(0) S(2) V(1) ...; peer CTA: forwards "Q half
//              landed" to the leader. Latent chunks are loaded with 2-SM tensor
//              TMA (UTMALDG.2CTA) by both CTAs and complete on the LEADER's
//              barriers, so no per-chunk relay is needed.
// Per-tile pair exchanges avoid cluster-scope fences: the column maxima and
// the peer's half of P^T travel as st.async (completing tx on the peer's
// mbarrier); only the per-item head sums use release/acquire.
#include "common.cuh"
#include "kernels.h"
#include "kv_layout.cuh"
#include "tc05.cuh"
#include "xfrag.cuh"
#ifdef HX_MLA_TRACE
#include <cstdio>
#endif

namespace hx {

namespace {
// Threads: NWG softmax warpgroups (warps 0 .. 4 NWG - 1) + S producer, MMA
// issuer, V producer, second S producer.
__host__ __device__ constexpr int mla_threads(int nwg) { return 32 * (4 * nwg + 4); }

// Per-variant geometry. bf16 latents (F8 = false): kind::f16, K = 16 per MMA;
// FP8 latents (F8 = true, kv_layout.cuh mla_kv_offset8): kind::f8f6f4 with e4m3
// latents, an e4m3 query image (per-head power-of-two scale) and e4m3 P, K = 32
// per MMA -- the same tile shapes at half the bytes and twice the MMA rate.
template <bool F8>
struct MlaCfg {
  static constexpr uint32_t kQHalf = F8 ? 36u * 1024u : kMlaW * 64u * 2u;  // query image half (64 heads)
  static constexpr int kSRows = F8 ? 12 : 8;          // 2 KB page rows per S chunk (192 / 64 dims)
  static constexpr uint32_t kSChunk = kSRows * 2048u;  // 24 / 16 KB
  static constexpr int kSChunks = F8 ? 3 : 9;
  static constexpr int kSMmas = F8 ? 6 : 4;            // MMAs per S chunk (2 dim groups each)
  static constexpr int kVRows = F8 ? 8 : 16;           // 128 value dims x 128 rows
  static constexpr uint32_t kVBlock = kVRows * 2048u;
  static constexpr int kSSlots = 3, kVSlots = F8 ? 4 : 2;  // barrier slots: S <= 3, V <= 4
  static_assert(kSSlots <= 3 && kVSlots <= 4, "mbarrier index layout (mla_decode_kernel)");
  static constexpr uint32_t kPTPage = F8 ? 8192u : 16384u;  // P^T of 128 tokens x 64 heads
  static constexpr uint32_t kPT = 2 * kPTPage;
  static constexpr uint32_t kPTLbo = F8 ? 512u : 1024u;     // P^T stride between 8-token groups
  static constexpr int kPVMmas = F8 ? 4 : 8;                // MMAs per 128-token page (K = 32 / 16)
  static constexpr uint32_t kPVAStep = F8 ? 512u : 256u;    // V^T bytes per MMA along K (tokens)
  static constexpr uint32_t kIdescST = F8 ? umma_idesc_e4m3(256, 128, false, false) : umma_idesc_bf16(256, 128, false, false);
  static constexpr uint32_t kIdescOT = F8 ? umma_idesc_e4m3(256, 128, true, true) : umma_idesc_bf16(256, 128, true, true);
  // shared-memory carve-up
  static constexpr uint32_t kOffQ = 0;
  static constexpr uint32_t kOffS = kOffQ + kQHalf;
  static constexpr uint32_t kOffV = kOffS + kSSlots * kSChunk;
  // P^T buffers: FP8 double-buffers (softmax(g+1) writes while P.V(g) runs; the
  // bf16 variant has no shared memory left for a second 32 KB buffer)
  static constexpr int kPTBufs = F8 ? 2 : 1;
  static constexpr uint32_t kOffPT = kOffV + kVSlots * kVBlock;
  static constexpr uint32_t kOffRed = kOffPT + kPTBufs * kPT;  // float [8 warps][64 heads] (max / sum)
  static constexpr uint32_t kOffMin = kOffRed + 4 * 128 * 4;  // float [2][128] peer maxima
  static constexpr uint32_t kOffMuse = kOffMin + 2 * 128 * 4;
  static constexpr uint32_t kOffAlpha = kOffMuse + 128 * 4;
  static constexpr uint32_t kOffZin = kOffAlpha + 128 * 4;    // float [2][128] peer sums
  static constexpr uint32_t kOffZs = kOffZin + 2 * 128 * 4;
  static constexpr uint32_t kOffCs = kOffZs + 128 * 4;        // float [128] score scale per head (FP8 q)
  static constexpr uint32_t kOffFl = kOffCs + 128 * 4;       // float [2] the peer's "some head grows" flag
  static constexpr uint32_t kOffBar = kOffFl + 16;
  static constexpr int kNumBars = 32;
  static constexpr uint32_t kSmem = kOffBar + kNumBars * 8 + 16;
};

struct MlaItem {
  int b, sl, pg0, pg1, ntok;
};

__device__ __forceinline__ MlaItem decode_item(const AttnParams& p, int item) {
  MlaItem it;
  const int split = item / p.n_streams;
  const int stream = item - split * p.n_streams;
  const int bl = stream % p.stream_batch;
  it.sl = stream / p.stream_batch;
  it.b = bl + p.b_begin;
  const int rank = (it.sl + p.slot_base) % p.kvp;
  it.ntok = static_cast<int>(rr_count(p.total[it.b], rank, p.chunk, p.kvp));
  const int pages = (it.ntok + kMlaPageRows - 1) / kMlaPageRows;
  it.pg0 = static_cast<int>((static_cast<long long>(split) * pages) / p.splits);
  it.pg1 = static_cast<int>((static_cast<long long>(split + 1) * pages) / p.splits);
  return it;
}

// Consumption order of an item's stages (producer, forwarder and MMA agree):
//   S(0), S(1), V(0), S(2), V(1), ..., S(n-1), V(n-2), V(n-1)
__device__ __forceinline__ void mla_step(int k, int n, int& tile, bool& value) {
  if (n == 1) {
    tile = 0;
    value = k == 1;
    return;
  }
  if (k < 2) {
    tile = k;
    value = false;
    return;
  }
  const int j = k - 2;
  tile = j / 2 + ((j & 1) ? 2 : 0);
  value = (j & 1) == 0;
  if (tile >= n) {
    tile = n - 1;
    value = true;
  }
}
#ifdef HX_MLA_TRACE
// per-tile event times of the first CTA pair's leader (debug builds: HX_NVCC_FLAGS=-DHX_MLA_TRACE)
__device__ unsigned long long g_mla_trace[64][12];
__device__ __forceinline__ unsigned long long mla_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define MLA_TRACE(g, ev, cond) \
  do { if (blockIdx.x == 0 && (g) < 64 && (cond)) g_mla_trace[g][ev] = mla_gtime(); } while (0)
#else
#define MLA_TRACE(g, ev, cond) do {} while (0)
#endif

// four floats -> four e4m3 bytes (RNE, saturating), a in the lowest byte
__device__ __forceinline__ uint32_t pack_e4m3x4(float a, float b, float c, float d) {
  uint32_t r;
  asm("{\n.reg .b16 lo, hi;\ncvt.rn.satfinite.e4m3x2.f32 lo, %2, %1;\ncvt.rn.satfinite.e4m3x2.f32 hi, %4, %3;\n"
      "mov.b32 %0, {lo, hi};\n}"
      : "=r"(r)
      : "f"(a), "f"(b), "f"(c), "f"(d));
  return r;
}
}  // namespace

template <bool F8, int NWG>
__global__ void __launch_bounds__(mla_threads(NWG), 1) mla_decode_kernel(const AttnParams p, const __grid_constant__ CUtensorMap tm_s,
                                                                   const __grid_constant__ CUtensorMap tm_v) {
  using C = MlaCfg<F8>;
  constexpr uint32_t kQHalf = C::kQHalf, kSChunk = C::kSChunk, kVBlock = C::kVBlock;
  constexpr int kSChunks = C::kSChunks, kSSlots = C::kSSlots, kVSlots = C::kVSlots;
  constexpr uint32_t kOffQ = C::kOffQ, kOffS = C::kOffS, kOffV = C::kOffV, kOffPT = C::kOffPT;
  constexpr uint32_t kOffRed = C::kOffRed, kOffMin = C::kOffMin, kOffMuse = C::kOffMuse, kOffAlpha = C::kOffAlpha;
  constexpr uint32_t kOffZin = C::kOffZin, kOffZs = C::kOffZs, kOffBar = C::kOffBar;
  constexpr int kNumBars = C::kNumBars;
  const uint32_t page_bytes = mla_page_bytes(F8), q_bytes = mla_q_bytes(F8);
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint64_t* full_s = bars + 0;       // [3]
  uint64_t* empty_s = bars + 3;      // [3]
  uint64_t* full_v = bars + 6;       // [kVSlots <= 4]
  uint64_t* empty_v = bars + 10;     // [kVSlots <= 4]
  uint64_t* q_full = bars + 15;
  uint64_t* q_free = bars + 16;
  uint64_t* pq_full = bars + 17;     // leader: peer's Q half landed
  uint64_t* s_full = bars + 18;      // [2] per S^T buffer
  uint64_t* pt_full = bars + 20;     // [kPTBufs] P^T of this CTA complete: 256 local arrivals + the peer's st.async bytes
                                     // (+1: the peer's forward, leader only)
  uint64_t* pv_done = bars + 22;     // [kPTBufs] P.V(g) complete (g % kPTBufs)
  uint64_t* o_free = bars + 24;      // leader: both CTAs' softmax threads read O^T
  uint64_t* mx_bar = bars + 25;      // [2] peer maxima arrived (1 arrival + 512 tx bytes)
  uint64_t* zx_bar = bars + 27;      // [2] peer sums arrived (128 arrivals)
  uint64_t* fl_bar = bars + 29;      // [2] peer flag arrived (1 arrival + 4 tx bytes)
  constexpr int NPT = C::kPTBufs;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + kNumBars);
  float* red = reinterpret_cast<float*>(smem + kOffRed);
  float* m_in = reinterpret_cast<float*>(smem + kOffMin);
  float* m_use = reinterpret_cast<float*>(smem + kOffMuse);
  float* alpha_s = reinterpret_cast<float*>(smem + kOffAlpha);
  float* z_in = reinterpret_cast<float*>(smem + kOffZin);
  float* zs = reinterpret_cast<float*>(smem + kOffZs);
  float* cs = reinterpret_cast<float*>(smem + C::kOffCs);  // FP8: qscale * 2^-e_h per head

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t cta = cluster_ctarank();
  const uint32_t peer = cta ^ 1u;
  const bool leader = cta == 0;
  const int cluster_id = blockIdx.x >> 1, n_clusters = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kSSlots; ++s) {
      mbar_init(&full_s[s], 1);
      mbar_init(&empty_s[s], 1);
    }
    for (int s = 0; s < kVSlots; ++s) {
      mbar_init(&full_v[s], 1);
      mbar_init(&empty_v[s], 1);
    }
    mbar_init(q_full, 1);
    mbar_init(q_free, 1);
    mbar_init(pq_full, 1);
    mbar_init(&s_full[0], 1);
    mbar_init(&s_full[1], 1);
    for (int i = 0; i < NPT; ++i) {
      mbar_init(&pt_full[i], 128 * NWG + (leader ? 1 : 0));
      mbar_init(&pv_done[i], 1);
    }
    mbar_init(o_free, 2 * 128 * NWG);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&mx_bar[i], 1);  // + 512 tx bytes of peer maxima per phase
      mbar_init(&zx_bar[i], 128);
      mbar_init(&fl_bar[i], 1);
    }
    fence_mbar_init();
  }
  constexpr int SW = 4 * NWG;                       // first non-softmax warp
  constexpr int kWarpS0 = SW, kWarpMma = SW + 1, kWarpV = SW + 2, kWarpS1 = SW + 3;
  constexpr int HPW = 128 / NWG;                     // heads per softmax warpgroup
  constexpr int kBarAll = 8;                         // named barrier of all softmax warps (warpgroups: 1 .. NWG)
  if (warp == kWarpMma) tmem_alloc_pair(tmem_slot, 512);
  tc_fence_before();
  cluster_sync_all();  // barriers of both CTAs initialised, TMEM allocated
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  griddep_launch_dependents();

  if (warp == kWarpS0 || warp == kWarpV || warp == kWarpS1) {
    // ------------------------------------------------------------ producers (S: two warps; V: one)
    if (lane == 0) {
      const bool sprod = warp != kWarpV;
      const uint32_t l_full_s = mapa_shared(smem_u32(full_s), 0), l_full_v = mapa_shared(smem_u32(full_v), 0);
      const int sparity = warp == kWarpS0 ? 0 : 1;  // S chunks issued by this warp: us % 2 == sparity
      int us = 0, uv = 0, qcount = 0;
      bool waited = false;
      for (int item = cluster_id; item < p.n_items; item += n_clusters) {
        const MlaItem it = decode_item(p, item);
        if (it.pg1 <= it.pg0) continue;
        if (!waited) {  // query images and the appended latent come from the QKV kernel
          griddep_wait();
          waited = true;
        }
        const uint8_t* kvb =
            p.kv + (static_cast<size_t>(it.sl) * p.batch + it.b) * p.page_cap * static_cast<size_t>(page_bytes);
        const int n = (it.pg1 - it.pg0 + 1) / 2;
        auto page_of = [&](int tile, int c) {
          const int pg = it.pg0 + 2 * tile + c;
          return kvb + static_cast<size_t>(pg < it.pg1 ? pg : it.pg0) * page_bytes;  // ghost: masked
        };
        if (sprod) {
          if (sparity == 0) {
            if (qcount > 0) mbar_wait(q_free, (qcount - 1) & 1);
            mbar_arrive_expect_tx(q_full, kQHalf);
            bulk_g2s(smem + kOffQ, p.qimg + static_cast<size_t>(it.b) * q_bytes + cta * kQHalf, kQHalf, q_full);
            ++qcount;
          }
          for (int tile = 0; tile < n; ++tile) {
            const int row0 = static_cast<int>((page_of(tile, static_cast<int>(cta)) - p.kv) >> 11);  // 2 KB rows
            for (int j = 0; j < kSChunks; ++j, ++us) {
              if ((us & 1) != sparity) continue;
              const int s = us % kSSlots;
              if (us >= kSSlots) mbar_wait(&empty_s[s], ((us / kSSlots) - 1) & 1);
              // both CTAs' chunks complete on the LEADER's full barrier (2-SM TMA)
              if (leader) mbar_arrive_expect_tx(&full_s[s], 2 * kSChunk);
              tma_load_2d_pair(sbase + kOffS + s * kSChunk, &tm_s, 0, row0 + j * C::kSRows, l_full_s + s * 8);
            }
          }
        } else {
          for (int tile = 0; tile < n; ++tile)
            for (int jb = 0; jb < 2; ++jb)
              for (int pp = 0; pp < 2; ++pp, ++uv) {
                const int s = uv % kVSlots;
                if (uv >= kVSlots) mbar_wait(&empty_v[s], ((uv / kVSlots) - 1) & 1);
                if (leader) mbar_arrive_expect_tx(&full_v[s], 2 * kVBlock);
                // this CTA's 128 value dims of block jb: [256 jb + 128 cta, +128), rows of CTA pp's page
                const int row0 = static_cast<int>((page_of(tile, pp) - p.kv) >> 11) + (2 * jb + static_cast<int>(cta)) * C::kVRows;
                tma_load_2d_pair(sbase + kOffV + s * kVBlock, &tm_v, 0, row0, l_full_v + s * 8);
              }
        }
      }
      if (!waited) griddep_wait();
    }
  } else if (warp == kWarpMma) {
    if (lane == 0 && !leader) {
      // ---------------------------------------------------------- peer: forward "Q half landed"
      // (latent chunks complete directly on the leader's barriers through 2-SM TMA)
      const uint32_t l_pq = mapa_shared(smem_u32(pq_full), 0);
      int qcount = 0;
      for (int item = cluster_id; item < p.n_items; item += n_clusters) {
        const MlaItem it = decode_item(p, item);
        if (it.pg1 <= it.pg0) continue;
        mbar_wait(q_full, qcount & 1);
        ++qcount;
        mbar_arrive_cluster_relaxed(l_pq);
      }
    } else if (leader) {
      // ---------------------------------------------------------- leader: MMA issue
      // order S(0) S(1) V(0) S(2) V(1) ... (a non-blocking scheduler interleaving
      // the two streams measured slower: both rings are latency-bound anyway).
      // The whole warp walks the loop and waits; one elected lane issues (a
      // lone-lane issue loop cost ~145 cycles per tcgen05.mma, tc05.cuh elect_one).
      int us = 0, uv = 0, qcount = 0, g0 = 0, items = 0;
      for (int item = cluster_id; item < p.n_items; item += n_clusters) {
        const MlaItem it = decode_item(p, item);
        if (it.pg1 <= it.pg0) continue;
        mbar_wait(q_full, qcount & 1);
        mbar_wait(pq_full, qcount & 1);
        ++qcount;
        tc_fence_after();
        const int n = (it.pg1 - it.pg0 + 1) / 2;
        for (int k = 0; k < 2 * n; ++k) {
          int tile;
          bool value;
          mla_step(k, n, tile, value);
          const int g = g0 + tile;
          if (!value) {
            // S^T(g) -> buffer g&1 (its previous reader, softmax(g-2), completed pt_full(g-2),
            // which this thread waited before issuing P.V(g-2))
            const uint32_t d = tbase + 128u * (g & 1);
            MLA_TRACE(g, 6, lane == 0);
            for (int j = 0; j < kSChunks; ++j, ++us) {
              const int s = us % kSSlots;
              mbar_wait(&full_s[s], (us / kSSlots) & 1);  // both CTAs' chunks (2-SM TMA)
              tc_fence_after();
              // A: the chunk's dim groups (2 KB apart) x 8-token groups (128 B); B: the
              // query image's dim groups (1 KB apart) x 8-head groups; 2 dim groups per MMA
              const uint64_t a0 = umma_desc(sbase + kOffS + s * kSChunk, 2048, 128);
              const uint64_t b0 = umma_desc(sbase + kOffQ + j * C::kSRows * 1024, 1024, 128);
              if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < C::kSMmas; ++kk) {
                  const uint64_t a = a0 + static_cast<uint64_t>((kk * 4096) >> 4);
                  const uint64_t b = b0 + static_cast<uint64_t>((kk * 2048) >> 4);
                  if constexpr (F8)
                    umma_ss_pair_f8(d, a, b, C::kIdescST, (j | kk) != 0);
                  else
                    umma_ss_pair(d, a, b, C::kIdescST, (j | kk) != 0);
                }
                umma_commit_pair(&empty_s[s]);
              }
              __syncwarp();
            }
            MLA_TRACE(g, 7, lane == 0);
            if (elect_one()) {
              if (tile == n - 1) umma_commit_pair(q_free);
              umma_commit_pair(&s_full[g & 1]);
            }
            __syncwarp();
          } else {
            mbar_wait(&pt_full[g % NPT], (g / NPT) & 1);
            MLA_TRACE(g, 8, lane == 0);
            if (tile == 0 && items > 0) mbar_wait_cluster(o_free, (items - 1) & 1);
            fence_proxy_async();
            tc_fence_after();
            for (int jb = 0; jb < 2; ++jb)
              for (int pp = 0; pp < 2; ++pp, ++uv) {
                const int s = uv % kVSlots;
                mbar_wait(&full_v[s], (uv / kVSlots) & 1);  // both CTAs' blocks (2-SM TMA)
                tc_fence_after();
                // MN-major both: A = V^T (8-token groups 128 B apart along K, dim
                // groups 2 KB apart along M), B = P^T (8-token groups kPTLbo apart,
                // head groups 128 B apart along N)
                const uint64_t a0 = umma_desc(sbase + kOffV + s * kVBlock, 128, 2048);
                const uint64_t b0 = umma_desc(sbase + kOffPT + (g % NPT) * C::kPT + pp * C::kPTPage, C::kPTLbo, 128);
                const bool acc0 = tile > 0 || pp > 0;
                if (elect_one()) {
#pragma unroll
                  for (int kk = 0; kk < C::kPVMmas; ++kk) {
                    const uint64_t a = a0 + static_cast<uint64_t>((kk * C::kPVAStep) >> 4);
                    const uint64_t b = b0 + static_cast<uint64_t>((kk * 2048) >> 4);
                    if constexpr (F8)
                      umma_ss_pair_f8(tbase + 256 + 128 * jb, a, b, C::kIdescOT, (acc0 || kk > 0) ? 1u : 0u);
                    else
                      umma_ss_pair(tbase + 256 + 128 * jb, a, b, C::kIdescOT, (acc0 || kk > 0) ? 1u : 0u);
                  }
                  umma_commit_pair(&empty_v[s]);
                }
                __syncwarp();
              }
            MLA_TRACE(g, 9, lane == 0);
            if (elect_one()) umma_commit_pair(&pv_done[g % NPT]);
            __syncwarp();
          }
        }
        g0 += n;
        ++items;
      }
    }
  } else {
    // ------------------------------------------------------------ softmax / correction (warps 0 .. SW - 1)
    const int wg = warp >> 2, wq = warp & 3;
    const int t = wq * 32 + lane;  // token lane of S^T, dim lane of O^T
    const int hbase = HPW * wg;    // this warpgroup's heads
    const int wg_bar = 1 + wg;     // named barrier of the warpgroup
    const uint32_t lrow = tbase + (static_cast<uint32_t>(wq * 32) << 16);
    const uint32_t peer_min = mapa_shared(sbase + kOffMin, peer), peer_zin = mapa_shared(sbase + kOffZin, peer);
    const uint32_t peer_mx = mapa_shared(smem_u32(mx_bar), peer), peer_zx = mapa_shared(smem_u32(zx_bar), peer);
    const uint32_t peer_fl = mapa_shared(sbase + C::kOffFl, peer), peer_flbar = mapa_shared(smem_u32(fl_bar), peer);
    const float* fl_in = reinterpret_cast<const float*>(smem + C::kOffFl);
    int fcnt = 0, ecnt = 0;  // flag exchanges / maxima exchanges so far (the same sequence in both CTAs)
    const uint32_t peer_pt0 = mapa_shared(sbase + kOffPT, peer), peer_ptfull0 = mapa_shared(smem_u32(pt_full), peer);
    const uint32_t l_ptfull0 = mapa_shared(smem_u32(pt_full), 0), l_ofree = mapa_shared(smem_u32(o_free), 0);
    const bool pt_remote = (hbase >> 6) != static_cast<int>(cta);  // P^T of heads [64k, 64k + 64) lives in CTA k
    const int hl0 = hbase & 63;                                      // first head within that P^T
    const int h_own = hbase + t;  // head owned for max/sum bookkeeping (t < HPW)
    if constexpr (F8) griddep_wait();  // the query images' head scales are read from global below
    int g = 0, items = 0;
    for (int item = cluster_id; item < p.n_items; item += n_clusters) {
      const MlaItem it = decode_item(p, item);
      if (it.pg1 <= it.pg0) {  // empty split: zero fragment rows, LSE -inf
        for (int jb = 0; jb < 2; ++jb) {
          const int dim = 256 * jb + 128 * static_cast<int>(cta) + t;
          for (int h = hbase; h < hbase + HPW && h < p.q_heads; ++h)
            p.part_o[(static_cast<size_t>(item) * kMlaHeads + h) * kMlaDV + dim] = 0.f;
        }
        if (leader && t < HPW && h_own < p.q_heads) p.part_lse2[static_cast<size_t>(item) * kMlaHeads + h_own] = -INFINITY;
        continue;
      }
      float z[HPW];
#pragma unroll
      for (int h = 0; h < HPW; ++h) z[h] = 0.f;
      float m_run = -INFINITY;  // reference max of head h_own (log2 units), threads t < HPW
      if constexpr (F8) {  // per-head score scale: qscale x the query image's 2^-e_h (published by the barriers below)
        if (t < HPW)
          cs[h_own] = p.qscale * reinterpret_cast<const float*>(p.qimg + static_cast<size_t>(it.b) * q_bytes +
                                                                kMlaW * kMlaHeads)[h_own];
      }
      const int n = (it.pg1 - it.pg0 + 1) / 2;
      for (int tile = 0; tile < n; ++tile, ++g) {
        const int buf = g & 1;
        const int pg = it.pg0 + 2 * tile + static_cast<int>(cta);
        const int valid = pg < it.pg1 ? min(kMlaPageRows, it.ntok - pg * kMlaPageRows) : 0;
        const bool mine = t < valid;
        const uint32_t srow = lrow + 128u * buf + hbase;
        mbar_wait(&s_full[buf], (g >> 1) & 1);
        tc_fence_after();
        MLA_TRACE(g, 0, threadIdx.x == 0);
        // ---- does any head's column maximum (over the pair's 256 tokens) exceed its
        // reference max by more than 2^8? Only then (and at an item's first tile, where
        // the references start at -inf) are the exact column maxima needed: the lazy
        // rescale leaves every reference unchanged otherwise, so skipping them when no
        // score is that large gives the same m_use as computing them.
        bool exact = tile == 0;
        if (!exact) {
          float dmax = -INFINITY;
#pragma unroll
          for (int j = 0; j < HPW / 32; ++j) {
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              float v[16];
              tmem_ld16(srow + 32 * j + 16 * hh, v);
#pragma unroll
              for (int q4 = 0; q4 < 4; ++q4) {
                const int hl = 32 * j + 16 * hh + 4 * q4;
                const float4 mm = *reinterpret_cast<const float4*>(m_use + hbase + hl);
                float4 cc;
                if constexpr (F8)
                  cc = *reinterpret_cast<const float4*>(cs + hbase + hl);
                else
                  cc = make_float4(p.qscale, p.qscale, p.qscale, p.qscale);
                dmax = fmaxf(dmax, fmaxf(fmaxf(fmaf(v[4 * q4], cc.x, -mm.x), fmaf(v[4 * q4 + 1], cc.y, -mm.y)),
                                         fmaxf(fmaf(v[4 * q4 + 2], cc.z, -mm.z), fmaf(v[4 * q4 + 3], cc.w, -mm.w))));
              }
            }
          }
          const bool any_local = bar_red_or(kBarAll, 128 * NWG, mine && dmax > 8.f);
          const int f = fcnt & 1;
          if (threadIdx.x == 0) {
            mbar_arrive_expect_tx(&fl_bar[f], 4);
            st_async_f32(peer_fl + f * 4, any_local ? 1.f : 0.f, peer_flbar + f * 8);
          }
          mbar_wait(&fl_bar[f], (fcnt >> 1) & 1);
          exact = any_local || fl_in[f] != 0.f;
          ++fcnt;
          MLA_TRACE(g, 10, threadIdx.x == 0);
        }
        bool any = false, pv_waited = false;
        if (exact) {
        const int e = ecnt & 1;
        if (threadIdx.x == 0) mbar_arrive_expect_tx(&mx_bar[e], 128 * 4);  // the peer's maxima
        // ---- column (per-head) maxima over this CTA's 128 tokens, this warpgroup's HPW heads
#pragma unroll 1
        for (int j = 0; j < HPW / 32; ++j) {
          float keep = -INFINITY;
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {  // 16 columns per TMEM load (register budget of NWG = 4)
            float v[16];
            tmem_ld16(srow + 32 * j + 16 * hh, v);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float r = redux_max_f32(mine ? v[i] : -INFINITY);
              if (lane == 16 * hh + i) keep = r;
            }
          }
          red[warp * HPW + 32 * j + lane] = keep;
        }
        MLA_TRACE(g, 1, threadIdx.x == 0);
        named_bar(wg_bar, 128);
        bool grow = false;
        if (t < HPW) {
          float mc = fmaxf(fmaxf(red[(4 * wg) * HPW + t], red[(4 * wg + 1) * HPW + t]),
                           fmaxf(red[(4 * wg + 2) * HPW + t], red[(4 * wg + 3) * HPW + t]));
          mc *= F8 ? cs[h_own] : p.qscale;
          st_async_f32(peer_min + (e * 128 + h_own) * 4, mc, peer_mx + e * 8);
          mbar_wait(&mx_bar[e], (ecnt >> 1) & 1);
          MLA_TRACE(g, 2, threadIdx.x == 0);
          const float mt = fmaxf(mc, m_in[e * 128 + h_own]);
          grow = mt > m_run + 8.f;  // lazy: keep the reference max within 2^8
          const float m_new = grow ? mt : m_run;
          alpha_s[h_own] = grow ? exp2f(m_run - m_new) : 1.f;
          m_use[h_own] = m_new;
          m_run = m_new;
        }
        any = bar_red_or(kBarAll, 128 * NWG, grow);  // also publishes m_use / alpha_s
        ++ecnt;
        }
        MLA_TRACE(g, 3, threadIdx.x == 0);
        if (any) {
#pragma unroll
          for (int h = 0; h < HPW; ++h) z[h] *= alpha_s[hbase + h];
          if (tile > 0) {  // O^T holds tiles < tile: wait for P.V(g-1), rescale this warpgroup's head columns
            mbar_wait(&pv_done[(g - 1) % NPT], ((g - 1) / NPT) & 1);
            tc_fence_after();
            pv_waited = true;
#pragma unroll 1
            for (int c = 0; c < 2 * (HPW / 32); ++c) {
              const int jb = c / (HPW / 32), cc = c % (HPW / 32);
              const uint32_t col = 256 + 128 * jb + hbase + 32 * cc;
              float v[32];
              tmem_ld32(lrow + col, v);
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] *= alpha_s[hbase + 32 * cc + i];
              tmem_st32(lrow + col, v);
            }
            tmem_wait_st();
          }
        }
        // this tile's P^T buffer is free once P.V(g - NPT) completed (earlier items: waited at their end)
        if (tile >= NPT && !pv_waited) mbar_wait(&pv_done[g % NPT], ((g - NPT) / NPT) & 1);
        MLA_TRACE(g, 4, threadIdx.x == 0);
        const uint32_t pt_local = sbase + kOffPT + (g % NPT) * C::kPT;
        const uint32_t peer_pt = peer_pt0 + (g % NPT) * C::kPT, peer_ptfull = peer_ptfull0 + (g % NPT) * 8;
        // ---- P for this token, this warpgroup's HPW heads -> P^T of CTA hbase / 64 (local or st.async)
        const int k = 128 * static_cast<int>(cta) + t;
        if constexpr (F8) {
          // e4m3 P^T [tg 32][16-head group 4][token%8][16 heads]; the head sums keep
          // the unrounded fp32 p (RNE errors are unbiased; the tolerance covers them)
          const uint32_t rowoff = static_cast<uint32_t>(k >> 3) * 512 + (k & 7) * 16;
#pragma unroll
          for (int j = 0; j < HPW / 32; ++j) {
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              float v[16];
              tmem_ld16(srow + 32 * j + 16 * q, v);
              uint32_t w4[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int hl = 32 * j + 16 * q + 4 * e;  // head index within the warpgroup
                const float4 mm = *reinterpret_cast<const float4*>(m_use + hbase + hl);
                const float4 cc = *reinterpret_cast<const float4*>(cs + hbase + hl);
                const float* vv = v + 4 * e;
                const float p0 = mine ? ex2_approx(fmaf(vv[0], cc.x, -mm.x)) : 0.f;
                const float p1 = mine ? ex2_approx(fmaf(vv[1], cc.y, -mm.y)) : 0.f;
                const float p2 = mine ? ex2_approx(fmaf(vv[2], cc.z, -mm.z)) : 0.f;
                const float p3 = mine ? ex2_approx(fmaf(vv[3], cc.w, -mm.w)) : 0.f;
                z[hl] += p0;
                z[hl + 1] += p1;
                z[hl + 2] += p2;
                z[hl + 3] += p3;
                w4[e] = pack_e4m3x4(p0, p1, p2, p3);
              }
              const uint32_t off = rowoff + static_cast<uint32_t>((hl0 >> 4) + 2 * j + q) * 128;
              const uint4 val = make_uint4(w4[0], w4[1], w4[2], w4[3]);
              if (pt_remote)
                st_async_v4(peer_pt + off, val, peer_ptfull);
              else
                sts128(pt_local + off, val);
            }
          }
        } else {
          const uint32_t rowoff = (static_cast<uint32_t>(k >> 3) * 64 + (k & 7)) * 16;
#pragma unroll
          for (int j = 0; j < HPW / 32; ++j) {
#pragma unroll
            for (int qq = 0; qq < 2; ++qq) {
              float v[16];  // 16 columns per TMEM load (register budget of NWG = 4)
              tmem_ld16(srow + 32 * j + 16 * qq, v);
#pragma unroll
              for (int q2 = 0; q2 < 2; ++q2) {
                const int q = 2 * qq + q2;
                const float4 ma = *reinterpret_cast<const float4*>(m_use + hbase + 32 * j + 8 * q);
                const float4 mb = *reinterpret_cast<const float4*>(m_use + hbase + 32 * j + 8 * q + 4);
                const float mm[8] = {ma.x, ma.y, ma.z, ma.w, mb.x, mb.y, mb.z, mb.w};
                uint32_t w4[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const int hl = 32 * j + 8 * q + 2 * e;  // head index within the warpgroup
                  const float p0 = mine ? ex2_approx(fmaf(v[8 * q2 + 2 * e], p.qscale, -mm[2 * e])) : 0.f;
                  const float p1 = mine ? ex2_approx(fmaf(v[8 * q2 + 2 * e + 1], p.qscale, -mm[2 * e + 1])) : 0.f;
                  const __nv_bfloat162 pb = __floats2bfloat162_rn(p0, p1);
                  z[hl] += __low2float(pb);
                  z[hl + 1] += __high2float(pb);
                  w4[e] = *reinterpret_cast<const uint32_t*>(&pb);
                }
                // P^T core (token row k, heads 8-group (hl0 / 8 + 4j + q) of this CTA's 64)
                const uint32_t off = rowoff + static_cast<uint32_t>((hl0 >> 3) + 4 * j + q) * 128;
                const uint4 val = make_uint4(w4[0], w4[1], w4[2], w4[3]);
                if (pt_remote)
                  st_async_v4(peer_pt + off, val, peer_ptfull);
                else
                  sts128(pt_local + off, val);
              }
            }
          }
        }
        fence_proxy_async();
        tc_fence_before();
        if (threadIdx.x == 0)
          mbar_arrive_expect_tx(&pt_full[g % NPT], 128 * 64 * (F8 ? 1 : 2));  // + the peer warpgroup's st.async into this P^T
        else
          mbar_arrive(&pt_full[g % NPT]);
        if (!leader && threadIdx.x == 0) {  // forward "peer P^T complete" to the leader's MMA issuer
          mbar_wait(&pt_full[g % NPT], (g / NPT) & 1);
          fence_proxy_async();
          mbar_arrive_cluster_relaxed(l_ptfull0 + (g % NPT) * 8);
        }
      }
      // ---- item done: head sums over the pair, then O^T / z
      mbar_wait(&pv_done[(g - 1) % NPT], ((g - 1) / NPT) & 1);
      tc_fence_after();
      // transpose-reduce the HPW per-head partials across the warp: lane ends with heads [hb, hb + HPW / 32)
      int hb = 0;
#pragma unroll
      for (int o = 16, cnt = HPW / 2; o >= 1; o >>= 1, cnt >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < cnt; ++i) {
          const float send = up ? z[i] : z[i + cnt];
          const float keep = up ? z[i + cnt] : z[i];
          z[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
        if (up) hb += cnt;
      }
      named_bar(wg_bar, 128);  // red[] free (last tile's maxima consumed)
#pragma unroll
      for (int i = 0; i < HPW / 32; ++i) red[warp * HPW + hb + i] = z[i];
      named_bar(wg_bar, 128);
      const int zb = items & 1;
      float zc = 0.f;
      if (t < HPW) {
        zc = (red[(4 * wg) * HPW + t] + red[(4 * wg + 1) * HPW + t]) +
             (red[(4 * wg + 2) * HPW + t] + red[(4 * wg + 3) * HPW + t]);
        st_cluster_f32(peer_zin + (zb * 128 + h_own) * 4, zc);
        mbar_arrive_cluster(peer_zx + zb * 8);
        mbar_wait_cluster(&zx_bar[zb], (items >> 1) & 1);
        const float ztot = leader ? zc + z_in[zb * 128 + h_own] : z_in[zb * 128 + h_own] + zc;  // CTA 0's sum first
        zs[h_own] = ztot > 0.f ? 1.f / ztot : 0.f;
        if (leader && h_own < p.q_heads)
          p.part_lse2[static_cast<size_t>(item) * kMlaHeads + h_own] = ztot > 0.f ? m_run + log2f(ztot) : -INFINITY;
      }
      named_bar(kBarAll, 128 * NWG);
#pragma unroll 1
      for (int c = 0; c < 2 * (HPW / 32); ++c) {
        const int jb = c / (HPW / 32), hc = hbase + 32 * (c % (HPW / 32));
        const int dim = 256 * jb + 128 * static_cast<int>(cta) + t;
        float v[32];
        tmem_ld32(lrow + 256 + 128 * jb + hc, v);
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int h = hc + i;
          if (h < p.q_heads) p.part_o[(static_cast<size_t>(item) * kMlaHeads + h) * kMlaDV + dim] = v[i] * zs[h];
        }
      }
      tc_fence_before();
      mbar_arrive_cluster(l_ofree);
      ++items;
    }
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (warp == kWarpMma) tmem_dealloc_pair(tbase, 512);
#ifdef HX_MLA_TRACE
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const unsigned long long t0 = g_mla_trace[8][0];
    for (int i = 8; i < 24; ++i)
      printf("tile %2d  sm: sfull %6lld flag %6lld max %6lld mx %6lld vote %6lld pbuf %6lld pdone %6lld | mma: S %6lld-%6lld ptfull %6lld pv %6lld\n",
             i, (long long)(g_mla_trace[i][0] - t0), (long long)(g_mla_trace[i][10] - t0), (long long)(g_mla_trace[i][1] - t0), (long long)(g_mla_trace[i][2] - t0),
             (long long)(g_mla_trace[i][3] - t0), (long long)(g_mla_trace[i][4] - t0), (long long)(g_mla_trace[i][5] - t0),
             (long long)(g_mla_trace[i][6] - t0), (long long)(g_mla_trace[i][7] - t0), (long long)(g_mla_trace[i][8] - t0),
             (long long)(g_mla_trace[i][9] - t0));
  }
#endif
}

// Merge a stream's split partials (split order, deterministic) into the
// rank's fragment [slot][b][head][512] + natural-log lse (HeadFragment).
// One CTA per (stream, head): warp w merges splits w, w+8, ... in order (all its
// loads issued together), the 8 warp partials are combined in warp order
// (deterministic). part_o of a launch (<= 19 MB at the C4 shard) is L2-resident.
__global__ void __launch_bounds__(256) mla_split_reduce_kernel(const AttnParams p, float* frag_o, float* frag_lse) {
  griddep_wait();
  griddep_launch_dependents();
  __shared__ float s_m[8], s_l[8];
  __shared__ float s_o[8][kMlaDV];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = blockIdx.x % p.q_heads, stream = blockIdx.x / p.q_heads;
  const int bl = stream % p.stream_batch, sl = stream / p.stream_batch, b = bl + p.b_begin;
  const int rank = (sl + p.slot_base) % p.kvp;
  const int ntok = static_cast<int>(rr_count(p.total[b], rank, p.chunk, p.kvp));
  const int pages = (ntok + kMlaPageRows - 1) / kMlaPageRows;
  auto valid = [&](int s) {
    const int pg0 = static_cast<int>((static_cast<long long>(s) * pages) / p.splits);
    const int pg1 = static_cast<int>((static_cast<long long>(s + 1) * pages) / p.splits);
    return pg1 > pg0;
  };
  float M = -INFINITY;
  for (int s = warp * 32 + lane; s < p.splits; s += 256)
    if (valid(s)) M = fmaxf(M, p.part_lse2[static_cast<size_t>(s * p.n_streams + stream) * kMlaHeads + h]);
#pragma unroll
  for (int o2 = 16; o2 > 0; o2 >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o2));
  if (lane == 0) s_m[warp] = M;
  __syncthreads();
  M = s_m[0];
#pragma unroll
  for (int w = 1; w < 8; ++w) M = fmaxf(M, s_m[w]);
  float o[16] = {};
  float L = 0.f;
  for (int s0 = warp; s0 < p.splits; s0 += 16) {
    float w2[2], v[2][16];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int s = s0 + 8 * j;
      const bool ok = s < p.splits && valid(s);
      const size_t item = static_cast<size_t>(s * p.n_streams + stream);
      w2[j] = ok ? p.part_lse2[item * kMlaHeads + h] : -INFINITY;
#pragma unroll
      for (int i = 0; i < 16; ++i) v[j][i] = ok ? p.part_o[(item * kMlaHeads + h) * kMlaDV + lane + 32 * i] : 0.f;
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const float e = w2[j] == -INFINITY ? 0.f : exp2f(w2[j] - M);
      L += e;
#pragma unroll
      for (int i = 0; i < 16; ++i) o[i] += e * v[j][i];
    }
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) s_o[warp][lane + 32 * i] = o[i];
  if (lane == 0) s_l[warp] = L;
  __syncthreads();
  // all 8 warps write: warp w finalises dims [64w, 64w + 64)
  float Lt = 0.f;
#pragma unroll
  for (int w = 0; w < 8; ++w) Lt += s_l[w];
  const size_t fo = (static_cast<size_t>(sl) * p.batch + b) * p.q_per_slot + h;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int d = warp * 64 + lane + 32 * i;
    float ot = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) ot += s_o[w][d];
    frag_o[fo * kMlaDV + d] = Lt > 0.f ? ot / Lt : 0.f;
  }
  if (threadIdx.x == 0) frag_lse[fo] = Lt > 0.f ? (M + log2f(Lt)) * 0.69314718055994530942f : -INFINITY;
}

template <bool F8, int NWG>
static cudaError_t launch_mla_t(const AttnParams& p, int grid, cudaStream_t stream, const void* tm_s, const void* tm_v) {
  constexpr uint32_t kSmem = MlaCfg<F8>::kSmem;
  {
    const cudaError_t e = smem_optin<mla_decode_kernel<F8, NWG>>(kSmem);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(2 * grid));  // grid = number of CTA pairs
  cfg.blockDim = dim3(mla_threads(NWG));
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, mla_decode_kernel<F8, NWG>, p, *static_cast<const CUtensorMap*>(tm_s),
                            *static_cast<const CUtensorMap*>(tm_v));
}

cudaError_t launch_mla_decode(const AttnParams& p, int grid, cudaStream_t stream, const void* tm_s, const void* tm_v) {
  if (p.q_heads > kMlaHeads || p.q_heads < 1) return cudaErrorInvalidValue;
  // two softmax warpgroups of 64 heads (NWG = 4, 32 heads each, measured 10-20% slower:
  // 20 warps cap registers at 96 and spill the per-head sums)
  return p.kv8 ? launch_mla_t<true, 2>(p, grid, stream, tm_s, tm_v) : launch_mla_t<false, 2>(p, grid, stream, tm_s, tm_v);
}

cudaError_t make_mla_tensor_maps(const void* pool, size_t bytes, void* tm_s, void* tm_v, bool f8) {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || !fn) return e != cudaSuccess ? e : cudaErrorNotSupported;
    encode = reinterpret_cast<EncodeFn>(fn);
  }
  if (bytes % 2048) return cudaErrorInvalidValue;
  const cuuint64_t dims[2] = {256, bytes / 2048};  // u64 elements per 2 KB row, rows
  const cuuint64_t strides[1] = {2048};
  const cuuint32_t estr[2] = {1, 1};
  const cuuint32_t box_s[2] = {256, f8 ? 12u : 8u}, box_v[2] = {256, f8 ? 8u : 16u};
  CUresult r = encode(static_cast<CUtensorMap*>(tm_s), CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<void*>(pool), dims,
                      strides, box_s, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  r = encode(static_cast<CUtensorMap*>(tm_v), CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<void*>(pool), dims, strides,
             box_v, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t launch_mla_split_reduce(const AttnParams& p, float* frag_o, float* frag_lse, cudaStream_t stream) {
  const long long ctas = static_cast<long long>(p.n_streams) * p.q_heads;  // one per (stream, head)
  return launch_k(mla_split_reduce_kernel, dim3(static_cast<unsigned>(ctas)), dim3(256), 0, stream, p, frag_o,
                  frag_lse);
}

// ---------------------------------------------------------------------------
// Hash fill of the latent cache (layer_oracle.hpp MLA): element d of global
// token g of request b = hash_unit(seed, stream_k, ((b << 32) + g) * W + d).
// One thread per 16-byte core-matrix row (8 dims of one local row); rows
// outside the appended range keep their contents.
__device__ __forceinline__ long long mla_rr_global(long long row, int rank, int chunk, int kvp) {
  return (row / chunk) * static_cast<long long>(chunk) * kvp + static_cast<long long>(rank) * chunk + row % chunk;
}

__global__ void kv_fill_hash_mla_kernel(uint8_t* kv, const int* total, int batch, int kvp, int chunk, int page_cap,
                                        int slot_base, int n_local_slots, long long n, uint64_t seed,
                                        uint64_t stream_k, bool f8) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int dims = f8 ? 16 : 8;  // latent dims per 16-byte row
  const int kRowsPerPage = kMlaPageRows * (kMlaW / dims);  // 16-byte rows per page
  const long long per_stream = static_cast<long long>(page_cap) * kRowsPerPage;
  if (idx >= static_cast<long long>(n_local_slots) * batch * per_stream) return;
  const long long st = idx / per_stream;  // slot_local * B + b
  const long long rem = idx - st * per_stream;
  const int page = static_cast<int>(rem / kRowsPerPage);
  const int ci = static_cast<int>(rem % kRowsPerPage);  // (dg * 16 + tg) * 8 + r8
  const int r8 = ci & 7, tg = (ci >> 3) & 15, dg = ci >> 7;
  const int b = static_cast<int>(st % batch);
  const int rank = (static_cast<int>(st / batch) + slot_base) % kvp;
  const long long row = static_cast<long long>(page) * kMlaPageRows + tg * 8 + r8;
  const long long g = mla_rr_global(row, rank, chunk, kvp);
  const long long t0 = total[b];
  if (g < t0 || g >= t0 + n) return;
  const uint64_t kseed = splitmix64(seed ^ (stream_k * 0xD1B54A32D192ED03ull));
  const uint64_t base = ((static_cast<uint64_t>(b) << 32) + static_cast<uint64_t>(g)) * kMlaW + dg * dims;
  uint8_t* pg = kv + (static_cast<size_t>(st) * page_cap + page) * static_cast<size_t>(mla_page_bytes(f8));
  if (f8) {  // the double draw rounded straight to e4m3 (oracle: round_e4m3 of the same draw)
    uint8_t c[16];
#pragma unroll
    for (int e = 0; e < 16; ++e)
      c[e] = e4m3_from_double(2.0 * (static_cast<double>(splitmix64(kseed + base + e) >> 11) * 0x1.0p-53) - 1.0);
    *reinterpret_cast<uint4*>(pg + static_cast<size_t>(ci) * 16) = *reinterpret_cast<const uint4*>(c);
    return;
  }
  uint32_t w[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    uint16_t lo, hi;
    {
      const uint64_t z = splitmix64(kseed + base + 2 * e);
      const __nv_bfloat16 v = double_to_bf16_rne(2.0 * (static_cast<double>(z >> 11) * 0x1.0p-53) - 1.0);
      lo = *reinterpret_cast<const uint16_t*>(&v);
    }
    {
      const uint64_t z = splitmix64(kseed + base + 2 * e + 1);
      const __nv_bfloat16 v = double_to_bf16_rne(2.0 * (static_cast<double>(z >> 11) * 0x1.0p-53) - 1.0);
      hi = *reinterpret_cast<const uint16_t*>(&v);
    }
    w[e] = static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
  }
  *reinterpret_cast<uint4*>(pg + static_cast<size_t>(ci) * 16) = make_uint4(w[0], w[1], w[2], w[3]);
}

__global__ void add_total_mla_kernel(int* total, int batch, int n) {
  for (int b = threadIdx.x; b < batch; b += blockDim.x) total[b] += n;
}

cudaError_t launch_kv_fill_hash_mla(uint8_t* kv, int* total, int batch, int kvp, int chunk, int page_cap,
                                    int slot_base, int n_local_slots, long long n, uint64_t seed, uint64_t stream_k,
                                    cudaStream_t stream, bool f8) {
  const long long work = static_cast<long long>(n_local_slots) * batch * page_cap * kMlaPageRows * (kMlaW / (f8 ? 16 : 8));
  if (n > 0)
    kv_fill_hash_mla_kernel<<<static_cast<unsigned>((work + 255) / 256), 256, 0, stream>>>(
        kv, total, batch, kvp, chunk, page_cap, slot_base, n_local_slots, n, seed, stream_k, f8);
  add_total_mla_kernel<<<1, 64, 0, stream>>>(total, batch, static_cast<int>(n));
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Decode-time weight absorption around the latent attention (layer_oracle.hpp):
// the QKV GEMV streams the reference-shaped W_q [H x Q*Hsz] (roofline.hpp:17-48),
// these two small per-head products turn its output into the 576-wide latent
// query and the 512-wide latent attention output back into head_size values.

// One per-head product out[b][h][j] = sum_d in[b][h][d] * W[h][d][j] (d < din,
// j < dout), used twice:
//   ABSORB: in = n [B][Q][dp] (QKV epilogue), W = W_UK [Q][hs][576], out -> bf16 q image;
//   UV:     in = att [B][nh*512] (merged latent output), W = W_UV [nh][512][hs],
//           out -> x-fragments of v [B][nh*hs] (the O-projection's K operand).
// Grid (head, column chunk); thread = (8-column group, d-slice): one 16-byte
// weight load per d feeds 8 requests x 8 columns of FMAs, eight loads in flight
// per thread; the DS d-slice partials are summed in slice order (deterministic).
// Requests in passes of 8, staged in shared memory as [d][8].
// Q8 (ABSORB for FP8 latents, one CTA per head): the head's 576 values of each
// request are scaled by 2^e_h, the largest power of two keeping max |q_h| <= 448,
// and stored as e4m3 with 2^-e_h beside the image (mla_q_offset8).
template <bool ABSORB, int DS, bool Q8 = false>
__global__ void __launch_bounds__(512) mla_head_gemm_kernel(const float* in, int in_head_stride, int in_row_stride,
                                                             const __nv_bfloat16* w, int din, int dout, int batch,
                                                             uint8_t* out, int xf16) {
  constexpr int NB = 8;
  extern __shared__ __align__(16) float hsm[];
  float* s_in = hsm;                    // [din][NB]
  const int cols = dout / gridDim.y, c0 = blockIdx.y * cols;
  float* red = hsm + din * NB;          // [DS][NB][cols]
  const int h = blockIdx.x;
  const int groups = cols / 8;
  const int cg = threadIdx.x % groups, ds = threadIdx.x / groups;
  const int dper = din / DS, d0 = ds * dper;
  const __nv_bfloat16* wh = w + static_cast<size_t>(h) * din * dout + c0 + cg * 8;
  griddep_wait();
  griddep_launch_dependents();
  for (int bc = 0; bc < batch; bc += NB) {
    const int nb = min(NB, batch - bc);
    // stage the inputs: 8 independent loads per thread in flight before any store
    for (int i0 = threadIdx.x; i0 < NB * din; i0 += 8 * blockDim.x) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * blockDim.x;
        const int b = i / din, d = i - b * din;
        v[u] = (i < NB * din && b < nb)
                   ? in[static_cast<size_t>(bc + b) * in_row_stride + static_cast<size_t>(h) * in_head_stride + d]
                   : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * blockDim.x;
        if (i < NB * din) s_in[(i % din) * NB + i / din] = v[u];
      }
    }
    __syncthreads();
    if (ds < DS) {
      float acc[NB][8];
#pragma unroll
      for (int b = 0; b < NB; ++b)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[b][c] = 0.f;
      for (int dc = d0; dc < d0 + dper; dc += 8) {
        uint4 wv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          wv[u] = dc + u < d0 + dper ? __ldg(reinterpret_cast<const uint4*>(wh + static_cast<size_t>(dc + u) * dout))
                                     : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (dc + u >= d0 + dper) break;
          float wf[8];
          const __nv_bfloat162* w2 = reinterpret_cast<const __nv_bfloat162*>(&wv[u]);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            wf[2 * c] = __low2float(w2[c]);
            wf[2 * c + 1] = __high2float(w2[c]);
          }
          const float4* x4 = reinterpret_cast<const float4*>(s_in + (dc + u) * NB);
#pragma unroll
          for (int b4 = 0; b4 < NB / 4; ++b4) {
            const float4 x = x4[b4];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              acc[4 * b4 + 0][c] += x.x * wf[c];
              acc[4 * b4 + 1][c] += x.y * wf[c];
              acc[4 * b4 + 2][c] += x.z * wf[c];
              acc[4 * b4 + 3][c] += x.w * wf[c];
            }
          }
        }
      }
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        float4* r4 = reinterpret_cast<float4*>(red + (static_cast<size_t>(ds) * NB + b) * cols + cg * 8);
        r4[0] = make_float4(acc[b][0], acc[b][1], acc[b][2], acc[b][3]);
        r4[1] = make_float4(acc[b][4], acc[b][5], acc[b][6], acc[b][7]);
      }
    }
    __syncthreads();
    if constexpr (Q8) {
      __shared__ float s_scale[NB];
      for (int e = threadIdx.x; e < nb * cols; e += blockDim.x) {  // sums in place (slice 0 of each element)
        const int b = e / cols, jc = e - b * cols;
        float v = 0.f;
#pragma unroll
        for (int s = 0; s < DS; ++s) v += red[(s * NB + b) * cols + jc];
        red[b * cols + jc] = v;
      }
      __syncthreads();
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      if (warp < nb) {
        float mx = 0.f;
        for (int jc = lane; jc < cols; jc += 32) mx = fmaxf(mx, fabsf(red[warp * cols + jc]));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        int ex = 0;
        if (mx > 0.f) {
          ex = static_cast<int>(floorf(log2f(448.f / mx)));
          while (ex > -120 && ldexpf(mx, ex) > 448.f) --ex;
          while (ex < 120 && ldexpf(mx, ex + 1) <= 448.f) ++ex;
        }
        if (lane == 0) {
          s_scale[warp] = ldexpf(1.f, ex);
          reinterpret_cast<float*>(out + static_cast<size_t>(bc + warp) * mla_q_bytes(true) + kMlaW * kMlaHeads)[h] =
              ldexpf(1.f, -ex);
        }
      }
      __syncthreads();
      for (int e = threadIdx.x; e < nb * cols; e += blockDim.x) {
        const int b = e / cols, jc = e - b * cols;
        out[static_cast<size_t>(bc + b) * mla_q_bytes(true) + mla_q_offset8(h, c0 + jc)] =
            e4m3_from_double(static_cast<double>(red[b * cols + jc] * s_scale[b]));
      }
    } else {
      for (int e = threadIdx.x; e < nb * cols; e += blockDim.x) {
        const int b = e / cols, jc = e - b * cols, jj = c0 + jc;
        float v = 0.f;
#pragma unroll
        for (int s = 0; s < DS; ++s) v += red[(s * NB + b) * cols + jc];
        if (ABSORB)
          *reinterpret_cast<__nv_bfloat16*>(out + static_cast<size_t>(bc + b) * mla_q_bytes() + mla_q_offset(h, jj)) =
              __float2bfloat16_rn(v);
        else
          xf_write(out, xf_nb8(batch), bc + b, h * dout + jj, v, xf16);
      }
    }
    __syncthreads();
  }
}

template <bool ABSORB, int DS, bool Q8 = false>
static cudaError_t launch_head_gemm_t(const float* in, int in_head_stride, int in_row_stride, const uint16_t* w,
                                      int din, int dout, int batch, int heads, int col_chunks, uint8_t* out,
                                      cudaStream_t stream, int xf16 = 0) {
  while (col_chunks > 1 && dout % (8 * col_chunks)) --col_chunks;
  const int cols = dout / col_chunks;
  if (cols % 8 || din % DS || (cols / 8) * DS > 512) return cudaErrorInvalidValue;
  const size_t smem = (static_cast<size_t>(din) * 8 + static_cast<size_t>(DS) * 8 * cols) * sizeof(float);
  {
    const cudaError_t e = smem_optin<mla_head_gemm_kernel<ABSORB, DS, Q8>>(smem);
    if (e != cudaSuccess) return e;
  }
  const int threads = (cols / 8) * DS;
  if (Q8 && (col_chunks != 1 || threads < 32 * 8)) return cudaErrorInvalidValue;  // one CTA per head, a warp per request
  return launch_k(mla_head_gemm_kernel<ABSORB, DS, Q8>, dim3(heads, col_chunks), dim3((threads + 31) / 32 * 32), smem,
                  stream, in,
                  in_head_stride, in_row_stride, reinterpret_cast<const __nv_bfloat16*>(w), din, dout, batch, out, xf16);
}

cudaError_t launch_mla_absorb_q(const float* n, const uint16_t* wuk, int batch, int q_heads, int hs, int dp,
                                uint8_t* qimg, cudaStream_t stream, bool f8) {
  if (hs > 128) return cudaErrorInvalidValue;  // 3 chunks of 24 column groups x 8 d-slices
  if (f8)  // one CTA per head (the per-head scale spans all 576 columns): 72 column groups x 4 d-slices
    return launch_head_gemm_t<true, 4, true>(n, dp, q_heads * dp, wuk, hs, kMlaW, batch, q_heads, 1, qimg, stream);
  return launch_head_gemm_t<true, 8>(n, dp, q_heads * dp, wuk, hs, kMlaW, batch, q_heads, 3, qimg, stream);
}

cudaError_t launch_mla_uv(const float* att, const uint16_t* wuv, int batch, int n_heads, int hs, uint8_t* xf,
                          cudaStream_t stream, int xf16) {
  if (hs > 128) return cudaErrorInvalidValue;  // 4 chunks of hs/32 column groups x 32 d-slices of 16
  return launch_head_gemm_t<false, 32>(att, kMlaDV, n_heads * kMlaDV, wuv, kMlaDV, hs, batch, n_heads, 4, xf,
                                       stream, xf16);
}

}  // namespace hx
