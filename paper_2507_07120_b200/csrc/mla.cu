// MLA decode attention on the 5th-generation tensor cores (tcgen05 + TMEM).
//
// Per (rank shard, request): 128 query heads (zero-padded) share one latent
// KV "head" of width W = 576 (keys = the latent, values = its first 512 dims):
//   S = Q . C^T * (1/sqrt(W)),  P = exp(S - m),  O = P . C[:, :512]
// -- partial_head_attention (attention.hpp:65-78) for every head of the
// rank, with the LSE of each head (HeadFragment) so the fragments merge
// exactly as merge_head_fragments (:118-137).
//
// At ~242 FLOP per KV byte MLA sits at the B200 ridge, so both GEMMs run on
// tcgen05 (UMMA M = 128 heads, fp32 accumulators in TMEM). The fp32 output
// [128 x 512] alone would fill all 512 TMEM columns, so a work item owns one
// VALUE HALF (256 dims): the two items of a (split, stream) pair each compute
// S for the whole tile and accumulate their half of O (the QK^T product is
// issued twice; the KV bytes come from HBM once and from L2 twice).
//
// TMEM (512 columns x 128 lanes fp32):
//   S/P buffer 0 [0, 128)   S/P buffer 1 [128, 256)   O half [256, 512)
// Tiles are 128-row pages; S of tile t+1 is computed while the softmax of
// tile t runs, and P.V(t) follows. Shared memory: the Q image (147,456 B,
// K-major A operand, once per item) + a 5 x 16 KB ring of latent chunks
// (64 dims x 128 rows, contiguous in the page layout).
// Roles (192 threads):
//   warps 0-3  softmax: thread = head row = TMEM lane. Row max, lazy rescale
//              of O (only when the max grows by > 2^8, FA4-style; decided per
//              warp), P = exp2 in bf16 written into TMEM over S (the A operand
//              of P.V), row sum of the bf16-rounded P, final O / z and LSE.
//   warp 4     producer: cp.async.bulk of the Q image and latent chunks in
//              the MMA's consumption order.
//   warp 5     TMEM allocation + MMA issue (one thread):
//                S(t)  = 36 x UMMA SS  M128 N128 K16 (Q smem, latent K-major)
//                O    += 32 x UMMA TS  M128 N64  K16 (P in TMEM, latent MN-major)
// Items (split, stream, value half) are statically strided over the grid.
#include "common.cuh"
#include "kernels.h"
#include "kv_layout.cuh"
#include "tc05.cuh"

namespace hx {

namespace {
constexpr uint32_t kQBytes = kMlaW * kMlaHeads * 2;  // 147456
constexpr uint32_t kChunk = 64 * kMlaPageRows * 2;   // 16384: 64 latent dims x 128 rows
constexpr int kSChunks = kMlaW / 64;                 // 9
constexpr int kVChunks = kMlaDV / 2 / 64;            // 4 per value half
constexpr int kSlots = 5;
constexpr uint32_t kDgStride = kMlaPageRows / 8 * 128;  // bytes between 8-dim groups of a chunk
constexpr uint32_t kIdescS = umma_idesc_bf16(128, kMlaPageRows, false, false);
constexpr uint32_t kIdescPV = umma_idesc_bf16(128, 64, false, true);
constexpr int kThreads = 192;

struct MlaItem {
  int b, sl, half, pg0, pg1, ntok;
};

__device__ __forceinline__ MlaItem decode_item(const AttnParams& p, int item) {
  MlaItem it;
  it.half = item & 1;
  const int ps = item >> 1;  // split * n_streams + stream
  const int split = ps / p.n_streams;
  const int stream = ps - split * p.n_streams;
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

// Consumption order of an item's chunks (producer and MMA agree on it):
//   S(0), S(1), V(0), S(2), V(1), S(3), ..., V(n-1)
// step k of an item with n tiles -> (tile, is_value)
__device__ __forceinline__ void mla_step(int k, int n, int& tile, bool& value) {
  if (k < 2 || n == 1) {
    if (n == 1) {
      tile = 0;
      value = k == 1;
    } else {
      tile = k;
      value = false;
    }
    return;
  }
  const int j = k - 2;  // V(j/2) then S(j/2 + 2)
  tile = j / 2 + ((j & 1) ? 2 : 0);
  value = (j & 1) == 0;
  if (tile >= n) {  // past the last S: only V remains
    tile = n - 1;
    value = true;
  }
}
}  // namespace

__global__ void __launch_bounds__(kThreads, 1) mla_decode_kernel(const AttnParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* qs = smem;
  uint8_t* ring = smem + kQBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + kSlots * kChunk);
  uint64_t* full = bars;                // [kSlots]
  uint64_t* empty = bars + kSlots;      // [kSlots]
  uint64_t* q_full = bars + 2 * kSlots;
  uint64_t* q_free = q_full + 1;
  uint64_t* s_full = q_full + 2;   // [2] per S buffer
  uint64_t* p_full = q_full + 4;   // [2]
  uint64_t* pv_done = q_full + 6;  // [2]
  uint64_t* o_free = q_full + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_full + 9);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSlots; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(q_full, 1);
    mbar_init(q_free, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 128);
      mbar_init(&pv_done[i], 1);
    }
    mbar_init(o_free, 128);
    fence_mbar_init();
  }
  if (warp == 5) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  griddep_launch_dependents();

  if (warp == 4) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      int it_slot = 0, qcount = 0;
      bool waited = false;
      for (int item = blockIdx.x; item < p.n_items; item += gridDim.x) {
        const MlaItem it = decode_item(p, item);
        if (it.pg1 <= it.pg0) continue;
        if (!waited) {  // the query images come from the QKV kernel
          griddep_wait();
          waited = true;
        }
        if (qcount > 0) mbar_wait(q_free, (qcount - 1) & 1);
        mbar_arrive_expect_tx(q_full, kQBytes);
        bulk_g2s(qs, p.qimg + static_cast<size_t>(it.b) * kQBytes, kQBytes, q_full);
        ++qcount;
        const uint8_t* kvb =
            p.kv + (static_cast<size_t>(it.sl) * p.batch + it.b) * p.page_cap * static_cast<size_t>(mla_page_bytes());
        const int n = it.pg1 - it.pg0;
        for (int k = 0; k < 2 * n; ++k) {
          int tile;
          bool value;
          mla_step(k, n, tile, value);
          const uint8_t* page = kvb + static_cast<size_t>(it.pg0 + tile) * mla_page_bytes();
          const int nch = value ? kVChunks : kSChunks;
          for (int j = 0; j < nch; ++j) {
            const int blk = value ? 4 * it.half + j : j;  // 64-dim block of the page
            const int s = it_slot % kSlots;
            if (it_slot >= kSlots) mbar_wait(&empty[s], ((it_slot / kSlots) - 1) & 1);
            mbar_arrive_expect_tx(&full[s], kChunk);
            bulk_g2s(ring + s * kChunk, page + static_cast<size_t>(blk) * kChunk, kChunk, &full[s]);
            ++it_slot;
          }
        }
      }
      if (!waited) griddep_wait();
    }
  } else if (warp == 5) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t q_addr = smem_u32(qs), ring_addr = smem_u32(ring);
      int it_slot = 0, qcount = 0, g0 = 0, items = 0;  // g0: global index of the item's first tile
      for (int item = blockIdx.x; item < p.n_items; item += gridDim.x) {
        const MlaItem it = decode_item(p, item);
        if (it.pg1 <= it.pg0) continue;
        mbar_wait(q_full, qcount & 1);
        ++qcount;
        tc_fence_after();
        const int n = it.pg1 - it.pg0;
        for (int k = 0; k < 2 * n; ++k) {
          int tile;
          bool value;
          mla_step(k, n, tile, value);
          const int g = g0 + tile, buf = g & 1;
          if (!value) {
            // S(tile) into buffer buf: the P.V that last read this buffer must be done
            if (g >= 2) mbar_wait(&pv_done[buf], ((g >> 1) - 1) & 1);
            tc_fence_after();
            for (int j = 0; j < kSChunks; ++j) {
              const int s = it_slot % kSlots;
              mbar_wait(&full[s], (it_slot / kSlots) & 1);
              tc_fence_after();
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) {
                const uint64_t a = umma_desc(q_addr + (4 * j + kk) * 4096, 2048, 128);
                const uint64_t bd = umma_desc(ring_addr + s * kChunk + kk * 2 * kDgStride, kDgStride, 128);
                umma_ss(tbase + buf * 128, a, bd, kIdescS, (j | kk) != 0);
              }
              umma_commit(&empty[s]);
              ++it_slot;
            }
            if (tile == n - 1) umma_commit(q_free);
            umma_commit(&s_full[buf]);
          } else {
            mbar_wait(&p_full[buf], (g >> 1) & 1);
            if (tile == 0 && items > 0) mbar_wait(o_free, (items - 1) & 1);  // previous O read out
            tc_fence_after();
            for (int v = 0; v < kVChunks; ++v) {
              const int s = it_slot % kSlots;
              mbar_wait(&full[s], (it_slot / kSlots) & 1);
              tc_fence_after();
#pragma unroll
              for (int kk = 0; kk < kMlaPageRows / 16; ++kk) {
                const uint64_t bd = umma_desc(ring_addr + s * kChunk + kk * 256, 128, kDgStride);
                umma_ts(tbase + 256 + 64 * v, tbase + buf * 128 + 8 * kk, bd, kIdescPV,
                        (tile > 0 || kk > 0) ? 1u : 0u);
              }
              umma_commit(&empty[s]);
              ++it_slot;
            }
            umma_commit(&pv_done[buf]);
          }
        }
        g0 += n;
        ++items;
      }
    }
  } else {
    // ------------------------------------------------------------ softmax (warps 0-3)
    const int h = threadIdx.x;  // head row == TMEM lane
    const uint32_t lrow = tbase + (static_cast<uint32_t>(warp * 32) << 16);
    int g = 0;
    for (int item = blockIdx.x; item < p.n_items; item += gridDim.x) {
      const MlaItem it = decode_item(p, item);
      float* po = p.part_o + (static_cast<size_t>(item) * kMlaHeads + h) * 256;
      float* pl = p.part_lse2 + static_cast<size_t>(item) * kMlaHeads + h;
      if (it.pg1 <= it.pg0) {
        if (h < p.q_heads) {
          for (int i = 0; i < 256; i += 4) *reinterpret_cast<float4*>(po + i) = make_float4(0.f, 0.f, 0.f, 0.f);
          *pl = -INFINITY;
        }
        continue;
      }
      float m = -INFINITY, z = 0.f;
      const int n = it.pg1 - it.pg0;
      for (int t = 0; t < n; ++t, ++g) {
        const int buf = g & 1;
        const uint32_t sb = lrow + buf * 128;
        const int valid = min(kMlaPageRows, it.ntok - (it.pg0 + t) * kMlaPageRows);
        mbar_wait(&s_full[buf], (g >> 1) & 1);
        tc_fence_after();
        float mt = -INFINITY;
#pragma unroll 1
        for (int c = 0; c < kMlaPageRows / 32; ++c) {
          float v[32];
          tmem_ld32(sb + 32 * c, v);
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (32 * c + i < valid) mt = fmaxf(mt, v[i]);
        }
        mt *= p.qscale;
        // Lazy rescale: a row keeps its reference max unless the tile max exceeds
        // it by 2^8. Decided per warp (tcgen05.ld/st are warp-collective); rows
        // that did not grow rescale by exactly 1.
        const bool grow = mt > m + 8.f;
        if (__any_sync(0xffffffffu, grow)) {
          const float m_new = grow ? mt : m;
          const float alpha = grow ? exp2f(m - m_new) : 1.f;  // 0 on the first tile
          if (t > 0) {
            // O holds tiles < t: wait for P.V(t-1), then rescale it in TMEM
            mbar_wait(&pv_done[(g - 1) & 1], ((g - 1) >> 1) & 1);
            tc_fence_after();
#pragma unroll 1
            for (int c = 0; c < 8; ++c) {
              float v[32];
              tmem_ld32(lrow + 256 + 32 * c, v);
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] *= alpha;
              tmem_st32(lrow + 256 + 32 * c, v);
            }
          }
          z *= alpha;
          m = m_new;
        }
#pragma unroll 1
        for (int c = 0; c < kMlaPageRows / 32; ++c) {
          float v[32];
          tmem_ld32(sb + 32 * c, v);
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float p0 = (32 * c + 2 * i < valid) ? exp2f(fmaf(v[2 * i], p.qscale, -m)) : 0.f;
            const float p1 = (32 * c + 2 * i + 1 < valid) ? exp2f(fmaf(v[2 * i + 1], p.qscale, -m)) : 0.f;
            const __nv_bfloat162 pb = __floats2bfloat162_rn(p0, p1);  // .x = low half = even token
            z += __low2float(pb) + __high2float(pb);
            pk[i] = *reinterpret_cast<const uint32_t*>(&pb);
          }
          tmem_st16(sb + 16 * c, pk);  // P over the S columns already read
        }
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&p_full[buf]);
      }
      mbar_wait(&pv_done[(g - 1) & 1], ((g - 1) >> 1) & 1);
      tc_fence_after();
      const float inv = z > 0.f ? 1.f / z : 0.f;
#pragma unroll 1
      for (int c = 0; c < 8; ++c) {
        float v[32];
        tmem_ld32(lrow + 256 + 32 * c, v);
        if (h < p.q_heads)
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            *reinterpret_cast<float4*>(po + 32 * c + i) =
                make_float4(v[i] * inv, v[i + 1] * inv, v[i + 2] * inv, v[i + 3] * inv);
      }
      if (h < p.q_heads) *pl = z > 0.f ? m + log2f(z) : -INFINITY;
      tc_fence_before();
      mbar_arrive(o_free);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 5) tmem_dealloc(tbase, 512);
}

// Merge a stream's split partials (split order, deterministic) into the
// rank's fragment [slot][b][head][512] + natural-log lse (HeadFragment).
__global__ void mla_split_reduce_kernel(const AttnParams p, float* frag_o, float* frag_lse) {
  griddep_wait();
  griddep_launch_dependents();
  const int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int h = wg % p.q_heads, stream = wg / p.q_heads;
  if (stream >= p.n_streams) return;
  const int bl = stream % p.stream_batch, sl = stream / p.stream_batch, b = bl + p.b_begin;
  const int rank = (sl + p.slot_base) % p.kvp;
  const int ntok = static_cast<int>(rr_count(p.total[b], rank, p.chunk, p.kvp));
  const int pages = (ntok + kMlaPageRows - 1) / kMlaPageRows;
  float M = -INFINITY;
  for (int s = 0; s < p.splits; ++s) {
    const int pg0 = static_cast<int>((static_cast<long long>(s) * pages) / p.splits);
    const int pg1 = static_cast<int>((static_cast<long long>(s + 1) * pages) / p.splits);
    if (pg1 > pg0)
      M = fmaxf(M, p.part_lse2[static_cast<size_t>(((s * p.n_streams + stream) * 2) * kMlaHeads) + h]);
  }
  float o[16] = {};
  float L = 0.f;
  for (int s = 0; s < p.splits; ++s) {
    const int pg0 = static_cast<int>((static_cast<long long>(s) * pages) / p.splits);
    const int pg1 = static_cast<int>((static_cast<long long>(s + 1) * pages) / p.splits);
    if (pg1 <= pg0) continue;
    const size_t i0 = static_cast<size_t>((s * p.n_streams + stream) * 2);
    const float w = exp2f(p.part_lse2[i0 * kMlaHeads + h] - M);
    L += w;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int d = lane + 32 * i, half = d >> 8;
      o[i] += w * p.part_o[((i0 + half) * kMlaHeads + h) * 256 + (d & 255)];
    }
  }
  const size_t fo = (static_cast<size_t>(sl) * p.batch + b) * p.q_per_slot + h;
#pragma unroll
  for (int i = 0; i < 16; ++i) frag_o[fo * kMlaDV + lane + 32 * i] = L > 0.f ? o[i] / L : 0.f;
  if (lane == 0) frag_lse[fo] = L > 0.f ? (M + log2f(L)) * 0.69314718055994530942f : -INFINITY;
}

size_t mla_smem_bytes() { return kQBytes + kSlots * kChunk + (2 * kSlots + 12) * 8; }

cudaError_t launch_mla_decode(const AttnParams& p, int grid, cudaStream_t stream) {
  if (p.q_heads > kMlaHeads || p.q_heads < 1) return cudaErrorInvalidValue;
  static bool configured = false;
  const size_t smem = mla_smem_bytes();
  if (!configured) {
    cudaError_t e =
        cudaFuncSetAttribute(mla_decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  return launch_k(mla_decode_kernel, dim3(grid), dim3(kThreads), smem, stream, p);
}

cudaError_t launch_mla_split_reduce(const AttnParams& p, float* frag_o, float* frag_lse, cudaStream_t stream) {
  const long long warps = static_cast<long long>(p.n_streams) * p.q_heads;
  const int threads = 256;
  return launch_k(mla_split_reduce_kernel, dim3(static_cast<unsigned>((warps * 32 + threads - 1) / threads)),
                  dim3(threads), 0, stream, p, frag_o, frag_lse);
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
                                        uint64_t stream_k) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  constexpr int kRowsPerPage = kMlaPageRows * (kMlaW / 8);  // 16-byte rows per page
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
  const uint64_t base = ((static_cast<uint64_t>(b) << 32) + static_cast<uint64_t>(g)) * kMlaW + dg * 8;
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
  uint8_t* pg = kv + (static_cast<size_t>(st) * page_cap + page) * static_cast<size_t>(mla_page_bytes());
  *reinterpret_cast<uint4*>(pg + static_cast<size_t>(ci) * 16) = make_uint4(w[0], w[1], w[2], w[3]);
}

__global__ void add_total_mla_kernel(int* total, int batch, int n) {
  for (int b = threadIdx.x; b < batch; b += blockDim.x) total[b] += n;
}

cudaError_t launch_kv_fill_hash_mla(uint8_t* kv, int* total, int batch, int kvp, int chunk, int page_cap,
                                    int slot_base, int n_local_slots, long long n, uint64_t seed, uint64_t stream_k,
                                    cudaStream_t stream) {
  const long long work = static_cast<long long>(n_local_slots) * batch * page_cap * kMlaPageRows * (kMlaW / 8);
  if (n > 0)
    kv_fill_hash_mla_kernel<<<static_cast<unsigned>((work + 255) / 256), 256, 0, stream>>>(
        kv, total, batch, kvp, chunk, page_cap, slot_base, n_local_slots, n, seed, stream_k);
  add_total_mla_kernel<<<1, 64, 0, stream>>>(total, batch, static_cast<int>(n));
  return cudaGetLastError();
}

}  // namespace hx
