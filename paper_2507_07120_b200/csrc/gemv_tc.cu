// Weight-streaming GEMM on the 5th-generation tensor cores for batches above
// 16 (north star (3): "tcgen05 is used only once the batch makes the
// contraction dense"). Same split-K partials and epilogue kernel as the
// mma.sync GEMV (gemv.cu); the inner product moves to tcgen05:
//
//   D[128 rows x N] (TMEM, fp32) += W[128 rows x 16 k] . X^T[16 k x N]   per k-step, x term, row block
//
// A tile is TWO 128-row blocks (256 output features) x one k-chunk, so every
// x slice staged in shared memory feeds two row blocks. Both operands are
// K-major canonical core matrices (no swizzle): the weights are initialised in
// that image (per row block and k-step 4 KB = [row group 16][k-half 2][row 8]
// [8 k], misc.cu) and the x-fragments switch to it for nb8 >= 4 (xfrag.cuh:
// per k-step [term][batch group]), so the TMA bulk copies land as ready
// operands. One MMA multiplies the hi and mid terms at once (N = 2 x 8 nb8 =
// 64 or 128 columns; the drain adds the two column halves); the QKV
// projection's third term is a second MMA (N = 8 nb8) accumulating into the
// hi half.
//
// Roles (224 threads): warp 4 weight producer (tile queue; two bulk copies per
// stage, one per row block), warp 6 x producer (one copy per term; a warp
// issues ~1 bulk copy per 300 ns), warp 5 TMEM allocation + single-thread MMA
// issue, warps 0-3 drain finished tiles (tcgen05.ld, TMEM lane = feature row)
// into the split-K partials while the next tile accumulates in the other TMEM
// buffer.
#include "common.cuh"
#include "kernels.h"
#include "tc05.cuh"
#include "xfrag.cuh"

namespace hx {

namespace {
constexpr int kTcThreads = 224;
constexpr int kTcDone = -1;
// ring geometry: KSTEPS k-steps per stage x NSTAGE stages
struct TcMeta {
  int tile, pb, kc, gi, nks, first, last, k0;
};
template <int NB8, int KSTEPS>
constexpr uint32_t tc_stage_bytes() {
  return KSTEPS * (2 * 4096u + kXfTerms * NB8 * 256u);  // all three terms: one x copy per stage
}
template <int NB8, int KSTEPS, int NSTAGE>
constexpr size_t tc_smem_bytes() {
  return NSTAGE * tc_stage_bytes<NB8, KSTEPS>() + NSTAGE * sizeof(TcMeta) + 8 * sizeof(int) + (3 * NSTAGE + 6) * 8 +
         16 + 128;
}
}  // namespace

template <int NB8, int XS, int KSTEPS, int NSTAGE>
__global__ void __launch_bounds__(kTcThreads, 1) gemv_tc_kernel(const GemvParams p) {
  static_assert(NB8 == 4 || NB8 == 8, "tcgen05 GEMV: N = 32 or 64 batch rows");
  constexpr int NST = NSTAGE;
  constexpr int kTcSteps = KSTEPS;
  constexpr uint32_t XT = NB8 * 256u;                     // x bytes per (k-step, term)
  constexpr uint32_t XSTEP = kXfTerms * XT;               // x bytes per k-step (all terms)
  constexpr uint32_t SW = kTcSteps * 4096u;               // weight bytes per stage and row block
  constexpr uint32_t SB = tc_stage_bytes<NB8, KSTEPS>();
  constexpr int N = 8 * NB8;                              // batch rows
  constexpr int NC = 2 * N;                               // accumulator columns: [hi | mid]
  constexpr uint32_t COLS = 4 * NC;                       // 2 buffers x 2 row blocks
  constexpr uint32_t IDESC2 = umma_idesc_bf16(128, NC, false, false);
  constexpr uint32_t IDESC1 = umma_idesc_bf16(128, N, false, false);

  extern __shared__ __align__(1024) uint8_t smem[];
  TcMeta* meta = reinterpret_cast<TcMeta*>(smem + NST * SB);
  int* acc_meta = reinterpret_cast<int*>(meta + NST);  // [2 buffers][pb, kc, gi, done]
  uint64_t* full = reinterpret_cast<uint64_t*>(acc_meta + 8);
  uint64_t* empty = full + NST;
  uint64_t* acc_full = empty + NST;     // [2] all MMAs of the tile done (tcgen05.commit)
  uint64_t* acc_ready = acc_full + 2;   // [2] the tile's (pb, kc, gi) written
  uint64_t* acc_empty = acc_ready + 2;  // [2] drained by the 128 epilogue threads
  uint64_t* meta_full = acc_empty + 2;  // [NST] stage meta written (weight producer -> x producer)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(meta_full + NST);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KST = p.K >> 4;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&meta_full[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_ready[i], 1);
      mbar_init(&acc_empty[i], 128);
    }
    fence_mbar_init();
  }
  if (warp == 5) tmem_alloc(tslot, COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  griddep_launch_dependents();

  if (warp == 4) {
    // ------------------------------------------------------------ weight producer (tile queue)
    if (lane == 0) {
      int st = 0;
      int n_tiles = p.n_tiles;
      if (p.group_count) {  // the active-expert list is produced by the routing kernel
        griddep_wait();
        n_tiles = *p.group_count * p.tiles_per_group;
      }
      for (;;) {
        const int tile = atomicAdd(p.work_counter, 1);
        const bool done = tile >= n_tiles;
        const int gi = (done || !p.group_count) ? 0 : tile / p.tiles_per_group;
        const int rem = done ? 0 : tile - gi * p.tiles_per_group;
        const int pb = rem / p.ksplit;  // row-block pair
        const int kc = rem - pb * p.ksplit;
        const int k0 = kc * p.kr_steps;
        const int k1 = min(k0 + p.kr_steps, KST);
        const int nstage = done ? 1 : (k1 - k0 + kTcSteps - 1) / kTcSteps;
        const uint8_t* wg = reinterpret_cast<const uint8_t*>(p.w);
        if (!done && p.group_count) wg += static_cast<size_t>(p.group_ids[gi] - p.group_base) * p.w_group_stride;
        for (int si = 0; si < nstage; ++si, ++st) {
          const int s = st % NST;
          if (st >= NST) mbar_wait(&empty[s], ((st / NST) & 1) ^ 1);
          TcMeta& m = meta[s];
          if (done) {
            m.tile = kTcDone;
            mbar_arrive(&meta_full[s]);
            mbar_arrive(&full[s]);
            break;
          }
          const int a = k0 + si * kTcSteps;
          const int n = min(kTcSteps, k1 - a);
          m.tile = tile;
          m.pb = pb;
          m.kc = kc;
          m.gi = gi;
          m.nks = n;
          m.first = si == 0;
          m.last = si == nstage - 1;
          m.k0 = a;
          uint8_t* dst = smem + s * SB;
          mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(n) * (2 * 4096u + XSTEP));
          mbar_arrive(&meta_full[s]);  // the x producer may now issue its copies (tx already expected)
#pragma unroll
          for (int r2 = 0; r2 < 2; ++r2)
            bulk_g2s(dst + r2 * SW, wg + (static_cast<size_t>(2 * pb + r2) * KST + a) * 4096,
                     static_cast<uint32_t>(n) * 4096u, &full[s]);
        }
        if (done) break;
      }
    }
  } else if (warp == 6) {
    // ------------------------------------------------------------ x producer
    if (lane == 0) {
      griddep_wait();  // the x fragments are the previous kernel's output
      for (int st = 0;; ++st) {
        const int s = st % NST;
        mbar_wait(&meta_full[s], (st / NST) & 1);
        const TcMeta m = meta[s];
        if (m.tile == kTcDone) break;
        const uint8_t* xg = p.xf + (p.group_count ? static_cast<size_t>(m.gi) * p.xf_group_stride : 0) +
                            static_cast<size_t>(m.k0) * XSTEP;
        bulk_g2s(smem + s * SB + 2 * SW, xg, static_cast<uint32_t>(m.nks) * XSTEP, &full[s]);
      }
    }
  } else if (warp == 5) {
    // ------------------------------------------------------------ MMA issue (one elected lane of
    // the converged warp: tc05.cuh elect_one -- a lone-lane issue loop costs ~145 cycles per MMA)
    {
      const uint32_t ring = smem_u32(smem);
      int uses = 0;  // accumulator buffer uses (tile t -> buffer t & 1)
      for (int st = 0;; ++st) {
        const int s = st % NST;
        mbar_wait(&full[s], (st / NST) & 1);
        const TcMeta m = meta[s];
        const int buf = uses & 1;
        if (m.tile == kTcDone || m.first) {
          if (uses >= 2) mbar_wait(&acc_empty[buf], ((uses >> 1) - 1) & 1);  // drained two tiles ago
          if (lane == 0) {
            acc_meta[buf * 4 + 0] = m.pb;
            acc_meta[buf * 4 + 1] = m.kc;
            acc_meta[buf * 4 + 2] = m.gi;
            acc_meta[buf * 4 + 3] = m.tile == kTcDone;
            mbar_arrive(&acc_ready[buf]);
          }
          __syncwarp();
          if (m.tile == kTcDone) break;
        }
        tc_fence_after();
        const uint32_t sw = ring + s * SB, sx = sw + 2 * SW;
        const uint64_t a0 = umma_desc(sw, 128, 256), x0 = umma_desc(sx, 128, 256);
        const uint32_t d0 = tbase + static_cast<uint32_t>(2 * buf * NC);
        if (elect_one()) {
          for (int kk = 0; kk < m.nks; ++kk) {
#pragma unroll
            for (int r2 = 0; r2 < 2; ++r2) {
              const uint64_t a = a0 + static_cast<uint64_t>((r2 * SW + kk * 4096u) >> 4);
              const uint64_t x = x0 + static_cast<uint64_t>((kk * XSTEP) >> 4);
              const uint32_t acc = (m.first && kk == 0) ? 0u : 1u;
              umma_ss(d0 + r2 * NC, a, x, IDESC2, acc);  // [hi | mid]
              if (XS == 3) umma_ss(d0 + r2 * NC, a, x + static_cast<uint64_t>((2 * XT) >> 4), IDESC1, 1u);  // lo -> hi
            }
          }
          umma_commit(&empty[s]);  // the stage is free once these MMAs have read it
          if (m.last) umma_commit(&acc_full[buf]);
        }
        __syncwarp();
        if (m.last) ++uses;
      }
    }
  } else {
    // ------------------------------------------------------------ drain (warps 0-3: TMEM lanes = rows)
    for (int uses = 0;; ++uses) {
      const int buf = uses & 1;
      mbar_wait(&acc_ready[buf], (uses >> 1) & 1);
      if (acc_meta[buf * 4 + 3]) break;
      const int pb = acc_meta[buf * 4 + 0], kc = acc_meta[buf * 4 + 1], gi = acc_meta[buf * 4 + 2];
      mbar_wait(&acc_full[buf], (uses >> 1) & 1);
      tc_fence_after();
      float* yp = p.ypart + static_cast<size_t>(gi) * p.part_group_stride +
                  static_cast<size_t>(kc) * p.batch * p.Npad;
#pragma unroll
      for (int r2 = 0; r2 < 2; ++r2) {
        const int row = (2 * pb + r2) * 128 + warp * 32 + lane;
        const uint32_t col = tbase + static_cast<uint32_t>((2 * buf + r2) * NC) + (static_cast<uint32_t>(warp * 32) << 16);
#pragma unroll
        for (int c0 = 0; c0 < N; c0 += 32) {
          float v[32], w[32];
          tmem_ld32(col + c0, v);       // W . x_hi (+ W . x_lo)
          tmem_ld32(col + N + c0, w);   // W . x_mid
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (c0 + i < p.batch) yp[static_cast<size_t>(c0 + i) * p.Npad + row] = v[i] + w[i];
        }
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[buf]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc(tbase, COLS);
  }
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(p.work_counter + 1, 1) == static_cast<int>(gridDim.x) - 1) {
      p.work_counter[0] = 0;  // every CTA drained the queue: reset for the next launch
      p.work_counter[1] = 0;
      __threadfence();
    }
  }
}

template <int NB8, int XS, int KSTEPS, int NSTAGE>
static cudaError_t launch_tc_t(const GemvParams& p, int grid, cudaStream_t stream) {
  constexpr size_t smem = tc_smem_bytes<NB8, KSTEPS, NSTAGE>();
  static_assert(smem <= 227 * 1024, "tcgen05 GEMV ring exceeds shared memory");
  const cudaError_t e = smem_optin<gemv_tc_kernel<NB8, XS, KSTEPS, NSTAGE>>(smem);
  if (e != cudaSuccess) return e;
  return launch_k(gemv_tc_kernel<NB8, XS, KSTEPS, NSTAGE>, dim3(grid), dim3(kTcThreads), smem, stream, p);
}

// 4 k-steps x 4 stages (2 x 8 measured the same at B = 64)
template <int NB8, int XS>
static cudaError_t launch_tc_ring(const GemvParams& p, int grid, cudaStream_t stream) {
  return launch_tc_t<NB8, XS, 4, 4>(p, grid, stream);
}

cudaError_t launch_gemv_tc(const GemvParams& p, int nb8, int xs, int grid, cudaStream_t stream) {
  if ((p.Npad % 256) || ((p.K >> 4) % 4) || (p.kr_steps % 4)) return cudaErrorInvalidValue;
  if (nb8 == 4) return xs == 3 ? launch_tc_ring<4, 3>(p, grid, stream) : launch_tc_ring<4, 2>(p, grid, stream);
  if (nb8 == 8) return xs == 3 ? launch_tc_ring<8, 3>(p, grid, stream) : launch_tc_ring<8, 2>(p, grid, stream);
  return cudaErrorInvalidValue;
}

}  // namespace hx
