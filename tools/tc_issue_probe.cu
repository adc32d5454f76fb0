// Issue and completion cost of small-N tcgen05.mma (kind::f16, M = 128) from
// one elected lane of a converged warp: A from TMEM (ts) or shared memory (ss),
// N in {16, 32, 64, 256}; 8 fully unrolled MMAs (K = 128) per round.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2507_07120_b200/csrc tools/tc_issue_probe.cu -o tools/tc_issue_probe
#include <cstdio>

#include "common.cuh"
#include "tc05.cuh"

using namespace hx;

__host__ __device__ constexpr uint32_t idesc_f16(int m, int n, bool a_mn, bool b_mn) {
  return (1u << 4) | (static_cast<uint32_t>(a_mn) << 15) | (static_cast<uint32_t>(b_mn) << 16) |
         (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
}

HX_DEV bool elect_one() {
  uint32_t pred;
  asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}" : "=r"(pred));
  return pred != 0;
}

template <int MODE, int N>
__global__ void probe(int rounds, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];  // A 32 KB | B 64 KB
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&tslot, 512);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < (96 << 10) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tslot;
  if (warp == 0) {
    const uint32_t a = smem_u32(sm), b = a + (32 << 10);
    constexpr uint32_t id = idesc_f16(128, N, false, false);
    const uint64_t bd0 = umma_desc(b, (N / 8) * 128, 128), ad0 = umma_desc(a, 16 * 128, 128);
    __syncwarp();
    const unsigned long long t0 = clock64();
    for (int r = 0; r < rounds; ++r) {
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint64_t bd = bd0 + static_cast<uint64_t>((k * 2 * (N / 8) * 128) >> 4);
          if constexpr (MODE == 0)
            umma_ts(tb + 256 + (r & 1) * 128, tb + k * 8, bd, id, k > 0);
          else
            umma_ss(tb + 256 + (r & 1) * 128, ad0 + static_cast<uint64_t>((k * 2 * 16 * 128) >> 4), bd, id, k > 0);
        }
      }
      __syncwarp();
    }
    const unsigned long long t1 = clock64();
    if (elect_one()) umma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    const unsigned long long t2 = clock64();
    if (threadIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tb, 512);
}

template <int MODE, int N>
void run(unsigned long long* d) {
  cudaFuncSetAttribute(probe<MODE, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 << 10);
  for (int rounds : {1, 16}) {
    probe<MODE, N><<<1, 128, 96 << 10>>>(rounds, d);
    unsigned long long h[2];
    if (cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost) != cudaSuccess) {
      printf("error\n");
      return;
    }
    printf("%s N=%3d mmas=%3d: issue %6llu cyc (%5.1f/mma)  done %6llu cyc (%5.1f/mma)\n", MODE ? "ss" : "ts", N,
           8 * rounds, h[0], double(h[0]) / (8 * rounds), h[1], double(h[1]) / (8 * rounds));
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  run<0, 16>(d); run<0, 32>(d); run<0, 64>(d); run<0, 256>(d);
  run<1, 16>(d); run<1, 32>(d); run<1, 64>(d); run<1, 256>(d);
  return 0;
}
