// Probe of the tcgen05 operand forms the quantised GQA decode kernel
// (attention_tc.cu) relies on, checked against a host product:
//   test 0: D[128 x N] = A[128 x 128] . B^T, A f16 in TMEM (lane = row m,
//           column j = elements k = 2j, 2j+1), B f16 K-major in shared memory
//   test 1: same A, B f16 MN-major in shared memory ([n/8][k/8][k%8][n%8])
//   test 2: A f16 K-major in shared memory (control)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2507_07120_b200/csrc tools/tc_probe.cu -o tools/tc_probe
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>

#include "common.cuh"
#include "tc05.cuh"

using namespace hx;

constexpr int M = 128, K = 128;

__host__ __device__ constexpr uint32_t idesc_f16(int m, int n, bool a_mn, bool b_mn) {
  return (1u << 4) | (static_cast<uint32_t>(a_mn) << 15) | (static_cast<uint32_t>(b_mn) << 16) |
         (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
}

__host__ __device__ float aval(int m, int k) { return (((m * 7 + k * 3) % 9) - 4) * 0.25f; }
__host__ __device__ float bval(int n, int k) { return (((n * 5 + k) % 7) - 3) * 0.5f; }

template <int N>
__global__ void probe(int test, float* out) {
  __shared__ __align__(1024) __half bs[N * K];
  __shared__ __align__(1024) __half as[M * K];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) tmem_alloc(&tbase, 256);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  // B image
  for (int i = tid; i < N * K; i += 128) {
    const int n = i / K, k = i % K;
    int off;
    if (test == 1)
      off = (((n >> 3) * (K / 8) + (k >> 3)) * 8 + (k & 7)) * 8 + (n & 7);  // MN-major
    else
      off = (((k >> 3) * (N / 8) + (n >> 3)) * 8 + (n & 7)) * 8 + (k & 7);  // K-major
    bs[off] = __float2half(bval(n, k));
  }
  for (int i = tid; i < M * K; i += 128) {  // A K-major smem image (test 2)
    const int m = i / K, k = i % K;
    as[(((k >> 3) * (M / 8) + (m >> 3)) * 8 + (m & 7)) * 8 + (k & 7)] = __float2half(aval(m, k));
  }
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  // A into TMEM columns [0, 64): lane = row
  {
    const int m = tid;
    uint32_t r[16];
    for (int c0 = 0; c0 < 64; c0 += 16) {
      for (int j = 0; j < 16; ++j) {
        const int k = 2 * (c0 + j);
        __half2 h = __floats2half2_rn(aval(m, k), aval(m, k + 1));
        r[j] = *reinterpret_cast<uint32_t*>(&h);
      }
      tmem_st16(tm + (static_cast<uint32_t>(warp * 32) << 16) + c0, r);
    }
    tmem_wait_st();
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    const uint32_t d = tm + 128;
    for (int ks = 0; ks < K / 16; ++ks) {
      if (test == 2) {
        const uint64_t a = umma_desc(smem_u32(as) + ks * 2 * (M / 8) * 128, (M / 8) * 128, 128);
        const uint64_t b = umma_desc(smem_u32(bs) + ks * 2 * (N / 8) * 128, (N / 8) * 128, 128);
        umma_ss(d, a, b, idesc_f16(M, N, false, false), ks > 0);
      } else if (test == 1) {
        const uint64_t b = umma_desc(smem_u32(bs) + ks * 2 * 128, 128, (K / 8) * 128);
        umma_ts(d, tm + ks * 8, b, idesc_f16(M, N, false, true), ks > 0);
      } else {
        const uint64_t b = umma_desc(smem_u32(bs) + ks * 2 * (N / 8) * 128, (N / 8) * 128, 128);
        umma_ts(d, tm + ks * 8, b, idesc_f16(M, N, false, false), ks > 0);
      }
    }
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  float v[32];
  tmem_ld32(tm + (static_cast<uint32_t>(warp * 32) << 16) + 128, v);
  for (int n = 0; n < N; ++n) out[tid * N + n] = v[n];
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 256);
}

template <int N>
int run(int test) {
  float* d;
  cudaMalloc(&d, M * N * 4);
  cudaMemset(d, 0, M * N * 4);
  probe<N><<<1, 128>>>(test, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("test %d N=%d: CUDA error %s\n", test, N, cudaGetErrorString(e));
    return 1;
  }
  float h[M * N];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double err = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double r = 0;
      for (int k = 0; k < K; ++k) r += static_cast<double>(aval(m, k)) * bval(n, k);
      err = fmax(err, fabs(r - h[m * N + n]));
    }
  printf("test %d N=%d: max |err| = %g  (D[0][0..3] = %g %g %g %g)\n", test, N, err, h[0], h[1], h[2], h[3]);
  cudaFree(d);
  return err > 1e-3;
}

// test 3: kind::f8f6f4, A e4m3 K-major [128 x 128] and B e4m3 K-major [N x 128]
// from shared memory (core matrix = 8 rows x 16 bytes), 4 MMAs of K = 32
__host__ __device__ float a8(int m, int k) { return (((m * 5 + k * 3) % 7) - 3) * 0.5f; }
__host__ __device__ float b8(int n, int k) { return (((n * 3 + k) % 5) - 2) * 0.25f; }
__device__ uint8_t to_e4m3(float x) {
  uint16_t r;
  asm("{\n.reg .b16 t;\ncvt.rn.satfinite.e4m3x2.f32 t, %1, %1;\nmov.b16 %0, t;\n}" : "=h"(r) : "f"(x));
  return static_cast<uint8_t>(r & 0xFF);
}
template <int N>
__global__ void probe8(float* out) {
  __shared__ __align__(1024) uint8_t as[128 * 128];
  __shared__ __align__(1024) uint8_t bs[N * 128];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) tmem_alloc(&tbase, 256);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  // K-major 8-bit: [k/16][row/8][row%8][k%16]
  for (int i = tid; i < 128 * 128; i += 128) {
    const int m = i / 128, k = i % 128;
    as[(((k >> 4) * 16 + (m >> 3)) * 8 + (m & 7)) * 16 + (k & 15)] = to_e4m3(a8(m, k));
  }
  for (int i = tid; i < N * 128; i += 128) {
    const int n = i / 128, k = i % 128;
    bs[(((k >> 4) * (N / 8) + (n >> 3)) * 8 + (n & 7)) * 16 + (k & 15)] = to_e4m3(b8(n, k));
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  // idesc kind::f8f6f4: D f32 (bit 4), A/B format E4M3 = 0, K-major both, N>>3 at 17, M>>4 at 24
  const uint32_t id = (1u << 4) | (static_cast<uint32_t>(N >> 3) << 17) | (128u >> 4 << 24);
  if (warp == 0) {
    if (elect_one()) {
      for (int ks = 0; ks < 4; ++ks) {  // K = 32 per MMA: two 16-byte core matrices along K
        const uint64_t a = umma_desc(smem_u32(as) + ks * 2 * 16 * 128, 16 * 128, 128);
        const uint64_t b = umma_desc(smem_u32(bs) + ks * 2 * (N / 8) * 128, (N / 8) * 128, 128);
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n}\n" ::"r"(tm + 128),
            "l"(a), "l"(b), "r"(id), "r"(ks > 0 ? 1u : 0u)
            : "memory");
      }
      umma_commit(&bar);
    }
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int n0 = 0; n0 < N; n0 += 32) {
    float v[32];
    tmem_ld32(tm + (static_cast<uint32_t>(warp * 32) << 16) + 128 + n0, v);
    for (int n = 0; n < 32; ++n) out[tid * N + n0 + n] = v[n];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 256);
}
template <int N>
int run8() {
  float* d;
  cudaMalloc(&d, 128 * N * 4);
  probe8<N><<<1, 128>>>(d);
  if (cudaDeviceSynchronize() != cudaSuccess) {
    printf("f8 test N=%d: CUDA error\n", N);
    return 1;
  }
  float h[128 * N];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double err = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      double r = 0;
      for (int k = 0; k < 128; ++k) r += static_cast<double>(a8(m, k)) * b8(n, k);
      err = fmax(err, fabs(r - h[m * N + n]));
    }
  printf("f8f6f4 e4m3 K-major N=%d: max |err| = %g (D[0][0..1] = %g %g)\n", N, err, h[0], h[1]);
  cudaFree(d);
  return err > 1e-3;
}

// test 4: kind::f8f6f4 with A and B both MN-major e4m3 (the MLA FP8 P.V form):
// [mn/16][k/8][k%8][mn%16] bytes -- a core matrix is 8 K-rows x 16 bytes along
// M/N; K-direction stride 128 B (LBO), M/N-direction stride (K/8)*128 B (SBO)
template <int N>
__global__ void probe8mn(float* out) {
  constexpr int KK = 128;
  __shared__ __align__(1024) uint8_t as[128 * KK];
  __shared__ __align__(1024) uint8_t bs[N * KK];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) tmem_alloc(&tbase, 256);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  for (int i = tid; i < 128 * KK; i += 128) {
    const int m = i / KK, k = i % KK;
    as[(((m >> 4) * (KK / 8) + (k >> 3)) * 8 + (k & 7)) * 16 + (m & 15)] = to_e4m3(a8(m, k));
  }
  for (int i = tid; i < N * KK; i += 128) {
    const int n = i / KK, k = i % KK;
    bs[(((n >> 4) * (KK / 8) + (k >> 3)) * 8 + (k & 7)) * 16 + (n & 15)] = to_e4m3(b8(n, k));
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  const uint32_t id = (1u << 4) | (1u << 15) | (1u << 16) | (static_cast<uint32_t>(N >> 3) << 17) | (128u >> 4 << 24);
  if (warp == 0) {
    if (elect_one()) {
      for (int ks = 0; ks < KK / 32; ++ks) {  // K = 32 per MMA: four 8-row core matrices along K
        const uint64_t a = umma_desc(smem_u32(as) + ks * 4 * 128, 128, (KK / 8) * 128);
        const uint64_t b = umma_desc(smem_u32(bs) + ks * 4 * 128, 128, (KK / 8) * 128);
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n}\n" ::"r"(tm + 128),
            "l"(a), "l"(b), "r"(id), "r"(ks > 0 ? 1u : 0u)
            : "memory");
      }
      umma_commit(&bar);
    }
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int n0 = 0; n0 < N; n0 += 32) {
    float v[32];
    tmem_ld32(tm + (static_cast<uint32_t>(warp * 32) << 16) + 128 + n0, v);
    for (int n = 0; n < 32; ++n) out[tid * N + n0 + n] = v[n];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 256);
}
template <int N>
int run8mn() {
  float* d;
  cudaMalloc(&d, 128 * N * 4);
  probe8mn<N><<<1, 128>>>(d);
  if (cudaDeviceSynchronize() != cudaSuccess) {
    printf("f8 MN-major test N=%d: CUDA error\n", N);
    return 1;
  }
  float h[128 * N];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double err = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      double r = 0;
      for (int k = 0; k < 128; ++k) r += static_cast<double>(a8(m, k)) * b8(n, k);
      err = fmax(err, fabs(r - h[m * N + n]));
    }
  printf("f8f6f4 e4m3 MN-major A and B N=%d: max |err| = %g (D[0][0..1] = %g %g)\n", N, err, h[0], h[1]);
  cudaFree(d);
  return err > 1e-3;
}

int main() {
  int bad = 0;
  bad += run<16>(2);
  bad += run<32>(2);
  bad += run<16>(0);
  bad += run<32>(0);
  bad += run<16>(1);
  bad += run<32>(1);
  bad += run8<32>();
  bad += run8<64>();
  bad += run8mn<32>();
  bad += run8mn<64>();
  printf(bad ? "PROBE FAILED\n" : "PROBE OK\n");
  return bad;
}
