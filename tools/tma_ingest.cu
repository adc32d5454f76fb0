// Microbenchmark: per-SM cp.async.bulk ingest from an L2-resident buffer vs
// bytes in flight (one CTA per SM, one producer thread, mbarrier ring).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const uint8_t* src, size_t src_bytes, int chunk, int slots, int iters, unsigned long long* sink) {
  extern __shared__ __align__(128) uint8_t smem_all[];
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint8_t* sm = smem_all + (size_t)w * (slots * chunk + 128);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + slots * chunk);
  if ((threadIdx.x & 31) == 0) {
    for (int s = 0; s < slots; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if ((threadIdx.x & 31) != 0) return;
  size_t off = ((size_t)blockIdx.x * 7919 + w * 104729) * 128 % src_bytes;
  unsigned long long acc = 0;
  for (int i = 0; i < iters + slots; ++i) {
    const int s = i % slots;
    if (i >= slots) {  // wait for the copy issued `slots` iterations ago
      const uint32_t par = ((i / slots) - 1) & 1;
      asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}\n" :: "r"(su(&full[s])), "r"(par));
      acc += sm[s * chunk];
    }
    if (i < iters) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su(&full[s])), "r"(chunk));
      off = (off + chunk * 13) % (src_bytes - chunk);
      off &= ~(size_t)127;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(su(sm + s * chunk)), "l"(src + off), "r"(chunk), "r"(su(&full[s])) : "memory");
    }
  }
  sink[blockIdx.x] = acc;
}
// lanes 0..L-1 of one warp each copy chunk/L bytes of the same slot in one (converged) instruction
__global__ void kl(const uint8_t* src, size_t src_bytes, int chunk, int slots, int iters, int L, unsigned long long* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + slots * chunk);
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < slots; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  size_t off = (size_t)blockIdx.x * 7919 * 128 % src_bytes;
  unsigned long long acc = 0;
  const int part = chunk / L;
  for (int i = 0; i < iters + slots; ++i) {
    const int s = i % slots;
    if (i >= slots) {
      const uint32_t par = ((i / slots) - 1) & 1;
      asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}\n" :: "r"(su(&full[s])), "r"(par));
      acc += sm[s * chunk];
    }
    if (i < iters) {
      off = (off + chunk * 13) % (src_bytes - chunk);
      off &= ~(size_t)127;
      if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su(&full[s])), "r"(chunk));
      __syncwarp();
      if (lane < L)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(su(sm + s * chunk + lane * part)), "l"(src + off + lane * part), "r"(part), "r"(su(&full[s])) : "memory");
      __syncwarp();
    }
  }
  if (lane == 0) sink[blockIdx.x] = acc;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  size_t bytes = 64u << 20;  // L2-resident
  uint8_t* src; cudaMalloc(&src, bytes); cudaMemset(src, 1, bytes);
  unsigned long long* sink; cudaMalloc(&sink, sms * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  struct C { int chunk, slots, warps; };
  C cs[] = {{4096, 8, 1}, {8192, 8, 1}, {16384, 4, 1}, {32768, 4, 1}, {65536, 3, 1}, {98304, 2, 1},
            {16384, 4, 2}, {16384, 3, 4}, {8192, 4, 4}, {32768, 3, 2}, {4096, 4, 8}};
  for (auto c : cs) {
    size_t per = (size_t)c.chunk * c.slots + 128, smem = per * c.warps;
    if (smem > 227 * 1024) continue;
    int iters = (int)(200000000ll / c.chunk / c.warps / sms * 10);
    k<<<sms, 32 * c.warps, smem>>>(src, bytes, c.chunk, c.slots, 20, sink);
    cudaEventRecord(a);
    k<<<sms, 32 * c.warps, smem>>>(src, bytes, c.chunk, c.slots, iters, sink);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double gbs = (double)c.chunk * iters * c.warps * sms / (ms * 1e-3) / 1e9;
    printf("chunk %6d x %d slots x %d issuers: %8.1f GB/s total, %6.1f GB/s per SM, %5.0f ns per copy per SM\n",
           c.chunk, c.slots, c.warps, gbs, gbs / sms, c.chunk / (gbs / sms));
  }
  cudaFuncSetAttribute(kl, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  for (int L : {1, 2, 4, 8}) for (int chunk : {16384, 32768}) {
    int slots = 3; size_t smem = (size_t)chunk * slots + 128;
    int iters = (int)(200000000ll / chunk / sms * 10);
    kl<<<sms, 32, smem>>>(src, bytes, chunk, slots, 20, L, sink);
    cudaEventRecord(a);
    kl<<<sms, 32, smem>>>(src, bytes, chunk, slots, iters, L, sink);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double gbs = (double)chunk * iters * sms / (ms * 1e-3) / 1e9;
    printf("one warp, %d lanes x %6d B per %6d-B slot: %8.1f GB/s total, %6.1f GB/s per SM\n", L, chunk / L, chunk, gbs, gbs / sms);
  }
  cudaError_t e = cudaGetLastError(); if (e) printf("err %s\n", cudaGetErrorString(e));
  return 0;
}
