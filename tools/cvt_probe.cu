// Throughput of the FP8 / FP4 widening converts (F2FP unpack) and f16x2 math
// per SM sub-partition: W warps per SMSP, 256 independent converts per thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/cvt_probe.cu -o tools/cvt_probe
#include <cstdio>
#include <cstdint>

template <int OP>
__global__ void k(uint32_t seed, uint32_t* out, unsigned long long* cyc) {
  uint32_t a[8];
  for (int i = 0; i < 8; ++i) a[i] = seed * (threadIdx.x + 7 * i + 1);
  __syncthreads();
  const unsigned long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < 32; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      uint32_t r;
      if constexpr (OP == 0) {
        asm volatile("{\n.reg .b16 x, y;\nmov.b32 {x, y}, %1;\ncvt.rn.f16x2.e4m3x2 %0, x;\n}" : "=r"(r) : "r"(a[i]));
      } else if constexpr (OP == 1) {
        asm volatile("{\n.reg .b8 b0, b1, b2, b3;\nmov.b32 {b0, b1, b2, b3}, %1;\ncvt.rn.f16x2.e2m1x2 %0, b0;\n}" : "=r"(r) : "r"(a[i]));
      } else if constexpr (OP == 2) {
        asm volatile("mul.rn.f16x2 %0, %1, %1;" : "=r"(r) : "r"(a[i]));
      } else {
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %1;" : "=r"(r) : "f"(__uint_as_float(a[i])));
      }
      a[i] = r ^ it;
    }
  }
  const unsigned long long t1 = clock64();
  uint32_t x = 0;
  for (int i = 0; i < 8; ++i) x ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  uint32_t* o;
  unsigned long long* c;
  cudaMalloc(&o, 1 << 20);
  cudaMalloc(&c, 1024);
  const char* names[4] = {"cvt e4m3x2->f16x2", "cvt e2m1x2->f16x2", "mul.f16x2", "cvt f32x2->f16x2"};
  for (int op = 0; op < 4; ++op)
    for (int w : {4, 16}) {
      void (*f)(uint32_t, uint32_t*, unsigned long long*) = op == 0 ? k<0> : op == 1 ? k<1> : op == 2 ? k<2> : k<3>;
      f<<<1, 32 * w>>>(3u, o, c);
      unsigned long long h;
      cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
      printf("%-20s %2d warps/SM: %5.2f cycles per warp-instruction per SMSP\n", names[op], w,
             double(h) / (32 * 8) / (w / 4));
    }
  return 0;
}
