// Throughput micro-benchmark of the special-function / conversion paths the softmax uses:
// MUFU.EX2 (f32, f16x2, bf16x2), F2FP.BF16 pack, polynomial exp2 on the FMA pipe.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/xu_bench scripts/xu_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t ex2_bf16x2(uint32_t x) {
  uint32_t y;
  asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint32_t ex2_f16x2(uint32_t x) {
  uint32_t y;
  asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_cvt(float a, float b) {
  uint32_t r;
  asm volatile("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(r) : "f"(a), "f"(b));
  return r;
}
// 2^x on the FMA pipe: round-to-nearest split via the 1.5*2^23 trick, degree-3 poly on
// [-0.5, 0.5], exponent added with an integer multiply-add.
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -126.f);
  const float t = x + 12582912.f;
  const float f = x - (t - 12582912.f);
  float p = fmaf(f, 0.05550410866f, 0.2402265070f);
  p = fmaf(p, f, 0.6931471806f);
  p = fmaf(p, f, 1.0f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

template <int MODE>
__global__ void k(float* out, int iters) {
  float a[8];
  uint32_t u[8];
  for (int i = 0; i < 8; i++) {
    a[i] = -(threadIdx.x + i) * 1e-3f;
    u[i] = 0x3c003c00u + threadIdx.x + i;
  }
  uint32_t acc = 0;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      if (MODE == 0) a[i] = ex2(a[i]) - 1.0f;
      if (MODE == 1) u[i] = ex2_bf16x2(u[i]) ^ 0x80008000u;
      if (MODE == 2) u[i] = ex2_f16x2(u[i]) ^ 0x80008000u;
      if (MODE == 3) { uint32_t r = pack_cvt(a[i], a[(i + 3) & 7]); a[i] = __uint_as_float(r ^ acc); acc += r; }
      if (MODE == 4) a[i] = ex2_poly(a[i]) - 1.0f;
      if (MODE == 5) a[i] = fmaf(a[i], 0.999f, -1e-3f);
    }
  }
  float s = 0;
  for (int i = 0; i < 8; i++) s += a[i] + (float)u[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + (float)acc;
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 8 * 1024 * sizeof(float));
  const char* names[] = {"MUFU.EX2 f32", "ex2 bf16x2 (2 elem/op)", "ex2 f16x2 (2 elem/op)",
                         "cvt.rn.bf16x2.f32", "poly exp2 (FMA pipe)", "FFMA"};
  for (int mode = 0; mode < 6; mode++) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096, blocks = 148 * 4, threads = 512;
    auto launch = [&] {
      if (mode == 0) k<0><<<blocks, threads>>>(out, iters);
      if (mode == 1) k<1><<<blocks, threads>>>(out, iters);
      if (mode == 2) k<2><<<blocks, threads>>>(out, iters);
      if (mode == 3) k<3><<<blocks, threads>>>(out, iters);
      if (mode == 4) k<4><<<blocks, threads>>>(out, iters);
      if (mode == 5) k<5><<<blocks, threads>>>(out, iters);
    };
    launch();
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double ops = (double)blocks * threads * iters * 8;
    const double cycles = ms * 1e-3 * clk * 1e3;
    printf("%-26s %8.3f ms  %7.2f instr/clk/SM (x lanes; at %d MHz nominal)\n", names[mode], ms,
           ops / cycles / 148, clk / 1000);
  }
  return 0;
}
