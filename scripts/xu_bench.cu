// Throughput micro-benchmark of the special-function / conversion paths the softmax
// uses (MUFU.EX2, F2FP.BF16 pack, integer RNE pack, polynomial exp2 on FMA).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o xu_bench scripts/xu_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_cvt(float a, float b) {
  uint32_t r;
  asm volatile("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ uint32_t pack_int(float a, float b) {
  uint32_t ua = __float_as_uint(a), ub = __float_as_uint(b);
  ua += 0x7FFFu + ((ua >> 16) & 1u);
  ub += 0x7FFFu + ((ub >> 16) & 1u);
  return __byte_perm(ua, ub, 0x7632);
}
// 2^x for x <= 0 on the FMA pipe: Cody-Waite split + degree-3 minimax polynomial.
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -127.f);
  const float fl = floorf(x);
  const float f = x - fl;
  float p = fmaf(f, 0.0555041086648216f, 0.2402264923172690f);
  p = fmaf(p, f, 0.6931471805599453f);
  p = fmaf(p, f, 1.0f);
  return __uint_as_float(__float_as_uint(p) + ((int)fl << 23));
}

template <int MODE>
__global__ void k(float* out, int iters) {
  float a[8];
  for (int i = 0; i < 8; i++) a[i] = -(threadIdx.x + i) * 1e-3f;
  uint32_t acc = 0;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      if (MODE == 0) a[i] = ex2(a[i]) - 1.0f;
      if (MODE == 1) acc ^= pack_cvt(a[i], a[(i + 1) & 7]), a[i] += 1e-7f;
      if (MODE == 2) acc ^= pack_int(a[i], a[(i + 1) & 7]), a[i] += 1e-7f;
      if (MODE == 3) a[i] = ex2_poly(a[i]) - 1.0f;
      if (MODE == 4) a[i] = fmaf(a[i], 0.999f, -1e-3f);
    }
  }
  float s = 0;
  for (int i = 0; i < 8; i++) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + (float)acc;
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 8 * 1024 * sizeof(float));
  const char* names[] = {"MUFU.EX2", "cvt.rn.bf16x2 (F2FP)", "int RNE pack", "poly exp2 (FMA)", "FFMA"};
  const double per_it[] = {8, 8, 8, 8, 8};  // ops per thread per iteration
  for (int mode = 0; mode < 5; mode++) {
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
    const double ops = (double)blocks * threads * iters * per_it[mode];
    const double cycles = ms * 1e-3 * clk * 1e3;
    printf("%-24s %8.3f ms  %7.2f elem-ops/clk/SM (at %d MHz nominal)\n", names[mode], ms,
           ops / cycles / 148, clk / 1000);
  }
  return 0;
}
