// Issue-rate micro-benchmark of the tcgen05.mma shapes the attention kernels use.
// Reports clocks per "unit" = one 128x128x128 product per SM (512 clk at the nominal
// dense bf16 rate).  Operand contents are irrelevant (zeros).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/umma_bench scripts/umma_bench.cu
#include <cstdio>
#include <cstdlib>
#include "../paper_2311_09431_b200/csrc/common.cuh"

using namespace sa;

__device__ int g_reps = 64;

// variant: bit0 = A from TMEM, bit1 = B MN-major, N in template
template <bool kPair, bool kTS, bool kBmn, int N>
__global__ void bench_kernel(long long* out, int mode, const uint8_t* gsrc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase_s;
  const uint32_t warp = warp_id();
  // mode bit0: random operands (else zeros); bit1: warps 1-3 stream TMEM loads meanwhile
  for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x) {
    uint4 w = make_uint4(0, 0, 0, 0);
    if (mode & 1) {  // random bf16 in +-[0.5, 2): random sign, exponent 126/127, mantissa
      uint32_t z = (i + 1) * 2654435761u ^ (blockIdx.x * 40503u);
      uint32_t* wp = &w.x;
      for (int k = 0; k < 4; k++) {
        z ^= z << 13; z ^= z >> 17; z ^= z << 5;
        const uint32_t m = z & 0x80FF80FFu;  // sign + low exponent bit + 7 mantissa bits
        wp[k] = 0x3F003F00u | m;
      }
    }
    reinterpret_cast<uint4*>(smem)[i] = w;
  }
  __shared__ volatile int done;
  if (threadIdx.x == 0) done = 0;
  if (warp == 0) {
    if constexpr (kPair) tmem_alloc2<512>(&tbase_s); else tmem_alloc<512>(&tbase_s);
  }
  if (threadIdx.x == 32) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  if constexpr (kPair) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tbase_s;
  const uint32_t rank = kPair ? cluster_rank() : 0;
  if ((mode & 1) && warp < 4) {  // realistic (random bf16) A operand in TMEM cols [384, 448)
    uint32_t r[32];
    uint32_t z = (threadIdx.x + 1) * 2654435761u ^ (blockIdx.x * 40503u);
    for (int c = 0; c < 2; c++) {
      for (int k = 0; k < 32; k++) {
        z ^= z << 13; z ^= z >> 17; z ^= z << 5;
        r[k] = 0x3F003F00u | (z & 0x80FF80FFu);
      }
      SA_TMEM_ST32(tbase + ((warp * 32) << 16) + 384 + 32 * c, r);
    }
    tmem_st_wait();
  }
  tc_fence_before();
  if constexpr (kPair) cluster_sync(); else __syncthreads();
  tc_fence_after();
  // per CTA: A 128 rows x 128 K (32 KB), B: N/(kPair?2:1) rows (K-major) or K x N cols (MN)
  const uint32_t sa_ = smem_u32(smem), sb = smem_u32(smem + 32768);
  constexpr uint32_t kM = kPair ? 256 : 128;
  constexpr uint32_t kNc = kPair ? N / 2 : N;  // B extent held per CTA
  const uint32_t id = idesc_bf16(kM, N, (mode & 16) ? 1 : 0, kBmn ? 1 : 0);
  constexpr uint32_t hi = sdesc_hi(1024);
  if (threadIdx.x == 0 && rank == 0) {
    long long t0 = clock64();
    const int kReps = g_reps;
    for (int r = 0; r < kReps; r++) {
      for (int kk = 0; kk < 8; kk++) {
        const uint32_t a = (mode & 16) ? sdesc_lo(sa_ + kk * 2048, 16384)
                                       : sdesc_lo(sa_ + (kk >> 2) * 16384 + (kk & 3) * 32, 16);
        uint32_t b;
        if (kBmn) b = sdesc_lo(sb + kk * 2048, 128 * 128);  // K rows x 64-col panels
        else b = sdesc_lo(sb + (kk >> 2) * (kNc * 128) + (kk & 3) * 32, 16);
        const uint32_t d = tbase;
        if constexpr (kPair) {
          if (kTS) mma2_ts(d, tbase + 256 * 0 + 448 - 64 + kk * 8 - 0, b, hi, id, kk > 0);
          else mma2_ss(d, a, hi, b, hi, id, kk > 0);
        } else {
          if (kTS) mma_ts2(d, tbase + 448 + kk * 8 - 64, b, hi, id, kk > 0);
          else mma_ss2(d, a, hi, b, hi, id, kk > 0);
        }
      }
    }
    if constexpr (kPair) mma2_commit_both(&bar); else mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
    done = 1;
  } else if (kPair && threadIdx.x == 0) {
    mbar_wait(&bar, 0);
    done = 1;
  } else if ((mode & 32) && warp == 1 && (threadIdx.x & 31) == 0) {
    // background TMA-style bulk copies global -> smem (16 KB chunks, 3 in flight)
    __shared__ uint64_t cbar[3];
    for (int i = 0; i < 3; i++) mbar_init(&cbar[i], 1);
    fence_barrier_init();
    uint32_t it = 0;
    while (!done) {
      const int b = it % 3;
      if (it >= 3) mbar_wait(&cbar[b], ((it / 3) - 1) & 1);
      mbar_arrive_expect_tx(&cbar[b], 16384);
      const uint8_t* src = gsrc + (size_t)((blockIdx.x * 7919u + it) % 4096u) * 16384;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(smem + 112 * 1024 + b * 16384)), "l"(src), "r"(16384),
                     "r"(smem_u32(&cbar[b])) : "memory");
      it++;
    }
    for (uint32_t k = it >= 3 ? it - 3 : 0; k < it; k++) mbar_wait(&cbar[k % 3], (k / 3) & 1);
  } else if ((mode & 4) && warp >= 4) {
    // softmax-like TMEM traffic: 128 columns loaded, 64 stored, per pass
    uint32_t r[128];
    float acc = 0.f;
    const uint32_t t = tbase + (((warp & 3) * 32) << 16) + 128 + 128 * ((warp >> 2) & 1);
    while (!done) {
      SA_TMEM_LD32(t + 0, (r + 0));
      SA_TMEM_LD32(t + 32, (r + 32));
      SA_TMEM_LD32(t + 64, (r + 64));
      SA_TMEM_LD32(t + 96, (r + 96));
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 64; i++) r[i] = r[2 * i] ^ r[2 * i + 1];
      SA_TMEM_ST32(t + 0, (r + 0));
      SA_TMEM_ST32(t + 32, (r + 32));
      tmem_st_wait();
      if (mode & 8) __nanosleep(500);
    }
    acc = __uint_as_float(r[5]);
    if (acc == 1234.5f) out[0] = 0;
  } else if ((mode & 2) && warp >= 1) {
    uint32_t r[32];
    float acc = 0.f;
    while (!done) {
      SA_TMEM_LD32(tbase + ((warp * 32) << 16) + 256 + 64 * (warp & 1), r);
      tmem_ld_wait();
      acc += __uint_as_float(r[0]) + __uint_as_float(r[31]);
    }
    if (acc == 1234.5f) out[0] = 0;
  }
  tc_fence_before();
  if constexpr (kPair) cluster_sync(); else __syncthreads();
  if (warp == 0) {
    if constexpr (kPair) tmem_dealloc2<512>(tbase); else tmem_dealloc<512>(tbase);
  }
}

template <bool kPair, bool kTS, bool kBmn, int N>
void run(const char* name, int grid, int mode) {
  long long* d;
  cudaMalloc(&d, grid * sizeof(long long));
  cudaMemset(d, 0, grid * sizeof(long long));
  auto k = bench_kernel<kPair, kTS, kBmn, N>;
  const int smem = 160 * 1024 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(384);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kPair ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  static uint8_t* gsrc = nullptr;
  if (!gsrc) cudaMalloc(&gsrc, (size_t)4096 * 16384);
  cudaLaunchKernelEx(&cfg, k, d, mode, (const uint8_t*)gsrc);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, k, d, mode, (const uint8_t*)gsrc);
  cudaEventRecord(e1);
  cudaError_t e = cudaDeviceSynchronize();
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[296];
  cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < grid; i++) mx = h[i] > mx ? h[i] : mx;
  // units per SM: kReps * (N / 128) (pair: each SM does 128 rows x N)
  int reps = 64;
  cudaMemcpyFromSymbol(&reps, g_reps, sizeof(int));
  const double units = reps * (N / 128.0);
  printf("%-34s grid %3d mode %d: %8.1f clk/unit  %.3f ms  => %.0f MHz  %.0f TF/s (%s)\n", name, grid, mode,
         mx / units, ms, mx / (ms * 1e3), grid * units * 4194304.0 / (ms * 1e9) * (kPair ? 1 : 1), cudaGetErrorString(e));
  cudaFree(d);
}

// Attention-like MMA sequence on a CTA pair: per rep, PV(r) (TS, A = P in buffer r%3,
// D = O) then S (SS, D = buffer (r + shift) % 3).  shift 0 = S overwrites the buffer PV
// just read (the fwd kernel's order).
__global__ void __cluster_dims__(2, 1, 1) seq_kernel(long long* out, int shift, int reps, int commits, int mode) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar, dummy[4], never;
  __shared__ volatile int done;
  __shared__ uint32_t tbase_s;
  const uint32_t warp = warp_id();
  for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x) {
    uint32_t z = (i + 1) * 2654435761u ^ (blockIdx.x * 40503u);
    uint4 w;
    uint32_t* wp = &w.x;
    for (int k = 0; k < 4; k++) {
      z ^= z << 13; z ^= z >> 17; z ^= z << 5;
      wp[k] = 0x3F003F00u | (z & 0x80FF80FFu);
    }
    reinterpret_cast<uint4*>(smem)[i] = w;
  }
  if (warp == 0) tmem_alloc2<512>(&tbase_s);
  if (threadIdx.x == 32) {
    mbar_init(&bar, 1);
    for (int i = 0; i < 4; i++) mbar_init(&dummy[i], (mode & 4) && i == 0 ? 2 : 1 << 19);
    mbar_init(&never, 1);
    done = 0;
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tbase = tbase_s;
  const uint32_t rank = cluster_rank();
  const uint32_t sq = smem_u32(smem), sk = smem_u32(smem + 32768), sv = smem_u32(smem + 65536);
  constexpr uint32_t id_s = idesc_bf16(256, 128, 0, 0), id_o = idesc_bf16(256, 128, 0, 1);
  constexpr uint32_t hi = sdesc_hi(1024);
  if (threadIdx.x == 0 && rank == 0) {
    long long t0 = clock64();
    for (int r = 0; r < reps; r++) {
      for (int kk = 0; kk < 8; kk++)
        mma2_ts(tbase + 384, tbase + 128 * (r % 3) + kk * 8, sdesc_lo(sv + kk * 2048, 16384), hi, id_o, 1);
      for (int c = 0; c < commits; c++) mma2_commit_both(&dummy[c]);
      const uint32_t d = tbase + 128 * ((r + shift) % 3);
      for (int kk = 0; kk < 8; kk++)
        mma2_ss(d, sdesc_lo(sq + (kk >> 2) * 16384 + (kk & 3) * 32, 16), hi,
                sdesc_lo(sk + (kk >> 2) * 8192 + (kk & 3) * 32, 16), hi, id_s, kk > 0);
      for (int c = 0; c < commits; c++) mma2_commit_both(&dummy[2 + c % 2]);
      if (mode & 4) {  // serialise: wait for each rep (latency of PV + S)
        mma2_commit_both(&dummy[0]);
        mbar_wait(&dummy[0], r & 1);
      }
    }
    mma2_commit_both(&bar);
    mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - t0;
    done = 1;
  } else if (threadIdx.x == 0) {
    mbar_wait(&bar, 0);
    done = 1;
  } else if ((mode & 1) && warp >= 1) {  // polling pressure: try_wait on a barrier that never completes
    while (!done) mbar_try_wait(&never, 0);
  } else if (mode & 8) {  // idle warps sleep instead of waiting at the cluster barrier
    while (!done) __nanosleep(1000);
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 0) tmem_dealloc2<512>(tbase);
}

void run_seq(int shift, int reps, int commits, int mode) {
  long long* d;
  const int grid = 148;
  cudaMalloc(&d, grid * sizeof(long long));
  const int smem = 160 * 1024 + 1024;
  cudaFuncSetAttribute(seq_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  seq_kernel<<<grid, 384, smem>>>(d, shift, reps, commits, mode);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < grid; i += 2) mx = h[i] > mx ? h[i] : mx;
  printf("seq PV->S shift %d commits %d mode %d: %8.1f clk per MMA (%s)\n", shift, commits, mode, mx / (2.0 * reps), cudaGetErrorString(e));
  cudaFree(d);
}

int main(int argc, char** argv) {
  int reps = argc > 1 ? atoi(argv[1]) : 64;
  cudaMemcpyToSymbol(g_reps, &reps, sizeof(int));
  // mode bits: 1 random operands, 4 softmax-like TMEM traffic (8 warps), 16 A MN-major,
  // 32 background bulk copies global -> smem
  if (argc > 2) {  // sustained (power-capped) run of the shapes the backward could use
    const int mode = atoi(argv[2]);
    for (int rep = 0; rep < 2; rep++) {
      run<false, false, false, 128>("1cta SS  M128 N128 Bk", 148, mode);
      run<false, false, true, 128>("1cta SS  M128 N128 Bmn", 148, mode);
      run<false, true, false, 128>("1cta TS  M128 N128 Bk", 148, mode);
      run<false, true, true, 128>("1cta TS  M128 N128 Bmn", 148, mode);
      run<false, true, false, 64>("1cta TS  M128 N64 Bk", 148, mode);
      run<true, false, false, 128>("pair SS M256 N128 Bk", 148, mode);
      run<true, true, true, 128>("pair TS M256 N128 Bmn", 148, mode);
    }
    return 0;
  }
  for (int mode : {1, 17, 33, 49, 37}) {
    const int grid = 148;
    run<false, false, false, 128>("1cta SS  M128 N128 Bk", grid, mode);
    run<false, false, true, 128>("1cta SS  M128 N128 Bmn", grid, mode);
    run<false, false, false, 64>("1cta SS  M128 N64 Bk", grid, mode);
    run<false, false, true, 64>("1cta SS  M128 N64 Bmn", grid, mode);
    run<false, true, true, 128>("1cta TS  M128 N128 Bmn", grid, mode);
    run<true, false, false, 128>("pair SS M256 N128 Bk", grid, mode);
    run<true, false, false, 256>("pair SS M256 N256 Bk", grid, mode);
  }
  return 0;
}
