// Test-only probe of the tcgen05 / TMA operand layouts used by the attention kernels.
//   s = a b^T          (SS MMA, both operands K-major: the QK^T shape)
//   o = bf16(s) v      (TS MMA, A from TMEM, B MN-major: the PV shape)
//   y = b^T v          (SS MMA, A MN-major, B MN-major: the dS^T Q / dS K shapes)
#include "common.cuh"
#include "internal.h"

namespace sa {
namespace {

constexpr uint32_t kPanel = 128 * 128;  // one 64-col x 128-row bf16 panel, bytes

__global__ void __launch_bounds__(128, 1)
probe_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
             const __grid_constant__ CUtensorMap tv, float* s_out, float* o_out, float* y_out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa_ = smem;
  uint8_t* sb = smem + 2 * kPanel;
  uint8_t* sv = smem + 4 * kPanel;
  __shared__ uint64_t bar_load, bar_mma;
  __shared__ uint32_t tmem_base_s;

  const uint32_t tid = threadIdx.x, warp = warp_id();
  if (warp == 0) tmem_alloc<512>(&tmem_base_s);
  if (tid == 32) {
    mbar_init(&bar_load, 1);
    mbar_init(&bar_mma, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base_s;

  if (tid == 0) {
    mbar_arrive_expect_tx(&bar_load, 6 * kPanel);
    for (int p = 0; p < 2; p++) {
      tma_load_2d(sa_ + p * kPanel, &ta, &bar_load, 64 * p, 0);
      tma_load_2d(sb + p * kPanel, &tb, &bar_load, 64 * p, 0);
      tma_load_2d(sv + p * kPanel, &tv, &bar_load, 64 * p, 0);
    }
  }
  mbar_wait(&bar_load, 0);

  if (tid == 0) {
    tc_fence_after();
    const uint32_t id = idesc_bf16(128, 128, 0, 0);
    for (uint32_t kk = 0; kk < 8; kk++) {
      const uint32_t off = (kk >> 2) * kPanel + (kk & 3) * 32;
      mma_ss(tbase + 0, sdesc(smem_u32(sa_) + off, 16, 1024), sdesc(smem_u32(sb) + off, 16, 1024),
             id, kk > 0);
    }
    mma_commit(&bar_mma);
  }
  mbar_wait(&bar_mma, 0);
  tc_fence_after();

  const uint32_t row = tid;  // warp w owns TMEM lanes 32w..32w+31
  const uint32_t lane_base = (warp * 32) << 16;
  uint32_t r[32];
  for (uint32_t ch = 0; ch < 4; ch++) {
    SA_TMEM_LD32(tbase + lane_base + ch * 32, r);
    tmem_ld_wait();
    uint32_t pk[16];
    for (int i = 0; i < 32; i++) s_out[row * 128 + ch * 32 + i] = __uint_as_float(r[i]);
    for (int i = 0; i < 16; i++) pk[i] = pack_bf16(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
    SA_TMEM_ST16(tbase + lane_base + 384 + ch * 16, pk);
  }
  tmem_st_wait();
  tc_fence_before();
  __syncthreads();

  if (tid == 0) {
    tc_fence_after();
    const uint32_t id_pv = idesc_bf16(128, 128, 0, 1);
    for (uint32_t kk = 0; kk < 8; kk++)
      mma_ts(tbase + 128, tbase + 384 + kk * 8, sdesc(smem_u32(sv) + kk * 2048, kPanel, 1024), id_pv,
             kk > 0);
    const uint32_t id_tt = idesc_bf16(128, 128, 1, 1);
    for (uint32_t kk = 0; kk < 8; kk++)
      mma_ss(tbase + 256, sdesc(smem_u32(sb) + kk * 2048, kPanel, 1024),
             sdesc(smem_u32(sv) + kk * 2048, kPanel, 1024), id_tt, kk > 0);
    mma_commit(&bar_mma);
  }
  mbar_wait(&bar_mma, 1);
  tc_fence_after();
  for (uint32_t ch = 0; ch < 4; ch++) {
    SA_TMEM_LD32(tbase + lane_base + 128 + ch * 32, r);
    tmem_ld_wait();
    for (int i = 0; i < 32; i++) o_out[row * 128 + ch * 32 + i] = __uint_as_float(r[i]);
    SA_TMEM_LD32(tbase + lane_base + 256 + ch * 32, r);
    tmem_ld_wait();
    for (int i = 0; i < 32; i++) y_out[row * 128 + ch * 32 + i] = __uint_as_float(r[i]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tbase);
}

}  // namespace

int launch_probe(const void* a, const void* b, const void* v, float* s, float* o, float* y,
                 cudaStream_t st) {
  CUtensorMap ta, tb, tv;
  if (int r = make_tmap_2d(&ta, a, 128, 128, 128)) return r;
  if (int r = make_tmap_2d(&tb, b, 128, 128, 128)) return r;
  if (int r = make_tmap_2d(&tv, v, 128, 128, 128)) return r;
  const int smem = 6 * kPanel + 1024;
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe_kernel<<<1, 128, smem, st>>>(ta, tb, tv, s, o, y);
  return check_launch("probe_kernel");
}

}  // namespace sa
