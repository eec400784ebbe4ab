// Test-only probe of the tcgen05 / TMA operand layouts used by the attention kernels.
//   s = a b^T          (SS MMA, both operands K-major: the QK^T shape)
//   o = bf16(s) v      (TS MMA, A from TMEM, B MN-major: the PV shape)
//   y = b^T v          (SS MMA, A MN-major, B MN-major: the dS^T Q / dS K shapes)
// Built into tests/csrc/libsa_probe.so (test infrastructure, not the product library).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <string>

#include "common.cuh"

namespace sa {
namespace {
thread_local std::string g_probe_err;

int probe_check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    g_probe_err = std::string(what) + ": " + cudaGetErrorString(e);
    return -static_cast<int>(e);
  }
  return 0;
}

// 2-D bf16 [rows, cols] map, box (64 x box_rows), SW128.
int make_tmap_2d(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int32_t box_rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess || q != cudaDriverEntryPointSuccess) {
      g_probe_err = "cuTensorMapEncodeTiled unavailable";
      return 1;
    }
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  cuuint64_t sizes[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), sizes,
                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    g_probe_err = "cuTensorMapEncodeTiled(2d) failed";
    return 1;
  }
  return 0;
}
}  // namespace
}  // namespace sa

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
  return probe_check_launch("probe_kernel");
}

}  // namespace sa

// ---------------------------------------------------------------------------------------
// Test-only probe of the CTA-pair (cta_group::2) primitives the 2-CTA kernels rely on.
//   s  = a b^T        (SS, M=256 across the pair: CTA r holds a rows [128r,128r+128) and
//                      b rows [64r,64r+64) -- B split by N)
//   o  = bf16(s) v    (TS: P from each CTA's TMEM; v columns [64r,64r+64) in CTA r)
//   s2 = a b^T with A read from TMEM (the operand staged by the threads)
namespace sa {
namespace {

SA_DEV void tma_load_2d_pair(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)),
        "r"(map_to_rank(smem_u32(bar), 0)), "r"(c0), "r"(c1)
      : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
probe_pair_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                  const __grid_constant__ CUtensorMap tv, float* s_out, float* o_out, float* s2_out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa_ = smem;                  // 2 panels x 128 rows (32 KB)
  uint8_t* sb = smem + 2 * kPanel;      // 2 panels x 64 rows (16 KB)
  uint8_t* sv = smem + 3 * kPanel;      // 1 panel x 128 rows (16 KB)
  __shared__ uint64_t bar_load, bar_mma, bar_p;
  __shared__ uint32_t tmem_base_s;
  const uint32_t tid = threadIdx.x, warp = warp_id(), rank = cluster_rank();
  if (warp == 0) tmem_alloc2<512>(&tmem_base_s);
  if (tid == 32) {
    mbar_init(&bar_load, 1);
    mbar_init(&bar_mma, 1);
    mbar_init(&bar_p, 2);
    fence_barrier_init();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tbase = tmem_base_s;
  if (tid == 0) {
    if (rank == 0) mbar_arrive_expect_tx(&bar_load, 2 * 4 * kPanel);
    for (int pn = 0; pn < 2; pn++) {
      tma_load_2d_pair(sa_ + pn * kPanel, &ta, &bar_load, 64 * pn, 128 * rank);
      tma_load_2d_pair(sb + pn * (kPanel / 2), &tb, &bar_load, 64 * pn, 64 * rank);
    }
    tma_load_2d_pair(sv, &tv, &bar_load, 64 * rank, 0);
  }
  constexpr uint32_t hi = sdesc_hi(1024);
  if (rank == 0 && tid == 0) {
    mbar_wait(&bar_load, 0);
    tc_fence_after();
    const uint32_t id = idesc_bf16(256, 128, 0, 0);
    for (uint32_t kk = 0; kk < 8; kk++) {
      mma2_ss(tbase, sdesc_lo(smem_u32(sa_) + (kk >> 2) * kPanel + (kk & 3) * 32, 16), hi,
              sdesc_lo(smem_u32(sb) + (kk >> 2) * (kPanel / 2) + (kk & 3) * 32, 16), hi, id, kk > 0);
    }
    mma2_commit_both(&bar_mma);
  }
  mbar_wait(&bar_mma, 0);
  tc_fence_after();
  const uint32_t row = tid, lane_base = (warp * 32) << 16;
  const uint32_t grow = rank * 128 + row;
  uint32_t r[32];
  for (uint32_t ch = 0; ch < 4; ch++) {
    SA_TMEM_LD32(tbase + lane_base + ch * 32, r);
    tmem_ld_wait();
    uint32_t pk[16];
    for (int i = 0; i < 32; i++) s_out[grow * 128 + ch * 32 + i] = __uint_as_float(r[i]);
    for (int i = 0; i < 16; i++) pk[i] = pack_bf16(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
    SA_TMEM_ST16(tbase + lane_base + 256 + ch * 16, pk);
  }
  // stage this row of a (bf16, 128 K) into TMEM cols [384, 448) as an A operand
  for (uint32_t pn = 0; pn < 2; pn++) {
    uint32_t q[32];
    for (uint32_t cidx = 0; cidx < 8; cidx++) {
      const uint4 w = *reinterpret_cast<const uint4*>(sa_ + pn * kPanel + sw128_off(row, cidx));
      q[4 * cidx] = w.x;
      q[4 * cidx + 1] = w.y;
      q[4 * cidx + 2] = w.z;
      q[4 * cidx + 3] = w.w;
    }
    SA_TMEM_ST32(tbase + lane_base + 384 + pn * 32, q);
  }
  tmem_st_wait();
  tc_fence_before();
  __syncthreads();
  if (tid == 0) mbar_arrive_cluster(map_to_rank(smem_u32(&bar_p), 0));
  if (rank == 0 && tid == 0) {
    mbar_wait(&bar_p, 0);
    tc_fence_after();
    const uint32_t id_pv = idesc_bf16(256, 128, 0, 1);
    for (uint32_t kk = 0; kk < 8; kk++)
      mma2_ts(tbase + 128, tbase + 256 + kk * 8, sdesc_lo(smem_u32(sv) + kk * 2048, kPanel), hi,
              id_pv, kk > 0);
    const uint32_t id = idesc_bf16(256, 128, 0, 0);
    for (uint32_t kk = 0; kk < 8; kk++)
      mma2_ts(tbase, tbase + 384 + kk * 8,
              sdesc_lo(smem_u32(sb) + (kk >> 2) * (kPanel / 2) + (kk & 3) * 32, 16), hi, id, kk > 0);
    mma2_commit_both(&bar_mma);
  }
  mbar_wait(&bar_mma, 1);
  tc_fence_after();
  for (uint32_t ch = 0; ch < 4; ch++) {
    SA_TMEM_LD32(tbase + lane_base + 128 + ch * 32, r);
    tmem_ld_wait();
    for (int i = 0; i < 32; i++) o_out[grow * 128 + ch * 32 + i] = __uint_as_float(r[i]);
    SA_TMEM_LD32(tbase + lane_base + ch * 32, r);
    tmem_ld_wait();
    for (int i = 0; i < 32; i++) s2_out[grow * 128 + ch * 32 + i] = __uint_as_float(r[i]);
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 0) tmem_dealloc2<512>(tbase);
}

}  // namespace

int launch_probe_pair(const void* a, const void* b, const void* v, float* s, float* o, float* s2,
                      cudaStream_t st) {
  CUtensorMap ta, tb, tv;
  if (int r = make_tmap_2d(&ta, a, 256, 128, 128)) return r;
  if (int r = make_tmap_2d(&tb, b, 128, 128, 64)) return r;
  if (int r = make_tmap_2d(&tv, v, 128, 128, 128)) return r;
  const int smem = 4 * kPanel + 1024;
  cudaFuncSetAttribute(probe_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe_pair_kernel<<<2, 128, smem, st>>>(ta, tb, tv, s, o, s2);
  return probe_check_launch("probe_pair_kernel");
}

}  // namespace sa

// ---------------------------------------------------------------------------------------
extern "C" {
const char* sa_probe_last_error(void) { return sa::g_probe_err.c_str(); }

int sa_probe_umma(const void* a, const void* b, const void* v, float* s, float* o, float* y,
                  void* stream) {
  if (!a || !b || !v || !s || !o || !y) return 1;
  return sa::launch_probe(a, b, v, s, o, y, static_cast<cudaStream_t>(stream));
}

int sa_probe_pair(const void* a, const void* b, const void* v, float* s, float* o, float* s2,
                  void* stream) {
  if (!a || !b || !v || !s || !o || !s2) return 1;
  return sa::launch_probe_pair(a, b, v, s, o, s2, static_cast<cudaStream_t>(stream));
}
}  // extern "C"
