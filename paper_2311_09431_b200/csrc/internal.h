// Host-side internals shared by the .cu translation units (not part of the ABI).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <string>

#ifndef SA_PERF_TRACE
#define SA_PERF_TRACE 0  // see common.cuh
#endif

namespace sa {

void set_error(const std::string& msg);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per device: set it once per device
// the kernel is launched on (bit d of *mask), thread-safely.  Returns 0 or -(cudaError).
template <typename Kernel>
int set_smem_attr_once(Kernel kernel, int bytes, unsigned long long* mask) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  const unsigned long long bit = 1ull << (dev & 63);
  if (__atomic_load_n(mask, __ATOMIC_ACQUIRE) & bit) return 0;
  const cudaError_t e =
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) {
    set_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    return -static_cast<int>(e);
  }
  __atomic_fetch_or(mask, bit, __ATOMIC_RELEASE);
  return 0;
}
int fail_arg(const std::string& msg);             // returns 1
int check_launch(const char* what);               // 0 or -(cudaError)
void count_launch(int n = 1);

// 3-D tensor map over a token-major bf16 tensor [rows, heads, dim] with a
// (64 x 1 x box_rows) box and 128-byte swizzle (one smem "panel" per box).
int make_tmap_rows(CUtensorMap* map, const void* base, int64_t rows, int32_t heads, int32_t dim,
                   int32_t box_rows);
// fp32 [rows, heads, dim] map, box (32 x 1 x box_rows), SW128 (accumulator TMA reduce-add).
int make_tmap_rows_f32(CUtensorMap* map, const void* base, int64_t rows, int32_t heads,
                       int32_t dim, int32_t box_rows);

int launch_permute(const void* src, void* dst, int64_t n_seq, int32_t n_dev, int64_t row_bytes,
                   int32_t scheme, int32_t direction, int32_t device, cudaStream_t st);
bool fwd_pair_enabled(int32_t d);
int launch_fwd_pair(const void* q, const void* k, const void* v, float* o_acc, float* lse,
                    void* out, int64_t c, int32_t hq, int32_t hkv, float scale, int32_t kind,
                    int32_t first, int32_t last, int64_t* tiles, cudaStream_t st);
int launch_fwd(const void* q, const void* k, const void* v, float* o_acc, float* lse, void* out,
               int64_t c, int32_t hq, int32_t hkv, int32_t d, float scale, int32_t kind,
               int32_t first, int32_t last, int64_t* tiles, cudaStream_t st);
int launch_bwd_pre(const void* out, const void* dout, float* dsum, float* dq_acc, int64_t c,
                   int32_t hq, int32_t d, cudaStream_t st);
// dk_out / dv_out non-null: "final" mode, dK / dV written as bf16 (dk / dv unused)
int launch_bwd(const void* q, const void* k, const void* v, const void* dout, const float* lse,
               const float* dsum, float* dq, float* dk, float* dv, int64_t c, int32_t hq,
               int32_t hkv, int32_t d, float scale, int32_t kind, cudaStream_t st,
               void* dk_out = nullptr, void* dv_out = nullptr, int32_t kv_tile_begin = 0,
               int32_t kv_tile_end = -1, int32_t* dq_sem = nullptr);
int launch_cast(const float* src, void* dst, int64_t n, cudaStream_t st);
int launch_fill_state(float* o_acc, float* lse, int64_t c, int32_t hq, int32_t d, cudaStream_t st);

}  // namespace sa
