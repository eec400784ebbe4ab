// HBM-bound kernels: stripe permute (K1), bwd preprocess (K4), casts / state fill.
#include "../../include/striped_attn.h"
#include "common.cuh"
#include "internal.h"

namespace sa {
namespace {

constexpr int kNumSMs = 148;

// K1.  Layout.partition / Layout.gather (layout.py:81-117) as a row gather.
// Each warp moves whole rows; 16-byte vectors when the row allows it.
__device__ __forceinline__ int64_t global_row(int64_t d, int64_t x, int64_t c, int64_t n_dev,
                                              int scheme) {
  return scheme == SA_SCHEME_STRIPED ? d + x * n_dev : d * c + x;  // layout.py:62-70
}

template <typename V>
__global__ void __launch_bounds__(256) permute_kernel(const uint8_t* __restrict__ src,
                                                      uint8_t* __restrict__ dst, int64_t rows,
                                                      int64_t c, int64_t n_dev, int64_t row_vecs,
                                                      int scheme, int direction, int device) {
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int lane = threadIdx.x & 31;
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows;
       r += warps) {
    // r indexes the permuted (device-major) side: device d, local x.
    const int64_t d = device >= 0 ? device : r / c;
    const int64_t x = device >= 0 ? r : r % c;
    const int64_t g = global_row(d, x, c, n_dev, scheme);
    const int64_t p = device >= 0 ? x : r;  // row in the shard buffer
    const V* s;
    V* o;
    if (direction == SA_PARTITION) {
      s = reinterpret_cast<const V*>(src) + g * row_vecs;
      o = reinterpret_cast<V*>(dst) + p * row_vecs;
    } else {
      s = reinterpret_cast<const V*>(src) + p * row_vecs;
      o = reinterpret_cast<V*>(dst) + g * row_vecs;
    }
    int64_t i = lane;
    for (; i + 96 < row_vecs; i += 128) {  // 4 loads in flight per lane
      V a = s[i], b = s[i + 32], cc = s[i + 64], e = s[i + 96];
      o[i] = a;
      o[i + 32] = b;
      o[i + 64] = cc;
      o[i + 96] = e;
    }
    for (; i < row_vecs; i += 32) o[i] = s[i];
  }
}

__global__ void cast_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                            int64_t n) {
  int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 8;
  for (; i + 8 <= n; i += stride) {
    float4 a = *reinterpret_cast<const float4*>(src + i);
    float4 b = *reinterpret_cast<const float4*>(src + i + 4);
    uint4 w;
    w.x = pack_bf16(a.x, a.y);
    w.y = pack_bf16(a.z, a.w);
    w.z = pack_bf16(b.x, b.y);
    w.w = pack_bf16(b.z, b.w);
    *reinterpret_cast<uint4*>(dst + i) = w;
  }
}

__global__ void cast_scalar_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                                   int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    dst[i] = __float2bfloat16_rn(src[i]);
}

__global__ void fill_state_kernel(float* __restrict__ o_acc, float* __restrict__ lse, int64_t n_o,
                                  int64_t n_l) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_o; i += stride) o_acc[i] = 0.f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_l; i += stride)
    lse[i] = -INFINITY;
}

// K4.  dsum[h, x] = <dout[x,h,:], out[x,h,:]>; one warp per (x, h) row; also zero dq_acc.
template <int D>
__global__ void __launch_bounds__(256) bwd_pre_kernel(const __nv_bfloat16* __restrict__ out,
                                                      const __nv_bfloat16* __restrict__ dout,
                                                      float* __restrict__ dsum,
                                                      float* __restrict__ dq_acc, int64_t c,
                                                      int hq) {
  const int64_t rows = c * hq;
  const int64_t warps = (int64_t)gridDim.x * 8;
  const int lane = threadIdx.x & 31;
  for (int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); r < rows; r += warps) {
    float acc = 0.f;
    constexpr int kPer = D / 32;  // 2 or 4 bf16 per lane
    const __nv_bfloat16* a = out + r * D + lane * kPer;
    const __nv_bfloat16* b = dout + r * D + lane * kPer;
#pragma unroll
    for (int i = 0; i < kPer; i += 2) {
      float2 x = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(a + i));
      float2 y = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(b + i));
      acc += x.x * y.x + x.y * y.y;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      const int64_t x = r / hq, h = r % hq;
      dsum[h * c + x] = acc;
    }
    float* z = dq_acc + r * D + lane * kPer;
#pragma unroll
    for (int i = 0; i < kPer; i++) z[i] = 0.f;
  }
}

int grid_for(int64_t work, int per_block) {
  int64_t g = (work + per_block - 1) / per_block;
  int64_t cap = int64_t(kNumSMs) * 16;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

}  // namespace

int launch_permute(const void* src, void* dst, int64_t n_seq, int32_t n_dev, int64_t row_bytes,
                   int32_t scheme, int32_t direction, int32_t device, cudaStream_t st) {
  const int64_t c = n_seq / n_dev;
  const int64_t rows = device >= 0 ? c : n_seq;
  const int grid = grid_for(rows, 8);
  const auto* s = static_cast<const uint8_t*>(src);
  auto* o = static_cast<uint8_t*>(dst);
  const bool v16 = row_bytes % 16 == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
  if (v16)
    permute_kernel<uint4><<<grid, 256, 0, st>>>(s, o, rows, c, n_dev, row_bytes / 16, scheme,
                                                direction, device);
  else
    permute_kernel<uint32_t><<<grid, 256, 0, st>>>(s, o, rows, c, n_dev, row_bytes / 4, scheme,
                                                   direction, device);
  return check_launch("permute_kernel");
}

int launch_cast(const float* src, void* dst, int64_t n, cudaStream_t st) {
  const bool vec = (reinterpret_cast<uintptr_t>(src) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
  const int64_t n8 = vec ? n - n % 8 : 0;
  if (n8) cast_kernel<<<grid_for(n8 / 8, 256), 256, 0, st>>>(src, static_cast<__nv_bfloat16*>(dst), n8);
  if (n > n8)
    cast_scalar_kernel<<<grid_for(n - n8, 256), 256, 0, st>>>(
        src + n8, static_cast<__nv_bfloat16*>(dst) + n8, n - n8);
  return check_launch("cast_kernel");
}

int launch_fill_state(float* o_acc, float* lse, int64_t c, int32_t hq, int32_t d, cudaStream_t st) {
  fill_state_kernel<<<grid_for(c * hq * d, 256), 256, 0, st>>>(o_acc, lse, c * hq * d, c * hq);
  return check_launch("fill_state_kernel");
}

int launch_bwd_pre(const void* out, const void* dout, float* dsum, float* dq_acc, int64_t c,
                   int32_t hq, int32_t d, cudaStream_t st) {
  const int grid = grid_for(c * hq, 8);
  const auto* o = static_cast<const __nv_bfloat16*>(out);
  const auto* g = static_cast<const __nv_bfloat16*>(dout);
  if (d == 128)
    bwd_pre_kernel<128><<<grid, 256, 0, st>>>(o, g, dsum, dq_acc, c, hq);
  else
    bwd_pre_kernel<64><<<grid, 256, 0, st>>>(o, g, dsum, dq_acc, c, hq);
  return check_launch("bwd_pre_kernel");
}

}  // namespace sa
