// C ABI entry points (include/striped_attn.h): argument validation + dispatch.
#include "../../include/striped_attn.h"
#include "internal.h"

#include <atomic>
#include <cstdio>
#include <cudaTypedefs.h>
#include <mutex>

namespace sa {

static thread_local std::string g_err;
static std::atomic<int64_t> g_launches{0};

void set_error(const std::string& m) { g_err = m; }
int fail_arg(const std::string& m) {
  g_err = m;
  return 1;
}
void count_launch(int n) { g_launches += n; }
int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    g_err = std::string(what) + ": " + cudaGetErrorString(e);
    return -static_cast<int>(e);
  }
  count_launch();
  return 0;
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

int make_tmap_rows(CUtensorMap* map, const void* base, int64_t rows, int32_t heads, int32_t dim,
                   int32_t box_rows) {
  auto fn = encode_fn();
  if (!fn) return fail_arg("cuTensorMapEncodeTiled unavailable");
  cuuint64_t sizes[3] = {(cuuint64_t)dim, (cuuint64_t)heads, (cuuint64_t)rows};
  cuuint64_t strides[2] = {(cuuint64_t)dim * 2, (cuuint64_t)heads * dim * 2};
  cuuint32_t box[3] = {64, 1, (cuuint32_t)box_rows};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), sizes,
                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[128];
    snprintf(buf, sizeof buf, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return fail_arg(buf);
  }
  return 0;
}

int make_tmap_rows_f32(CUtensorMap* map, const void* base, int64_t rows, int32_t heads,
                       int32_t dim, int32_t box_rows) {
  auto fn = encode_fn();
  if (!fn) return fail_arg("cuTensorMapEncodeTiled unavailable");
  cuuint64_t sizes[3] = {(cuuint64_t)dim, (cuuint64_t)heads, (cuuint64_t)rows};
  cuuint64_t strides[2] = {(cuuint64_t)dim * 4, (cuuint64_t)heads * dim * 4};
  cuuint32_t box[3] = {32, 1, (cuuint32_t)box_rows};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), sizes, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : fail_arg("cuTensorMapEncodeTiled(f32) failed");
}

static int check_heads(int64_t c, int32_t hq, int32_t hkv, int32_t d) {
  if (c < 1) return fail_arg("block length c must be >= 1");
  if (c > (int64_t(1) << 31) - 256) return fail_arg("block length too large");
  if (hq < 1 || hkv < 1 || hq % hkv) return fail_arg("need hq >= 1, hkv >= 1, hq % hkv == 0");
  if (d != 64 && d != 128) return fail_arg("head dim must be 64 or 128");
  return 0;
}
static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace sa

using namespace sa;

extern "C" {

int sa_abi_version(void) { return 1; }
const char* sa_last_error(void) { return g_err.c_str(); }
int64_t sa_launch_count(void) { return g_launches.load(); }

int sa_permute(const void* src, void* dst, int64_t n_seq, int32_t n_dev, int64_t row_bytes,
               int32_t scheme, int32_t direction, int32_t device, void* stream) {
  if (!src || !dst) return fail_arg("null pointer");
  if (n_dev < 1 || n_seq < n_dev || n_seq % n_dev)
    return fail_arg("n_dev must evenly divide n_seq");  // layout.py:50-56
  if (row_bytes <= 0 || row_bytes % 4) return fail_arg("row_bytes must be a positive multiple of 4");
  if (scheme != SA_SCHEME_CONTIGUOUS && scheme != SA_SCHEME_STRIPED) return fail_arg("bad scheme");
  if (direction != SA_PARTITION && direction != SA_GATHER) return fail_arg("bad direction");
  if (device >= n_dev) return fail_arg("device out of range");
  return launch_permute(src, dst, n_seq, n_dev, row_bytes, scheme, direction, device,
                        static_cast<cudaStream_t>(stream));
}

int sa_fwd_block(const void* q, const void* k, const void* v, float* o_acc, float* lse, void* out,
                 int64_t c, int32_t hq, int32_t hkv, int32_t d, float softmax_scale,
                 int32_t mask_kind, int32_t first_step, int32_t last_step,
                 int64_t* tiles_computed, void* stream) {
  if (int r = check_heads(c, hq, hkv, d)) return r;
  if (!q || !k || !v || !lse) return fail_arg("null q/k/v/lse");
  if (!aligned16(q) || !aligned16(k) || !aligned16(v)) return fail_arg("q/k/v must be 16B aligned");
  if ((o_acc && !aligned16(o_acc)) || (out && !aligned16(out)))
    return fail_arg("o_acc/out must be 16B aligned");  // vector epilogue loads / stores
  if (!(first_step && last_step) && !o_acc) return fail_arg("o_acc required across ring steps");
  if (last_step && !out) return fail_arg("out required on the last step");
  if (mask_kind < 0 || mask_kind > 3) return fail_arg("bad mask kind");
  if (!(softmax_scale > 0.f)) return fail_arg("softmax_scale must be > 0");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (mask_kind == SA_MASK_FULLY_MASKED) {
    // Nothing to fold (attention.py:198: SKIP).  Keep the state well defined.
    if (first_step) {
      if (last_step) return fail_arg("a single fully-masked step leaves every row dead");
      if (int r = launch_fill_state(o_acc, lse, c, hq, d, st)) return r;
    }
    if (last_step) return launch_cast(o_acc, out, c * hq * d, st);
    return 0;
  }
  return launch_fwd(q, k, v, o_acc, lse, out, c, hq, hkv, d, softmax_scale, mask_kind, first_step,
                    last_step, tiles_computed, st);
}

int sa_bwd_preprocess(const void* out, const void* dout, float* dsum, float* dq_acc, int64_t c,
                      int32_t hq, int32_t d, void* stream) {
  if (int r = check_heads(c, hq, hq, d)) return r;
  if (!out || !dout || !dsum || !dq_acc) return fail_arg("null pointer");
  return launch_bwd_pre(out, dout, dsum, dq_acc, c, hq, d, static_cast<cudaStream_t>(stream));
}

int sa_bwd_block(const void* q, const void* k, const void* v, const void* dout, const float* lse,
                 const float* dsum, float* dq_acc, float* dk_acc, float* dv_acc, int64_t c,
                 int32_t hq, int32_t hkv, int32_t d, float softmax_scale, int32_t mask_kind,
                 void* stream) {
  if (int r = check_heads(c, hq, hkv, d)) return r;
  if (!q || !k || !v || !dout || !lse || !dsum || !dq_acc || !dk_acc || !dv_acc)
    return fail_arg("null pointer");
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(dout) || !aligned16(dq_acc) ||
      !aligned16(dk_acc) || !aligned16(dv_acc))
    return fail_arg("q/k/v/dout and the accumulators must be 16B aligned");
  if (mask_kind < 0 || mask_kind > 3) return fail_arg("bad mask kind");
  if (!(softmax_scale > 0.f)) return fail_arg("softmax_scale must be > 0");
  if (mask_kind == SA_MASK_FULLY_MASKED) return 0;
  return launch_bwd(q, k, v, dout, lse, dsum, dq_acc, dk_acc, dv_acc, c, hq, hkv, d,
                    softmax_scale, mask_kind, static_cast<cudaStream_t>(stream));
}

int sa_bwd_block_range(const void* q, const void* k, const void* v, const void* dout,
                       const float* lse, const float* dsum, float* dq_acc, float* dk_acc,
                       float* dv_acc, int64_t c, int32_t hq, int32_t hkv, int32_t d,
                       float softmax_scale, int32_t mask_kind, int32_t key_row_begin,
                       int32_t key_row_end, void* stream) {
  if (int r = check_heads(c, hq, hkv, d)) return r;
  if (!q || !k || !v || !dout || !lse || !dsum || !dq_acc || !dk_acc || !dv_acc)
    return fail_arg("null pointer");
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(dout) || !aligned16(dq_acc) ||
      !aligned16(dk_acc) || !aligned16(dv_acc))
    return fail_arg("q/k/v/dout and the accumulators must be 16B aligned");
  if (mask_kind < 0 || mask_kind > 3) return fail_arg("bad mask kind");
  if (!(softmax_scale > 0.f)) return fail_arg("softmax_scale must be > 0");
  if (key_row_begin < 0 || key_row_end > c || key_row_begin > key_row_end ||
      key_row_begin % 128 || (key_row_end % 128 && key_row_end != c))
    return fail_arg("key rows must be a 128-aligned sub-range of [0, c)");
  if (mask_kind == SA_MASK_FULLY_MASKED || key_row_begin == key_row_end) return 0;
  return launch_bwd(q, k, v, dout, lse, dsum, dq_acc, dk_acc, dv_acc, c, hq, hkv, d,
                    softmax_scale, mask_kind, static_cast<cudaStream_t>(stream), nullptr,
                    nullptr, key_row_begin / 128, (key_row_end + 127) / 128);
}

int sa_bwd_block_final(const void* q, const void* k, const void* v, const void* dout,
                       const float* lse, const float* dsum, float* dq_acc, void* dk, void* dv,
                       int64_t c, int32_t hq, int32_t hkv, int32_t d, float softmax_scale,
                       int32_t mask_kind, void* stream) {
  if (int r = check_heads(c, hq, hkv, d)) return r;
  if (!q || !k || !v || !dout || !lse || !dsum || !dq_acc || !dk || !dv)
    return fail_arg("null pointer");
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(dout) || !aligned16(dq_acc) ||
      !aligned16(dk) || !aligned16(dv))
    return fail_arg("q/k/v/dout, dq_acc and dk/dv must be 16B aligned");
  if (mask_kind < 0 || mask_kind > 3) return fail_arg("bad mask kind");
  if (!(softmax_scale > 0.f)) return fail_arg("softmax_scale must be > 0");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (mask_kind == SA_MASK_FULLY_MASKED) {  // no pair: the gradients are zero
    const size_t bytes = static_cast<size_t>(c) * hkv * d * 2;
    if (cudaMemsetAsync(dk, 0, bytes, st) != cudaSuccess || cudaMemsetAsync(dv, 0, bytes, st) != cudaSuccess)
      return check_launch("memset dk/dv");
    return 0;
  }
  return launch_bwd(q, k, v, dout, lse, dsum, dq_acc, nullptr, nullptr, c, hq, hkv, d,
                    softmax_scale, mask_kind, st, dk, dv);
}

int sa_bwd_block_ex(const void* q, const void* k, const void* v, const void* dout,
                    const float* lse, const float* dsum, float* dq_acc, float* dk_acc,
                    float* dv_acc, void* dk_out, void* dv_out, int64_t c, int32_t hq, int32_t hkv,
                    int32_t d, float softmax_scale, int32_t mask_kind, int32_t key_row_begin,
                    int32_t key_row_end, int32_t* dq_semaphore, void* stream) {
  if (int r = check_heads(c, hq, hkv, d)) return r;
  const bool final_out = dk_out || dv_out;
  if (final_out && (!dk_out || !dv_out)) return fail_arg("dk_out and dv_out go together");
  if (!final_out && (!dk_acc || !dv_acc)) return fail_arg("need dk_acc/dv_acc or dk_out/dv_out");
  if (!q || !k || !v || !dout || !lse || !dsum || !dq_acc) return fail_arg("null pointer");
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(dout) || !aligned16(dq_acc) ||
      (dk_acc && !aligned16(dk_acc)) || (dv_acc && !aligned16(dv_acc)) ||
      (dk_out && !aligned16(dk_out)) || (dv_out && !aligned16(dv_out)))
    return fail_arg("q/k/v/dout, dq_acc and the dK/dV buffers must be 16B aligned");
  if (mask_kind < 0 || mask_kind > 3) return fail_arg("bad mask kind");
  if (!(softmax_scale > 0.f)) return fail_arg("softmax_scale must be > 0");
  if (key_row_end < 0) key_row_end = static_cast<int32_t>(c);
  if (key_row_begin < 0 || key_row_end > c || key_row_begin > key_row_end ||
      key_row_begin % 128 || (key_row_end % 128 && key_row_end != c))
    return fail_arg("key rows must be a 128-aligned sub-range of [0, c)");
  if (final_out && (key_row_begin != 0 || key_row_end != c))
    return fail_arg("bf16 dK/dV outputs need the whole key range");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (mask_kind == SA_MASK_FULLY_MASKED || key_row_begin == key_row_end) {
    if (final_out) {
      const size_t bytes = static_cast<size_t>(c) * hkv * d * 2;
      if (cudaMemsetAsync(dk_out, 0, bytes, st) != cudaSuccess ||
          cudaMemsetAsync(dv_out, 0, bytes, st) != cudaSuccess)
        return check_launch("memset dk/dv");
    }
    return 0;
  }
  return launch_bwd(q, k, v, dout, lse, dsum, dq_acc, dk_acc, dv_acc, c, hq, hkv, d,
                    softmax_scale, mask_kind, st, dk_out, dv_out, key_row_begin / 128,
                    (key_row_end + 127) / 128, dq_semaphore);
}

int sa_cast_f32_bf16(const float* src, void* dst, int64_t n, void* stream) {
  if (!src || !dst || n < 0) return fail_arg("bad cast arguments");
  if (n == 0) return 0;
  return launch_cast(src, dst, n, static_cast<cudaStream_t>(stream));
}

int sa_memcpy2d_async(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width,
                      int64_t height, void* stream) {
  if (!dst || !src || width < 0 || height < 0 || dpitch < width || spitch < width)
    return fail_arg("bad 2-D copy arguments");
  if (width == 0 || height == 0) return 0;
  cudaError_t e = cudaMemcpy2DAsync(dst, (size_t)dpitch, src, (size_t)spitch, (size_t)width,
                                    (size_t)height, cudaMemcpyDefault,
                                    static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) {
    set_error(std::string("cudaMemcpy2DAsync: ") + cudaGetErrorString(e));
    return -static_cast<int>(e);
  }
  return 0;
}

int sa_memcpy_async(void* dst, const void* src, int64_t bytes, void* stream) {
  if (!dst || !src || bytes < 0) return fail_arg("bad copy arguments");
  if (bytes == 0) return 0;
  cudaError_t e = cudaMemcpyAsync(dst, src, static_cast<size_t>(bytes), cudaMemcpyDefault,
                                  static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) {
    set_error(std::string("cudaMemcpyAsync: ") + cudaGetErrorString(e));
    return -static_cast<int>(e);
  }
  return 0;
}

}  // extern "C"
