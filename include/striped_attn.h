/* striped_attn.h -- C ABI of the B200 (sm_100a) striped / ring causal attention path.
 *
 * Drop-in boundary for the reference's hot path (ringsim, /root/reference/pkg/src/ringsim).
 * The reference has no FFI: its seams are pure-Python functions.  Each entry point
 * below names the reference function it replaces.  A ctypes binding of exactly these
 * symbols is paper_2311_09431_b200/_lib.py; INTEGRATION.md shows the binding a
 * ringsim maintainer would add.
 *
 * Conventions (all entry points):
 *   - Caller-owned DEVICE buffers, plain pointers and element counts; the library never
 *     allocates device memory and never throws across the ABI.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Return 0 = OK, >0 = invalid argument (nothing launched), <0 = CUDA error.
 *     sa_last_error() returns a thread-local message for the last non-zero status.
 *   - Thread-safe across distinct streams.
 *   - Token-major layouts: Q/K/V/O/dO are bf16 [c, H, D] (row = token, heads
 *     interleaved, D contiguous).  LSE / Dsum are fp32 [H, c].  Accumulators fp32.
 *   - D (head dim) in {64, 128}; Hq % Hkv == 0 (grouped-query attention).
 *   - softmax_scale multiplies QK^T (the reference's scale=True is 1/sqrt(D),
 *     attention.py:137-138 / simulator.py:365).
 */
#ifndef STRIPED_ATTN_H_
#define STRIPED_ATTN_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* MaskKind, attention.py:42-46 (same order). */
enum sa_mask_kind {
  SA_MASK_FULLY_MASKED = 0,    /* no pair allowed: block skipped                    */
  SA_MASK_FULLY_UNMASKED = 1,  /* every pair allowed                                */
  SA_MASK_CAUSAL_INCLUSIVE = 2,/* allowed iff key row y <= query row x              */
  SA_MASK_CAUSAL_EXCLUSIVE = 3 /* allowed iff y < x (striped, key stripe > q stripe) */
};

/* Scheme, layout.py:20-22. */
enum sa_scheme { SA_SCHEME_CONTIGUOUS = 0, SA_SCHEME_STRIPED = 1 };

/* Direction of sa_permute. */
enum sa_direction { SA_PARTITION = 0, SA_GATHER = 1 };

int sa_abi_version(void);
const char* sa_last_error(void);
/* Number of device kernels this library launched since load (for bench "gpu_launches"). */
int64_t sa_launch_count(void);

/* K1 -- stripe permute / unpermute of a row-major [n_seq, row_bytes] tensor.
 * Replaces Layout.partition (layout.py:81-101) and Layout.gather (layout.py:103-117).
 *   SA_PARTITION, device < 0 : dst = concat_d shard_d   (dst row d*c + x <- src row global_of(d, x))
 *   SA_PARTITION, device = d : dst = shard_d only       ([c, row_bytes])
 *   SA_GATHER,    device < 0 : dst[global_of(d, x)] <- src[d*c + x]   (exact inverse)
 *   SA_GATHER,    device = d : scatter shard d (src [c, row]) into its rows of dst [n_seq, row]
 * global_of: striped d + x*N, contiguous d*c + x (layout.py:62-70).  Bit-exact byte copy;
 * works for any payload (Q/K/V rows, int64 position ids, ...).  row_bytes % 4 == 0. */
int sa_permute(const void* src, void* dst, int64_t n_seq, int32_t n_dev, int64_t row_bytes,
               int32_t scheme, int32_t direction, int32_t device, void* stream);

/* K2+K3 -- one ring step of the forward for one rank (one query stripe vs the held
 * key/value stripe), all heads.  Replaces _process_round (simulator.py:144-186) ->
 * classify_tiles / accumulate_tile / _fold (attention.py:213-225, 296-328) and, on the last
 * step, finalize (attention.py:331-336) plus the implied LSE = m + ln l.
 *   q [c, hq, d], k/v [c, hkv, d] bf16.
 *   o_acc [c, hq, d] fp32, lse [hq, c] fp32: running (normalised) output and LSE of the ring
 *     steps so far; merged in place with this block's result (-inf safe).  first_step: the
 *     previous state is ignored (o_acc may be NULL when first_step && last_step).
 *   out [c, hq, d] bf16: written when last_step (may be NULL otherwise).
 *   mask_kind: sa_mask_kind for (query stripe j, key stripe k), chosen by the host with
 *     get_mask_striped / get_mask_ring (attention.py:155-183).  Tiles of 128x128 are
 *     classified in-kernel with the reference rule (attention.py:194-210); SKIP tiles are
 *     never computed.  Rows with no allowed key (strict mask, local row 0) leave the state
 *     unchanged.  tiles_computed (nullable, device int64[1]) is incremented by the number
 *     of 128x128 tiles computed per head (the reference's RoundStats counters). */
int sa_fwd_block(const void* q, const void* k, const void* v, float* o_acc, float* lse, void* out,
                 int64_t c, int32_t hq, int32_t hkv, int32_t d, float softmax_scale,
                 int32_t mask_kind, int32_t first_step, int32_t last_step,
                 int64_t* tiles_computed, void* stream);

/* K4 -- backward preprocess: dsum[h, x] = sum_d dout[x,h,d] * out[x,h,d]; zeroes dq_acc.
 * (No reference counterpart: ringsim has no backward.) */
int sa_bwd_preprocess(const void* out, const void* dout, float* dsum, float* dq_acc, int64_t c,
                      int32_t hq, int32_t d, void* stream);

/* K5 -- one ring step of the backward for one rank (no reference counterpart).
 * Recomputes P = exp(scale*QK^T - lse) under mask_kind with the GLOBAL lse, then
 *   dq_acc [c,hq,d] fp32 += scale * dS K          (this rank's queries)
 *   dk_acc [c,hkv,d] fp32 += scale * dS^T Q       (the held key stripe; travels with K)
 *   dv_acc [c,hkv,d] fp32 += P^T dO               (travels with V)
 * with dS = P o (dO V^T - dsum).  Same tile classification / skipping as sa_fwd_block. */
int sa_bwd_block(const void* q, const void* k, const void* v, const void* dout, const float* lse,
                 const float* dsum, float* dq_acc, float* dk_acc, float* dv_acc, int64_t c,
                 int32_t hq, int32_t hkv, int32_t d, float softmax_scale, int32_t mask_kind,
                 void* stream);

/* sa_bwd_block restricted to the keys [key_row_begin, key_row_end) of the held stripe
 * (128-aligned; the end may be c): only those dK / dV rows and their dQ contributions.
 * The ring launches a block in parts so each part's dK / dV rows can travel to the next
 * rank while the next part computes. */
int sa_bwd_block_range(const void* q, const void* k, const void* v, const void* dout,
                       const float* lse, const float* dsum, float* dq_acc, float* dk_acc,
                       float* dv_acc, int64_t c, int32_t hq, int32_t hkv, int32_t d,
                       float softmax_scale, int32_t mask_kind, int32_t key_row_begin,
                       int32_t key_row_end, void* stream);

/* Single-step backward ("final"): as sa_bwd_block, but dK / dV are written (not added)
 * as bf16 [c, Hkv, D] straight from the kernel's accumulators: no fp32 accumulators, no
 * zero-fill, no cast.  For a block that is the ONLY contribution to dK / dV (N = 1, or
 * the caller's own non-ring use); the ring's travelling accumulators use sa_bwd_block. */
int sa_bwd_block_final(const void* q, const void* k, const void* v, const void* dout,
                       const float* lse, const float* dsum, float* dq_acc, void* dk, void* dv,
                       int64_t c, int32_t hq, int32_t hkv, int32_t d, float softmax_scale,
                       int32_t mask_kind, void* stream);

/* All options of K5 in one entry point:
 *   - dk_acc / dv_acc (fp32, reduce-added) OR dk_out / dv_out (bf16, written; whole key
 *     range only) -- exactly one pair non-NULL;
 *   - key rows [key_row_begin, key_row_end) as sa_bwd_block_range (key_row_end < 0 = c);
 *   - dq_semaphore (nullable): DETERMINISTIC dQ.  int32 [hq, ceil(c/64)], zero-filled
 *     once by the caller and left zero by every launch; the key tiles then add into each
 *     query tile of dq_acc in ascending order, so reruns are bit-identical (the
 *     reference requires reproducible runs: verify.py:216-227).  Slower: the
 *     reduce-adds of one query tile serialise across CTAs. */
int sa_bwd_block_ex(const void* q, const void* k, const void* v, const void* dout,
                    const float* lse, const float* dsum, float* dq_acc, float* dk_acc,
                    float* dv_acc, void* dk_out, void* dv_out, int64_t c, int32_t hq, int32_t hkv,
                    int32_t d, float softmax_scale, int32_t mask_kind, int32_t key_row_begin,
                    int32_t key_row_end, int32_t* dq_semaphore, void* stream);

/* dst_bf16[i] = bf16(src[i]) (finalises dq/dk/dv accumulators and skipped last steps). */
int sa_cast_f32_bf16(const float* src, void* dst, int64_t n, void* stream);

/* Strided host<->device row copy (cudaMemcpy2DAsync): `height` rows of `width` bytes,
 * row pitches in bytes.  Used by the host-streaming API to move one head group of a
 * token-major [c, H, D] tensor without a host-side gather. */
int sa_memcpy2d_async(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width,
                      int64_t height, void* stream);

/* Device<->device (or peer) copy of `bytes` bytes on `stream` (cudaMemcpyAsync with
 * cudaMemcpyDefault: a copy engine, NVLink between peers).  The ring's copy-engine hop
 * (ring.LocalComm, ipc.IpcComm) -- the reference's per-round message hand-off,
 * simulator.py:211-215 -- issued without NCCL kernels on the SMs. */
int sa_memcpy_async(void* dst, const void* src, int64_t bytes, void* stream);

/* CUDA IPC for the one-process-per-GPU copy-engine hop (ipc.IpcComm), handles exchanged
 * once per buffer: 64-byte opaque handles.  sa_ipc_mem_handle returns the handle of the
 * allocation containing `ptr` and ptr's byte offset in it. */
int sa_ipc_mem_handle(const void* ptr, void* handle_out, int64_t* offset_out);
int sa_ipc_mem_open(const void* handle, void** base_out);
int sa_ipc_mem_close(void* base);
int sa_ipc_event_create(void** event_out, void* handle_out);
int sa_ipc_event_open(const void* handle, void** event_out);
int sa_event_record(void* event, void* stream);
int sa_stream_wait_event(void* stream, void* event);
int sa_event_destroy(void* event);

#ifdef __cplusplus
}
#endif
#endif /* STRIPED_ATTN_H_ */
