// Shared sm_100a device helpers: mbarriers, TMA, tcgen05 (UMMA + TMEM), descriptors.
//
// Everything here is inline PTX for -gencode arch=compute_100a,code=sm_100a.
// Layout conventions used by every kernel in this library:
//   * bf16 operand tiles live in shared memory in the 128-byte-swizzle layout that
//     TMA writes (CU_TENSOR_MAP_SWIZZLE_128B): a "panel" is 64 bf16 columns (128 B)
//     x R rows, row r at byte r*128, 16-byte chunk j stored at chunk (j ^ (r & 7)).
//     Panels are 1024-byte aligned.
//   * K-major UMMA operand (K contiguous): one panel per 64 K-elements, SBO = 1024.
//   * MN-major UMMA operand (MN contiguous): one panel per 64 MN-elements, rows are K,
//     LBO = panel stride (next 64 MN elements), SBO = 1024 (next 8 K rows).
#pragma once
#include <cstdint>
#include "../../include/striped_attn.h"  // SA_MASK_* (the softmax helpers)
#include <cuda_bf16.h>
#include <cuda.h>

#define SA_DEV __device__ __forceinline__

// Perf-experiment instrumentation (clock64 timelines, debug knobs read from the
// environment).  OFF in the product build: the launch paths then read no environment,
// allocate nothing and never synchronise.  Build with SA_NVCC_EXTRA=-DSA_PERF_TRACE=1.
#ifndef SA_PERF_TRACE
#define SA_PERF_TRACE 0
#endif

namespace sa {

SA_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

SA_DEV uint32_t warp_id() { return threadIdx.x >> 5; }
SA_DEV uint32_t lane_id() { return threadIdx.x & 31; }

// One lane of a fully active warp.  INVARIANT relied on by every MMA issuer: with the
// full member mask elect.sync picks the same (lowest active) lane every time, so all of a
// warp's tcgen05.mma / tcgen05.commit come from ONE thread -- a commit tracks only the
// earlier tcgen05 ops of its own thread (bwd.cu's DP_FULL / KV_DONE commits depend on it).
// Call only from warps whose 32 lanes are all active.
SA_DEV bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t.reg .b32 r;\n\t"
      "elect.sync r|P, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// ------------------------------------------------------------------ mbarrier
SA_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
SA_DEV void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
SA_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
SA_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;"
               ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// try_wait suspends the warp (it wakes when the phase completes) for up to a time limit;
// without a hint that limit is short and a waiting warp spins every few tens of cycles,
// taking issue slots from the compute warps on its SM sub-partition.  The hint is in ns.
#ifndef SA_MBAR_SUSPEND_NS
#define SA_MBAR_SUSPEND_NS 0x989680
#endif
SA_DEV bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
#if SA_MBAR_SUSPEND_NS
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P, [%1], %2, %3;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "n"(SA_MBAR_SUSPEND_NS)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
#endif
  return ok != 0;
}
SA_DEV uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Non-blocking probe of a phase (for issuers that poll several barriers).
SA_DEV bool mbar_test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "mbarrier.test_wait.parity.acquire.cta.shared::cta.b64 P, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Bounded wait: a pipeline bug traps (launch error) instead of hanging the GPU -- after
// 4 s of waiting on one phase (every legitimate wait here is microseconds).
SA_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  if (mbar_try_wait(bar, parity)) return;
  const uint64_t t0 = globaltimer_ns();
  while (!mbar_try_wait(bar, parity)) {
    if (globaltimer_ns() - t0 > 4000000000ull) __trap();
  }
}

// ------------------------------------------------------------------ TMA
SA_DEV void prefetch_tmap(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
SA_DEV void tma_load_3d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2,
                        uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)),
        "r"(c0), "r"(c1), "r"(c2), "l"(policy)
      : "memory");
}
SA_DEV void tma_load_2d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
SA_DEV uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
SA_DEV uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// ------------------------------------------------------------------ tcgen05 / TMEM
template <uint32_t kCols>
SA_DEV void tmem_alloc(uint32_t* dst_smem) {  // whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
               ::"r"(smem_u32(dst_smem)), "n"(kCols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
template <uint32_t kCols>
SA_DEV void tmem_dealloc(uint32_t taddr) {  // whole warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols));
}
SA_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
SA_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] * B[smem]
SA_DEV void mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc)
      : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem]
SA_DEV void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
      ::"r"(d_tmem), "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc)
      : "memory");
}
// Same, with the descriptors given as (lo, hi) 32-bit halves: only the lo word (start
// address, LBO) varies across k-steps, so callers keep one 32-bit value per operand.
SA_DEV void mma_ss2(uint32_t d_tmem, uint32_t a_lo, uint32_t a_hi, uint32_t b_lo, uint32_t b_hi,
                    uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b64 da, db;\n\t"
      "mov.b64 da, {%1, %2};\n\tmov.b64 db, {%3, %4};\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, p;\n\t}"
      ::"r"(d_tmem), "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(acc)
      : "memory");
}
SA_DEV void mma_ts2(uint32_t d_tmem, uint32_t a_tmem, uint32_t b_lo, uint32_t b_hi, uint32_t idesc,
                    uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b64 db;\n\t"
      "mov.b64 db, {%2, %3};\n\t"
      "setp.ne.b32 p, %5, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], db, %4, p;\n\t}"
      ::"r"(d_tmem), "r"(a_tmem), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(acc)
      : "memory");
}
// lo / hi words of sdesc(): lo = start>>4 | (LBO>>4)<<16, hi = SBO>>4 | version | SW128.
SA_DEV constexpr uint32_t sdesc_lo(uint32_t saddr, uint32_t lbo_bytes) {
  return ((saddr >> 4) & 0x3FFFu) | (((lbo_bytes >> 4) & 0x3FFFu) << 16);
}
SA_DEV constexpr uint32_t sdesc_hi(uint32_t sbo_bytes) {
  return ((sbo_bytes >> 4) & 0x3FFFu) | (1u << 14) | (2u << 29);
}

// Opaque copy: stops the compiler from hoisting per-k-step descriptor arithmetic out of
// the issue loop (which costs registers in the 56-register MMA warp).
SA_DEV uint32_t opaque(uint32_t x) {
  asm volatile("mov.b32 %0, %0;" : "+r"(x));
  return x;
}

// Arrive on an mbarrier when all previously issued tcgen05 ops of this thread finish.
SA_DEV void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               ::"r"(smem_u32(bar)) : "memory");
}

// Instruction descriptor: kind::f16, bf16 x bf16 -> f32, dense.
__host__ __device__ constexpr uint32_t idesc_bf16(uint32_t M, uint32_t N, uint32_t a_mn_major,
                                                  uint32_t b_mn_major) {
  return (1u << 4)            // D format f32
         | (1u << 7)          // A bf16
         | (1u << 10)         // B bf16
         | (a_mn_major << 15) | (b_mn_major << 16)
         | ((N >> 3) << 17) | ((M >> 4) << 24);
}

// Shared-memory matrix descriptor, SWIZZLE_128B, sm100 version bit.
SA_DEV uint64_t sdesc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu)
         | (static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFFu) << 16)
         | (static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFFu) << 32)
         | (1ull << 46)     // version (sm100)
         | (2ull << 61);    // SWIZZLE_128B
}

// TMEM -> registers: 32 lanes x 32 bit, N consecutive columns per thread.
#define SA_TMEM_LD32(taddr, r)                                                                    \
  asm volatile(                                                                                   \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"   \
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"          \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),      \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),  \
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),            \
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),            \
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])             \
      : "r"(taddr))

#define SA_TMEM_LD16(taddr, r)                                                                    \
  asm volatile(                                                                                   \
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"   \
      "%14,%15}, [%16];"                                                                          \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),      \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),  \
        "=r"(r[14]), "=r"(r[15])                                                                  \
      : "r"(taddr))

#define SA_TMEM_ST16(taddr, r)                                                                    \
  asm volatile(                                                                                   \
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"    \
      "%13,%14,%15,%16};"                                                                         \
      ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), \
        "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]),         \
        "r"(r[14]), "r"(r[15])                                                                    \
      : "memory")

#define SA_TMEM_ST32(taddr, r)                                                                    \
  asm volatile(                                                                                   \
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"    \
      "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"        \
      ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), \
        "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]),         \
        "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]),      \
        "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),      \
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])                                            \
      : "memory")

SA_DEV void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
SA_DEV void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Make generic-proxy smem writes visible to the async proxy (UMMA / TMA reads).
SA_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// Order global-memory accesses of the async proxy (TMA) with the generic proxy.
SA_DEV void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
SA_DEV int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
SA_DEV void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

SA_DEV void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <uint32_t kRegs>
SA_DEV void regs_dec() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegs)); }
template <uint32_t kRegs>
SA_DEV void regs_inc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegs)); }

SA_DEV uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);  // .x = lo (low 16 bits)
  return *reinterpret_cast<uint32_t*>(&v);
}

SA_DEV float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ---- CTA pairs (cluster of 2, tcgen05 cta_group::2)
SA_DEV uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
SA_DEV void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}
// Shared::cluster address of the same smem offset in CTA `rank` of the cluster.
SA_DEV uint32_t map_to_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// Arrive on a (possibly remote) barrier of the cluster.  Default .release.cta semantics:
// .release.cluster costs ~1000 clk per arrive on sm_100 and is not needed for the
// tcgen05 hand-off (tcgen05.wait::st + fence::before_thread_sync order the TMEM writes).
SA_DEV void mbar_arrive_cluster(uint32_t cluster_saddr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_saddr) : "memory");
}
template <uint32_t kCols>
SA_DEV void tmem_alloc2(uint32_t* dst_smem) {  // one warp in EACH CTA of the pair
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
               ::"r"(smem_u32(dst_smem)), "n"(kCols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
template <uint32_t kCols>
SA_DEV void tmem_dealloc2(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols));
}
// 2-CTA MMAs, issued by the leader CTA only; A rows split across the pair, B split by N.
SA_DEV void mma2_ss(uint32_t d_tmem, uint32_t a_lo, uint32_t a_hi, uint32_t b_lo, uint32_t b_hi,
                    uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b64 da, db;\n\t"
      "mov.b64 da, {%1, %2};\n\tmov.b64 db, {%3, %4};\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, p;\n\t}"
      ::"r"(d_tmem), "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(acc)
      : "memory");
}
SA_DEV void mma2_ts(uint32_t d_tmem, uint32_t a_tmem, uint32_t b_lo, uint32_t b_hi, uint32_t idesc,
                    uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b64 db;\n\t"
      "mov.b64 db, {%2, %3};\n\t"
      "setp.ne.b32 p, %5, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], db, %4, p;\n\t}"
      ::"r"(d_tmem), "r"(a_tmem), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(acc)
      : "memory");
}
// Commit of the leader's MMAs, arriving on the barrier at the same offset in both CTAs.
SA_DEV void mma2_commit_both(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)), "h"((uint16_t)3)
      : "memory");
}
// TMA load broadcast to the CTAs of `mask`: same smem offset and same barrier offset in each.
SA_DEV void tma_load_3d_mc(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2,
                           uint64_t policy, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      ".multicast::cluster.L2::cache_hint [%0], [%1, {%3, %4, %5}], [%2], %6, %7;"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)),
        "r"(c0), "r"(c1), "r"(c2), "h"(mask), "l"(policy)
      : "memory");
}
// 1-CTA MMA commit arriving on the barrier at the same offset in every CTA of `mask`.
SA_DEV void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
// TMA load into this CTA's smem whose transaction bytes complete on the LEADER's barrier.
SA_DEV void tma_load_3d_pair(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2,
                             uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%3, %4, %5}], [%2], %6;"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)),
        "r"(map_to_rank(smem_u32(bar), 0)), "r"(c0), "r"(c1), "r"(c2), "l"(policy)
      : "memory");
}

// ---- packed fp32x2 arithmetic (sm_100 FFMA2 / FADD2 / FMUL2: two lanes' worth per issue)
SA_DEV void fma2(float& d0, float& d1, float a0, float a1, float b0, float b1, float c0, float c1) {
  asm("{\n\t.reg .b64 a, b, c, d;\n\t"
      "mov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\tmov.b64 c, {%6, %7};\n\t"
      "fma.rn.f32x2 d, a, b, c;\n\tmov.b64 {%0, %1}, d;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}
SA_DEV void add2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  asm("{\n\t.reg .b64 a, b, d;\n\t"
      "mov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
      "add.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
SA_DEV void mul2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  asm("{\n\t.reg .b64 a, b, d;\n\t"
      "mov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
      "mul.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}

// 2^x for a pair on the FMA pipe (offloads the MUFU unit, which alone caps the softmax):
// round-to-nearest split x = j + f with the 1.5*2^23 trick, f in [-0.5, 0.5], degree-3
// polynomial (max rel. error 7.7e-5, far below the bf16 rounding P gets next), exponent
// added as an integer.  Valid for x in [-125, 126]; smaller x clamps to 2^-125.
SA_DEV void ex2_poly2(float& y0, float& y1, float x0, float x1) {
  constexpr float kMagic = 12582912.f;  // 1.5 * 2^23
  x0 = fmaxf(x0, -125.f);
  x1 = fmaxf(x1, -125.f);
  float t0, t1, r0, r1, f0, f1, p0, p1;
  add2(t0, t1, x0, x1, kMagic, kMagic);
  add2(r0, r1, t0, t1, -kMagic, -kMagic);
  add2(f0, f1, x0, x1, -r0, -r1);
  fma2(p0, p1, f0, f1, 0.05509095639f, 0.05509095639f, 0.2426045388f, 0.2426045388f);
  fma2(p0, p1, p0, p1, f0, f1, 0.6932758689f, 0.6932758689f);
  fma2(p0, p1, p0, p1, f0, f1, 0.9999288917f, 0.9999288917f);
  y0 = __int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23));
  y1 = __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23));
}

// ---- forward softmax of one S row (128 keys held by one thread), shared by fwd.cu and
// fwd_pair.cu: the reference's tile fold (attention.py:310-328) in the exp2 domain.
// Key column limit of a masked (diagonal and/or ragged) tile: keys >= the returned value
// are masked -- inclusive y <= x, strict y < x (attention.py:155-183), ragged y < c.
SA_DEV int key_limit(int kind, int x, int c, int j) {
  const int last = kind == SA_MASK_CAUSAL_INCLUSIVE ? x + 1 : kind == SA_MASK_CAUSAL_EXCLUSIVE ? x : c;
  return min(last, c) - j * 128;
}
// Keys >= lim of a masked tile -> -inf (before the row maximum).
SA_DEV void mask_row(uint32_t (&r)[128], int lim) {
#pragma unroll
  for (int i = 0; i < 128; i++)
    if (i >= lim) r[i] = __float_as_uint(-INFINITY);
}
// Row maximum of the raw scores.  Eight independent partial maxima: no 128-long
// dependency chain (ptxas pairs them into FMNMX3).
SA_DEV float s_row_max(const uint32_t (&r)[128]) {
  float mx8[8];
#pragma unroll
  for (int u = 0; u < 8; u++) mx8[u] = __uint_as_float(r[u]);
#pragma unroll
  for (int i = 8; i < 128; i++) mx8[i & 7] = fmaxf(mx8[i & 7], __uint_as_float(r[i]));
  return fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
               fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
}
// p = 2^(s * scale_log2 - m) (neg_m = -m, 0 for a row with no key yet), packed as bf16
// pairs in place into r[0..63] for the PV MMA; returns the fp32 row sum of the unrounded
// p.  Pairs go through FFMA2; kPoly of every 16 pairs take the FMA-pipe polynomial (the
// rest MUFU.EX2) so the two pipes share the exponentials; four FADD2 chains for the sum.
template <bool kMasked, int kPoly>
SA_DEV float s_row_exp_pack(uint32_t (&r)[128], float scale_log2, float neg_m, int lim) {
  float sa[4] = {0.f, 0.f, 0.f, 0.f}, sb[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int i = 0; i < 64; i++) {
    float x0, x1, p0, p1;
    fma2(x0, x1, __uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]), scale_log2,
         scale_log2, neg_m, neg_m);
    if ((i & 15) < kPoly) {
      ex2_poly2(p0, p1, x0, x1);
    } else {
      p0 = ex2(x0);
      p1 = ex2(x1);
    }
    if constexpr (kMasked) {
      p0 = 2 * i < lim ? p0 : 0.f;
      p1 = 2 * i + 1 < lim ? p1 : 0.f;
    }
    add2(sa[i & 3], sb[i & 3], sa[i & 3], sb[i & 3], p0, p1);
    r[i] = pack_bf16(p0, p1);
  }
  return ((sa[0] + sa[1]) + (sa[2] + sa[3])) + ((sb[0] + sb[1]) + (sb[2] + sb[3]));
}
// Lazy rescale of one thread's O row in TMEM (D fp32 columns) by `factor`.
template <int D>
SA_DEV void tmem_scale_row(uint32_t t_o, float factor) {
#pragma unroll 1
  for (int ch = 0; ch < D / 32; ch++) {
    uint32_t o[32];
    SA_TMEM_LD32(t_o + ch * 32, o);
    tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 32; i++) o[i] = __float_as_uint(__uint_as_float(o[i]) * factor);
    SA_TMEM_ST32(t_o + ch * 32, o);
  }
}

// ---- forward epilogue shared by fwd.cu (D = 64) and fwd_pair.cu (D = 128): merge one
// block's result into the running (o_acc, lse) state of the ring steps so far -- the
// reference's carry rules (attention.py:321-328) and finalize (331-336), -inf safe: a row
// that attended no key in this block (lse_blk = -inf) keeps its state bit for bit.
struct LseMerge {
  float w_prev;   // weight of the carried o_acc
  float s_blk;    // scale of this block's unnormalised O (weight / l)
  float lse_new;  // merged log-sum-exp (natural log)
};
SA_DEV LseMerge lse_merge(float lse_blk, float inv_l, bool first, const float* lse_prev_ptr) {
  LseMerge r{0.f, inv_l, lse_blk};
  if (!first) {
    const float lse_prev = *lse_prev_ptr;
    const float mx = fmaxf(lse_prev, lse_blk);
    if (mx == -INFINITY) {
      r.w_prev = 1.f;
      r.s_blk = 0.f;
      r.lse_new = -INFINITY;
    } else {
      const float a = __expf(lse_prev - mx), bb = __expf(lse_blk - mx);
      r.lse_new = mx + __logf(a + bb);
      r.w_prev = a / (a + bb);
      r.s_blk = bb / (a + bb) * inv_l;
    }
  }
  return r;
}
// 32 consecutive output columns of one row: v = O * s_blk (+ w_prev * o_acc); written as
// bf16 to `out_row` on the last ring step, else as fp32 back to `acc_row`.
SA_DEV void merge_store32(const uint32_t* o, const LseMerge& mw, bool first, bool last,
                          float* acc_row, __nv_bfloat16* out_row) {
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; i++) v[i] = __uint_as_float(o[i]) * mw.s_blk;
  if (!first) {
    const float4* src = reinterpret_cast<const float4*>(acc_row);
#pragma unroll
    for (int i = 0; i < 8; i++) {
      const float4 a = src[i];
      v[4 * i] += mw.w_prev * a.x;
      v[4 * i + 1] += mw.w_prev * a.y;
      v[4 * i + 2] += mw.w_prev * a.z;
      v[4 * i + 3] += mw.w_prev * a.w;
    }
  }
  if (last) {
    uint4* dst = reinterpret_cast<uint4*>(out_row);
#pragma unroll
    for (int i = 0; i < 4; i++)
      dst[i] = make_uint4(pack_bf16(v[8 * i], v[8 * i + 1]), pack_bf16(v[8 * i + 2], v[8 * i + 3]),
                          pack_bf16(v[8 * i + 4], v[8 * i + 5]), pack_bf16(v[8 * i + 6], v[8 * i + 7]));
  } else {
    float4* dst = reinterpret_cast<float4*>(acc_row);
#pragma unroll
    for (int i = 0; i < 8; i++) dst[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
  }
}

// Byte offset of 16-byte chunk `chunk` (0..7) of row `row` inside a SW128 panel.
SA_DEV uint32_t sw128_off(uint32_t row, uint32_t chunk) {
  return row * 128u + ((chunk ^ (row & 7u)) << 4);
}

SA_DEV void named_bar_arrive(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Explicit shared-space accesses (32-bit shared addresses; never generic).
SA_DEV void sts128(uint32_t saddr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(saddr), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}
SA_DEV float4 lds128f(uint32_t saddr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(saddr)
               : "memory");
  return v;
}
SA_DEV float lds32f(uint32_t saddr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(saddr) : "memory");
  return v;
}
SA_DEV void sts32f(uint32_t saddr, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(saddr), "f"(v) : "memory");
}

// TMA bulk tensor reduce-add (fp32) smem -> global, bulk-group completion.
SA_DEV void tma_reduce_add_3d(const CUtensorMap* m, const void* src, int c0, int c1, int c2) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group"
      " [%0, {%2, %3, %4}], [%1];"
      ::"l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
SA_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
SA_DEV void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
SA_DEV void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

}  // namespace sa
