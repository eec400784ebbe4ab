// K5: striped / ring block backward on tcgen05 (no reference counterpart: ringsim has no
// backward).  Same block mask, tile classification and skipping as the forward
// (attention.py:155-183, 194-210), recomputing P from the GLOBAL lse.
//
// One CTA = one 128-row key/value tile j of one kv head g; it loops over the q heads of its
// GQA group and the non-SKIP 128-row query tiles i, accumulating dK and dV in TMEM.
// Transposed orientation (TMEM lane = key row):
//   S^T  = K Q_i^T            (SS, both K-major)                       -> TMEM [0,128)
//   dP^T = V dO_i^T           (SS, both K-major)                       -> TMEM [128,256)
//   P^T  = exp2(S^T*scale*log2e - lse*log2e)     (compute WGs, written back as bf16 over S^T)
//   dV  += P^T dO_i           (TS; dO MN-major)                         -> [256,256+D)
//   dS^T = P^T o (dP^T - dsum)                    (compute WGs, bf16 into smem, SW128)
//   dK  += dS^T Q_i           (SS: dS^T K-major; Q MN-major)            -> [256+D,256+2D)
//   dQ_i = dS K               (SS: dS = MN-major view of the same smem) -> [128,128+D)
// dQ_i is drained TMEM -> registers -> a dedicated smem staging buffer -> TMA bulk
// reduce-add into the fp32 dq_acc; dK / dV are added into the travelling fp32 accumulators
// with TMA reduce-add once per CTA (the CTA owns those rows: deterministic).
//
// MMA issue order (one elected lane of warp 1):
//   prologue S(0) dP(0);  per i:  [P(i)] dV(i)  [Q(i+1)] S(i+1)  [dS(i)] dQ(i) dK(i)
//                                 [dQ(i) drained, dO(i+1)] dP(i+1)
// so the compute warpgroups run P(i+1) right after dS(i) while the tensor core works
// through dQ(i), dK(i), dP(i+1): the two sides overlap instead of alternating.
//
// CTA pairs (SA_BWD_PAIR, default): the grid is launched in clusters of two adjacent key
// tiles that walk the same query-tile sequence in lockstep.  Each Q_i / dO_i tile is read
// from L2 once and multicast into both CTAs (each CTA issues one of the two D=128 panels);
// a stage is reloaded once BOTH CTAs' MMAs released it (the release commits are multicast).
// Halving the per-SM Q / dO fetches measured +3% on the backward at c = 64k.
//
// Warp groups (512 threads):
//   WG0: warp 0 TMA producer (+ lse/dsum staging), warp 1 MMA issuer, warp 2 TMEM alloc.
//   WG1 / WG2: compute, query columns [0,64) / [64,128) of each tile (two warps per SMSP).
//   WG3: dQ drain, then the dK epilogue.  WG1 also runs the dV epilogue.
// Shared memory (D=128): K, V 32 KB each; Q 2 stages; dO 1 stage (refilled as soon as
// dV(i) retires); dS 32 KB; dQ staging 2 x 16 KB; lse / dsum 2 stages.
#include "../../include/striped_attn.h"
// Plain (short-suspend) try_wait loops here: the suspend hint measured neutral on this
// kernel (+0.1 %), while it gains 1.2 % on the forward.
#ifndef SA_MBAR_SUSPEND_NS
#define SA_MBAR_SUSPEND_NS 0
#endif
#include "common.cuh"
#include "internal.h"

#include <cstdio>
#include <cstdlib>

namespace sa {
namespace {

constexpr uint32_t kPanelBytes = 128 * 128;  // 128 rows x 128 B
constexpr float kLog2e = 1.4426950408889634f;
#ifndef SA_BWD_DP_PREFETCH
#define SA_BWD_DP_PREFETCH 1  // both dP^T chunks loaded before the first wait
#endif
#ifndef SA_BWD_POLY
#define SA_BWD_POLY 0  // quads of every 8 whose exp2 runs on the FMA-pipe polynomial
#endif
#ifndef SA_BWD_PAIR
#define SA_BWD_PAIR 1  // clusters of two key tiles sharing multicast Q / dO loads (A/B: 0)
#endif
#ifndef SA_BWD_PACKED
#define SA_BWD_PACKED 0  // packed fp32x2 dS arithmetic (A/B)
#endif

struct BwdParams {
  CUtensorMap tq, tk, tv, tdo;   // bf16 [c, H, D], box 64 x 1 x 128
  CUtensorMap tdq, tdk, tdv;     // fp32 [c, H, D], box 32 x 1 x 128 (reduce-add)
  const float* lse;
  const float* dsum;
  // "final" mode (single-step backward, sa_bwd_block_final): dK / dV are written once as
  // bf16 straight from TMEM instead of reduce-added into fp32 accumulators
  __nv_bfloat16* dk_out;
  __nv_bfloat16* dv_out;
  // deterministic dQ (nullable): int32 [hq, n_t] ordering the reduce-adds into each query
  // tile by ascending key tile; zero at launch, left zero by the launch
  int* dq_sem;
  int c, hq, hkv, n_t;
  int j_begin, n_j;  // key tiles [j_begin, j_begin + n_j) of the block (a part of it)
  float scale, scale_log2;
  int kind;
  int debug;         // perf experiments only: bit0 = skip the dQ reduction
  long long* trace;  // perf experiments only: per-iteration clock64 stamps of one CTA
  int trace_cta;
};

#define SA_TR(slot)                                                                     \
  do {                                                                                  \
    if (SA_PERF_TRACE && p.trace && blockIdx.x == p.trace_cta && it < 16) p.trace[it * 32 + (slot)] = clock64(); \
  } while (0)

template <int D>
struct BwdSmem {
  static constexpr uint32_t kTile = D / 64 * kPanelBytes;  // 128 rows x D bf16
  static constexpr uint32_t kK = 0, kV = kTile, kQ = 2 * kTile, kDO = 4 * kTile, kDS = 5 * kTile;
  static constexpr uint32_t kStg = kDS + 2 * kPanelBytes;   // dQ staging, 2 x 16 KB
  static constexpr uint32_t kLse = kStg + 2 * kPanelBytes;  // 2 stages x 128 fp32
  static constexpr uint32_t kDsum = kLse + 1024;
  static constexpr uint32_t kBar = kDsum + 1024;
  static constexpr uint32_t kBytes = kBar + 256;
  static constexpr uint32_t kAlloc = kBytes + 1024 <= 232448 ? kBytes + 1024 : 232448;
};

enum : int {
  B_KV_FULL = 0, B_S_FULL, B_DP_FULL, B_P_READY, B_DS_READY, B_DQ_FULL, B_DQ_FREE, B_DS_EMPTY,
  B_KV_DONE, B_DO_FULL, B_DO_EMPTY, B_Q_FULL = 11 /* x2 */, B_LSE_FULL = 13 /* x2 */,
  B_Q_EMPTY = 15 /* x2 */, B_COUNT = 17
};

__device__ __forceinline__ bool allowed_bwd(int kind, int x, int y, int c) {
  if (x >= c || y >= c) return false;
  if (kind == SA_MASK_CAUSAL_INCLUSIVE) return y <= x;
  if (kind == SA_MASK_CAUSAL_EXCLUSIVE) return y < x;
  return true;
}

// One key row (TMEM lane) of a dK / dV accumulator -> bf16 global row y of kv head g.
template <int D>
__device__ __forceinline__ void store_row_bf16(__nv_bfloat16* base, uint32_t t_row, float scale,
                                               int y, int g, const BwdParams& p) {
  __nv_bfloat16* dst = base + ((int64_t)y * p.hkv + g) * D;
  const bool live = y < p.c;
#pragma unroll 1
  for (int ch = 0; ch < D / 32; ch++) {
    uint32_t o[32];
    SA_TMEM_LD32(t_row + ch * 32, o);
    tmem_ld_wait();
    if (!live) continue;
    uint4* d4 = reinterpret_cast<uint4*>(dst + ch * 32);
#pragma unroll
    for (int i = 0; i < 4; i++) {
      const float* f = reinterpret_cast<const float*>(o + 8 * i);
      d4[i] = make_uint4(pack_bf16(f[0] * scale, f[1] * scale), pack_bf16(f[2] * scale, f[3] * scale),
                         pack_bf16(f[4] * scale, f[5] * scale), pack_bf16(f[6] * scale, f[7] * scale));
    }
  }
}

template <int D, bool kPair>
__global__ void __launch_bounds__(512, 1) bwd_kernel(const __grid_constant__ BwdParams p) {
  using L = BwdSmem<D>;
  constexpr int kPanels = D / 64;
  constexpr int kKSteps = D / 16;
  constexpr int kChunks = D / 32;  // 32-column fp32 chunks of dQ / dK / dV
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint32_t* tmem_base_s = reinterpret_cast<uint32_t*>(bar + B_COUNT);
  const uint32_t sbase = smem_u32(smem);

  const uint32_t warp = warp_id(), lane = lane_id();
  if (smem + L::kBytes > smem_raw + L::kAlloc) __trap();  // alignment slack exhausted

  // Head-major order: the ~148 concurrent CTAs share one kv head, so that head's Q / dO
  // and its dq_acc rows (the reduce-add target) stay L2-resident.  Within a head, small j
  // (most query tiles) first (LPT).
  // kPair: clusters of two adjacent key tiles (j_begin + 2m, j_begin + 2m + 1) walk the
  // SAME query tiles in lockstep, so each Q_i / dO_i tile is fetched from L2 once and
  // multicast to both CTAs (each CTA issues half of the loads).  The odd CTA's first tile
  // (i = j - 1) is fully masked, and an odd tile count gets a "ghost" partner that
  // contributes nothing.
  const int nj_grid = kPair ? (p.n_j + 1) & ~1 : p.n_j;
  const int jj = blockIdx.x % nj_grid;
  const int g = blockIdx.x / nj_grid;
  const int j = p.j_begin + jj;
  const bool ghost = kPair && jj >= p.n_j;
  const uint32_t rank = kPair ? (jj & 1) : 0;
  const int group = p.hq / p.hkv;
  const bool causal = p.kind != SA_MASK_FULLY_UNMASKED;
  const int i0 = causal ? (kPair ? j - static_cast<int>(rank) : j) : 0;
  const int n_i = p.n_t - i0;
  const int n_it = group * n_i;

  if (warp == 2) tmem_alloc<512>(tmem_base_s);
  if (warp == 1 && lane == 0) {
    for (int b = 0; b < B_COUNT; b++) mbar_init(&bar[b], 1);
    mbar_init(&bar[B_LSE_FULL], 32);
    mbar_init(&bar[B_LSE_FULL + 1], 32);
    mbar_init(&bar[B_P_READY], 256);
    mbar_init(&bar[B_DS_READY], 256);
    mbar_init(&bar[B_DQ_FREE], 128);
    if (kPair) {  // both CTAs' MMAs must have released a Q / dO stage before its reload
      mbar_init(&bar[B_Q_EMPTY], 2);
      mbar_init(&bar[B_Q_EMPTY + 1], 2);
      mbar_init(&bar[B_DO_EMPTY], 2);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&p.tq);
    prefetch_tmap(&p.tdo);
    prefetch_tmap(&p.tdq);
  }
  tc_fence_before();
  if (kPair)
    cluster_sync();  // the partner's barriers are initialised before any multicast lands
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_base_s;
  const uint32_t t_st = tbase, t_dpt = tbase + 128, t_dv = tbase + 256, t_dk = tbase + 256 + D;

  if (warp < 4) {
    regs_dec<56>();
    if (warp == 0) {
      // ---------------------------------------------------------- producer
      const uint64_t pol_kv = policy_evict_first(), pol_q = policy_evict_last();
      // kPair: which multicast Q / dO loads this CTA issues for both (D=128: one panel each;
      // D=64: whole tiles, alternating by iteration)
      auto fetches = [&](int pn, int it) {
        return kPanels == 2 ? pn == static_cast<int>(rank) : (it & 1) == static_cast<int>(rank);
      };
      if (lane == 0) {
        mbar_arrive_expect_tx(&bar[B_KV_FULL], 2 * L::kTile);
        for (int pn = 0; pn < kPanels; pn++) {
          tma_load_3d(smem + L::kK + pn * kPanelBytes, &p.tk, &bar[B_KV_FULL], 64 * pn, g, 128 * j,
                      pol_kv);
          tma_load_3d(smem + L::kV + pn * kPanelBytes, &p.tv, &bar[B_KV_FULL], 64 * pn, g, 128 * j,
                      pol_kv);
        }
      }
      for (int it = 0; it < n_it; it++) {
        const int s = it & 1;
        const int h = g * group + it / n_i;
        const int i = i0 + it % n_i;
        // Q_i (2 stages) and lse/dsum (2 stages): free once dK(i-2) retired
        if (it >= 2) mbar_wait(&bar[B_Q_EMPTY + s], ((it >> 1) - 1) & 1);
        if (lane == 0) {
          SA_TR(21);
          mbar_arrive_expect_tx(&bar[B_Q_FULL + s], L::kTile);
          for (int pn = 0; pn < kPanels; pn++) {
            uint8_t* dst = smem + L::kQ + s * L::kTile + pn * kPanelBytes;
            if (!kPair)
              tma_load_3d(dst, &p.tq, &bar[B_Q_FULL + s], 64 * pn, h, 128 * i, pol_q);
            else if (fetches(pn, it))
              tma_load_3d_mc(dst, &p.tq, &bar[B_Q_FULL + s], 64 * pn, h, 128 * i, pol_q, 3);
          }
        }
#pragma unroll
        for (int e = 0; e < 4; e++) {
          const int xl = lane * 4 + e, x = 128 * i + xl;
          float lv = INFINITY, dv = 0.f;  // rows past the block: P = 0
          if (x < p.c) {
            const float raw = p.lse[(int64_t)h * p.c + x];
            lv = raw == -INFINITY ? INFINITY : raw * kLog2e;  // dead row -> P = 0
            dv = p.dsum[(int64_t)h * p.c + x];
          }
          sts32f(sbase + L::kLse + s * 512 + xl * 4, lv);
          sts32f(sbase + L::kDsum + s * 512 + xl * 4, dv);
        }
        mbar_arrive(&bar[B_LSE_FULL + s]);
        // dO_i (single buffer): free once dV(i-1) retired
        if (it >= 1) mbar_wait(&bar[B_DO_EMPTY], (it - 1) & 1);
        if (lane == 0) {
          SA_TR(22);
          mbar_arrive_expect_tx(&bar[B_DO_FULL], L::kTile);
          for (int pn = 0; pn < kPanels; pn++) {
            uint8_t* dst = smem + L::kDO + pn * kPanelBytes;
            if (!kPair)
              tma_load_3d(dst, &p.tdo, &bar[B_DO_FULL], 64 * pn, h, 128 * i, pol_q);
            else if (fetches(pn, it))
              tma_load_3d_mc(dst, &p.tdo, &bar[B_DO_FULL], 64 * pn, h, 128 * i, pol_q, 3);
          }
        }
      }
      if (kPair) {
        // consume the partner's last stage releases, so it cannot arrive on this CTA's
        // barriers after this CTA has exited (the final cluster barrier orders the rest)
        for (int it = n_it > 2 ? n_it - 2 : 0; it < n_it; it++)
          mbar_wait(&bar[B_Q_EMPTY + (it & 1)], (it >> 1) & 1);
        if (n_it > 0) mbar_wait(&bar[B_DO_EMPTY], (n_it - 1) & 1);
      }
    } else if (SA_PERF_TRACE && warp == 3 && lane == 0 && p.trace && blockIdx.x == p.trace_cta) {
      // perf experiments only: completion time of every MMA group, in issue order
      // dV(it) S(it+1) dQ(it) dK(it) dP(it+1)
      for (int it = 0; it < n_it && it < 16; it++) {
        mbar_wait(&bar[B_DO_EMPTY], it & 1);
        SA_TR(24);
        if (it + 1 < n_it) {
          mbar_wait(&bar[B_S_FULL], (it + 1) & 1);
          SA_TR(25);
        }
        mbar_wait(&bar[B_DQ_FULL], it & 1);
        SA_TR(26);
        mbar_wait(&bar[B_Q_EMPTY + (it & 1)], (it >> 1) & 1);
        SA_TR(27);
        if (it + 1 < n_it) {
          mbar_wait(&bar[B_DP_FULL], (it + 1) & 1);
          SA_TR(28);
        }
      }
    } else if (warp == 1) {
      // ---------------------------------------------------------- MMA issuer
      // The whole warp walks the schedule (descriptor words stay warp-uniform); one elected
      // lane issues.  Descriptor lo words: start >> 4 | LBO >> 4 << 16; hi word is shared.
      constexpr uint32_t id_s = idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t id_kv = idesc_bf16(128, D, 0, 1);
      constexpr uint32_t id_q = idesc_bf16(128, D, 1, 1);
      constexpr uint32_t hi = sdesc_hi(1024);
      const uint32_t k_km = sdesc_lo(sbase + L::kK, 16), v_km = sdesc_lo(sbase + L::kV, 16);
      const uint32_t k_mn = sdesc_lo(sbase + L::kK, kPanelBytes);
      const uint32_t do_km = sdesc_lo(sbase + L::kDO, 16);
      const uint32_t do_mn = sdesc_lo(sbase + L::kDO, kPanelBytes);
      const uint32_t ds_km = sdesc_lo(sbase + L::kDS, 16);
      const uint32_t ds_mn = sdesc_lo(sbase + L::kDS, kPanelBytes);
      auto kmaj = [](int kk) -> uint32_t {  // k-step offset inside K-major SW128 panels (16 B units)
        return ((kk >> 2) * kPanelBytes + (kk & 3) * 32) >> 4;
      };
      auto issue_s = [&](int it) {  // S^T(it) = K Q_it^T
        const int s = it & 1;
        mbar_wait(&bar[B_Q_FULL + s], (it >> 1) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a = opaque(k_km), b = opaque(sdesc_lo(sbase + L::kQ + s * L::kTile, 16));
#pragma unroll
          for (int kk = 0; kk < kKSteps; kk++)
            mma_ss2(t_st, a + kmaj(kk), hi, b + kmaj(kk), hi, id_s, kk > 0);
          mma_commit(&bar[B_S_FULL]);
        }
        __syncwarp();
        SA_TR(1);
      };
      auto issue_dp = [&](int it) {  // dP^T(it) = V dO_it^T, once dQ(it-1) left TMEM
        mbar_wait(&bar[B_DO_FULL], it & 1);
        if (it > 0) mbar_wait(&bar[B_DQ_FREE], (it - 1) & 1);
        SA_TR(2);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a = opaque(v_km), b = opaque(do_km);
#pragma unroll
          for (int kk = 0; kk < kKSteps; kk++)
            mma_ss2(t_dpt, a + kmaj(kk), hi, b + kmaj(kk), hi, id_s, kk > 0);
          mma_commit(&bar[B_DP_FULL]);
        }
        __syncwarp();
        SA_TR(3);
      };
      mbar_wait(&bar[B_KV_FULL], 0);
      {
        const int it = 0;
        SA_TR(0);
      }
      issue_s(0);
      issue_dp(0);
      for (int it = 0; it < n_it; it++) {
        const int s = it & 1;
        mbar_wait(&bar[B_P_READY], it & 1);
        SA_TR(4);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t b = opaque(do_mn);
#pragma unroll
          for (int kk = 0; kk < 8; kk++)  // P^T: q cols [0,64) at TMEM [0,32), [64,128) at [64,96)
            mma_ts2(t_dv, t_st + (kk < 4 ? kk * 8 : 64 + (kk - 4) * 8), b + kk * 128, hi, id_kv,
                    (it > 0 || kk > 0) ? 1u : 0u);
          if (kPair)
            mma_commit_mc(&bar[B_DO_EMPTY], 3);  // frees the stage in both CTAs' view
          else
            mma_commit(&bar[B_DO_EMPTY]);
        }
        __syncwarp();
        SA_TR(5);
        if (it + 1 < n_it) issue_s(it + 1);  // S^T cols are free once dV(it) read P^T
        mbar_wait(&bar[B_DS_READY], it & 1);
        SA_TR(6);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a = opaque(ds_mn), b = opaque(k_mn);
#pragma unroll
          for (int kk = 0; kk < 8; kk++)  // MN-major k-step = 16 rows = 2048 B = 128 units
            mma_ss2(t_dpt, a + kk * 128, hi, b + kk * 128, hi, id_q, kk > 0);
          mma_commit(&bar[B_DQ_FULL]);
          const uint32_t c = opaque(ds_km),
                         e = opaque(sdesc_lo(sbase + L::kQ + s * L::kTile, kPanelBytes));
#pragma unroll
          for (int kk = 0; kk < 8; kk++)
            mma_ss2(t_dk, c + kmaj(kk), hi, e + kk * 128, hi, id_kv, (it > 0 || kk > 0) ? 1u : 0u);
          // one commit: Q stage s and the dS tile are both free once dK(it) retired
          if (kPair)
            mma_commit_mc(&bar[B_Q_EMPTY + s], 3);
          else
            mma_commit(&bar[B_Q_EMPTY + s]);
        }
        __syncwarp();
        SA_TR(7);
        if (it + 1 < n_it) issue_dp(it + 1);
      }
      if (elect_one()) mma_commit(&bar[B_KV_DONE]);
      __syncwarp();
    }
  } else if (warp < 12) {
    regs_inc<152>();
    // ------------------------------------------------------------ compute WGs
    const int half = (warp - 4) >> 2;  // query columns [64*half, 64*half + 64)
    const uint32_t row = (warp & 3) * 32 + lane;
    const uint32_t lane_off = ((warp & 3) * 32) << 16;
    const int y = 128 * j + row;
    const uint32_t ds_panel = sbase + L::kDS + half * kPanelBytes;
    const bool tr = lane == 0 && warp == 4;
    for (int it = 0; it < n_it; it++) {
      const int s = it & 1;
      const int i = i0 + it % n_i;
      const bool masked = (causal && i <= j) || (i + 1) * 128 > p.c || (j + 1) * 128 > p.c || ghost;
      const uint32_t lse_a = sbase + L::kLse + s * 512 + half * 256;
      const uint32_t dsum_a = sbase + L::kDsum + s * 512 + half * 256;
      const int xbase = 128 * i + 64 * half;
      mbar_wait(&bar[B_S_FULL], it & 1);
      if (tr) SA_TR(8);
      tc_fence_after();
      mbar_wait(&bar[B_LSE_FULL + s], (it >> 1) & 1);
      if (SA_PERF_TRACE && (p.debug & 4)) {  // perf experiments only: no compute, just the hand-offs
        tc_fence_before();
        mbar_arrive(&bar[B_P_READY]);
        mbar_wait(&bar[B_DP_FULL], it & 1);
        tc_fence_after();
        if (it > 0) mbar_wait(&bar[B_Q_EMPTY + ((it - 1) & 1)], ((it - 1) >> 1) & 1);
        fence_proxy_async_smem();
        tc_fence_before();
        mbar_arrive(&bar[B_DS_READY]);
        continue;
      }
      float pv[64];
#pragma unroll
      for (int ch = 0; ch < 2; ch++) {
        uint32_t sr[32];
        SA_TMEM_LD32(t_st + lane_off + half * 64 + ch * 32, sr);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; e += 4) {
          const float4 l4 = lds128f(lse_a + (ch * 32 + e) * 4);
          const float x0 = fmaf(__uint_as_float(sr[e + 0]), p.scale_log2, -l4.x);
          const float x1 = fmaf(__uint_as_float(sr[e + 1]), p.scale_log2, -l4.y);
          const float x2 = fmaf(__uint_as_float(sr[e + 2]), p.scale_log2, -l4.z);
          const float x3 = fmaf(__uint_as_float(sr[e + 3]), p.scale_log2, -l4.w);
          if (((ch * 32 + e) / 4) % 8 < SA_BWD_POLY) {  // FMA-pipe exp2 for a share of quads
            ex2_poly2(pv[ch * 32 + e + 0], pv[ch * 32 + e + 1], x0, x1);
            ex2_poly2(pv[ch * 32 + e + 2], pv[ch * 32 + e + 3], x2, x3);
          } else {
            pv[ch * 32 + e + 0] = ex2(x0);
            pv[ch * 32 + e + 1] = ex2(x1);
            pv[ch * 32 + e + 2] = ex2(x2);
            pv[ch * 32 + e + 3] = ex2(x3);
          }
        }
        if (masked) {
#pragma unroll
          for (int e = 0; e < 32; e++)
            if (ghost || !allowed_bwd(p.kind, xbase + ch * 32 + e, y, p.c)) pv[ch * 32 + e] = 0.f;
        }
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; e++) pk[e] = pack_bf16(pv[ch * 32 + 2 * e], pv[ch * 32 + 2 * e + 1]);
        SA_TMEM_ST16(t_st + lane_off + half * 64 + ch * 16, pk);
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&bar[B_P_READY]);
      if (tr) SA_TR(10);

      mbar_wait(&bar[B_DP_FULL], it & 1);
      if (tr) SA_TR(11);
      tc_fence_after();
      // dQ/dK(it-1) must have read dS^T before it is overwritten: implied by DP_FULL(it),
      // whose commit was issued after dK(it-1) (a commit tracks ALL prior MMAs of the
      // issuing thread), so no separate wait sits on the dS -> dQ -> dP critical cycle
      if (tr) SA_TR(12);
#if SA_BWD_DP_PREFETCH
      uint32_t dr_all[64];  // both dP^T chunks in flight before the first wait
      SA_TMEM_LD32(t_dpt + lane_off + half * 64, (dr_all + 0));
      SA_TMEM_LD32(t_dpt + lane_off + half * 64 + 32, (dr_all + 32));
      tmem_ld_wait();
#endif
#pragma unroll
      for (int ch = 0; ch < 2; ch++) {
#if SA_BWD_DP_PREFETCH
        const uint32_t* dr = dr_all + ch * 32;
#else
        uint32_t dr[32];
        SA_TMEM_LD32(t_dpt + lane_off + half * 64 + ch * 32, dr);
        tmem_ld_wait();
#endif
        uint32_t dk[16];
#pragma unroll
        for (int e = 0; e < 32; e += 4) {
          const float4 d4 = lds128f(dsum_a + (ch * 32 + e) * 4);
#if SA_BWD_PACKED  // FADD2 / FMUL2: half the ALU issues of the dS arithmetic
          float t0, t1, t2, t3, a0, a1, a2, a3;
          add2(t0, t1, __uint_as_float(dr[e + 0]), __uint_as_float(dr[e + 1]), -d4.x, -d4.y);
          add2(t2, t3, __uint_as_float(dr[e + 2]), __uint_as_float(dr[e + 3]), -d4.z, -d4.w);
          mul2(a0, a1, pv[ch * 32 + e + 0], pv[ch * 32 + e + 1], t0, t1);
          mul2(a2, a3, pv[ch * 32 + e + 2], pv[ch * 32 + e + 3], t2, t3);
#else
          const float a0 = pv[ch * 32 + e + 0] * (__uint_as_float(dr[e + 0]) - d4.x);
          const float a1 = pv[ch * 32 + e + 1] * (__uint_as_float(dr[e + 1]) - d4.y);
          const float a2 = pv[ch * 32 + e + 2] * (__uint_as_float(dr[e + 2]) - d4.z);
          const float a3 = pv[ch * 32 + e + 3] * (__uint_as_float(dr[e + 3]) - d4.w);
#endif
          dk[e / 2] = pack_bf16(a0, a1);
          dk[e / 2 + 1] = pack_bf16(a2, a3);
        }
        // dS^T row `row`, this half's query columns [32ch, 32ch+32) -> 16 B chunks 4ch..4ch+3
#pragma unroll
        for (int qd = 0; qd < 4; qd++)
          sts128(ds_panel + sw128_off(row, ch * 4 + qd), dk[4 * qd], dk[4 * qd + 1], dk[4 * qd + 2],
                 dk[4 * qd + 3]);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&bar[B_DS_READY]);
      if (tr) SA_TR(13);
    }
    if (half == 0 && !ghost) {
      // ---------------------------------------------------------- dV epilogue
      mbar_wait(&bar[B_KV_DONE], 0);
      tc_fence_after();
      if (p.dv_out) {
        store_row_bf16<D>(p.dv_out, t_dv + lane_off, 1.f, 128 * j + static_cast<int>(row), g, p);
      } else {
      const uint32_t stage = sbase + L::kQ;  // Q stages are free now
#pragma unroll 1
      for (int ch = 0; ch < kChunks; ch++) {
        uint32_t o[32];
        SA_TMEM_LD32(t_dv + lane_off + ch * 32, o);
        tmem_ld_wait();
#pragma unroll
        for (int qd = 0; qd < 8; qd++)
          sts128(stage + ch * kPanelBytes + sw128_off(row, qd), o[4 * qd], o[4 * qd + 1],
                 o[4 * qd + 2], o[4 * qd + 3]);
      }
      fence_proxy_async_smem();
      named_bar_sync(2, 128);
      if (warp == 4 && lane == 0) {
        for (int ch = 0; ch < kChunks; ch++)
          tma_reduce_add_3d(&p.tdv, smem + L::kQ + ch * kPanelBytes, 32 * ch, g, 128 * j);
        bulk_commit();
        bulk_wait<0>();
      }
      }
    }
  } else {
    regs_inc<152>();
    // ------------------------------------------------------------ dQ drain + dK epilogue
    const uint32_t row = (warp & 3) * 32 + lane;
    const uint32_t lane_off = ((warp & 3) * 32) << 16;
    const bool leader = warp == 12 && lane == 0;
    for (int it = 0; it < n_it; it++) {
      const int h = g * group + it / n_i;
      const int i = i0 + it % n_i;
      mbar_wait(&bar[B_DQ_FULL], it & 1);
      if (leader) SA_TR(17);
      tc_fence_after();
      uint32_t o[kChunks][32];  // the whole dQ row, so the TMEM columns free up at once
#pragma unroll
      for (int ch = 0; ch < kChunks; ch++) SA_TMEM_LD32(t_dpt + lane_off + ch * 32, o[ch]);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(&bar[B_DQ_FREE]);
      if (leader) SA_TR(18);
      if (SA_PERF_TRACE && (p.debug & 1)) continue;
      int* sem = p.dq_sem ? p.dq_sem + (int64_t)h * p.n_t + i : nullptr;
      if (ghost || (causal && i < j)) continue;  // kPair's all-masked tiles: dQ is exactly 0
      if (sem && leader) {
        // deterministic dQ: the key tiles add into query tile i in ascending j order.  The
        // CTAs of lower j have lower blockIdx (scheduled earlier), so the wait cannot
        // deadlock; the semaphore counts this launch's contributions to tile i.
        const int want = j - p.j_begin;
        if (ld_acquire_gpu(sem) != want) {
          const uint64_t t0 = globaltimer_ns();  // bounded: trap after 4 s (as mbar_wait)
          while (ld_acquire_gpu(sem) != want)
            if (globaltimer_ns() - t0 > 4000000000ull) __trap();
        }
        fence_proxy_async_global();  // the previous adder's TMA writes before ours
      }
      __syncwarp();  // reconverge warp 12 before the named barriers below
#pragma unroll
      for (int ch = 0; ch < kChunks; ch++) {
        const uint32_t buf = sbase + L::kStg + (ch & 1) * kPanelBytes;
        if (leader) bulk_wait_read<1>();  // the reduce that last read this buffer is done
        named_bar_sync(1, 128);
#pragma unroll
        for (int qd = 0; qd < 8; qd++)
          sts128(buf + sw128_off(row, qd),
                 __float_as_uint(__uint_as_float(o[ch][4 * qd]) * p.scale),
                 __float_as_uint(__uint_as_float(o[ch][4 * qd + 1]) * p.scale),
                 __float_as_uint(__uint_as_float(o[ch][4 * qd + 2]) * p.scale),
                 __float_as_uint(__uint_as_float(o[ch][4 * qd + 3]) * p.scale));
        fence_proxy_async_smem();
        named_bar_sync(1, 128);
        if (leader) {
          if (!(SA_PERF_TRACE && (p.debug & 8)))  // perf experiments only: bit 3 stages dQ but skips the reduce
            tma_reduce_add_3d(&p.tdq, smem + L::kStg + (ch & 1) * kPanelBytes, 32 * ch, h, 128 * i);
          bulk_commit();
        }
      }
      if (sem && leader) {
        bulk_wait<0>();              // our adds are complete in global memory
        fence_proxy_async_global();
        // the last contributor of this launch leaves the semaphore zeroed for the next one
        const int j_last = causal ? min(i, p.j_begin + p.n_j - 1) : p.j_begin + p.n_j - 1;
        st_release_gpu(sem, j == j_last ? 0 : j - p.j_begin + 1);
      }
      if (leader) SA_TR(19);
    }
    if (leader) bulk_wait<0>();
    // ------------------------------------------------------------ dK epilogue
    mbar_wait(&bar[B_KV_DONE], 0);
    tc_fence_after();
    if (ghost) {
      // the ghost partner owns no key rows
    } else if (p.dk_out) {
      store_row_bf16<D>(p.dk_out, t_dk + lane_off, p.scale, 128 * j + static_cast<int>(row), g, p);
    } else {
    const uint32_t kst = sbase + L::kDO;  // dO + dS buffers (contiguous) are free now
#pragma unroll 1
    for (int ch = 0; ch < kChunks; ch++) {
      uint32_t o[32];
      SA_TMEM_LD32(t_dk + lane_off + ch * 32, o);
      tmem_ld_wait();
#pragma unroll
      for (int qd = 0; qd < 8; qd++)
        sts128(kst + ch * kPanelBytes + sw128_off(row, qd),
               __float_as_uint(__uint_as_float(o[4 * qd]) * p.scale),
               __float_as_uint(__uint_as_float(o[4 * qd + 1]) * p.scale),
               __float_as_uint(__uint_as_float(o[4 * qd + 2]) * p.scale),
               __float_as_uint(__uint_as_float(o[4 * qd + 3]) * p.scale));
    }
    fence_proxy_async_smem();
    named_bar_sync(1, 128);
    if (leader) {
      for (int ch = 0; ch < kChunks; ch++)
        tma_reduce_add_3d(&p.tdk, smem + L::kDO + ch * kPanelBytes, 32 * ch, g, 128 * j);
      bulk_commit();
      bulk_wait<0>();
    }
    }
  }
  tc_fence_before();
  if (kPair)
    cluster_sync();  // no CTA leaves while its partner's multicasts / commits may target it
  else
    __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

template <int D, bool kPair>
int launch_bwd_d(BwdParams& prm, cudaStream_t st) {
  const int smem = BwdSmem<D>::kAlloc;
  static unsigned long long attr_devices = 0;
  if (int r = set_smem_attr_once(bwd_kernel<D, kPair>, smem, &attr_devices)) return r;
  if (!kPair) {
    bwd_kernel<D, false><<<prm.n_j * prm.hkv, 512, smem, st>>>(prm);
    return check_launch("bwd_kernel");
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(((prm.n_j + 1) & ~1) * prm.hkv);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  (void)cudaLaunchKernelEx(&cfg, bwd_kernel<D, true>, prm);  // errors surface in check_launch
  return check_launch("bwd_kernel(pair)");
}

}  // namespace

int launch_bwd(const void* q, const void* k, const void* v, const void* dout, const float* lse,
               const float* dsum, float* dq, float* dk, float* dv, int64_t c, int32_t hq,
               int32_t hkv, int32_t d, float scale, int32_t kind, cudaStream_t st,
               void* dk_out, void* dv_out, int32_t kv_tile_begin, int32_t kv_tile_end,
               int32_t* dq_sem) {
  BwdParams prm;
  prm.dq_sem = dq_sem;
  prm.dk_out = static_cast<__nv_bfloat16*>(dk_out);
  prm.dv_out = static_cast<__nv_bfloat16*>(dv_out);
  if (int r = make_tmap_rows(&prm.tq, q, c, hq, d, 128)) return r;
  if (int r = make_tmap_rows(&prm.tk, k, c, hkv, d, 128)) return r;
  if (int r = make_tmap_rows(&prm.tv, v, c, hkv, d, 128)) return r;
  if (int r = make_tmap_rows(&prm.tdo, dout, c, hq, d, 128)) return r;
  if (int r = make_tmap_rows_f32(&prm.tdq, dq, c, hq, d, 128)) return r;
  if (!dk_out)
    if (int r = make_tmap_rows_f32(&prm.tdk, dk, c, hkv, d, 128)) return r;
  if (!dv_out)
    if (int r = make_tmap_rows_f32(&prm.tdv, dv, c, hkv, d, 128)) return r;
  prm.lse = lse;
  prm.dsum = dsum;
  prm.c = static_cast<int>(c);
  prm.hq = hq;
  prm.hkv = hkv;
  prm.n_t = static_cast<int>((c + 127) / 128);
  prm.j_begin = kv_tile_begin;
  prm.n_j = (kv_tile_end < 0 ? prm.n_t : kv_tile_end) - kv_tile_begin;
  if (prm.n_j <= 0) return 0;
  prm.scale = scale;
  prm.scale_log2 = scale * kLog2e;
  prm.kind = kind;
  prm.debug = 0;
  prm.trace = nullptr;
  prm.trace_cta = 0;
#if SA_PERF_TRACE
  const char* dbg = getenv("SA_BWD_DEBUG");
  prm.debug = dbg ? atoi(dbg) : 0;
  static long long* trace_buf = nullptr;
  const char* tr = getenv("SA_BWD_TRACE");  // perf experiments: dump one CTA's timeline
  if (tr) {
    if (!trace_buf) cudaMalloc(&trace_buf, 16 * 32 * sizeof(long long));
    cudaMemsetAsync(trace_buf, 0, 16 * 32 * sizeof(long long), st);
    prm.trace = trace_buf;
    prm.trace_cta = atoi(tr);
  }
#endif
  int r;
  if (SA_BWD_PAIR)
    r = d == 128 ? launch_bwd_d<128, true>(prm, st) : launch_bwd_d<64, true>(prm, st);
  else
    r = d == 128 ? launch_bwd_d<128, false>(prm, st) : launch_bwd_d<64, false>(prm, st);
#if SA_PERF_TRACE
  if (tr && r == 0) {
    long long h[16 * 32];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, trace_buf, sizeof h, cudaMemcpyDeviceToHost);
    const long long t0 = h[0];
    for (int it = 0; it < 16; it++) {
      fprintf(stderr, "it%2d", it);
      for (int k = 0; k < 29; k++) fprintf(stderr, " %6lld", h[it * 32 + k] ? h[it * 32 + k] - t0 : -1);
      fprintf(stderr, "\n");
    }
  }
#endif
  return r;
}

}  // namespace sa
