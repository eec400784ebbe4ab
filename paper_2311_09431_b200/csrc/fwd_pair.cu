// K2 + K3 for D = 128 on a CTA pair (cluster of 2, tcgen05 cta_group::2).
//
// Same block op as fwd.cu (simulator.py:144-186 -> attention.py:213-225, 296-336) with a
// different mapping onto the SM pair:
//   * a pair owns 256 query rows of one head; CTA r holds query tile tg = 2*qp + r.
//   * every MMA is M = 256 across the pair and issued by the leader (rank 0):
//       S(j)  = Q K_j^T   A = this CTA's Q tile (smem), B = K_j split by keys: CTA r holds
//                         keys [64r, 64r+64) of the tile (16 KB)
//       O    += P(j) V_j  A = P from TMEM, B = V_j split by D: CTA r holds columns
//                         [64r, 64r+64) (16 KB)
//     Per kv tile each SM reads 32+16+16 KB of operands from shared memory and receives
//     32 KB of TMA (the 1-CTA kernel: 192 + 64 KB per two tiles).
//   * S is triple-buffered in TMEM and the two softmax warpgroups take alternate kv tiles
//     (warps 4-7 even j, warps 8-11 odd j; thread = query row, all 128 key columns), so
//     one group's exponentials overlap the other's loads / maxima / stores and the
//     tensor pipe always has the next S queued.
//   * both groups share ONE running max per row: tile j hands m_j to the group of tile
//     j+1 through shared memory (a 64-thread producer/consumer named barrier per 32
//     rows).  Each group keeps its own partial row sum relative to the last max it saw;
//     the two are combined in the epilogue.  O is shared; a (lazy, > 2^8) max increase at
//     tile j rescales O after PV(j-1) and before P(j) is released.
// TMEM (512 cols, same in both CTAs): S/P buffers [0,128) [128,256) [256,384), O [384,512).
//
// Synchronisation.  Loads of both CTAs complete on the leader's q_full / k_full / v_full;
// the leader's MMA commits arrive (multicast) on s_full (after S(j)) and pv_done (after
// PV(j): frees the K/V stage and tells the softmax O is current; o_final for the last
// tile) of BOTH CTAs -- one commit per MMA group, since each commit costs tensor-pipe
// time; each softmax warp arrives remotely on the leader's p_full (8 arrivals per phase).
#include "../../include/striped_attn.h"
#include "common.cuh"
#include "internal.h"

#include <cstdio>
#include <cstdlib>

namespace sa {
namespace {

constexpr int kSt = 4;                      // K/V stages
constexpr int kSBuf = 3;                    // S/P buffers in TMEM
constexpr uint32_t kPanel = 128 * 128;      // 128 rows x 64 bf16
constexpr uint32_t kHalfPanel = 64 * 128;   // 64 rows x 64 bf16
constexpr uint32_t kQOff = 0;                             // 2 panels (this CTA's 128 rows)
constexpr uint32_t kKOff = 2 * kPanel;                    // kSt x (2 half panels)
constexpr uint32_t kVOff = kKOff + kSt * 2 * kHalfPanel;  // kSt x (1 panel: D cols [64r,64r+64))
constexpr uint32_t kMPubOff = kVOff + kSt * kPanel;       // float [2 group][128] running max
constexpr uint32_t kEpiOff = kMPubOff + 2 * 128 * 4;      // float [2 group][2 (m,l)][128]
constexpr uint32_t kBarOff = kEpiOff + 2 * 2 * 128 * 4;
constexpr uint32_t kSmemBytes = kBarOff + 256 + 1024;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kRescaleThreshold = 8.0f;
#ifndef SA_PROD_WARP
#define SA_PROD_WARP 0
#endif
#ifndef SA_FWD_POLY
#define SA_FWD_POLY 2
#endif

struct PairParams {
  CUtensorMap tq, tk, tv;
  float* o_acc;
  float* lse;
  __nv_bfloat16* out;
  unsigned long long* tiles;
  int c, hq, hkv, n_pair;
  float scale_log2;
  int kind, first, last;
  long long* trace;  // perf experiments only: per-tile clock64 stamps of the leader of pair 0
};

#define SA_TR(slot)                                                                       \
  do {                                                                                    \
    if (SA_PERF_TRACE && p.trace && blockIdx.x == 0 && j < 16) p.trace[j * 32 + (slot)] = clock64();      \
  } while (0)

struct Bars {
  uint64_t q_full, k_full[kSt], v_full[kSt], pv_done[kSt], s_full[kSBuf], p_full[kSBuf], o_final;
  uint32_t tmem_base;
};
static_assert(sizeof(Bars) <= 256, "barrier block");

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
fwd_pair_kernel(const __grid_constant__ PairParams p) {
  constexpr int D = 128;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  Bars& bar = *reinterpret_cast<Bars*>(smem + kBarOff);
  const uint32_t m_pub = smem_u32(smem + kMPubOff), epi = smem_u32(smem + kEpiOff);  // fp32 arrays

  const uint32_t warp = warp_id(), lane = lane_id(), rank = cluster_rank();
  const int pair = blockIdx.x >> 1;
  // head-major, heaviest pairs first (as fwd.cu)
  const int h = pair / p.n_pair;
  const int qp = p.n_pair - 1 - pair % p.n_pair;
  const int kvh = h / (p.hq / p.hkv);
  const int tg = qp * 2 + static_cast<int>(rank);
  const int r0 = tg * 128;
  const bool causal = p.kind != SA_MASK_FULLY_UNMASKED;
  const int n_kv = (p.c + 127) / 128;
  const int n = causal ? min(qp * 2 + 2, n_kv) : n_kv;  // kv tiles the pair walks
  const int n_mine = r0 < p.c ? (causal ? min(tg + 1, n_kv) : n_kv) : 0;

  if (warp == 2) tmem_alloc2<512>(&bar.tmem_base);
  if (warp == 1 && lane == 0) {
    mbar_init(&bar.q_full, 1);
    for (int s = 0; s < kSt; s++) {
      mbar_init(&bar.k_full[s], 1);
      mbar_init(&bar.v_full[s], 1);
      mbar_init(&bar.pv_done[s], 1);
    }
    for (int b = 0; b < kSBuf; b++) {
      mbar_init(&bar.s_full[b], 1);
      mbar_init(&bar.p_full[b], 8);
    }
    mbar_init(&bar.o_final, 1);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&p.tq);
    prefetch_tmap(&p.tk);
    prefetch_tmap(&p.tv);
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tbase = bar.tmem_base;

  if (warp < 4) {
    regs_dec<56>();
    if (warp == SA_PROD_WARP && lane == 0) {
      // ------------------------------------------------------------ TMA producer (both CTAs)
      const uint64_t pol_q = policy_evict_first(), pol_kv = policy_evict_last();
      if (rank == 0) mbar_arrive_expect_tx(&bar.q_full, 2 * 2 * kPanel);
      for (int pn = 0; pn < 2; pn++)
        tma_load_3d_pair(smem + kQOff + pn * kPanel, &p.tq, &bar.q_full, 64 * pn, h, r0, pol_q);
      for (int j = 0; j < n; j++) {
        const int s = j % kSt;
        const uint32_t ph = (j / kSt) & 1;
        if (j >= kSt) mbar_wait(&bar.pv_done[s], ph ^ 1);  // S(j-kSt) and PV(j-kSt) done
        if (rank == 0) mbar_arrive_expect_tx(&bar.k_full[s], 2 * 2 * kHalfPanel);
        for (int pn = 0; pn < 2; pn++)
          tma_load_3d_pair(smem + kKOff + s * 2 * kHalfPanel + pn * kHalfPanel, &p.tk,
                           &bar.k_full[s], 64 * pn, kvh, 128 * j + 64 * static_cast<int>(rank),
                           pol_kv);
        if (rank == 0) mbar_arrive_expect_tx(&bar.v_full[s], 2 * kPanel);
        tma_load_3d_pair(smem + kVOff + s * kPanel, &p.tv, &bar.v_full[s],
                         64 * static_cast<int>(rank), kvh, 128 * j, pol_kv);
      }
      // drain: the leader's last commits must land before this CTA may exit
      for (int j = max(0, n - kSt); j < n - 1; j++) mbar_wait(&bar.pv_done[j % kSt], (j / kSt) & 1);
      mbar_wait(&bar.o_final, 0);
    } else if (warp == 3 - SA_PROD_WARP && rank == 0 && lane == 0 && SA_PERF_TRACE && p.trace && blockIdx.x == 0) {
      // perf experiments only: completion times of S(j) / PV(j) for the first 16 tiles
      for (int j = 0; j < 16 && j < n - 1; j++) {
        mbar_wait(&bar.s_full[j % kSBuf], (j / kSBuf) & 1);
        SA_TR(5);
        mbar_wait(&bar.pv_done[j % kSt], (j / kSt) & 1);
        SA_TR(6);
      }
    } else if (warp == 1 && rank == 0) {
      // ------------------------------------------------------------ MMA issuer (leader)
      constexpr uint32_t id_s = idesc_bf16(256, 128, 0, 0);
      constexpr uint32_t id_o = idesc_bf16(256, D, 0, 1);
      constexpr uint32_t hi = sdesc_hi(1024);
      const uint32_t sbase = smem_u32(smem);
      auto issue_s = [&](int j) {
        const int s = j % kSt;
        mbar_wait(&bar.k_full[s], (j / kSt) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a = opaque(sdesc_lo(sbase + kQOff, 16));
          const uint32_t b = opaque(sdesc_lo(sbase + kKOff + s * 2 * kHalfPanel, 16));
#pragma unroll
          for (int kk = 0; kk < 8; kk++)
            mma2_ss(tbase + 128 * (j % kSBuf), a + (((kk >> 2) * kPanel + (kk & 3) * 32) >> 4), hi,
                    b + (((kk >> 2) * kHalfPanel + (kk & 3) * 32) >> 4), hi, id_s, kk > 0);
          mma2_commit_both(&bar.s_full[j % kSBuf]);
        }
        __syncwarp();
      };
      mbar_wait(&bar.q_full, 0);
      for (int j = 0; j < kSBuf && j < n; j++) issue_s(j);
      for (int j = 0; j < n; j++) {
        const int s = j % kSt;
        mbar_wait(&bar.v_full[s], (j / kSt) & 1);
        mbar_wait(&bar.p_full[j % kSBuf], (j / kSBuf) & 1);
        SA_TR(0);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t b = opaque(sdesc_lo(sbase + kVOff + s * kPanel, kPanel));
#pragma unroll
          for (int kk = 0; kk < 8; kk++)
            mma2_ts(tbase + 384, tbase + 128 * (j % kSBuf) + kk * 8, b + kk * 128, hi, id_o,
                    (j > 0 || kk > 0) ? 1u : 0u);
          // one commit per MMA group: each costs tensor-pipe time (scripts/umma_bench.cu)
          mma2_commit_both(j == n - 1 ? &bar.o_final : &bar.pv_done[s]);
        }
        __syncwarp();
        SA_TR(1);
        if (j + kSBuf < n) issue_s(j + kSBuf);
        SA_TR(2);
      }
    }
  } else {
    regs_inc<224>();
    // -------------------------------------------------------------- softmax / epilogue
    const uint32_t grp = (warp - 4) >> 2;  // takes kv tiles j = grp, grp + 2, ...
    const uint32_t rg = warp & 3;          // row group: TMEM lanes [32 rg, 32 rg + 32)
    const uint32_t row = rg * 32 + lane;
    const uint32_t lane_off = (rg * 32) << 16;
    const uint32_t bar_out = 1 + rg + 4 * grp, bar_in = 1 + rg + 4 * (grp ^ 1);
    const int x = r0 + static_cast<int>(row);
    const uint32_t t_o = tbase + lane_off + 384;
    const bool trace_lane = lane == 0 && rg == 0;

    float m_seen = -INFINITY, l = 0.f;  // this group's partial row sum is relative to m_seen
    for (int j = static_cast<int>(grp); j < n; j += 2) {
      const uint32_t buf = j % kSBuf;
      const uint32_t t_s = tbase + lane_off + 128 * buf;
      mbar_wait(&bar.s_full[buf], (j / kSBuf) & 1);
      if (trace_lane) SA_TR(grp ? 12 : 8);
      tc_fence_after();
      uint32_t r[128];
      const bool live_tile = j < n_mine;
      const bool masked = (causal && j == tg) || (j + 1) * 128 > p.c;
      int lim = 128;
      float mx = -INFINITY;
      if (live_tile) {
        SA_TMEM_LD32(t_s + 0, (r + 0));
        SA_TMEM_LD32(t_s + 32, (r + 32));
        SA_TMEM_LD32(t_s + 64, (r + 64));
        SA_TMEM_LD32(t_s + 96, (r + 96));
        tmem_ld_wait();
        if (masked) {
          lim = key_limit(p.kind, x, p.c, j);
          mask_row(r, lim);
        }
        mx = s_row_max(r);
      }
      // running max hand-off: m_{j-1} from the other group, m_j to it
      float m_prev = -INFINITY;
      if (j > 0) {
        named_bar_sync(bar_in, 64);
        m_prev = lds32f(m_pub + ((grp ^ 1) * 128 + row) * 4);
      }
      if (trace_lane) SA_TR(grp ? 13 : 9);
      const float mt = mx * p.scale_log2;
      float m_new = m_prev;
      bool resc = false;
      if (m_prev == -INFINITY) {
        m_new = mt;
      } else if (mt > m_prev + kRescaleThreshold) {
        m_new = mt;
        resc = true;
      }
      if (j + 1 < n) {
        sts32f(m_pub + (grp * 128 + row) * 4, m_new);
        named_bar_arrive(bar_out, 64);
      }
      if (m_new != m_seen) {
        l = l > 0.f ? l * ex2(m_seen - m_new) : 0.f;
        m_seen = m_new;
      }
      if (live_tile) {
        const float neg_m = (m_new == -INFINITY) ? 0.f : -m_new;
        l += masked ? s_row_exp_pack<true, SA_FWD_POLY>(r, p.scale_log2, neg_m, lim)
                    : s_row_exp_pack<false, SA_FWD_POLY>(r, p.scale_log2, neg_m, lim);
        if (trace_lane) SA_TR(grp ? 14 : 10);
        SA_TMEM_ST32(t_s + 0, (r + 0));
        SA_TMEM_ST32(t_s + 32, (r + 32));
      } else {
        uint32_t z[32];  // tile above this CTA's diagonal: P = 0
#pragma unroll
        for (int i = 0; i < 32; i++) z[i] = 0u;
        SA_TMEM_ST32(t_s + 0, z);
        SA_TMEM_ST32(t_s + 32, z);
      }
      if (__any_sync(0xffffffffu, resc)) {
        // O holds PV(0..j-1) relative to m_prev: rescale once PV(j-1) has landed
        mbar_wait(&bar.pv_done[(j - 1) % kSt], ((j - 1) / kSt) & 1);
        tc_fence_after();
        tmem_scale_row<D>(t_o, resc ? ex2(m_prev - m_new) : 1.f);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(map_to_rank(smem_u32(&bar.p_full[buf]), 0));
      if (trace_lane) SA_TR(grp ? 15 : 11);
    }
    // ---------------------------------------------------------- epilogue + LSE merge
    sts32f(epi + ((grp * 2 + 0) * 128 + row) * 4, m_seen);
    sts32f(epi + ((grp * 2 + 1) * 128 + row) * 4, l);
    mbar_wait(&bar.o_final, 0);
    tc_fence_after();
    named_bar_sync(9 + rg, 64);
    if (n_mine > 0) {
      const float m0 = lds32f(epi + (0 * 128 + row) * 4), l0 = lds32f(epi + (1 * 128 + row) * 4);
      const float m1 = lds32f(epi + (2 * 128 + row) * 4), l1 = lds32f(epi + (3 * 128 + row) * 4);
      const float m_f = fmaxf(m0, m1);  // the running max only grows: the later one
      const float l_tot = (l0 > 0.f ? l0 * ex2(m0 - m_f) : 0.f) + (l1 > 0.f ? l1 * ex2(m1 - m_f) : 0.f);
      const bool live = x < p.c;
      const float lse_blk = l_tot > 0.f ? (m_f + __log2f(l_tot)) * kLn2 : -INFINITY;
      const int64_t lse_idx = (int64_t)h * p.c + x;
      const LseMerge mw = lse_merge(lse_blk, l_tot > 0.f ? 1.f / l_tot : 0.f, p.first || !live,
                                    p.lse + lse_idx);
      const int64_t row_off = ((int64_t)x * p.hq + h) * D + grp * 64;
#pragma unroll 1
      for (int ch = 0; ch < 2; ch++) {  // this group's half of the D columns
        uint32_t o[32];
        SA_TMEM_LD32(t_o + grp * 64 + ch * 32, o);
        tmem_ld_wait();
        if (live)
          merge_store32(o, mw, p.first, p.last, p.o_acc + row_off + ch * 32,
                        p.out + row_off + ch * 32);
      }
      if (live && grp == 0) p.lse[lse_idx] = mw.lse_new;
    }
    if (p.tiles && warp == 4 && lane == 0) atomicAdd(p.tiles, (unsigned long long)n_mine);
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc2<512>(tbase);
  }
}

}  // namespace

bool fwd_pair_enabled(int32_t d) {
#if SA_PERF_TRACE
  static const bool off = getenv("SA_FWD_SINGLE") != nullptr;  // A/B against fwd.cu
#else
#ifdef SA_FWD_FORCE_SINGLE  // A/B build: the 1-CTA fwd_kernel<128> for D = 128
  constexpr bool off = true;
#else
  constexpr bool off = false;
#endif
#endif
  return d == 128 && !off;
}

int launch_fwd_pair(const void* q, const void* k, const void* v, float* o_acc, float* lse,
                    void* out, int64_t c, int32_t hq, int32_t hkv, float scale, int32_t kind,
                    int32_t first, int32_t last, int64_t* tiles, cudaStream_t st) {
  PairParams prm;
  if (int r = make_tmap_rows(&prm.tq, q, c, hq, 128, 128)) return r;
  if (int r = make_tmap_rows(&prm.tk, k, c, hkv, 128, 64)) return r;
  if (int r = make_tmap_rows(&prm.tv, v, c, hkv, 128, 128)) return r;
  prm.o_acc = o_acc;
  prm.lse = lse;
  prm.out = static_cast<__nv_bfloat16*>(out);
  prm.tiles = reinterpret_cast<unsigned long long*>(tiles);
  prm.c = static_cast<int>(c);
  prm.hq = hq;
  prm.hkv = hkv;
  prm.n_pair = static_cast<int>((c + 255) / 256);
  prm.scale_log2 = scale * 1.4426950408889634f;
  prm.kind = kind;
  prm.first = first;
  prm.last = last;
  prm.trace = nullptr;
#if SA_PERF_TRACE
  static long long* trace_buf = nullptr;
  const bool tr = getenv("SA_FWD_PAIR_TRACE") != nullptr;
#else
  constexpr bool tr = false;
  long long* trace_buf = nullptr;
#endif
  if (tr) {
    if (!trace_buf) cudaMalloc(&trace_buf, 32 * 32 * sizeof(long long));
    cudaMemsetAsync(trace_buf, 0, 32 * 32 * sizeof(long long), st);
    prm.trace = trace_buf;
  }
  static unsigned long long attr_devices = 0;
  if (int r = set_smem_attr_once(fwd_pair_kernel, kSmemBytes, &attr_devices)) return r;
  fwd_pair_kernel<<<2 * prm.n_pair * hq, 384, kSmemBytes, st>>>(prm);
#if SA_PERF_TRACE
  if (tr) {
    long long hbuf[32 * 32];
    cudaStreamSynchronize(st);
    cudaMemcpy(hbuf, trace_buf, sizeof hbuf, cudaMemcpyDeviceToHost);
    const long long t0 = hbuf[8];
    for (int jj = 0; jj < 16; jj++) {
      fprintf(stderr, "j%2d", jj);
      for (int k = 0; k < 16; k++)
        fprintf(stderr, " %6lld", hbuf[jj * 32 + k] ? hbuf[jj * 32 + k] - t0 : -1);
      fprintf(stderr, "\n");
    }
  }
#endif
  return check_launch("fwd_pair_kernel");
}

}  // namespace sa
