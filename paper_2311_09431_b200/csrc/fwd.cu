// K2 + K3: striped / ring block forward on tcgen05 with the LSE merge fused in the epilogue.
//
// One CTA = one head x 256 query rows (two 128-row query tiles, "Q0" and "Q1"), streaming
// 128-row key/value tiles of the held stripe.  Replaces the reference's per-(rank, round)
// block op: _process_round (simulator.py:144-186) -> classify_tiles (attention.py:213-225)
// -> accumulate_tile / _fold (attention.py:296-328) -> finalize (attention.py:331-336).
//
// Warp roles (384 threads):
//   warp 0      TMA producer: Q0/Q1 once, then K_j / V_j into a 2-stage ring.
//   warp 1      MMA issuer (one thread): S_t = Q_t K_j^T (SS), O_t += P_t V_j (TS, P in TMEM).
//   warp 2      TMEM allocator.  warp 3 idle.
//   warps 4-7   softmax for Q0 (thread = query row = TMEM lane), warps 8-11 for Q1.
// TMEM (512 cols): S0 [0,128)  S1 [128,256)  O0 [256,256+D)  O1 [256+D,256+2D);
// P_t (bf16) overwrites the first 64 columns of S_t.
// Issue order PV_0(j) S_0(j+1) PV_1(j) S_1(j+1): each softmax group overlaps the other
// group's MMAs (FA4-style ping-pong).  Online softmax in the log2 domain with lazy
// rescaling (O is only rescaled when the running max grows by > 8, i.e. 256x).
//
// Mask (attention.py:155-183, 194-210): key tile j of query tile tg is SKIP iff j > tg
// for both causal kinds; the diagonal tile applies y <= x (inclusive) or y < x (strict);
// ragged blocks (c % 128 != 0) mask y >= c.  Rows with no allowed key keep m = -inf,
// l = 0 and contribute lse = -inf / o = 0 to the merge, which leaves the carried state
// untouched (the reference leaves such rows bit-unchanged, attention.py:310-316).
#include "../../include/striped_attn.h"
// Plain try_wait loops in this kernel: the suspend hint that gains 1.2 % in the CTA-pair
// forward costs 1.5 % here (D = 64, 32k x 32).
#ifndef SA_MBAR_SUSPEND_NS
#define SA_MBAR_SUSPEND_NS 0
#endif
#include "common.cuh"
#include "internal.h"

#include <cstdio>
#include <type_traits>
#include <cstdlib>

namespace sa {
namespace {

constexpr int kStages = 2;
constexpr uint32_t kPanelBytes = 128 * 128;  // 128 rows x 64 bf16
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kRescaleThreshold = 8.0f;     // log2 units
// pairs of every 16 whose exp2 runs on the FMA-pipe polynomial.  At D = 64 the MMAs are
// half as long as at D = 128 for the same exponentials, so more of them go to the FMA
// pipe: swept 4 / 6 / 8 / 10 / 12 on B200, 8 is best (+6 % over 4 on the causal block).
#ifndef SA_FWD_POLY_D64
#define SA_FWD_POLY_D64 8
#endif
#ifndef SA_FWD_POLY_D128
#define SA_FWD_POLY_D128 4
#endif

struct FwdParams {
  CUtensorMap tq, tk, tv;
  float* o_acc;
  float* lse;
  __nv_bfloat16* out;
  unsigned long long* tiles;
  int c, hq, hkv, n_qblk;
  float scale_log2;
  int kind, first, last;
  long long* trace;  // perf experiments only: per-iteration clock64 stamps of one CTA
  int trace_cta;
};

#define SA_TR(slot)                                                                     \
  do {                                                                                  \
    if (SA_PERF_TRACE && p.trace && blockIdx.x == p.trace_cta && j < 16) p.trace[j * 32 + (slot)] = clock64(); \
  } while (0)

template <int D>
struct FwdSmem {
  static constexpr uint32_t kTile = D / 64 * kPanelBytes;  // one 128-row tile
  static constexpr uint32_t kQ0 = 0, kQ1 = kTile, kK = 2 * kTile, kV = kK + kStages * kTile;
  static constexpr uint32_t kBytes = kV + kStages * kTile + 1024;  // + alignment slack
};

__device__ __forceinline__ bool allowed(int kind, int x, int y, int c) {
  if (y >= c) return false;
  if (kind == SA_MASK_CAUSAL_INCLUSIVE) return y <= x;
  if (kind == SA_MASK_CAUSAL_EXCLUSIVE) return y < x;
  return true;
}

template <int D>
__global__ void __launch_bounds__(384, 1) fwd_kernel(const __grid_constant__ FwdParams p) {
  using L = FwdSmem<D>;
  constexpr int kPanels = D / 64;
  constexpr int kKSteps = D / 16;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  __shared__ uint64_t q_full, k_full[kStages], k_empty[kStages], v_full[kStages],
      v_empty[kStages], s_full[2], p_full[2], o_done[2];
  __shared__ uint32_t tmem_base_s;

  const uint32_t warp = warp_id(), lane = lane_id();
  const int b = blockIdx.x;
  // Head-major order keeps the K/V of ~1 head (a few MB) L2-resident while the ~148
  // concurrent CTAs stream it; within a head the heaviest query blocks go first (LPT).
  const int h = b / p.n_qblk;
  const int qb = p.n_qblk - 1 - b % p.n_qblk;
  const int kvh = h / (p.hq / p.hkv);
  const int r0 = qb * 256;
  const bool causal = p.kind != SA_MASK_FULLY_UNMASKED;
  const int n_kv = (p.c + 127) / 128;
  int n_t[2];
#pragma unroll
  for (int t = 0; t < 2; t++) {
    const int tg = qb * 2 + t;
    const bool valid = tg * 128 < p.c;
    n_t[t] = !valid ? 0 : (causal ? min(tg + 1, n_kv) : n_kv);
  }
  const int n_cta = max(n_t[0], n_t[1]);

  if (warp == 2) tmem_alloc<512>(&tmem_base_s);
  if (warp == 1 && lane == 0) {
    mbar_init(&q_full, 1);
    for (int s = 0; s < kStages; s++) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int t = 0; t < 2; t++) {
      mbar_init(&s_full[t], 1);
      mbar_init(&p_full[t], 128);
      mbar_init(&o_done[t], 1);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&p.tq);
    prefetch_tmap(&p.tk);
    prefetch_tmap(&p.tv);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base_s;
  if (warp < 4) {
   regs_dec<56>();
   if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      const uint64_t pol_q = policy_evict_first(), pol_kv = policy_evict_last();
      const int nq = n_t[1] > 0 ? 2 : 1;
      mbar_arrive_expect_tx(&q_full, nq * L::kTile);
      for (int t = 0; t < nq; t++)
        for (int pn = 0; pn < kPanels; pn++)
          tma_load_3d(smem + (t ? L::kQ1 : L::kQ0) + pn * kPanelBytes, &p.tq, &q_full, 64 * pn, h,
                      r0 + 128 * t, pol_q);
      for (int j = 0; j < n_cta; j++) {
        const int s = j % kStages;
        const uint32_t ph = (j / kStages) & 1;
        if (j >= kStages) mbar_wait(&k_empty[s], ph ^ 1);
        SA_TR(12);
        mbar_arrive_expect_tx(&k_full[s], L::kTile);
        for (int pn = 0; pn < kPanels; pn++)
          tma_load_3d(smem + L::kK + s * L::kTile + pn * kPanelBytes, &p.tk, &k_full[s], 64 * pn,
                      kvh, 128 * j, pol_kv);
        if (j >= kStages) mbar_wait(&v_empty[s], ph ^ 1);
        SA_TR(13);
        mbar_arrive_expect_tx(&v_full[s], L::kTile);
        for (int pn = 0; pn < kPanels; pn++)
          tma_load_3d(smem + L::kV + s * L::kTile + pn * kPanelBytes, &p.tv, &v_full[s], 64 * pn,
                      kvh, 128 * j, pol_kv);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // Whole warp walks the schedule (descriptor words warp-uniform); one elected lane issues.
    {
      constexpr uint32_t id_s = idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t id_o = idesc_bf16(128, D, 0, 1);
      constexpr uint32_t hi = sdesc_hi(1024);
      const uint32_t sbase = smem_u32(smem);
      auto issue_s = [&](int t, int s) {
        if (elect_one()) {
          const uint32_t a = opaque(sdesc_lo(sbase + (t ? L::kQ1 : L::kQ0), 16));
          const uint32_t b = opaque(sdesc_lo(sbase + L::kK + s * L::kTile, 16));
#pragma unroll
          for (int kk = 0; kk < kKSteps; kk++) {
            const uint32_t off = ((kk >> 2) * kPanelBytes + (kk & 3) * 32) >> 4;
            mma_ss2(tbase + t * 128, a + off, hi, b + off, hi, id_s, kk > 0);
          }
          mma_commit(&s_full[t]);
        }
        __syncwarp();
      };
      mbar_wait(&q_full, 0);
      mbar_wait(&k_full[0], 0);
      tc_fence_after();
      for (int t = 0; t < 2; t++)
        if (n_t[t] > 0) issue_s(t, 0);
      if (elect_one()) mma_commit(&k_empty[0]);
      __syncwarp();
      for (int j = 0; j < n_cta; j++) {
        const int sv = j % kStages;
        mbar_wait(&v_full[sv], (j / kStages) & 1);
        bool k_next = false;
        const int sk = (j + 1) % kStages;
        for (int t = 0; t < 2; t++) {
          if (j < n_t[t]) {
            mbar_wait(&p_full[t], j & 1);
            SA_TR(t ? 3 : 0);
            tc_fence_after();
            if (elect_one()) {
              const uint32_t b = opaque(sdesc_lo(sbase + L::kV + sv * L::kTile, kPanelBytes));
#pragma unroll
              for (int kk = 0; kk < 8; kk++)
                mma_ts2(tbase + 256 + t * D, tbase + t * 128 + kk * 8, b + kk * 128, hi, id_o,
                        (j > 0 || kk > 0) ? 1u : 0u);
              mma_commit(&o_done[t]);
            }
            __syncwarp();
            SA_TR(t ? 4 : 1);
          }
          if (j + 1 < n_t[t]) {
            if (!k_next) {
              mbar_wait(&k_full[sk], ((j + 1) / kStages) & 1);
              tc_fence_after();
              k_next = true;
            }
            issue_s(t, sk);
            SA_TR(t ? 5 : 2);
          }
        }
        if (elect_one()) {
          mma_commit(&v_empty[sv]);
          if (k_next) mma_commit(&k_empty[sk]);
        }
        __syncwarp();
      }
      if (p.tiles && lane == 0) atomicAdd(p.tiles, (unsigned long long)(n_t[0] + n_t[1]));
    }
   }
  } else {
    regs_inc<224>();
    // ------------------------------------------------------------ softmax / epilogue
    const int t = (warp - 4) >> 2;
    const uint32_t row = (warp & 3) * 32 + lane;
    const uint32_t lane_off = ((warp & 3) * 32) << 16;
    const uint32_t t_s = tbase + lane_off + t * 128;
    const uint32_t t_o = tbase + lane_off + 256 + t * D;
    const int x = r0 + t * 128 + row;  // local query row of this thread
    const int n = n_t[t];
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < n; j++) {
      mbar_wait(&s_full[t], j & 1);
      if (lane == 0 && (warp & 3) == 0) SA_TR(t ? 10 : 8);
      tc_fence_after();
      uint32_t r[128];
      SA_TMEM_LD32(t_s + 0, (r + 0));
      SA_TMEM_LD32(t_s + 32, (r + 32));
      SA_TMEM_LD32(t_s + 64, (r + 64));
      SA_TMEM_LD32(t_s + 96, (r + 96));
      tmem_ld_wait();
      // Diagonal / ragged tile: key columns >= lim are masked (y <= x, y < x, y < c).
      const bool masked = (causal && j == (qb * 2 + t)) || (j + 1) * 128 > p.c;
      float factor = 1.f;
      bool resc = false;
      // Two instantiations so the common (unmasked) tile carries no per-element selects.
      auto tile = [&](auto masked_tag) {
        constexpr bool kMasked = decltype(masked_tag)::value;
        const int lim = kMasked ? key_limit(p.kind, x, p.c, j) : 128;
        if constexpr (kMasked) mask_row(r, lim);
        const float mt = s_row_max(r) * p.scale_log2;
        if (m == -INFINITY) {
          m = mt;
        } else if (mt > m + kRescaleThreshold) {
          factor = ex2(m - mt);
          m = mt;
          resc = true;
        }
        const float neg_m = (m == -INFINITY) ? 0.f : -m;
        return s_row_exp_pack<kMasked, D == 64 ? SA_FWD_POLY_D64 : SA_FWD_POLY_D128>(
            r, p.scale_log2, neg_m, lim);
      };
      const float sum = masked ? tile(std::true_type{}) : tile(std::false_type{});
      l = l * factor + sum;
      SA_TMEM_ST32(t_s + 0, (r + 0));
      SA_TMEM_ST32(t_s + 32, (r + 32));
      if (__any_sync(0xffffffffu, resc) && j > 0) {
        mbar_wait(&o_done[t], (j - 1) & 1);
        tc_fence_after();
        tmem_scale_row<D>(t_o, factor);
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&p_full[t]);
      if (lane == 0 && (warp & 3) == 0) SA_TR(t ? 11 : 9);
    }
    if (n > 0) {
      // -------------------------------------------------------- epilogue + LSE merge
      mbar_wait(&o_done[t], (n - 1) & 1);
      tc_fence_after();
      const bool live = x < p.c;
      const float lse_blk = l > 0.f ? (m + __log2f(l)) * kLn2 : -INFINITY;
      const int64_t lse_idx = (int64_t)h * p.c + x;
      const LseMerge mw = lse_merge(lse_blk, l > 0.f ? 1.f / l : 0.f, p.first || !live,
                                    p.lse + lse_idx);
      const int64_t row_off = ((int64_t)x * p.hq + h) * D;
#pragma unroll 1
      for (int ch = 0; ch < D / 32; ch++) {
        uint32_t o[32];
        SA_TMEM_LD32(t_o + ch * 32, o);
        tmem_ld_wait();
        if (live)
          merge_store32(o, mw, p.first, p.last, p.o_acc + row_off + ch * 32,
                        p.out + row_off + ch * 32);
      }
      if (live) p.lse[lse_idx] = mw.lse_new;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

template <int D>
int launch_fwd_d(FwdParams& prm, cudaStream_t st) {
  const int smem = FwdSmem<D>::kBytes;
  static unsigned long long attr_devices = 0;
  if (int r = set_smem_attr_once(fwd_kernel<D>, smem, &attr_devices)) return r;
  const int grid = prm.n_qblk * prm.hq;
  fwd_kernel<D><<<grid, 384, smem, st>>>(prm);
  return check_launch("fwd_kernel");
}

}  // namespace

int launch_fwd(const void* q, const void* k, const void* v, float* o_acc, float* lse, void* out,
               int64_t c, int32_t hq, int32_t hkv, int32_t d, float scale, int32_t kind,
               int32_t first, int32_t last, int64_t* tiles, cudaStream_t st) {
  if (fwd_pair_enabled(d) && !(SA_PERF_TRACE && getenv("SA_FWD_TRACE")))
    return launch_fwd_pair(q, k, v, o_acc, lse, out, c, hq, hkv, scale, kind, first, last, tiles, st);
  FwdParams prm;
  if (int r = make_tmap_rows(&prm.tq, q, c, hq, d, 128)) return r;
  if (int r = make_tmap_rows(&prm.tk, k, c, hkv, d, 128)) return r;
  if (int r = make_tmap_rows(&prm.tv, v, c, hkv, d, 128)) return r;
  prm.o_acc = o_acc;
  prm.lse = lse;
  prm.out = static_cast<__nv_bfloat16*>(out);
  prm.tiles = reinterpret_cast<unsigned long long*>(tiles);
  prm.c = static_cast<int>(c);
  prm.hq = hq;
  prm.hkv = hkv;
  prm.n_qblk = static_cast<int>((c + 255) / 256);
  prm.scale_log2 = scale * 1.4426950408889634f;
  prm.kind = kind;
  prm.first = first;
  prm.last = last;
  prm.trace = nullptr;
  prm.trace_cta = 0;
#if SA_PERF_TRACE
  static long long* trace_buf = nullptr;
  const char* tr = getenv("SA_FWD_TRACE");  // perf experiments: dump one CTA's timeline
  if (tr) {
    if (!trace_buf) cudaMalloc(&trace_buf, 16 * 32 * sizeof(long long));
    cudaMemsetAsync(trace_buf, 0, 16 * 32 * sizeof(long long), st);
    prm.trace = trace_buf;
    prm.trace_cta = atoi(tr);
  }
  if (tr) {
    int r = d == 128 ? launch_fwd_d<128>(prm, st) : launch_fwd_d<64>(prm, st);
    long long hbuf[16 * 32];
    cudaStreamSynchronize(st);
    cudaMemcpy(hbuf, trace_buf, sizeof hbuf, cudaMemcpyDeviceToHost);
    const long long t0 = hbuf[12];
    for (int jj = 0; jj < 16; jj++) {
      fprintf(stderr, "j%2d", jj);
      for (int k = 0; k < 14; k++)
        fprintf(stderr, " %6lld", hbuf[jj * 32 + k] ? hbuf[jj * 32 + k] - t0 : -1);
      fprintf(stderr, "\n");
    }
    return r;
  }
#endif
  return d == 128 ? launch_fwd_d<128>(prm, st) : launch_fwd_d<64>(prm, st);
}

}  // namespace sa
