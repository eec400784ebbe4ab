// K5: striped / ring block backward on tcgen05 (no reference counterpart: ringsim has no
// backward).  Same block mask, tile classification and skipping as the forward
// (attention.py:155-183, 194-210), recomputing P from the GLOBAL lse.
//
// One CTA = one 128-row key/value tile of one kv head; it loops over the q heads of its
// GQA group and the non-SKIP 128-row query tiles, accumulating dK and dV in TMEM.
// Transposed orientation (TMEM lane = key row):
//   S^T  = K Q^T              (SS, both K-major)            -> TMEM [0,128)
//   dP^T = V dO^T             (SS, both K-major)            -> TMEM [128,256)
//   P^T  = exp2(S^T*scale*log2e - lse*log2e), dS^T = P^T o (dP^T - dsum)   (compute WG)
//   dV  += P^T dO             (TS: P^T bf16 in TMEM over S^T; dO MN-major)  -> [256,256+D)
//   dK  += dS^T Q             (SS: dS^T smem K-major; Q MN-major)           -> [256+D,256+2D)
//   dQ_i = dS K               (SS: dS = MN-major view of the same smem; K MN-major) -> [128,...)
// dQ_i is drained by a second warpgroup with fp32 vector atomics into dq_acc; dK/dV are
// added into the travelling fp32 accumulators once per CTA (the CTA owns those rows).
//
// Warps: 0 TMA producer (+ lse/dsum staging), 1 MMA issuer, 2 TMEM allocator, 3 idle,
//        4-7 compute (P^T, dS^T) + final dV, 8-11 dQ drain + final dK.
#include "../../include/striped_attn.h"
#include "common.cuh"
#include "internal.h"

namespace sa {
namespace {

constexpr uint32_t kPanelBytes = 128 * 128;
constexpr float kLog2e = 1.4426950408889634f;

struct BwdParams {
  CUtensorMap tq, tk, tv, tdo;
  const float* lse;
  const float* dsum;
  float* dq;
  float* dk;
  float* dv;
  int c, hq, hkv, n_t;
  float scale, scale_log2;
  int kind;
};

template <int D>
struct BwdSmem {
  static constexpr uint32_t kTile = D / 64 * kPanelBytes;
  static constexpr uint32_t kK = 0, kV = kTile, kQ = 2 * kTile, kDO = 4 * kTile, kDS = 6 * kTile;
  static constexpr uint32_t kLse = kDS + 2 * kPanelBytes;  // 2 stages x 128 fp32
  static constexpr uint32_t kDsum = kLse + 1024;
  static constexpr uint32_t kBar = kDsum + 1024;  // mbarriers + TMEM address (no static smem)
  static constexpr uint32_t kBytes = kBar + 128;
  static constexpr uint32_t kAlloc = kBytes + 1024 <= 232448 ? kBytes + 1024 : 232448;
};

__device__ __forceinline__ bool allowed_bwd(int kind, int x, int y, int c) {
  if (x >= c || y >= c) return false;
  if (kind == SA_MASK_CAUSAL_INCLUSIVE) return y <= x;
  if (kind == SA_MASK_CAUSAL_EXCLUSIVE) return y < x;
  return true;
}

template <int D>
__global__ void __launch_bounds__(384, 1) bwd_kernel(const __grid_constant__ BwdParams p) {
  using L = BwdSmem<D>;
  constexpr int kPanels = D / 64;
  constexpr int kKSteps = D / 16;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t &kv_full = bars[0], &st_full = bars[1], &ds_full = bars[2], &ds_empty = bars[3],
           &dq_full = bars[4], &dq_empty = bars[5], &kv_done = bars[6];
  uint64_t* q_full = bars + 7;
  uint64_t* lse_full = bars + 9;
  uint64_t* q_empty = bars + 11;
  uint32_t& tmem_base_s = *reinterpret_cast<uint32_t*>(bars + 13);

  const uint32_t warp = warp_id(), lane = lane_id();
  if (smem + L::kBytes > smem_raw + L::kAlloc) __trap();  // alignment slack exhausted

  const int j = blockIdx.x / p.hkv;  // key tile: small j = most query tiles (LPT first)
  const int g = blockIdx.x % p.hkv;
  const int group = p.hq / p.hkv;
  const bool causal = p.kind != SA_MASK_FULLY_UNMASKED;
  const int i0 = causal ? j : 0;
  const int n_i = p.n_t - i0;
  const int n_it = group * n_i;
  const float* lse_g = p.lse;

  if (warp == 2) tmem_alloc<512>(&tmem_base_s);
  if (warp == 1 && lane == 0) {
    mbar_init(&kv_full, 1);
    for (int s = 0; s < 2; s++) {
      mbar_init(&q_full[s], 1);
      mbar_init(&lse_full[s], 32);
      mbar_init(&q_empty[s], 1);
    }
    mbar_init(&st_full, 1);
    mbar_init(&ds_full, 128);
    mbar_init(&ds_empty, 1);
    mbar_init(&dq_full, 1);
    mbar_init(&dq_empty, 128);
    mbar_init(&kv_done, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base_s;
  const uint32_t t_st = tbase, t_dpt = tbase + 128, t_dv = tbase + 256, t_dk = tbase + 256 + D;

  if (warp < 4) {
    regs_dec<56>();
    if (warp == 0) {
      // ---------------------------------------------------------- producer
      const uint64_t pol_kv = policy_evict_first(), pol_q = policy_evict_last();
      if (lane == 0) {
        mbar_arrive_expect_tx(&kv_full, 2 * L::kTile);
        for (int pn = 0; pn < kPanels; pn++) {
          tma_load_3d(smem + L::kK + pn * kPanelBytes, &p.tk, &kv_full, 64 * pn, g, 128 * j, pol_kv);
          tma_load_3d(smem + L::kV + pn * kPanelBytes, &p.tv, &kv_full, 64 * pn, g, 128 * j, pol_kv);
        }
      }
      for (int it = 0; it < n_it; it++) {
        const int s = it & 1;
        const int h = g * group + it / n_i;
        const int i = i0 + it % n_i;
        if (it >= 2) mbar_wait(&q_empty[s], ((it >> 1) - 1) & 1);
        if (lane == 0) {
          mbar_arrive_expect_tx(&q_full[s], 2 * L::kTile);
          for (int pn = 0; pn < kPanels; pn++) {
            tma_load_3d(smem + L::kQ + s * L::kTile + pn * kPanelBytes, &p.tq, &q_full[s], 64 * pn,
                        h, 128 * i, pol_q);
            tma_load_3d(smem + L::kDO + s * L::kTile + pn * kPanelBytes, &p.tdo, &q_full[s],
                        64 * pn, h, 128 * i, pol_q);
          }
        }
        float* lse_s = reinterpret_cast<float*>(smem + L::kLse + s * 512);
        float* dsum_s = reinterpret_cast<float*>(smem + L::kDsum + s * 512);
#pragma unroll
        for (int e = 0; e < 4; e++) {
          const int xl = lane * 4 + e, x = 128 * i + xl;
          float lv = INFINITY, dv = 0.f;
          if (x < p.c) {
            const float raw = lse_g[(int64_t)h * p.c + x];
            lv = raw == -INFINITY ? INFINITY : raw * kLog2e;  // dead row -> P = 0
            dv = p.dsum[(int64_t)h * p.c + x];
          }
          lse_s[xl] = lv;
          dsum_s[xl] = dv;
        }
        mbar_arrive(&lse_full[s]);
      }
    } else if (warp == 1) {
      // ---------------------------------------------------------- MMA issuer
      if (lane == 0) {
        const uint32_t id_s = idesc_bf16(128, 128, 0, 0);
        const uint32_t id_kv = idesc_bf16(128, D, 0, 1);
        const uint32_t id_q = idesc_bf16(128, D, 1, 1);
        const uint32_t k_addr = smem_u32(smem + L::kK), v_addr = smem_u32(smem + L::kV);
        const uint32_t ds_addr = smem_u32(smem + L::kDS);
        mbar_wait(&kv_full, 0);
        for (int it = 0; it < n_it; it++) {
          const int s = it & 1;
          const uint32_t q_addr = smem_u32(smem + L::kQ + s * L::kTile);
          const uint32_t do_addr = smem_u32(smem + L::kDO + s * L::kTile);
          mbar_wait(&q_full[s], (it >> 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < kKSteps; kk++) {
            const uint32_t off = (kk >> 2) * kPanelBytes + (kk & 3) * 32;
            mma_ss(t_st, sdesc(k_addr + off, 16, 1024), sdesc(q_addr + off, 16, 1024), id_s, kk > 0);
          }
          if (it > 0) {
            mbar_wait(&dq_empty, (it - 1) & 1);
            tc_fence_after();
          }
#pragma unroll
          for (int kk = 0; kk < kKSteps; kk++) {
            const uint32_t off = (kk >> 2) * kPanelBytes + (kk & 3) * 32;
            mma_ss(t_dpt, sdesc(v_addr + off, 16, 1024), sdesc(do_addr + off, 16, 1024), id_s, kk > 0);
          }
          mma_commit(&st_full);
          mbar_wait(&ds_full, it & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < 8; kk++)
            mma_ts(t_dv, t_st + kk * 8, sdesc(do_addr + kk * 2048, kPanelBytes, 1024), id_kv,
                   (it > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
          for (int kk = 0; kk < 8; kk++)
            mma_ss(t_dk, sdesc(ds_addr + (kk >> 2) * kPanelBytes + (kk & 3) * 32, 16, 1024),
                   sdesc(q_addr + kk * 2048, kPanelBytes, 1024), id_kv, (it > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
          for (int kk = 0; kk < 8; kk++)
            mma_ss(t_dpt, sdesc(ds_addr + kk * 2048, kPanelBytes, 1024),
                   sdesc(k_addr + kk * 2048, kPanelBytes, 1024), id_q, kk > 0);
          mma_commit(&dq_full);
          mma_commit(&ds_empty);
          mma_commit(&q_empty[s]);
        }
        mma_commit(&kv_done);
      }
    }
  } else {
    regs_inc<224>();
    const uint32_t row = (warp & 3) * 32 + lane;
    const uint32_t lane_off = ((warp & 3) * 32) << 16;
    const int y = 128 * j + row;  // key row (compute WG) / query row within tile (dQ WG)
    if (warp < 8) {
      // ---------------------------------------------------------- compute WG: P^T, dS^T
      uint8_t* ds_smem = smem + L::kDS;
      for (int it = 0; it < n_it; it++) {
        const int s = it & 1;
        const int i = i0 + it % n_i;
        mbar_wait(&st_full, it & 1);
        tc_fence_after();
        mbar_wait(&lse_full[s], (it >> 1) & 1);
        if (it > 0) mbar_wait(&ds_empty, (it - 1) & 1);
        const float* lse_s = reinterpret_cast<const float*>(smem + L::kLse + s * 512);
        const float* dsum_s = reinterpret_cast<const float*>(smem + L::kDsum + s * 512);
        const bool masked = (causal && i == j) || (i + 1) * 128 > p.c || (j + 1) * 128 > p.c;
#pragma unroll 1
        for (int ch = 0; ch < 4; ch++) {
          uint32_t sr[32], dr[32];
          SA_TMEM_LD32(t_st + lane_off + ch * 32, sr);
          SA_TMEM_LD32(t_dpt + lane_off + ch * 32, dr);
          tmem_ld_wait();
          uint32_t pk[16], dk[16];
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            float pp[2], dd[2];
#pragma unroll
            for (int u = 0; u < 2; u++) {
              const int xl = ch * 32 + e + u;
              float pv = ex2(fmaf(__uint_as_float(sr[e + u]), p.scale_log2, -lse_s[xl]));
              if (masked && !allowed_bwd(p.kind, 128 * i + xl, y, p.c)) pv = 0.f;
              pp[u] = pv;
              dd[u] = pv * (__uint_as_float(dr[e + u]) - dsum_s[xl]);
            }
            pk[e / 2] = pack_bf16(pp[0], pp[1]);
            dk[e / 2] = pack_bf16(dd[0], dd[1]);
          }
          SA_TMEM_ST16(t_st + lane_off + ch * 16, pk);
          // dS^T row `row`, query columns [32ch, 32ch+32): panel ch/2, 16B chunks (ch&1)*4 + q
          uint8_t* panel = ds_smem + (ch >> 1) * kPanelBytes;
#pragma unroll
          for (int qd = 0; qd < 4; qd++) {
            const uint32_t off = sw128_off(row, (ch & 1) * 4 + qd);
            *reinterpret_cast<uint4*>(panel + off) =
                make_uint4(dk[4 * qd], dk[4 * qd + 1], dk[4 * qd + 2], dk[4 * qd + 3]);
          }
        }
        tmem_st_wait();
        fence_proxy_async_smem();
        tc_fence_before();
        mbar_arrive(&ds_full);
      }
      // final dV (this CTA owns key rows [128j, 128j+128) of kv head g)
      mbar_wait(&kv_done, 0);
      tc_fence_after();
      const int64_t base = ((int64_t)y * p.hkv + g) * D;
#pragma unroll 1
      for (int ch = 0; ch < D / 32; ch++) {
        uint32_t o[32];
        SA_TMEM_LD32(t_dv + lane_off + ch * 32, o);
        tmem_ld_wait();
        if (y < p.c) {
          float4* dst = reinterpret_cast<float4*>(p.dv + base + ch * 32);
#pragma unroll
          for (int e = 0; e < 8; e++) {
            float4 a = dst[e];
            a.x += __uint_as_float(o[4 * e]);
            a.y += __uint_as_float(o[4 * e + 1]);
            a.z += __uint_as_float(o[4 * e + 2]);
            a.w += __uint_as_float(o[4 * e + 3]);
            dst[e] = a;
          }
        }
      }
    } else {
      // ---------------------------------------------------------- dQ drain WG
      for (int it = 0; it < n_it; it++) {
        const int h = g * group + it / n_i;
        const int i = i0 + it % n_i;
        mbar_wait(&dq_full, it & 1);
        tc_fence_after();
        const int x = 128 * i + row;
        float* dst = p.dq + ((int64_t)x * p.hq + h) * D;
#pragma unroll 1
        for (int ch = 0; ch < D / 32; ch++) {
          uint32_t o[32];
          SA_TMEM_LD32(t_dpt + lane_off + ch * 32, o);
          tmem_ld_wait();
          if (x < p.c) {
#pragma unroll
            for (int e = 0; e < 8; e++)
              atomicAdd(reinterpret_cast<float4*>(dst + ch * 32 + 4 * e),
                        make_float4(__uint_as_float(o[4 * e]) * p.scale,
                                    __uint_as_float(o[4 * e + 1]) * p.scale,
                                    __uint_as_float(o[4 * e + 2]) * p.scale,
                                    __uint_as_float(o[4 * e + 3]) * p.scale));
          }
        }
        tc_fence_before();
        mbar_arrive(&dq_empty);
      }
      // final dK
      mbar_wait(&kv_done, 0);
      tc_fence_after();
      const int64_t base = ((int64_t)y * p.hkv + g) * D;
#pragma unroll 1
      for (int ch = 0; ch < D / 32; ch++) {
        uint32_t o[32];
        SA_TMEM_LD32(t_dk + lane_off + ch * 32, o);
        tmem_ld_wait();
        if (y < p.c) {
          float4* dst = reinterpret_cast<float4*>(p.dk + base + ch * 32);
#pragma unroll
          for (int e = 0; e < 8; e++) {
            float4 a = dst[e];
            a.x += __uint_as_float(o[4 * e]) * p.scale;
            a.y += __uint_as_float(o[4 * e + 1]) * p.scale;
            a.z += __uint_as_float(o[4 * e + 2]) * p.scale;
            a.w += __uint_as_float(o[4 * e + 3]) * p.scale;
            dst[e] = a;
          }
        }
      }
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
int launch_bwd_d(BwdParams& prm, cudaStream_t st) {
  const int smem = BwdSmem<D>::kAlloc;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(bwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr_set = true;
  }
  bwd_kernel<D><<<prm.n_t * prm.hkv, 384, smem, st>>>(prm);
  return check_launch("bwd_kernel");
}

}  // namespace

int launch_bwd(const void* q, const void* k, const void* v, const void* dout, const float* lse,
               const float* dsum, float* dq, float* dk, float* dv, int64_t c, int32_t hq,
               int32_t hkv, int32_t d, float scale, int32_t kind, cudaStream_t st) {
  BwdParams prm;
  if (int r = make_tmap_rows(&prm.tq, q, c, hq, d, 128)) return r;
  if (int r = make_tmap_rows(&prm.tk, k, c, hkv, d, 128)) return r;
  if (int r = make_tmap_rows(&prm.tv, v, c, hkv, d, 128)) return r;
  if (int r = make_tmap_rows(&prm.tdo, dout, c, hq, d, 128)) return r;
  prm.lse = lse;
  prm.dsum = dsum;
  prm.dq = dq;
  prm.dk = dk;
  prm.dv = dv;
  prm.c = static_cast<int>(c);
  prm.hq = hq;
  prm.hkv = hkv;
  prm.n_t = static_cast<int>((c + 127) / 128);
  prm.scale = scale;
  prm.scale_log2 = scale * kLog2e;
  prm.kind = kind;
  return d == 128 ? launch_bwd_d<128>(prm, st) : launch_bwd_d<64>(prm, st);
}

}  // namespace sa
