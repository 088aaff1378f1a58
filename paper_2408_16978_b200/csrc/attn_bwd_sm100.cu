// Backward chunk-pair attention for sm_100a (KV-stationary; tcgen05 + TMEM + TMA).
//
// One launch = one (key/value chunk j, query chunk i) step of FPDT's nested backward loop
// (fig:bw_db: "The outer loop is on key and value, while the inner one is on query"),
// or, in the resident mode, key/value chunk j against the whole query range [jC, S).
// A CTA owns one 128-row key/value tile of one KV head and walks the query tiles of the range and the
// G query heads of its group; per (query tile, head) it computes:
//   S^T  = K Q^T            P^T  = exp2(S^T*scale*log2e - lse2)       (recompute, no stored P)
//   dP^T = V dO^T           dS^T = P^T o (dP^T - D)
//   dV  += P^T dO           dK  += dS^T Q          dQ_partial = dS K  (reduced into fp32 dq_acc)
// dK/dV accumulate in TMEM across the whole walk and leave once per launch (accumulated across the
// inner loop of the offloaded schedule in fp32 HBM; final bf16 at the last inner step).
//
// Warps (448 threads):
//   0-3   softmax-gradient, query columns [0,64)   (thread = key row = TMEM lane); final dK
//   4-7   softmax-gradient, query columns [64,128)                                ; final dV
//   8-11  dQ read-out (thread = query row) and reduction into dq_acc: TMA bulk reduce-add (D <= 80)
//         or vector atomics (D = 128)
//   12    TMA producer;  13  TMEM allocator + single-thread MMA issuer
// TMEM: S^T [0,128) -> P^T bf16 [0,64) + dS^T bf16 [64,128) (A operands of dV, dK);  dP^T [128,256);
//       dS is also stored to smem (MN-major 128B-swizzled) as the A operand of dQ = dS K;
//       D <= 80: dQ [256,256+D), dK, dV next (496 columns at D = 80)  -> dP^T of the next tile can be
//                issued before the current dQ is read out;
//       D = 128: dQ aliases dP^T; dK [256,384); dV [384,512).
// MMA issue order per tile n: dV_n, dK_n, S^T_{n+1}, dQ_n, dP^T_{n+1}: S^T_{n+1} overwrites P^T_n/dS^T_n only
// after dV_n/dK_n in issue order (tcgen05 MMAs of one thread execute in order), so the next tile's
// exponentials overlap the dQ_n and dP^T_{n+1} MMAs.  dV, dK, dQ are single N = D instructions per
// 16-row contraction step (attn_tile.cuh), the minimum tcgen05 instruction count.
#include "attn_tile.cuh"
#include "kernels.h"
#include "smem_layout.cuh"
#include "tma_host.h"

#include <cstdlib>
#include <cstring>

namespace fpdt {
namespace {

using namespace ptx;

constexpr int kThreads = 448;
#ifndef FPDT_BWD_TMA_DQ
#define FPDT_BWD_TMA_DQ 1
#endif

template <int D>
struct BwdCfg {
  using T = Tile<D>;
  static constexpr bool kSepDQ = (D <= 80);
  static constexpr bool kTmaDQ = FPDT_BWD_TMA_DQ && (D <= 80);
  static constexpr int QS = 2;
  static constexpr int kStage = 2 * T::kBytes;                 // Q + dO
  static constexpr int kDS = 128 * 128 * 2;
  static constexpr int kDQ = kTmaDQ ? 128 * D * 4 : 0;
  static constexpr int kStats = 1024;                          // lse2[128] + D[128]
  static constexpr int oK = 0, oV = T::kBytes, oStage = 2 * T::kBytes;
  static constexpr int oDS = oStage + QS * kStage;
  static constexpr int oDQ = oDS + kDS;
  static constexpr int oStats = oDQ + kDQ;
  static constexpr int oBars = oStats + QS * kStats;
  static constexpr int kSmem = oBars + 256;
  // TMEM columns
  static constexpr uint32_t tS = 0, tdP = 128;
  static constexpr uint32_t tdQ = kSepDQ ? 256 : 128;
  static constexpr uint32_t tdK = kSepDQ ? 256 + D : 256;
  static constexpr uint32_t tdV = kSepDQ ? 256 + 2 * D : 384;
  static_assert(!kSepDQ || 256 + 3 * D <= 512, "TMEM budget");
};

struct TmapSet {
  CUtensorMap q, k, v, o, dq;
};

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the FMA pipe (see attn_fwd_sm100.cu): degree-3 minimax, max rel. error 7.5e-5; -127 <= x <= 127.
__device__ __forceinline__ float exp2_poly(float x) {
  x = fmaxf(x, -127.f);
  const float j = __fadd_rn(x, 12582912.f);
  const float f = __fsub_rn(x, __fsub_rn(j, 12582912.f));
  float p = fmaf(f, 0.055169348f, 0.24260798f);
  p = fmaf(p, f, 0.69326115f);
  p = fmaf(p, f, 0.9999283f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(j) << 23));
}

__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void tma_reduce_add_3d(const CUtensorMap* m, uint32_t src, int c0, int c1, int c2) {
  asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(src), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
attn_bwd_kernel(const __grid_constant__ TmapSet tm, const __grid_constant__ BwdArgs a) {
  using T = Tile<D>;
  using C = BwdCfg<D>;
  constexpr int QS = C::QS;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023) != 0) __trap();
  const uint32_t base = smem_u32(smem);
  const uint32_t sK = base + C::oK, sV = base + C::oV, sDS = base + C::oDS, sDQ = base + C::oDQ;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::oBars);
  const uint32_t b_kv = smem_u32(&bars[0]);
  auto b_qfull = [&](int s) { return smem_u32(&bars[1 + s]); };
  auto b_qempty = [&](int s) { return smem_u32(&bars[3 + s]); };
  const uint32_t b_s = smem_u32(&bars[5]), b_dp = smem_u32(&bars[6]), b_p = smem_u32(&bars[7]),
                 b_ds = smem_u32(&bars[8]), b_dsfree = smem_u32(&bars[9]), b_dqfull = smem_u32(&bars[10]),
                 b_dqempty = smem_u32(&bars[11]), b_kvdone = smem_u32(&bars[12]);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::oBars + 16 * 8);

  const uint32_t warp = warp_id(), lane = lane_id();
  const int kt = blockIdx.x;
  const int g = blockIdx.y;
  const int G = a.G;
  const int64_t kv_base = a.kv_pos0 + (int64_t)kt * 128;
  int qt_first = 0;
  const int n_qt_total = a.n_q_rows / 128;
  if (a.causal) {
    const int64_t rel = kv_base - a.q_pos0;  // first query tile that can see this key tile
    if (rel > 0) qt_first = (int)(rel / 128);
    if (qt_first > n_qt_total) qt_first = n_qt_total;
  }
  const int n_iter = (n_qt_total - qt_first) * G;
  // debug timeline (a.trace != nullptr): SM clock of protocol events of CTA (trace_cta, 0)
  const bool tracing = a.trace != nullptr && blockIdx.x == a.trace_cta && blockIdx.y == 0;
#define TRACE(ev, n)                                                        \
  do {                                                                      \
    if (tracing && (n) < 4096) a.trace[(ev) * 4096 + (n)] = clock64();      \
  } while (0)

  if (warp == 13) tmem_alloc<512>(smem_u32(tmem_slot));
  if (warp == 12 && lane == 0) {
    mbar_init(b_kv, 1);
    for (int s = 0; s < QS; ++s) {
      mbar_init(b_qfull(s), 1);
      mbar_init(b_qempty(s), 1);
    }
    mbar_init(b_s, 1);
    mbar_init(b_dp, 1);
    mbar_init(b_p, 256);
    mbar_init(b_ds, 256);
    mbar_init(b_dsfree, 1);
    mbar_init(b_dqfull, 1);
    mbar_init(b_dqempty, 128);
    mbar_init(b_kvdone, 1);
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 12) {
    // ------------------------------------------------------------------ producer
    if (elect_one() && n_iter > 0) {
      const uint64_t pol_kv = policy_evict_first(), pol_q = policy_evict_last();
      mbar_expect_tx(b_kv, 2 * T::kBytes);
      const int krow = (int)(a.kv_row0 + (int64_t)kt * 128);
      T::load(sK, &tm.k, b_kv, a.k.head0 + g, krow, pol_kv);
      T::load(sV, &tm.v, b_kv, a.v.head0 + g, krow, pol_kv);
      for (int n = 0; n < n_iter; ++n) {
        const int s = n % QS;
        if (n >= QS) mbar_wait(b_qempty(s), ((n / QS) - 1) & 1);
        TRACE(12, n);
        const int qt = qt_first + n / G, hh = n % G;
        const int h = g * G + hh;
        const uint32_t st = base + C::oStage + s * C::kStage;
        const uint32_t stats = base + C::oStats + s * C::kStats;
        const int qrow = (int)(a.q_row0 + (int64_t)qt * 128);
        mbar_expect_tx(b_qfull(s), 2 * T::kBytes + 1024);
        T::load(st, &tm.q, b_qfull(s), a.q.head0 + h, qrow, pol_q);
        T::load(st + T::kBytes, &tm.o, b_qfull(s), a.dout.head0 + h, qrow, pol_q);
        bulk_load(stats, a.lse2 + (int64_t)h * a.stat_ld + (int64_t)qt * 128, 512, b_qfull(s));
        bulk_load(stats + 512, a.Dstat + (int64_t)h * a.stat_ld + (int64_t)qt * 128, 512, b_qfull(s));
      }
    }
  } else if (warp == 13) {
    // ------------------------------------------------------------------ MMA issuer
    if (elect_one() && n_iter > 0) {
      const uint32_t idS = idesc_bf16(128, 128, 0, 0);           // S^T, dP^T: A,B K-major
      const uint32_t idG = idesc_bf16(128, D, 0, 1);             // dV, dK: A = TMEM, B MN-major
      const uint32_t idQ = idesc_bf16(128, D, 1, 1);             // dQ: A = dS MN-major smem, B = K MN-major
      const uint32_t tS = tmem + C::tS, tdP = tmem + C::tdP, tdQ = tmem + C::tdQ, tdK = tmem + C::tdK,
                     tdV = tmem + C::tdV;
      auto stage_q = [&](int n) { return base + C::oStage + (n % QS) * C::kStage; };
      auto issue_S = [&](int n) {
        const uint32_t sQ = stage_q(n);
#pragma unroll
        for (int kk = 0; kk < T::kKSteps; ++kk) mma_ss(tS, T::desc_kmajor(sK, kk), T::desc_kmajor(sQ, kk), idS, kk > 0);
        mma_commit(b_s);
      };
      auto issue_dP = [&](int n) {
        const uint32_t sO = stage_q(n) + T::kBytes;
#pragma unroll
        for (int kk = 0; kk < T::kKSteps; ++kk) mma_ss(tdP, T::desc_kmajor(sV, kk), T::desc_kmajor(sO, kk), idS, kk > 0);
        mma_commit(b_dp);
      };
      mbar_wait(b_kv, 0);
      mbar_wait(b_qfull(0), 0);
      tc_fence_after();
      issue_S(0);
      issue_dP(0);
      for (int n = 0; n < n_iter; ++n) {
        const int s = n % QS;
        const uint32_t sQ = stage_q(n), sO = sQ + T::kBytes;
        // dV += P^T dO   (A = P^T from TMEM)
        mbar_wait(b_p, n & 1);
        TRACE(4, n);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) mma_ts(tdV, tS + kk * 8, T::desc_mn(sO, kk), idG, (n > 0 || kk > 0));
        // dK += dS^T Q   (A = dS^T from TMEM)
        mbar_wait(b_ds, n & 1);
        TRACE(5, n);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) mma_ts(tdK, tS + 64 + kk * 8, T::desc_mn(sQ, kk), idG, (n > 0 || kk > 0));
        mma_commit(b_qempty(s));  // Q_n / dO_n consumed (dQ reads dS and K only)
        // S^T_{n+1} may overwrite P^T_n / dS^T_n now (dV_n, dK_n precede it in issue order)
        const bool more = n + 1 < n_iter;
        if (more) {
          mbar_wait(b_qfull((n + 1) % QS), ((n + 1) / QS) & 1);
          tc_fence_after();
          issue_S(n + 1);
          TRACE(6, n);
        }
        // dQ_n = dS K  (A = dS from smem, MN-major; its TMEM columns must be read out for n-1)
        if (n > 0) {
          mbar_wait(b_dqempty, (n - 1) & 1);
          TRACE(7, n);
          tc_fence_after();
        }
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) mma_ss(tdQ, desc_a_mn_sw128(sDS, kk), T::desc_mn(sK, kk), idQ, kk > 0);
        mma_commit(b_dqfull);
        mma_commit(b_dsfree);
        if (more) {
          if constexpr (!C::kSepDQ) {  // dP^T aliases dQ: wait until dQ_n has been read out
            mbar_wait(b_dqempty, n & 1);
            tc_fence_after();
          }
          issue_dP(n + 1);
          TRACE(8, n);
        }
      }
      mma_commit(b_kvdone);
    }
  } else if (warp < 8) {
    // ------------------------------------------------------------------ softmax gradient (key rows)
    const int half = warp >> 2;  // query columns [64*half, 64*half+64)
    const int r = (warp & 3) * 32 + lane;
    const uint32_t lane_off = ((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + C::tS + lane_off, tdP = tmem + C::tdP + lane_off;
    const int64_t kpos = kv_base + r;
    const float sl2 = a.scale_log2;
    for (int n = 0; n < n_iter; ++n) {
      const int s = n % QS;
      const int qt = qt_first + n / G;
      const float* lse2 = reinterpret_cast<const float*>(smem + C::oStats + s * C::kStats) + 64 * half;
      const float* Dq = lse2 + 128;
      mbar_wait(b_s, n & 1);
      if (warp == 0 && lane == 0) TRACE(0, n);
      tc_fence_after();
      float p[64];
      tmem_ld32(tS + 64 * half, reinterpret_cast<uint32_t*>(p));
      tmem_ld32(tS + 64 * half + 32, reinterpret_cast<uint32_t*>(p) + 32);
      tmem_wait_ld();
      if (warp == 0 && lane == 0) TRACE(13, n);
      // query column index (within the tile) < lim is masked (query position < key position)
      int64_t lim64 = (a.causal ? (kpos - (a.q_pos0 + (int64_t)qt * 128)) : -1) - 64 * half;
      const int lim = (int)(lim64 < -1 ? -1 : (lim64 > 64 ? 64 : lim64));
      if (__any_sync(0xffffffffu, lim > 0)) {
        // tile straddling the diagonal: MUFU only (maps to exact zeros under the mask)
#pragma unroll
        for (int i = 0; i < 64; ++i) {
          const float v = ex2(fmaf(p[i], sl2, -lse2[i]));
          p[i] = (i < lim) ? 0.f : v;
        }
      } else {
        // every 4th exponential on the FMA pipe (exp2_poly), the rest on MUFU
#pragma unroll
        for (int i = 0; i < 64; i += 4) {
          p[i] = ex2(fmaf(p[i], sl2, -lse2[i]));
          p[i + 1] = ex2(fmaf(p[i + 1], sl2, -lse2[i + 1]));
          p[i + 2] = ex2(fmaf(p[i + 2], sl2, -lse2[i + 2]));
          p[i + 3] = exp2_poly(fmaf(p[i + 3], sl2, -lse2[i + 3]));
        }
      }
      if (warp == 0 && lane == 0) TRACE(14, n);
#pragma unroll
      for (int c = 0; c < 64; c += 32) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) pk[i / 2] = pack_bf16x2(p[c + i], p[c + i + 1]);
        tmem_st16(tS + 32 * half + c / 2, pk);
      }
      tmem_wait_st();
      if (warp == 0 && lane == 0) TRACE(15, n);
      tc_fence_before();
      mbar_arrive(b_p);
      if (warp == 0 && lane == 0) TRACE(1, n);
      mbar_wait(b_dp, n & 1);
      if (warp == 0 && lane == 0) TRACE(2, n);
      if (n > 0) mbar_wait(b_dsfree, (n - 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < 64; c += 32) {
        // dS = P o (dP - D)
        float dp[32];
        tmem_ld32(tdP + 64 * half + c, reinterpret_cast<uint32_t*>(dp));
        tmem_wait_ld();
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const float d0 = p[c + i] * (dp[i] - Dq[c + i]);
          const float d1 = p[c + i + 1] * (dp[i + 1] - Dq[c + i + 1]);
          pk[i / 2] = pack_bf16x2(d0, d1);
        }
        tmem_st16(tS + 64 + 32 * half + c / 2, pk);
#pragma unroll
        for (int m8 = 0; m8 < 4; ++m8) {
          const uint32_t w[4] = {pk[m8 * 4], pk[m8 * 4 + 1], pk[m8 * 4 + 2], pk[m8 * 4 + 3]};
          st_shared_v4(sDS + mn_sw128_offset(64 * half + c + m8 * 8, r), w);
        }
      }
      tmem_wait_st();
      fence_async_shared();
      tc_fence_before();
      mbar_arrive(b_ds);
      if (warp == 0 && lane == 0) TRACE(3, n);
    }
    // ---- final dK (half 0) / dV (half 1), thread = key row
    const int64_t row = (int64_t)kt * 128 + r;  // row within the launch's key range
    const int hkv = a.hq / G;
    float* acc = (half ? a.dv_acc : a.dk_acc) + (row * hkv + g) * D;
    const float sc = half ? 1.f : a.scale;
    __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(half ? a.dv_out : a.dk_out);
    if (a.kv_final) out += row * a.kv_out_ld + (int64_t)(a.kv_out_head0 + g) * D;
    if (n_iter > 0) {
      mbar_wait(b_kvdone, 0);
      tc_fence_after();
    }
#pragma unroll
    for (int c = 0; c < D; c += 16) {
      float v[16];
      if (n_iter > 0) {
        tmem_ld16(tmem + (half ? C::tdV : C::tdK) + lane_off + c, reinterpret_cast<uint32_t(&)[16]>(v));
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] *= sc;
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = 0.f;
      }
      if (!a.kv_acc_init) {
#pragma unroll
        for (int i = 0; i < 16; i += 4) {
          const float4 x = *reinterpret_cast<const float4*>(acc + c + i);
          v[i] += x.x; v[i + 1] += x.y; v[i + 2] += x.z; v[i + 3] += x.w;
        }
      }
      if (a.kv_final) {
#pragma unroll
        for (int i = 0; i < 16; i += 8) {
          uint4 w;
          w.x = pack_bf16x2(v[i], v[i + 1]); w.y = pack_bf16x2(v[i + 2], v[i + 3]);
          w.z = pack_bf16x2(v[i + 4], v[i + 5]); w.w = pack_bf16x2(v[i + 6], v[i + 7]);
          *reinterpret_cast<uint4*>(out + c + i) = w;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 16; i += 4)
          *reinterpret_cast<float4*>(acc + c + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
      }
    }
  } else {
    // ------------------------------------------------------------------ dQ read-out (query rows)
    const int r = (warp - 8) * 32 + lane;
    const int t128 = threadIdx.x - 256;
    const uint32_t lane_off = ((warp & 3) * 32) << 16;
    const uint32_t tdQ = tmem + C::tdQ + lane_off;
    for (int n = 0; n < n_iter; ++n) {
      const int qt = qt_first + n / G, hh = n % G;
      const int h = g * G + hh;
      mbar_wait(b_dqfull, n & 1);
      TRACE(9, n);
      tc_fence_after();
      if constexpr (C::kTmaDQ) {
        float v[D];
#pragma unroll
        for (int c = 0; c < D; c += 16) tmem_ld16(tdQ + c, reinterpret_cast<uint32_t(&)[16]>(v[c]));
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(b_dqempty);
        TRACE(10, n);
        // the previous bulk reduce must have finished reading the staging tile
        if (t128 == 0) bulk_wait_read0();
        named_bar(1, 128);
        float* dst = reinterpret_cast<float*>(smem + C::oDQ) + r * D;
#pragma unroll
        for (int c = 0; c < D; c += 4)
          *reinterpret_cast<float4*>(dst + c) = make_float4(v[c] * a.scale, v[c + 1] * a.scale, v[c + 2] * a.scale,
                                                            v[c + 3] * a.scale);
        fence_async_shared();
        named_bar(1, 128);
        if (t128 == 0) {
          tma_reduce_add_3d(&tm.dq, sDQ, 0, qt * 128, h);
          bulk_commit();
          TRACE(11, n);
        }
      } else {
        const int64_t qrow = (int64_t)qt * 128 + r;
        float4* dst = reinterpret_cast<float4*>(a.dq_acc + (int64_t)h * a.dq_head_stride + qrow * D);
#pragma unroll
        for (int hf = 0; hf < D; hf += 64) {
          float v[64];
#pragma unroll
          for (int c = 0; c < 64; c += 16) tmem_ld16(tdQ + hf + c, reinterpret_cast<uint32_t(&)[16]>(v[c]));
          tmem_wait_ld();
          if (hf + 64 >= D) {
            tc_fence_before();
            mbar_arrive(b_dqempty);
          }
#pragma unroll
          for (int c = 0; c < 64; c += 4)
            atomicAdd(dst + (hf + c) / 4,
                      make_float4(v[c] * a.scale, v[c + 1] * a.scale, v[c + 2] * a.scale, v[c + 3] * a.scale));
        }
      }
    }
    if constexpr (C::kTmaDQ) {
      if (t128 == 0) bulk_wait0();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 13) tmem_dealloc<512>(tmem);
}

template <int D>
int launch_bwd(const BwdArgs& a, cudaStream_t s) {
  using C = BwdCfg<D>;
  TmapSet tm;
  bool ok = make_tile_tmap<D>(&tm.q, a.q.base, a.q.rows, a.q.heads);
  ok &= make_tile_tmap<D>(&tm.k, a.k.base, a.k.rows, a.k.heads);
  ok &= make_tile_tmap<D>(&tm.v, a.v.base, a.v.rows, a.v.heads);
  ok &= make_tile_tmap<D>(&tm.o, a.dout.base, a.dout.rows, a.dout.heads);
  if constexpr (C::kTmaDQ)
    ok &= make_tmap_f32_head_major(&tm.dq, a.dq_acc, a.n_q_rows, a.hq, D, a.dq_head_stride, D, 128,
                                   CU_TENSOR_MAP_SWIZZLE_NONE);
  if (!ok) return -1;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(attn_bwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    attr_set = true;
  }
  dim3 grid(a.n_kv_rows / 128, a.hq / a.G);
  attn_bwd_kernel<D><<<grid, kThreads, C::kSmem, s>>>(tm, a);
  return (int)cudaGetLastError();
}

}  // namespace

// head_dim 64 / 80 run the software-pipelined kernel (attn_bwd_pipe_sm100.cu) unless FPDT_BWD_KERNEL=v2 selects
// this one (A/B measurements); head_dim 128 always runs this one.
int launch_attn_bwd_bf16(const BwdArgs& a, int head_dim, cudaStream_t s) {
  // FPDT_BWD_KERNEL: unset = attn_bwd_q64 for d = 128 and attn_bwd_pipe for 64/80; "q64" / "pipe" / "v2" (this
  // file's kernel) force one kernel for every head_dim it supports
  static const int which = [] {
    const char* e = getenv("FPDT_BWD_KERNEL");
    if (e && strcmp(e, "v2") == 0) return 2;
    if (e && strcmp(e, "q64") == 0) return 1;
    if (e && strcmp(e, "pipe") == 0) return 3;
    return 0;
  }();
  if (which == 1 || (which == 0 && head_dim == 128)) return launch_attn_bwd_q64_bf16(a, head_dim, s);
  if (which == 0 || which == 3) return launch_attn_bwd_pipe_bf16(a, head_dim, s);
  switch (head_dim) {
    case 64: return launch_bwd<64>(a, s);
    case 80: return launch_bwd<80>(a, s);
    case 128: return launch_bwd<128>(a, s);
  }
  return -2;
}

}  // namespace fpdt
