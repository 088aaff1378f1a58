// Backward chunk-pair attention for sm_100a, head_dim 128: 64-row query tiles and a transposed dQ product.
//
// Same operation as attn_bwd_pipe_sm100.cu: one (key/value chunk j, query chunk i) step of FPDT's nested backward
// loop (fig:bw_db). The CTA is KV-stationary: one 128-row key/value tile of one KV head, walking the
// query tiles of the range and the G query heads of its group.
//   S^T  = K Q^T             P^T  = exp2(S^T*scale*log2e - lse2)       (recompute)
//   dP^T = V dO^T            dS^T = P^T o (dP^T - D)
//   dV  += P^T dO            dK  += dS^T Q
//   dQ^T = K^T dS^T          (the partial dQ of the tile, TMA bulk reduce-added into the fp32 dq accumulator)
//
// Why a separate kernel for d = 128. With 128-row query tiles, Sᵀ, dPᵀ, dK and dV fill all 512 TMEM columns, and
// K, V, the Q/dO stages and dS fill shared memory. There is then no room to stage the 64 KB dQ partial for a TMA
// reduce-add, so attn_bwd_sm100.cu reduces it with vector atomics (≈ 630 TFLOP/s).
// With 64-row query tiles:
//   * every product keeps M = 128; dQ is computed transposed (M = head_dim = 128, N = 64 query rows) with
//     A = Kᵀ read MN-major from the resident K tile and B = dS read MN-major from the tile the softmax warps
//     write;
//   * TMEM: Sᵀ 64 | dPᵀ 64 | dQᵀ 2 × 64 (double-buffered) | dK 128 | dV 128 = 512 columns;
//   * shared memory: K, V 64 KB | 3 Q + 2 dO stages 80 KB | dS 16 KB | dQ staging 2 × 32 KB | stats (226 KB).
// The dQ read-out thread owns one head_dim column (a TMEM lane) and 64 query rows. It stages [64 rows][64 cols]
// fp32 halves without swizzle (a warp writes 128 contiguous bytes per row), and each half leaves as one TMA
// reduce-add box.
// Warp roles and the issue order are those of attn_bwd_pipe_sm100.cu.
#include "attn_tile.cuh"
#include "kernels.h"
#include "smem_layout.cuh"
#include "tma_host.h"

namespace fpdt {
namespace {

using namespace ptx;

constexpr int kThreads = 512;
constexpr int kLaunchRegs = (65536 / kThreads) & ~7;  // 128
constexpr int kRegsSoftmax = 168, kRegsDQ = 104, kRegsCtl = 72;
static_assert(2 * 128 * (kRegsSoftmax - kLaunchRegs) <= 128 * (2 * kLaunchRegs - kRegsDQ - kRegsCtl), "register pool");
#ifndef FPDT_BWD_POLY_EVERY
#define FPDT_BWD_POLY_EVERY 4
#endif

constexpr int D = 128, BQ = 64;

// [R rows x 128 cols] bf16 operand tile: two 128B-swizzled atoms of [R rows x 64 cols] (TMA box = one atom)
template <int R>
struct T128 {
  static constexpr int kAtom = R * 128;
  static constexpr int kBytes = 2 * kAtom;
  // K-major (rows = M or N, contraction over the 128 columns), step kk = 16 columns
  static __device__ __forceinline__ uint64_t kmajor(uint32_t t, int kk) {
    return smem_desc(t + (kk >> 2) * kAtom + (kk & 3) * 32, 16, 1024, kSw128);
  }
  // MN-major (contraction over the R rows, M or N = the 128 columns in two atoms kAtom apart), step kk = 16 rows
  static __device__ __forceinline__ uint64_t mn(uint32_t t, int kk) { return smem_desc(t + kk * 2048, kAtom, 1024, kSw128); }
  static __device__ __forceinline__ void load(uint32_t t, const CUtensorMap* m, uint32_t bar, int head, int row0,
                                              uint64_t pol) {
    tma_load_3d(t, m, bar, 0, head, row0, pol);
    tma_load_3d(t + kAtom, m, bar, 64, head, row0, pol);
  }
};
using TK = T128<128>;
using TQ = T128<BQ>;

struct Cfg {
  static constexpr int QS = 3, OS = 2;
  static constexpr int kDS = 128 * BQ * 2;    // dS, [128 keys][64 queries] bf16, MN-major (queries contiguous)
  static constexpr int kDQH = BQ * 64 * 4;    // one staging half: [64 query rows][64 cols] fp32
  static constexpr int kStats = 2 * BQ * 4;   // lse2[64] + D[64]
  static constexpr int oK = 0, oV = TK::kBytes, oQ = 2 * TK::kBytes, oO = oQ + QS * TQ::kBytes;
  static constexpr int oDS = oO + OS * TQ::kBytes;
  static constexpr int oDQ = oDS + kDS;
  static constexpr int oStats = oDQ + 4 * kDQH;
  static constexpr int oBars = oStats + QS * kStats;
  static constexpr int kSmem = oBars + 256;
  static_assert(oDS % 1024 == 0, "swizzle atoms are 1 KB aligned");
  static_assert(kSmem <= 227 * 1024, "shared memory budget");
  static constexpr uint32_t tS = 0, tdP = 64, tdQ = 128, tdK = 256, tdV = 384;
};

struct TmapSet {
  CUtensorMap q, k, v, o, dq;
};

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 2^x for a pair on the FMA pipe (degree-3 minimax on the fraction, exponent added as an integer; max rel. error
// 7.5e-5); x clamped to >= -127
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
  x.x = fmaxf(x.x, -127.f);
  x.y = fmaxf(x.y, -127.f);
  const float2 kRnd = make_float2(12582912.f, 12582912.f);
  const float2 j = __fadd2_rn(x, kRnd);
  const float2 f = __fadd2_rn(x, __fadd2_rn(kRnd, make_float2(-j.x, -j.y)));
  float2 p = __ffma2_rn(f, make_float2(0.055169348f, 0.055169348f), make_float2(0.24260798f, 0.24260798f));
  p = __ffma2_rn(p, f, make_float2(0.69326115f, 0.69326115f));
  p = __ffma2_rn(p, f, make_float2(0.9999283f, 0.9999283f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(j.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(j.y) << 23)));
}
__device__ __forceinline__ void tma_reduce_add_3d(const CUtensorMap* m, uint32_t src, int c0, int c1, int c2) {
  asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(src), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void sts32(uint32_t addr, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}

__global__ void __launch_bounds__(kThreads, 1)
attn_bwd_q64_kernel(const __grid_constant__ TmapSet tm, const __grid_constant__ BwdArgs a) {
  using C = Cfg;
  constexpr int QS = C::QS, OS = C::OS;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = smem_u32(smem);
  const uint32_t sK = base + C::oK, sV = base + C::oV, sDS = base + C::oDS, sDQ = base + C::oDQ;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::oBars);
  auto bar = [&](int i) { return smem_u32(&bars[i]); };
  constexpr int B_KV = 0, B_QF = 1, B_QE = B_QF + QS, B_OF = B_QE + QS, B_OE = B_OF + OS, B_S = B_OE + OS,
                B_SFREE = B_S + 1, B_DP = B_SFREE + 1, B_P = B_DP + 1, B_DS = B_P + 1, B_DSFREE = B_DS + 1,
                B_DQF = B_DSFREE + 1, B_DQE = B_DQF + 2, B_KVDONE = B_DQE + 2, B_NUM = B_KVDONE + 1;
  static_assert(B_NUM <= 30, "barrier area");
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::oBars + 30 * 8);

  const uint32_t warp = warp_id(), lane = lane_id();
  const int kt = blockIdx.x;
  const int g = blockIdx.y;
  const int G = a.G;
  const int64_t kv_base = a.kv_pos0 + (int64_t)kt * 128;
  int qt_first = 0;
  const int n_qt_total = a.n_q_rows / BQ;
  if (a.causal) {
    const int64_t rel = kv_base - a.q_pos0;  // first query tile that can see this key tile
    if (rel > 0) qt_first = (int)(rel / BQ);
    if (qt_first > n_qt_total) qt_first = n_qt_total;
  }
  const int n_iter = (n_qt_total - qt_first) * G;

  if (warp == 13) tmem_alloc<512>(smem_u32(tmem_slot));
  if (warp == 12 && lane == 0) {
    mbar_init(bar(B_KV), 1);
    for (int s = 0; s < QS; ++s) {
      mbar_init(bar(B_QF + s), 1);
      mbar_init(bar(B_QE + s), 1);
    }
    for (int s = 0; s < OS; ++s) {
      mbar_init(bar(B_OF + s), 1);
      mbar_init(bar(B_OE + s), 1);
    }
    mbar_init(bar(B_S), 1);
    mbar_init(bar(B_SFREE), 256);
    mbar_init(bar(B_DP), 1);
    mbar_init(bar(B_P), 256);
    mbar_init(bar(B_DS), 256);
    mbar_init(bar(B_DSFREE), 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(bar(B_DQF + b), 1);
      mbar_init(bar(B_DQE + b), 128);
    }
    mbar_init(bar(B_KVDONE), 1);
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp >= 12) {
    setmaxnreg_dec<kRegsCtl>();
    if (warp == 12) {
      // ---------------------------------------------------------------- TMA producer
      if (elect_one() && n_iter > 0) {
        const uint64_t pol_kv = policy_evict_first(), pol_q = policy_evict_last();
        mbar_expect_tx(bar(B_KV), 2 * TK::kBytes);
        const int krow = (int)(a.kv_row0 + (int64_t)kt * 128);
        TK::load(sK, &tm.k, bar(B_KV), a.k.head0 + g, krow, pol_kv);
        TK::load(sV, &tm.v, bar(B_KV), a.v.head0 + g, krow, pol_kv);
        for (int n = 0; n < n_iter; ++n) {
          const int qs = n % QS, os = n % OS;
          const int qt = qt_first + n / G, h = g * G + n % G;
          const int qrow = (int)(a.q_row0 + (int64_t)qt * BQ);
          if (n >= QS) mbar_wait(bar(B_QE + qs), ((n / QS) - 1) & 1);
          const uint32_t fq = bar(B_QF + qs);
          const uint32_t stats = base + C::oStats + qs * C::kStats;
          mbar_expect_tx(fq, TQ::kBytes + C::kStats);
          TQ::load(base + C::oQ + qs * TQ::kBytes, &tm.q, fq, a.q.head0 + h, qrow, pol_q);
          bulk_load(stats, a.lse2 + (int64_t)h * a.stat_ld + (int64_t)qt * BQ, BQ * 4, fq);
          bulk_load(stats + BQ * 4, a.Dstat + (int64_t)h * a.stat_ld + (int64_t)qt * BQ, BQ * 4, fq);
          if (n >= OS) mbar_wait(bar(B_OE + os), ((n / OS) - 1) & 1);
          mbar_expect_tx(bar(B_OF + os), TQ::kBytes);
          TQ::load(base + C::oO + os * TQ::kBytes, &tm.o, bar(B_OF + os), a.dout.head0 + h, qrow, pol_q);
        }
      }
    } else if (warp == 13) {
      // ---------------------------------------------------------------- MMA issuer
      if (elect_one() && n_iter > 0) {
        const uint32_t idS = idesc_bf16(128, BQ, 0, 0);  // S^T, dP^T: A = K / V rows, B = Q / dO rows, K-major
        const uint32_t idG = idesc_bf16(128, D, 0, 1);   // dV, dK: A = P^T / dS^T in TMEM, B = dO / Q MN-major
        const uint32_t idQ = idesc_bf16(128, BQ, 1, 1);  // dQ^T: A = K^T (K tile MN-major), B = dS MN-major
        const uint32_t tS = tmem + C::tS, tdP = tmem + C::tdP, tdK = tmem + C::tdK, tdV = tmem + C::tdV;
        auto sQ = [&](int n) { return base + C::oQ + (n % QS) * TQ::kBytes; };
        auto sO = [&](int n) { return base + C::oO + (n % OS) * TQ::kBytes; };
        auto issue_S = [&](int n) {
          mbar_wait(bar(B_QF + n % QS), (n / QS) & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) mma_ss(tS, TK::kmajor(sK, kk), TQ::kmajor(sQ(n), kk), idS, kk > 0);
          mma_commit(bar(B_S));
        };
        auto issue_dP = [&](int n) {
          mbar_wait(bar(B_OF + n % OS), (n / OS) & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) mma_ss(tdP, TK::kmajor(sV, kk), TQ::kmajor(sO(n), kk), idS, kk > 0);
          mma_commit(bar(B_DP));
        };
        mbar_wait(bar(B_KV), 0);
        issue_S(0);
        issue_dP(0);
        // per query tile n: S^T_{n+1} after SFREE(n); dV_n after P(n); dK_n after DS(n); dP^T_{n+1} (overwrites
        // P^T_n / dS^T_n, after dV_n and dK_n in issue order); dQ^T_n into buffer n&1 once dQ^T_{n-2} is read out
        for (int n = 0; n < n_iter; ++n) {
          const bool more = n + 1 < n_iter;
          if (more) {
            mbar_wait(bar(B_SFREE), n & 1);
            issue_S(n + 1);
          }
          mbar_wait(bar(B_P), n & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < BQ / 16; ++kk)
            mma_ts(tdV, tdP + 32 * (kk >> 1) + (kk & 1) * 8, TQ::mn(sO(n), kk), idG, (n > 0 || kk > 0));
          mma_commit(bar(B_OE + n % OS));
          mbar_wait(bar(B_DS), n & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < BQ / 16; ++kk)
            mma_ts(tdK, tdP + 32 * (kk >> 1) + 16 + (kk & 1) * 8, TQ::mn(sQ(n), kk), idG, (n > 0 || kk > 0));
          mma_commit(bar(B_QE + n % QS));
          if (more) issue_dP(n + 1);
          const int buf = n & 1;
          if (n >= 2) {
            mbar_wait(bar(B_DQE + buf), ((n >> 1) - 1) & 1);
            tc_fence_after();
          }
#pragma unroll
          for (int kk = 0; kk < 128 / 16; ++kk)
            mma_ss(tmem + C::tdQ + 64 * buf, TK::mn(sK, kk), smem_desc(sDS + kk * 2048, 8192, 1024, kSw128), idQ,
                   kk > 0);
          mma_commit(bar(B_DQF + buf));
          mma_commit(bar(B_DSFREE));
        }
        mma_commit(bar(B_KVDONE));
      }
    }
  } else if (warp < 8) {
    setmaxnreg_inc<kRegsSoftmax>();
    // ------------------------------------------------------------------ softmax gradient (key rows)
    const int half = warp >> 2;  // query columns [32*half, 32*half+32) of the tile
    const int r = (warp & 3) * 32 + lane;
    uint32_t tS = tmem + C::tS + (((warp & 3) * 32) << 16) + 32 * half;
    uint32_t tdP = tS + (C::tdP - C::tS);
    asm volatile("" : "+r"(tS), "+r"(tdP));
    // key row r of the dS tile: 128 bytes (64 queries) in a 1 KB 8-row group; 16-byte chunk c at chunk c ^ (r & 7)
    const uint32_t sDSr = sDS + (uint32_t)(r >> 3) * 1024 + (uint32_t)(r & 7) * 128;
    const uint32_t xr = (uint32_t)(r & 7);
    const int64_t kpos = kv_base + r;
    const float sl2 = a.scale_log2;
    for (int n = 0; n < n_iter; ++n) {
      const int qt = qt_first + n / G;
      const float* st = reinterpret_cast<const float*>(smem + C::oStats + (n % QS) * C::kStats) + 32 * half;
      mbar_wait(bar(B_S), n & 1);
      tc_fence_after();
      float p[32];
      tmem_ld32(tS, reinterpret_cast<uint32_t*>(p));
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(bar(B_SFREE));
      // query column (within this half) < lim is masked: its query position is before the key position
      const int64_t lim64 = (a.causal ? (kpos - (a.q_pos0 + (int64_t)qt * BQ)) : -1) - 32 * half;
      const int lim = (int)(lim64 < 0 ? 0 : (lim64 > 32 ? 32 : lim64));
      if (__any_sync(0xffffffffu, lim > 0)) {
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const float4 l = *reinterpret_cast<const float4*>(st + i);
          const float2 x0 = __ffma2_rn(make_float2(p[i], p[i + 1]), make_float2(sl2, sl2), make_float2(-l.x, -l.y));
          const float2 x1 =
              __ffma2_rn(make_float2(p[i + 2], p[i + 3]), make_float2(sl2, sl2), make_float2(-l.z, -l.w));
          p[i] = i < lim ? 0.f : ex2(x0.x);
          p[i + 1] = i + 1 < lim ? 0.f : ex2(x0.y);
          p[i + 2] = i + 2 < lim ? 0.f : ex2(x1.x);
          p[i + 3] = i + 3 < lim ? 0.f : ex2(x1.y);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const float4 l = *reinterpret_cast<const float4*>(st + i);
          const float2 x0 = __ffma2_rn(make_float2(p[i], p[i + 1]), make_float2(sl2, sl2), make_float2(-l.x, -l.y));
          const float2 x1 =
              __ffma2_rn(make_float2(p[i + 2], p[i + 3]), make_float2(sl2, sl2), make_float2(-l.z, -l.w));
          p[i] = ex2(x0.x);
          p[i + 1] = ex2(x0.y);
          if ((i / 4) % (FPDT_BWD_POLY_EVERY / 2) == (FPDT_BWD_POLY_EVERY / 2) - 1) {
            const float2 e = ex2_poly2(x1);
            p[i + 2] = e.x;
            p[i + 3] = e.y;
          } else {
            p[i + 2] = ex2(x1.x);
            p[i + 3] = ex2(x1.y);
          }
        }
      }
      // dP^T_n -> registers; this half's 32 dP^T columns then receive P^T_n [0,16) and dS^T_n [16,32) (bf16)
      mbar_wait(bar(B_DP), n & 1);
      tc_fence_after();
      float dp[32];
      tmem_ld32(tdP, reinterpret_cast<uint32_t*>(dp));
      tmem_wait_ld();
      {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) pk[i / 2] = pack_bf16x2(p[i], p[i + 1]);
        tmem_st16(tdP, pk);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(bar(B_P));
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        const float4 dd = *reinterpret_cast<const float4*>(st + BQ + i);
        const float2 a0 = __fmul2_rn(make_float2(p[i], p[i + 1]),
                                     __fadd2_rn(make_float2(dp[i], dp[i + 1]), make_float2(-dd.x, -dd.y)));
        const float2 a1 = __fmul2_rn(make_float2(p[i + 2], p[i + 3]),
                                     __fadd2_rn(make_float2(dp[i + 2], dp[i + 3]), make_float2(-dd.z, -dd.w)));
        pk[i / 2] = pack_bf16x2(a0.x, a0.y);
        pk[i / 2 + 1] = pack_bf16x2(a1.x, a1.y);
      }
      tmem_st16(tdP + 16, pk);
      if (n > 0) mbar_wait(bar(B_DSFREE), (n - 1) & 1);
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const uint32_t w[4] = {pk[m * 4], pk[m * 4 + 1], pk[m * 4 + 2], pk[m * 4 + 3]};
        st_shared_v4(sDSr + ((((uint32_t)(4 * half + m)) ^ xr) << 4), w);
      }
      tmem_wait_st();
      fence_async_shared();
      tc_fence_before();
      mbar_arrive(bar(B_DS));
    }
    // ---- final dK (half 0) / dV (half 1), thread = key row
    const int64_t row = (int64_t)kt * 128 + r;
    const int hkv = a.hq / G;
    float* acc = (half ? a.dv_acc : a.dk_acc) + (row * hkv + g) * D;
    const float sc = half ? 1.f : a.scale;
    __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(half ? a.dv_out : a.dk_out);
    if (a.kv_final) out += row * a.kv_out_ld + (int64_t)(a.kv_out_head0 + g) * D;
    if (n_iter > 0) {
      mbar_wait(bar(B_KVDONE), 0);
      tc_fence_after();
    }
    const uint32_t tacc = tmem + (half ? C::tdV : C::tdK) + (((warp & 3) * 32) << 16);
#pragma unroll
    for (int c = 0; c < D; c += 16) {
      float v[16];
      if (n_iter > 0) {
        tmem_ld16(tacc + c, reinterpret_cast<uint32_t(&)[16]>(v));
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
    setmaxnreg_dec<kRegsDQ>();
    // ------------------------------------------------------------------ dQ read-out: thread = one head_dim column
    const int e = (warp & 3) * 32 + lane;  // TMEM lane of dQ^T = head_dim index
    const int chalf = e >> 6, el = e & 63;  // staging half (columns [64*chalf, +64)) and column within it
    const bool lead = el == 0;
    uint32_t tdQ = tmem + C::tdQ + (((warp & 3) * 32) << 16);
    asm volatile("" : "+r"(tdQ));
    const float sc = a.scale;
    for (int n = 0; n < n_iter; ++n) {
      const int qt = qt_first + n / G, h = g * G + n % G;
      const int buf = n & 1;
      mbar_wait(bar(B_DQF + buf), (n >> 1) & 1);
      tc_fence_after();
      float v[BQ];
      tmem_ld32(tdQ + 64 * buf, reinterpret_cast<uint32_t*>(v));
      tmem_ld32(tdQ + 64 * buf + 32, reinterpret_cast<uint32_t*>(v) + 32);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(bar(B_DQE + buf));
      if (lead) bulk_wait_read1();  // the reduce-add of tile n-2 (same staging buffer) has read its source
      named_bar(2 + chalf, 64);
      const uint32_t stg = sDQ + (uint32_t)(buf * 2 + chalf) * C::kDQH + (uint32_t)el * 4;
#pragma unroll
      for (int q = 0; q < BQ; ++q) sts32(stg + q * 256, v[q] * sc);
      fence_async_shared();
      named_bar(2 + chalf, 64);
      if (lead) {
        tma_reduce_add_3d(&tm.dq, sDQ + (uint32_t)(buf * 2 + chalf) * C::kDQH, 64 * chalf, qt * BQ, h);
        bulk_commit();
      }
    }
    if (lead) bulk_wait0();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 13) tmem_dealloc<512>(tmem);
}

}  // namespace

int launch_attn_bwd_q64_bf16(const BwdArgs& a, int head_dim, cudaStream_t s) {
  if (head_dim != D) return -2;
  TmapSet tm;
  bool ok = make_tmap_rows_heads_dim(&tm.q, a.q.base, a.q.rows, a.q.heads, D, 64, BQ, CU_TENSOR_MAP_SWIZZLE_128B);
  ok &= make_tmap_rows_heads_dim(&tm.o, a.dout.base, a.dout.rows, a.dout.heads, D, 64, BQ, CU_TENSOR_MAP_SWIZZLE_128B);
  ok &= make_tile_tmap<D>(&tm.k, a.k.base, a.k.rows, a.k.heads);
  ok &= make_tile_tmap<D>(&tm.v, a.v.base, a.v.rows, a.v.heads);
  ok &= make_tmap_f32_head_major(&tm.dq, a.dq_acc, a.n_q_rows, a.hq, D, a.dq_head_stride, 64, BQ,
                                 CU_TENSOR_MAP_SWIZZLE_NONE);
  if (!ok) return -1;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(attn_bwd_q64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem);
    attr_set = true;
  }
  attn_bwd_q64_kernel<<<dim3(a.n_kv_rows / 128, a.hq / a.G), kThreads, Cfg::kSmem, s>>>(tm, a);
  return (int)cudaGetLastError();
}

}  // namespace fpdt
