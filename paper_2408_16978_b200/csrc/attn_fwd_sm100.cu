// Forward chunk-pair attention for sm_100a: TMA-fed tcgen05 MMAs with TMEM accumulators.
//
// Computes, for one (query range, key/value range) pair of FPDT's chunk loop (PAPER.md L218-230,
// fig:pipele_case2), the online-softmax attention of the query rows against the key/value rows and
// merges it with the running partial result of earlier pairs by log-sum-exp (the "online attention
// policy").  Causal masking on global token positions (key pos <= query pos; reading R3).
//
// CTA = 2 query tiles of 128 rows of ONE query head (sharing every K/V tile), 12 warps (3 warpgroups):
//   WG0 (0-3)   softmax + correction + epilogue of query tile 0 (thread = query row = TMEM lane)
//   WG1 (4-7)   same for query tile 1
//   WG2 (8)     TMA producer (Q once, then a K/V ring of kStages stages); (9) TMEM allocator +
//               single-thread tcgen05.mma issuer; (10, 11) idle
// (Measured alternative, not kept: two threads per row, 16 softmax warps — the exponential phase of a tile took
// as long, the pipes being shared per SMSP, and the registers per thread dropped to 104.)
// TMEM (512 columns): S0 [0,128) S1 [128,256) O0 [256,256+NO) O1 [384,384+NO); P_t (bf16) aliases S_t[0,64).
// MMA order per key tile j:  PV0_j, S0_{j+1}, PV1_j, S1_{j+1} — tcgen05 MMAs of one thread execute in
// issue order, so S_t{j+1} overwriting P_t_j after PV_t_j is safe, and the commit that signals S_t{j+1}
// also guarantees PV_t_j has finished (so the softmax warps may rescale O_t in TMEM then).
// Softmax (the bottleneck at d <= 80: per (row, key) the exponential costs more than the 4d MMA FLOPs):
//   * row max with three-input FMNMX3, scale/subtract with packed FFMA2;
//   * a fifth (d = 80) / an eighth (d = 128) of the exponential pairs as a degree-3 polynomial on the FMA pipe, the
//     rest on MUFU (FwdCfg::kPolyEvery);
//   * d = 80: the row sum of P comes from the tensor core — each V stage carries a 16-column atom of ones,
//     so PV has N = 96 and O column 80 accumulates sum(P) with the same rescaling as O (and the same bf16 P
//     the numerator uses); d = 64 / 128 sum with packed FADD2.
// Lazy rescale: the running max used for exponentiation is only raised when a row max exceeds it by
// more than 8 (log2 units), bounding P by 2^8 (exact result either way; rescale skipped otherwise).
#include <cuda_fp16.h>

#include "attn_tile.cuh"
#include "kernels.h"
#include "tma_host.h"

namespace fpdt {
namespace {

using namespace ptx;

constexpr int kThreads = 384;
// setmaxnreg budget: the CTA's register pool is what the launch allocated (kLaunchRegs per thread); the two
// softmax warpgroups may only grow by what WG2 gives back (an over-subscribed setmaxnreg.inc never returns)
constexpr int kLaunchRegs = (65536 / kThreads) & ~7;  // 168
// measured (tools/gpu_regs_sweep.sh, d = 80 C = 64K pair): 200/88 -> 958-988, 208/88 -> 943-968 TFLOP/s
#ifndef FPDT_FWD_REGS_SOFTMAX
#define FPDT_FWD_REGS_SOFTMAX 200
#define FPDT_FWD_REGS_OTHER 88
#endif
constexpr int kRegsSoftmax = FPDT_FWD_REGS_SOFTMAX, kRegsOther = FPDT_FWD_REGS_OTHER;
static_assert(2 * 128 * (kRegsSoftmax - kLaunchRegs) <= 128 * (kLaunchRegs - kRegsOther), "register pool");
constexpr float kRescaleThreshold = 8.0f;
// One exponential pair in N on the FMA pipe, the rest on MUFU (0 = all MUFU), per head_dim.  Measured on the
// C = 64K, 32-head diagonal pair (tools/gpu_poly_sweep_fwd.sh, two sessions; run-to-run noise about 2%):
//   d = 80:  0, 1, 2, 3 -> 800, 669, 811, 865; 4 -> 940-948 / 966-985; 5 -> 954-955 / 957-987; 6 -> 915-935; 8 -> 902-941
//   d = 128: 0 -> 1147-1149; 4 -> 1142-1145; 5 -> 1147-1148; 6 -> 1151-1159; 8 -> 1147-1162; 12, 16 -> 1139-1152
// Inside the bench step on one box (tools/gpu_ab_fwdpoly.sh), d = 80: 4 -> 895, 5 -> 910, 6 -> 876 TFLOP/s.
// With the MMA-SMSP split below (round 2, bench step, same box, A/B/A/B): 4 -> fwd 909, 5 -> 901 TFLOP/s (and 4 with no
// MMA-SMSP split 894-896).
#ifndef FPDT_FWD_POLY_EVERY
#define FPDT_FWD_POLY_EVERY 4
#endif
#ifndef FPDT_FWD_STAGES
#define FPDT_FWD_STAGES 3  // K/V ring depth at d <= 80 (d = 128: 2, the shared-memory limit); in the bench step on one
                           // box (tools/gpu_ab_stages.sh) 3 stages: fwd 912, 4 stages: 885-886 TFLOP/s
#endif
// The softmax warps that share an SMSP with the MMA-issuing warp (9: warps 1 and 5) run one exponential pair in
// FPDT_FWD_POLY_MMA_SMSP on the FMA pipe (0 = the same split as the others).  MUFU instructions go through the SMSP's
// MIO queue, where the MMA instructions waiting for the tensor pipe hold them up: per-warp traces (tools/trace_pair.py)
// showed warp 1 finishing its exponentials ~600 clk after warps 2 and 3 every key tile, and PV_0 waits for the slowest
// warp.  Measured (round 2, same box): 3 -> the four warps even, standalone pair 953 vs 947, in the bench step fwd 912
// vs 891 TFLOP/s; 4 -> 891; 2 -> 901 standalone (warp 1 then FMA-bound).  (Also measured: making the MMA thread wait
// for each MMA group to complete before issuing the next evens the warps too, but serialises the pipe: 870-917.  A third
// code path -- warps 0 and 4, beside the TMA producer, with their own split -- dropped the forward to 785-803 in the
// step: the unrolled exponential loops are large, and each SMSP's path has to stay in the instruction caches.  Also
// measured and not kept: exponentials with the running max first and the row max formed alongside them (a second
// pass only when a rescale is due; the same results): 748 vs 893 in the step -- the restructured loop costs more than
// the ~290 clk row-max phase it takes off the critical path.  The producer as lane 1 of the MMA warp (SMSP 0 free of
// control threads): 651 vs 766 -- and the control roles selected by `lane == 0` instead of elect.sync alone already
// cost 905 -> 766 TFLOP/s in the step.)
#ifndef FPDT_FWD_POLY_MMA_SMSP
#define FPDT_FWD_POLY_MMA_SMSP 3
#endif
// P aliased onto S (d = 128): PV issued in FPDT_FWD_SPLIT_PV key chunks (1, 2 or 4), each as soon as its P is in TMEM,
// so that the first half of PV_t(j) runs during the exponentials of keys 64-127 (S_t(j+1) has to wait for all of PV_t(j)
// there).  Measured (C = 64K, 32 x 128, diagonal / full pair, same box): 1 -> 1131 / 1151-1158, 2 -> 1160-1172 /
// 1181-1186, 4 -> 1149 / 1155 TFLOP/s.
#ifndef FPDT_FWD_SPLIT_PV
#define FPDT_FWD_SPLIT_PV 2
#endif
// d = 128 with the split PV (round 2, C = 64K, 32 x 128, diagonal / full pair, same box): 3 -> 1174 / 1197,
// 4 -> 1172 / 1193-1195, 5 -> 1182-1188 / 1193-1194, 6 -> 1169 / 1181, 8 -> 1165-1170 / 1179-1180, 12 -> 1175 / 1179
#ifndef FPDT_FWD_POLY_EVERY_D128
#define FPDT_FWD_POLY_EVERY_D128 5
#endif

template <int D>
struct FwdCfg {
  using T = Tile<D>;
  static constexpr bool kSumMMA = (D == 80);     // row sums from a ones column of V (SW32 atoms only)
  static constexpr int NO = kSumMMA ? D + 16 : D;  // PV N / O columns
  // separate P buffer (d <= 80): S0, S1, P, O0, O1 fit the 512 TMEM columns, so S_t(j+1) can be computed while the
  // softmax of S_t(j) runs; d = 128 keeps P aliased onto S_t (S_t(j+1) then waits for PV_t(j))
  static constexpr bool kSepP = 2 * 128 + 64 + 2 * NO <= 512;
  static constexpr uint32_t tP = 256, tO0 = kSepP ? 320 : 256, tOstride = kSepP ? NO : 128;
  static constexpr int kStages = (D == 128) ? 2 : FPDT_FWD_STAGES;
  // P aliased onto S (d = 128): PV issued in FPDT_FWD_SPLIT_PV key chunks (1, 2 or 4; see the macro)
  static constexpr int kPVChunks = kSepP ? 1 : FPDT_FWD_SPLIT_PV;
  static_assert(kPVChunks == 1 || kPVChunks == 2 || kPVChunks == 4, "PV chunks");
  static constexpr int kPolyEvery = (D == 128) ? FPDT_FWD_POLY_EVERY_D128 : FPDT_FWD_POLY_EVERY;
  static constexpr int kQBytes = 2 * T::kBytes;
  static constexpr int kOnes = kSumMMA ? 128 * 16 * 2 : 0;      // the ones atom right after each V tile
  static constexpr int kStageBytes = 2 * T::kBytes + kOnes;       // K + V (+ ones)
  static constexpr int kSmem = kQBytes + kStages * kStageBytes + 1024;
};

struct TmapSet {
  CUtensorMap q, k, v;
  CUtensorMap k64, v64;  // 64-row boxes: each CTA of a cluster pair multicasts one half of a K / V tile (MC)
};

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float max3(float a, float b, float c) {
  float y;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(y) : "f"(a), "f"(b), "f"(c));
  return y;
}

// (Measured and not kept: the MUFU exponentials as ex2.approx.f16x2 on f16-rounded arguments (ptxas splits it into two
// MUFU.EX2.F16 and a PRMT, no faster per element than MUFU.EX2): with a conversion back to bf16, 924 vs 956 TFLOP/s on
// the d = 80 pair; with fp16 P and an fp16 PV product (V converted in shared memory by the idle warps), 844 vs 954
// (round 2, tools/gpu_ab.sh) — more accurate (lse error 2x lower, dQ on drift32 3.4e-3 vs 8.3e-3) but slower.  A
// mixed fp16 x bf16 kind::f16 MMA is an illegal instruction.)

// P = exp2(x*sl2 - mb) for the 128 columns of a row, packed to bf16 and stored to TMEM columns [tS, tS+64); returns
// the sum of the fp32 values when kSum (else 0).  kEvery > 0: every kEvery-th pair on the FMA pipe.
template <int kEvery, bool kSum, bool kStore = true>
__device__ __forceinline__ float exp_pack_store(const float* x, float sl2, float mb, uint32_t tS,
                                                uint32_t* pko = nullptr, int c0 = 0, int c1 = 128) {
  float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
  const float2 s2 = make_float2(sl2, sl2), nm = make_float2(-mb, -mb);
#pragma unroll
  for (int c = 0; c < 128; c += 32) {
    if (c < c0 || c >= c1) continue;  // c0, c1 are compile-time after unrolling
    uint32_t pkl[16];
    uint32_t* pk = kStore ? pkl : pko + c / 2;
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      const float2 e = __ffma2_rn(make_float2(x[c + i], x[c + i + 1]), s2, nm);
      float2 pr;
      if (kEvery > 0 && (i / 2) % (kEvery > 0 ? kEvery : 1) == kEvery - 1) {
        pr = ex2_poly2(e);
      } else {
        pr = make_float2(ex2(e.x), ex2(e.y));
      }
      if (kSum) {
        if ((i / 2) & 1)
          acc1 = __fadd2_rn(acc1, pr);
        else
          acc0 = __fadd2_rn(acc0, pr);
      }
      pk[i / 2] = pack_bf16x2(pr.x, pr.y);
    }
    if (kStore) tmem_st16(tS + c / 2, pk);
  }
  return kSum ? (acc0.x + acc0.y) + (acc1.x + acc1.y) : 0.f;
}

// MC: clusters of two CTAs on adjacent query-tile pairs of one head, which walk the same key / value tiles (for the
// causal diagonal the pair's longer range; the shorter CTA's extra tiles are fully masked); each CTA loads one 64-row
// half of every K and V tile and multicasts it into both, and a stage is refilled once both have consumed it.
#ifndef FPDT_FWD_MC
#define FPDT_FWD_MC 1
#endif
template <int D, bool MC>
__global__ void __launch_bounds__(kThreads, 1)
attn_fwd_kernel(const __grid_constant__ TmapSet tm, const __grid_constant__ FwdArgs a) {
  using T = Tile<D>;
  using C = FwdCfg<D>;
  constexpr int ST = C::kStages;
  constexpr int kPVChunks = C::kPVChunks;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar_q, bar_k[ST], bar_v[ST], bar_kv_empty[ST], bar_s[2], bar_p[2], bar_o[2], bar_sfree[2],
      bar_pvdone[2], bar_pa[2][3];
  __shared__ uint32_t tmem_slot;

  const uint32_t warp = warp_id(), lane = lane_id();
  const uint32_t sQ = smem_u32(smem);
  const uint32_t sKV = sQ + C::kQBytes;
  const int h = blockIdx.y;
  const int g = h / a.G;
  // longest-first: for the causal diagonal block the last query tiles have the most key tiles
  const int pair = gridDim.x - 1 - blockIdx.x;
  const int64_t q_pos_first = a.q_pos0 + (int64_t)pair * 256;
  int n_tiles = a.n_kv_rows / 128;
  const uint32_t crank = MC ? cluster_ctarank() : 0;
  if (a.causal) {
    // keys visible to the last row of the CTA (MC: of the cluster's later query-tile pair, rank 0)
    const int64_t last_first = MC ? a.q_pos0 + (int64_t)(gridDim.x - 1 - (blockIdx.x & ~1u)) * 256 : q_pos_first;
    const int64_t reach = last_first + 256 - a.kv_pos0;
    const int64_t need = (reach + 127) / 128;
    n_tiles = (int)(need < n_tiles ? need : n_tiles);
  }
  const bool tracing = a.trace != nullptr && blockIdx.x == a.trace_cta && blockIdx.y == 0;
#define TRACE(ev, n)                                                        \
  do {                                                                      \
    if (tracing && (n) < 4096) a.trace[(ev) * 4096 + (n)] = clock64();      \
  } while (0)

  if (warp == 9) tmem_alloc<512>(smem_u32(&tmem_slot));
  if constexpr (C::kSumMMA) {
    // the ones atom after every V tile (constant; MN-major B columns D..D+15 of PV): all 16 columns = 1.0, so
    // the swizzle does not matter and O column D accumulates sum(P)
    if (warp >= 10) {
      const int t = threadIdx.x - 320;
      for (int s2 = 0; s2 < ST; ++s2) {
        uint4* dst = reinterpret_cast<uint4*>(smem + C::kQBytes + s2 * C::kStageBytes + 2 * T::kBytes);
        for (int i = t; i < C::kOnes / 16; i += 64)
          dst[i] = make_uint4(0x3f803f80u, 0x3f803f80u, 0x3f803f80u, 0x3f803f80u);
      }
      fence_async_shared();
    }
  }
  if (warp == 8 && lane == 0) {
    mbar_init(smem_u32(&bar_q), 1);
    for (int s = 0; s < ST; ++s) {
      mbar_init(smem_u32(&bar_k[s]), 1);
      mbar_init(smem_u32(&bar_v[s]), 1);
      mbar_init(smem_u32(&bar_kv_empty[s]), MC ? 2 : 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(smem_u32(&bar_s[t]), 1);
      mbar_init(smem_u32(&bar_p[t]), 128);
      mbar_init(smem_u32(&bar_o[t]), 1);
      mbar_init(smem_u32(&bar_sfree[t]), 128);
      mbar_init(smem_u32(&bar_pvdone[t]), 1);
      for (int k = 0; k < 3; ++k) mbar_init(smem_u32(&bar_pa[t][k]), 128);
    }
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if constexpr (MC) cluster_sync();  // the partner's barriers exist before any multicast load or commit reaches them
  const uint32_t tmem = tmem_slot;

  if (warp >= 8) {
   setmaxnreg_dec<kRegsOther>();
   if (warp == 8) {
    // ------------------------------------------------------------------ TMA producer
    if (elect_one()) {
      tma_prefetch_desc(&tm.q);
      tma_prefetch_desc(&tm.k);
      tma_prefetch_desc(&tm.v);
      const uint64_t pol_q = policy_evict_first(), pol_kv = policy_evict_last();
      const uint32_t bq = smem_u32(&bar_q);
      mbar_expect_tx(bq, C::kQBytes);
      const int qrow = (int)(a.q_row0 + (int64_t)pair * 256);
      T::load(sQ, &tm.q, bq, a.q.head0 + h, qrow, pol_q);
      T::load(sQ + T::kBytes, &tm.q, bq, a.q.head0 + h, qrow + 128, pol_q);
      for (int j = 0; j < n_tiles; ++j) {
        const int s = j % ST;
        if (j >= ST) mbar_wait(smem_u32(&bar_kv_empty[s]), ((j / ST) - 1) & 1);
        TRACE(7, j);
        const uint32_t sk = sKV + s * C::kStageBytes, sv = sk + T::kBytes;
        const int krow = (int)(a.kv_row0 + (int64_t)j * 128);
        mbar_expect_tx(smem_u32(&bar_k[s]), T::kBytes);
        mbar_expect_tx(smem_u32(&bar_v[s]), T::kBytes);
        if constexpr (MC) {
#pragma unroll
          for (int at = 0; at < T::kAtoms; ++at) {
            const uint32_t off = at * T::kAtomBytes + crank * 64 * T::kRowBytes;
            tma_load_3d_mc(sk + off, &tm.k64, smem_u32(&bar_k[s]), at * T::kAtomCols, a.k.head0 + g,
                           krow + 64 * (int)crank, 3, pol_kv);
            tma_load_3d_mc(sv + off, &tm.v64, smem_u32(&bar_v[s]), at * T::kAtomCols, a.v.head0 + g,
                           krow + 64 * (int)crank, 3, pol_kv);
          }
        } else {
          T::load(sk, &tm.k, smem_u32(&bar_k[s]), a.k.head0 + g, krow, pol_kv);
          T::load(sv, &tm.v, smem_u32(&bar_v[s]), a.v.head0 + g, krow, pol_kv);
        }
      }
    }
   } else if (warp == 9) {
    // ------------------------------------------------------------------ MMA issuer
    if (elect_one()) {
      const uint32_t idS = idesc_bf16(128, 128, 0, 0);
      const uint32_t idPV = idesc_bf16(128, C::NO, 0, 1);
      const uint32_t tS[2] = {tmem, tmem + 128};
      const uint32_t tO[2] = {tmem + C::tO0, tmem + C::tO0 + C::tOstride};
      const uint32_t tPa[2] = {C::kSepP ? tmem + C::tP : tS[0], C::kSepP ? tmem + C::tP : tS[1]};
      auto issue_S = [&](int t, int s) {
        const uint32_t sq = sQ + t * T::kBytes, sk = sKV + s * C::kStageBytes;
#pragma unroll
        for (int kk = 0; kk < T::kKSteps; ++kk)
          mma_ss(tS[t], T::desc_kmajor(sq, kk), T::desc_kmajor(sk, kk), idS, kk > 0);
      };
      auto issue_PV = [&](int t, int s, int j, int k0 = 0, int k1 = 8) {
        const uint32_t sv = sKV + s * C::kStageBytes + T::kBytes;
#pragma unroll
        for (int kk = k0; kk < k1; ++kk)
          mma_ts(tO[t], tPa[t] + kk * 8, T::desc_mn(sv, kk), idPV, (j > 0 || kk > 0) ? 1u : 0u);
      };
      // kPVChunks > 1: PV_t(j) in key chunks, each as soon as its P is in TMEM
      auto issue_PV_split = [&](int t, int s, int j) {
        if constexpr (kPVChunks > 1) {
          constexpr int KS = 8 / kPVChunks;  // 16-key MMA steps per chunk
#pragma unroll
          for (int k = 0; k < kPVChunks - 1; ++k) {
            mbar_wait(smem_u32(&bar_pa[t][k]), j & 1);
            tc_fence_after();
            issue_PV(t, s, j, k * KS, (k + 1) * KS);
          }
          mbar_wait(smem_u32(&bar_p[t]), j & 1);
          TRACE(4 + t, j);
          tc_fence_after();
          issue_PV(t, s, j, 8 - KS, 8);
        } else {
          mbar_wait(smem_u32(&bar_p[t]), j & 1);
          TRACE(4 + t, j);
          tc_fence_after();
          issue_PV(t, s, j);
        }
      };
      mbar_wait(smem_u32(&bar_q), 0);
      tc_fence_after();
      if constexpr (C::kSepP) {
        // per key tile j: S_t(j+1) as soon as the softmax warps have read S_t(j) out of TMEM; PV_t(j) when P_t(j)
        // is in the shared P buffer (the softmax warps of the other tile wait for PV_t(j) before overwriting it).
        // (Measured, not kept: the order S_0(j+1), PV_1(j-1), S_1(j+1), PV_0(j), which serves each warpgroup's events
        // in arrival order: same speed, 910-926 vs 911-927 TFLOP/s, tools/round1/gpu_ab_fwdorder.sh — the S tiles
        // were never late enough to matter; the exponential phases, 2.0 elem/clk per warp, set the pace.)
        mbar_wait(smem_u32(&bar_k[0]), 0);
        tc_fence_after();
        issue_S(0, 0);
        mma_commit(smem_u32(&bar_s[0]));
        issue_S(1, 0);
        mma_commit(smem_u32(&bar_s[1]));
        for (int j = 0; j < n_tiles; ++j) {
          const int s = j % ST, s2 = (j + 1) % ST;
          const uint32_t ph = (j / ST) & 1;
          const bool more = j + 1 < n_tiles;
          if (more) {
            mbar_wait(smem_u32(&bar_k[s2]), ((j + 1) / ST) & 1);
            mbar_wait(smem_u32(&bar_sfree[0]), j & 1);
            TRACE(6, j);
            tc_fence_after();
            issue_S(0, s2);
            mma_commit(smem_u32(&bar_s[0]));
            if (j < 1024) TRACE(6, 1024 + j);  // S_0(j+1) issued
            mbar_wait(smem_u32(&bar_sfree[1]), j & 1);
            tc_fence_after();
            issue_S(1, s2);
            mma_commit(smem_u32(&bar_s[1]));
            if (j < 1024) TRACE(6, 2048 + j);  // S_1(j+1) issued
          }
          mbar_wait(smem_u32(&bar_v[s]), ph);
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            mbar_wait(smem_u32(&bar_p[t]), j & 1);
            TRACE(4 + t, j);
            tc_fence_after();
            issue_PV(t, s, j);
            mma_commit(smem_u32(&bar_pvdone[t]));
            if (t == 1) {
              if constexpr (MC) mma_commit_mc(smem_u32(&bar_kv_empty[s]), 3);  // stage s consumed, in both CTAs
              else mma_commit(smem_u32(&bar_kv_empty[s]));
            }
            if (!more) mma_commit(smem_u32(&bar_o[t]));
            if (j < 1024) TRACE(4 + t, 1024 + j);  // PV_t(j) issued and committed
          }
        }
      } else
      for (int j = 0; j < n_tiles; ++j) {
        const int s = j % ST;
        const uint32_t ph = (j / ST) & 1;
        if (j == 0) {
          mbar_wait(smem_u32(&bar_k[s]), ph);
          tc_fence_after();
          issue_S(0, s);
          mma_commit(smem_u32(&bar_s[0]));
          issue_S(1, s);
          mma_commit(smem_u32(&bar_s[1]));
        }
        mbar_wait(smem_u32(&bar_v[s]), ph);
        issue_PV_split(0, s, j);
        const bool more = j + 1 < n_tiles;
        const int s2 = (j + 1) % ST;
        if (more) {
          mbar_wait(smem_u32(&bar_k[s2]), ((j + 1) / ST) & 1);
          TRACE(6, j);
          tc_fence_after();
          issue_S(0, s2);
          mma_commit(smem_u32(&bar_s[0]));
        } else {
          mma_commit(smem_u32(&bar_o[0]));
        }
        issue_PV_split(1, s, j);
        if constexpr (MC) mma_commit_mc(smem_u32(&bar_kv_empty[s]), 3);
        else mma_commit(smem_u32(&bar_kv_empty[s]));
        if (more) {
          issue_S(1, s2);
          mma_commit(smem_u32(&bar_s[1]));
        } else {
          mma_commit(smem_u32(&bar_o[1]));
        }
      }
    }
   }
  } else {
    setmaxnreg_inc<kRegsSoftmax>();
    // ------------------------------------------------------------------ softmax / correction / epilogue
    const int t = warp >> 2;
    const int r = (warp & 3) * 32 + lane;
    const uint32_t lane_off = ((warp & 3) * 32) << 16;
    uint32_t tS = tmem + t * 128 + lane_off;
    uint32_t tO = tmem + C::tO0 + t * C::tOstride + lane_off;
    uint32_t tPw = C::kSepP ? tmem + C::tP + lane_off : tS;
    asm volatile("" : "+r"(tS), "+r"(tO), "+r"(tPw));
    const int64_t qpos = q_pos_first + t * 128 + r;
    const float sl2 = a.scale_log2;
    float m_run = -INFINITY, l_run = 0.f;
    for (int j = 0; j < n_tiles; ++j) {
      mbar_wait(smem_u32(&bar_s[t]), j & 1);
      if ((warp & 3) == 0 && lane == 0) TRACE(0 + 2 * t, j);
      tc_fence_after();
      float x[128];
      tmem_ld32(tS + 0, reinterpret_cast<uint32_t*>(x));
      tmem_ld32(tS + 32, reinterpret_cast<uint32_t*>(x) + 32);
      tmem_ld32(tS + 64, reinterpret_cast<uint32_t*>(x) + 64);
      tmem_ld32(tS + 96, reinterpret_cast<uint32_t*>(x) + 96);
      tmem_wait_ld();
      if constexpr (C::kSepP) {
        tc_fence_before();
        mbar_arrive(smem_u32(&bar_sfree[t]));  // S_t(j) is in registers: the MMA warp may compute S_t(j+1)
      }
      if ((warp & 3) == 0 && lane == 0) TRACE(8 + 4 * t, j);
      // causal mask: only on the tile(s) that straddle the diagonal (warp-uniform fast path otherwise)
      const int64_t lim64 = qpos - (a.kv_pos0 + (int64_t)j * 128);
      const bool masked = a.causal && lim64 < 127;
      const bool any_masked = __any_sync(0xffffffffu, masked);
      if (masked) {
        const int lim = (int)(lim64 < -1 ? -1 : lim64);
#pragma unroll
        for (int i = 0; i < 128; ++i)
          if (i > lim) x[i] = -INFINITY;
      }
      // row max: 8 independent three-input max chains over columns 8..119, then the last 8 columns
      float m8[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) m8[k] = x[k];
#pragma unroll
      for (int i = 8; i + 16 <= 128; i += 16) {
#pragma unroll
        for (int k = 0; k < 8; ++k) m8[k] = max3(m8[k], x[i + k], x[i + 8 + k]);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) m8[k] = fmaxf(m8[k], x[120 + k]);
      float mx = max3(max3(m8[0], m8[1], m8[2]), max3(m8[3], m8[4], m8[5]), fmaxf(m8[6], m8[7]));
      mx *= sl2;
      if ((warp & 3) == 0 && lane == 0) TRACE(9 + 4 * t, j);
      const bool need = mx > m_run + kRescaleThreshold;
      if (__any_sync(0xffffffffu, need)) {
        const float m_new = need ? mx : m_run;
        const float alpha = need ? ex2(m_run - m_new) : 1.f;
        if constexpr (!C::kSumMMA) l_run *= alpha;
        if (j > 0) {
          if constexpr (C::kSepP) {
            mbar_wait(smem_u32(&bar_pvdone[t]), (j - 1) & 1);  // PV_t(j-1) has accumulated into O_t
            tc_fence_after();
          }
#pragma unroll
          for (int c = 0; c < C::NO; c += 16) {
            uint32_t o[16];
            tmem_ld16(tO + c, o);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st16(tO + c, o);
          }
        }
        m_run = m_new;
      }
      const float mb = (m_run == -INFINITY) ? 0.f : m_run;
      // P = exp2(S*scale*log2e - m): every FPDT_FWD_POLY_EVERY-th pair on the FMA pipe, the rest on MUFU, except on
      // masked tiles (MUFU maps -inf to exactly 0)
      constexpr bool kSumHere = !C::kSumMMA;
      float sum;
      if constexpr (C::kSepP) {
        // P in registers first; then the shared P buffer: P_0(j) after PV_1(j-1) has read it, P_1(j) after PV_0(j)
        uint32_t pk[64];
        if (any_masked)
          sum = exp_pack_store<0, kSumHere, false>(x, sl2, mb, 0, pk);
        else if (FPDT_FWD_POLY_MMA_SMSP > 0 && (warp & 3) == 1)
          sum = exp_pack_store<(FPDT_FWD_POLY_MMA_SMSP > 0 ? FPDT_FWD_POLY_MMA_SMSP : 1), kSumHere, false>(x, sl2, mb, 0,
                                                                                                     pk);
        else
          sum = exp_pack_store<C::kPolyEvery, kSumHere, false>(x, sl2, mb, 0, pk);
        if (t == 0 && j > 0) mbar_wait(smem_u32(&bar_pvdone[1]), (j - 1) & 1);
        if (t == 1) mbar_wait(smem_u32(&bar_pvdone[0]), j & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < 64; c += 16) tmem_st16(tPw + c, pk + c);
      } else {
        if constexpr (kPVChunks > 1) {
          // P in key chunks: each lets the MMA warp run PV_t(j) over that part of the contraction while the
          // exponentials of the next chunk run
          constexpr int W = 128 / kPVChunks;
          sum = 0.f;
#pragma unroll
          for (int k = 0; k < kPVChunks - 1; ++k) {
            sum += any_masked ? exp_pack_store<0, kSumHere, true>(x, sl2, mb, tPw, nullptr, k * W, (k + 1) * W)
                              : exp_pack_store<C::kPolyEvery, kSumHere, true>(x, sl2, mb, tPw, nullptr, k * W,
                                                                              (k + 1) * W);
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(smem_u32(&bar_pa[t][k]));
          }
          sum += any_masked ? exp_pack_store<0, kSumHere, true>(x, sl2, mb, tPw, nullptr, 128 - W, 128)
                            : exp_pack_store<C::kPolyEvery, kSumHere, true>(x, sl2, mb, tPw, nullptr, 128 - W, 128);
        } else {
          sum = any_masked ? exp_pack_store<0, kSumHere>(x, sl2, mb, tPw)
                           : exp_pack_store<C::kPolyEvery, kSumHere>(x, sl2, mb, tPw);
        }
      }
      if constexpr (kSumHere) l_run += sum;
      if (lane == 0 && j < 1024) TRACE(10 + 4 * t, 1024 * (warp & 3) + j);
      tmem_wait_st();
      if ((warp & 3) == 0 && lane == 0) TRACE(11 + 4 * t, j);
      tc_fence_before();
      mbar_arrive(smem_u32(&bar_p[t]));
      if (lane == 0 && j < 1024) TRACE(1 + 2 * t, 1024 * (warp & 3) + j);
    }
    // epilogue: normalise, merge with the running partial result, write
    mbar_wait(smem_u32(&bar_o[t]), 0);
    tc_fence_after();
    float o[C::NO];
#pragma unroll
    for (int c = 0; c < C::NO; c += 16) tmem_ld16(tO + c, reinterpret_cast<uint32_t(&)[16]>(o[c]));
    tmem_wait_ld();
    if constexpr (C::kSumMMA) l_run = o[D];
    const float inv_l = 1.f / l_run;
    float lse_b = m_run + lg2(l_run);
    const int64_t row = (int64_t)pair * 256 + t * 128 + r;  // row within the launch's query range
    float wb = inv_l;
    float wa = 0.f;
    float* acc_row = a.o_acc ? a.o_acc + (row * a.hq + h) * D : nullptr;
    if (a.has_prev) {
      const float lse_a = a.lse_acc[(int64_t)h * a.n_q_rows + row];
      const float mxl = fmaxf(lse_a, lse_b);
      const float ea = ex2(lse_a - mxl), eb = ex2(lse_b - mxl);
      const float lse = mxl + lg2(ea + eb);
      wa = ex2(lse_a - lse);
      wb = inv_l * ex2(lse_b - lse);
      lse_b = lse;
    }
#pragma unroll
    for (int c = 0; c < D; c += 4) {
      float4 v = make_float4(o[c] * wb, o[c + 1] * wb, o[c + 2] * wb, o[c + 3] * wb);
      if (a.has_prev) {
        const float4 pa = *reinterpret_cast<const float4*>(acc_row + c);
        v.x += wa * pa.x; v.y += wa * pa.y; v.z += wa * pa.z; v.w += wa * pa.w;
      }
      o[c] = v.x; o[c + 1] = v.y; o[c + 2] = v.z; o[c + 3] = v.w;
    }
    if (a.is_final) {
      __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(a.o_out) + row * a.o_ld + (int64_t)(a.o_head0 + h) * D;
#pragma unroll
      for (int c = 0; c < D; c += 8) {
        uint4 w;
        w.x = pack_bf16x2(o[c], o[c + 1]);
        w.y = pack_bf16x2(o[c + 2], o[c + 3]);
        w.z = pack_bf16x2(o[c + 4], o[c + 5]);
        w.w = pack_bf16x2(o[c + 6], o[c + 7]);
        *reinterpret_cast<uint4*>(out + c) = w;
        if (a.o_resid) {
          // residual O - bf16(O), so the backward can form D from the fp32 output (R22)
          const __nv_bfloat162* wb2 = reinterpret_cast<const __nv_bfloat162*>(&w);
          uint4 rw;
          uint32_t* rp = reinterpret_cast<uint32_t*>(&rw);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float2 f = __bfloat1622float2(wb2[i]);
            rp[i] = pack_bf16x2(o[c + 2 * i] - f.x, o[c + 2 * i + 1] - f.y);
          }
          *reinterpret_cast<uint4*>(a.o_resid + row * a.o_resid_ld + (int64_t)h * D + c) = rw;
        }
      }
      a.lse_save[(int64_t)h * a.lse_save_ld + row] = lse_b;
      if (a.lse_user) a.lse_user[row * a.lse_user_ld + a.lse_user_head0 + h] = lse_b * 0.69314718055994531f;
    } else {
#pragma unroll
      for (int c = 0; c < D; c += 4)
        *reinterpret_cast<float4*>(acc_row + c) = make_float4(o[c], o[c + 1], o[c + 2], o[c + 3]);
      a.lse_acc[(int64_t)h * a.n_q_rows + row] = lse_b;
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (MC) cluster_sync();  // no CTA leaves while its partner may still multicast into it or arrive on it
  if (warp == 9) tmem_dealloc<512>(tmem);
}

template <int D>
int launch_fwd(const FwdArgs& a, cudaStream_t s) {
  using C = FwdCfg<D>;
  TmapSet tm;
  bool ok = make_tile_tmap<D>(&tm.q, a.q.base, a.q.rows, a.q.heads);
  ok &= make_tile_tmap<D>(&tm.k, a.k.base, a.k.rows, a.k.heads);
  ok &= make_tile_tmap<D>(&tm.v, a.v.base, a.v.rows, a.v.heads);
  constexpr CUtensorMapSwizzle kSw = D == 80 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_128B;
  ok &= make_tmap_rows_heads_dim(&tm.k64, a.k.base, a.k.rows, a.k.heads, D, Tile<D>::kAtomCols, 64, kSw);
  ok &= make_tmap_rows_heads_dim(&tm.v64, a.v.base, a.v.rows, a.v.heads, D, Tile<D>::kAtomCols, 64, kSw);
  if (!ok) return -1;
  dim3 grid(a.n_q_rows / 256, a.hq);
  // d = 128 only: there the K/V tiles are 32 KB each (C = 64K, 32 heads: 1228-1240 vs 1213-1228 TFLOP/s, diagonal / full
  // pair); at d = 80 the pairs lost 1-2% (957 / 964 vs 977 / 972 standalone, 924 vs 930 in the bench step)
  if (FPDT_FWD_MC && D == 128 && grid.x % 2 == 0) {
    if (int e = set_max_dynamic_smem((const void*)attn_fwd_kernel<D, true>, C::kSmem)) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = C::kSmem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaError_t e = cudaLaunchKernelEx(&cfg, attn_fwd_kernel<D, true>, tm, a)) return (int)e;
    return (int)cudaGetLastError();
  }
  if (int e = set_max_dynamic_smem((const void*)attn_fwd_kernel<D, false>, C::kSmem)) return e;
  attn_fwd_kernel<D, false><<<grid, kThreads, C::kSmem, s>>>(tm, a);
  return (int)cudaGetLastError();
}

}  // namespace

int launch_attn_fwd_bf16(const FwdArgs& a, int head_dim, cudaStream_t s) {
  switch (head_dim) {
    case 64: return launch_fwd<64>(a, s);
    case 80: return launch_fwd<80>(a, s);
    case 128: return launch_fwd<128>(a, s);
  }
  return -2;
}

}  // namespace fpdt
