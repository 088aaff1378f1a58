// Backward chunk-pair attention for sm_100a, head_dim 64 / 80: software-pipelined across query tiles; the dQ product in
// fp16 (see PipeCfg).
//
// Same operation as attn_bwd_sm100.cu (one (key/value chunk j, query chunk i) step of FPDT's nested backward
// loop, fig:bw_db; KV-stationary CTA = one 128-row key/value tile of one KV head walking the
// query tiles of the range and the G query heads of its group):
//   S^T  = K Q^T            P^T  = exp2(S^T*scale*log2e - lse2)       (recompute)
//   dP^T = V dO^T           dS^T = P^T o (dP^T - D)
//   dV  += P^T dO           dK  += dS^T Q          dQ_partial = dS K  (TMA bulk reduce-add into fp32 dq_acc)
//
// What differs from the non-pipelined kernel: P^T_n and dS^T_n (bf16) are written into the dP^T TMEM columns
// once the softmax warps hold dP^T_n in registers, so the S^T columns hold nothing but S^T and S^T_{n+1} is
// issued as soon as S^T_n has been read out — it runs during the exponentials of tile n, and the softmax warps go
// straight from dS_n to the exponentials of tile n+1.  dV and dK are TS-MMAs (A from TMEM): shared memory, not
// the tensor pipe, is the scarce resource here (128 B/clk/SM; an SS-MMA with M = 128, N <= 128 already needs all
// of it), so per query tile only dQ = dS K (A = the dS smem tile) reads two smem operands.  Shared-memory bytes per
// tile (d = 80): TMA Q, dO 40K + MMA operands 172K + dS 32K + dQ staging 80K.
// (Round 2: per-warp traces show the softmax warps on SMSPs 0 and 1 -- with the TMA and MMA issuing warps, whose
// instructions share the MIO queue with MUFU -- ~200-400 clk behind those on SMSPs 2 and 3 per tile; moving one
// exponential pair in 2 / 4 / 8 of those warps to the FMA pipe evened them but left the step at 843-847 vs 848 TFLOP/s:
// the tile period here is set by the dQ reduce-add chain, not by the slowest softmax warp.  Moving the TMA / MMA warps
// to SMSPs 2 / 3 (warps 14 / 15) changed nothing either: 844.5-845.1 vs 844.8-845.3 in the step.)
// Element-wise math uses packed f32x2 FMA-pipe instructions (FFMA2/FADD2/FMUL2); the exponentials all run on MUFU
// (an FA4-style polynomial offload of a fraction of them measured slower here: one pair in 4 / 8 / 16 on the FMA pipe
// gave 848-858 / 868 / 871 TFLOP/s against 872-875 all on MUFU, C = 64K, 32 x 80 diagonal pair).
//
// Launched in clusters of two CTAs (adjacent key tiles of one head, same query-tile walk) that multicast the halves of
// every Q and dO tile to each other (template flag MC, see the kernel): 877 vs 862 TFLOP/s on the d = 80 diagonal pair,
// 859 vs 846 on a full pair (tools/gpu_ab.sh, same box).  Measured along the way (timing-only builds, results wrong):
// no dQ reduce-add 1000 / 1011, no Q / dO loads 944 / 959, neither 1038 / 1075 TFLOP/s; Q / dO through the
// load/store unit (cp.async by two warps) instead of TMA 574-695 (slower); each CTA of the pair reduce-adding only its
// 64 query rows of the pair's summed dQ partials, the other 64 rows sent to the partner with st.shared::cluster (DSMEM)
// 556-562 (the remote stores move ~4 B/clk/SM; parity-green, not kept).
// Warps (512 threads = 4 warpgroups, registers rebalanced with setmaxnreg):
//   WG0 (0-3)   softmax-gradient, query columns [0,64)   (thread = key row = TMEM lane); final dK    168 regs
//   WG1 (4-7)   softmax-gradient, query columns [64,128)                                ; final dV    168 regs
//   WG2 (8-11)  dQ read-out (thread = query row) -> smem staging -> TMA bulk reduce-add              104 regs
//   WG3 (12)    TMA producer; (13) TMEM allocator + single-thread MMA issuer; (14, 15) the dO' atoms of the D
//               fold (d = 80, PipeCfg::kFoldD: dP^T = V dO^T - D as a sixth k-step)                   72 regs
// Shared memory (d = 80: 226 KB): K, V | 2 Q stages (+ lse2 rows) | 2 dO stages | fp16 K | dS (fp16) | dQ staging |
// V' atom | 2 dO' atoms.
// TMEM: S^T [0,128) | dP^T [128,256), then per query half h: P^T [128+64h, +32), dS^T [160+64h, +32) (bf16) |
//       dQ [256,256+D) | dK | dV  (496 columns at d = 80).
#include "attn_tile.cuh"
#include "kernels.h"
#include "smem_layout.cuh"
#include "tma_host.h"

namespace fpdt {
namespace {

using namespace ptx;

constexpr int kThreads = 512;
// setmaxnreg budget: the softmax warpgroups grow only by what WG2 / WG3 give back (pool = launch allocation)
constexpr int kLaunchRegs = (65536 / kThreads) & ~7;  // 128
// measured (tools/gpu_regs_sweep.sh, d = 80 C = 64K pair): 168/104/72 -> 872-876, 176/96/64 -> 863-865,
// 160/120/72 -> 837-841 TFLOP/s
#ifndef FPDT_BWD_REGS_SOFTMAX
#define FPDT_BWD_REGS_SOFTMAX 168
#define FPDT_BWD_REGS_DQ 104
#define FPDT_BWD_REGS_CTL 72
#endif
// dQ staging groups: 32 rows (each dQ warp stages its rows and issues their reduce-add: a warp waits only for its own
// previous reduce-add to have read its staging) or 64 (two halves, a named barrier each).  In the bench step (same box,
// A/B/A/B): 32 -> bwd 838 at 1560 MHz, 64 -> 829 at 1590 MHz; 16 (half warps) -> 818-819 vs 830-831 for 32.
#ifndef FPDT_BWD_DQ_ROWS
#define FPDT_BWD_DQ_ROWS 32
#endif
constexpr int kDQRows = FPDT_BWD_DQ_ROWS;
static_assert(kDQRows == 32 || kDQRows == 64, "dQ staging group");
// multicast cluster: kCS CTAs on adjacent key tiles, each loading kCR = 128 / kCS rows of every Q / dO tile (4: bwd
// 811 vs 849 TFLOP/s in the step, A/B/A/B -- four CTAs in lockstep wait on each other more than the loads cost)
#ifndef FPDT_BWD_CLUSTER
#define FPDT_BWD_CLUSTER 2
#endif
constexpr int kCS = FPDT_BWD_CLUSTER, kCR = 128 / kCS;
constexpr uint16_t kCMask = (uint16_t)((1u << kCS) - 1);
static_assert(kCS == 2 || kCS == 4, "multicast cluster size");
#ifndef FPDT_BWD_FOLD_D
#define FPDT_BWD_FOLD_D 1
#endif
constexpr int kRegsSoftmax = FPDT_BWD_REGS_SOFTMAX, kRegsDQ = FPDT_BWD_REGS_DQ, kRegsCtl = FPDT_BWD_REGS_CTL;
static_assert(2 * 128 * (kRegsSoftmax - kLaunchRegs) <= 128 * (2 * kLaunchRegs - kRegsDQ - kRegsCtl), "register pool");
// The dQ product runs in fp16 (dS and a copy of K rounded to fp16, fp32 accumulation): its sum cancels
// (sum_j dS_ij = 0), so a common offset of the keys multiplies the rounding error of dS -- a key drift of 32 in one
// dimension (fpdt_inputs "drift") costs ~1.2e-2 normwise in dQ with bf16 dS, ~1.5e-3 with fp16 (measured: bf16
// 0.012-0.026 on the GPU drift cases).  The fp16 copy of K takes the shared memory of a third Q stage (2 stages:
// 858 vs 871 TFLOP/s for the bf16 product with 3 stages, C = 64K, 32 x 80 diagonal pair).  The third stage is not
// what the 1.5% went to (tools/gpu_ab_qs.sh, same box): d = 64, where it fits, gains 0.5% from it (817 -> 821), and
// at d = 80 buying it back with a 3-slot 16-column dQ staging ring per half (a wait for the reduce-add to read the
// ring in the middle of every tile) loses 13% (856 -> 746): the bulk reduce-add's read of the staging is slow enough
// that the staging must hold a whole tile.
template <int D>
struct PipeCfg {
  using T = Tile<D>;
  static constexpr int QS = 2, OS = 2;
  static constexpr int TB = T::kBytes;
  static constexpr int kDS = 128 * 128 * 2;  // dS (fp16)
  static constexpr int kDQ = 128 * D * 4;
  static constexpr int kStats = 1024;  // lse2[128] + D[128] fp32
  static constexpr int oK = 0, oV = TB, oQ = 2 * TB, oO = oQ + QS * TB;
  static constexpr int oKH = ((oO + OS * TB + 1023) / 1024) * 1024;  // fp16 copy of K (B of dQ)
  static constexpr int oDS = oKH + ((TB + 1023) / 1024) * 1024;
  static constexpr int oDQ = oDS + kDS;
  static constexpr int oStats = oDQ + kDQ;
  // kFoldD: D enters dP^T = V dO^T - D as one more 16-column k-step -- a constant atom of V' (columns -1, -1, 0, ...)
  // and, per dO stage, an atom of dO' (bf16 hi / lo of D in columns 0 / 1) -- instead of the softmax warps' broadcast
  // shared-memory reads of D and their subtraction
  static constexpr bool kFoldD = FPDT_BWD_FOLD_D != 0 && D == 80;  // the extra atoms use the d = 80 (SW32) format
  static constexpr int kXAtom = 128 * 16 * 2;  // one 16-column SW32 atom of 128 rows
  static constexpr int oVX = ((oStats + QS * kStats + 1023) / 1024) * 1024;
  static constexpr int oOX = oVX + (kFoldD ? kXAtom : 0);
  static constexpr int oBars = oOX + (kFoldD ? OS * kXAtom : 0);
  static constexpr int kSmem = oBars + 256;
  static_assert(kSmem <= 227 * 1024, "shared memory budget");
  static constexpr uint32_t tS = 0, tdP = 128, tdQ = 256, tdK = 256 + D, tdV = 256 + 2 * D;
  static_assert(256 + 3 * D <= 512, "TMEM budget");
};

struct TmapSet {
  CUtensorMap q, k, v, o;
  CUtensorMap q64, o64;  // 64-row boxes: each CTA of a cluster pair multicasts one half of a Q / dO tile
  CUtensorMap dq32h, dq16h;  // fp32 dq_acc, 64-row boxes: 32 columns (128B swizzle) / 16 columns (64B swizzle)
};

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
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
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
[[maybe_unused]] __device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ float4 lds4(const float* p) { return *reinterpret_cast<const float4*>(p); }

__device__ __forceinline__ uint32_t pack_f16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// MC: launched in clusters of two CTAs on adjacent key tiles of one head, which walk the same query tiles; each CTA
// loads one 64-row half of every Q and dO tile and multicasts it into both, so each SM's TMA engine issues half of the
// loads (it also carries the dQ reduce-adds, and the loads queued behind them were late: skipping the Q or the dO
// loads in a timing-only build ran the pair at 946 / 901 instead of 850 TFLOP/s).  A stage is refilled once both CTAs
// have consumed it (the MMA commit arrives on the empty barrier of both).
template <int D, bool MC>
__global__ void __launch_bounds__(kThreads, 1)
attn_bwd_pipe_kernel(const __grid_constant__ TmapSet tm, const __grid_constant__ BwdArgs a) {
  using T = Tile<D>;
  using C = PipeCfg<D>;
  constexpr int QS = C::QS, OS = C::OS;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = smem_u32(smem);
  const uint32_t sK = base + C::oK, sV = base + C::oV, sDS = base + C::oDS, sDQ = base + C::oDQ;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::oBars);
  auto bar = [&](int i) { return smem_u32(&bars[i]); };
  // barrier indices
  constexpr int B_KV = 0, B_QF = 1, B_QE = B_QF + QS, B_OF = B_QE + QS, B_OE = B_OF + OS, B_S = B_OE + OS,
                B_SFREE = B_S + 1, B_DP = B_SFREE + 1, B_P = B_DP + 1, B_DS = B_P + 1,
                B_DSFREE = B_DS + 1, B_DQF = B_DSFREE + 1, B_DQE = B_DQF + 1, B_KVDONE = B_DQE + 1,
                B_KH = B_KVDONE + 1, B_NUM = B_KH + 1;
  static_assert(B_NUM <= 30, "barrier area");
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::oBars + 30 * 8);

  const uint32_t warp = warp_id(), lane = lane_id();
  const int kt = blockIdx.x;
  const int g = blockIdx.y;
  const int G = a.G;
  const int64_t kv_base = a.kv_pos0 + (int64_t)kt * 128;
  const uint32_t crank = MC ? cluster_ctarank() : 0;
  int qt_first = 0;
  const int n_qt_total = a.n_q_rows / 128;
  if (a.causal) {
    // first query tile that can see this key tile (MC: the pair's first key tile; the second CTA's first tile of a
    // diagonal pair is then fully masked, P = 0)
    const int64_t rel = a.kv_pos0 + (int64_t)(MC ? (kt & ~(kCS - 1)) : kt) * 128 - a.q_pos0;
    if (rel > 0) qt_first = (int)(rel / 128);
    if (qt_first > n_qt_total) qt_first = n_qt_total;
  }
  const int n_iter = (n_qt_total - qt_first) * G;
  const bool tracing = a.trace != nullptr && blockIdx.x == a.trace_cta && blockIdx.y == 0;
#define TRACE(ev, n)                                                        \
  do {                                                                      \
    if (tracing && (n) < 4096) a.trace[(ev) * 4096 + (n)] = clock64();      \
  } while (0)

  if (warp == 13) tmem_alloc<512>(smem_u32(tmem_slot));
  if (warp == 12 && lane == 0) {
    mbar_init(bar(B_KV), 1);
    for (int s = 0; s < QS; ++s) {
      mbar_init(bar(B_QF + s), 1);
      mbar_init(bar(B_QE + s), MC ? kCS : 1);
    }
    for (int s = 0; s < OS; ++s) {
      mbar_init(bar(B_OF + s), C::kFoldD ? 1 + 64 : 1);  // + the 64 threads writing the stage's dO' atom
      mbar_init(bar(B_OE + s), MC ? kCS : 1);
    }
    mbar_init(bar(B_S), 1);
    mbar_init(bar(B_SFREE), 256);
    mbar_init(bar(B_DP), 1);
    mbar_init(bar(B_P), 256);
    mbar_init(bar(B_DS), 256);
    mbar_init(bar(B_DSFREE), 1);
    mbar_init(bar(B_DQF), 1);
    mbar_init(bar(B_DQE), 128);
    mbar_init(bar(B_KVDONE), 1);
    mbar_init(bar(B_KH), 4);
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if constexpr (MC) cluster_sync();  // the partner's barriers exist before any multicast load or commit reaches them
  const uint32_t tmem = *tmem_slot;

  if (warp >= 12) {
    setmaxnreg_dec<kRegsCtl>();
    if (warp == 12) {
      // ---------------------------------------------------------------- TMA producer
      if (elect_one() && n_iter > 0) {
        const uint64_t pol_kv = policy_evict_first(), pol_q = policy_evict_last();
        mbar_expect_tx(bar(B_KV), 2 * C::TB);
        const int krow = (int)(a.kv_row0 + (int64_t)kt * 128);
        T::load(sK, &tm.k, bar(B_KV), a.k.head0 + g, krow, pol_kv);
        T::load(sV, &tm.v, bar(B_KV), a.v.head0 + g, krow, pol_kv);
        for (int n = 0; n < n_iter; ++n) {
          const int qs = n % QS, os = n % OS;
          const int qt = qt_first + n / G, h = g * G + n % G;
          const int qrow = (int)(a.q_row0 + (int64_t)qt * 128);
          if (n >= QS) mbar_wait(bar(B_QE + qs), ((n / QS) - 1) & 1);
          TRACE(12, n);
          const uint32_t fq = bar(B_QF + qs);
          const uint32_t stats = base + C::oStats + qs * C::kStats;
          mbar_expect_tx(fq, C::TB + (C::kFoldD ? 512 : 1024));
          if constexpr (MC) {
#pragma unroll
            for (int at = 0; at < T::kAtoms; ++at)
              tma_load_3d_mc(base + C::oQ + qs * C::TB + at * T::kAtomBytes + crank * kCR * T::kRowBytes, &tm.q64,
                             fq, at * T::kAtomCols, a.q.head0 + h, qrow + kCR * (int)crank, kCMask, pol_q);
          } else {
            T::load(base + C::oQ + qs * C::TB, &tm.q, fq, a.q.head0 + h, qrow, pol_q);
          }
          bulk_load(stats, a.lse2 + (int64_t)h * a.stat_ld + (int64_t)qt * 128, 512, fq);
          if constexpr (!C::kFoldD) bulk_load(stats + 512, a.Dstat + (int64_t)h * a.stat_ld + (int64_t)qt * 128, 512, fq);
          if (n >= OS) mbar_wait(bar(B_OE + os), ((n / OS) - 1) & 1);
          mbar_expect_tx(bar(B_OF + os), C::TB);
          if constexpr (MC) {
#pragma unroll
            for (int at = 0; at < T::kAtoms; ++at)
              tma_load_3d_mc(base + C::oO + os * C::TB + at * T::kAtomBytes + crank * kCR * T::kRowBytes, &tm.o64,
                             bar(B_OF + os), at * T::kAtomCols, a.dout.head0 + h, qrow + kCR * (int)crank, kCMask,
                             pol_q);
          } else {
            T::load(base + C::oO + os * C::TB, &tm.o, bar(B_OF + os), a.dout.head0 + h, qrow, pol_q);
          }
        }
      }
    } else if (warp == 13) {
      // ---------------------------------------------------------------- MMA issuer
      if (elect_one() && n_iter > 0) {
        const uint32_t idS = idesc_bf16(128, 128, 0, 0);  // S^T, dP^T: A (K or V rows), B (Q or dO rows) K-major
        const uint32_t idG = idesc_bf16(128, D, 0, 1);    // dV, dK: A = P^T / dS^T K-major smem, B MN-major
        // dQ: A = dS MN-major smem, B = K MN-major, both fp16 (kind::f16 with fp16 inputs)
        const uint32_t idQ = (1u << 4) | (1u << 15) | (1u << 16) | ((uint32_t)(D >> 3) << 17) | ((128u >> 4) << 24);
        const uint32_t sKQ = base + C::oKH;  // the fp16 copy of K
        const uint32_t tS = tmem + C::tS, tdP = tmem + C::tdP, tdQ = tmem + C::tdQ, tdK = tmem + C::tdK,
                       tdV = tmem + C::tdV;
        auto sQ = [&](int n) { return base + C::oQ + (n % QS) * C::TB; };
        auto sO = [&](int n) { return base + C::oO + (n % OS) * C::TB; };
        auto issue_S = [&](int n) {
          mbar_wait(bar(B_QF + n % QS), (n / QS) & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < T::kKSteps; ++kk)
            mma_ss(tS, T::desc_kmajor(sK, kk), T::desc_kmajor(sQ(n), kk), idS, kk > 0);
          mma_commit(bar(B_S));
        };
        auto issue_dP = [&](int n) {
          mbar_wait(bar(B_OF + n % OS), (n / OS) & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < T::kKSteps; ++kk)
            mma_ss(tdP, T::desc_kmajor(sV, kk), T::desc_kmajor(sO(n), kk), idS, kk > 0);
          if constexpr (C::kFoldD)
            mma_ss(tdP, T::desc_kmajor(base + C::oVX, 0), T::desc_kmajor(base + C::oOX + (n % OS) * C::kXAtom, 0), idS,
                   1u);
          mma_commit(bar(B_DP));
        };
        mbar_wait(bar(B_KV), 0);
        issue_S(0);
        issue_dP(0);
        // Issue order per query tile n (blocking waits: a spinning probe loop would steal the shared-memory pipe
        // the tensor core reads its operands through):
        //   S^T_{n+1}  after SFREE(n) (S^T_n read out) and Q_{n+1} loaded
        //   dV_n       after P^T_n in TMEM
        //   group n    dK_n, dP^T_{n+1}, dQ_n after dS^T_n in TMEM and dS_n in smem; dP^T_{n+1} overwrites P^T_n /
        //              dS^T_n after dV_n and dK_n in issue order; dQ_n after dQ_{n-1} has been read out
        for (int n = 0; n < n_iter; ++n) {
          const bool more = n + 1 < n_iter;
          if (more) {
            mbar_wait(bar(B_SFREE), n & 1);
            TRACE(6, n);
            issue_S(n + 1);
          }
          // dV += P^T dO_n   (A = P^T in TMEM)
          mbar_wait(bar(B_P), n & 1);
          TRACE(4, n);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            mma_ts(tdV, tdP + 64 * (kk >> 2) + (kk & 3) * 8, T::desc_mn(sO(n), kk), idG, (n > 0 || kk > 0));
          if constexpr (MC) mma_commit_mc(bar(B_OE + n % OS), kCMask);  // dO_n consumed (dP_n precedes dV_n), both CTAs
          else mma_commit(bar(B_OE + n % OS));
          // dK += dS^T Q_n   (A = dS^T in TMEM); first, so that Q_n is released early
          mbar_wait(bar(B_DS), n & 1);
          TRACE(5, n);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            mma_ts(tdK, tdP + 64 * (kk >> 2) + 32 + (kk & 3) * 8, T::desc_mn(sQ(n), kk), idG, (n > 0 || kk > 0));
          if constexpr (MC) mma_commit_mc(bar(B_QE + n % QS), kCMask);  // Q_n consumed
          else mma_commit(bar(B_QE + n % QS));
          if (more) issue_dP(n + 1);
          // dQ_n = dS K   (A = the dS smem tile, MN-major)
          if (n > 0) {
            mbar_wait(bar(B_DQE), (n - 1) & 1);
            tc_fence_after();
          } else {
            mbar_wait(bar(B_KH), 0);  // the fp16 copy of K is built
            tc_fence_after();
          }
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) mma_ss(tdQ, desc_a_mn_sw128(sDS, kk), T::desc_mn(sKQ, kk), idQ, kk > 0);
          mma_commit(bar(B_DQF));
          mma_commit(bar(B_DSFREE));
          TRACE(8, n);
        }
        mma_commit(bar(B_KVDONE));
      }
    } else if (C::kFoldD && warp >= 14) {
      // ---------------------------------------------------------------- the extra dP^T k-step's atoms (kFoldD)
      // thread t writes rows t and t + 64: the constant V' atom and the zero halves once, then per query tile the
      // bf16 hi / lo split of D into the dO stage's dO' atom (SW32: 16-byte piece c of row r at c ^ ((r >> 2) & 1))
      const int t = (int)threadIdx.x - 448;
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int r = t + 64 * k;
        const uint32_t sw = (uint32_t)(r >> 2) & 1u;
        uint8_t* vx = smem + C::oVX + r * 32;
        *reinterpret_cast<uint4*>(vx + ((0u ^ sw) << 4)) = make_uint4(0xbf80bf80u, 0u, 0u, 0u);  // -1, -1 (bf16)
        *reinterpret_cast<uint4*>(vx + ((1u ^ sw) << 4)) = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
        for (int s2 = 0; s2 < OS; ++s2)
          *reinterpret_cast<uint4*>(smem + C::oOX + s2 * C::kXAtom + r * 32 + ((1u ^ sw) << 4)) =
              make_uint4(0u, 0u, 0u, 0u);
      }
      for (int n = 0; n < n_iter; ++n) {
        const int os = n % OS;
        const int qt = qt_first + n / G, h = g * G + n % G;
        if (n >= OS) mbar_wait(bar(B_OE + os), ((n / OS) - 1) & 1);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int r = t + 64 * k;
          const float dv = a.Dstat[(int64_t)h * a.stat_ld + (int64_t)qt * 128 + r];
          const __nv_bfloat16 hi = __float2bfloat16_rn(dv);
          const float lo = dv - __bfloat162float(hi);
          *reinterpret_cast<uint4*>(smem + C::oOX + os * C::kXAtom + r * 32 + ((0u ^ ((uint32_t)(r >> 2) & 1u)) << 4)) =
              make_uint4(pack_bf16x2(__bfloat162float(hi), lo), 0u, 0u, 0u);
        }
        fence_async_shared();  // generic-proxy writes -> the tensor core's operand reads
        mbar_arrive(bar(B_OF + os));
      }
    }
  } else if (warp < 8) {
    setmaxnreg_inc<kRegsSoftmax>();
    // ------------------------------------------------------------------ softmax gradient (key rows)
    const int half = warp >> 2;  // query columns [64*half, 64*half+64)
    const int r = (warp & 3) * 32 + lane;
    // TMEM addresses of this warp's lanes; the empty asm keeps them in registers (no per-iteration S2R)
    uint32_t tS = tmem + C::tS + (((warp & 3) * 32) << 16) + 64 * half;
    uint32_t tdP = tS + (C::tdP - C::tS);
    asm volatile("" : "+r"(tS), "+r"(tdP));
    // row r's 128-byte line in the SW128 tiles; the 16-byte chunk m8 of it lives at chunk m8 ^ (r & 7)
    const uint32_t xr = (uint32_t)(r & 7) << 4;
    const uint32_t sDSr = sDS + mn_sw128_offset(64 * half, r) - xr;
    const int64_t kpos = kv_base + r;
    const float sl2 = a.scale_log2;
    for (int n = 0; n < n_iter; ++n) {
      const int qt = qt_first + n / G;
      const float* st = reinterpret_cast<const float*>(smem + C::oStats + (n % QS) * C::kStats) + 64 * half;
      mbar_wait(bar(B_S), n & 1);
      if (warp == 0 && lane == 0) TRACE(0, n);
      tc_fence_after();
      float p[64];
      tmem_ld32(tS, reinterpret_cast<uint32_t*>(p));
      tmem_ld32(tS + 32, reinterpret_cast<uint32_t*>(p) + 32);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(bar(B_SFREE));
      if (warp == 0 && lane == 0) TRACE(13, n);
      // query column (within this half) < lim is masked: its query position is before the key position
      const int64_t lim64 = (a.causal ? (kpos - (a.q_pos0 + (int64_t)qt * 128)) : -1) - 64 * half;
      const int lim = (int)(lim64 < 0 ? 0 : (lim64 > 64 ? 64 : lim64));
      if (__any_sync(0xffffffffu, lim > 0)) {
        // tile straddling the diagonal: MUFU only (exact zeros under the mask)
#pragma unroll
        for (int i = 0; i < 64; i += 4) {
          const float4 l = lds4(st + i);
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
        for (int i = 0; i < 64; i += 4) {
          const float4 l = lds4(st + i);
          const float2 x0 = __ffma2_rn(make_float2(p[i], p[i + 1]), make_float2(sl2, sl2), make_float2(-l.x, -l.y));
          const float2 x1 =
              __ffma2_rn(make_float2(p[i + 2], p[i + 3]), make_float2(sl2, sl2), make_float2(-l.z, -l.w));
          p[i] = ex2(x0.x);
          p[i + 1] = ex2(x0.y);
          p[i + 2] = ex2(x1.x);
          p[i + 3] = ex2(x1.y);
        }
      }
      if (lane == 0 && n < 512) TRACE(14, 512 * warp + n);  // per softmax warp: slot 512 * warp + n
      // dP^T_n -> registers; its TMEM columns then receive P^T_n and dS^T_n (bf16), the A operands of dV and dK
      mbar_wait(bar(B_DP), n & 1);
      if (warp == 0 && lane == 0) TRACE(2, n);
      tc_fence_after();
      float dp[64];
      tmem_ld32(tdP, reinterpret_cast<uint32_t*>(dp));
      tmem_ld32(tdP + 32, reinterpret_cast<uint32_t*>(dp) + 32);
      tmem_wait_ld();
      if (warp == 0 && lane == 0) TRACE(15, n);
#pragma unroll
      for (int c = 0; c < 64; c += 32) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) pk[i / 2] = pack_bf16x2(p[c + i], p[c + i + 1]);
        tmem_st16(tdP + c / 2, pk);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(bar(B_P));
      if (lane == 0 && n < 512) TRACE(1, 512 * warp + n);  // per softmax warp: slot 512 * warp + n
      // dS = P o (dP - D) -> TMEM (dS^T bf16, A of dK) and smem (MN-major dS tile fp16, A of dQ)
      uint32_t pk[32];
      {
        // dS in place of dP (fp32), bf16 to TMEM; the fp16 copy for the smem tile is packed below
#pragma unroll
        for (int i = 0; i < 64; i += 4) {
          float2 a0, a1;
          if constexpr (C::kFoldD) {  // dP^T already holds dP - D
            a0 = __fmul2_rn(make_float2(p[i], p[i + 1]), make_float2(dp[i], dp[i + 1]));
            a1 = __fmul2_rn(make_float2(p[i + 2], p[i + 3]), make_float2(dp[i + 2], dp[i + 3]));
          } else {
            const float4 dd = lds4(st + 128 + i);
            a0 = __fmul2_rn(make_float2(p[i], p[i + 1]),
                            __fadd2_rn(make_float2(dp[i], dp[i + 1]), make_float2(-dd.x, -dd.y)));
            a1 = __fmul2_rn(make_float2(p[i + 2], p[i + 3]),
                            __fadd2_rn(make_float2(dp[i + 2], dp[i + 3]), make_float2(-dd.z, -dd.w)));
          }
          dp[i] = a0.x; dp[i + 1] = a0.y; dp[i + 2] = a1.x; dp[i + 3] = a1.y;
        }
#pragma unroll
        for (int c = 0; c < 64; c += 32) {
#pragma unroll
          for (int i = 0; i < 32; i += 2) pk[i / 2] = pack_bf16x2(dp[c + i], dp[c + i + 1]);
          tmem_st16(tdP + 32 + c / 2, pk);
        }
#pragma unroll
        for (int i = 0; i < 64; i += 2) pk[i / 2] = pack_f16x2(dp[i], dp[i + 1]);
      }
      if (n > 0) mbar_wait(bar(B_DSFREE), (n - 1) & 1);
      if (warp == 0 && lane == 0) TRACE(10, n);
#pragma unroll
      for (int m8 = 0; m8 < 8; ++m8) {
        const uint32_t w[4] = {pk[m8 * 4], pk[m8 * 4 + 1], pk[m8 * 4 + 2], pk[m8 * 4 + 3]};
        st_shared_v4(sDSr + (((uint32_t)m8 << 4) ^ xr), w);
      }
      tmem_wait_st();
      fence_async_shared();
      tc_fence_before();
      mbar_arrive(bar(B_DS));
      if (lane == 0 && n < 512) TRACE(3, 512 * warp + n);  // per softmax warp: slot 512 * warp + n
    }
    // ---- final dK (half 0) / dV (half 1), thread = key row
    const int64_t row = (int64_t)kt * 128 + r;  // row within the launch's key range
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
    // ------------------------------------------------------------------ dQ read-out (query rows)
    const int r = (warp - 8) * 32 + lane;
    {
      // fp16 copy of the K tile, same (swizzled) layout, elementwise
      if (n_iter > 0) mbar_wait(bar(B_KV), 0);
      const uint4* src = reinterpret_cast<const uint4*>(smem + C::oK);
      uint4* dst = reinterpret_cast<uint4*>(smem + C::oKH);
      for (int i = r; i < C::TB / 16; i += 128) {
        const uint4 x = src[i];
        const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
        uint32_t ws[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xs[q]));
          ws[q] = pack_f16x2(f.x, f.y);
        }
        dst[i] = make_uint4(ws[0], ws[1], ws[2], ws[3]);
      }
      fence_async_shared();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(B_KH));
    }
    uint32_t tdQ = tmem + C::tdQ + (((warp & 3) * 32) << 16);
    asm volatile("" : "+r"(tdQ));
    for (int n = 0; n < n_iter; ++n) {
      const int qt = qt_first + n / G, h = g * G + n % G;
      mbar_wait(bar(B_DQF), n & 1);
      TRACE(9, n);
      tc_fence_after();
      float v[D];
#pragma unroll
      for (int c = 0; c < D; c += 16) tmem_ld16(tdQ + c, reinterpret_cast<uint32_t(&)[16]>(v[c]));
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(bar(B_DQE));
      // Independent row groups of kDQRows rows (one per dQ warp at 32), each with its own part of the staging, barrier
      // and issuing thread: while one group waits for its previous reduce-add to finish reading its staging, the TMA
      // engine works on the others'.  Staging per group: D/32 column chunks [GR rows][32 fp32] (128B-swizzled) + a
      // [GR][16] chunk (64B-swizzled) when D % 32 == 16 — the 16-byte piece j of row rr lives at piece j ^ (rr & 7)
      // (resp. j ^ ((rr >> 1) & 3)), so the 32 rows of a warp hit all 32 banks.
      constexpr int GR = kDQRows;  // rows per staging group (one issuing thread, one named barrier or warp)
      const int hrow = r / GR, rr = r % GR;
      const bool hlead = rr == 0;
      constexpr uint32_t HB = GR * D * 4;
      auto gsync = [&] {
        if constexpr (GR == 32) __syncwarp();
        else named_bar(2 + hrow, GR);
      };
      if (hlead) bulk_wait_read0();
      gsync();
      const float2 sc = make_float2(a.scale, a.scale);
      uint8_t* stg = smem + C::oDQ + hrow * HB;
#pragma unroll
      for (int c = 0; c < D; c += 4) {
        const float2 x0 = __fmul2_rn(make_float2(v[c], v[c + 1]), sc);
        const float2 x1 = __fmul2_rn(make_float2(v[c + 2], v[c + 3]), sc);
        const int j = (c & 31) >> 2;
        const uint32_t off = c < (D / 32) * 32 ? (c >> 5) * (GR * 128) + rr * 128 + ((j ^ (rr & 7)) << 4)
                                               : (D / 32) * (GR * 128) + rr * 64 + ((j ^ ((rr >> 1) & 3)) << 4);
        *reinterpret_cast<float4*>(stg + off) = make_float4(x0.x, x0.y, x1.x, x1.y);
      }
      fence_async_shared();
      gsync();
      if (hlead) {
        const uint32_t sb = sDQ + hrow * HB;
        const int row0 = qt * 128 + GR * hrow;
#pragma unroll
        for (int cc = 0; cc < D / 32; ++cc) tma_reduce_add_3d(&tm.dq32h, sb + cc * (GR * 128), cc * 32, row0, h);
        if (D % 32) tma_reduce_add_3d(&tm.dq16h, sb + (D / 32) * (GR * 128), (D / 32) * 32, row0, h);
        bulk_commit();
        if (hrow == 0) TRACE(11, n);
      }
    }
    if (r % kDQRows == 0) bulk_wait0();
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (MC) cluster_sync();  // no CTA leaves while its partner may still multicast into it or arrive on it
  if (warp == 13) tmem_dealloc<512>(tmem);
#undef TRACE
}

template <int D>
int launch_pipe(const BwdArgs& a, cudaStream_t s) {
  using C = PipeCfg<D>;
  TmapSet tm;
  constexpr uint32_t kAtomCols = Tile<D>::kAtomCols;
  constexpr CUtensorMapSwizzle kSw = D == 80 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_128B;
  bool ok = make_tile_tmap<D>(&tm.q, a.q.base, a.q.rows, a.q.heads);
  ok &= make_tmap_rows_heads_dim(&tm.q64, a.q.base, a.q.rows, a.q.heads, D, kAtomCols, kCR, kSw);
  ok &= make_tmap_rows_heads_dim(&tm.o64, a.dout.base, a.dout.rows, a.dout.heads, D, kAtomCols, kCR, kSw);
  ok &= make_tile_tmap<D>(&tm.k, a.k.base, a.k.rows, a.k.heads);
  ok &= make_tile_tmap<D>(&tm.v, a.v.base, a.v.rows, a.v.heads);
  ok &= make_tile_tmap<D>(&tm.o, a.dout.base, a.dout.rows, a.dout.heads);
  ok &= make_tmap_f32_head_major(&tm.dq32h, a.dq_acc, a.n_q_rows, a.hq, D, a.dq_head_stride, 32, kDQRows,
                                 CU_TENSOR_MAP_SWIZZLE_128B);
  ok &= make_tmap_f32_head_major(&tm.dq16h, a.dq_acc, a.n_q_rows, a.hq, D, a.dq_head_stride, 16, kDQRows,
                                 CU_TENSOR_MAP_SWIZZLE_64B);
  if (!ok) return -1;
  const dim3 grid(a.n_kv_rows / 128, a.hq / a.G);
#ifndef FPDT_BWD_MC
#define FPDT_BWD_MC 1
#endif
  if (FPDT_BWD_MC && grid.x % kCS == 0) {
    if (int e = set_max_dynamic_smem((const void*)attn_bwd_pipe_kernel<D, true>, C::kSmem)) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = C::kSmem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kCS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaError_t e = cudaLaunchKernelEx(&cfg, attn_bwd_pipe_kernel<D, true>, tm, a)) return (int)e;
    return (int)cudaGetLastError();
  }
  if (int e = set_max_dynamic_smem((const void*)attn_bwd_pipe_kernel<D, false>, C::kSmem)) return e;
  attn_bwd_pipe_kernel<D, false><<<grid, kThreads, C::kSmem, s>>>(tm, a);
  return (int)cudaGetLastError();
}

}  // namespace

// head_dim 64 / 80: this kernel; head_dim 128 runs attn_bwd_q64_sm100.cu (no TMEM room here for a 128-column dQ
// next to S^T, dP^T, dK and dV, nor shared memory for its staging)
int launch_attn_bwd_pipe_bf16(const BwdArgs& a, int head_dim, cudaStream_t s) {
  switch (head_dim) {
    case 64: return launch_pipe<64>(a, s);
    case 80: return launch_pipe<80>(a, s);
  }
  return -2;
}

// The bf16 backward pair kernel for each head_dim: this file's kernel at 64 / 80, the 64-row query-tile kernel at 128.
// (A CTA-pair variant, tcgen05 cta_group::2, is in the diagnostics library: correct but slower.)
int launch_attn_bwd_bf16(const BwdArgs& a, int head_dim, cudaStream_t s) {
  if (head_dim == 128) return launch_attn_bwd_q64_bf16(a, head_dim, s);
  return launch_attn_bwd_pipe_bf16(a, head_dim, s);
}

}  // namespace fpdt
