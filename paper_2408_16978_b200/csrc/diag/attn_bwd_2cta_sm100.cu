// Backward chunk-pair attention for sm_100a, head_dim 64 / 80, on CTA PAIRS (tcgen05 cta_group::2).
//
// DIAGNOSTICS LIBRARY ONLY (libfpdt_diag.so, fpdt_debug_pair which = 3): parity-green against the oracle but slower
// than the single-CTA kernel (686 vs 858 TFLOP/s on the C = 64K, 32 x 80 pair; DESIGN.md §6 has the timeline), so the
// FPDT schedule does not use it.
//
// Same operation as the other backward kernels: one (key/value chunk j, query chunk i) step of FPDT's nested backward
// loop (fig:bw_db).  KV-stationary: a cluster of two CTAs on two SMs holds 256 key
// rows of one KV head (CTA r: rows [128 r, 128 r + 128)) and walks the 128-row query tiles of the range and the G
// query heads of its group:
//   S^T  = K Q^T            P^T  = exp2(S^T*scale*log2e - lse2)       (recompute)
//   dP^T = V dO^T           dS^T = P^T o (dP^T - D)
//   dV  += P^T dO           dK  += dS^T Q          dQ_partial = dS K over all 256 keys (TMA bulk reduce-add)
//
// Why a pair: the single-CTA kernel is bound by shared-memory bandwidth (an SS-MMA with M = 128 and
// N <= 128 consumes all 128 B/clk/SM) and by the per-SM write path of the fp32 dQ reduce-add (40 KB per 128 x 128
// unit).  With M = 256 the pair's two tensor cores share every Q / dO operand (each CTA supplies half of the N rows),
// and the dQ product contracts over 256 keys, so each CTA reduce-adds 64 query rows (20 KB per unit) instead of 128.
//
// Numerics: the dQ product runs in fp16 (dS and K rounded to fp16, fp32 accumulation) instead of bf16.  dQ_i =
// sigma sum_j dS_ij k_j is a sum whose terms cancel (sum_j dS_ij = 0 for the exact gradient), so a common offset of
// the keys multiplies the rounding error of dS: with bf16 dS a key drift of 32 in one dimension (fpdt_inputs "drift")
// costs ~1e-2 relative error in dQ, fp16's three extra mantissa bits make it ~1.5e-3.  dS^T stays bf16 for dK += dS^T Q
// (no such cancellation there).
//
// Operand layouts (shared memory, SW32 atoms of 16 columns x rows; every MMA descriptor must address the same bytes
// in both CTAs of the pair):
//   KA, V   own 128 key rows, all head_dim atoms (A of S^T and dP^T, K-major)
//   Q, dO   per query tile, two regions:
//             E: the CTA's 64 query rows (64 r .. 64 r + 63) of every atom (B of S^T / dP^T, K-major, N split)
//             R: all 128 query rows of the CTA's half of the padded head_dim columns (B of dK / dV, MN-major, N split)
//           2 stages each.
//   KB      fp16 K of all 256 keys, the CTA's half of the padded head_dim columns (B of dQ, MN-major, N split)
//   dS      fp16 [256 keys x 64 query rows of this CTA] MN-major SW128 (A of dQ): the partner's keys' half arrives
//           over DSMEM as one 16 KB bulk copy (TMA engine) from the partner's staging buffer, completing on this CTA's
//           mbarrier (128 threads x 8 st.async of 16 B measured ~4 B/clk)
// TMEM (per CTA): S^T [0,128) | dP^T [128,256) (then P^T, dS^T bf16 per query half) | dQ (2x2 layout: lanes 0-63 hold
//   columns [0, DP/2) of the CTA's 64 query rows, lanes 64-127 columns [DP/2, DP)) | dK | dV.
// Warps (512 threads): 0-7 softmax gradient (thread = key row; warpgroup h = query columns [64 h, 64 h + 64)), 8-11 dQ
//   read-out and reduce-add, 12 TMA producer, 13 TMEM allocator + (leader CTA only) the single MMA-issuing thread.
#include "kernels.h"
#include "sm100_ptx.cuh"
#include "smem_layout.cuh"
#include "tma_host.h"

namespace fpdt {
namespace {

using namespace ptx;

constexpr int kThreads = 512;
constexpr int kLaunchRegs = (65536 / kThreads) & ~7;  // 128
constexpr int kRegsSoftmax = 168, kRegsDQ = 104, kRegsCtl = 72;
static_assert(2 * 128 * (kRegsSoftmax - kLaunchRegs) <= 128 * (2 * kLaunchRegs - kRegsDQ - kRegsCtl), "register pool");

template <int D>
struct Cfg2 {
  static_assert(D == 64 || D == 80, "head_dim 64 or 80");
  static constexpr int DP = D == 80 ? 96 : 64;  // padded head_dim of the N-split products (N % 32 for TS-MMAs)
  static constexpr int NA = D / 16;              // SW32 atoms of head_dim
  static constexpr int NH = DP / 32;             // atoms per CTA half of DP
  static constexpr int AT = 4096;                // one [128 x 16] bf16 atom
  static constexpr int QE = 2, QR = 2, OE = 2, OR = 2, ST = 2;
  static constexpr int kE = NA * 2048;           // E region: 64 rows x NA atoms
  static constexpr int kR = NH * AT;             // R region: 128 rows x NH atoms
  static constexpr int oKA = 0, oV = NA * AT, oKB = 2 * NA * AT;
  static constexpr int kKB = NH * 2 * AT;        // 256 rows x NH atoms (fp16)
  static constexpr int oQE = oKB + kKB, oQR = oQE + QE * kE, oOE = oQR + QR * kR, oOR = oOE + OE * kE;
  static constexpr int oDS = ((oOR + OR * kR + 1023) / 1024) * 1024;
  static constexpr int kDS = 256 * 64 * 2;
  static constexpr int oSTG = oDS + kDS;           // staging of the dS half that goes to the partner (16 KB)
  static constexpr int oDQ = oSTG + kDS / 2;
  static constexpr int kDQ = 64 * D * 4;
  static constexpr int oStats = oDQ + kDQ;
  static constexpr int oBars = oStats + ST * 1024;
  static constexpr int kSmem = oBars + 512;
  static_assert(kSmem <= 227 * 1024, "shared memory budget");
  static constexpr uint32_t tS = 0, tdP = 128, tdQ = 256, tdK = 256 + DP / 2, tdV = tdK + DP;
  static_assert(tdV + DP <= 512, "TMEM budget");
};

struct TmapSet2 {
  CUtensorMap qe, qr, oe, orr, ka, v, dq32h, dq16h;
};

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_f16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
// instruction descriptor, kind::f16 with fp16 A and B, fp32 D
__host__ __device__ constexpr uint32_t idesc_f16(uint32_t M, uint32_t N, uint32_t a_mn, uint32_t b_mn) {
  return (1u << 4) | (a_mn << 15) | (b_mn << 16) | ((N >> 3) << 17) | ((M >> 4) << 24);
}
__device__ __forceinline__ void mma2_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma2_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(id), "r"(acc));
}
// arrive on the mbarrier at the same offset in BOTH CTAs of the pair when the issued MMAs complete
__device__ __forceinline__ void commit2(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"((uint16_t)3)
      : "memory");
}
// TMA tile load into this CTA's shared memory, completing on an mbarrier of either CTA of the pair
__device__ __forceinline__ void tma_load_3d_pair(uint32_t dst, const CUtensorMap* m, uint32_t cluster_bar, int c0, int c1,
                                                 int c2, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(cluster_bar), "l"(policy)
      : "memory");
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
// arrive (count 1) on an mbarrier given by its shared::cluster address, releasing this thread's prior writes
// (shared memory and, after tcgen05.fence::before_thread_sync, TMEM) at cluster scope
__device__ __forceinline__ void arrive_cluster(uint32_t cluster_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar) : "memory");
}
// the same without memory ordering: for hand-offs of TMEM (ordered by tcgen05.wait + fence::before_thread_sync) --
// a release at cluster scope waits for every prior memory operation of the thread (measured ~1000+ clk here)
__device__ __forceinline__ void arrive_cluster_relaxed(uint32_t cluster_bar) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar) : "memory");
}
// bulk copy of this CTA's shared memory into the partner's (shared::cluster address), complete_tx on its mbarrier
__device__ __forceinline__ void bulk_copy_to_peer(uint32_t dst_cluster, uint32_t src, uint32_t bytes, uint32_t bar_cluster) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   dst_cluster),
               "r"(src), "r"(bytes), "r"(bar_cluster)
               : "memory");
}
[[maybe_unused]] __device__ __forceinline__ void st_async_u4(uint32_t cluster_addr, const uint32_t (&w)[4], uint32_t cluster_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                   cluster_addr),
               "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(cluster_bar)
               : "memory");
}

template <int D>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
attn_bwd_2cta_kernel(const __grid_constant__ TmapSet2 tm, const __grid_constant__ BwdArgs a) {
  using C = Cfg2<D>;
  constexpr int NA = C::NA, NH = C::NH, DP = C::DP;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = smem_u32(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::oBars);
  auto bar = [&](int i) { return smem_u32(&bars[i]); };
  // Barriers.  "leader": waited on by the MMA thread of CTA 0, arrivals / transactions from both CTAs;
  // "both": completed in both CTAs by a multicast MMA commit; "local": this CTA only.
  constexpr int B_KV = 0,                                  // leader: K, V tiles of both CTAs
      B_QEF = 1, B_QEE = B_QEF + C::QE,                    // leader full / both empty: Q E-region stages
      B_QRF = B_QEE + C::QE, B_QRE = B_QRF + C::QR,        // Q R-region stages
      B_OEF = B_QRE + C::QR, B_OEE = B_OEF + C::OE,        // dO E-region stages
      B_ORF = B_OEE + C::OE, B_ORE = B_ORF + C::OR,        // dO R-region stages
      B_STF = B_ORE + C::OR, B_STE = B_STF + C::ST,        // local: stats stages (full / consumed by 8 warps)
      B_S = B_STE + C::ST, B_DP = B_S + 1,                 // both: S^T_n, dP^T_n in TMEM
      B_SFREE = B_DP + 1, B_P = B_SFREE + 1, B_DST = B_P + 1,  // leader: 16 warp arrivals each (dS^T_n in TMEM)
      B_DSS = B_DST + 1,                                   // leader: 8 warp arrivals (both CTAs' dS_n tiles complete)
      B_DSRX = B_DSS + 1,                                  // local: the partner's half of dS_n has arrived
      B_DSL = B_DSRX + 1,                                  // local: this CTA's own half of dS_n is written (4 warps)
      B_DSFREE = B_DSL + 1, B_DQF = B_DSFREE + 1,         // both: dQ_n has read dS_n / dQ_n in TMEM
      B_DQE = B_DQF + 1, B_KB = B_DQE + 1,                 // leader: 8 warp arrivals each
      B_KVDONE = B_KB + 1, B_NUM = B_KVDONE + 1;           // both
  static_assert(B_NUM <= 60, "barrier area");
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::oBars + 60 * 8);

  const uint32_t warp = warp_id(), lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  auto lead = [&](int i) { return mapa(bar(i), 0); };  // shared::cluster address of barrier i of CTA 0
  const int pair = blockIdx.x >> 1;
  const int g = blockIdx.y;
  const int G = a.G;
  const int64_t pair_kbase = a.kv_pos0 + (int64_t)pair * 256;
  const int64_t kv_base = pair_kbase + 128 * rank;
  int qt_first = 0;
  const int n_qt_total = a.n_q_rows / 128;
  if (a.causal) {
    const int64_t rel = pair_kbase - a.q_pos0;  // first query tile that can see a key of the pair
    if (rel > 0) qt_first = (int)(rel / 128);
    if (qt_first > n_qt_total) qt_first = n_qt_total;
  }
  const int n_iter = (n_qt_total - qt_first) * G;
  // debug timeline (fpdt_debug_pair trace): CTA blockIdx.x == trace_cta of head 0
  const bool tracing = a.trace != nullptr && (int)blockIdx.x == a.trace_cta && blockIdx.y == 0;
#define TRACE(ev, n)                                                        \
  do {                                                                      \
    if (tracing && (n) < 4096) a.trace[(ev) * 4096 + (n)] = clock64();      \
  } while (0)

  if (warp == 13) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (warp == 12 && lane == 0) {
    mbar_init(bar(B_KV), 1);
    for (int s = 0; s < C::QE; ++s) { mbar_init(bar(B_QEF + s), 1); mbar_init(bar(B_QEE + s), 1); }
    for (int s = 0; s < C::QR; ++s) { mbar_init(bar(B_QRF + s), 1); mbar_init(bar(B_QRE + s), 1); }
    for (int s = 0; s < C::OE; ++s) { mbar_init(bar(B_OEF + s), 1); mbar_init(bar(B_OEE + s), 1); }
    for (int s = 0; s < C::OR; ++s) { mbar_init(bar(B_ORF + s), 1); mbar_init(bar(B_ORE + s), 1); }
    for (int s = 0; s < C::ST; ++s) { mbar_init(bar(B_STF + s), 1); mbar_init(bar(B_STE + s), 8); }
    mbar_init(bar(B_S), 1);
    mbar_init(bar(B_DP), 1);
    mbar_init(bar(B_SFREE), 16);
    mbar_init(bar(B_P), 16);
    mbar_init(bar(B_DST), 16);
    mbar_init(bar(B_DSS), 2);
    mbar_init(bar(B_DSL), 4);
    mbar_init(bar(B_DSRX), 1);
    mbar_init(bar(B_DSFREE), 1);
    mbar_init(bar(B_DQF), 1);
    mbar_init(bar(B_DQE), 8);
    mbar_init(bar(B_KB), 8);
    mbar_init(bar(B_KVDONE), 1);
    fence_mbar_init();
  }
  tc_fence_before();
  cluster_sync();  // both CTAs' barriers are initialised before any remote arrive, st.async or pair TMA
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sKA = base + C::oKA, sV = base + C::oV, sKB = base + C::oKB, sDS = base + C::oDS,
                 sDQ = base + C::oDQ;
  auto sQE = [&](int n) { return base + C::oQE + (n % C::QE) * C::kE; };
  auto sQR = [&](int n) { return base + C::oQR + (n % C::QR) * C::kR; };
  auto sOE = [&](int n) { return base + C::oOE + (n % C::OE) * C::kE; };
  auto sOR = [&](int n) { return base + C::oOR + (n % C::OR) * C::kR; };

  if (warp >= 12) {
    setmaxnreg_dec<kRegsCtl>();
    if (warp == 12) {
      // ---------------------------------------------------------------- TMA producer (both CTAs)
      if (elect_one() && n_iter > 0) {
        const uint64_t pol_kv = policy_evict_first(), pol_q = policy_evict_last();
        const int krow = (int)(a.kv_row0 + (int64_t)pair * 256 + 128 * rank);
        if (rank == 0) mbar_expect_tx(bar(B_KV), 2 * 2 * NA * C::AT);
        for (int t = 0; t < NA; ++t) {
          tma_load_3d_pair(sKA + t * C::AT, &tm.ka, lead(B_KV), 16 * t, a.k.head0 + g, krow, pol_kv);
          tma_load_3d_pair(sV + t * C::AT, &tm.v, lead(B_KV), 16 * t, a.v.head0 + g, krow, pol_kv);
        }
        for (int n = 0; n < n_iter; ++n) {
          const int qt = qt_first + n / G, h = g * G + n % G;
          const int qrow = (int)(a.q_row0 + (int64_t)qt * 128);
          {  // stats of the 128 query rows (local): lse2 [0,512) and D [512,1024)
            const int s = n % C::ST;
            if (n >= C::ST) mbar_wait(bar(B_STE + s), ((n / C::ST) - 1) & 1);
            const uint32_t fb = bar(B_STF + s), dst = base + C::oStats + s * 1024;
            mbar_expect_tx(fb, 1024);
            bulk_load(dst, a.lse2 + (int64_t)h * a.stat_ld + (int64_t)qt * 128, 512, fb);
            bulk_load(dst + 512, a.Dstat + (int64_t)h * a.stat_ld + (int64_t)qt * 128, 512, fb);
          }
          {  // Q, E region: this CTA's 64 rows of every atom
            const int s = n % C::QE;
            if (n >= C::QE) mbar_wait(bar(B_QEE + s), ((n / C::QE) - 1) & 1);
            if (rank == 0) mbar_expect_tx(bar(B_QEF + s), 2 * C::kE);
            for (int t = 0; t < NA; ++t)
              tma_load_3d_pair(sQE(n) + t * 2048, &tm.qe, lead(B_QEF + s), 16 * t, a.q.head0 + h, qrow + 64 * rank,
                               pol_q);
          }
          {  // dO, E region
            const int s = n % C::OE;
            if (n >= C::OE) mbar_wait(bar(B_OEE + s), ((n / C::OE) - 1) & 1);
            if (rank == 0) mbar_expect_tx(bar(B_OEF + s), 2 * C::kE);
            for (int t = 0; t < NA; ++t)
              tma_load_3d_pair(sOE(n) + t * 2048, &tm.oe, lead(B_OEF + s), 16 * t, a.dout.head0 + h,
                               qrow + 64 * rank, pol_q);
          }
          {  // dO, R region: 128 rows of this CTA's half of the (padded) head_dim; columns >= D read as zero
            const int s = n % C::OR;
            if (n >= C::OR) mbar_wait(bar(B_ORE + s), ((n / C::OR) - 1) & 1);
            if (rank == 0) mbar_expect_tx(bar(B_ORF + s), 2 * C::kR);
            for (int t = 0; t < NH; ++t)
              tma_load_3d_pair(sOR(n) + t * C::AT, &tm.orr, lead(B_ORF + s), 16 * (rank * NH + t), a.dout.head0 + h,
                               qrow, pol_q);
          }
          {  // Q, R region
            const int s = n % C::QR;
            if (n >= C::QR) mbar_wait(bar(B_QRE + s), ((n / C::QR) - 1) & 1);
            if (rank == 0) mbar_expect_tx(bar(B_QRF + s), 2 * C::kR);
            for (int t = 0; t < NH; ++t)
              tma_load_3d_pair(sQR(n) + t * C::AT, &tm.qr, lead(B_QRF + s), 16 * (rank * NH + t), a.q.head0 + h,
                               qrow, pol_q);
          }
        }
      }
    } else if (warp == 13) {
      // ---------------------------------------------------------------- MMA issuer (CTA 0 of the pair)
      if (rank == 0 && elect_one() && n_iter > 0) {
        const uint32_t idS = idesc_bf16(256, 128, 0, 0);  // S^T, dP^T: A = K / V rows, B = Q / dO rows, K-major
        const uint32_t idG = idesc_bf16(256, DP, 0, 1);   // dV, dK: A = P^T / dS^T in TMEM, B MN-major
        const uint32_t idQ = idesc_f16(128, DP, 1, 1);    // dQ: A = dS (fp16, MN-major), B = K (fp16, MN-major)
        const uint32_t tS = tmem + C::tS, tdP = tmem + C::tdP, tdQ = tmem + C::tdQ, tdK = tmem + C::tdK,
                       tdV = tmem + C::tdV;
        // Descriptors advance by adding (byte offset >> 4) to their start-address field; the loops stay rolled so that
        // no table of 64-bit descriptors is kept live in this warp's 72 registers.
        auto issue_S = [&](int n) {
          mbar_wait_cluster(bar(B_QEF + n % C::QE), (n / C::QE) & 1);
          tc_fence_after();
          uint64_t da = smem_desc(sKA, 16, 256, kSw32), db = smem_desc(sQE(n), 16, 256, kSw32);
#pragma unroll 1
          for (int kk = 0; kk < NA; ++kk, da += C::AT >> 4, db += 2048 >> 4) mma2_ss(tS, da, db, idS, kk > 0);
          commit2(bar(B_QEE + n % C::QE));
          commit2(bar(B_S));
        };
        auto issue_dP = [&](int n) {
          mbar_wait_cluster(bar(B_OEF + n % C::OE), (n / C::OE) & 1);
          tc_fence_after();
          uint64_t da = smem_desc(sV, 16, 256, kSw32), db = smem_desc(sOE(n), 16, 256, kSw32);
#pragma unroll 1
          for (int kk = 0; kk < NA; ++kk, da += C::AT >> 4, db += 2048 >> 4) mma2_ss(tdP, da, db, idS, kk > 0);
          commit2(bar(B_OEE + n % C::OE));
          commit2(bar(B_DP));
        };
        mbar_wait_cluster(bar(B_KV), 0);
        issue_S(0);
        issue_dP(0);
        for (int n = 0; n < n_iter; ++n) {
          const bool more = n + 1 < n_iter;
          if (more) {
            mbar_wait_cluster(bar(B_SFREE), n & 1);
            TRACE(6, n);
            issue_S(n + 1);
          }
          // dV += P^T dO_n
          mbar_wait_cluster(bar(B_P), n & 1);
          TRACE(4, n);
          mbar_wait_cluster(bar(B_ORF + n % C::OR), (n / C::OR) & 1);
          tc_fence_after();
          {
            uint64_t db = smem_desc(sOR(n), C::AT, 256, kSw32);
#pragma unroll 1
            for (int kk = 0; kk < 8; ++kk, db += 512 >> 4)
              mma2_ts(tdV, tdP + 64 * (kk >> 2) + (kk & 3) * 8, db, idG, (n > 0 || kk > 0));
          }
          commit2(bar(B_ORE + n % C::OR));
          // dK += dS^T Q_n
          mbar_wait_cluster(bar(B_DST), n & 1);
          TRACE(5, n);
          mbar_wait_cluster(bar(B_QRF + n % C::QR), (n / C::QR) & 1);
          tc_fence_after();
          {
            uint64_t db = smem_desc(sQR(n), C::AT, 256, kSw32);
#pragma unroll 1
            for (int kk = 0; kk < 8; ++kk, db += 512 >> 4)
              mma2_ts(tdK, tdP + 64 * (kk >> 2) + 32 + (kk & 3) * 8, db, idG, (n > 0 || kk > 0));
          }
          commit2(bar(B_QRE + n % C::QR));
          if (more) issue_dP(n + 1);  // overwrites P^T_n / dS^T_n after dV_n, dK_n in issue order
          TRACE(8, n);
          // dQ_n = dS K over the pair's 256 keys (fp16)
          mbar_wait_cluster(bar(B_DSS), n & 1);
          TRACE(7, n);
          if (n == 0) mbar_wait_cluster(bar(B_KB), 0);
          else mbar_wait_cluster(bar(B_DQE), (n - 1) & 1);
          tc_fence_after();
          {
            uint64_t da = smem_desc(sDS, 16384, 1024, kSw128), db = smem_desc(sKB, 2 * C::AT, 256, kSw32);
#pragma unroll 1
            for (int kk = 0; kk < 16; ++kk, da += 2048 >> 4, db += 512 >> 4) mma2_ss(tdQ, da, db, idQ, kk > 0);
          }
          commit2(bar(B_DQF));
          commit2(bar(B_DSFREE));
        }
        commit2(bar(B_KVDONE));
      }
    } else if (warp == 14) {
      // ---------------------------------------------------------------- dS hand-off (both CTAs)
      // this CTA's dS tile is complete once its own half is written (DSL) and the partner's bulk copy has landed
      // (DSRX); then the leader may issue dQ_n.  Kept off the softmax warps, which go on with the next tile.
      if (elect_one() && n_iter > 0) {
        mbar_expect_tx(bar(B_DSRX), 128 * 128);
        for (int n = 0; n < n_iter; ++n) {
          mbar_wait_cluster(bar(B_DSRX), n & 1);
          if (n + 1 < n_iter) mbar_expect_tx(bar(B_DSRX), 128 * 128);
          mbar_wait(bar(B_DSL), n & 1);
          TRACE(12, n);
          arrive_cluster_relaxed(lead(B_DSS));
        }
      }
    }
  } else if (warp < 8) {
    setmaxnreg_inc<kRegsSoftmax>();
    // ------------------------------------------------------------------ softmax gradient (key rows of this CTA)
    const int half = warp >> 2;  // query columns [64*half, 64*half+64)
    const int r = (warp & 3) * 32 + lane;
    uint32_t tS = tmem + C::tS + (((warp & 3) * 32) << 16) + 64 * half;
    uint32_t tdP = tS + (C::tdP - C::tS);
    asm volatile("" : "+r"(tS), "+r"(tdP));
    // dS_n (fp16) row of key kr = 128 rank + r, query columns of this half: to CTA `half` (the one whose dQ rows
    // these queries are), locally or over DSMEM
    // (the partner's rows are staged in this CTA first; their block of the partner's tile is contiguous:
    // rows [128 rank, 128 rank + 128) are bytes [16 KB rank, 16 KB (rank + 1)))
    const uint32_t row_off = (uint32_t)((r >> 3) * 1024 + (r & 7) * 128), xr = (uint32_t)(r & 7);
    const bool local = half == (int)rank;
    const uint32_t dsdst = local ? sDS + rank * 16384 + row_off : base + C::oSTG + row_off;
    const uint32_t peer_blk = mapa(sDS + rank * 16384, half), rxbar = mapa(bar(B_DSRX), half);
    const bool tx_owner = !local && (warp & 3) == 0 && lane == 0;  // issues the bulk copy to the partner
    const int64_t kpos = kv_base + r;
    const float sl2 = a.scale_log2;
    for (int n = 0; n < n_iter; ++n) {
      const int qt = qt_first + n / G;
      const int s = n % C::ST;
      mbar_wait(bar(B_STF + s), (n / C::ST) & 1);
      const float* st = reinterpret_cast<const float*>(smem + C::oStats + s * 1024) + 64 * half;
      mbar_wait(bar(B_S), n & 1);
      if (warp == 0 && lane == 0) TRACE(0, n);
      tc_fence_after();
      float p[64];
      tmem_ld32(tS, reinterpret_cast<uint32_t*>(p));
      tmem_ld32(tS + 32, reinterpret_cast<uint32_t*>(p) + 32);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) arrive_cluster_relaxed(lead(B_SFREE));
      if (warp == 0 && lane == 0) TRACE(13, n);
      const int64_t lim64 = (a.causal ? (kpos - (a.q_pos0 + (int64_t)qt * 128)) : -1) - 64 * half;
      const int lim = (int)(lim64 < 0 ? 0 : (lim64 > 64 ? 64 : lim64));
      if (__any_sync(0xffffffffu, lim > 0)) {
#pragma unroll
        for (int i = 0; i < 64; i += 4) {
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
        for (int i = 0; i < 64; i += 4) {
          const float4 l = *reinterpret_cast<const float4*>(st + i);
          const float2 x0 = __ffma2_rn(make_float2(p[i], p[i + 1]), make_float2(sl2, sl2), make_float2(-l.x, -l.y));
          const float2 x1 =
              __ffma2_rn(make_float2(p[i + 2], p[i + 3]), make_float2(sl2, sl2), make_float2(-l.z, -l.w));
          p[i] = ex2(x0.x);
          p[i + 1] = ex2(x0.y);
          p[i + 2] = ex2(x1.x);
          p[i + 3] = ex2(x1.y);
        }
      }
      // dP^T_n -> registers; its TMEM columns then receive P^T_n and dS^T_n (bf16), the A operands of dV and dK
      if (warp == 0 && lane == 0) TRACE(14, n);
      mbar_wait(bar(B_DP), n & 1);
      if (warp == 0 && lane == 0) TRACE(2, n);
      tc_fence_after();
      float dp[64];
      tmem_ld32(tdP, reinterpret_cast<uint32_t*>(dp));
      tmem_ld32(tdP + 32, reinterpret_cast<uint32_t*>(dp) + 32);
      tmem_wait_ld();
#pragma unroll
      for (int c = 0; c < 64; c += 32) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) pk[i / 2] = pack_bf16x2(p[c + i], p[c + i + 1]);
        tmem_st16(tdP + c / 2, pk);
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) arrive_cluster_relaxed(lead(B_P));
      if (warp == 0 && lane == 0) TRACE(1, n);
      // dS = P o (dP - D): bf16 to TMEM (dS^T, A of dK) first -- dK_n and dP^T_{n+1} wait only for that -- then fp16
      // to the dS tile of CTA `half` (A of dQ), locally or over DSMEM
      // dS in place of dP (fp32), so that P's registers die as dS is formed
#pragma unroll
      for (int i = 0; i < 64; i += 4) {
        const float4 dd = *reinterpret_cast<const float4*>(st + 128 + i);
        const float2 a0 = __fmul2_rn(make_float2(p[i], p[i + 1]),
                                     __fadd2_rn(make_float2(dp[i], dp[i + 1]), make_float2(-dd.x, -dd.y)));
        const float2 a1 = __fmul2_rn(make_float2(p[i + 2], p[i + 3]),
                                     __fadd2_rn(make_float2(dp[i + 2], dp[i + 3]), make_float2(-dd.z, -dd.w)));
        dp[i] = a0.x; dp[i + 1] = a0.y; dp[i + 2] = a1.x; dp[i + 3] = a1.y;
      }
#pragma unroll
      for (int c = 0; c < 64; c += 32) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) pk[i / 2] = pack_bf16x2(dp[c + i], dp[c + i + 1]);
        tmem_st16(tdP + 32 + c / 2, pk);
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        arrive_cluster_relaxed(lead(B_DST));
        mbar_arrive(bar(B_STE + s));  // stats stage consumed
      }
      if (n > 0) mbar_wait(bar(B_DSFREE), (n - 1) & 1);  // dQ_{n-1} has read both dS tiles
      if (warp == 0 && lane == 0) TRACE(10, n);
#pragma unroll
      for (int m8 = 0; m8 < 8; ++m8) {  // 16-byte chunk = 8 queries, fp16
        const uint32_t w[4] = {pack_f16x2(dp[m8 * 8], dp[m8 * 8 + 1]), pack_f16x2(dp[m8 * 8 + 2], dp[m8 * 8 + 3]),
                               pack_f16x2(dp[m8 * 8 + 4], dp[m8 * 8 + 5]), pack_f16x2(dp[m8 * 8 + 6], dp[m8 * 8 + 7])};
        st_shared_v4(dsdst + ((((uint32_t)m8) ^ xr) << 4), w);
      }
      if (!local) {
        // the partner's half: staged here, then one bulk DSMEM copy (the staging is free again once dQ_n is done,
        // which the DSFREE wait of the next tile observes)
        fence_async_shared();
        named_bar(4, 128);
        if (tx_owner) bulk_copy_to_peer(peer_blk, base + C::oSTG, 16384, rxbar);
      }
      if (warp == 0 && lane == 0) TRACE(15, n);
      if (local) {
        // the own half (generic stores) is made visible to the async proxy by each thread's proxy fence; warp 14
        // combines it with the partner's half and tells the leader (the arrive there carries no memory ordering:
        // a release at cluster scope costs ~1500 clk here, measured)
        fence_async_shared();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar(B_DSL));
        if (warp == 0 && lane == 0) TRACE(3, n);
      }
    }
    // ---- final dK (half 0) / dV (half 1), thread = key row
    const int64_t row = (int64_t)pair * 256 + 128 * rank + r;  // row within the launch's key range
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
    // ------------------------------------------------------------------ KB build, then dQ read-out
    const int t = (int)threadIdx.x - 256;  // 0..127
    {
      // KB = fp16 K of the pair's 256 keys, this CTA's half of the padded head_dim columns: atom at (kr, 16-byte
      // chunk j) holds K[kr][col0 + 8 j .. +8] at chunk j ^ ((kr >> 2) & 1) of row kr (the 32B swizzle TMA uses)
      const __nv_bfloat16* kb = reinterpret_cast<const __nv_bfloat16*>(a.k.base);
      const int64_t row0 = a.kv_row0 + (int64_t)pair * 256;
      for (int e = t; e < NH * 256 * 2; e += 128) {
        const int at = e / 512, kr2 = (e % 512) >> 1, j = e & 1;
        const int col0 = (int)(rank * NH + at) * 16 + 8 * j;
        uint32_t w[4] = {0u, 0u, 0u, 0u};
        if (col0 < D) {
          const uint4 x = *reinterpret_cast<const uint4*>(
              kb + ((row0 + kr2) * a.k.heads + a.k.head0 + g) * (int64_t)D + col0);
          const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xs[q]));
            w[q] = pack_f16x2(f.x, f.y);
          }
        }
        st_shared_v4(sKB + at * 2 * C::AT + kr2 * 32 + ((j ^ ((kr2 >> 2) & 1)) << 4), w);
      }
      fence_async_shared();
      __syncwarp();
      if (lane == 0 && n_iter > 0) arrive_cluster(lead(B_KB));
    }
    // dQ_n of this CTA's 64 query rows: TMEM lanes 0-63 hold columns [0, DP/2), lanes 64-127 [DP/2, DP)
    const int lg = (int)(warp & 3);
    const int rr = (lg * 32 + (int)lane) & 63;
    const int cbase = lg >= 2 ? DP / 2 : 0;
    uint32_t tdQ = tmem + C::tdQ + ((uint32_t)(lg * 32) << 16);
    asm volatile("" : "+r"(tdQ));
    const bool lead_thr = t == 0;
    for (int n = 0; n < n_iter; ++n) {
      const int qt = qt_first + n / G, h = g * G + n % G;
      mbar_wait(bar(B_DQF), n & 1);
      if (t == 0) TRACE(9, n);
      tc_fence_after();
      float v[DP / 2];
#pragma unroll
      for (int c = 0; c < DP / 2; c += 16) tmem_ld16(tdQ + c, reinterpret_cast<uint32_t(&)[16]>(v[c]));
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) arrive_cluster_relaxed(lead(B_DQE));
      // staging [64 rows x D] fp32: 32-column chunks 128B-swizzled, then a 16-column chunk 64B-swizzled (D = 80)
      if (lead_thr) bulk_wait_read0();  // the previous tile's reduce-add has read the staging
      named_bar(2, 128);
      const float2 sc = make_float2(a.scale, a.scale);
      uint8_t* stg = smem + C::oDQ;
#pragma unroll
      for (int i = 0; i < DP / 2; i += 4) {
        const int c = cbase + i;
        if (c >= D) break;
        const float2 x0 = __fmul2_rn(make_float2(v[i], v[i + 1]), sc);
        const float2 x1 = __fmul2_rn(make_float2(v[i + 2], v[i + 3]), sc);
        const int j = (c & 31) >> 2;
        const uint32_t off = c < (D / 32) * 32 ? (c >> 5) * 8192 + rr * 128 + ((j ^ (rr & 7)) << 4)
                                               : (D / 32) * 8192 + rr * 64 + ((j ^ ((rr >> 1) & 3)) << 4);
        *reinterpret_cast<float4*>(stg + off) = make_float4(x0.x, x0.y, x1.x, x1.y);
      }
      fence_async_shared();
      named_bar(2, 128);
      if (lead_thr) {
        const int row0 = qt * 128 + 64 * (int)rank;
#pragma unroll
        for (int cc = 0; cc < D / 32; ++cc) tma_reduce_add_3d(&tm.dq32h, sDQ + cc * 8192, cc * 32, row0, h);
        if (D % 32) tma_reduce_add_3d(&tm.dq16h, sDQ + (D / 32) * 8192, (D / 32) * 32, row0, h);
        bulk_commit();
        TRACE(11, n);
      }
    }
    if (lead_thr) bulk_wait0();
  }
  tc_fence_before();
  cluster_sync();  // neither CTA leaves while the partner may still write into its shared memory or TMEM
  if (warp == 13) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
#undef TRACE
}

template <int D>
int launch_2cta(const BwdArgs& a, cudaStream_t s) {
  using C = Cfg2<D>;
  if (a.n_kv_rows % 256) return -2;
  TmapSet2 tm;
  const CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_32B;
  bool ok = make_tmap_rows_heads_dim(&tm.qe, a.q.base, a.q.rows, a.q.heads, D, 16, 64, sw);
  ok &= make_tmap_rows_heads_dim(&tm.qr, a.q.base, a.q.rows, a.q.heads, D, 16, 128, sw);
  ok &= make_tmap_rows_heads_dim(&tm.oe, a.dout.base, a.dout.rows, a.dout.heads, D, 16, 64, sw);
  ok &= make_tmap_rows_heads_dim(&tm.orr, a.dout.base, a.dout.rows, a.dout.heads, D, 16, 128, sw);
  ok &= make_tmap_rows_heads_dim(&tm.ka, a.k.base, a.k.rows, a.k.heads, D, 16, 128, sw);
  ok &= make_tmap_rows_heads_dim(&tm.v, a.v.base, a.v.rows, a.v.heads, D, 16, 128, sw);
  ok &= make_tmap_f32_head_major(&tm.dq32h, a.dq_acc, a.n_q_rows, a.hq, D, a.dq_head_stride, 32, 64,
                                 CU_TENSOR_MAP_SWIZZLE_128B);
  ok &= make_tmap_f32_head_major(&tm.dq16h, a.dq_acc, a.n_q_rows, a.hq, D, a.dq_head_stride, 16, 64,
                                 CU_TENSOR_MAP_SWIZZLE_64B);
  if (!ok) return -1;
  if (int e = set_max_dynamic_smem((const void*)attn_bwd_2cta_kernel<D>, C::kSmem)) return e;
  attn_bwd_2cta_kernel<D><<<dim3(a.n_kv_rows / 128, a.hq / a.G), kThreads, C::kSmem, s>>>(tm, a);
  return (int)cudaGetLastError();
}

}  // namespace

int launch_attn_bwd_2cta_bf16(const BwdArgs& a, int head_dim, cudaStream_t s) {
  switch (head_dim) {
    case 64: return launch_2cta<64>(a, s);
    case 80: return launch_2cta<80>(a, s);
  }
  return -2;
}

}  // namespace fpdt
