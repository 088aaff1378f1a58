// libfpdt host runtime, internal header (not installed, not part of the C-ABI): the context and in-process group
// objects, the schedule configuration, and the runtime services the chunk schedules are built from -- device buffer
// pool, events, the pinned host chunk store, the copy / all-to-all / point-to-point transfers, kernel launch wrappers
// with timing, the projection GEMM wrappers and the key/value fetch strategies.
//   fpdt_runtime.cpp   those services
//   schedule_fwd.cpp   the forward chunk schedule (§4.1)
//   schedule_bwd.cpp   the backward chunk schedules (fig:bw_db; §8(a) B1-B8, NEXT-1 Q-outer order)
//   fpdt_ctx.cpp       the C-ABI entry points of include/fpdt.h
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <chrono>
#include <cmath>
#include <condition_variable>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "fpdt.h"
#include "kernels.h"

namespace fpdt_rt {
using namespace fpdt;

extern thread_local std::string g_last_error;

struct Fail {
  int code;
};

#define FPDT_CHECK_CUDA(x)                                                                          \
  do {                                                                                              \
    cudaError_t e_ = (x);                                                                           \
    if (e_ != cudaSuccess) {                                                                        \
      g_last_error = std::string(#x) + ": " + cudaGetErrorString(e_);                               \
      throw Fail{e_ == cudaErrorMemoryAllocation ? FPDT_ERR_DEVICE_OOM : FPDT_ERR_CUDA};            \
    }                                                                                               \
  } while (0)

#define FPDT_CHECK_NCCL(x)                                                                          \
  do {                                                                                              \
    ncclResult_t r_ = (x);                                                                          \
    if (r_ != ncclSuccess) {                                                                        \
      g_last_error = std::string(#x) + ": " + ncclGetErrorString(r_);                               \
      throw Fail{FPDT_ERR_NCCL};                                                                    \
    }                                                                                               \
  } while (0)

#define FPDT_CHECK_LAUNCH(x)                                                                        \
  do {                                                                                              \
    int r_ = (x);                                                                                   \
    if (r_ != 0) {                                                                                  \
      g_last_error = std::string(#x) + " failed: " +                                                \
                     (r_ > 0 ? cudaGetErrorString((cudaError_t)r_) : "tensor map / argument error"); \
      throw Fail{FPDT_ERR_CUDA};                                                                    \
    }                                                                                               \
  } while (0)

// The communicator is non-blocking (so that a rank that never joins makes ncclCommInitRank time out instead of hang):
// any NCCL call may return ncclInProgress; poll the communicator until the call has been accepted.
void nccl_settle(ncclComm_t comm, double timeout_s, const char* what);

[[noreturn]] void fail(int code, const std::string& msg);

struct Config {
  int64_t s_local = 0;
  int Hq = 0, Hkv = 0, d = 0, causal = 1;
  int64_t C = 0;
  int p = 1, dtype = 0, offload = 1;
  float scale = 0.f;
  // derived
  int64_t c = 0, u = 0, S = 0;
  int hq = 0, hkv = 0, G = 1, eb = 2;
  bool operator==(const Config& o) const {
    return s_local == o.s_local && Hq == o.Hq && Hkv == o.Hkv && d == o.d && causal == o.causal && C == o.C &&
           p == o.p && dtype == o.dtype && offload == o.offload && scale == o.scale;
  }
};

// Fused QKV projection of fpdt_block_fwd / fpdt_block_bwd; nullptr = the
// attention-only calls.  Row-major: x, dx [s_local][hidden]; w [hidden][(Hq + 2 Hkv) * d] (q heads, k, v); dw fp32.
// Optional output projection after the attention: w_o [Hq * d][hidden], y = o w_o [s_local][hidden]; backward from
// dy: dO = dy w_o^T, dw_o = o^T dy (fp32).
struct Proj {
  const void* x = nullptr;
  const void* w = nullptr;
  void* dx = nullptr;
  float* dw = nullptr;
  int hidden = 0;
  const void* w_o = nullptr;
  void* y = nullptr;
  float* dw_o = nullptr;
};

struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
};

enum BufId {
  B_OACC, B_LSEACC, B_LSESAVE, B_OHAT, B_KVSLOT0, B_KVSLOT1, B_A2A_SEND0, B_A2A_SEND1, B_A2A_RECV0, B_A2A_RECV1,
  B_STORE, B_D, B_DQDEV, B_QSLOT0, B_QSLOT1, B_DOSLOT0, B_DOSLOT1, B_DQSLOT0, B_DQSLOT1, B_DKACC, B_DVACC,
  B_BWD_SEND, B_BWD_RECV, B_LSE_T, B_LSE_RECV, B_DOSTORE, B_ORESID, B_RESSTORE, B_DORES, B_DQRES, B_DKVSLOT0,
  B_DKVSLOT1, B_DKVRES, B_KVSLOT2, B_KVSLOT3, B_DKVSLOT2, B_DKVSLOT3, B_QOSEND, B_QORECV, B_PROJ0, B_PROJ1,
  B_PROJ2, B_DOUT, B_OHAT1, B_BWD_SEND1, B_BWD_RECV1, B_KVALL0, B_KVALL1, B_KVSTAGE, B_KVGATHER, B_X0, B_X1,
  B_HQ, B_HK, B_HV, B_HO, B_HLSE, B_HDO, B_HDQ, B_HDK, B_HDV, B_NUM
};
}  // namespace fpdt_rt

// In-process group (fpdt_group_create): world_size ranks in ONE process on ONE device, one host thread per
// rank.  Its all-to-all is a copy-engine exchange with NCCL's send/recv layout (recv block q = rank q's send
// block r); everything else is the code the NCCL path runs.  For single-GPU multi-rank tests.
struct fpdt_group {
  int p = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  int64_t generation = 0;
  std::vector<const void*> send;
  std::vector<std::vector<const void*>> send_to;  // p2p: per rank, its send buffer for each destination (or null)
  std::vector<uint64_t> arg_hash;  // fpdt_set_debug_checks
  std::vector<cudaEvent_t> ev_sent, ev_read;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const int64_t gen = generation;
    if (++arrived == p) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

struct fpdt_ctx {
  int p = 1, rank = 0, device = 0;
  ncclComm_t comm = nullptr;
  fpdt_group* group = nullptr;  // non-null: in-process group instead of NCCL
  // world size 1 created with an NCCL id: the sequence-parallel path with a one-rank communicator (every exchange an
  // ncclAlltoAll of the rank with itself), so that one GPU runs the production NCCL data plane
  bool xch1 = false;
  cudaStream_t s_comm = nullptr, s_h2d = nullptr, s_d2h = nullptr;
  // Q-outer backward: second compute stream (pairs of one query chunk run two at a time) and its slot events
  cudaStream_t s_comp2 = nullptr;
  int qo_streams = 2;  // FPDT_BWD_QO_STREAMS (1 or 2)
  double nccl_timeout_s = 300.0;  // FPDT_NCCL_TIMEOUT_S: bound on waiting for NCCL initialisation / call acceptance
  bool check_args = false;        // fpdt_set_debug_checks: compare the call arguments across ranks first
  // scheduler stress (debug, FPDT_STRESS_NS > 0): a random sleep kernel of up to stress_ns ns goes onto the stream of
  // every copy, all-to-all, GEMM and attention launch, before it (SURVEY §4 tier 5)
  uint32_t stress_ns = 0;
  uint64_t stress_state = 0x9E3779B97F4A7C15ull;
  cudaEvent_t ev_qo_free[4] = {}, ev_qo_filled[4] = {}, ev_qo_done[4] = {}, ev_qo_send[3] = {}, ev_fork = nullptr,
              ev_join = nullptr;
  uint8_t* host = nullptr;
  size_t host_bytes = 0;
  uint8_t* host_dkv = nullptr;  // Q-outer backward: fp32 dK/dV partials [u][2][C][hkv][d] (fpdt_set_bwd_order)
  // fetch strategy B (fpdt_set_fetch_strategy, rank 0 only): every rank's key/value chunks [u][p][C][2hkv][d]
  uint8_t* host_kvall = nullptr;
  size_t host_kvall_bytes = 0;
  // hidden-state offload of the block calls (fpdt_set_hidden_offload): x chunks [u][c][hidden]
  uint8_t* host_x = nullptr;
  size_t host_x_bytes = 0;
  bool hidden_offload = false, saved_hidden_offload = false;
  std::vector<cudaEvent_t> ev_xoff;
  cudaEvent_t ev_x_free[2] = {}, ev_x_filled[2] = {};
  size_t host_dkv_bytes = 0;
  fpdt_rt::DevBuf bufs[fpdt_rt::B_NUM];
  // per-chunk events
  std::vector<cudaEvent_t> ev_off, ev_doff, ev_dqoff, ev_dkvoff, ev_a2a, ev_up;
  cudaEvent_t ev_enter = nullptr, ev_slot_free[2] = {}, ev_slot_filled[2] = {}, ev_q_free[2] = {}, ev_q_filled[2] = {},
              ev_dq_ready[2] = {}, ev_kv_free[2] = {}, ev_kv_filled[2] = {}, ev_recv_used_c[2] = {},
              ev_recv_used_d[2] = {}, ev_ohat_free[2] = {}, ev_bsend_free[2] = {}, ev_kvall_free[2] = {}, ev_kvall_filled[2] = {},
              ev_kvg_free = nullptr, ev_o_ready = nullptr, ev_comm_done = nullptr, ev_d2h_done = nullptr,
              ev_h2d_done = nullptr, ev_tmp = nullptr;
  // saved state
  bool fwd_done = false;
  fpdt_rt::Config saved;
  int saved_hidden = 0;  // > 0: the saved forward was fpdt_block_fwd with this hidden size
  bool saved_has_wo = false;  // ... with the output projection
  // block-sparsity plan (fpdt_set_sparsity): keep[m*u + i] over (query chunk m, key chunk i); empty = dense.
  // The forward copies it into saved_plan; the backward of that forward uses the copy.
  std::vector<uint8_t> plan, saved_plan;
  int64_t plan_u = 0;
  const void *saved_q = nullptr, *saved_k = nullptr, *saved_v = nullptr;
  // the saved forward was fpdt_attn_fwd_host: its caller's host q (the world-size-1 backward fetches q_i from it) and
  // host o (the backward's o argument; the forward's device mirror of it still holds the output)
  bool saved_hostio = false;
  const void *saved_host_q = nullptr, *saved_host_o = nullptr;
  // HBM residency budget (fpdt_set_residency): key/value chunks i < res_kv and query-side chunks i >= u - res_q stay
  // on the device (offload = 1 only); the forward copies the setting, its backward uses the copy
  int64_t res_kv = 0, res_q = 0, saved_res_kv = 0, saved_res_q = 0;
  int bwd_order = FPDT_BWD_KV_OUTER;  // fpdt_set_bwd_order
  int fetch_strategy = FPDT_FETCH_PER_RANK, saved_fetch = FPDT_FETCH_PER_RANK;  // fpdt_set_fetch_strategy
  fpdt_stats stats{};
  // kernel timing
  bool timing = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> t_fwd, t_bwd;
  std::vector<std::pair<cudaStream_t, int64_t>> t_fwd_src, t_bwd_src;  // launch stream and call number per launch
  size_t n_fwd = 0, n_bwd = 0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> t_a2a;  // all-to-all timing (p > 1), with the kernel timing
  std::vector<int64_t> t_a2a_bytes;
  size_t n_a2a = 0;
  int64_t call_seq = 0;  // fpdt_attn_* / fpdt_block_* calls so far (kernel-gap accounting)
  // every event created once in create_ctx (destroyed by fpdt_ctx_destroy; null handles are skipped)
  std::vector<cudaEvent_t> fixed_events() const {
    std::vector<cudaEvent_t> v = {ev_enter, ev_o_ready, ev_comm_done, ev_d2h_done, ev_h2d_done, ev_tmp, ev_fork, ev_join,
                                  ev_kvg_free};
    for (int b = 0; b < 2; ++b)
      for (cudaEvent_t e : {ev_slot_free[b], ev_slot_filled[b], ev_q_free[b], ev_q_filled[b], ev_dq_ready[b],
                            ev_kv_free[b], ev_kv_filled[b], ev_recv_used_c[b], ev_recv_used_d[b], ev_ohat_free[b],
                            ev_bsend_free[b], ev_kvall_free[b], ev_kvall_filled[b], ev_x_free[b], ev_x_filled[b]})
        v.push_back(e);
    for (int b = 0; b < 4; ++b) v.insert(v.end(), {ev_qo_free[b], ev_qo_filled[b], ev_qo_done[b]});
    for (int b = 0; b < 3; ++b) v.push_back(ev_qo_send[b]);
    return v;
  }
};

namespace fpdt_rt {

// true when the schedules run the sequence-parallel exchanges (world size > 1, or world size 1 with a one-rank NCCL
// communicator: fpdt_ctx::xch1); false: world size 1 works on the caller's rows in place
inline bool exchanges(const fpdt_ctx* ctx) { return ctx->p > 1 || ctx->xch1; }

void* dev(fpdt_ctx* ctx, int id, size_t bytes);

// Which chunks stay on the device under the residency budget.  Key/value chunk i is resident
// when i < rkv: the forward fetches chunk i for every later query chunk, so the first chunks save the most fetches.
// Query-side chunk i (q_i, dO_i and its dq partial) is resident when i >= u - rq: the backward fetches chunk i for
// every key chunk j <= i, so the last chunks save the most.  slot[m]: index of chunk m in the resident device store
// (p > 1: the whole head-layout chunk after the all-to-all), qslot[m]: index among the query-side resident chunks.
struct Residency {
  int64_t u = 0, rkv = 0, rq = 0, n = 0, nq = 0;
  std::vector<int64_t> slot, qslot;
  bool kv(int64_t i) const { return i < rkv; }
  bool q(int64_t i) const { return i >= u - rq; }
};

Residency make_residency(int64_t u, int64_t rkv, int64_t rq);

// NVTX ranges (header-only NVTX3: no-ops unless a tool such as nsys is attached) around the host-side enqueue of each
// chunk's work, each exchange and each pair launch, so a timeline tool can line them up with the streams.
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
};

void ensure_events(std::vector<cudaEvent_t>& v, size_t n);

void rec(cudaEvent_t e, cudaStream_t s);

// scheduler stress: a sleep of a random length in [0, stress_ns) on stream s (no-op unless FPDT_STRESS_NS is set)
void stress(fpdt_ctx* ctx, cudaStream_t s);

void wait(cudaStream_t s, cudaEvent_t e);

Config make_config(int64_t s_local, int Hq, int Hkv, int d, int causal, int64_t C, int p, int dtype, int offload,
                   float scale);

// Host chunk store layout (offload=1): per chunk m, q_m [C][hq][d], kv_m [C][2hkv][d], dO_m [C][hq][d] (eb bytes),
// dq_acc_m [hq][C][d] fp32 (head-major, the layout of the device dq accumulators).
struct HostLayout {
  size_t q_bytes, kv_bytes, do_bytes, dq_bytes, total;
  size_t q(int64_t m) const { return (size_t)m * q_bytes; }
  size_t kv(int64_t m, int64_t u) const { return (size_t)u * q_bytes + (size_t)m * kv_bytes; }
  size_t dO(int64_t m, int64_t u) const { return (size_t)u * (q_bytes + kv_bytes) + (size_t)m * do_bytes; }
  size_t dq(int64_t m, int64_t u) const { return (size_t)u * (q_bytes + kv_bytes + do_bytes) + (size_t)m * dq_bytes; }
};

HostLayout host_layout(const Config& c);

// Host-link bytes (H2D + D2H) of the offloaded backward's chunk loop in either order (fpdt_set_bwd_order), for
// FPDT_BWD_AUTO.  keep(i, j): block (query chunk i, key chunk j) is computed; kres / qres: residency.
//   KV-outer: per j kv_j; per kept (i, j): q_i, dO_i, and the dq partial of i in (unless first) and out
//     (unless i == j, where dq_i is final).
//   Q-outer: per i q_i, dO_i; per kept (i, j): kv_j, and the dK/dV partial of j in (unless first) and out (unless
//     i is the last query chunk attending j).
template <class Keep>
int64_t bwd_host_bytes(int order, const Config& c, int64_t rkv, int64_t rq, const Keep& keep) {
  const int64_t u = c.u;
  const int64_t kv = c.C * 2 * c.hkv * c.d * c.eb, qc = c.C * c.hq * c.d * c.eb;
  const int64_t dqc = c.C * c.hq * c.d * 4, dkvc = c.C * 2 * c.hkv * c.d * 4;
  auto kres = [&](int64_t i) { return i < rkv; };
  auto qres = [&](int64_t i) { return i >= u - rq; };
  int64_t b = 0;
  if (order == FPDT_BWD_KV_OUTER) {
    std::vector<char> started((size_t)u, 0);
    for (int64_t j = 0; j < u; ++j) {
      if (!kres(j)) b += kv;
      for (int64_t i = j; i < u; ++i) {
        if (!keep(i, j)) continue;
        if (!qres(i)) b += 2 * qc + (started[(size_t)i] ? dqc : 0) + (i != j ? dqc : 0);
        started[(size_t)i] = 1;
      }
    }
  } else {
    std::vector<int64_t> last((size_t)u, 0);
    for (int64_t j = 0; j < u; ++j)
      for (int64_t i = j; i < u; ++i)
        if (keep(i, j)) last[(size_t)j] = i;
    std::vector<char> started((size_t)u, 0);
    for (int64_t i = 0; i < u; ++i) {
      if (!qres(i)) b += 2 * qc;
      for (int64_t j = 0; j <= i; ++j) {
        if (!keep(i, j)) continue;
        if (!kres(j)) b += kv + (started[(size_t)j] ? dkvc : 0) + (i != last[(size_t)j] ? dkvc : 0);
        started[(size_t)j] = 1;
      }
    }
  }
  return b;
}

void ensure_host(fpdt_ctx* ctx, size_t bytes);

void h2d(fpdt_ctx* ctx, void* dst, const void* src, size_t bytes);

void d2h(fpdt_ctx* ctx, void* dst, const void* src, size_t bytes);

// the caller's rows of the host-memory calls (fpdt_attn_fwd_host / fpdt_attn_bwd_host), on the same two copy streams
void h2d_io(fpdt_ctx* ctx, void* dst, const void* src, size_t bytes);

void d2h_io(fpdt_ctx* ctx, void* dst, const void* src, size_t bytes);

void d2h_2d(fpdt_ctx* ctx, void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t rows);

// All-to-all on the comm stream: send [p][count] -> recv [p][count], recv block q = rank q's send block `rank`.
void alltoall(fpdt_ctx* ctx, const void* send, void* recv, size_t count_per_peer, int dtype);

// Debug check (fpdt_set_debug_checks): every rank must enter each collective call with the same arguments (SPMD);
// a mismatch would otherwise hang or corrupt the all-to-alls.  The ranks compare a 64-bit hash of them first
// (NCCL: max-reductions of h and ~h on the comm stream plus a host sync; local group: through the group object).
uint64_t hash_mix(uint64_t h, uint64_t v);

void check_collective_args(fpdt_ctx* ctx, int call, const Config& c, int hidden);

// Point-to-point exchange on the comm stream (strategy B of the key/value fetch, fpdt_set_fetch_strategy): this rank
// sends send_to[q] (bytes, nullable) to rank q and receives recv_from[q] (nullable) from rank q; the ranks' calls
// pair up (a send to q for every receive of q).  Self-transfers are device copies.
void p2p(fpdt_ctx* ctx, const void* const* send_to, void* const* recv_from, size_t bytes);

struct TimedScope {
  fpdt_ctx* ctx;
  bool fwd;
  cudaStream_t s;
  std::pair<cudaEvent_t, cudaEvent_t>* ev = nullptr;
  TimedScope(fpdt_ctx* c, bool f, cudaStream_t st) : ctx(c), fwd(f), s(st) {
    if (!ctx->timing) return;
    auto& v = fwd ? ctx->t_fwd : ctx->t_bwd;
    auto& src = fwd ? ctx->t_fwd_src : ctx->t_bwd_src;
    size_t& n = fwd ? ctx->n_fwd : ctx->n_bwd;
    if (v.size() <= n) {
      cudaEvent_t a, b;
      FPDT_CHECK_CUDA(cudaEventCreate(&a));
      FPDT_CHECK_CUDA(cudaEventCreate(&b));
      v.push_back({a, b});
      src.push_back({nullptr, 0});
    }
    src[n] = {s, ctx->call_seq};
    ev = &v[n++];
    rec(ev->first, s);
  }
  ~TimedScope() {
    if (ev) cudaEventRecord(ev->second, s);
  }
};

void launch_fwd(fpdt_ctx* ctx, const Config& c, const FwdArgs& a, cudaStream_t s);

void launch_bwd(fpdt_ctx* ctx, const Config& c, const BwdArgs& a, cudaStream_t s);

// ------------------------------------------------------------------------------------------ projection GEMMs
// Hand-written GEMMs (gemm_sm100.cu): tcgen05 with fp32 accumulation in bf16 mode, true-FP32 SIMT in fp32 mode.
// Y[rows][n] (row stride ldy) = X[rows][k] (ldx) W[k][n] (ldw)       (forward projection); with `sc` the
// output is scattered straight into the all-to-all send layout instead (the F3 pack fused into the GEMM)
void gemm_xw(fpdt_ctx* ctx, int dtype, const void* X, int64_t ldx, const void* W, int64_t ldw, void* Y, int64_t ldy,
             int64_t rows, int64_t k, int64_t n, cudaStream_t s, const ScatterOut* sc = nullptr);

// dX[rows][k] (ldx) = dY[rows][n] (ldy) W^T                            (hidden-state gradient)
void gemm_dx(fpdt_ctx* ctx, int dtype, const void* dY, int64_t ldy, const void* W, int64_t ldw, void* dX, int64_t ldx,
             int64_t rows, int64_t k, int64_t n, cudaStream_t s);

// dW[k][n] fp32 (= or +=) X[rows][k]^T dY[rows][n]                       (weight gradient, summed over chunks)
void gemm_dw(fpdt_ctx* ctx, int dtype, const void* X, int64_t ldx, const void* dY, int64_t ldy, float* dW, int64_t rows,
             int64_t k, int64_t n, bool accumulate, cudaStream_t s);

// ------------------------------------------------------------------------------------------ key/value fetch strategies
// (fig:avg_time: "each GPU fetches its own chunk" (A) vs "one GPU fetches and
// scatters over NVLink" (B)).  A: every rank offloads its head-layout key/value chunk to its own pinned store and
// fetches it back over its own host link.  B: rank 0 holds every rank's key/value chunks: at the offload each rank
// sends its chunk to rank 0 (gather), which writes the p blocks to its pinned store; at a fetch rank 0 moves the p
// blocks host -> device and sends rank r its block (scatter).  Query-side chunks (q, dO, dq partials) stay per rank.
struct KvFetch {
  fpdt_ctx* ctx;
  const Config& c;
  bool leader_mode;  // strategy B at p > 1
  size_t blk;        // bytes of one rank's key/value chunk [C][2hkv][d]
  uint8_t* kvall[2] = {nullptr, nullptr};
  uint8_t *stage = nullptr, *gather = nullptr;

  KvFetch(fpdt_ctx* x, const Config& cfg, int strategy) : ctx(x), c(cfg) {
    leader_mode = strategy == FPDT_FETCH_LEADER && c.p > 1 && c.offload;
    blk = (size_t)c.C * 2 * c.hkv * c.d * c.eb;
    if (!leader_mode) return;
    stage = (uint8_t*)dev(ctx, B_KVSTAGE, blk);
    if (ctx->rank == 0) {
      gather = (uint8_t*)dev(ctx, B_KVGATHER, blk * c.p);
      for (int b = 0; b < 2; ++b) kvall[b] = (uint8_t*)dev(ctx, b ? B_KVALL1 : B_KVALL0, blk * c.p);
      const size_t need = (size_t)c.u * c.p * blk;
      if (ctx->host_kvall_bytes < need) {
        if (ctx->host_kvall) {
          FPDT_CHECK_CUDA(cudaDeviceSynchronize());
          cudaFreeHost(ctx->host_kvall);
          ctx->host_kvall = nullptr;
          ctx->host_kvall_bytes = 0;
        }
        void* hp = nullptr;
        cudaError_t e = cudaHostAlloc(&hp, need, cudaHostAllocDefault);
        if (e != cudaSuccess) {
          cudaGetLastError();
          fail(FPDT_ERR_HOST_OOM, "pinned all-rank key/value store of " + std::to_string(need) + " bytes: " +
                                      cudaGetErrorString(e));
        }
        ctx->host_kvall = static_cast<uint8_t*>(hp);
        ctx->host_kvall_bytes = need;
      }
    }
  }
  void init_events(cudaStream_t cs) {
    if (!leader_mode) return;
    for (int b = 0; b < 2; ++b) rec(ctx->ev_kvall_free[b], cs);
    rec(ctx->ev_kvg_free, cs);
  }
  // offload of chunk m's key/value block (head layout, rows `pitch` bytes apart) after ev_a2a[m]; records ev_off[m]
  // once the block is in the store it will be fetched from
  void offload(int64_t m, const uint8_t* kv_src, size_t pitch, const HostLayout& hl) {
    const size_t row_kv2 = (size_t)2 * c.hkv * c.d * c.eb;
    if (!leader_mode) {
      wait(ctx->s_d2h, ctx->ev_a2a[m]);
      d2h_2d(ctx, ctx->host + hl.kv(m, c.u), row_kv2, kv_src, pitch, row_kv2, c.C);
      return;
    }
    const int p = c.p, r = ctx->rank;
    FPDT_CHECK_CUDA(cudaMemcpy2DAsync(stage, row_kv2, kv_src, pitch, row_kv2, c.C, cudaMemcpyDeviceToDevice,
                                      ctx->s_comm));
    std::vector<const void*> send(p, nullptr);
    std::vector<void*> recv(p, nullptr);
    send[0] = stage;
    if (r == 0) {
      wait(ctx->s_comm, ctx->ev_kvg_free);
      for (int q = 0; q < p; ++q) recv[q] = gather + (size_t)q * blk;
    }
    p2p(ctx, send.data(), recv.data(), blk);
    if (r == 0) {
      rec(ctx->ev_tmp, ctx->s_comm);
      wait(ctx->s_d2h, ctx->ev_tmp);
      d2h(ctx, ctx->host_kvall + (size_t)m * p * blk, gather, (size_t)p * blk);
      rec(ctx->ev_kvg_free, ctx->s_d2h);
    }
  }
  // fetch of key/value chunk i into `slot` after ev_free (the slot's last reader); records ev_filled
  void fetch(int64_t i, uint8_t* slot, int sl, cudaEvent_t ev_free, cudaEvent_t ev_filled, const HostLayout& hl) {
    if (!leader_mode) {
      wait(ctx->s_h2d, ev_free);
      wait(ctx->s_h2d, ctx->ev_off[i]);
      h2d(ctx, slot, ctx->host + hl.kv(i, c.u), blk);
      rec(ev_filled, ctx->s_h2d);
      return;
    }
    const int p = c.p, r = ctx->rank;
    if (r == 0) {
      wait(ctx->s_h2d, ctx->ev_kvall_free[sl]);
      wait(ctx->s_h2d, ctx->ev_off[i]);
      h2d(ctx, kvall[sl], ctx->host_kvall + (size_t)i * p * blk, (size_t)p * blk);
      rec(ctx->ev_kvall_filled[sl], ctx->s_h2d);
      wait(ctx->s_comm, ctx->ev_kvall_filled[sl]);
    }
    wait(ctx->s_comm, ev_free);
    std::vector<const void*> send(p, nullptr);
    std::vector<void*> recv(p, nullptr);
    recv[0] = slot;
    if (r == 0)
      for (int q = 0; q < p; ++q) send[q] = kvall[sl] + (size_t)q * blk;
    p2p(ctx, send.data(), recv.data(), blk);
    rec(ev_filled, ctx->s_comm);
    if (r == 0) rec(ctx->ev_kvall_free[sl], ctx->s_comm);
  }
};

// Caller rows in host memory (fpdt_attn_fwd_host / fpdt_attn_bwd_host).  forward() and backward() then run on device
// mirrors of the caller's tensors (the q, k, v, o, ... arguments) and stage the caller's rows through them chunk by
// chunk on the library's own copy streams: chunk m's upload is enqueued just ahead of its first reader (one chunk
// ahead of the compute, in the same stream order as the chunk fetches), each chunk's output rows leave as soon as
// they are final.  World size 1 also fetches q_i and dO_i for the backward straight from the caller's host rows
// (their layout is the host store's), so those are never offloaded.
struct HostIO {
  const void *q = nullptr, *k = nullptr, *v = nullptr, *dout = nullptr;  // host inputs
  void *o = nullptr, *dq = nullptr, *dk = nullptr, *dv = nullptr;        // host outputs
  float* lse = nullptr;
  bool upload_o = false;  // backward: o is not the saved forward's output (its mirror is stale): upload it first
};

// the chunk schedules (schedule_fwd.cpp, schedule_bwd.cpp); pj: the fused projection of fpdt_block_fwd/bwd, io: the
// caller's rows in host memory (fpdt_attn_fwd_host/bwd_host)
void forward(fpdt_ctx* ctx, const Config& c, const void* q, const void* k, const void* v, void* o, float* lse,
             cudaStream_t cs, const Proj* pj = nullptr, const HostIO* io = nullptr);
void backward(fpdt_ctx* ctx, const Config& c, const void* o, const void* dout, void* dq, void* dk, void* dv,
              cudaStream_t cs, const Proj* pj = nullptr, const HostIO* io = nullptr);

}  // namespace fpdt_rt
