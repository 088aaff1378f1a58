// libfpdt host runtime: context, pinned host chunk store, device slots, stream/event chunk scheduler,
// NCCL all-to-all, and the C-ABI entry points declared in include/fpdt.h.
//
// Schedules (§4.1-4.2):
//   forward, offload=1:  per chunk m: [comm] all-to-all of q,k,v chunk m (p>1)  [d2h] offload q_m, kv_m
//                        [compute] diagonal pair (m,m) ; for i<m: [h2d] fetch kv_i -> slot i%2,
//                        [compute] pair (m,i) with LSE merge ; [comm] all-to-all of O_m back (p>1)
//   forward, offload=0:  per chunk m one launch over the resident key range [0,(m+1)C)
//   backward, offload=1: D preprocess; per chunk all-to-all of (O,dO) (p>1); offload dO_m;
//                        for j (outer, key/value): [h2d] fetch kv_j; for i>=j (inner, query):
//                        [h2d] fetch q_i, dO_i, dq_acc_i (j>0) -> slot ; [compute] pair (i,j) ;
//                        i>j: [d2h] dq_acc_i -> host ; i==j: dq_j final ; after the inner loop dk_j, dv_j
//                        final -> [comm] all-to-all of dq_j,dk_j,dv_j back (p>1)
//   backward, offload=0: per j one launch over the resident query range [jC, S)
// Streams: compute (= the caller's stream), comm, h2d, d2h; every cross-stream dependency is an event.
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

using namespace fpdt;

namespace {

thread_local std::string g_last_error;

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
void nccl_settle(ncclComm_t comm, double timeout_s, const char* what) {
  ncclResult_t st = ncclInProgress;
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const ncclResult_t r = ncclCommGetAsyncError(comm, &st);
    if (r != ncclSuccess) st = r;
    if (st != ncclInProgress) break;
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s) {
      g_last_error = std::string(what) + ": timed out after " + std::to_string(timeout_s) +
                     " s (a rank did not join, or the ranks' calls differ)";
      throw Fail{FPDT_ERR_NCCL};
    }
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
  if (st != ncclSuccess) {
    g_last_error = std::string(what) + ": " + ncclGetErrorString(st);
    throw Fail{FPDT_ERR_NCCL};
  }
}

[[noreturn]] void fail(int code, const std::string& msg) {
  g_last_error = msg;
  throw Fail{code};
}

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

}  // namespace

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
  DevBuf bufs[B_NUM];
  // per-chunk events
  std::vector<cudaEvent_t> ev_off, ev_doff, ev_dqoff, ev_dkvoff, ev_a2a, ev_up;
  cudaEvent_t ev_enter = nullptr, ev_slot_free[2] = {}, ev_slot_filled[2] = {}, ev_q_free[2] = {}, ev_q_filled[2] = {},
              ev_dq_ready[2] = {}, ev_kv_free[2] = {}, ev_kv_filled[2] = {}, ev_recv_used_c[2] = {},
              ev_recv_used_d[2] = {}, ev_ohat_free[2] = {}, ev_bsend_free[2] = {}, ev_kvall_free[2] = {}, ev_kvall_filled[2] = {},
              ev_kvg_free = nullptr, ev_o_ready = nullptr, ev_comm_done = nullptr, ev_d2h_done = nullptr,
              ev_h2d_done = nullptr, ev_tmp = nullptr;
  // saved state
  bool fwd_done = false;
  Config saved;
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

namespace {

void* dev(fpdt_ctx* ctx, int id, size_t bytes) {
  DevBuf& b = ctx->bufs[id];
  if (b.bytes < bytes) {
    if (b.ptr) {
      FPDT_CHECK_CUDA(cudaDeviceSynchronize());
      FPDT_CHECK_CUDA(cudaFree(b.ptr));
      ctx->stats.device_bytes -= (int64_t)b.bytes;
      b.ptr = nullptr;
      b.bytes = 0;
    }
    cudaError_t e = cudaMalloc(&b.ptr, bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      b.ptr = nullptr;
      fail(FPDT_ERR_DEVICE_OOM, "cudaMalloc of " + std::to_string(bytes) + " bytes failed: " + cudaGetErrorString(e));
    }
    b.bytes = bytes;
    ctx->stats.device_bytes += (int64_t)bytes;
  }
  return b.ptr;
}

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
Residency make_residency(int64_t u, int64_t rkv, int64_t rq) {
  Residency r;
  r.u = u;
  r.rkv = std::min(rkv, u);
  r.rq = std::min(rq, u);
  r.slot.assign((size_t)u, -1);
  r.qslot.assign((size_t)u, -1);
  for (int64_t m = 0; m < u; ++m) {
    if (r.kv(m) || r.q(m)) r.slot[(size_t)m] = r.n++;
    if (r.q(m)) r.qslot[(size_t)m] = r.nq++;
  }
  return r;
}

// NVTX ranges (header-only NVTX3: no-ops unless a tool such as nsys is attached) around the host-side enqueue of each
// chunk's work, each exchange and each pair launch, so a timeline tool can line them up with the streams.
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
};

void ensure_events(std::vector<cudaEvent_t>& v, size_t n) {
  while (v.size() < n) {
    cudaEvent_t e;
    FPDT_CHECK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    v.push_back(e);
  }
}

void rec(cudaEvent_t e, cudaStream_t s) { FPDT_CHECK_CUDA(cudaEventRecord(e, s)); }
// scheduler stress: a sleep of a random length in [0, stress_ns) on stream s (no-op unless FPDT_STRESS_NS is set)
void stress(fpdt_ctx* ctx, cudaStream_t s) {
  if (!ctx->stress_ns) return;
  uint64_t& x = ctx->stress_state;
  x ^= x << 13;
  x ^= x >> 7;
  x ^= x << 17;
  FPDT_CHECK_LAUNCH(launch_stress_sleep((uint32_t)(x % ctx->stress_ns), s));
  ctx->stats.stress_sleeps++;
}
void wait(cudaStream_t s, cudaEvent_t e) { FPDT_CHECK_CUDA(cudaStreamWaitEvent(s, e, 0)); }

Config make_config(int64_t s_local, int Hq, int Hkv, int d, int causal, int64_t C, int p, int dtype, int offload,
                   float scale) {
  Config c;
  c.s_local = s_local; c.Hq = Hq; c.Hkv = Hkv; c.d = d; c.causal = causal; c.C = C; c.p = p;
  c.dtype = dtype; c.offload = offload ? 1 : 0;
  c.scale = scale > 0.f ? scale : (float)(1.0 / std::sqrt((double)d));
  if (s_local <= 0 || Hq <= 0 || Hkv <= 0 || C <= 0 || p <= 0) fail(FPDT_ERR_ARG, "non-positive size argument");
  if (d != 64 && d != 80 && d != 128) fail(FPDT_ERR_UNSUPPORTED, "head_dim must be 64, 80 or 128");
  if (causal != 1) fail(FPDT_ERR_UNSUPPORTED, "only causal attention (causal=1) is supported");
  if (dtype != FPDT_BF16 && dtype != FPDT_FP32) fail(FPDT_ERR_UNSUPPORTED, "dtype must be FPDT_BF16 or FPDT_FP32");
  if (C % p) fail(FPDT_ERR_DIVISIBILITY, "chunk_size % world_size != 0");
  c.c = C / p;
  if (s_local % c.c) fail(FPDT_ERR_DIVISIBILITY, "s_local % (chunk_size / world_size) != 0 (S % C != 0)");
  if (C % 256) fail(FPDT_ERR_DIVISIBILITY, "chunk_size must be a multiple of 256");
  if (Hq % p || Hkv % p) fail(FPDT_ERR_DIVISIBILITY, "head counts must be divisible by world_size");
  if (Hq % Hkv) fail(FPDT_ERR_DIVISIBILITY, "n_q_heads % n_kv_heads != 0");
  c.u = s_local / c.c;
  c.S = c.u * C;
  c.hq = Hq / p;
  c.hkv = Hkv / p;
  c.G = Hq / Hkv;
  c.eb = dtype == FPDT_BF16 ? 2 : 4;
  return c;
}

// Host chunk store layout (offload=1): per chunk m, q_m [C][hq][d], kv_m [C][2hkv][d], dO_m [C][hq][d] (eb bytes),
// dq_acc_m [hq][C][d] fp32 (head-major, the layout of the device dq accumulators).
struct HostLayout {
  size_t q_bytes, kv_bytes, do_bytes, dq_bytes, total;
  size_t q(int64_t m) const { return (size_t)m * q_bytes; }
  size_t kv(int64_t m, int64_t u) const { return (size_t)u * q_bytes + (size_t)m * kv_bytes; }
  size_t dO(int64_t m, int64_t u) const { return (size_t)u * (q_bytes + kv_bytes) + (size_t)m * do_bytes; }
  size_t dq(int64_t m, int64_t u) const { return (size_t)u * (q_bytes + kv_bytes + do_bytes) + (size_t)m * dq_bytes; }
};
HostLayout host_layout(const Config& c) {
  HostLayout h;
  h.q_bytes = (size_t)c.C * c.hq * c.d * c.eb;
  h.kv_bytes = (size_t)c.C * 2 * c.hkv * c.d * c.eb;
  h.do_bytes = h.q_bytes;
  h.dq_bytes = (size_t)c.C * c.hq * c.d * 4;
  h.total = (size_t)c.u * (h.q_bytes + h.kv_bytes + h.do_bytes + h.dq_bytes);
  return h;
}

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

void ensure_host(fpdt_ctx* ctx, size_t bytes) {
  if (ctx->host_bytes >= bytes) return;
  if (ctx->host) {
    FPDT_CHECK_CUDA(cudaDeviceSynchronize());
    cudaFreeHost(ctx->host);
    ctx->host = nullptr;
    ctx->host_bytes = 0;
  }
  void* p = nullptr;
  cudaError_t e = cudaHostAlloc(&p, bytes, cudaHostAllocDefault);
  if (e != cudaSuccess) {
    cudaGetLastError();
    fail(FPDT_ERR_HOST_OOM, "pinned host store of " + std::to_string(bytes) + " bytes: " + cudaGetErrorString(e));
  }
  ctx->host = static_cast<uint8_t*>(p);
  ctx->host_bytes = bytes;
  ctx->stats.host_arena_bytes = (int64_t)bytes;
}

void h2d(fpdt_ctx* ctx, void* dst, const void* src, size_t bytes) {
  Nvtx nv("fpdt:fetch_h2d");
  stress(ctx, ctx->s_h2d);
  FPDT_CHECK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->s_h2d));
  ctx->stats.bytes_h2d += (int64_t)bytes;
}
void d2h(fpdt_ctx* ctx, void* dst, const void* src, size_t bytes) {
  Nvtx nv("fpdt:offload_d2h");
  stress(ctx, ctx->s_d2h);
  FPDT_CHECK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->s_d2h));
  ctx->stats.bytes_d2h += (int64_t)bytes;
}
// the caller's rows of the host-memory calls (fpdt_attn_fwd_host / fpdt_attn_bwd_host), on the same two copy streams
void h2d_io(fpdt_ctx* ctx, void* dst, const void* src, size_t bytes) {
  Nvtx nv("fpdt:io_h2d");
  stress(ctx, ctx->s_h2d);
  FPDT_CHECK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->s_h2d));
  ctx->stats.bytes_io_h2d += (int64_t)bytes;
}
void d2h_io(fpdt_ctx* ctx, void* dst, const void* src, size_t bytes) {
  Nvtx nv("fpdt:io_d2h");
  stress(ctx, ctx->s_d2h);
  FPDT_CHECK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->s_d2h));
  ctx->stats.bytes_io_d2h += (int64_t)bytes;
}
void d2h_2d(fpdt_ctx* ctx, void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t rows) {
  Nvtx nv("fpdt:offload_d2h");
  stress(ctx, ctx->s_d2h);
  FPDT_CHECK_CUDA(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, rows, cudaMemcpyDeviceToHost, ctx->s_d2h));
  ctx->stats.bytes_d2h += (int64_t)(width * rows);
}

// All-to-all on the comm stream: send [p][count] -> recv [p][count], recv block q = rank q's send block `rank`.
void alltoall(fpdt_ctx* ctx, const void* send, void* recv, size_t count_per_peer, int dtype) {
  Nvtx nv("fpdt:alltoall");
  const size_t eb = dtype == FPDT_BF16 ? 2 : 4;
  stress(ctx, ctx->s_comm);
  std::pair<cudaEvent_t, cudaEvent_t>* tev = nullptr;
  if (ctx->timing) {
    if (ctx->t_a2a.size() <= ctx->n_a2a) {
      cudaEvent_t e0, e1;
      FPDT_CHECK_CUDA(cudaEventCreate(&e0));
      FPDT_CHECK_CUDA(cudaEventCreate(&e1));
      ctx->t_a2a.push_back({e0, e1});
      ctx->t_a2a_bytes.push_back(0);
    }
    ctx->t_a2a_bytes[ctx->n_a2a] = (int64_t)(count_per_peer * (ctx->p - 1) * eb);
    tev = &ctx->t_a2a[ctx->n_a2a++];
    rec(tev->first, ctx->s_comm);
  }
  if (!ctx->group) {
    const ncclResult_t r = ncclAlltoAll(send, recv, count_per_peer, dtype == FPDT_BF16 ? ncclBfloat16 : ncclFloat32,
                                        ctx->comm, ctx->s_comm);
    if (r != ncclSuccess && r != ncclInProgress) {
      g_last_error = std::string("ncclAlltoAll: ") + ncclGetErrorString(r);
      throw Fail{FPDT_ERR_NCCL};
    }
    nccl_settle(ctx->comm, ctx->nccl_timeout_s, "ncclAlltoAll");
  } else {
    // local group: publish the send buffer and its ready event, pull every peer's block, then hold the
    // comm stream until every peer has read ours (a send buffer is rewritten only after that).
    fpdt_group* g = ctx->group;
    const int r = ctx->rank, p = ctx->p;
    const size_t bytes = count_per_peer * eb;
    g->send[r] = send;
    FPDT_CHECK_CUDA(cudaEventRecord(g->ev_sent[r], ctx->s_comm));
    g->barrier();
    for (int q = 0; q < p; ++q) {
      FPDT_CHECK_CUDA(cudaStreamWaitEvent(ctx->s_comm, g->ev_sent[q], 0));
      FPDT_CHECK_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(recv) + q * bytes,
                                      static_cast<const uint8_t*>(g->send[q]) + r * bytes, bytes,
                                      cudaMemcpyDeviceToDevice, ctx->s_comm));
    }
    FPDT_CHECK_CUDA(cudaEventRecord(g->ev_read[r], ctx->s_comm));
    g->barrier();
    for (int q = 0; q < p; ++q) FPDT_CHECK_CUDA(cudaStreamWaitEvent(ctx->s_comm, g->ev_read[q], 0));
    g->barrier();  // nobody re-records ev_sent / ev_read before every rank has enqueued its waits
  }
  if (tev) rec(tev->second, ctx->s_comm);
  ctx->stats.bytes_a2a += (int64_t)(count_per_peer * (ctx->p - 1) * eb);
}

// Debug check (fpdt_set_debug_checks): every rank must enter each collective call with the same arguments (SPMD);
// a mismatch would otherwise hang or corrupt the all-to-alls.  The ranks compare a 64-bit hash of them first
// (NCCL: max-reductions of h and ~h on the comm stream plus a host sync; local group: through the group object).
uint64_t hash_mix(uint64_t h, uint64_t v) {
  h ^= v + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
  return h * 0xD1B54A32D192ED03ull;
}
void check_collective_args(fpdt_ctx* ctx, int call, const Config& c, int hidden) {
  if (!ctx->check_args || ctx->p == 1) return;
  uint64_t h = hash_mix(0, (uint64_t)call);
  for (uint64_t v : {(uint64_t)c.s_local, (uint64_t)c.Hq, (uint64_t)c.Hkv, (uint64_t)c.d, (uint64_t)c.causal,
                     (uint64_t)c.C, (uint64_t)c.p, (uint64_t)c.dtype, (uint64_t)c.offload, (uint64_t)hidden,
                     (uint64_t)ctx->bwd_order, (uint64_t)ctx->res_kv, (uint64_t)ctx->res_q, (uint64_t)ctx->plan_u,
                     (uint64_t)ctx->fetch_strategy,
                     (uint64_t)__builtin_bit_cast(uint32_t, c.scale)})
    h = hash_mix(h, v);
  for (uint8_t k : ctx->plan) h = hash_mix(h, k);
  uint64_t lo = h, hi = h;
  if (ctx->group) {
    fpdt_group* g = ctx->group;
    g->arg_hash[ctx->rank] = h;
    g->barrier();
    for (uint64_t x : g->arg_hash) lo = std::min(lo, x), hi = std::max(hi, x);
    g->barrier();
  } else {
    uint64_t* buf = nullptr;
    FPDT_CHECK_CUDA(cudaMallocAsync((void**)&buf, 16, ctx->s_comm));
    const uint64_t hv[2] = {h, ~h};
    FPDT_CHECK_CUDA(cudaMemcpyAsync(buf, hv, 16, cudaMemcpyHostToDevice, ctx->s_comm));
    const ncclResult_t r = ncclAllReduce(buf, buf, 2, ncclUint64, ncclMax, ctx->comm, ctx->s_comm);
    if (r != ncclSuccess && r != ncclInProgress) fail(FPDT_ERR_NCCL, std::string("ncclAllReduce: ") + ncclGetErrorString(r));
    nccl_settle(ctx->comm, ctx->nccl_timeout_s, "argument check");
    uint64_t out[2];
    FPDT_CHECK_CUDA(cudaMemcpyAsync(out, buf, 16, cudaMemcpyDeviceToHost, ctx->s_comm));
    FPDT_CHECK_CUDA(cudaFreeAsync(buf, ctx->s_comm));
    FPDT_CHECK_CUDA(cudaStreamSynchronize(ctx->s_comm));
    hi = out[0];
    lo = ~out[1];
  }
  if (lo != hi) fail(FPDT_ERR_ARG, "collective call arguments differ across ranks (fpdt_set_debug_checks)");
}

// Point-to-point exchange on the comm stream (strategy B of the key/value fetch, fpdt_set_fetch_strategy): this rank
// sends send_to[q] (bytes, nullable) to rank q and receives recv_from[q] (nullable) from rank q; the ranks' calls
// pair up (a send to q for every receive of q).  Self-transfers are device copies.
void p2p(fpdt_ctx* ctx, const void* const* send_to, void* const* recv_from, size_t bytes) {
  const int p = ctx->p, r = ctx->rank;
  stress(ctx, ctx->s_comm);
  if (send_to[r] && recv_from[r])
    FPDT_CHECK_CUDA(cudaMemcpyAsync(recv_from[r], send_to[r], bytes, cudaMemcpyDeviceToDevice, ctx->s_comm));
  if (!ctx->group) {
    FPDT_CHECK_NCCL(ncclGroupStart());
    for (int q = 0; q < p; ++q) {
      if (q == r) continue;
      if (send_to[q]) {
        const ncclResult_t e = ncclSend(send_to[q], bytes, ncclUint8, q, ctx->comm, ctx->s_comm);
        if (e != ncclSuccess && e != ncclInProgress) fail(FPDT_ERR_NCCL, std::string("ncclSend: ") + ncclGetErrorString(e));
      }
      if (recv_from[q]) {
        const ncclResult_t e = ncclRecv(recv_from[q], bytes, ncclUint8, q, ctx->comm, ctx->s_comm);
        if (e != ncclSuccess && e != ncclInProgress) fail(FPDT_ERR_NCCL, std::string("ncclRecv: ") + ncclGetErrorString(e));
      }
    }
    const ncclResult_t e = ncclGroupEnd();
    if (e != ncclSuccess && e != ncclInProgress) fail(FPDT_ERR_NCCL, std::string("ncclGroupEnd: ") + ncclGetErrorString(e));
    nccl_settle(ctx->comm, ctx->nccl_timeout_s, "p2p exchange");
  } else {
    fpdt_group* g = ctx->group;
    for (int q = 0; q < p; ++q) g->send_to[r][q] = send_to[q];
    FPDT_CHECK_CUDA(cudaEventRecord(g->ev_sent[r], ctx->s_comm));
    g->barrier();
    for (int q = 0; q < p; ++q) {
      if (q == r || !recv_from[q]) continue;
      if (!g->send_to[q][r]) fail(FPDT_ERR_STATE, "p2p: receive without a matching send");
      FPDT_CHECK_CUDA(cudaStreamWaitEvent(ctx->s_comm, g->ev_sent[q], 0));
      FPDT_CHECK_CUDA(cudaMemcpyAsync(recv_from[q], g->send_to[q][r], bytes, cudaMemcpyDeviceToDevice, ctx->s_comm));
    }
    FPDT_CHECK_CUDA(cudaEventRecord(g->ev_read[r], ctx->s_comm));
    g->barrier();
    for (int q = 0; q < p; ++q) FPDT_CHECK_CUDA(cudaStreamWaitEvent(ctx->s_comm, g->ev_read[q], 0));
    g->barrier();
  }
  for (int q = 0; q < p; ++q)
    if (q != r && send_to[q]) ctx->stats.bytes_a2a += (int64_t)bytes;
}

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

void launch_fwd(fpdt_ctx* ctx, const Config& c, const FwdArgs& a, cudaStream_t s) {
  Nvtx nv("fpdt:pair_fwd");
  stress(ctx, s);
  TimedScope t(ctx, true, s);
  if (c.dtype == FPDT_BF16)
    FPDT_CHECK_LAUNCH(launch_attn_fwd_bf16(a, c.d, s));
  else
    FPDT_CHECK_LAUNCH(launch_attn_fwd_f32(a, c.d, s));
  ctx->stats.kernel_launches++;
  ctx->stats.attn_launches++;
}
void launch_bwd(fpdt_ctx* ctx, const Config& c, const BwdArgs& a, cudaStream_t s) {
  Nvtx nv("fpdt:pair_bwd");
  stress(ctx, s);
  TimedScope t(ctx, false, s);
  if (c.dtype == FPDT_BF16)
    FPDT_CHECK_LAUNCH(launch_attn_bwd_bf16(a, c.d, s));
  else
    FPDT_CHECK_LAUNCH(launch_attn_bwd_f32(a, c.d, s));
  ctx->stats.kernel_launches += c.dtype == FPDT_BF16 ? 1 : 2;
  ctx->stats.attn_launches++;
}

// ------------------------------------------------------------------------------------------ projection GEMMs
// Hand-written GEMMs (gemm_sm100.cu): tcgen05 with fp32 accumulation in bf16 mode, true-FP32 SIMT in fp32 mode.
// Y[rows][n] (row stride ldy) = X[rows][k] (ldx) W[k][n] (ldw)       (forward projection); with `sc` the
// output is scattered straight into the all-to-all send layout instead (the F3 pack fused into the GEMM)
void gemm_xw(fpdt_ctx* ctx, int dtype, const void* X, int64_t ldx, const void* W, int64_t ldw, void* Y, int64_t ldy,
             int64_t rows, int64_t k, int64_t n, cudaStream_t s, const ScatterOut* sc = nullptr) {
  stress(ctx, s);
  FPDT_CHECK_LAUNCH(launch_gemm_xw(dtype == FPDT_FP32, X, ldx, W, ldw, Y, ldy, rows, k, n, sc, s));
  ctx->stats.kernel_launches++;
}
// dX[rows][k] (ldx) = dY[rows][n] (ldy) W^T                            (hidden-state gradient)
void gemm_dx(fpdt_ctx* ctx, int dtype, const void* dY, int64_t ldy, const void* W, int64_t ldw, void* dX, int64_t ldx,
             int64_t rows, int64_t k, int64_t n, cudaStream_t s) {
  stress(ctx, s);
  FPDT_CHECK_LAUNCH(launch_gemm_dx(dtype == FPDT_FP32, dY, ldy, W, ldw, dX, ldx, rows, k, n, s));
  ctx->stats.kernel_launches++;
}
// dW[k][n] fp32 (= or +=) X[rows][k]^T dY[rows][n]                       (weight gradient, summed over chunks)
void gemm_dw(fpdt_ctx* ctx, int dtype, const void* X, int64_t ldx, const void* dY, int64_t ldy, float* dW, int64_t rows,
             int64_t k, int64_t n, bool accumulate, cudaStream_t s) {
  stress(ctx, s);
  FPDT_CHECK_LAUNCH(launch_gemm_dw(dtype == FPDT_FP32, X, ldx, dY, ldy, dW, rows, k, n, accumulate, s));
  ctx->stats.kernel_launches++;
}

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

// ------------------------------------------------------------------------------------------ forward
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

void forward(fpdt_ctx* ctx, const Config& c, const void* q, const void* k, const void* v, void* o, float* lse,
             cudaStream_t cs, const Proj* pj = nullptr, const HostIO* io = nullptr) {
  Nvtx nv("fpdt:forward");
  const int64_t C = c.C, u = c.u;
  const int d = c.d, hq = c.hq, hkv = c.hkv, eb = c.eb, p = c.p;
  const size_t row_q = (size_t)hq * d * eb, row_kv2 = (size_t)2 * hkv * d * eb;
  const int hcomb = hq + 2 * hkv;  // combined head-layout buffer: q heads, k heads, v heads
  const float sl2 = c.scale * 1.4426950408889634f;
  float* lse_save = (float*)dev(ctx, B_LSESAVE, (size_t)hq * c.S * 4);
  __nv_bfloat16* o_resid = c.dtype == FPDT_BF16 ? (__nv_bfloat16*)dev(ctx, B_ORESID, (size_t)c.S * hq * d * 2) : nullptr;
  float* o_acc = nullptr;
  float* lse_acc = nullptr;
  if (c.offload) {
    o_acc = (float*)dev(ctx, B_OACC, (size_t)C * hq * d * 4);
    lse_acc = (float*)dev(ctx, B_LSEACC, (size_t)hq * C * 4);
  }
  ++ctx->call_seq;
  ensure_events(ctx->ev_off, u);
  ensure_events(ctx->ev_a2a, u);
  ensure_events(ctx->ev_xoff, u);
  if (io) ensure_events(ctx->ev_up, u);
  if (pj && ctx->saved_hidden_offload) {
    const size_t need = (size_t)u * c.c * pj->hidden * c.eb;
    if (ctx->host_x_bytes < need) {
      if (ctx->host_x) {
        FPDT_CHECK_CUDA(cudaDeviceSynchronize());
        cudaFreeHost(ctx->host_x);
        ctx->host_x = nullptr;
        ctx->host_x_bytes = 0;
      }
      void* hp = nullptr;
      cudaError_t e = cudaHostAlloc(&hp, need, cudaHostAllocDefault);
      if (e != cudaSuccess) {
        cudaGetLastError();
        fail(FPDT_ERR_HOST_OOM, "pinned hidden-state store of " + std::to_string(need) + " bytes: " + cudaGetErrorString(e));
      }
      ctx->host_x = static_cast<uint8_t*>(hp);
      ctx->host_x_bytes = need;
    }
  }
  rec(ctx->ev_enter, cs);
  for (cudaStream_t s : {ctx->s_comm, ctx->s_h2d, ctx->s_d2h}) wait(s, ctx->ev_enter);
  HostLayout hl{};
  if (c.offload) {
    hl = host_layout(c);
    ensure_host(ctx, hl.total);
  }
  // device store for resident mode with p > 1: gathered [S][hcomb][d]
  uint8_t* store = nullptr;
  if (!c.offload && p > 1) store = (uint8_t*)dev(ctx, B_STORE, (size_t)c.S * hcomb * d * eb);
  // head-layout output of a chunk before its return all-to-all (p > 1), double-buffered so that chunk m+1's pairs
  // run while chunk m's output is exchanged
  uint8_t* o_hat[2] = {nullptr, nullptr};
  if (p > 1)
    for (int b = 0; b < 2; ++b) o_hat[b] = (uint8_t*)dev(ctx, b ? B_OHAT1 : B_OHAT, (size_t)C * hq * d * eb);
  uint8_t* a2a_send[2] = {nullptr, nullptr};
  uint8_t* a2a_recv[2] = {nullptr, nullptr};
  if (p > 1) {
    for (int b = 0; b < 2; ++b) {
      a2a_send[b] = (uint8_t*)dev(ctx, B_A2A_SEND0 + b, (size_t)C * hcomb * d * eb);
      if (c.offload) a2a_recv[b] = (uint8_t*)dev(ctx, B_A2A_RECV0 + b, (size_t)C * hcomb * d * eb);
    }
  }
  // fused projection (fpdt_block_fwd): chunk m of the hidden state is projected on the comm stream just before
  // its all-to-all; the GEMM's epilogue writes the all-to-all send layout [p][c][hq + 2hkv][d] directly
  // (the pack fused into the GEMM); at p = 1 that layout is the combined head layout [C][Hq + 2Hkv][d] itself.
  const bool proj = pj != nullptr, headbuf = p > 1 || proj;
  const int64_t ntot = (int64_t)(c.Hq + 2 * c.Hkv) * d;
  ScatterOut scat;
  scat.d = d; scat.Hq = c.Hq; scat.Hkv = c.Hkv; scat.hq = hq; scat.hkv = hkv;
  scat.peer_stride = c.c * hcomb * d;
  if (proj && p == 1)
    for (int b = 0; b < 2; ++b) a2a_recv[b] = (uint8_t*)dev(ctx, B_A2A_RECV0 + b, (size_t)C * hcomb * d * eb);
  const Residency R = make_residency(u, c.offload ? ctx->saved_res_kv : 0, c.offload ? ctx->saved_res_q : 0);
  uint8_t* resstore = (p > 1 && R.n > 0) ? (uint8_t*)dev(ctx, B_RESSTORE, (size_t)R.n * C * hcomb * d * eb) : nullptr;
  auto res_chunk = [&](int64_t m) { return resstore + (size_t)R.slot[(size_t)m] * C * hcomb * d * eb; };
  uint8_t* kv_slot[2] = {nullptr, nullptr};
  KvFetch kvf(ctx, c, ctx->saved_fetch);
  kvf.init_events(cs);
  if (c.offload) {
    kv_slot[0] = (uint8_t*)dev(ctx, B_KVSLOT0, (size_t)C * row_kv2);
    kv_slot[1] = (uint8_t*)dev(ctx, B_KVSLOT1, (size_t)C * row_kv2);
    for (int b = 0; b < 2; ++b) rec(ctx->ev_slot_free[b], cs);
  }
  for (int b = 0; b < 2; ++b) {
    rec(ctx->ev_recv_used_c[b], cs);
    rec(ctx->ev_recv_used_d[b], cs);
    rec(ctx->ev_ohat_free[b], cs);
  }
  // host rows: chunk m's q, k, v rows -> the device mirrors (records ev_up[m])
  auto upload = [&](int64_t m) {
    const size_t bq = (size_t)c.c * c.Hq * d * eb, bkv = (size_t)c.c * c.Hkv * d * eb;
    h2d_io(ctx, (uint8_t*)q + (size_t)m * bq, (const uint8_t*)io->q + (size_t)m * bq, bq);
    h2d_io(ctx, (uint8_t*)k + (size_t)m * bkv, (const uint8_t*)io->k + (size_t)m * bkv, bkv);
    h2d_io(ctx, (uint8_t*)v + (size_t)m * bkv, (const uint8_t*)io->v + (size_t)m * bkv, bkv);
    rec(ctx->ev_up[(size_t)m], ctx->s_h2d);
  };
  // p == 1, host rows: upload chunk m, then offload its key/value rows (q_m stays in the caller's host rows, from
  // which the backward fetches it)
  auto stage_p1 = [&](int64_t m) {
    upload(m);
    wait(ctx->s_d2h, ctx->ev_up[(size_t)m]);
    const size_t wkv = (size_t)hkv * d * eb;
    d2h_2d(ctx, ctx->host + hl.kv(m, u), row_kv2, (const uint8_t*)k + (size_t)m * C * wkv, wkv, wkv, C);
    d2h_2d(ctx, ctx->host + hl.kv(m, u) + wkv, row_kv2, (const uint8_t*)v + (size_t)m * C * wkv, wkv, wkv, C);
    rec(ctx->ev_off[(size_t)m], ctx->s_d2h);
  };
  const bool io_p1 = io && p == 1;
  if (io_p1) stage_p1(0);
  // p == 1 with offload: the head-layout chunk IS the caller's rows; offload all chunks up front
  if (p == 1 && c.offload && !proj && !io) {
    for (int64_t m = 0; m < u; ++m) {
      if (!R.q(m)) d2h(ctx, ctx->host + hl.q(m), (const uint8_t*)q + (size_t)m * C * row_q, (size_t)C * row_q);
      if (!R.kv(m)) {
        const size_t wkv = (size_t)hkv * d * eb;
        d2h_2d(ctx, ctx->host + hl.kv(m, u), row_kv2, (const uint8_t*)k + (size_t)m * C * wkv, wkv, wkv, C);
        d2h_2d(ctx, ctx->host + hl.kv(m, u) + wkv, row_kv2, (const uint8_t*)v + (size_t)m * C * wkv, wkv, wkv, C);
      }
      rec(ctx->ev_off[m], ctx->s_d2h);
    }
  }
  // receive buffer of chunk m in the head layout (headbuf)
  auto recv_of = [&](int64_t m) -> uint8_t* {
    return !c.offload ? store + (size_t)m * C * hcomb * d * eb : R.slot[(size_t)m] >= 0 ? res_chunk(m)
                                                                                      : a2a_recv[m & 1];
  };
  // F3/F4/F5 for chunk m on the comm (and d2h) stream: projection or pack, all-to-all seq -> head, offload of q_m
  // and kv_m from the receive buffer.  Enqueued one chunk AHEAD of the compute (software pipeline): the exchange of
  // chunk m+1 is on the comm stream before the output exchange of chunk m, so it runs during chunk m's pairs and only
  // the first chunk's exchange (and the last chunk's output return) is exposed.
  auto exchange = [&](int64_t m) {
    const int b = (int)(m & 1);
    uint8_t* recv = recv_of(m);
    wait(ctx->s_comm, ctx->ev_recv_used_c[b]);
    wait(ctx->s_comm, ctx->ev_recv_used_d[b]);
    const size_t per_peer = (size_t)c.c * hcomb * d;
    if (proj) {
      // The projection GEMM runs on the compute stream, between the pairs of chunk m-1 (it is enqueued one chunk
      // ahead); its all-to-all still overlaps chunk m-1's pairs on the comm stream.  Measured at the bench shape: on
      // the comm stream, concurrently with the pair kernels, it only breaks their waves (block overhead 79 vs 68 ms).
      if (p == 1) wait(cs, ctx->ev_recv_used_d[b]);              // the offload of chunk m-2 has read this buffer
      else if (m >= 2) wait(cs, ctx->ev_a2a[m - 2]);             // chunk m-2's all-to-all has read the send buffer
      const uint8_t* xm = (const uint8_t*)pj->x + (size_t)m * c.c * pj->hidden * eb;
      gemm_xw(ctx, c.dtype, xm, pj->hidden, pj->w, ntot, p == 1 ? recv : a2a_send[b], ntot, c.c, pj->hidden, ntot, cs,
              &scat);
      rec(ctx->ev_tmp, cs);
      wait(ctx->s_comm, ctx->ev_tmp);
      if (ctx->saved_hidden_offload) {
        // the input hidden state chunk goes to the pinned store; the backward prefetches it for the projection
        // backward of chunk m ("the prefetching of the input hidden state h_0 will only be synced in the
        // projection backward")
        const size_t xb = (size_t)c.c * pj->hidden * eb;
        wait(ctx->s_d2h, ctx->ev_tmp);
        d2h(ctx, ctx->host_x + (size_t)m * xb, xm, xb);
        rec(ctx->ev_xoff[m], ctx->s_d2h);
      }
    } else {
      if (io) {
        upload(m);
        wait(ctx->s_comm, ctx->ev_up[(size_t)m]);
      }
      const uint8_t *qm = (const uint8_t*)q + (size_t)m * c.c * c.Hq * d * eb,
                    *km = (const uint8_t*)k + (size_t)m * c.c * c.Hkv * d * eb,
                    *vm = (const uint8_t*)v + (size_t)m * c.c * c.Hkv * d * eb;
      FPDT_CHECK_LAUNCH(launch_pack_seq2head(qm, c.c, c.Hq, d, p, eb, a2a_send[b], per_peer, (int64_t)hcomb * d, 0,
                                             ctx->s_comm));
      FPDT_CHECK_LAUNCH(launch_pack_seq2head(km, c.c, c.Hkv, d, p, eb, a2a_send[b], per_peer, (int64_t)hcomb * d, hq,
                                             ctx->s_comm));
      FPDT_CHECK_LAUNCH(launch_pack_seq2head(vm, c.c, c.Hkv, d, p, eb, a2a_send[b], per_peer, (int64_t)hcomb * d,
                                             hq + hkv, ctx->s_comm));
      ctx->stats.kernel_launches += 3;
    }
    if (p > 1) alltoall(ctx, a2a_send[b], recv, per_peer, c.dtype);
    rec(ctx->ev_a2a[m], ctx->s_comm);
    if (c.offload) {
      wait(ctx->s_d2h, ctx->ev_a2a[m]);
      const size_t pitch = (size_t)hcomb * d * eb;
      if (!R.q(m)) d2h_2d(ctx, ctx->host + hl.q(m), row_q, recv, pitch, row_q, C);
      if (!R.kv(m)) kvf.offload(m, recv + row_q, pitch, hl);
      rec(ctx->ev_off[m], ctx->s_d2h);
      rec(ctx->ev_recv_used_d[b], ctx->s_d2h);
      if (kvf.leader_mode) {  // the gather read the receive buffer on the comm stream
        rec(ctx->ev_tmp, ctx->s_comm);
        wait(ctx->s_d2h, ctx->ev_tmp);
        rec(ctx->ev_recv_used_d[b], ctx->s_d2h);
      }
    }
  };
  int fetch = 0;
  int64_t high = 0;
  // block sparsity (§5.6): skipped key chunks are neither fetched nor computed
  const std::vector<uint8_t>& plan = ctx->saved_plan;
  auto keep = [&](int64_t m, int64_t i) { return plan.empty() || plan[(size_t)(m * u + i)] != 0; };
  if (headbuf) exchange(0);
  for (int64_t m = 0; m < u; ++m) {
    if (headbuf && m + 1 < u) exchange(m + 1);
    if (io_p1 && m + 1 < u) stage_p1(m + 1);  // overlaps chunk m's pairs, ahead of their fetches on s_h2d
    int64_t last_kept = -1;  // the last earlier key chunk chunk m attends
    for (int64_t i = 0; i < m; ++i)
      if (keep(m, i)) last_kept = i;
    // ---- views of the current chunk's q, k, v in the head layout
    HeadView qv, kv, vv;
    int64_t q_row0, kv_row0_cur;
    if (!headbuf) {
      if (io_p1) wait(cs, ctx->ev_up[(size_t)m]);
      qv = {q, c.S, hq, 0};
      kv = {k, c.S, hkv, 0};
      vv = {v, c.S, hkv, 0};
      q_row0 = m * C;
      kv_row0_cur = m * C;
    } else {
      wait(cs, ctx->ev_a2a[m]);
      const uint8_t* base = c.offload ? recv_of(m) : store;
      qv = {base, c.offload ? C : c.S, hcomb, 0};
      kv = {base, c.offload ? C : c.S, hcomb, hq};
      vv = {base, c.offload ? C : c.S, hcomb, hq + hkv};
      q_row0 = c.offload ? 0 : m * C;
      kv_row0_cur = c.offload ? 0 : m * C;
    }
    FwdArgs a;
    a.q = qv;
    a.q_row0 = q_row0;
    a.n_q_rows = (int)C;
    a.q_pos0 = m * C;
    a.causal = 1;
    a.hq = hq;
    a.G = c.G;
    a.scale_log2 = sl2;
    a.o_acc = o_acc;
    a.lse_acc = lse_acc;
    if (p == 1) {
      a.o_out = (uint8_t*)o + (size_t)m * C * c.Hq * d * eb;
      a.o_ld = (int64_t)c.Hq * d;
      a.lse_user = lse ? lse + (size_t)m * C * c.Hq : nullptr;
      a.lse_user_ld = c.Hq;
    } else {
      wait(cs, ctx->ev_ohat_free[m & 1]);  // chunk m-2's output has left this buffer
      a.o_out = o_hat[m & 1];
      a.o_ld = (int64_t)hq * d;
    }
    a.lse_save = lse_save + m * C;
    a.lse_save_ld = c.S;
    a.o_resid = o_resid ? o_resid + (size_t)m * C * hq * d : nullptr;
    a.o_resid_ld = (int64_t)hq * d;
    if (!c.offload) {
      // resident: one launch over keys [0, (m+1)C)
      a.k = kv;
      a.v = vv;
      a.kv_row0 = 0;
      a.n_kv_rows = (int)((m + 1) * C);
      a.kv_pos0 = 0;
      a.has_prev = 0;
      a.is_final = 1;
      launch_fwd(ctx, c, a, cs);
    } else {
      // F6: diagonal block with the resident chunk
      a.k = kv;
      a.v = vv;
      a.kv_row0 = kv_row0_cur;
      a.n_kv_rows = (int)C;
      a.kv_pos0 = m * C;
      a.has_prev = 0;
      a.is_final = (last_kept < 0);
      launch_fwd(ctx, c, a, cs);
      // F7/F8: earlier chunks fetched from the host store, double-buffered
      for (int64_t i = 0; i < m; ++i) {
        if (!keep(m, i)) continue;
        a.kv_pos0 = i * C;
        a.has_prev = 1;
        a.is_final = (i == last_kept);
        if (R.kv(i)) {  // resident key/value chunk: no fetch
          if (!headbuf) {
            a.k = {k, c.S, hkv, 0};
            a.v = {v, c.S, hkv, 0};
            a.kv_row0 = i * C;
          } else {
            a.k = {res_chunk(i), C, hcomb, hq};
            a.v = {res_chunk(i), C, hcomb, hq + hkv};
            a.kv_row0 = 0;
          }
          launch_fwd(ctx, c, a, cs);
          continue;
        }
        const int sl = fetch & 1;
        kvf.fetch(i, kv_slot[sl], sl, ctx->ev_slot_free[sl], ctx->ev_slot_filled[sl], hl);
        high = std::max<int64_t>(high, std::min<int64_t>(fetch + 1, 2));  // slots 0/1 alternate
        wait(cs, ctx->ev_slot_filled[sl]);
        a.k = {kv_slot[sl], C, 2 * hkv, 0};
        a.v = {kv_slot[sl], C, 2 * hkv, hkv};
        a.kv_row0 = 0;
        a.kv_pos0 = i * C;
        a.has_prev = 1;
        a.is_final = (i == last_kept);
        launch_fwd(ctx, c, a, cs);
        rec(ctx->ev_slot_free[sl], cs);
        ++fetch;
      }
    }
    // chunk m's receive buffer (its q rows) is read by every pair (m, i) above: free it only after the last one
    if (headbuf) rec(ctx->ev_recv_used_c[m & 1], cs);
    // output projection of chunk m (fpdt_block_fwd with w_o): y_m = o_m w_o once O_m is final in the sequence layout
    const int64_t od = (int64_t)c.Hq * d;
    if (proj && pj->w_o && p == 1)
      gemm_xw(ctx, c.dtype, (const uint8_t*)o + (size_t)m * C * od * eb, od, pj->w_o, pj->hidden,
              (uint8_t*)pj->y + (size_t)m * C * pj->hidden * eb, pj->hidden, C, od, pj->hidden, cs);
    // host rows: chunk m's output rows (final now at p == 1, after the return exchange at p > 1) leave at once
    auto download_o = [&](cudaStream_t from) {
      rec(ctx->ev_tmp, from);
      wait(ctx->s_d2h, ctx->ev_tmp);
      const size_t bo = (size_t)c.c * od * eb;
      d2h_io(ctx, (uint8_t*)io->o + (size_t)m * bo, (const uint8_t*)o + (size_t)m * bo, bo);
      if (io->lse) {
        const size_t bl = (size_t)c.c * c.Hq * 4;
        d2h_io(ctx, (uint8_t*)io->lse + (size_t)m * bl, (const uint8_t*)lse + (size_t)m * bl, bl);
      }
    };
    if (io_p1) download_o(cs);
    if (p > 1) {
      // F10: all-to-all of O_m back to the sequence layout, then unpack into the caller's rows of slot m (on the comm
      // stream behind chunk m+1's exchange, so it overlaps chunk m+1's pairs)
      rec(ctx->ev_o_ready, cs);
      wait(ctx->s_comm, ctx->ev_o_ready);
      uint8_t* back = (uint8_t*)dev(ctx, B_BWD_RECV, (size_t)C * hq * d * eb);
      alltoall(ctx, o_hat[m & 1], back, (size_t)c.c * hq * d, c.dtype);
      rec(ctx->ev_ohat_free[m & 1], ctx->s_comm);
      FPDT_CHECK_LAUNCH(launch_unpack_head2seq(back, (int64_t)c.c * hq * d, (int64_t)hq * d, 0, c.c, c.Hq, d, p, eb,
                                               (uint8_t*)o + (size_t)m * c.c * c.Hq * d * eb, ctx->s_comm));
      ctx->stats.kernel_launches++;
      if (proj && pj->w_o)
        gemm_xw(ctx, c.dtype, (const uint8_t*)o + (size_t)m * c.c * od * eb, od, pj->w_o, pj->hidden,
                (uint8_t*)pj->y + (size_t)m * c.c * pj->hidden * eb, pj->hidden, c.c, od, pj->hidden, ctx->s_comm);
      if (lse) {
        // lse of this chunk: [hq][C] log2 -> [C][hq] natural, all-to-all (fp32), unpack to [c][Hq]
        float* lt = (float*)dev(ctx, B_LSE_T, (size_t)C * hq * 4);
        float* lr = (float*)dev(ctx, B_LSE_RECV, (size_t)C * hq * 4);
        FPDT_CHECK_LAUNCH(launch_lse_to_user(lse_save + m * C, c.S, C, hq, lt, hq, 0, ctx->s_comm));
        alltoall(ctx, lt, lr, (size_t)c.c * hq, FPDT_FP32);
        // unpack [p][c][hq] -> [c][Hq]: rank r's block holds heads [r hq, (r+1) hq) of every row
        for (int r = 0; r < p; ++r)
          FPDT_CHECK_CUDA(cudaMemcpy2DAsync(lse + (size_t)m * c.c * c.Hq + (size_t)r * hq, (size_t)c.Hq * 4,
                                            lr + (size_t)r * c.c * hq, (size_t)hq * 4, (size_t)hq * 4, c.c,
                                            cudaMemcpyDeviceToDevice, ctx->s_comm));
        ctx->stats.kernel_launches++;
      }
      if (io) download_o(ctx->s_comm);
    }
  }
  ctx->stats.fetch_slots_highwater = std::max(ctx->stats.fetch_slots_highwater, high);
  // the caller may reuse q/k/v after the call: every offload must have read them
  rec(ctx->ev_d2h_done, ctx->s_d2h);
  wait(cs, ctx->ev_d2h_done);
  rec(ctx->ev_comm_done, ctx->s_comm);
  wait(cs, ctx->ev_comm_done);
}

// ------------------------------------------------------------------------------------------ backward
// Arguments of the backward pair kernel for (query chunk i, key chunk j) of the offloaded schedule, both
// loop orders: q/dO/k/v views, the chunk's saved lse2 and D, its fp32 dq accumulator and dK/dV accumulators.  The
// caller sets the final-output pointers (dk_out, dv_out, kv_out_ld, kv_out_head0).
BwdArgs pair_bwd_args(const Config& c, const HeadView& qi, const HeadView& doi, const HeadView& kj, const HeadView& vj,
                      int64_t q_row0, int64_t kv_row0, int64_t i, int64_t j, const float* lse_save, const float* Dh,
                      float* dq_acc, float* dk_acc, float* dv_acc, bool acc_init, bool kv_final) {
  BwdArgs a;
  a.q = qi;
  a.dout = doi;
  a.k = kj;
  a.v = vj;
  a.q_row0 = q_row0;
  a.kv_row0 = kv_row0;
  a.n_q_rows = (int)c.C;
  a.n_kv_rows = (int)c.C;
  a.q_pos0 = i * c.C;
  a.kv_pos0 = j * c.C;
  a.causal = 1;
  a.hq = c.hq;
  a.G = c.G;
  a.scale = c.scale;
  a.scale_log2 = c.scale * 1.4426950408889634f;
  a.lse2 = lse_save + i * c.C;
  a.Dstat = Dh + i * c.C;
  a.stat_ld = c.S;
  a.dq_acc = dq_acc;  // head-major [hq][C][d]
  a.dq_head_stride = c.C * c.d;
  a.dk_acc = dk_acc;
  a.dv_acc = dv_acc;
  a.kv_acc_init = acc_init;
  a.kv_final = kv_final;
  return a;
}

// Q-outer chunk loop of the offloaded backward (fpdt_set_bwd_order FPDT_BWD_Q_OUTER).  The pair
// kernels and their arguments are the paper order's; only the loop nesting and what round-trips the host
// differ: for query chunk i (outer) fetch q_i, dO_i once and keep the fp32 dq_i accumulator on the device; for each
// key chunk j <= i (inner) fetch kv_j and the fp32 dK_j/dV_j partial (unless it is j's first pair), run pair (i, j),
// and write the partial back (unless i is the last query chunk attending j, where the kernel writes the final dK_j,
// dV_j).  After the inner loop dq_i is final.  p > 1: dq_i and (dk_j, dv_j) return to their owner ranks by separate
// all-to-alls, each as soon as it is final.
template <class Keep>
void backward_q_outer(fpdt_ctx* ctx, const Config& c, const Residency& R, const Keep& keep, const void* do_h,
                      int64_t do_rows, int do_heads, int do_head0, uint8_t* dores, void* dq, void* dk, void* dv,
                      cudaStream_t cs) {
  const int64_t C = c.C, u = c.u;
  const int d = c.d, hq = c.hq, hkv = c.hkv, eb = c.eb, p = c.p;
  const int hcomb = hq + 2 * hkv;
  const size_t row_q = (size_t)hq * d * eb, row_kv2 = (size_t)2 * hkv * d * eb;
  const size_t dkv_elems = (size_t)C * 2 * hkv * d, dkv_bytes = dkv_elems * 4;
  float* lse_save = (float*)ctx->bufs[B_LSESAVE].ptr;
  float* Dh = (float*)ctx->bufs[B_D].ptr;
  const HostLayout hl = host_layout(c);
  uint8_t* resstore = (uint8_t*)ctx->bufs[B_RESSTORE].ptr;
  auto res_chunk = [&](int64_t m) { return resstore + (size_t)R.slot[(size_t)m] * C * hcomb * d * eb; };

  std::vector<int64_t> last_i((size_t)u, 0);  // the last query chunk attending key chunk j
  for (int64_t j = 0; j < u; ++j)
    for (int64_t i = j; i < u; ++i)
      if (keep(i, j)) last_i[(size_t)j] = i;
  // pinned store of the dK/dV partials (grow-only, separate from the forward's store so the latter stays valid)
  if (R.rkv < u && u > 1) {
    const size_t need = (size_t)u * dkv_bytes;
    if (ctx->host_dkv_bytes < need) {
      if (ctx->host_dkv) {
        FPDT_CHECK_CUDA(cudaDeviceSynchronize());
        cudaFreeHost(ctx->host_dkv);
        ctx->host_dkv = nullptr;
        ctx->host_dkv_bytes = 0;
      }
      void* hp = nullptr;
      cudaError_t e = cudaHostAlloc(&hp, need, cudaHostAllocDefault);
      if (e != cudaSuccess) {
        cudaGetLastError();
        fail(FPDT_ERR_HOST_OOM, "pinned dK/dV partial store of " + std::to_string(need) + " bytes: " + cudaGetErrorString(e));
      }
      ctx->host_dkv = static_cast<uint8_t*>(hp);
      ctx->host_dkv_bytes = need;
      ctx->stats.host_dkv_bytes = (int64_t)need;
    }
  }
  ensure_events(ctx->ev_dkvoff, u);
  // The pairs (i, j) of one query chunk i share only dq_i, which the kernels reduce-add (order-free), so they run
  // two at a time on two compute streams: the second kernel's CTAs fill the SMs the first one's last wave leaves
  // idle (a full pair is 512 CTAs, 3.5 waves, when one kv head per rank is left: configs[4] at p = 8).
  // Key/value slots: two per stream (fetch of the next pair while the current one computes).
  // (bf16 only: the fp32 validation kernels add dQ with a plain read-modify-write, one owner per launch)
  const int ns = c.dtype == FPDT_BF16 ? ctx->qo_streams : 1, nslots = 2 * ns;
  cudaStream_t streams[2] = {cs, ctx->s_comp2};
  static const int kv_ids[4] = {B_KVSLOT0, B_KVSLOT1, B_KVSLOT2, B_KVSLOT3};
  static const int dkv_ids[4] = {B_DKVSLOT0, B_DKVSLOT1, B_DKVSLOT2, B_DKVSLOT3};
  uint8_t* kvs[4] = {};
  float* dkvs[4] = {};
  for (int b = 0; b < nslots; ++b) {
    kvs[b] = (uint8_t*)dev(ctx, kv_ids[b], (size_t)C * row_kv2);
    dkvs[b] = (float*)dev(ctx, dkv_ids[b], dkv_bytes);
  }
  float* dkvres = R.rkv > 0 ? (float*)dev(ctx, B_DKVRES, (size_t)R.rkv * dkv_bytes) : nullptr;
  uint8_t* qs[2] = {(uint8_t*)dev(ctx, B_QSLOT0, (size_t)C * row_q), (uint8_t*)dev(ctx, B_QSLOT1, (size_t)C * row_q)};
  uint8_t* dos[2] = {(uint8_t*)dev(ctx, B_DOSLOT0, (size_t)C * row_q), (uint8_t*)dev(ctx, B_DOSLOT1, (size_t)C * row_q)};
  float* dqs[2] = {(float*)dev(ctx, B_DQSLOT0, (size_t)C * hq * d * 4), (float*)dev(ctx, B_DQSLOT1, (size_t)C * hq * d * 4)};
  // p > 1 send / receive buffers: [C][hq][d] for dq, then two [C][2hkv][d] parts for (dk, dv), alternating between
  // final key chunks (ev_qo_send[0] = dq part free, [1 + r] = part r free)
  uint8_t *qsend = nullptr, *qrecv = nullptr;
  const size_t kvpart = (size_t)C * row_kv2;
  if (p > 1) {
    qsend = (uint8_t*)dev(ctx, B_QOSEND, (size_t)C * row_q + 2 * kvpart);
    qrecv = (uint8_t*)dev(ctx, B_QORECV, (size_t)C * row_q + 2 * kvpart);
    for (int b = 0; b < 3; ++b) rec(ctx->ev_qo_send[b], cs);
  }
  for (int b = 0; b < nslots; ++b) rec(ctx->ev_qo_free[b], cs);
  for (int b = 0; b < 2; ++b) rec(ctx->ev_q_free[b], cs);
  // B7 (p > 1): a final part goes back to the sequence layout of its owner ranks, after the kernel on `st`
  auto send_back = [&](cudaStream_t st, int part, int64_t chunk) {
    const bool is_dq = part == 0;
    const size_t off = is_dq ? 0 : (size_t)C * row_q + (size_t)(part - 1) * kvpart;
    const int heads = is_dq ? hq : 2 * hkv;
    rec(ctx->ev_o_ready, st);
    wait(ctx->s_comm, ctx->ev_o_ready);
    const int64_t pst = (int64_t)c.c * heads * d, rld = (int64_t)heads * d;
    alltoall(ctx, qsend + off, qrecv + off, (size_t)pst, c.dtype);
    if (is_dq) {
      FPDT_CHECK_LAUNCH(launch_unpack_head2seq(qrecv + off, pst, rld, 0, c.c, c.Hq, d, p, eb,
                                               (uint8_t*)dq + (size_t)chunk * c.c * c.Hq * d * eb, ctx->s_comm));
      ctx->stats.kernel_launches += 1;
    } else {
      FPDT_CHECK_LAUNCH(launch_unpack_head2seq(qrecv + off, pst, rld, 0, c.c, c.Hkv, d, p, eb,
                                               (uint8_t*)dk + (size_t)chunk * c.c * c.Hkv * d * eb, ctx->s_comm));
      FPDT_CHECK_LAUNCH(launch_unpack_head2seq(qrecv + off, pst, rld, hkv, c.c, c.Hkv, d, p, eb,
                                               (uint8_t*)dv + (size_t)chunk * c.c * c.Hkv * d * eb, ctx->s_comm));
      ctx->stats.kernel_launches += 2;
    }
    rec(ctx->ev_qo_send[part], ctx->s_comm);  // the part's send / receive buffers are free again
  };
  std::vector<char> dkv_started((size_t)u, 0);
  int kstep = 0, nfinal = 0;
  for (int64_t i = 0; i < u; ++i) {
    const int qsl = (int)(i & 1);
    HeadView qi, doi;
    int64_t q_row0 = 0;
    if (R.q(i)) {
      if (p == 1) {
        qi = {ctx->saved_q, c.S, hq, 0};
        doi = {do_h, do_rows, do_heads, do_head0};
        q_row0 = i * C;
      } else {
        qi = {res_chunk(i), C, hcomb, 0};
        doi = {dores + (size_t)R.qslot[(size_t)i] * C * 2 * hq * d * eb, C, 2 * hq, hq};
        wait(cs, ctx->ev_a2a[i]);  // its (O, dO) exchange and D_i
      }
    } else {
      // B4 (once per outer iteration): fetch q_i, dO_i
      wait(ctx->s_h2d, ctx->ev_q_free[qsl]);
      wait(ctx->s_h2d, ctx->ev_doff[i]);
      h2d(ctx, qs[qsl], ctx->host + hl.q(i), (size_t)C * row_q);
      h2d(ctx, dos[qsl], ctx->host + hl.dO(i, u), (size_t)C * row_q);
      rec(ctx->ev_q_filled[qsl], ctx->s_h2d);
      wait(cs, ctx->ev_q_filled[qsl]);
      qi = {qs[qsl], C, hq, 0};
      doi = {dos[qsl], C, hq, 0};
    }
    float* dqi = dqs[qsl];
    FPDT_CHECK_CUDA(cudaMemsetAsync(dqi, 0, (size_t)C * hq * d * 4, cs));
    if (ns > 1) {  // the second stream starts after everything enqueued on the caller's stream so far
      rec(ctx->ev_fork, cs);
      wait(ctx->s_comp2, ctx->ev_fork);
    }
    int n = 0;  // pair index within this query chunk
    for (int64_t j = 0; j <= i; ++j) {
      if (!keep(i, j)) continue;
      cudaStream_t st = streams[(n++) % ns];
      const bool first = !dkv_started[(size_t)j], fin = (i == last_i[(size_t)j]);
      HeadView kj, vj;
      int64_t kv_row0 = 0;
      float* acc = nullptr;
      int sl = -1;
      if (R.kv(j)) {
        if (p == 1) {
          kj = {ctx->saved_k, c.S, hkv, 0};
          vj = {ctx->saved_v, c.S, hkv, 0};
          kv_row0 = j * C;
        } else {
          kj = {res_chunk(j), C, hcomb, hq};
          vj = {res_chunk(j), C, hcomb, hq + hkv};
        }
        acc = dkvres + (size_t)j * dkv_elems;
      } else {
        // B3 per pair: kv_j and (after its first pair) the dK_j/dV_j partial
        sl = (kstep++) % nslots;
        wait(ctx->s_h2d, ctx->ev_qo_free[sl]);
        wait(ctx->s_h2d, ctx->ev_off[j]);
        h2d(ctx, kvs[sl], ctx->host + hl.kv(j, u), (size_t)C * row_kv2);
        if (!first) {
          wait(ctx->s_h2d, ctx->ev_dkvoff[j]);
          h2d(ctx, dkvs[sl], ctx->host_dkv + (size_t)j * dkv_bytes, dkv_bytes);
        }
        rec(ctx->ev_qo_filled[sl], ctx->s_h2d);
        wait(st, ctx->ev_qo_filled[sl]);
        kj = {kvs[sl], C, 2 * hkv, 0};
        vj = {kvs[sl], C, 2 * hkv, hkv};
        acc = dkvs[sl];
      }
      BwdArgs a = pair_bwd_args(c, qi, doi, kj, vj, q_row0, kv_row0, i, j, lse_save, Dh, dqi, acc,
                                acc + (size_t)C * hkv * d, first, fin);
      int part = 0;
      if (p == 1) {
        a.dk_out = (uint8_t*)dk + (size_t)j * C * c.Hkv * d * eb;
        a.dv_out = (uint8_t*)dv + (size_t)j * C * c.Hkv * d * eb;
        a.kv_out_ld = (int64_t)c.Hkv * d;
      } else {
        part = fin ? 1 + (nfinal++ & 1) : 0;
        uint8_t* kvsend = qsend + (size_t)C * row_q + (size_t)(part ? part - 1 : 0) * kvpart;
        if (fin) wait(st, ctx->ev_qo_send[part]);
        a.dk_out = kvsend;
        a.dv_out = kvsend + (size_t)hkv * d * eb;
        a.kv_out_ld = (int64_t)2 * hkv * d;
      }
      a.kv_out_head0 = 0;
      launch_bwd(ctx, c, a, st);
      dkv_started[(size_t)j] = 1;
      if (sl >= 0) {
        if (!fin) {
          // B6 (Q-outer): the dK_j/dV_j partial goes back to the host store
          rec(ctx->ev_qo_done[sl], st);
          wait(ctx->s_d2h, ctx->ev_qo_done[sl]);
          d2h(ctx, ctx->host_dkv + (size_t)j * dkv_bytes, dkvs[sl], dkv_bytes);
          rec(ctx->ev_dkvoff[j], ctx->s_d2h);
          rec(ctx->ev_qo_free[sl], ctx->s_d2h);
        } else {
          rec(ctx->ev_qo_free[sl], st);
        }
      }
      if (fin && p > 1) send_back(st, part, j);
    }
    if (ns > 1) {  // join: dq_i is complete when both streams' pairs are
      rec(ctx->ev_join, ctx->s_comp2);
      wait(cs, ctx->ev_join);
    }
    // dq_i is final after its last key chunk
    if (p > 1) wait(cs, ctx->ev_qo_send[0]);
    FPDT_CHECK_LAUNCH(launch_convert_out(dqi, C, hq, d, C * d, 1.f,
                                         p == 1 ? (uint8_t*)dq + (size_t)i * C * c.Hq * d * eb : qsend, c.dtype,
                                         p == 1 ? (int64_t)c.Hq * d : (int64_t)hq * d, 0, cs));
    ctx->stats.kernel_launches++;
    if (p > 1) send_back(cs, 0, i);
    if (!R.q(i)) rec(ctx->ev_q_free[qsl], cs);
  }
  if (p > 1) {
    rec(ctx->ev_comm_done, ctx->s_comm);
    wait(cs, ctx->ev_comm_done);
  }
}

void backward(fpdt_ctx* ctx, const Config& c, const void* o, const void* dout, void* dq, void* dk, void* dv,
              cudaStream_t cs, const Proj* pj = nullptr, const HostIO* io = nullptr) {
  Nvtx nv("fpdt:backward");
  const int64_t C = c.C, u = c.u;
  const int d = c.d, hq = c.hq, hkv = c.hkv, eb = c.eb, p = c.p;
  const int hcomb = hq + 2 * hkv;
  const size_t row_q = (size_t)hq * d * eb, row_kv2 = (size_t)2 * hkv * d * eb;
  const float sl2 = c.scale * 1.4426950408889634f;
  float* lse_save = (float*)ctx->bufs[B_LSESAVE].ptr;
  float* Dh = (float*)dev(ctx, B_D, (size_t)hq * c.S * 4);
  const __nv_bfloat16* o_resid = c.dtype == FPDT_BF16 ? (const __nv_bfloat16*)ctx->bufs[B_ORESID].ptr : nullptr;
  if (pj && pj->w_o) {
    // output projection backward (fpdt_block_bwd with w_o): `dout` is dy [s_local][hidden]; dO = dy w_o^T for every
    // local row and dw_o = o^T dy, before the attention backward needs dO
    const int64_t od = (int64_t)c.Hq * d;
    void* dO = dev(ctx, B_DOUT, (size_t)c.s_local * od * eb);
    gemm_dx(ctx, c.dtype, dout, pj->hidden, pj->w_o, pj->hidden, dO, od, c.s_local, od, pj->hidden, cs);
    gemm_dw(ctx, c.dtype, o, od, dout, pj->hidden, pj->dw_o, c.s_local, od, pj->hidden, false, cs);
    dout = dO;
  }
  ++ctx->call_seq;
  ensure_events(ctx->ev_doff, u);
  ensure_events(ctx->ev_dqoff, u);
  ensure_events(ctx->ev_a2a, u);
  if (io) ensure_events(ctx->ev_up, u);
  rec(ctx->ev_enter, cs);
  for (cudaStream_t s : {ctx->s_comm, ctx->s_h2d, ctx->s_d2h}) wait(s, ctx->ev_enter);
  HostLayout hl{};
  if (c.offload) hl = host_layout(c);
  const bool io_p1 = io && p == 1;
  if (io && io->upload_o) {
    // o is not the saved forward's output: its device mirror is stale
    h2d_io(ctx, const_cast<void*>(o), io->o, (size_t)c.s_local * c.Hq * d * eb);
    rec(ctx->ev_tmp, ctx->s_h2d);
    wait(cs, ctx->ev_tmp);
    wait(ctx->s_comm, ctx->ev_tmp);
  }
  const Residency R = make_residency(u, c.offload ? ctx->saved_res_kv : 0, c.offload ? ctx->saved_res_q : 0);
  uint8_t* resstore = (uint8_t*)ctx->bufs[B_RESSTORE].ptr;  // p > 1: the forward's resident head-layout chunks
  auto res_chunk = [&](int64_t m) { return resstore + (size_t)R.slot[(size_t)m] * C * hcomb * d * eb; };
  uint8_t* dores = (p > 1 && R.nq > 0) ? (uint8_t*)dev(ctx, B_DORES, (size_t)R.nq * C * 2 * hq * d * eb) : nullptr;
  float* dqres = R.nq > 0 ? (float*)dev(ctx, B_DQRES, (size_t)R.nq * C * hq * d * 4) : nullptr;
  // ---- B1/B2: D and the head-layout dO
  const void* do_h = dout;            // head-layout dO view base (p == 1: the caller's dO)
  int64_t do_rows = c.S;
  int do_heads = hq, do_head0 = 0;
  uint8_t* gathered = nullptr;        // p > 1: [S or C][2hq][d] gathered (O, dO)
  if (io_p1) {
    // host rows: D_i is formed at the first pair of query chunk i from its fetched dO_i (below); dO_i and q_i are
    // fetched from the caller's host rows
  } else if (p == 1) {
    FPDT_CHECK_LAUNCH(launch_bwd_preprocess_D(o, dout, c.dtype, c.S, hq, d, (int64_t)c.Hq * d, o_resid,
                                              (int64_t)hq * d, Dh, c.S, cs));
    ctx->stats.kernel_launches++;
    if (c.offload) {
      rec(ctx->ev_tmp, cs);
      wait(ctx->s_d2h, ctx->ev_tmp);
      for (int64_t m = 0; m < u; ++m) {
        if (!R.q(m)) d2h(ctx, ctx->host + hl.dO(m, u), (const uint8_t*)dout + (size_t)m * C * row_q, (size_t)C * row_q);
        rec(ctx->ev_doff[m], ctx->s_d2h);
      }
    }
  } else {
    // all-to-all of (O, dO) per chunk; D from the gathered head-layout chunks
    const size_t per_peer = (size_t)c.c * 2 * hq * d;
    uint8_t* send = (uint8_t*)dev(ctx, B_A2A_SEND0, (size_t)C * 2 * hq * d * eb);
    gathered = (uint8_t*)dev(ctx, B_DOSTORE, (size_t)(c.offload ? 2 * C : c.S) * 2 * hq * d * eb);
    for (int64_t m = 0; m < u; ++m) {
      // query-side resident chunks (a suffix of m) keep their (O, dO) chunk; the others share a double buffer
      uint8_t* recv = !c.offload ? gathered + (size_t)m * C * 2 * hq * d * eb
                      : R.q(m)   ? dores + (size_t)R.qslot[(size_t)m] * C * 2 * hq * d * eb
                                 : gathered + (size_t)(m & 1) * C * 2 * hq * d * eb;
      if (c.offload && !R.q(m) && m >= 2) wait(ctx->s_comm, ctx->ev_doff[m - 2]);
      if (io) {
        const size_t bo = (size_t)c.c * c.Hq * d * eb;
        h2d_io(ctx, (uint8_t*)dout + (size_t)m * bo, (const uint8_t*)io->dout + (size_t)m * bo, bo);
        rec(ctx->ev_up[(size_t)m], ctx->s_h2d);
        wait(ctx->s_comm, ctx->ev_up[(size_t)m]);
      }
      FPDT_CHECK_LAUNCH(launch_pack_seq2head((const uint8_t*)o + (size_t)m * c.c * c.Hq * d * eb, c.c, c.Hq, d, p, eb,
                                             send, per_peer, (int64_t)2 * hq * d, 0, ctx->s_comm));
      FPDT_CHECK_LAUNCH(launch_pack_seq2head((const uint8_t*)dout + (size_t)m * c.c * c.Hq * d * eb, c.c, c.Hq, d, p,
                                             eb, send, per_peer, (int64_t)2 * hq * d, hq, ctx->s_comm));
      ctx->stats.kernel_launches += 2;
      alltoall(ctx, send, recv, per_peer, c.dtype);
      // D for rows [mC, (m+1)C) in the head layout (o = heads [0,hq), dO = heads [hq,2hq) of recv)
      FPDT_CHECK_LAUNCH(launch_bwd_preprocess_D(recv, recv + row_q, c.dtype, C, hq, d, (int64_t)2 * hq * d,
                                                o_resid ? o_resid + (size_t)m * C * hq * d : nullptr,
                                                (int64_t)hq * d, Dh + m * C, c.S, ctx->s_comm));
      ctx->stats.kernel_launches++;
      rec(ctx->ev_a2a[m], ctx->s_comm);
      if (c.offload && !R.q(m)) {
        wait(ctx->s_d2h, ctx->ev_a2a[m]);
        d2h_2d(ctx, ctx->host + hl.dO(m, u), row_q, recv + row_q, (size_t)2 * hq * d * eb, row_q, C);
        rec(ctx->ev_doff[m], ctx->s_d2h);
      }
    }
    // The chunk loop below waits for chunk i's exchange only where it reads chunk i (offloaded chunks through the
    // dO_i offload -> fetch chain, resident ones by ev_a2a[i]), so chunk 0's pairs start while the later (O, dO)
    // exchanges still run on the comm stream.  The resident-mode launches span many chunks: they wait for all.
    if (!c.offload) {
      rec(ctx->ev_comm_done, ctx->s_comm);
      wait(cs, ctx->ev_comm_done);
    }
    do_h = gathered;
    do_rows = c.S;
    do_heads = 2 * hq;
    do_head0 = hq;
  }

  float* dk_acc = (float*)dev(ctx, B_DKACC, (size_t)C * hkv * d * 4);
  float* dv_acc = (float*)dev(ctx, B_DVACC, (size_t)C * hkv * d * 4);
  // B7 buffers (p > 1), double-buffered by the outer index j: outer iteration j+1 fills one while chunk j's final
  // dq, dk, dv leave through the other
  uint8_t *bsend2[2] = {nullptr, nullptr}, *brecv2[2] = {nullptr, nullptr};
  for (int b = 0; b < 2; ++b) rec(ctx->ev_bsend_free[b], cs);
  if (p > 1)
    for (int b = 0; b < 2; ++b) {
      bsend2[b] = (uint8_t*)dev(ctx, b ? B_BWD_SEND1 : B_BWD_SEND, (size_t)C * hcomb * d * eb);
      brecv2[b] = (uint8_t*)dev(ctx, b ? B_BWD_RECV1 : B_BWD_RECV, (size_t)C * hcomb * d * eb);
    }
  uint8_t* bsend = nullptr;  // the send buffer of the current outer iteration

  // fused projection (fpdt_block_bwd): chunk j's final dq, dk, dv land in a chunk buffer of sequence rows
  // [c][Hq + 2Hkv][d] (double-buffered by j), from which the projection backward forms dx_j and adds x_j^T dqkv_j
  // to dW as soon as the chunk is final ("dq_0, dk_0, dv_0 are used to compute the gradient of the input
  // hidden state")
  const bool proj = pj != nullptr;
  const int64_t ntot = (int64_t)(c.Hq + 2 * c.Hkv) * d;
  uint8_t* dqkv_buf[2] = {nullptr, nullptr};
  if (proj)
    for (int b = 0; b < 2; ++b) dqkv_buf[b] = (uint8_t*)dev(ctx, B_PROJ1 + b, (size_t)c.c * ntot * eb);
  int proj_chunks_done = 0;
  // hidden-state chunks (x == nullptr: offloaded by the forward, fpdt_set_hidden_offload): prefetched into a double
  // buffer at the start of outer iteration j, synced only by the projection backward of chunk j
  const bool x_from_host = proj && pj->x == nullptr;
  const size_t xbytes = proj ? (size_t)c.c * pj->hidden * eb : 0;
  uint8_t* xslot[2] = {nullptr, nullptr};
  if (x_from_host)
    for (int b = 0; b < 2; ++b) {
      xslot[b] = (uint8_t*)dev(ctx, b ? B_X1 : B_X0, xbytes);
      rec(ctx->ev_x_free[b], cs);
    }
  auto prefetch_x = [&](int64_t j) {
    if (!x_from_host) return;
    wait(ctx->s_h2d, ctx->ev_x_free[j & 1]);
    wait(ctx->s_h2d, ctx->ev_xoff[j]);
    h2d(ctx, xslot[j & 1], ctx->host_x + (size_t)j * xbytes, xbytes);
    rec(ctx->ev_x_filled[j & 1], ctx->s_h2d);
  };
  auto proj_bwd = [&](int64_t j, cudaStream_t st) {
    if (!proj) return;
    const uint8_t* dy = dqkv_buf[j & 1];
    const size_t xoff = (size_t)j * c.c * pj->hidden * eb;
    gemm_dx(ctx, c.dtype, dy, ntot, pj->w, ntot, (uint8_t*)pj->dx + xoff, pj->hidden, c.c, pj->hidden, ntot, st);
    const uint8_t* xj = (const uint8_t*)pj->x + xoff;
    if (x_from_host) {
      wait(st, ctx->ev_x_filled[j & 1]);
      xj = xslot[j & 1];
    }
    gemm_dw(ctx, c.dtype, xj, pj->hidden, dy, ntot, pj->dw, c.c, pj->hidden, ntot, proj_chunks_done++ > 0, st);
    if (x_from_host) rec(ctx->ev_x_free[j & 1], st);
  };
  // B6: dq_j final (fp32, already scaled) -> the caller's rows (p == 1) or the head-side send buffer (p > 1)
  // dq_final: head-major fp32 rows of chunk j, heads head_stride elements apart
  auto emit_dq = [&](int64_t j, const float* dq_final, int64_t head_stride) {
    if (p == 1 && proj)
      FPDT_CHECK_LAUNCH(launch_convert_out(dq_final, C, hq, d, head_stride, 1.f, dqkv_buf[j & 1], c.dtype, ntot, 0,
                                           cs));
    else if (p == 1)
      FPDT_CHECK_LAUNCH(launch_convert_out(dq_final, C, hq, d, head_stride, 1.f,
                                           (uint8_t*)dq + (size_t)j * C * c.Hq * d * eb, c.dtype, (int64_t)c.Hq * d,
                                           0, cs));
    else
      FPDT_CHECK_LAUNCH(launch_convert_out(dq_final, C, hq, d, head_stride, 1.f, bsend, c.dtype, (int64_t)hcomb * d,
                                           0, cs));
    ctx->stats.kernel_launches++;
  };
  // B7: after outer iteration j, dq_j, dk_j, dv_j (in bsend) go back to their owner ranks (p > 1)
  auto send_back = [&](int64_t j) {
    if (p == 1) {
      // the projection backward of chunk j on the compute stream, right after its last pair (concurrent with the
      // pair kernels on another stream it only breaks their waves; at p > 1 it follows the return all-to-all below)
      if (!proj) return;
      proj_bwd(j, cs);
      rec(ctx->ev_bsend_free[j & 1], cs);
      return;
    }
    rec(ctx->ev_o_ready, cs);
    wait(ctx->s_comm, ctx->ev_o_ready);
    uint8_t* brecv = brecv2[j & 1];
    alltoall(ctx, bsend, brecv, (size_t)c.c * hcomb * d, c.dtype);
    const int64_t pst = (int64_t)c.c * hcomb * d, rld = (int64_t)hcomb * d;
    uint8_t *dqj = (uint8_t*)dq + (size_t)j * c.c * c.Hq * d * eb, *dkj = (uint8_t*)dk + (size_t)j * c.c * c.Hkv * d * eb,
            *dvj = (uint8_t*)dv + (size_t)j * c.c * c.Hkv * d * eb;
    int64_t dst_ld = 0;
    if (proj) {
      dqj = dqkv_buf[j & 1];
      dkj = dqj + (size_t)c.Hq * d * eb;
      dvj = dqj + (size_t)(c.Hq + c.Hkv) * d * eb;
      dst_ld = ntot;
    }
    FPDT_CHECK_LAUNCH(launch_unpack_head2seq(brecv, pst, rld, 0, c.c, c.Hq, d, p, eb, dqj, ctx->s_comm, dst_ld));
    FPDT_CHECK_LAUNCH(launch_unpack_head2seq(brecv, pst, rld, hq, c.c, c.Hkv, d, p, eb, dkj, ctx->s_comm, dst_ld));
    FPDT_CHECK_LAUNCH(launch_unpack_head2seq(brecv, pst, rld, hq + hkv, c.c, c.Hkv, d, p, eb, dvj, ctx->s_comm,
                                             dst_ld));
    ctx->stats.kernel_launches += 3;
    proj_bwd(j, ctx->s_comm);  // projection backward of chunk j overlaps the next outer iteration
    rec(ctx->ev_bsend_free[j & 1], ctx->s_comm);  // bsend / brecv [j & 1] reusable by outer iteration j + 2
  };
  auto set_kv_out = [&](BwdArgs& a, int64_t j) {
    if (p == 1 && proj) {
      a.dk_out = dqkv_buf[j & 1];
      a.dv_out = dqkv_buf[j & 1] + (size_t)hkv * d * eb;
      a.kv_out_ld = ntot;
      a.kv_out_head0 = hq;  // as the p > 1 send buffer: dk heads [hq, hq + hkv), dv pre-offset by hkv heads
    } else if (p == 1) {
      a.dk_out = (uint8_t*)dk + (size_t)j * C * c.Hkv * d * eb;
      a.dv_out = (uint8_t*)dv + (size_t)j * C * c.Hkv * d * eb;
      a.kv_out_ld = (int64_t)c.Hkv * d;
      a.kv_out_head0 = 0;
    } else {
      a.dk_out = bsend;
      a.dv_out = bsend + (size_t)hkv * d * eb;
      a.kv_out_ld = (int64_t)hcomb * d;
      a.kv_out_head0 = hq;  // heads [hq, hq+hkv) for dk; the dv pointer is pre-offset by hkv heads
    }
  };

  if (!c.offload) {
    ctx->stats.bwd_order = FPDT_BWD_KV_OUTER;
    // resident: one launch per outer j over the query range [jC, S)
    float* dq_dev = (float*)dev(ctx, B_DQDEV, (size_t)c.S * hq * d * 4);
    FPDT_CHECK_CUDA(cudaMemsetAsync(dq_dev, 0, (size_t)c.S * hq * d * 4, cs));
    HeadView qv, kv, vv;
    if (p == 1) {
      qv = {ctx->saved_q, c.S, hq, 0};
      kv = {ctx->saved_k, c.S, hkv, 0};
      vv = {ctx->saved_v, c.S, hkv, 0};
    } else {
      uint8_t* store = (uint8_t*)ctx->bufs[B_STORE].ptr;
      qv = {store, c.S, hcomb, 0};
      kv = {store, c.S, hcomb, hq};
      vv = {store, c.S, hcomb, hq + hkv};
    }
    for (int64_t j = 0; j < u; ++j) {
      if (p > 1 || proj) {
        if (p > 1) bsend = bsend2[j & 1];
        wait(cs, ctx->ev_bsend_free[j & 1]);
      }
      BwdArgs a;
      a.q = qv; a.k = kv; a.v = vv;
      a.dout = {do_h, do_rows, do_heads, do_head0};
      a.q_row0 = j * C;
      a.kv_row0 = j * C;
      a.n_q_rows = (int)(c.S - j * C);
      a.n_kv_rows = (int)C;
      a.q_pos0 = j * C;
      a.kv_pos0 = j * C;
      a.causal = 1;
      a.hq = hq;
      a.G = c.G;
      a.scale = c.scale;
      a.scale_log2 = sl2;
      a.lse2 = lse_save + j * C;
      a.Dstat = Dh + j * C;
      a.stat_ld = c.S;
      a.dq_acc = dq_dev + (size_t)j * C * d;  // head-major [hq][S][d]
      a.dq_head_stride = c.S * d;
      a.dk_acc = dk_acc;
      a.dv_acc = dv_acc;
      a.kv_acc_init = 1;
      a.kv_final = 1;
      set_kv_out(a, j);
      launch_bwd(ctx, c, a, cs);
      emit_dq(j, dq_dev + (size_t)j * C * d, c.S * d);
      send_back(j);
    }
  } else {
    const std::vector<uint8_t>& plan = ctx->saved_plan;
    auto keep = [&](int64_t i, int64_t j) { return i == j || plan.empty() || plan[(size_t)(i * u + j)] != 0; };
    int order = ctx->bwd_order;
    if (order == FPDT_BWD_AUTO)
      order = bwd_host_bytes(FPDT_BWD_Q_OUTER, c, R.rkv, R.rq, keep) < bwd_host_bytes(FPDT_BWD_KV_OUTER, c, R.rkv, R.rq, keep)
                  ? FPDT_BWD_Q_OUTER
                  : FPDT_BWD_KV_OUTER;
    if (proj) order = FPDT_BWD_KV_OUTER;  // the fused projection backward runs per final chunk j
    if (io) order = FPDT_BWD_KV_OUTER;    // host rows: chunk j's gradients leave after outer iteration j
    KvFetch kvf(ctx, c, ctx->saved_fetch);
    if (kvf.leader_mode) order = FPDT_BWD_KV_OUTER;  // strategy B is implemented for the paper's loop order
    kvf.init_events(cs);
    ctx->stats.bwd_order = order;
    if (order == FPDT_BWD_Q_OUTER && !proj) {
      backward_q_outer(ctx, c, R, keep, do_h, do_rows, do_heads, do_head0, dores, dq, dk, dv, cs);
    } else {
    uint8_t* kvs[2] = {(uint8_t*)dev(ctx, B_KVSLOT0, (size_t)C * row_kv2), (uint8_t*)dev(ctx, B_KVSLOT1, (size_t)C * row_kv2)};
    uint8_t* qs[2] = {(uint8_t*)dev(ctx, B_QSLOT0, (size_t)C * row_q), (uint8_t*)dev(ctx, B_QSLOT1, (size_t)C * row_q)};
    uint8_t* dos[2] = {(uint8_t*)dev(ctx, B_DOSLOT0, (size_t)C * row_q), (uint8_t*)dev(ctx, B_DOSLOT1, (size_t)C * row_q)};
    float* dqs[2] = {(float*)dev(ctx, B_DQSLOT0, (size_t)C * hq * d * 4), (float*)dev(ctx, B_DQSLOT1, (size_t)C * hq * d * 4)};
    for (int b = 0; b < 2; ++b) {
      rec(ctx->ev_kv_free[b], cs);
      rec(ctx->ev_q_free[b], cs);
    }
    int step = 0;
    std::vector<char> dq_started((size_t)u, 0);  // chunk i's dq partial already holds contributions (host store)
    std::vector<char> d_done((size_t)u, 0);      // host rows, p == 1: D_i formed
    // host-side source of q_i / dO_i: the store, or (host rows, p == 1) the caller's rows in the same layout
    auto src_q = [&](int64_t i) -> const uint8_t* {
      return io_p1 ? (const uint8_t*)io->q + (size_t)i * C * row_q : ctx->host + hl.q(i);
    };
    auto src_do = [&](int64_t i) -> const uint8_t* {
      return io_p1 ? (const uint8_t*)io->dout + (size_t)i * C * row_q : ctx->host + hl.dO(i, u);
    };
    for (int64_t j = 0; j < u; ++j) {
      const int ks = (int)(j & 1);
      if (p > 1 || proj) {
        if (p > 1) bsend = bsend2[j & 1];
        wait(cs, ctx->ev_bsend_free[j & 1]);  // chunk j-2's final gradients have left this buffer
      }
      int64_t last_i = j;  // the last query chunk that attends key chunk j
      for (int64_t i = j; i < u; ++i)
        if (keep(i, j)) last_i = i;
      prefetch_x(j);
      // B3: fetch kv_j (resident key/value chunks are read in place)
      HeadView kj, vj;
      int64_t kv_row0 = 0;
      if (R.kv(j)) {
        if (p == 1) {
          kj = {ctx->saved_k, c.S, hkv, 0};
          vj = {ctx->saved_v, c.S, hkv, 0};
          kv_row0 = j * C;
        } else {
          kj = {res_chunk(j), C, hcomb, hq};
          vj = {res_chunk(j), C, hcomb, hq + hkv};
        }
      } else {
        kvf.fetch(j, kvs[ks], ks, ctx->ev_kv_free[ks], ctx->ev_kv_filled[ks], hl);
        wait(cs, ctx->ev_kv_filled[ks]);
        kj = {kvs[ks], C, 2 * hkv, 0};
        vj = {kvs[ks], C, 2 * hkv, hkv};
      }
      for (int64_t i = j; i < u; ++i) {
        if (!keep(i, j)) continue;
        const bool qres = R.q(i);
        const int sl = qres ? 0 : (step++) & 1;
        HeadView qi, doi;
        int64_t q_row0 = 0;
        float* dqi = nullptr;
        if (qres) {
          // query-side resident chunk: q_i, dO_i in place, its dq partial accumulates in device memory
          if (p == 1) {
            qi = {ctx->saved_q, c.S, hq, 0};
            doi = {do_h, do_rows, do_heads, do_head0};
            q_row0 = i * C;
          } else {
            qi = {res_chunk(i), C, hcomb, 0};
            doi = {dores + (size_t)R.qslot[(size_t)i] * C * 2 * hq * d * eb, C, 2 * hq, hq};
          }
          dqi = dqres + (size_t)R.qslot[(size_t)i] * C * hq * d;
          if (p > 1) wait(cs, ctx->ev_a2a[i]);  // its (O, dO) exchange and D_i (a no-op after the first pair)
          if (!dq_started[i]) FPDT_CHECK_CUDA(cudaMemsetAsync(dqi, 0, (size_t)C * hq * d * 4, cs));
        } else {
          // B4: fetch q_i, dO_i and (when it already holds contributions) the dq partial of chunk i
          wait(ctx->s_h2d, ctx->ev_q_free[sl]);
          if (!io_p1) wait(ctx->s_h2d, ctx->ev_doff[i]);
          h2d(ctx, qs[sl], src_q(i), (size_t)C * row_q);
          h2d(ctx, dos[sl], src_do(i), (size_t)C * row_q);
          if (dq_started[i]) {
            wait(ctx->s_h2d, ctx->ev_dqoff[i]);
            h2d(ctx, dqs[sl], ctx->host + hl.dq(i, u), (size_t)C * hq * d * 4);
          }
          rec(ctx->ev_q_filled[sl], ctx->s_h2d);
          wait(cs, ctx->ev_q_filled[sl]);
          if (!dq_started[i]) FPDT_CHECK_CUDA(cudaMemsetAsync(dqs[sl], 0, (size_t)C * hq * d * 4, cs));
          if (io_p1 && !d_done[i]) {
            FPDT_CHECK_LAUNCH(launch_bwd_preprocess_D((const uint8_t*)o + (size_t)i * C * row_q, dos[sl], c.dtype, C,
                                                      hq, d, (int64_t)hq * d,
                                                      o_resid ? o_resid + (size_t)i * C * hq * d : nullptr,
                                                      (int64_t)hq * d, Dh + i * C, c.S, cs));
            ctx->stats.kernel_launches++;
            d_done[i] = 1;
          }
          qi = {qs[sl], C, hq, 0};
          doi = {dos[sl], C, hq, 0};
          dqi = dqs[sl];
        }
        BwdArgs a = pair_bwd_args(c, qi, doi, kj, vj, q_row0, kv_row0, i, j, lse_save, Dh, dqi, dk_acc, dv_acc,
                                  i == j, i == last_i);
        set_kv_out(a, j);
        launch_bwd(ctx, c, a, cs);
        if (qres) {
          dq_started[i] = 1;
          if (i == j) emit_dq(j, dqi, C * d);  // B6: final
        } else if (i == j) {
          // B6: dq_j is final after its last contribution (inner iteration i == j)
          emit_dq(j, dqs[sl], C * d);
          rec(ctx->ev_q_free[sl], cs);
        } else {
          // B6: write the dq partial back to the host store
          rec(ctx->ev_dq_ready[sl], cs);
          wait(ctx->s_d2h, ctx->ev_dq_ready[sl]);
          d2h(ctx, ctx->host + hl.dq(i, u), dqs[sl], (size_t)C * hq * d * 4);
          rec(ctx->ev_dqoff[i], ctx->s_d2h);
          dq_started[i] = 1;
          rec(ctx->ev_q_free[sl], ctx->s_d2h);
        }
      }
      send_back(j);  // dk_j, dv_j are final after the last inner iteration
      rec(ctx->ev_kv_free[ks], cs);
      if (io) {
        // host rows: chunk j's dq, dk, dv rows are final (p == 1: on the compute stream; p > 1: unpacked on the comm
        // stream by send_back)
        rec(ctx->ev_tmp, p == 1 ? cs : ctx->s_comm);
        wait(ctx->s_d2h, ctx->ev_tmp);
        const size_t bq = (size_t)c.c * c.Hq * d * eb, bkv = (size_t)c.c * c.Hkv * d * eb;
        d2h_io(ctx, (uint8_t*)io->dq + (size_t)j * bq, (const uint8_t*)dq + (size_t)j * bq, bq);
        d2h_io(ctx, (uint8_t*)io->dk + (size_t)j * bkv, (const uint8_t*)dk + (size_t)j * bkv, bkv);
        d2h_io(ctx, (uint8_t*)io->dv + (size_t)j * bkv, (const uint8_t*)dv + (size_t)j * bkv, bkv);
      }
    }
    }
  }
  rec(ctx->ev_d2h_done, ctx->s_d2h);
  wait(cs, ctx->ev_d2h_done);
  rec(ctx->ev_h2d_done, ctx->s_h2d);
  wait(cs, ctx->ev_h2d_done);
  rec(ctx->ev_comm_done, ctx->s_comm);  // the last chunk's gradients are in the caller's tensors
  wait(cs, ctx->ev_comm_done);
}

}  // namespace

// ============================================================================================ C ABI

namespace {
int run(const std::function<void()>& f) {
  try {
    f();
    return FPDT_OK;
  } catch (const Fail& e) {
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return FPDT_ERR_CUDA;
  }
}
}  // namespace

extern "C" {

const char* fpdt_last_error(void) { return g_last_error.c_str(); }

int64_t fpdt_global_token(int64_t local_t, int64_t chunk_size, int world_size, int rank) {
  const int64_t c = chunk_size / world_size;
  return ((local_t / c) * world_size + rank) * c + (local_t % c);
}

int fpdt_get_unique_id(unsigned char id[128]) {
  return run([&] {
    if (!id) fail(FPDT_ERR_ARG, "null id");
    ncclUniqueId u;
    FPDT_CHECK_NCCL(ncclGetUniqueId(&u));
    static_assert(sizeof(u.internal) == 128, "nccl id size");
    std::memcpy(id, u.internal, 128);
  });
}

namespace {
fpdt_ctx* create_ctx(int world_size, int rank, const unsigned char* nccl_id, fpdt_group* group, int device,
                     size_t host_arena_bytes) {
    FPDT_CHECK_CUDA(cudaSetDevice(device));
    fpdt_ctx* ctx = new fpdt_ctx();
    try {
    ctx->group = group;
    ctx->p = world_size;
    ctx->rank = rank;
    ctx->device = device;
    int lo = 0, hi = 0;
    FPDT_CHECK_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    FPDT_CHECK_CUDA(cudaStreamCreateWithPriority(&ctx->s_comm, cudaStreamNonBlocking, hi));
    FPDT_CHECK_CUDA(cudaStreamCreateWithFlags(&ctx->s_h2d, cudaStreamNonBlocking));
    FPDT_CHECK_CUDA(cudaStreamCreateWithFlags(&ctx->s_d2h, cudaStreamNonBlocking));
    FPDT_CHECK_CUDA(cudaStreamCreateWithFlags(&ctx->s_comp2, cudaStreamNonBlocking));
    if (const char* e = getenv("FPDT_BWD_QO_STREAMS")) ctx->qo_streams = atoi(e) == 1 ? 1 : 2;
    if (const char* e = getenv("FPDT_STRESS_NS")) ctx->stress_ns = (uint32_t)std::max(0, atoi(e));
    if (const char* e = getenv("FPDT_STRESS_SEED")) ctx->stress_state ^= (uint64_t)atoll(e) * 0xD1B54A32D192ED03ull;
    for (int b = 0; b < 4; ++b)
      for (cudaEvent_t* e : {&ctx->ev_qo_free[b], &ctx->ev_qo_filled[b], &ctx->ev_qo_done[b]})
        FPDT_CHECK_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    for (int b = 0; b < 3; ++b) FPDT_CHECK_CUDA(cudaEventCreateWithFlags(&ctx->ev_qo_send[b], cudaEventDisableTiming));
    FPDT_CHECK_CUDA(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
    FPDT_CHECK_CUDA(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
    cudaEvent_t* evs[] = {&ctx->ev_enter, &ctx->ev_o_ready, &ctx->ev_comm_done, &ctx->ev_d2h_done, &ctx->ev_h2d_done,
                          &ctx->ev_tmp, &ctx->ev_kvg_free};
    for (auto e : evs) FPDT_CHECK_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    for (int b = 0; b < 2; ++b) {
      cudaEvent_t* pe[] = {&ctx->ev_slot_free[b], &ctx->ev_slot_filled[b], &ctx->ev_q_free[b], &ctx->ev_q_filled[b],
                           &ctx->ev_dq_ready[b], &ctx->ev_kv_free[b], &ctx->ev_kv_filled[b], &ctx->ev_recv_used_c[b],
                           &ctx->ev_recv_used_d[b], &ctx->ev_ohat_free[b], &ctx->ev_bsend_free[b],
                           &ctx->ev_kvall_free[b], &ctx->ev_kvall_filled[b], &ctx->ev_x_free[b],
                           &ctx->ev_x_filled[b]};
      for (auto e : pe) FPDT_CHECK_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    }
    if (const char* e = getenv("FPDT_NCCL_TIMEOUT_S")) ctx->nccl_timeout_s = std::max(1.0, atof(e));
    if (world_size > 1 && !group) {
      ncclUniqueId u;
      std::memcpy(u.internal, nccl_id, 128);
      ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
      cfg.blocking = 0;
      const ncclResult_t r = ncclCommInitRankConfig(&ctx->comm, world_size, u, rank, &cfg);
      if (r != ncclSuccess && r != ncclInProgress) {
        g_last_error = std::string("ncclCommInitRankConfig: ") + ncclGetErrorString(r);
        throw Fail{FPDT_ERR_NCCL};
      }
      try {
        nccl_settle(ctx->comm, ctx->nccl_timeout_s, "ncclCommInitRank");
      } catch (...) {
        ncclCommAbort(ctx->comm);
        ctx->comm = nullptr;
        throw;
      }
    }
    if (host_arena_bytes) ensure_host(ctx, host_arena_bytes);
    } catch (...) {
      // release what was created (streams, events, communicator) and keep the failure's status and message
      const std::string msg = g_last_error;
      fpdt_ctx_destroy(ctx);
      g_last_error = msg;
      throw;
    }
    return ctx;
}
}  // namespace

int fpdt_ctx_create(int world_size, int rank, const unsigned char* nccl_id, int device, size_t host_arena_bytes,
                    fpdt_ctx** out) {
  return run([&] {
    if (!out || world_size < 1 || rank < 0 || rank >= world_size) fail(FPDT_ERR_ARG, "bad world_size/rank/out");
    if (world_size > 1 && !nccl_id) fail(FPDT_ERR_ARG, "nccl_id required for world_size > 1");
    *out = create_ctx(world_size, rank, nccl_id, nullptr, device, host_arena_bytes);
  });
}

int fpdt_group_create(int world_size, int device, fpdt_group** out) {
  return run([&] {
    if (!out || world_size < 1) fail(FPDT_ERR_ARG, "bad world_size/out");
    FPDT_CHECK_CUDA(cudaSetDevice(device));
    fpdt_group* g = new fpdt_group();
    g->p = world_size;
    g->send.assign(world_size, nullptr);
    g->send_to.assign(world_size, std::vector<const void*>(world_size, nullptr));
    g->arg_hash.assign(world_size, 0);
    g->ev_sent.assign(world_size, nullptr);
    g->ev_read.assign(world_size, nullptr);
    for (int r = 0; r < world_size; ++r) {
      FPDT_CHECK_CUDA(cudaEventCreateWithFlags(&g->ev_sent[r], cudaEventDisableTiming));
      FPDT_CHECK_CUDA(cudaEventCreateWithFlags(&g->ev_read[r], cudaEventDisableTiming));
    }
    *out = g;
  });
}

int fpdt_group_destroy(fpdt_group* g) {
  if (!g) return FPDT_OK;
  for (auto e : g->ev_sent)
    if (e) cudaEventDestroy(e);
  for (auto e : g->ev_read)
    if (e) cudaEventDestroy(e);
  delete g;
  return FPDT_OK;
}

int fpdt_ctx_create_local(fpdt_group* group, int rank, int device, size_t host_arena_bytes, fpdt_ctx** out) {
  return run([&] {
    if (!out || !group || rank < 0 || rank >= group->p) fail(FPDT_ERR_ARG, "bad group/rank/out");
    *out = create_ctx(group->p, rank, nullptr, group, device, host_arena_bytes);
  });
}

int fpdt_ctx_destroy(fpdt_ctx* ctx) {
  if (!ctx) return FPDT_OK;
  int rc = run([&] {
    cudaSetDevice(ctx->device);
    cudaDeviceSynchronize();
    if (ctx->comm) {
      // non-blocking communicator: finalize, wait (bounded) for it, then destroy
      if (ncclCommFinalize(ctx->comm) == ncclInProgress) {
        ncclResult_t st = ncclInProgress;
        const auto t0 = std::chrono::steady_clock::now();
        while (ncclCommGetAsyncError(ctx->comm, &st) == ncclSuccess && st == ncclInProgress &&
               std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() < ctx->nccl_timeout_s)
          std::this_thread::sleep_for(std::chrono::microseconds(100));
      }
      ncclCommDestroy(ctx->comm);
    }
    for (auto& b : ctx->bufs)
      if (b.ptr) cudaFree(b.ptr);
    if (ctx->host) cudaFreeHost(ctx->host);
    if (ctx->host_dkv) cudaFreeHost(ctx->host_dkv);
    if (ctx->host_kvall) cudaFreeHost(ctx->host_kvall);
    if (ctx->host_x) cudaFreeHost(ctx->host_x);
    for (auto v : {&ctx->ev_off, &ctx->ev_doff, &ctx->ev_dqoff, &ctx->ev_dkvoff, &ctx->ev_a2a, &ctx->ev_xoff, &ctx->ev_up})
      for (auto e : *v) cudaEventDestroy(e);
    for (cudaEvent_t e : ctx->fixed_events())
      if (e) cudaEventDestroy(e);
    for (auto& pr : ctx->t_fwd) cudaEventDestroy(pr.first), cudaEventDestroy(pr.second);
    for (auto& pr : ctx->t_bwd) cudaEventDestroy(pr.first), cudaEventDestroy(pr.second);
    for (auto& pr : ctx->t_a2a) cudaEventDestroy(pr.first), cudaEventDestroy(pr.second);
    cudaStreamDestroy(ctx->s_comm);
    cudaStreamDestroy(ctx->s_h2d);
    cudaStreamDestroy(ctx->s_d2h);
    cudaStreamDestroy(ctx->s_comp2);
  });
  delete ctx;
  return rc;
}

int fpdt_attn_fwd(fpdt_ctx* ctx, const void* q, const void* k, const void* v, void* o, float* lse, int64_t s_local,
                  int n_q_heads, int n_kv_heads, int head_dim, int causal, int64_t chunk_size, int world_size,
                  int dtype, int offload, float softmax_scale, void* stream) {
  return run([&] {
    if (!ctx || !q || !k || !v || !o) fail(FPDT_ERR_ARG, "null pointer argument");
    if (world_size != ctx->p) fail(FPDT_ERR_ARG, "world_size differs from the context's");
    Config c = make_config(s_local, n_q_heads, n_kv_heads, head_dim, causal, chunk_size, world_size, dtype, offload,
                           softmax_scale);
    FPDT_CHECK_CUDA(cudaSetDevice(ctx->device));
    if (!ctx->plan.empty()) {
      if (ctx->plan_u != c.u) fail(FPDT_ERR_ARG, "sparsity plan has " + std::to_string(ctx->plan_u) + " chunks, the call " + std::to_string(c.u));
      if (!c.offload) fail(FPDT_ERR_UNSUPPORTED, "block sparsity needs offload = 1 (per chunk-pair schedule)");
      for (int64_t m = 0; m < c.u; ++m)
        if (!ctx->plan[(size_t)(m * c.u + m)]) fail(FPDT_ERR_ARG, "sparsity plan drops a diagonal block");
    }
    check_collective_args(ctx, 1, c, 0);
    ctx->saved_fetch = ctx->fetch_strategy;
    ctx->saved_plan = ctx->plan;
    ctx->saved_res_kv = ctx->res_kv;
    ctx->saved_res_q = ctx->res_q;
    ctx->fwd_done = false;
    forward(ctx, c, q, k, v, o, lse, static_cast<cudaStream_t>(stream));
    ctx->saved_hidden = 0;
    ctx->saved_hostio = false;
    ctx->saved = c;
    ctx->saved_q = q;
    ctx->saved_k = k;
    ctx->saved_v = v;
    ctx->fwd_done = true;
  });
}

int fpdt_attn_bwd(fpdt_ctx* ctx, const void* o, const void* dout, void* dq, void* dk, void* dv, int64_t s_local,
                  int n_q_heads, int n_kv_heads, int head_dim, int causal, int64_t chunk_size, int world_size,
                  int dtype, int offload, float softmax_scale, void* stream) {
  return run([&] {
    if (!ctx || !o || !dout || !dq || !dk || !dv) fail(FPDT_ERR_ARG, "null pointer argument");
    if (world_size != ctx->p) fail(FPDT_ERR_ARG, "world_size differs from the context's");
    Config c = make_config(s_local, n_q_heads, n_kv_heads, head_dim, causal, chunk_size, world_size, dtype, offload,
                           softmax_scale);
    if (!ctx->fwd_done) fail(FPDT_ERR_STATE, "fpdt_attn_bwd without a preceding fpdt_attn_fwd on this context");
    if (!(c == ctx->saved)) fail(FPDT_ERR_STATE, "backward arguments differ from the saved forward's");
    if (ctx->saved_hidden) fail(FPDT_ERR_STATE, "the saved forward was fpdt_block_fwd: use fpdt_block_bwd");
    if (ctx->saved_hostio) fail(FPDT_ERR_STATE, "the saved forward was fpdt_attn_fwd_host: use fpdt_attn_bwd_host");
    FPDT_CHECK_CUDA(cudaSetDevice(ctx->device));
    check_collective_args(ctx, 2, c, 0);
    backward(ctx, c, o, dout, dq, dk, dv, static_cast<cudaStream_t>(stream));
  });
}

int fpdt_attn_fwd_host(fpdt_ctx* ctx, const void* q, const void* k, const void* v, void* o, float* lse,
                       int64_t s_local, int n_q_heads, int n_kv_heads, int head_dim, int causal, int64_t chunk_size,
                       int world_size, int dtype, int offload, float softmax_scale, void* stream) {
  return run([&] {
    if (!ctx || !q || !k || !v || !o) fail(FPDT_ERR_ARG, "null pointer argument");
    if (world_size != ctx->p) fail(FPDT_ERR_ARG, "world_size differs from the context's");
    Config c = make_config(s_local, n_q_heads, n_kv_heads, head_dim, causal, chunk_size, world_size, dtype, offload,
                           softmax_scale);
    if (!c.offload) fail(FPDT_ERR_UNSUPPORTED, "fpdt_attn_fwd_host needs offload = 1 (per-chunk staging)");
    if (ctx->res_kv || ctx->res_q) fail(FPDT_ERR_UNSUPPORTED, "fpdt_attn_fwd_host does not take a residency budget");
    FPDT_CHECK_CUDA(cudaSetDevice(ctx->device));
    if (!ctx->plan.empty()) {
      if (ctx->plan_u != c.u) fail(FPDT_ERR_ARG, "sparsity plan has " + std::to_string(ctx->plan_u) + " chunks, the call " + std::to_string(c.u));
      for (int64_t m = 0; m < c.u; ++m)
        if (!ctx->plan[(size_t)(m * c.u + m)]) fail(FPDT_ERR_ARG, "sparsity plan drops a diagonal block");
    }
    check_collective_args(ctx, 5, c, 0);
    const size_t bq = (size_t)s_local * n_q_heads * head_dim * c.eb, bkv = (size_t)s_local * n_kv_heads * head_dim * c.eb;
    void* qd = dev(ctx, B_HQ, bq);
    void* kd = dev(ctx, B_HK, bkv);
    void* vd = dev(ctx, B_HV, bkv);
    void* od = dev(ctx, B_HO, bq);
    float* ld = lse ? (float*)dev(ctx, B_HLSE, (size_t)s_local * n_q_heads * 4) : nullptr;
    HostIO io;
    io.q = q; io.k = k; io.v = v; io.o = o; io.lse = lse;
    ctx->saved_fetch = ctx->fetch_strategy;
    ctx->saved_plan = ctx->plan;
    ctx->saved_res_kv = ctx->saved_res_q = 0;
    ctx->fwd_done = false;
    forward(ctx, c, qd, kd, vd, od, ld, static_cast<cudaStream_t>(stream), nullptr, &io);
    ctx->saved_hidden = 0;
    ctx->saved = c;
    ctx->saved_q = qd;
    ctx->saved_k = kd;
    ctx->saved_v = vd;
    ctx->saved_hostio = true;
    ctx->saved_host_q = q;
    ctx->saved_host_o = o;
    ctx->fwd_done = true;
  });
}

int fpdt_attn_bwd_host(fpdt_ctx* ctx, const void* o, const void* dout, void* dq, void* dk, void* dv, int64_t s_local,
                       int n_q_heads, int n_kv_heads, int head_dim, int causal, int64_t chunk_size, int world_size,
                       int dtype, int offload, float softmax_scale, void* stream) {
  return run([&] {
    if (!ctx || !o || !dout || !dq || !dk || !dv) fail(FPDT_ERR_ARG, "null pointer argument");
    if (world_size != ctx->p) fail(FPDT_ERR_ARG, "world_size differs from the context's");
    Config c = make_config(s_local, n_q_heads, n_kv_heads, head_dim, causal, chunk_size, world_size, dtype, offload,
                           softmax_scale);
    if (!ctx->fwd_done) fail(FPDT_ERR_STATE, "fpdt_attn_bwd_host without a preceding fpdt_attn_fwd_host on this context");
    if (!(c == ctx->saved)) fail(FPDT_ERR_STATE, "backward arguments differ from the saved forward's");
    if (!ctx->saved_hostio) fail(FPDT_ERR_STATE, "the saved forward was not fpdt_attn_fwd_host: use fpdt_attn_bwd");
    FPDT_CHECK_CUDA(cudaSetDevice(ctx->device));
    check_collective_args(ctx, 6, c, 0);
    const size_t bq = (size_t)s_local * n_q_heads * head_dim * c.eb, bkv = (size_t)s_local * n_kv_heads * head_dim * c.eb;
    void* od = ctx->bufs[B_HO].ptr;
    void* dod = c.p > 1 ? dev(ctx, B_HDO, bq) : nullptr;  // p == 1 fetches dO_i from the caller's rows directly
    void* dqd = dev(ctx, B_HDQ, bq);
    void* dkd = dev(ctx, B_HDK, bkv);
    void* dvd = dev(ctx, B_HDV, bkv);
    HostIO io;
    io.q = ctx->saved_host_q; io.dout = dout; io.o = const_cast<void*>(o); io.dq = dq; io.dk = dk; io.dv = dv;
    io.upload_o = o != ctx->saved_host_o;
    backward(ctx, c, od, dod, dqd, dkd, dvd, static_cast<cudaStream_t>(stream), nullptr, &io);
  });
}

namespace {
void check_block_args(fpdt_ctx* ctx, const Config& c, int hidden) {
  if (hidden <= 0 || (hidden * c.eb) % 16) fail(FPDT_ERR_ARG, "hidden must be positive and a multiple of 16 bytes");
  if (!c.offload) fail(FPDT_ERR_UNSUPPORTED, "fpdt_block_fwd/bwd need offload = 1 (per-chunk projection schedule)");
  if (ctx->res_kv || ctx->res_q)
    fail(FPDT_ERR_UNSUPPORTED, "fpdt_block_fwd/bwd do not take an HBM residency budget (chunks are projected)");
}
}  // namespace

int fpdt_block_fwd(fpdt_ctx* ctx, const void* x, const void* w_qkv, const void* w_o, void* o, float* lse, void* y,
                   int64_t s_local, int hidden,
                   int n_q_heads, int n_kv_heads, int head_dim, int causal, int64_t chunk_size, int world_size,
                   int dtype, int offload, float softmax_scale, void* stream) {
  return run([&] {
    if (!ctx || !x || !w_qkv || !o || (w_o && !y)) fail(FPDT_ERR_ARG, "null pointer argument");
    if (world_size != ctx->p) fail(FPDT_ERR_ARG, "world_size differs from the context's");
    Config c = make_config(s_local, n_q_heads, n_kv_heads, head_dim, causal, chunk_size, world_size, dtype, offload,
                           softmax_scale);
    check_block_args(ctx, c, hidden);
    FPDT_CHECK_CUDA(cudaSetDevice(ctx->device));
    check_collective_args(ctx, 3, c, hidden);
    if (!ctx->plan.empty()) {
      if (ctx->plan_u != c.u) fail(FPDT_ERR_ARG, "sparsity plan has " + std::to_string(ctx->plan_u) + " chunks, the call " + std::to_string(c.u));
      for (int64_t m = 0; m < c.u; ++m)
        if (!ctx->plan[(size_t)(m * c.u + m)]) fail(FPDT_ERR_ARG, "sparsity plan drops a diagonal block");
    }
    ctx->saved_plan = ctx->plan;
    ctx->saved_fetch = ctx->fetch_strategy;
    ctx->saved_res_kv = 0;
    ctx->saved_res_q = 0;
    ctx->fwd_done = false;
    ctx->saved_hidden_offload = ctx->hidden_offload;
    Proj pj;
    pj.x = x;
    pj.w = w_qkv;
    pj.hidden = hidden;
    pj.w_o = w_o;
    pj.y = y;
    forward(ctx, c, nullptr, nullptr, nullptr, o, lse, static_cast<cudaStream_t>(stream), &pj);
    ctx->saved = c;
    ctx->saved_q = ctx->saved_k = ctx->saved_v = nullptr;
    ctx->saved_hidden = hidden;
    ctx->saved_hostio = false;
    ctx->saved_has_wo = w_o != nullptr;
    ctx->fwd_done = true;
  });
}

int fpdt_block_bwd(fpdt_ctx* ctx, const void* x, const void* w_qkv, const void* w_o, const void* o, const void* dout,
                   void* dx, float* dw_qkv, float* dw_o, int64_t s_local, int hidden, int n_q_heads, int n_kv_heads, int head_dim, int causal,
                   int64_t chunk_size, int world_size, int dtype, int offload, float softmax_scale, void* stream) {
  return run([&] {
    if (!ctx || !w_qkv || !o || !dout || !dx || !dw_qkv || (w_o && !dw_o))
      fail(FPDT_ERR_ARG, "null pointer argument");
    if (!x && !ctx->saved_hidden_offload)
      fail(FPDT_ERR_ARG, "x is NULL but the forward did not offload the hidden state (fpdt_set_hidden_offload)");
    if (world_size != ctx->p) fail(FPDT_ERR_ARG, "world_size differs from the context's");
    Config c = make_config(s_local, n_q_heads, n_kv_heads, head_dim, causal, chunk_size, world_size, dtype, offload,
                           softmax_scale);
    if (!ctx->fwd_done) fail(FPDT_ERR_STATE, "fpdt_block_bwd without a preceding fpdt_block_fwd on this context");
    if (!(c == ctx->saved) || ctx->saved_hidden != hidden || ctx->saved_has_wo != (w_o != nullptr))
      fail(FPDT_ERR_STATE, "backward arguments differ from the saved block forward's");
    FPDT_CHECK_CUDA(cudaSetDevice(ctx->device));
    check_collective_args(ctx, 4, c, hidden);
    Proj pj;
    pj.x = x;
    pj.w = w_qkv;
    pj.dx = dx;
    pj.dw = dw_qkv;
    pj.hidden = hidden;
    pj.w_o = w_o;
    pj.dw_o = dw_o;
    backward(ctx, c, o, dout, nullptr, nullptr, nullptr, static_cast<cudaStream_t>(stream), &pj);
  });
}

int fpdt_set_sparsity(fpdt_ctx* ctx, const uint8_t* keep, int64_t n_chunks) {
  return run([&] {
    if (!ctx || n_chunks < 0 || (n_chunks > 0 && !keep)) fail(FPDT_ERR_ARG, "bad sparsity plan arguments");
    if (n_chunks == 0)
      ctx->plan.clear();
    else
      ctx->plan.assign(keep, keep + (size_t)(n_chunks * n_chunks));
    ctx->plan_u = n_chunks;
  });
}

int fpdt_set_residency(fpdt_ctx* ctx, int64_t kv_chunks, int64_t q_chunks) {
  return run([&] {
    if (!ctx || kv_chunks < 0 || q_chunks < 0) fail(FPDT_ERR_ARG, "bad residency arguments");
    ctx->res_kv = kv_chunks;
    ctx->res_q = q_chunks;
  });
}

int fpdt_set_hidden_offload(fpdt_ctx* ctx, int enable) {
  if (!ctx) return FPDT_ERR_ARG;
  ctx->hidden_offload = enable != 0;
  return FPDT_OK;
}

int fpdt_set_fetch_strategy(fpdt_ctx* ctx, int strategy) {
  return run([&] {
    if (!ctx || (strategy != FPDT_FETCH_PER_RANK && strategy != FPDT_FETCH_LEADER)) fail(FPDT_ERR_ARG, "bad fetch strategy");
    ctx->fetch_strategy = strategy;
  });
}

int fpdt_set_debug_checks(fpdt_ctx* ctx, int enable) {
  if (!ctx) return FPDT_ERR_ARG;
  ctx->check_args = enable != 0;
  return FPDT_OK;
}

int fpdt_set_bwd_order(fpdt_ctx* ctx, int order) {
  return run([&] {
    if (!ctx || order < FPDT_BWD_KV_OUTER || order > FPDT_BWD_AUTO) fail(FPDT_ERR_ARG, "bad backward order");
    ctx->bwd_order = order;
  });
}

int fpdt_bwd_host_bytes(int order, int64_t s_local, int n_q_heads, int n_kv_heads, int head_dim, int64_t chunk_size,
                        int world_size, int dtype, int64_t kv_chunks, int64_t q_chunks, const uint8_t* keep,
                        int64_t n_chunks, int64_t* out) {
  return run([&] {
    if (!out || (order != FPDT_BWD_KV_OUTER && order != FPDT_BWD_Q_OUTER) || kv_chunks < 0 || q_chunks < 0)
      fail(FPDT_ERR_ARG, "bad arguments");
    const Config c = make_config(s_local, n_q_heads, n_kv_heads, head_dim, 1, chunk_size, world_size, dtype, 1, 0.f);
    if (keep && n_chunks != c.u) fail(FPDT_ERR_ARG, "sparsity plan size differs from the chunk count");
    const int64_t u = c.u;
    auto kept = [&](int64_t i, int64_t j) { return i == j || !keep || keep[(size_t)(i * u + j)] != 0; };
    *out = bwd_host_bytes(order, c, std::min(kv_chunks, u), std::min(q_chunks, u), kept);
  });
}

int fpdt_get_stats(const fpdt_ctx* ctx, fpdt_stats* out) {
  if (!ctx || !out) return FPDT_ERR_ARG;
  *out = ctx->stats;
  return FPDT_OK;
}

int fpdt_set_kernel_timing(fpdt_ctx* ctx, int enable) {
  if (!ctx) return FPDT_ERR_ARG;
  ctx->timing = enable != 0;
  return FPDT_OK;
}

int fpdt_kernel_time(fpdt_ctx* ctx, double* fwd_ms, int64_t* fwd_launches, double* bwd_ms, int64_t* bwd_launches,
                     int reset) {
  return run([&] {
    if (!ctx) fail(FPDT_ERR_ARG, "null ctx");
    double f = 0, b = 0;
    for (size_t i = 0; i < ctx->n_fwd; ++i) {
      float ms = 0;
      FPDT_CHECK_CUDA(cudaEventSynchronize(ctx->t_fwd[i].second));
      FPDT_CHECK_CUDA(cudaEventElapsedTime(&ms, ctx->t_fwd[i].first, ctx->t_fwd[i].second));
      f += ms;
    }
    for (size_t i = 0; i < ctx->n_bwd; ++i) {
      float ms = 0;
      FPDT_CHECK_CUDA(cudaEventSynchronize(ctx->t_bwd[i].second));
      FPDT_CHECK_CUDA(cudaEventElapsedTime(&ms, ctx->t_bwd[i].first, ctx->t_bwd[i].second));
      b += ms;
    }
    if (fwd_ms) *fwd_ms = f;
    if (bwd_ms) *bwd_ms = b;
    if (fwd_launches) *fwd_launches = (int64_t)ctx->n_fwd;
    if (bwd_launches) *bwd_launches = (int64_t)ctx->n_bwd;
    if (reset) ctx->n_fwd = ctx->n_bwd = ctx->n_a2a = 0;
  });
}

int fpdt_exchange_time(fpdt_ctx* ctx, double* total_ms, int64_t* n, int64_t* bytes, double* first_ms, double* last_ms) {
  return run([&] {
    if (!ctx || !total_ms || !n || !bytes) fail(FPDT_ERR_ARG, "null argument");
    double t = 0, f = 0, l = 0;
    int64_t b = 0;
    for (size_t i = 0; i < ctx->n_a2a; ++i) {
      float ms = 0;
      FPDT_CHECK_CUDA(cudaEventSynchronize(ctx->t_a2a[i].second));
      FPDT_CHECK_CUDA(cudaEventElapsedTime(&ms, ctx->t_a2a[i].first, ctx->t_a2a[i].second));
      t += ms;
      b += ctx->t_a2a_bytes[i];
      if (i == 0) f = ms;
      l = ms;
    }
    *total_ms = t;
    *n = (int64_t)ctx->n_a2a;
    *bytes = b;
    if (first_ms) *first_ms = f;
    if (last_ms) *last_ms = l;
  });
}

int fpdt_kernel_gaps(fpdt_ctx* ctx, double* gap_ms, int64_t* n_gaps) {
  return run([&] {
    if (!ctx || !gap_ms || !n_gaps) fail(FPDT_ERR_ARG, "null argument");
    double g = 0;
    int64_t n = 0;
    for (int fwd = 0; fwd < 2; ++fwd) {
      const auto& v = fwd ? ctx->t_fwd : ctx->t_bwd;
      const auto& src = fwd ? ctx->t_fwd_src : ctx->t_bwd_src;
      const size_t cnt = fwd ? ctx->n_fwd : ctx->n_bwd;
      for (size_t i = 0; i < cnt; ++i) {
        // the previous launch of the same call on the same stream
        for (size_t j = i; j-- > 0;) {
          if (src[j].second != src[i].second) break;
          if (src[j].first != src[i].first) continue;
          float ms = 0;
          FPDT_CHECK_CUDA(cudaEventSynchronize(v[i].first));
          FPDT_CHECK_CUDA(cudaEventElapsedTime(&ms, v[j].second, v[i].first));
          g += std::max(0.f, ms);
          ++n;
          break;
        }
      }
    }
    *gap_ms = g;
    *n_gaps = n;
  });
}

}  // extern "C"
