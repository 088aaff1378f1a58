// libfpdt host runtime services (fpdt_runtime.h): device buffer pool, events, scheduler stress, the pinned host chunk
// store, copies, the all-to-all and point-to-point exchanges (NCCL or the in-process group), the SPMD argument check,
// and the kernel / GEMM launch wrappers.
#include "fpdt_runtime.h"

namespace fpdt_rt {

thread_local std::string g_last_error;

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

HostLayout host_layout(const Config& c) {
  HostLayout h;
  h.q_bytes = (size_t)c.C * c.hq * c.d * c.eb;
  h.kv_bytes = (size_t)c.C * 2 * c.hkv * c.d * c.eb;
  h.do_bytes = h.q_bytes;
  h.dq_bytes = (size_t)c.C * c.hq * c.d * 4;
  h.total = (size_t)c.u * (h.q_bytes + h.kv_bytes + h.do_bytes + h.dq_bytes);
  return h;
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
             int64_t rows, int64_t k, int64_t n, cudaStream_t s, const ScatterOut* sc) {
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

}  // namespace fpdt_rt
