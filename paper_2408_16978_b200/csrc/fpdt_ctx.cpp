// libfpdt C-ABI entry points (include/fpdt.h): context and group life cycle, the attention / block / host-memory calls,
// the schedule options, stats and timing.  The schedules are in schedule_fwd.cpp / schedule_bwd.cpp, the runtime
// services in fpdt_runtime.cpp.
#include "fpdt_runtime.h"

using namespace fpdt_rt;

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
    if ((world_size > 1 || nccl_id) && !group) {
      ctx->xch1 = world_size == 1;
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
    // world_size 1 with an id: one-rank communicator, the exchange path (fpdt_ctx::xch1)
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
    void* dod = exchanges(ctx) ? dev(ctx, B_HDO, bq) : nullptr;  // p == 1 fetches dO_i from the caller's rows directly
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
