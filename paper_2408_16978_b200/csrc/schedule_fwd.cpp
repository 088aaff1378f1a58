// Forward chunk schedule of FPDT (§4.1, fig:pipele_case2):
//   offload=1:  per chunk m: [comm] all-to-all of q,k,v chunk m (p>1)  [d2h] offload q_m, kv_m
//               [compute] diagonal pair (m,m) ; for i<m: [h2d] fetch kv_i -> slot i%2,
//               [compute] pair (m,i) with LSE merge ; [comm] all-to-all of O_m back (p>1)
//   offload=0:  per chunk m one launch over the resident key range [0,(m+1)C)
// Streams: compute (= the caller's stream), comm, h2d, d2h; every cross-stream dependency is an event.
#include "fpdt_runtime.h"

namespace fpdt_rt {

void forward(fpdt_ctx* ctx, const Config& c, const void* q, const void* k, const void* v, void* o, float* lse,
             cudaStream_t cs, const Proj* pj, const HostIO* io) {
  Nvtx nv("fpdt:forward");
  const int64_t C = c.C, u = c.u;
  const int d = c.d, hq = c.hq, hkv = c.hkv, eb = c.eb, p = c.p;
  const bool X = exchanges(ctx);  // sequence-parallel exchanges (p > 1, or p = 1 through a one-rank communicator)
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
  if (!c.offload && X) store = (uint8_t*)dev(ctx, B_STORE, (size_t)c.S * hcomb * d * eb);
  // head-layout output of a chunk before its return all-to-all (p > 1), double-buffered so that chunk m+1's pairs
  // run while chunk m's output is exchanged
  uint8_t* o_hat[2] = {nullptr, nullptr};
  if (X)
    for (int b = 0; b < 2; ++b) o_hat[b] = (uint8_t*)dev(ctx, b ? B_OHAT1 : B_OHAT, (size_t)C * hq * d * eb);
  uint8_t* a2a_send[2] = {nullptr, nullptr};
  uint8_t* a2a_recv[2] = {nullptr, nullptr};
  if (X) {
    for (int b = 0; b < 2; ++b) {
      a2a_send[b] = (uint8_t*)dev(ctx, B_A2A_SEND0 + b, (size_t)C * hcomb * d * eb);
      if (c.offload) a2a_recv[b] = (uint8_t*)dev(ctx, B_A2A_RECV0 + b, (size_t)C * hcomb * d * eb);
    }
  }
  // fused projection (fpdt_block_fwd): chunk m of the hidden state is projected on the comm stream just before
  // its all-to-all; the GEMM's epilogue writes the all-to-all send layout [p][c][hq + 2hkv][d] directly
  // (the pack fused into the GEMM); at p = 1 that layout is the combined head layout [C][Hq + 2Hkv][d] itself.
  const bool proj = pj != nullptr, headbuf = X || proj;
  const int64_t ntot = (int64_t)(c.Hq + 2 * c.Hkv) * d;
  ScatterOut scat;
  scat.d = d; scat.Hq = c.Hq; scat.Hkv = c.Hkv; scat.hq = hq; scat.hkv = hkv;
  scat.peer_stride = c.c * hcomb * d;
  if (proj && !X)
    for (int b = 0; b < 2; ++b) a2a_recv[b] = (uint8_t*)dev(ctx, B_A2A_RECV0 + b, (size_t)C * hcomb * d * eb);
  const Residency R = make_residency(u, c.offload ? ctx->saved_res_kv : 0, c.offload ? ctx->saved_res_q : 0);
  uint8_t* resstore = (X && R.n > 0) ? (uint8_t*)dev(ctx, B_RESSTORE, (size_t)R.n * C * hcomb * d * eb) : nullptr;
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
  const bool io_p1 = io && !X;
  if (io_p1) stage_p1(0);
  // p == 1 with offload: the head-layout chunk IS the caller's rows; offload all chunks up front
  if (!X && c.offload && !proj && !io) {
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
      if (!X) wait(cs, ctx->ev_recv_used_d[b]);              // the offload of chunk m-2 has read this buffer
      else if (m >= 2) wait(cs, ctx->ev_a2a[m - 2]);             // chunk m-2's all-to-all has read the send buffer
      const uint8_t* xm = (const uint8_t*)pj->x + (size_t)m * c.c * pj->hidden * eb;
      gemm_xw(ctx, c.dtype, xm, pj->hidden, pj->w, ntot, !X ? recv : a2a_send[b], ntot, c.c, pj->hidden, ntot, cs,
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
    if (X) alltoall(ctx, a2a_send[b], recv, per_peer, c.dtype);
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
    if (!X) {
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
    if (proj && pj->w_o && !X)
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
    if (X) {
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

}  // namespace fpdt_rt
