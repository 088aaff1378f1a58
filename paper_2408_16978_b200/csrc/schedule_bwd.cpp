// Backward chunk schedules of FPDT (§4.2, fig:bw_db):
//   offload=1, KV-outer (the paper's order): D preprocess; per chunk all-to-all of (O,dO) (p>1); offload dO_m;
//               for j (outer, key/value): [h2d] fetch kv_j; for i>=j (inner, query):
//               [h2d] fetch q_i, dO_i, dq_acc_i (j>0) -> slot ; [compute] pair (i,j) ;
//               i>j: [d2h] dq_acc_i -> host ; i==j: dq_j final ; after the inner loop dk_j, dv_j
//               final -> [comm] all-to-all of dq_j,dk_j,dv_j back (p>1)
//   offload=1, Q-outer (fpdt_set_bwd_order): backward_q_outer below
//   offload=0:  per j one launch over the resident query range [jC, S)
#include "fpdt_runtime.h"

namespace fpdt_rt {

namespace {
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
  const bool X = exchanges(ctx);  // sequence-parallel exchanges (p > 1, or p = 1 through a one-rank communicator)
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
  if (X) {
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
      if (!X) {
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
        if (!X) {
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
      if (!X) {
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
      if (fin && X) send_back(st, part, j);
    }
    if (ns > 1) {  // join: dq_i is complete when both streams' pairs are
      rec(ctx->ev_join, ctx->s_comp2);
      wait(cs, ctx->ev_join);
    }
    // dq_i is final after its last key chunk
    if (X) wait(cs, ctx->ev_qo_send[0]);
    FPDT_CHECK_LAUNCH(launch_convert_out(dqi, C, hq, d, C * d, 1.f,
                                         !X ? (uint8_t*)dq + (size_t)i * C * c.Hq * d * eb : qsend, c.dtype,
                                         !X ? (int64_t)c.Hq * d : (int64_t)hq * d, 0, cs));
    ctx->stats.kernel_launches++;
    if (X) send_back(cs, 0, i);
    if (!R.q(i)) rec(ctx->ev_q_free[qsl], cs);
  }
  if (X) {
    rec(ctx->ev_comm_done, ctx->s_comm);
    wait(cs, ctx->ev_comm_done);
  }
}

}  // namespace

void backward(fpdt_ctx* ctx, const Config& c, const void* o, const void* dout, void* dq, void* dk, void* dv,
              cudaStream_t cs, const Proj* pj, const HostIO* io) {
  Nvtx nv("fpdt:backward");
  const int64_t C = c.C, u = c.u;
  const int d = c.d, hq = c.hq, hkv = c.hkv, eb = c.eb, p = c.p;
  const bool X = exchanges(ctx);  // sequence-parallel exchanges (p > 1, or p = 1 through a one-rank communicator)
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
  const bool io_p1 = io && !X;
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
  uint8_t* dores = (X && R.nq > 0) ? (uint8_t*)dev(ctx, B_DORES, (size_t)R.nq * C * 2 * hq * d * eb) : nullptr;
  float* dqres = R.nq > 0 ? (float*)dev(ctx, B_DQRES, (size_t)R.nq * C * hq * d * 4) : nullptr;
  // ---- B1/B2: D and the head-layout dO
  const void* do_h = dout;            // head-layout dO view base (p == 1: the caller's dO)
  int64_t do_rows = c.S;
  int do_heads = hq, do_head0 = 0;
  uint8_t* gathered = nullptr;        // p > 1: [S or C][2hq][d] gathered (O, dO)
  if (io_p1) {
    // host rows: D_i is formed at the first pair of query chunk i from its fetched dO_i (below); dO_i and q_i are
    // fetched from the caller's host rows
  } else if (!X) {
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
  if (X)
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
    if (!X && proj)
      FPDT_CHECK_LAUNCH(launch_convert_out(dq_final, C, hq, d, head_stride, 1.f, dqkv_buf[j & 1], c.dtype, ntot, 0,
                                           cs));
    else if (!X)
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
    if (!X) {
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
    if (!X && proj) {
      a.dk_out = dqkv_buf[j & 1];
      a.dv_out = dqkv_buf[j & 1] + (size_t)hkv * d * eb;
      a.kv_out_ld = ntot;
      a.kv_out_head0 = hq;  // as the p > 1 send buffer: dk heads [hq, hq + hkv), dv pre-offset by hkv heads
    } else if (!X) {
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
    if (!X) {
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
      if (X || proj) {
        if (X) bsend = bsend2[j & 1];
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
      if (X || proj) {
        if (X) bsend = bsend2[j & 1];
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
        if (!X) {
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
          if (!X) {
            qi = {ctx->saved_q, c.S, hq, 0};
            doi = {do_h, do_rows, do_heads, do_head0};
            q_row0 = i * C;
          } else {
            qi = {res_chunk(i), C, hcomb, 0};
            doi = {dores + (size_t)R.qslot[(size_t)i] * C * 2 * hq * d * eb, C, 2 * hq, hq};
          }
          dqi = dqres + (size_t)R.qslot[(size_t)i] * C * hq * d;
          if (X) wait(cs, ctx->ev_a2a[i]);  // its (O, dO) exchange and D_i (a no-op after the first pair)
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
        rec(ctx->ev_tmp, !X ? cs : ctx->s_comm);
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

}  // namespace fpdt_rt
