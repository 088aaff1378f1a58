// Diagnostic entry point: one chunk-pair attention kernel launched directly on caller buffers, with an
// optional per-CTA SM-clock timeline (kernels.h FwdArgs/BwdArgs::trace).  Not used by the FPDT schedule;
// it exists so a single pair kernel can be timed and its warp-role protocol inspected in isolation.
#include <cmath>

#include "fpdt.h"
#include "fpdt_diag.h"
#include "kernels.h"

namespace fpdt {
// CTA-pair backward (diag/attn_bwd_2cta_sm100.cu, this library only)
int launch_attn_bwd_2cta_bf16(const BwdArgs& a, int head_dim, cudaStream_t s);
}  // namespace fpdt

using namespace fpdt;

extern "C" int fpdt_debug_pair(int which, int head_dim, int causal, const void* q, const void* k, const void* v,
                               const void* dout, const float* lse2, const float* Dstat, void* out0, void* out1,
                               void* out2, int64_t n_rows, int n_q_heads, int n_kv_heads, long long* trace,
                               int trace_cta, void* stream) {
  if (head_dim != 64 && head_dim != 80 && head_dim != 128) return FPDT_ERR_UNSUPPORTED;
  // forward (2 query tiles per CTA) and the CTA-pair backward: 256-row multiples; the other backward kernels: 128
  if (n_rows % ((which == 0 || which == 3) ? 256 : 128) || n_q_heads % n_kv_heads) return FPDT_ERR_DIVISIBILITY;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const float scale = (float)(1.0 / std::sqrt((double)head_dim));
  if (which == 0) {
    FwdArgs a;
    a.q = {q, n_rows, n_q_heads, 0};
    a.k = {k, n_rows, n_kv_heads, 0};
    a.v = {v, n_rows, n_kv_heads, 0};
    a.n_q_rows = (int)n_rows;
    a.n_kv_rows = (int)n_rows;
    a.causal = causal;
    a.hq = n_q_heads;
    a.G = n_q_heads / n_kv_heads;
    a.scale_log2 = scale * 1.4426950408889634f;
    a.is_final = 1;
    a.o_out = out0;
    a.o_ld = (int64_t)n_q_heads * head_dim;
    a.lse_save = static_cast<float*>(out1);
    a.lse_save_ld = n_rows;
    a.trace = trace;
    a.trace_cta = trace_cta;
    return launch_attn_fwd_bf16(a, head_dim, s) == 0 ? FPDT_OK : FPDT_ERR_CUDA;
  }
  BwdArgs a;
  a.q = {q, n_rows, n_q_heads, 0};
  a.k = {k, n_rows, n_kv_heads, 0};
  a.v = {v, n_rows, n_kv_heads, 0};
  a.dout = {dout, n_rows, n_q_heads, 0};
  a.n_q_rows = (int)n_rows;
  a.n_kv_rows = (int)n_rows;
  a.causal = causal;
  a.hq = n_q_heads;
  a.G = n_q_heads / n_kv_heads;
  a.scale = scale;
  a.scale_log2 = scale * 1.4426950408889634f;
  a.lse2 = lse2;
  a.Dstat = Dstat;
  a.stat_ld = n_rows;
  a.dq_acc = static_cast<float*>(out0);
  a.dq_head_stride = n_rows * head_dim;
  a.kv_acc_init = 1;
  a.kv_final = 1;
  a.dk_out = out1;
  a.dv_out = out2;
  a.kv_out_ld = (int64_t)n_kv_heads * head_dim;
  a.trace = trace;
  a.trace_cta = trace_cta;
  // which 1: the kernel the library dispatches; 2: the single-CTA pipelined kernel (d = 64 / 80); 3: the CTA-pair
  // kernel (d = 64 / 80); 4: the 64-row query-tile kernel
  const int rc = which == 2   ? launch_attn_bwd_pipe_bf16(a, head_dim, s)
                 : which == 3 ? launch_attn_bwd_2cta_bf16(a, head_dim, s)
                 : which == 4 ? launch_attn_bwd_q64_bf16(a, head_dim, s)
                              : launch_attn_bwd_bf16(a, head_dim, s);
  return rc == 0 ? FPDT_OK : FPDT_ERR_CUDA;
}

// Diagnostic: one all-to-all layout kernel (F3/F10/B2/B7) on caller device buffers (include/fpdt_diag.h).
extern "C" int fpdt_debug_relayout(int which, const void* src, void* dst, int64_t c, int H, int head_dim, int p,
                                   int elem_bytes, int64_t hs_peer_stride, int64_t hs_row_ld, int hs_head0,
                                   int64_t seq_row_ld, void* stream) {
  using namespace fpdt;
  if ((which != 0 && which != 1) || !src || !dst || c <= 0 || H <= 0 || p <= 0 || H % p ||
      (elem_bytes != 2 && elem_bytes != 4) || (head_dim * elem_bytes) % 16 || hs_peer_stride <= 0 || hs_row_ld <= 0 ||
      hs_head0 < 0 || seq_row_ld < 0)
    return FPDT_ERR_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int rc = which == 0 ? launch_pack_seq2head(src, c, H, head_dim, p, elem_bytes, dst, hs_peer_stride, hs_row_ld,
                                                   hs_head0, s, seq_row_ld)
                            : launch_unpack_head2seq(src, hs_peer_stride, hs_row_ld, hs_head0, c, H, head_dim, p,
                                                     elem_bytes, dst, s, seq_row_ld);
  return rc == 0 ? FPDT_OK : FPDT_ERR_CUDA;
}
