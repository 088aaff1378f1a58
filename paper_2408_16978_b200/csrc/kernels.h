// Internal kernel launch interface of libfpdt (not part of the C-ABI).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <mutex>
#include <set>
#include <utility>

namespace fpdt {

// Opt kernel `kern` in to `bytes` of dynamic shared memory on the CURRENT device (cudaFuncSetAttribute acts per
// device), once per (kernel, device); thread-safe (the in-process group's rank threads launch concurrently).
// Returns the cudaError_t of the attribute call (0 on success).
inline int set_max_dynamic_smem(const void* kern, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return (int)e;
  std::lock_guard<std::mutex> lk(mu);
  if (done.count({kern, dev})) return 0;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return (int)e;
  done.insert({kern, dev});
  return 0;
}

// One tensor view for the attention kernels: a bf16 (or fp32) buffer laid out [rows][heads][head_dim].
struct HeadView {
  const void* base = nullptr;  // device pointer
  int64_t rows = 0;            // number of rows in the buffer
  int heads = 0;               // heads per row in the buffer
  int head0 = 0;               // first head of the view inside the buffer
};

// Forward chunk-pair attention: queries [q_row0, q_row0 + n_q_rows) of view q against keys/values
// [kv_row0, kv_row0 + n_kv_rows) of views k, v; online softmax inside, LSE merge with a previous partial
// result (o_acc, lse_acc) in the epilogue ("rescaled in the next chunk computation").
struct FwdArgs {
  HeadView q, k, v;
  int64_t q_row0 = 0, kv_row0 = 0;
  int n_q_rows = 0, n_kv_rows = 0;  // multiples of 256 / 128
  int64_t q_pos0 = 0, kv_pos0 = 0;  // global token positions (causal mask: key pos <= query pos)
  int causal = 1;
  int hq = 0, G = 1;                // local query heads, GQA group size
  float scale_log2 = 0.f;           // softmax_scale * log2(e)
  // running partial output (fp32, normalised) and its log2-domain lse; [n_q_rows][hq][D], [hq][n_q_rows]
  float* o_acc = nullptr;
  float* lse_acc = nullptr;
  int has_prev = 0, is_final = 0;
  // final outputs (is_final): O (bf16 or fp32 by dtype) at o_out[row*o_ld + (o_head0+h)*D + e]
  void* o_out = nullptr;
  int64_t o_ld = 0;
  int o_head0 = 0;
  float* lse_save = nullptr;        // log2-domain lse, lse_save[h*lse_save_ld + row]
  int64_t lse_save_ld = 0;
  float* lse_user = nullptr;        // optional natural-log lse, lse_user[row*lse_user_ld + lse_user_head0 + h]
  int64_t lse_user_ld = 0;
  int lse_user_head0 = 0;
  // bf16 mode: residual O_fp32 - bf16(O_fp32) (bf16) at o_resid[row*o_resid_ld + h*D + e], so that the backward's
  // D = rowsum(dO o O) is formed from the fp32 output (R9); nullptr = not saved.
  __nv_bfloat16* o_resid = nullptr;
  int64_t o_resid_ld = 0;
  long long* trace = nullptr;       // debug timeline (fpdt_debug_pair), [16][4096] SM clocks
  int trace_cta = 0;
};

// Backward chunk-pair attention (KV-stationary): keys/values [kv_row0, +n_kv_rows) against queries
// [q_row0, +n_q_rows) (outer loop on key/value, inner loop on query).
struct BwdArgs {
  HeadView q, k, v, dout;
  int64_t q_row0 = 0, kv_row0 = 0;
  int n_q_rows = 0, n_kv_rows = 0;  // multiples of 128
  int64_t q_pos0 = 0, kv_pos0 = 0;
  int causal = 1;
  int hq = 0, G = 1;
  float scale = 0.f, scale_log2 = 0.f;
  const float* lse2 = nullptr;      // log2-domain lse of the query rows, lse2[h*stat_ld + (row - q_row0)]
  const float* Dstat = nullptr;     // D = rowsum(dO o O), same indexing
  int64_t stat_ld = 0;
  float* dq_acc = nullptr;          // fp32 head-major [hq][dq_head_stride/D][D], rows [0, n_q_rows) of each head
  int64_t dq_head_stride = 0;       // elements between heads of dq_acc (>= n_q_rows * D); accumulated (scaled)
  // dK/dV: fp32 accumulators [n_kv_rows][hkv][D] (kv_acc_init: overwrite instead of add)
  float* dk_acc = nullptr;
  float* dv_acc = nullptr;
  int kv_acc_init = 0;
  int kv_final = 0;                 // 1: also write final dK/dV (bf16/fp32 by dtype) to dk_out/dv_out
  void* dk_out = nullptr;
  void* dv_out = nullptr;
  int64_t kv_out_ld = 0;            // elements per row of dk_out/dv_out
  int kv_out_head0 = 0;
  long long* trace = nullptr;       // debug timeline (fpdt_debug_pair), [16][4096] SM clocks
  int trace_cta = 0;
};

int launch_attn_fwd_bf16(const FwdArgs& a, int head_dim, cudaStream_t s);
int launch_attn_bwd_bf16(const BwdArgs& a, int head_dim, cudaStream_t s);
int launch_attn_bwd_pipe_bf16(const BwdArgs& a, int head_dim, cudaStream_t s);
int launch_attn_bwd_q64_bf16(const BwdArgs& a, int head_dim, cudaStream_t s);  // head_dim 128
int launch_attn_fwd_f32(const FwdArgs& a, int head_dim, cudaStream_t s);
int launch_attn_bwd_f32(const BwdArgs& a, int head_dim, cudaStream_t s);

// Support kernels (layout.cu)
// D[h*ld + t] = sum_e dO[t][h][e] * O[t][h][e]  (fp32 accumulate), t in [0,rows)
// (o and dout rows are row_ld elements apart; head h of row t starts at t*row_ld + h*head_dim)
// resid (bf16, nullable): O_fp32 - O, rows resid_ld elements apart, added to O before the dot product
int launch_bwd_preprocess_D(const void* o, const void* dout, int dtype, int64_t rows, int heads, int head_dim,
                            int64_t row_ld, const void* resid, int64_t resid_ld, float* D, int64_t ld,
                            cudaStream_t s);
// fp32 head-major src[h*src_head_stride + row*d + e] * scale -> bf16/fp32 dst[row*dst_ld + (dst_head0+h)*d + e]
int launch_convert_out(const float* src, int64_t rows, int heads, int head_dim, int64_t src_head_stride, float scale,
                       void* dst, int dtype, int64_t dst_ld, int dst_head0, cudaStream_t s);
// pack rows [c][H][d] of a sequence-layout tensor into send[p][c][H/p][d] (elem_bytes 2 or 4); source rows
// src_row_ld elements apart (0 = H*head_dim, dense)
int launch_pack_seq2head(const void* src, int64_t c, int H, int head_dim, int p, int elem_bytes, void* dst,
                         int64_t dst_peer_stride_elems, int64_t dst_row_ld, int dst_head0, cudaStream_t s,
                         int64_t src_row_ld = 0);
// unpack recv[p][c][H/p][d] into sequence-layout rows [c][H][d], rows dst_row_ld elements apart (0 = dense)
int launch_unpack_head2seq(const void* src, int64_t src_peer_stride_elems, int64_t src_row_ld, int src_head0,
                           int64_t c, int H, int head_dim, int p, int elem_bytes, void* dst, cudaStream_t s,
                           int64_t dst_row_ld = 0);
// Projection GEMMs (gemm_sm100.cu; fpdt_block_fwd/bwd).  Row-major operands with row strides in elements; bf16 mode
// (dtype_fp32 = 0) on tcgen05 with fp32 accumulation, fp32 mode on true-FP32 SIMT.  Returns 0, a cudaError_t, or -1
// (tensor map encoding failed).
// Optional scatter of the forward projection's output into the all-to-all send layout: column j of the projected
// rows (head j / d of the q | k | v heads) goes to send[peer][row][slot][e] (peer_stride elements per peer).
struct ScatterOut {
  int d = 0, Hq = 0, Hkv = 0, hq = 0, hkv = 0;
  int64_t peer_stride = 0;
};
// Y[rows][n] (ldy) = X[rows][k] (ldx) W[k][n] (ldw); scatter != nullptr: Y is the send buffer (ldy unused)
int launch_gemm_xw(int dtype_fp32, const void* X, int64_t ldx, const void* W, int64_t ldw, void* Y, int64_t ldy,
                   int64_t rows, int64_t k, int64_t n, const ScatterOut* scatter, cudaStream_t s);
// dX[rows][k] (ldx) = dY[rows][n] (ldy) W^T, W[k][n] (ldw)
int launch_gemm_dx(int dtype_fp32, const void* dY, int64_t ldy, const void* W, int64_t ldw, void* dX, int64_t ldx,
                   int64_t rows, int64_t k, int64_t n, cudaStream_t s);
// dW[k][n] fp32 (= or +=) X[rows][k]^T dY[rows][n]
int launch_gemm_dw(int dtype_fp32, const void* X, int64_t ldx, const void* dY, int64_t ldy, float* dW, int64_t rows,
                   int64_t k, int64_t n, bool accumulate, cudaStream_t s);

// debug: one thread sleeps about ns nanoseconds on stream s (scheduler stress, FPDT_STRESS_NS)
int launch_stress_sleep(uint32_t ns, cudaStream_t s);
// lse transpose: src[h*ld + t] (log2-domain) -> dst[t*dst_ld + dst_head0 + h] (natural log)
int launch_lse_to_user(const float* src, int64_t ld, int64_t rows, int heads, float* dst, int64_t dst_ld,
                       int dst_head0, cudaStream_t s);

}  // namespace fpdt
