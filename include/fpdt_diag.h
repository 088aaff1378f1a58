/* fpdt_diag.h — diagnostics of libfpdt, in a SEPARATE library (paper_2408_16978_b200/libfpdt_diag.so, linked
 * against libfpdt.so).  Nothing here is on the FPDT path (include/fpdt.h): these are micro-benchmarks and direct
 * kernel launches used by tests/ and tools/ to check operand formats, layout kernels and single pair kernels in
 * isolation.  All pointers are device pointers unless stated; every call is enqueued on `stream`.
 */
#ifndef FPDT_DIAG_H_
#define FPDT_DIAG_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Diagnostic self-test of the tcgen05/TMA operand formats (one 128-row tile product on one CTA).
 * variant 0: out[128x128] = A[128xD] B[128xD]^T;  1: out[128xD] = P[128x128] V[128xD] (P in TMEM);
 * 2: out[128xD] = A[128x128] V[128xD] (A MN-major smem).  a, b: device bf16; A/B tiles are rows
 * [0,128) of head n_heads-1 of [rows][n_heads][head_dim] tensors; P/A of variants 1-2 are [128][128].
 * out: device fp32.  Returns 0 or a CUDA error code. */
int fpdt_selftest_umma(int variant, int head_dim, const void* a, const void* b, int n_heads, int rows, void* out,
                       void* stream);

/* Diagnostic micro-benchmark (one CTA of 128 threads per SM, 148 CTAs): what = 0 SS tcgen05.mma
 * M=128 N=n K=16, 1 TS tcgen05.mma, 2 MUFU ex2 per thread, 3 tcgen05.ld 32x32b.x32 per warp, 4 FMA
 * polynomial exp2 per thread.  Writes SM cycles per operation (CTA 0) to out[0] (device fp32).
 * Returns 0 or a CUDA error code. */
int fpdt_selftest_perf(int what, int n, int iters, float* out, void* stream);

/* Diagnostic micro-benchmark of the forward softmax's exponential stage in registers (148 CTAs of `threads`):
 * what 0 = 128 columns per thread, 1 = 64; one pair in `every` as the FMA-pipe polynomial (0 = all MUFU).
 * Writes SM cycles per row per thread (CTA 0) to out[0] (device fp32).  Returns 0 or a CUDA error code. */
int fpdt_selftest_softmax(int what, int threads, int every, int iters, float* out, void* stream);

/* Diagnostic micro-benchmark of the dQ reduce-add path: 148 CTAs each reduce a 40 KB fp32 staging tile into global
 * memory `iters` times (mode 0: three swizzled tensor boxes as in the backward kernel, 1: one 1-D bulk reduce,
 * 2: ten 4 KB bulk reduces, 3: one unswizzled [128 x 80] box, 4: plain bulk store), `inflight` groups in flight
 * (1 or 2), into one region per CTA or (shared_target) the same region; 5: mode 0 plus a 40 KB bulk load per tile,
 * 6: the load alone.  gbuf: device fp32, >= 2*148*10240 floats.
 * out[0] = SM cycles per tile (device fp32).  Returns 0 or an error code. */
int fpdt_selftest_reduce(int mode, int iters, int inflight, int shared_target, float* gbuf, float* out, void* stream);

/* Diagnostic micro-benchmark of the CTA-pair MMA (groundwork for a CTA-pair backward): 148 CTAs in
 * clusters of 2, one per SM; mode 0: every CTA issues SS tcgen05.mma.cta_group::1 M=128 N=n K=16; mode 1: each
 * pair's leader issues SS tcgen05.mma.cta_group::2 M=256 N=n K=16 (each CTA supplies 128 rows of A and n/2 rows of B).
 * n: 16..256, multiple of 16.  out[0] = SM cycles per MMA (device fp32).  Returns 0, FPDT_ERR_ARG or a CUDA error. */
int fpdt_selftest_pair(int mode, int n, int iters, float* out, void* stream);

/* Diagnostic: run ONE all-to-all layout kernel on caller device buffers.
 *   which 0 (pack, sequence -> head-sharded send layout): src = c sequence rows [c][H][head_dim] (rows seq_row_ld
 *     elements apart, 0 = H * head_dim); dst element (peer, t, hh, e) = src (t, peer * H/p + hh, e), stored at
 *     dst[peer * hs_peer_stride + t * hs_row_ld + (hs_head0 + hh) * head_dim + e].
 *   which 1 (unpack): the inverse, src head-sharded, dst sequence rows.
 * elem_bytes 2 or 4 (the kernels move raw 16-byte vectors).  Returns FPDT_OK, FPDT_ERR_ARG or FPDT_ERR_CUDA. */
int fpdt_debug_relayout(int which, const void* src, void* dst, int64_t c, int H, int head_dim, int p, int elem_bytes,
                        int64_t hs_peer_stride, int64_t hs_row_ld, int hs_head0, int64_t seq_row_ld, void* stream);

/* Diagnostic: launch ONE bf16 chunk-pair kernel directly (no scheduler) on caller device buffers, rows
 * [0, n_rows) of q/k/v/dout against each other (the diagonal pair when causal = 1).
 *   which 0 (forward):  out0 = o bf16 [n_rows][n_q_heads][head_dim], out1 = log2-domain lse fp32 [n_q_heads][n_rows]
 *   which 1 (backward; 2 / 3 / 4 force the pipe kernel (multicast CTA pairs when n_rows / 128 is even), the
 *            cta_group::2 kernel or the 64-row-query-tile kernel): lse2 / Dstat fp32 [n_q_heads][n_rows] (log2-domain lse, rowsum(dO o O)),
 *                       out0 = dq accumulator fp32 [n_q_heads][n_rows][head_dim] (zeroed by the caller; scaled
 *                       dQ is added), out1 / out2 = dK / dV bf16 [n_rows][n_kv_heads][head_dim]
 * trace (nullable): device int64 [16][4096] receiving SM-clock timestamps of warp-role protocol events of
 * CTA (trace_cta, 0).  n_rows: a multiple of 256 for which 0 and 3, of 128 otherwise (else FPDT_ERR_DIVISIBILITY).
 * Returns FPDT_OK or a status. */
int fpdt_debug_pair(int which, int head_dim, int causal, const void* q, const void* k, const void* v, const void* dout,
                    const float* lse2, const float* Dstat, void* out0, void* out1, void* out2, int64_t n_rows,
                    int n_q_heads, int n_kv_heads, long long* trace, int trace_cta, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* FPDT_DIAG_H_ */
