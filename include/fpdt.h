/* fpdt.h — C ABI of libfpdt: the hot path of the Fully Pipelined Distributed Transformer
 * (FPDT, arXiv 2408.16978) on NVIDIA B200 (sm_100a).
 *
 * The library computes sequence-chunked, sequence-parallel (Ulysses) causal attention, forward and
 * backward, exactly as the paper's FPDT attention block does (§4.1-4.2):
 *   - every rank holds its local sequence shard [s_local, heads, head_dim] (b = 1 as in
 *     every experiment of the paper), in the rank-ordinal ("shuffled") token order of
 *     fig:seq_shuffle: local row t of rank r is global token
 *         ((t / c) * p + r) * c + (t % c),   c = chunk_size / world_size   (fpdt_global_token);
 *   - the shard is cut into u = s_local / c chunks T_i; per chunk an all-to-all scatters heads
 *     and gathers the sequence so each rank attends a contiguous chunk of
 *     C = chunk_size global tokens with H/p heads;
 *   - query chunk m attends the resident key/value chunk m (causal), then the earlier
 *     chunks i < m fetched one by one from pinned host memory, merging partial outputs with the
 *     online-softmax (log-sum-exp) policy (fig:pipele_case2);
 *   - q, k, v chunks are offloaded to host memory after use;
 *   - backward: outer loop over key/value chunks j, inner loop over query chunks i >= j, with the
 *     dq partials accumulated in host memory and dk_j, dv_j final after outer iteration j (P:L365,
 *     fig:bw_db); final gradients return to their owner ranks by the reverse all-to-all;
 *   - copies, all-to-all and compute run on separate CUDA streams with double-buffered device slots
 *     (§4.2 "Double buffering").
 *
 * Conventions for every call below
 *   - Tensor pointers are DEVICE pointers unless a name says host; tensors are contiguous row-major
 *     [s_local][heads][head_dim] (head_dim fastest), 16-byte aligned.  The caller owns them.
 *   - dtype FPDT_BF16: bf16 tensors, fp32 accumulation and softmax, tcgen05 tensor-core kernels.
 *     dtype FPDT_FP32: fp32 tensors and true-fp32 SIMT kernels (validation mode).
 *   - softmax_scale <= 0 selects 1/sqrt(head_dim) (the paper never states the scale; R1).
 *   - causal must be 1 (the paper's causal LLM setting; 0 returns FPDT_ERR_UNSUPPORTED).
 *   - All calls that take a context are collective over the sequence-parallel group (SPMD): every
 *     rank must make the same calls with the same shape arguments, in the same order.  A mismatch
 *     hangs NCCL; it is documented, not detected.
 *   - Calls are stream-ordered after `stream` (a cudaStream_t; NULL = legacy default stream) and
 *     return once the work is enqueued (no host synchronisation on the hot path).  Work that the
 *     caller enqueues on `stream` afterwards sees the results.
 *   - Return value: FPDT_OK (0) or one of fpdt_status; fpdt_last_error() gives a message.
 *     Asynchronous CUDA/NCCL faults surface as FPDT_ERR_CUDA / FPDT_ERR_NCCL on a later call.
 */
#ifndef FPDT_H_
#define FPDT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fpdt_ctx fpdt_ctx;

enum fpdt_status {
  FPDT_OK = 0,
  FPDT_ERR_ARG = 1,           /* null pointer, non-positive size, world_size/rank mismatch */
  FPDT_ERR_DIVISIBILITY = 2,  /* S % C, C % p, Hq % p, Hkv % p, Hq % Hkv, (C/p... tile) rules, see below */
  FPDT_ERR_UNSUPPORTED = 3,   /* head_dim not in {64, 80, 128}, causal == 0, unsupported dtype */
  FPDT_ERR_HOST_OOM = 4,      /* the pinned host chunk store cannot be allocated / is too small */
  FPDT_ERR_DEVICE_OOM = 5,    /* device working-set allocation failed */
  FPDT_ERR_STATE = 6,         /* backward without a matching forward on this context */
  FPDT_ERR_CUDA = 7,
  FPDT_ERR_NCCL = 8
};

enum fpdt_dtype { FPDT_BF16 = 0, FPDT_FP32 = 1 };

/* Rank 0 creates the NCCL unique id (128 bytes) for world_size > 1; the caller broadcasts it to the
 * other ranks (e.g. with torch.distributed).  Not needed when world_size == 1. */
int fpdt_get_unique_id(unsigned char id[128]);

/* Create a context on CUDA device `device` for rank `rank` of a group of `world_size` ranks.
 * nccl_id: the 128-byte id from fpdt_get_unique_id.  world_size == 1: NULL (the schedules work on the caller's rows
 *   in place), or an id of its own, which makes a one-rank NCCL communicator and runs the sequence-parallel path with
 *   every exchange an ncclAlltoAll of the rank with itself (pack, exchange, unpack; the results equal the NULL case):
 *   the production NCCL data plane on one GPU.
 * host_arena_bytes: pinned host chunk store to reserve now; 0 = allocate on the first offloaded
 * forward (sized for that call).  The context owns the NCCL communicator, its streams and events,
 * the pinned host store, the device slots and the saved state of ONE attention layer.
 * Returns FPDT_ERR_HOST_OOM if the store cannot be pinned, FPDT_ERR_NCCL if communicator set-up fails. */
int fpdt_ctx_create(int world_size, int rank, const unsigned char* nccl_id, int device, size_t host_arena_bytes,
                    fpdt_ctx** out);

/* In-process group: world_size ranks living in ONE process on ONE device `device`, one host thread per rank
 * (single-GPU multi-rank testing of the p > 1 path; SURVEY §8(e) "fallback if only 1 GPU is granted").
 * Contexts made with fpdt_ctx_create_local replace NCCL's all-to-all by a copy-engine exchange with exactly
 * ncclAlltoAll's layout (receive block q = rank q's send block r); packing, scheduling, offload and the reverse
 * all-to-alls are the same code as the NCCL path.  Rules: every rank's calls run on their own host thread and
 * their own `stream` (sharing one stream across ranks can deadlock the device), all ranks make the same calls;
 * a failing rank leaves the others blocked in the group barrier.  The group must outlive its contexts. */
typedef struct fpdt_group fpdt_group;
int fpdt_group_create(int world_size, int device, fpdt_group** out);
int fpdt_group_destroy(fpdt_group* group);
int fpdt_ctx_create_local(fpdt_group* group, int rank, int device, size_t host_arena_bytes, fpdt_ctx** out);

/* Release everything the context owns (synchronises the context's streams first). */
int fpdt_ctx_destroy(fpdt_ctx* ctx);

/* Forward.
 *   q [s_local, n_q_heads, head_dim], k, v [s_local, n_kv_heads, head_dim]  (inputs, rank-ordinal order)
 *   o [s_local, n_q_heads, head_dim]                                      (output, same dtype)
 *   lse [s_local, n_q_heads] fp32, natural log of the softmax denominator (output; may be NULL)
 *   chunk_size C: global tokens per chunk (the paper's "chunk size"); the global
 *     sequence S = s_local * world_size must satisfy S % C == 0, C % world_size == 0 and
 *     (C / world_size) * world_size == C with C a multiple of 256.
 *   n_q_heads % world_size == 0, n_kv_heads % world_size == 0, n_q_heads % n_kv_heads == 0 (GQA).
 *   offload 1: q, k, v chunks go to the pinned host store and earlier key/value chunks are fetched
 *     back double-buffered (the paper's FPDT with offloading).  offload 0: chunks stay in device
 *     memory ("FPDT chunking only"); with world_size == 1 the caller's q, k, v are used in
 *     place and must stay valid and unmodified until fpdt_attn_bwd.
 * Saves, for the backward, the per-row log-sum-exp and (offload 1) the chunk store. */
int fpdt_attn_fwd(fpdt_ctx* ctx, const void* q, const void* k, const void* v, void* o, float* lse, int64_t s_local,
                  int n_q_heads, int n_kv_heads, int head_dim, int causal, int64_t chunk_size, int world_size,
                  int dtype, int offload, float softmax_scale, void* stream);

/* Backward of the last fpdt_attn_fwd on this context, for upstream gradient dout.
 *   o, dout [s_local, n_q_heads, head_dim] (inputs: the forward output and dL/dO)
 *   dq [s_local, n_q_heads, head_dim], dk, dv [s_local, n_kv_heads, head_dim] (outputs, overwritten)
 * Every shape/flag argument must equal the forward's, else FPDT_ERR_STATE (also if no forward ran). */
int fpdt_attn_bwd(fpdt_ctx* ctx, const void* o, const void* dout, void* dq, void* dk, void* dv, int64_t s_local,
                  int n_q_heads, int n_kv_heads, int head_dim, int causal, int64_t chunk_size, int world_size,
                  int dtype, int offload, float softmax_scale, void* stream);

/* Forward and backward with the caller's tensors in HOST memory (the paper's setting: activations live in host
 * memory and each chunk is brought to the GPU when it is needed, "we offload ... to the host memory"
 * "the prefetching of the input hidden state").  Same arguments, shapes, layouts and errors as fpdt_attn_fwd /
 * fpdt_attn_bwd, except that q, k, v, o, lse (forward) and o, dout, dq, dk, dv (backward) are host pointers, pinned
 * (cudaHostAlloc / cudaHostRegister) for the copies to run asynchronously.  The library stages the rows through
 * device mirrors (library-owned, s_local rows of each tensor) chunk by chunk on its own copy streams: chunk m's upload
 * is enqueued just ahead of its first reader and each chunk's output rows leave as soon as they are final, so the
 * host copies share the host link with the chunk fetches in the schedule's own order.  With world_size 1 the backward
 * fetches q_i and dO_i straight from the caller's host rows (the forward does not offload q): the forward's host q
 * must stay valid and unmodified until fpdt_attn_bwd_host.  The backward reuses the forward's device copy of o when
 * `o` is the forward's output pointer (else it uploads o first).  Outputs are complete when `stream` reaches the end
 * of the call.  offload must be 1 and no residency budget set (FPDT_ERR_UNSUPPORTED); the backward runs the paper's
 * KV-outer order; the sparsity plan and the fetch strategy apply as for fpdt_attn_fwd.  fpdt_attn_bwd_host needs a
 * saved fpdt_attn_fwd_host (and fpdt_attn_bwd an fpdt_attn_fwd): else FPDT_ERR_STATE.  Host bytes moved for the
 * caller's rows are counted in fpdt_stats.bytes_io_h2d / bytes_io_d2h. */
int fpdt_attn_fwd_host(fpdt_ctx* ctx, const void* q, const void* k, const void* v, void* o, float* lse,
                       int64_t s_local, int n_q_heads, int n_kv_heads, int head_dim, int causal, int64_t chunk_size,
                       int world_size, int dtype, int offload, float softmax_scale, void* stream);
int fpdt_attn_bwd_host(fpdt_ctx* ctx, const void* o, const void* dout, void* dq, void* dk, void* dv, int64_t s_local,
                       int n_q_heads, int n_kv_heads, int head_dim, int causal, int64_t chunk_size, int world_size,
                       int dtype, int offload, float softmax_scale, void* stream);

/* Attention block with the chunked QKV projection fused in front.  PAPER.md P:L206: "we
 * directly slice the local sequence tensor into u chunks ... T_i is projected to query q_i, key k_i, and value v_i.
 * Then, we perform the Alltoall"; the final dq_j, dk_j, dv_j, all-to-all'd back, "are used to compute the
 * gradient of the input hidden state".  Per chunk the projection is the library's tcgen05 GEMM (fp32 accumulation;
 * fp32 mode: a SIMT fp32 GEMM) whose epilogue writes the all-to-all send layout, enqueued one chunk ahead of the
 * chunk's all-to-all, so the full-sequence q, k, v never exist;
 * in the backward each chunk's projection gradient runs as soon as its dq, dk, dv are final (the paper's KV-outer
 * order; fpdt_set_bwd_order is ignored here).
 *   x      [s_local][hidden]                         hidden state, rank-ordinal rows (as q of fpdt_attn_fwd)
 *   w_qkv  [hidden][(n_q_heads + 2 n_kv_heads) * head_dim]  row-major projection weight; columns are the q heads,
 *          then the k heads, then the v heads, head_dim fastest: [q | k | v] = x w_qkv (no bias)
 *   w_o    [n_q_heads * head_dim][hidden] or NULL: the output projection after the attention, y = o w_o (o flattened
 *          per token, head-major), computed per chunk as soon as the chunk's o is final; NULL = no output projection
 *   o, lse as fpdt_attn_fwd (o is always written: the backward needs it); y [s_local][hidden] (output; with w_o)
 *   dout   without w_o: dL/do [s_local][n_q_heads][head_dim]; with w_o: dL/dy [s_local][hidden], from which the
 *          library forms dL/do = dy w_o^T (held in library device memory, s_local * Hq * head_dim elements, for
 *          the duration of the call) and dw_o = o^T dy (fp32 [Hq d][hidden], output, overwritten)
 *   dx [s_local][hidden] (output, overwritten), dw_qkv fp32 [hidden][(Hq + 2 Hkv) d] (output, overwritten: the sum
 *   over this rank's rows of x^T dqkv; a data-parallel caller all-reduces dw_qkv and dw_o).
 * x, w_qkv, w_o must be unchanged between the two calls, and w_o NULL in both or in neither.  fpdt_block_bwd may take
 * x = NULL when the forward offloaded the hidden state (fpdt_set_hidden_offload): it is then prefetched per chunk.  All pointers are device pointers; dtype FPDT_BF16 (x, w, dx
 * bf16) or FPDT_FP32.  Errors: as fpdt_attn_fwd/bwd; hidden * elem bytes % 16 != 0: FPDT_ERR_ARG; offload = 0 or a
 * residency budget: FPDT_ERR_UNSUPPORTED; fpdt_attn_bwd after fpdt_block_fwd (or the reverse): FPDT_ERR_STATE. */
int fpdt_block_fwd(fpdt_ctx* ctx, const void* x, const void* w_qkv, const void* w_o, void* o, float* lse, void* y,
                   int64_t s_local, int hidden,
                   int n_q_heads, int n_kv_heads, int head_dim, int causal, int64_t chunk_size, int world_size,
                   int dtype, int offload, float softmax_scale, void* stream);
int fpdt_block_bwd(fpdt_ctx* ctx, const void* x, const void* w_qkv, const void* w_o, const void* o, const void* dout,
                   void* dx, float* dw_qkv, float* dw_o, int64_t s_local, int hidden, int n_q_heads, int n_kv_heads, int head_dim, int causal,
                   int64_t chunk_size, int world_size, int dtype, int offload, float softmax_scale, void* stream);

/* Block-sparse attention (§5.6, Table "MFU at different attention sparsity": "only part of the tokens in
 * key and value will be fetched from the host memory, while the query will always be the entire sequence").
 *   keep: host array [n_chunks][n_chunks], row m = query chunk, column i = key chunk (GLOBAL chunk indices, chunk
 *   size = the calls' chunk_size); nonzero = the block is computed.  Entries i > m are ignored (causally invisible);
 *   diagonal blocks must be kept.  Copied; n_chunks = 0 (keep NULL) restores dense attention.
 * Applies to the following fpdt_attn_fwd calls (which check n_chunks == S / chunk_size: FPDT_ERR_ARG, a dropped
 * diagonal: FPDT_ERR_ARG, offload == 0: FPDT_ERR_UNSUPPORTED); fpdt_attn_bwd uses the plan of its forward.
 * Dropped blocks are neither fetched from host memory nor computed: key j is visible to query i iff j <= i and
 * keep[i / C][j / C].  Collective: every rank passes the same plan. */
int fpdt_set_sparsity(fpdt_ctx* ctx, const uint8_t* keep, int64_t n_chunks);

/* HBM residency budget (the paper offloads every chunk).  With
 * offload = 1, keep some chunks in device memory instead of the pinned host store:
 *   kv_chunks: key/value chunks i < kv_chunks (global chunk index) are never offloaded nor fetched.  The forward
 *     fetches chunk i once for every later query chunk, so the first chunks save the most host-to-device bytes.
 *   q_chunks: query-side chunks i >= u - q_chunks (u = S / chunk_size) keep q_i, dO_i and their fp32 dq partial on
 *     the device.  The backward fetches chunk i for every key chunk j <= i, so the last chunks save the most.
 * Values larger than u mean u.  0, 0 (the default) is the paper's schedule.  Applies to the following
 * fpdt_attn_fwd calls; fpdt_attn_bwd uses the setting of its forward.  Results equal the offloaded schedule's up to
 * the order of the dq reduce-adds.  Device memory: world_size 1 reads the caller's q, k, v rows of resident chunks
 * in place (they must stay valid and unmodified until fpdt_attn_bwd) plus C * hq * head_dim * 4 bytes per
 * query-side chunk; world_size > 1 keeps each resident head-layout chunk, C * (hq + 2 hkv) * head_dim * elem
 * bytes, plus C * 2 hq * head_dim * elem bytes per query-side chunk.  Errors: FPDT_ERR_ARG for negative counts. */
int fpdt_set_residency(fpdt_ctx* ctx, int64_t kv_chunks, int64_t q_chunks);

/* Backward loop order (offload = 1 only, offload = 0 always runs the paper's order).
 *   FPDT_BWD_KV_OUTER (default): the paper's order (fig:bw_db): outer loop over key/value chunks j, inner
 *     loop over query chunks i >= j; the fp32 dq partial of every query chunk round-trips the host store
 *     (C * hq * head_dim * 4 bytes each way per pair).
 *   FPDT_BWD_Q_OUTER (GQA-aware): outer loop over query chunks i, inner loop over key/value chunks j <= i.  q_i, dO_i
 *     are fetched once per outer iteration and dq_i stays on the device until it is final; the fp32 dK_j/dV_j
 *     partials round-trip the host store instead (C * 2 hkv * head_dim * 4 bytes each way per pair).  With GQA
 *     (2 hkv < hq) that moves fewer host bytes; dK_j, dV_j are final only after the last query chunk that attends
 *     key chunk j (the chunk-wise dK/dV hand-off of P:L365 is lost for the dense mask).  Its extra pinned store
 *     (u * C * 2 hkv * head_dim * 4 bytes) is allocated by the first Q-outer backward.
 *   FPDT_BWD_AUTO: per backward call, the order whose schedule moves fewer host bytes (given the sparsity plan and
 *     residency budget of the forward); ties take KV_OUTER.
 * Both orders compute the same sums; results agree up to the order of the fp32 additions.  Applies to the following
 * fpdt_attn_bwd calls; fpdt_get_stats reports the order the last backward ran.  Errors: FPDT_ERR_ARG for an
 * unknown order. */
enum { FPDT_BWD_KV_OUTER = 0, FPDT_BWD_Q_OUTER = 1, FPDT_BWD_AUTO = 2 };
int fpdt_set_bwd_order(fpdt_ctx* ctx, int order);

/* The host-link bytes (host-to-device plus device-to-host) that the offloaded backward's chunk loop moves per rank
 * in `order` (FPDT_BWD_KV_OUTER or FPDT_BWD_Q_OUTER), for the given shape, residency budget (kv_chunks, q_chunks)
 * and sparsity plan (keep [n_chunks][n_chunks] host array as fpdt_set_sparsity, or NULL = dense): the model
 * FPDT_BWD_AUTO compares.  Host-only arithmetic (no device, no context).  Errors: FPDT_ERR_ARG,
 * FPDT_ERR_DIVISIBILITY / FPDT_ERR_UNSUPPORTED as fpdt_attn_fwd. */
int fpdt_bwd_host_bytes(int order, int64_t s_local, int n_q_heads, int n_kv_heads, int head_dim, int64_t chunk_size,
                        int world_size, int dtype, int64_t kv_chunks, int64_t q_chunks, const uint8_t* keep,
                        int64_t n_chunks, int64_t* out);

/* Message of the last non-OK status returned on this thread ("" if none). */
const char* fpdt_last_error(void);

/* Global token index of rank `rank`'s local row `local_t` (rank-ordinal layout). */
int64_t fpdt_global_token(int64_t local_t, int64_t chunk_size, int world_size, int rank);

/* Hidden-state offload of the block calls ("the prefetching of the input hidden state h_0 will only be
 * synced in the projection backward").  When enabled (enable != 0) before fpdt_block_fwd, the forward copies each
 * chunk's input rows x_m [c][hidden] to a pinned host store once its projection has read them, and fpdt_block_bwd may
 * then be called with x = NULL: the backward prefetches x_j into a double-buffered device slot at the start of outer
 * iteration j, and only the projection backward of chunk j (dW += x_j^T dqkv_j) waits for it, so the caller need not
 * keep the hidden states on the device between the passes.  A non-NULL x in fpdt_block_bwd is used in place either
 * way.  Read by the next fpdt_block_fwd.  Returns FPDT_OK or FPDT_ERR_ARG. */
int fpdt_set_hidden_offload(fpdt_ctx* ctx, int enable);

/* Key/value fetch strategy of the offloaded schedule (fig:avg_time, whose
 * latency study compares "every GPU fetches its own chunk" with "one GPU fetches and scatters over NVLink"):
 *   FPDT_FETCH_PER_RANK (default, A): each rank offloads its head-layout key/value chunks to its own pinned store and
 *     fetches them back over its own host link;
 *   FPDT_FETCH_LEADER (B): rank 0 keeps every rank's key/value chunks in its pinned store: at the offload each rank
 *     sends its chunk to rank 0 (gather over NCCL / the in-process group), at each fetch rank 0 moves all p blocks
 *     host -> device and sends rank r its block (scatter).  One host link carries p x the key/value bytes; the others
 *     carry none.  Query-side chunks stay per rank.  The backward then runs the paper's KV-outer order.
 * Collective setting (all ranks equal); read by the next forward and used by its backward; ignored at world size 1
 * or offload = 0.  Returns FPDT_OK or FPDT_ERR_ARG. */
enum { FPDT_FETCH_PER_RANK = 0, FPDT_FETCH_LEADER = 1 };
int fpdt_set_fetch_strategy(fpdt_ctx* ctx, int strategy);

/* Debug check of the SPMD contract: when enabled (enable != 0) and world_size > 1, every fpdt_attn_* / fpdt_block_*
 * call first compares a 64-bit hash of its arguments and schedule options (shape, chunk, dtype, offload, hidden,
 * backward order, residency, sparsity plan) across the ranks -- an NCCL max-reduction plus a host sync, or the
 * in-process group -- and returns FPDT_ERR_ARG on every rank if they differ, instead of entering mismatched
 * all-to-alls.  Off by default (it synchronises).  NCCL initialisation and every NCCL call are bounded by
 * FPDT_NCCL_TIMEOUT_S seconds (environment, default 300): a rank that never joins makes fpdt_ctx_create return
 * FPDT_ERR_NCCL instead of hanging.  Returns FPDT_OK or FPDT_ERR_ARG (null ctx). */
int fpdt_set_debug_checks(fpdt_ctx* ctx, int enable);

/* Counters of the context since creation (diagnostics for tests and the bench). */
typedef struct fpdt_stats {
  int64_t bytes_h2d;          /* host -> device chunk fetches */
  int64_t bytes_d2h;          /* device -> host chunk offloads */
  int64_t bytes_a2a;          /* bytes sent to other ranks by the all-to-alls */
  int64_t kernel_launches;    /* kernels enqueued by the library (attention + support kernels) */
  int64_t attn_launches;      /* attention pair kernels only */
  int64_t fetch_slots_highwater; /* max fetched key/value chunk sets resident at once (<= 2) */
  int64_t host_arena_bytes;   /* pinned host store reserved */
  int64_t device_bytes;       /* library-owned device working set */
  int64_t bwd_order;          /* loop order of the last fpdt_attn_bwd (FPDT_BWD_KV_OUTER / FPDT_BWD_Q_OUTER) */
  int64_t host_dkv_bytes;     /* pinned store of the Q-outer backward's dK/dV partials (0 until first used) */
  int64_t stress_sleeps;      /* debug sleep kernels enqueued by the scheduler stress mode (env FPDT_STRESS_NS) */
  int64_t bytes_io_h2d;       /* caller rows uploaded by fpdt_attn_fwd_host / fpdt_attn_bwd_host */
  int64_t bytes_io_d2h;       /* caller rows downloaded by fpdt_attn_fwd_host / fpdt_attn_bwd_host */
} fpdt_stats;
int fpdt_get_stats(const fpdt_ctx* ctx, fpdt_stats* out);

/* Per-launch timing of the attention pair kernels (for bench.py's roofline): when enabled, the library
 * records a CUDA event pair around every attention kernel on the stream it is launched on.
 * fpdt_kernel_time synchronises on those events and returns the summed kernel milliseconds and launch
 * counts of forward and backward attention kernels since the last reset (reset != 0 clears them). */
int fpdt_set_kernel_timing(fpdt_ctx* ctx, int enable);
int fpdt_kernel_time(fpdt_ctx* ctx, double* fwd_ms, int64_t* fwd_launches, double* bwd_ms, int64_t* bwd_launches,
                     int reset);

/* Compute-stream stall accounting (SURVEY §8(a) stream/event skeleton): over the attention launches recorded since the
 * last reset of fpdt_kernel_time, the summed time between the end of one launch and the start of the next launch of
 * the same fpdt call on the same stream (*gap_ms), and the number of such gaps (*n_gaps).  A gap is time the
 * compute stream spent waiting for a chunk exchange, a host fetch or a small support kernel instead of running pair
 * kernels.  Synchronises on the recorded events; call it before fpdt_kernel_time(..., reset = 1).
 * Returns FPDT_OK, FPDT_ERR_ARG or FPDT_ERR_CUDA. */
int fpdt_kernel_gaps(fpdt_ctx* ctx, double* gap_ms, int64_t* n_gaps);

/* All-to-all timing (p > 1, with fpdt_set_kernel_timing on): CUDA events around every exchange on the comm stream
 * since the last reset of fpdt_kernel_time.  *total_ms = summed exchange time, *n = exchanges, *bytes = bytes sent to
 * other ranks by them (for bus GB/s = bytes / time), *first_ms / *last_ms (nullable) = the first and the last exchange
 * (the pipeline fill and drain).  Synchronises on the events; call before fpdt_kernel_time(reset=1).
 * Returns FPDT_OK, FPDT_ERR_ARG or FPDT_ERR_CUDA. */
int fpdt_exchange_time(fpdt_ctx* ctx, double* total_ms, int64_t* n, int64_t* bytes, double* first_ms,
                       double* last_ms);

#ifdef __cplusplus
}
#endif

#endif /* FPDT_H_ */
