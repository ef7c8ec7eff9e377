/*
 * flexprefill.h -- C ABI of libflexprefill.so, a B200 (sm_100a) implementation
 * of FlexPrefill sparse prefill attention (arXiv 2502.20766).
 *
 * Citations: P:n = line n of the paper source; A1..A26 = the
 * readings of silent/ambiguous passages, listed in DESIGN.md §3.
 *
 * The method (Alg. 1 "Sparse Attention") runs per attention head:
 *   (i)   pattern determination  (Alg. 2)            -> fp_plan
 *   (ii)  sparse index selection (Alg. 3 P:340-369 / Alg. 4 P:377-403,
 *         forced blocks and minimum budget P:451)                 -> fp_select
 *   (iii) y = A(Q, K, V, S)                  -> fp_sparse_attn
 * plus a same-library dense causal kernel (the speedup denominator)
 *                                                                 -> fp_dense_causal_attn
 *
 * Conventions (all entry points):
 *  - Causal, bf16. The plain entry points take batch 1 with Q and O
 *    [heads][seq_len][head_dim] and K, V [kv_heads][seq_len][head_dim],
 *    row-major, contiguous; the *_ex entry points take an fp_layout (batch >= 1,
 *    any 16-byte-multiple strides, e.g. the token-major [batch][seq][heads][d]
 *    of a model's QKV projection). Q head h uses KV head
 *    floor(h * kv_heads / heads) (GQA, contiguous groups; A15).
 *  - seq_len is any n >= 128; nb = ceil(n / 128) blocks, the last one ragged
 *    when n % 128 != 0 (reading A26).
 *  - Every tensor / workspace pointer is a DEVICE pointer unless the name
 *    says host. The caller owns all memory; the library never allocates device
 *    memory, keeps no per-call state, and only enqueues work ordered on `stream`
 *    (no host syncs; fp_plan at short lengths forks one branch onto an internal
 *    side stream, one per calling thread and device, and joins it back through
 *    events before returning), so
 *    fp_plan -> fp_select -> fp_sparse_attn is CUDA-graph capturable. Stages
 *    communicate through the workspace; data-dependent sizes stay on device.
 *  - Validation is synchronous and happens before anything is enqueued; an
 *    invalid call enqueues nothing and returns a non-zero fp_status:
 *      FP_ERR_NULL      a required pointer is NULL
 *      FP_ERR_SHAPE     heads % kv_heads != 0, seq_len < 128, head_dim != 128,
 *                       block_size not 64 or 128 (128 is the
 *                       B200 tile, 64 the paper's alternative, A27), more than
 *                       8192 blocks (seq_len > 2^20 at b = 128, 2^19 at b = 64),
 *                       an fp_layout with batch < 1 or a stride < 128 elements
 *      FP_ERR_RANGE     gamma <= 0 or NaN; tau outside [0,1] or NaN; min_budget < 0
 *                       (gamma >= 1 is allowed and selects every causal block, A7)
 *      FP_ERR_ALIGN     a tensor pointer is not 16-byte aligned, or an fp_layout
 *                       stride is not a multiple of 8 elements (TMA requirement)
 *      FP_ERR_WORKSPACE ws_bytes < fp_workspace_bytes(...)
 *      FP_ERR_DEVICE    the current device is not compute capability 10.0
 *      FP_ERR_CUDA      a launch failed; fp_last_cuda_error() has the cudaError_t
 *    Asynchronous faults surface at the caller's next synchronisation.
 *    Outputs are undefined after any error.
 */
#ifndef FLEXPREFILL_H_
#define FLEXPREFILL_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FP_OK = 0,
  FP_ERR_NULL = 1,
  FP_ERR_SHAPE = 2,
  FP_ERR_RANGE = 3,
  FP_ERR_ALIGN = 4,
  FP_ERR_WORKSPACE = 5,
  FP_ERR_DEVICE = 6,
  FP_ERR_CUDA = 7
} fp_status;

/* Per-head selection statistics (fp_select). k_v / k_s: number of selected
 * vertical / slash lines (K_v, K_s of Alg. 3; block columns /
 * diagonal groups with vs_mode 1), 0 for QA heads; k_qa: K of Alg. 4 (
 * summed over rows with qa_mode 1), 0 for VS heads; nnz_blocks: computed
 * (q-block, k-block) pairs after forced blocks and the budgets; budget_added /
 * budget_removed: blocks added by the minimum budget (A12) / removed by
 * the maximum budget (A23); mass_*: achieved estimated mass of
 * the selected lines/blocks (fixed-point sum). */
typedef struct {
  int32_t k_v, k_s, k_qa, nnz_blocks, budget_added, pattern, budget_removed;
  double mass_v, mass_s, mass_qa;
} fp_select_stats;

/* Selection variants (fp_select_ex).
 *   vs_mode     0: Vertical-Slash lines selected at element level and rasterised
 *                  (Alg. 3 as written, reading A10/R1; default)
 *               1: block-pooled lines (f1, reading A24/R2): key-block columns by
 *                  topmass(a_hat), slash offset groups [D b, (D+1) b) by
 *                  topmass(As); a selected group marks block diagonals D, D+1
 *   qa_mode     0: flatten and normalise the pooled map, one topmass (Alg. 4)
 *               1: per query block ("wo/ flatten", A25)
 *   max_budget  tokens per query-block row, 0 = off (A23); rows
 *               above ceil(max_budget / 128) blocks keep their forced blocks
 *               and the best remaining blocks by row score */
typedef struct {
  int32_t vs_mode, qa_mode, max_budget;
} fp_select_options;

/* Tensor layout for the *_ex entry points (next row f3). Element (batch b,
 * head h, position i, dim c) of a tensor lives at
 *     base + b * stride[0] + h * stride[1] + i * stride[2] + c
 * (strides in bf16 ELEMENTS, each a multiple of 8 and >= 128; stride[0] is
 * ignored when batch == 1). K/V head indices run over kv_heads per batch
 * element, Q/O over heads. With a layout, every per-head array (pattern, jsd,
 * row_ptr, col_idx, stats, the workspace) covers batch * heads flattened heads
 * hh = b * heads + h: size the workspace with
 * fp_workspace_bytes(batch * heads, batch * kv_heads, ...) and call fp_select
 * with (batch * heads, batch * kv_heads). The caller guarantees that distinct
 * O rows do not overlap. */
typedef struct {
  int32_t batch;
  int64_t q_stride[3], k_stride[3], v_stride[3], o_stride[3];
} fp_layout;

/* Contiguous [batch][heads][seq][128] (head-major; the plain entry points'
 * layout) and [batch][seq][heads][128] (token-major, as produced by a QKV
 * projection) layouts; host-only helpers, no device work. */
fp_status fp_layout_bhsd(int batch, int heads, int kv_heads, int seq_len, fp_layout* out);
fp_status fp_layout_bshd(int batch, int heads, int kv_heads, int seq_len, fp_layout* out);

/* Device pointers into a workspace filled by fp_plan / fp_select (for tests
 * and stage-wise parity; read-only for the caller). Shapes, n = seq_len,
 * nb = ceil(n / 128):
 *   a_v, a_s   fp32 [heads][n]       vertical / slash line scores
 *   a_hat      fp32 [heads][nb]      true block distribution (A2)
 *   a_bar      fp32 [heads][nb]      estimated block distribution
 *   k_bar      fp32 [kv_heads][nb][128]  avg-pooled keys
 *   q_bar      fp32 [heads][nb][128]     avg-pooled queries (QA heads only)
 *   A_bar      fp32 [heads][nb(nb+1)/2]  flattened normalised pooled map
 *              (row-major over qb, kb <= qb; QA heads only)
 *   As         fp32 [heads][nb]      slash mass per block diagonal (A12)
 *   sel_v, sel_s  int32 [heads][n]   selected vertical / slash lines, ascending
 *   sel_qa     int32 [heads][nb(nb+1)/2]  selected flat QA indices, ascending
 *   sel_count  int32 [heads][3]      (K_v, K_s, K_qa)
 *   row_nnz_pre int32 [heads][nb]    blocks per row before the minimum budget
 */
typedef struct {
  const float *a_v, *a_s, *a_hat, *a_bar, *k_bar, *q_bar, *A_bar, *As;
  const int32_t *sel_v, *sel_s, *sel_qa, *sel_count, *row_nnz_pre;
  /* attention scheduler of the last fp_sparse_attn / fp_dense_causal_attn with
   * this ws (int32 [2]): [0] work counter, [1] number of work items (head,
   * query-block pair) that were redone with a row-max pass on every tile
   * because a score exceeded its row's reference by more than 64 (log2) */
  const int32_t *attn_sched;
} fp_debug_ptrs;

/* Bytes of device workspace needed by fp_plan/fp_select/fp_sparse_attn for
 * this shape (0 if the shape is invalid). */
size_t fp_workspace_bytes(int heads, int kv_heads, int seq_len, int head_dim, int block_size);

/* Per-head capacity (int32 entries) of col_idx: nb * (nb + 1) / 2, nb = ceil(n / 128). */
size_t fp_col_idx_capacity(int seq_len, int block_size);

/* Stage (i): Alg. 2 for every head, plus the Vertical-Slash line scores of
 * Alg. 3 from the same representative attention and, for Query-Aware
 * heads, the pooled map of Alg. 4 (it is the last step that reads Q).
 *   q, k      device bf16, layouts above (only the last 128 rows of each Q head
 *             and all of K are read, plus all of Q for Query-Aware heads)
 *   tau       pattern threshold, [0, 1]; QA iff D_JS < tau
 *   ws        device workspace of ws_bytes >= fp_workspace_bytes(...)
 *   pattern   device int32 [heads] out: 1 = query_specific (QA), 0 = vertical_slash
 *   jsd       device fp32 [heads] out: D_JS = sqrt(JSD(a_bar || a_hat)), base 2 (A1)
 */
fp_status fp_plan(const void* q, const void* k, int heads, int kv_heads, int seq_len, int head_dim,
                  int block_size, float tau, void* ws, size_t ws_bytes, int32_t* pattern,
                  float* jsd, void* stream);

/* fp_plan over an fp_layout (NULL = the plain layout, batch 1); heads and
 * kv_heads are per batch element, pattern / jsd are [batch * heads]. */
fp_status fp_plan_ex(const void* q, const void* k, int heads, int kv_heads, int seq_len,
                     int head_dim, int block_size, const fp_layout* layout, float tau, void* ws,
                     size_t ws_bytes, int32_t* pattern, float* jsd, void* stream);

/* Stage (ii): cumulative-attention selection for every head, then
 * forced first/diagonal key blocks (A11) and the minimum budget
 * (min_budget tokens per query-block row, 0 = off; A12). Reads the workspace
 * written by fp_plan on the same stream.
 *   gamma     cumulative threshold (0, 1); >= 1 selects all (A7)
 *   row_ptr   device int32 [heads][nb + 1] out: per-head CSR row offsets
 *   col_idx   device int32 [heads][fp_col_idx_capacity] out: key blocks of each
 *             query-block row, ascending (the diagonal block is last)
 *   stats     device fp_select_stats [heads] out, or NULL
 */
fp_status fp_select(int heads, int kv_heads, int seq_len, int head_dim, int block_size, float gamma,
                    int min_budget, void* ws, size_t ws_bytes, int32_t* row_ptr, int32_t* col_idx,
                    fp_select_stats* stats, void* stream);

/* fp_select with the selection variants of fp_select_options (NULL = the
 * defaults, identical to fp_select). FP_ERR_RANGE for a mode outside {0, 1},
 * max_budget < 0, or 0 < max_budget < min_budget (the cap is applied after the
 * floor, A23, and may not undercut it). Token budgets are converted to blocks
 * in 64-bit arithmetic and clamped to nb. */
fp_status fp_select_ex(int heads, int kv_heads, int seq_len, int head_dim, int block_size,
                       float gamma, int min_budget, const fp_select_options* opt, void* ws,
                       size_t ws_bytes, int32_t* row_ptr, int32_t* col_idx, fp_select_stats* stats,
                       void* stream);

/* Stage (iii): y = softmax((Q K^T + M_S) / sqrt(d)) V over exactly the blocks
 * in the CSR (intersected with j <= i), online softmax, GQA.
 *   o         device bf16 [heads][seq_len][128] out
 *   row_ptr, col_idx  the CSR from fp_select (or any CSR with kb <= qb, each row
 *             containing its diagonal block qb, kb ascending)
 *   ws        optional scheduler scratch: NULL, or a workspace of this shape
 *             (16-B aligned, ws_bytes >= fp_workspace_bytes(...), else
 *             FP_ERR_ALIGN / FP_ERR_WORKSPACE); the output does not depend on it
 */
fp_status fp_sparse_attn(const void* q, const void* k, const void* v, void* o, int heads,
                         int kv_heads, int seq_len, int head_dim, int block_size,
                         const int32_t* row_ptr, const int32_t* col_idx, void* ws, size_t ws_bytes,
                         void* stream);

/* fp_sparse_attn over an fp_layout (NULL = plain); row_ptr / col_idx cover the
 * batch * heads flattened heads. O rows past seq_len are never written. */
fp_status fp_sparse_attn_ex(const void* q, const void* k, const void* v, void* o, int heads,
                            int kv_heads, int seq_len, int head_dim, int block_size,
                            const fp_layout* layout, const int32_t* row_ptr,
                            const int32_t* col_idx, void* ws, size_t ws_bytes, void* stream);

/* Next row f4: fp_sparse_attn_ex whose epilogue also stores
 * every output row into n_peer further buffers -- the output exchange of the
 * head-partitioned multi-GPU layer (§8(e)) fused into the attention kernel.
 * Each peer buffer is another rank's output mapped into this process (CUDA IPC
 * / torch symmetric memory over NVLink), so a rank's heads reach every rank
 * tile by tile while its later tiles compute, instead of a separate
 * all-gather or broadcast after the kernel.
 *   peer_o   DEVICE array [n_peer] of device pointers (8-B aligned array);
 *            each buffer has o's layout (plain [heads][seq_len][128], or
 *            layout->o strides) and receives exactly the rows written to o
 *   n_peer   0..FP_MAX_PEERS (0: identical to fp_sparse_attn_ex)
 * Completion on the peers is the caller's: a cross-rank barrier ordered after
 * the kernel (e.g. the symmetric-memory barrier on the same stream) before a
 * peer reads its buffer. Errors: FP_ERR_RANGE n_peer < 0 or > FP_MAX_PEERS;
 * FP_ERR_NULL peer_o NULL with n_peer > 0; FP_ERR_ALIGN peer_o not 8-B
 * aligned (the pointer values are device data and are not checked). Both
 * block sizes (64 runs the same kernel on coarse 128 x 128 tiles). */
#define FP_MAX_PEERS 8
fp_status fp_sparse_attn_peers(const void* q, const void* k, const void* v, void* o,
                               const void* const* peer_o, int n_peer, int heads, int kv_heads,
                               int seq_len, int head_dim, int block_size, const fp_layout* layout,
                               const int32_t* row_ptr, const int32_t* col_idx, void* ws,
                               size_t ws_bytes, void* stream);

/* Dense causal attention A(Q, K, V) with the same kernel (every kb <= qb). */
fp_status fp_dense_causal_attn(const void* q, const void* k, const void* v, void* o, int heads,
                               int kv_heads, int seq_len, int head_dim, int block_size,
                               void* ws, size_t ws_bytes, void* stream);
fp_status fp_dense_causal_attn_ex(const void* q, const void* k, const void* v, void* o, int heads,
                                  int kv_heads, int seq_len, int head_dim, int block_size,
                                  const fp_layout* layout, void* ws, size_t ws_bytes,
                                  void* stream);

/* The whole layer (Alg. 1) from HOST buffers: copies q/k/v host->device into
 * the caller's device buffers (d_q, d_k, d_v), runs plan/select/attn, and
 * copies the output back to o_host. Pipelined per KV group: the host->device
 * copy of group c+1 and the device->host copy of group c-1 overlap the compute
 * of group c on internal streams, joined back into `stream` before return
 * (ws must hold fp_workspace_bytes of the whole layer; pattern, jsd, row_ptr,
 * col_idx are the full-layer arrays). Overlap needs pinned host buffers.
 * The results are bitwise those of fp_plan / fp_select / fp_sparse_attn on the
 * whole layer. Every argument (pointers, 16-B alignment of the device buffers
 * and ws, 4-B alignment of pattern / jsd / row_ptr / col_idx, shape, ranges,
 * workspace size, device) is validated before the first copy is enqueued.
 * The internal streams and events are created once per (calling thread,
 * device) and reused; calls from different threads never share them. */
fp_status fp_layer_host(const void* q_host, const void* k_host, const void* v_host, void* o_host,
                        void* d_q, void* d_k, void* d_v, void* d_o, int heads, int kv_heads,
                        int seq_len, int head_dim, int block_size, float gamma, float tau,
                        int min_budget, void* ws, size_t ws_bytes, int32_t* pattern, float* jsd,
                        int32_t* row_ptr, int32_t* col_idx, void* stream);

/* Fill *out with device pointers into ws (no device work). */
fp_status fp_debug_view(const void* ws, int heads, int kv_heads, int seq_len, int head_dim,
                        int block_size, fp_debug_ptrs* out);

/* Number of kernels fp_plan / fp_select / fp_sparse_attn enqueue per call. */
int fp_kernels_per_layer(void);

const char* fp_status_string(fp_status s);
int fp_last_cuda_error(void);

#ifdef __cplusplus
}
#endif
#endif /* FLEXPREFILL_H_ */
