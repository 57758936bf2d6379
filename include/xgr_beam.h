/*
 * xgr_beam.h -- C ABI of the B200-native xBeam decode-step selection library.
 *
 * The operation (PAPER.md = /root/reference/PAPER.md, line numbers L<n>):
 *   Per request and decode step t = 1..ND, the live beams' next-token logits are filtered to the
 *   legal children of each beam's prefix in the pre-built item trie ("valid path constraint",
 *   L361, section 6.1; dense/sparse mask storage, L371), normalised by an fp32 log-softmax over
 *   the legal tokens, added to the running beam score ("accumulates log-probabilities", L376,
 *   section 6.2) and the global Top-BW (parent beam, token) pairs are kept (L154-156, section
 *   2.2.2; L356, section 6), with early termination against a running BW-th threshold (L376-385,
 *   section 6.2) and fixed, reused beam structures (L392, section 6.3). After ND steps the TID
 *   tuples are the item IDs (L309, section 5).
 *   Exact result (readings R1-R21): the first min(BW, #legal) candidates under
 *   (S_b + x_{b,v} - LSE_{u in L_b} x_{b,u}) descending, ties to the lower flat index b*V + v.
 *
 * Sequencing: xgr_beam_init -> xgr_mask_build (once; the trie is immutable and reused) ->
 *   { exactly nd x xgr_beam_step -> xgr_beam_finalize } repeated per batch -> xgr_beam_destroy.
 *   Violations return XGR_ERR_SEQUENCE.
 *
 * Memory / ownership: the ctx owns the device trie and a fixed workspace sized at init for
 *   max_batch requests ("does not allocate entirely new data structure"):
 *   xgr_beam_step and xgr_beam_finalize never allocate. Pointers passed in are borrowed; device
 *   inputs must stay valid until the stream work completes.
 *
 * Streams: `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   xgr_beam_step validates on the host and only enqueues work: no host synchronisation, no
 *   allocation, so it can be captured in a CUDA graph.
 *
 * Errors: every call returns xgr_status; xgr_last_error() gives a thread-local message. Nothing
 *   aborts or exits. Device-detected NaN/+Inf logits at legal positions (or a row whose legal
 *   logits are all -Inf) set a sticky per-request flag reported by xgr_beam_request_status and
 *   by xgr_beam_finalize(..., outputs_on_device = 0) as XGR_ERR_NONFINITE; that request's output
 *   is undefined, other requests are unaffected. A legal -Inf logit is a zero-probability token.
 *
 * Threading: a ctx is single-stream and not thread-safe; distinct ctxs are independent.
 */
#ifndef XGR_BEAM_H
#define XGR_BEAM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define XGR_ABI_VERSION 2   /* 2: xgr_config allocator hooks, xgr_beam_step_host */

typedef struct xgr_ctx xgr_ctx; /* opaque; one per in-flight batch */

typedef enum {
  XGR_OK = 0,
  XGR_ERR_INVALID_ARG = 1, /* null pointer, size out of range, bad config */
  XGR_ERR_UNSUPPORTED = 2, /* valid but not implemented (0 < top_k < BW with nranks > 1, ...) */
  XGR_ERR_TOKEN_RANGE = 3, /* mask_build: a token < 0 or >= V */
  XGR_ERR_EMPTY_VOCAB = 4, /* mask_build: zero items (no beam could live) */
  XGR_ERR_SEQUENCE = 5,    /* call out of order */
  XGR_ERR_ALIGNMENT = 6,   /* logits not 16-byte aligned or ld % 4 != 0 */
  XGR_ERR_NONFINITE = 7,   /* a request saw NaN/+Inf at a legal position */
  XGR_ERR_CUDA = 8,
  XGR_ERR_NCCL = 9,
  XGR_ERR_OOM = 10
} xgr_status;

/* config.flags */
#define XGR_CFG_NO_PRUNE 0x1u /* theta = -inf: every legal candidate survives (test/ablation) */
#define XGR_CFG_COUNTERS 0x2u /* accumulate device counters (xgr_beam_counters) */
#define XGR_CFG_NO_SPARSE_KERNEL 0x4u /* route every step through the dense-step kernels */
#define XGR_CFG_TIMING 0x8u /* CUDA events around the dense-route streaming kernel           */
#define XGR_CFG_PAPER_HEAP 0x10u /* baseline: dense steps select with the paper's per-beam Top-K
                                    lists + sequential global min-heap instead of
                                    theta pruning; same results; V <= 16384, allocates
                                    max_batch * BW * K * 8 bytes of lists at init */

typedef struct {
  int32_t vocab;      /* V: tokens per level, 1..65536                                   */
  int32_t nd;         /* ND: tokens per item (trie depth), 1..8; nd*ceil(log2 V) <= 64    */
  int32_t beam_width; /* BW, 1..1024                                                      */
  int32_t top_k;      /* per-beam K: each beam keeps its K best candidates
                         (score desc, token asc) before the global Top-BW. 0 or >= BW: none.
                         0 < K < BW needs V <= 16384 and nranks == 1 (else UNSUPPORTED)    */
  int32_t max_batch;  /* max requests per step call, >= 1                                 */
  int32_t device;     /* CUDA device ordinal                                             */
  int32_t nranks;     /* codebook shards G >= 1 (1: no shard). G > 1: V % G == 0 and       */
                      /*   V/G a multiple of 128, <= 8192; use the xgr_shard_* calls      */
  int32_t rank;       /* this shard, 0 <= rank < nranks: columns [rank*V/G, (rank+1)*V/G) */
  const void* nccl_id;/* must be NULL: the caller performs the two all-gathers            */
  int32_t survivor_cap; /* per-request survivor buffer (keys); 0 = min(32*BW, 16384)      */
  int32_t theta_rows;   /* rows 0..theta_rows-1 seed the threshold; 0 = default (8)       */
  uint32_t flags;       /* XGR_CFG_*                                                      */
  /* Device-memory hooks, e.g. a framework's caching allocator; both or neither
   * (NULL, NULL: cudaMalloc / cudaFree). dev_alloc(bytes, alloc_user) returns >= 16-byte aligned
   * device memory on cfg.device or NULL (-> XGR_ERR_OOM); dev_free(ptr, alloc_user) takes it back.
   * Called only from xgr_beam_init, xgr_mask_build, the support calls that need scratch
   * (xgr_mask_children, xgr_beam_account), a growing xgr_beam_step_host and xgr_beam_destroy
   * (which synchronises the device first) -- never from a step, so steps stay graph-capturable. */
  void* (*dev_alloc)(size_t bytes, void* alloc_user);
  void (*dev_free)(void* ptr, void* alloc_user);
  void* alloc_user;
  int32_t reserved[5];  /* must be zero                                                   */
} xgr_config;

/* Create a context: validates cfg, selects the device, allocates the fixed beam workspace
 * (O(max_batch * BW * (nd + survivor_cap)) bytes). *out is NULL on failure. */
xgr_status xgr_beam_init(const xgr_config* cfg, xgr_ctx** out);

/* Build the device trie of legal items ("pre-built valid item vocabulary", PAPER.md L361;
 * "pre-generated during model loading", L371). items: HOST int32 [n_items][nd], any order;
 * duplicates are removed silently. Per level: nodes = distinct prefixes numbered in
 * lexicographic order, first_child offsets, each node's token label, and for nodes with
 * >= V/16 children a dense V-bit bitmap with a rank directory (otherwise the sorted labels of
 * its children act as the sparse list). Leaf id at level nd = the item's rank in the sorted,
 * de-duplicated list. Synchronous: returns after the build completed on `stream`.
 * Errors: XGR_ERR_TOKEN_RANGE, XGR_ERR_EMPTY_VOCAB, XGR_ERR_INVALID_ARG (n_items >= 2^32),
 * XGR_ERR_SEQUENCE (already built), XGR_ERR_OOM. */
xgr_status xgr_mask_build(xgr_ctx* ctx, const int32_t* items, int64_t n_items, void* stream);

/* One decode step for `batch` requests (step t = number of previous steps + 1).
 * logits: DEVICE fp32 [batch][rows][ld], request r's row b at logits + (r*rows + b)*ld; row b is
 *   the next-token distribution of live slot b of the previous step (slot 0 = the root at t=1).
 *   Rows >= n_live and columns outside the legal set are never read. 16-byte aligned, ld % 4 == 0,
 *   ld >= V. At t = 1 rows >= 1 (only row 0 is read); at t > 1 rows >= BW.
 * batch: 1..max_batch, fixed by the first step of a batch.
 * Route (no effect on results): a step whose requests' legal candidates fit on chip (rows x max
 * children of the level <= 16384) runs the sparse kernel; otherwise the dense streaming path --
 * one CTA per row up to 8192 columns, 2-CTA thread-block clusters for 16384, one CTA per row in
 * two passes for 32768 and 65536 (V % (128 C) == 0 for C = V/8192 rounded up to a power of two;
 * other V > 16384 return XGR_ERR_UNSUPPORTED on a dense step). A level that mixes dense and sparse
 * nodes takes both routes, per request (the previous step's commit counted its candidates).
 * Enqueues only (no sync, no allocation); graph-capturable. */
xgr_status xgr_beam_step(xgr_ctx* ctx, int32_t batch, const float* logits, int32_t rows,
                         int64_t ld, void* stream);

/* Logit element types for xgr_beam_step_ex. */
#define XGR_DTYPE_F32 0
#define XGR_DTYPE_BF16 1

/* xgr_beam_step with the logits' element type given (PAPER.md L361, L376
 * leave the dtype open). XGR_DTYPE_BF16: DEVICE bf16 [batch][rows][ld], 16-byte aligned rows
 * (ld % 8 == 0); every value is widened exactly to fp32 and the step computes in fp32 as for
 * XGR_DTYPE_F32 (the oracle widens the same values). bf16 dense steps need the streaming kernels
 * (V % 128 == 0; V > 8192 in column-split clusters); otherwise XGR_ERR_UNSUPPORTED, as for any
 * other dtype or a sharded ctx. XGR_DTYPE_F32 is exactly xgr_beam_step. */
xgr_status xgr_beam_step_ex(xgr_ctx* ctx, int32_t batch, const void* logits, int32_t dtype,
                            int32_t rows, int64_t ld, void* stream);

/* xgr_beam_step_ex with the logits in HOST memory (the end-to-end path: PAPER.md L376, logits
 * arrive from the model every step): the call copies host_logits [batch][rows][ld] (dtype
 * elements, ld >= V) into a ctx-owned device staging buffer with cudaMemcpyAsync on `stream`,
 * then enqueues the step on it. Use page-locked host memory for an asynchronous copy (pageable
 * memory makes the copy synchronous). The staging buffer holds one step: the next
 * xgr_beam_step_host on the same stream is ordered after this step's kernels. The first call, and
 * any call needing a larger buffer, synchronises `stream` and allocates (not graph-capturable
 * then); later calls only enqueue. Errors: as xgr_beam_step_ex; XGR_ERR_OOM. */
xgr_status xgr_beam_step_host(xgr_ctx* ctx, int32_t batch, const void* host_logits, int32_t dtype,
                              int32_t rows, int64_t ld, void* stream);

/* After exactly nd steps: item tuples of the final beams, in slot order (score descending).
 * The last step's kernels already wrote them into ctx-owned device buffers (fused finalize);
 * this call copies them out (device->device or device->host) and resets the ctx. With
 * outputs_on_device != 0 and all output pointers NULL it only resets: read the results in place
 * through xgr_beam_outputs (valid until the next batch's last step).
 * tokens [batch][BW][nd] int32, item_rank [batch][BW] int64 (rank in the sorted de-duplicated
 * item list), score [batch][BW] fp32 (sum of the per-step log-probabilities), n_live [batch].
 * Dead slots (n_live <= j < BW): tokens/item_rank -1, score -inf. Any output pointer may be NULL.
 * outputs_on_device != 0: pointers are device memory, call only enqueues.
 * outputs_on_device == 0: host memory; synchronises `stream`; returns XGR_ERR_NONFINITE if a
 * request was flagged. Resets the ctx for the next batch (the trie is kept). */
xgr_status xgr_beam_finalize(xgr_ctx* ctx, int32_t* tokens, int64_t* item_rank, float* score,
                             int32_t* n_live, int32_t outputs_on_device, void* stream);

xgr_status xgr_beam_destroy(xgr_ctx* ctx);
const char* xgr_last_error(void);
int32_t xgr_abi_version(void);

/* ---- support calls (tests, parity, accounting) ---------------------------------------- */

/* Device pointers to the latest step's beam state, each [batch][BW] (node ids are the trie
 * node of each slot's prefix at level t). Valid until the next step/finalize. */
xgr_status xgr_beam_view(const xgr_ctx* ctx, const int32_t** parent, const int32_t** token,
                         const float** score, const int32_t** n_live, const uint32_t** node);

/* Device pointers to step t's (1-based) parent/token history, each [batch][BW]. */
xgr_status xgr_beam_history(const xgr_ctx* ctx, int32_t step, const int32_t** parent,
                            const int32_t** token);

/* Per-request sticky status bits of the current batch, copied to HOST flags[batch]
 * (bit 0: non-finite logit, bit 1: survivor overflow -> exact fallback taken). Synchronous. */
xgr_status xgr_beam_request_status(const xgr_ctx* ctx, uint32_t* flags, int32_t batch,
                                   void* stream);

/* Legal children of n HOST prefixes [n][depth] (depth < nd), read from the representation the
 * step kernels use (dense bitmap or sparse labels). counts[i] = number of children (-1 if the
 * prefix is not in the trie, -2 if the node's rank/label views disagree); tokens[i][0..cap) the
 * first min(count, cap) children ascending. HOST outputs; synchronous. */
xgr_status xgr_mask_children(const xgr_ctx* ctx, const int32_t* prefixes, int32_t depth,
                             int64_t n, int32_t* counts, int32_t* tokens, int64_t cap,
                             void* stream);

/* Trie shape: n_items (after de-dup), nodes_per_level[nd+1], dense_per_level[nd+1] (levels
 * 0..nd; leaves are never dense), max_children_per_level[nd+1], device bytes held by the trie.
 * Any pointer may be NULL. */
xgr_status xgr_mask_info(const xgr_ctx* ctx, int64_t* n_items, int64_t* nodes_per_level,
                         int64_t* dense_per_level, int64_t* max_children_per_level,
                         int64_t* trie_bytes);

/* Device counters accumulated since the last call (needs XGR_CFG_COUNTERS), copied to HOST
 * out[XGR_NUM_COUNTERS], then zeroed. Synchronous. */
#define XGR_NUM_COUNTERS 8
#define XGR_CNT_ROWS_READ 0      /* rows whose logits were streamed by the dense-step pass   */
#define XGR_CNT_ROWS_SKIP_PRE 1  /* rows skipped before reading (S_b < theta)               */
#define XGR_CNT_ROWS_SKIP_POST 2 /* rows read but emitting nothing (S_b - ln Z_b < theta)   */
#define XGR_CNT_LEGAL 3          /* legal candidates of the rows read                       */
#define XGR_CNT_SURVIVORS 4      /* candidates emitted to the per-request survivor buffers  */
#define XGR_CNT_OVERFLOW 5       /* requests that took the exact overflow fallback          */
#define XGR_CNT_SPARSE_CANDS 6   /* candidates handled by the sparse-step kernel            */
#define XGR_CNT_DENSE_STEPS 7    /* (request, step) pairs run through the dense-step path   */
xgr_status xgr_beam_counters(xgr_ctx* ctx, uint64_t* out, void* stream);

/* Algorithmic HBM bytes of the LAST step: over live rows b with
 * S_b >= theta* (theta* = the BW-th selected score of that request): 32 B per 32-byte logit
 * sector holding >= 1 legal token, plus the mask bytes of the distinct dense nodes touched
 * (V/8 each) or 4 + 2|L| per sparse row, plus 16 B of state per row. Also the "full" bytes
 * (every live row, whole V). Host outputs; synchronous; not for the timed path. */
xgr_status xgr_beam_account(xgr_ctx* ctx, int64_t* alg_bytes, int64_t* full_bytes,
                            int64_t* legal_candidates, void* stream);

/* ---- codebook shard (nranks = G > 1) ---------------------------------------------
 * For vocabularies too large for one GPU, G ranks each hold the columns [rank*V/G, (rank+1)*V/G)
 * of every logits row, and the full trie (mask_build with the full item list on every rank).
 * A step runs in three phases around two all-gathers that the caller performs (NCCL through
 * torch.distributed; a plain copy when all ranks live in one process):
 *   1. xgr_shard_stats: per live row the local (m, Z) over this rank's legal tokens
 *      (m = -inf, Z = 0 when the row has none). *stats: device float pairs [batch][BW][2].
 *   2. all-gather the stats of every rank, rank-major: gstats [G][batch][BW][2].
 *   3. xgr_shard_select: global lse per row = fixed rank-order combine of the G pairs (identical
 *      on every rank, R20); theta-pruned local top-BW of this rank's candidates.
 *      *recs: device uint64 keys [batch][BW], sorted descending and 0-padded (no real key is 0),
 *      *rec_n: device int32 [batch] (the count of nonzero keys).
 *   4. all-gather the records: grecs [G][batch][BW] (and, optionally, grec_n [G][batch]).
 *   5. xgr_shard_merge: global top-BW of the union, committed identically on every rank.
 *      grec_n may be NULL: the merge then counts each rank's nonzero keys itself, so a step needs
 *      only two collectives (stats, records).
 * xgr_beam_init rejects (XGR_ERR_UNSUPPORTED) an nranks x beam_width the merge's shared memory
 * cannot hold on the device.
 * logits: this rank's columns only, [batch][rows][ld] with ld >= V/G; it must stay valid until
 * xgr_shard_select has completed on the stream. xgr_beam_step returns XGR_ERR_SEQUENCE on a
 * sharded ctx; finalize / view / history are unchanged. All calls only enqueue. */
xgr_status xgr_shard_stats(xgr_ctx* ctx, int32_t batch, const float* logits, int32_t rows, int64_t ld,
                           void* stream, const float** stats);
xgr_status xgr_shard_select(xgr_ctx* ctx, const float* gstats, void* stream, const uint64_t** recs,
                            const int32_t** rec_n);
xgr_status xgr_shard_merge(xgr_ctx* ctx, const uint64_t* grecs, const int32_t* grec_n, void* stream);

/* Device pointers to the ctx-owned final outputs (same layouts as xgr_beam_finalize): written by
 * the last step of every batch, valid until the next batch's last step. */
xgr_status xgr_beam_outputs(const xgr_ctx* ctx, const int32_t** tokens, const int64_t** item_rank,
                            const float** score, const int32_t** n_live);

/* Host-side count of the kernels this ctx has launched since init (step and finalize). */
int64_t xgr_beam_launch_count(const xgr_ctx* ctx);

/* Durations (ms, CUDA events on the launch stream) of the dense-route streaming kernel (k_main)
 * of every dense step since the last call, oldest first, with the step index of each; needs
 * XGR_CFG_TIMING. Writes min(recorded, cap) entries and *n; synchronises on the events. */
xgr_status xgr_beam_kernel_times(xgr_ctx* ctx, float* ms, int32_t* step, int32_t cap, int32_t* n);

/* ---- LM-head fusion at sparse steps (at the last steps each
 * row has only a few legal tokens). Instead of logits, the step takes the decoder's final hidden
 * states and the LM-head weight and computes only the legal tokens' logits
 *   x[b][v] = sum_{k < d} hidden[b][k] * head[v][k]  (+ bias[v] when bias != NULL)
 * (fp32 FMAs over bf16 inputs, a fixed order), then selects exactly as xgr_beam_step on those
 * values. hidden: DEVICE bf16 [batch][rows][ldh], row b of request r at hidden + (r*rows + b)*ldh
 * (ldh >= d, ldh % 8 == 0, 16-byte aligned); head: DEVICE bf16 [V][ldw] (ldw >= d, ldw % 8 == 0);
 * bias: DEVICE fp32 [V] or NULL; d % 8 == 0. Only for a step after the root that takes the sparse
 * route (xgr_beam_next_route == 1); otherwise XGR_ERR_UNSUPPORTED (produce logits with a GEMM and
 * call xgr_beam_step). Enqueues only; uses a ctx-owned buffer of max_batch * 16384 floats. */
xgr_status xgr_beam_step_head(xgr_ctx* ctx, int32_t batch, const void* hidden, int32_t rows, int64_t ldh,
                              const void* head, int64_t ldw, const float* bias, int32_t d, void* stream);

/* *sparse = 1 if the next step takes the sparse route (every request's legal candidates fit on
 * chip: rows x max children of the level <= 16384), 0 for the dense (streaming) route. */
xgr_status xgr_beam_next_route(const xgr_ctx* ctx, int32_t* sparse);

/* ---- KV-cache reorder after a step (section 5.1, Fig. 6:
 * the unshared per-beam cache "updates block contents based on beam indices").
 * For every request r < n_req, panel p < n_panel (e.g. a layer's K or V panel) and slot j < bw
 * with s = src[r*src_ld + j] >= 0: new row (r, p, j) = old row (r, p, s), in place. Row (r, p, j)
 * is the row_bytes bytes at cache + r*req_stride + p*panel_stride + j*beam_stride (DEVICE memory;
 * cache, row_bytes and every stride 16-byte aligned; beam_stride >= row_bytes). src: DEVICE int32,
 * e.g. a step's parent[] (xgr_beam_view / xgr_beam_history); s < 0 (dead slot) and s == j leave
 * the row untouched. Any map is allowed, not only SPEC's monotone plans: rows are moved in column
 * tiles staged in shared memory, so no row is overwritten before it has been read, without an
 * auxiliary copy of the cache. bw 1..1024. Enqueues only (graph-capturable); no ctx needed.
 * Errors: XGR_ERR_INVALID_ARG (sizes, NULL), XGR_ERR_ALIGNMENT, XGR_ERR_CUDA. */
xgr_status xgr_kv_reorder(void* cache, int32_t n_req, int32_t n_panel, int32_t bw, int64_t row_bytes,
                          int64_t beam_stride, int64_t panel_stride, int64_t req_stride,
                          const int32_t* src, int32_t src_ld, void* stream);

/* ---- Staged shared/unshared decode attention (second workload; PAPER.md
 * L339, section 5.2 "Staged Computation Allocation"; L324 KV cache separation; SPEC.md
 * S:L136-179). One decode step of one attention layer for n_req requests of bw beams:
 *   out[r][b][h] = softmax_j(scale * q[r][b][h] . k_j) v_j over j in the request's prompt
 *   positions (shared cache, one copy per request) followed by beam b's own generated tokens
 *   t < n_unshared (unshared cache), with query head h reading KV head h / (hq / hkv).
 * Layouts (DEVICE memory, bf16, element offsets; head_dim d = 128 only):
 *   q        [n_req][bw][hq][d] contiguous
 *   k_shared, v_shared  [n_req][ls][hkv][d] contiguous (prefill output, token-major)
 *   k_unshared, v_unshared: element (r, b, t, g, e) at base + r*u_req_stride + b*u_beam_stride
 *            + (t*hkv + g)*d + e (the unshared cache of PAPER.md L324, e.g. one layer's K or V
 *            panel of the cache xgr_kv_reorder moves; strides multiples of 8 elements)
 *   out      bf16 [n_req][bw][hq][d];  lse: fp32 [n_req][bw][hq] natural-log LSE, or NULL
 * The shared stage runs on the tensor cores (tcgen05, fp32 accumulation; softmax weights are
 * rounded to bf16 for the P.V product); the unshared stage and the merge run in its epilogue.
 * Constraints: d == 128, hq % hkv == 0, G = hq / hkv a power of two <= 128, 1 <= bw <= 65535,
 * n_req <= 65535, hkv <= 65535, 0 <= n_unshared <= 8, ls >= 0, ls + n_unshared >= 1 (S:L170:
 * both stages empty is undefined), all pointers 16-byte aligned. Enqueues only (no sync, no
 * allocation; graph-capturable). Errors: XGR_ERR_INVALID_ARG, XGR_ERR_UNSUPPORTED (d != 128 or
 * G not a power of two), XGR_ERR_ALIGNMENT, XGR_ERR_CUDA. */
xgr_status xgr_attn_staged(const void* q, const void* k_shared, const void* v_shared, int32_t ls,
                           const void* k_unshared, const void* v_unshared, int64_t u_req_stride,
                           int64_t u_beam_stride, int32_t n_unshared, void* out, float* lse,
                           int32_t n_req, int32_t bw, int32_t hq, int32_t hkv, int32_t d, float scale,
                           void* stream);

/* Shared stage alone (SPEC attend_shared): partials of every (r, b, h) over the
 * prompt, fp32 DEVICE outputs m [n_req][bw][hq] (max of the scaled logits), s (sum of
 * exp(logit - m)), o [n_req][bw][hq][d] (sum of exp(logit - m) v, unnormalised); ls == 0 gives
 * the empty partial (m = -inf, s = 0, o = 0). Same kernel, layouts and constraints as
 * xgr_attn_staged. */
xgr_status xgr_attn_shared(const void* q, const void* k_shared, const void* v_shared, int32_t ls,
                           float* m, float* s, float* o, int32_t n_req, int32_t bw, int32_t hq,
                           int32_t hkv, int32_t d, float scale, void* stream);

/* Unshared stage alone (SPEC attend_unshared): partials over beam b's own tokens
 * t < n_unshared (0 gives the empty partial), same output layout as xgr_attn_shared. */
xgr_status xgr_attn_unshared(const void* q, const void* k_unshared, const void* v_unshared,
                             int64_t u_req_stride, int64_t u_beam_stride, int32_t n_unshared,
                             float* m, float* s, float* o, int32_t n_req, int32_t bw, int32_t hq,
                             int32_t hkv, int32_t d, float scale, void* stream);

/* OnlineSoftmax merge of two partials (SPEC merge_partials): for rows i < rows,
 * M = max(m1, m2), w_k = exp(m_k - M) (0 for an empty partial), out[i] = (o1 w1 + o2 w2) /
 * (s1 w1 + s2 w2) (fp32 [rows][d]), lse[i] = M + ln(s1 w1 + s2 w2) if lse != NULL. A row with
 * both partials empty yields NaN (undefined). d == 128. */
xgr_status xgr_attn_merge(const float* m1, const float* s1, const float* o1, const float* m2,
                          const float* s2, const float* o2, int64_t rows, int32_t d, float* out,
                          float* lse, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* XGR_BEAM_H */
