/*
 * hylra.h — C ABI of the B200 (sm_100a) HyLRA decode-time hybrid attention path.
 *
 * This is the drop-in boundary for the reference's layer-policy interface
 * (reference: pkg/src/layerreuse/engine.py:129-209 `hybrid_decode`), split into
 * the primitives that interface is built from:
 *
 *   hylra_full_decode    <- attention.py:210-226 `full_attention` for every head of a
 *                           layer, plus engine.py:177-181 (per-head logits summed
 *                           into the selection score, zero-initialised, head order)
 *   hylra_topk_select    <- attention.py:264-275 `topk_of_logits` / :278-284
 *                           `topk_indices` (min(budget, N) highest, ties to the lower
 *                           index, ascending) and engine.py:169,183 (per-step clamp)
 *   hylra_reuse_decode   <- attention.py:229-241 `_subset_attention` and :244-261
 *                           `sparse_attention` (gather, subset-renormalised softmax)
 *   hylra_decode_step    <- engine.py:167-197, one decode step of Algorithm 2
 *                           (PAPER.md:223-247): FULL layers score the cache and publish
 *                           a selection, REUSE layers inherit the most recent FULL
 *                           layer's selection (engine.py:173,185-194)
 *   hylra_overlap_counts <- profiling.py:38-47 `overlap_ratio` numerators |S_i & S_j|
 *                           feeding profiling.py:126-145 `build_similarity_matrix`
 *   hylra_block_select,  <- attention.py:287-313 block pooling / topk_blocks and
 *   hylra_decode_step_blocks  engine.py:212-286 `hybrid_decode_blocks` (block mode)
 *   hylra_decode_step_ex <- hylra_decode_step with a side stream (selects and REUSE
 *                           gathers overlap FULL streaming) and per-layer completion events
 *   hylra_append_kv      <- synthetic.py:154-187 (the cache grows one row per step)
 *   hylra_decode_step_offload <- index-guided offload (the offload mirror
 *                           of engine.py:314-368 `cost_model`): REUSE layers' K/V in
 *                           page-locked host memory, only the selected rows cross the link
 *
 * Conventions
 *   - Every pointer is caller-owned DEVICE memory unless stated otherwise; the
 *     library allocates nothing and retains nothing. Work is enqueued on `stream`
 *     (a cudaStream_t passed as void*) and is asynchronous.
 *   - Workspaces must be zero-filled once before first use; the kernels leave them
 *     in the zero state they found them in, so a workspace can be reused by any
 *     number of calls and CUDA-graph replays on one stream. The words kernels expect
 *     zeroed (split-K counters, single-launch sync words) sit at offsets that depend
 *     only on the geometry's batch and kv_heads (and, for the decode step, the policy),
 *     never on n_valid, budget or the layer count of a call: one workspace serves every
 *     call on one (batch, kv_heads) geometry, e.g. a decoder whose cache grows each step.
 *     Re-zero it before using it with another geometry.
 *   - Stateless and re-entrant: concurrent calls are safe on distinct streams with
 *     non-aliasing outputs and workspaces, from any host thread and on any device
 *     (function attributes are set per device; grids are sized from the current
 *     device's SM count).
 *   - Status codes map 1:1 onto the reference's exception taxonomy
 *     (pkg/src/layerreuse/errors.py:4-21).
 */
#ifndef HYLRA_H
#define HYLRA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HYLRA_ABI_VERSION 7

enum hylra_status {
  HYLRA_OK = 0,
  HYLRA_ERR_CONFIGURATION = 1,     /* ConfigurationError    errors.py:8  */
  HYLRA_ERR_INVALID_INPUT = 2,     /* InvalidInputError     errors.py:20 */
  HYLRA_ERR_INVALID_SELECTION = 3, /* InvalidSelectionError errors.py:16 */
  HYLRA_ERR_NUMERIC_INPUT = 4,     /* NumericInputError     errors.py:12 */
  HYLRA_ERR_CUDA = 5               /* launch / driver failure            */
};

enum hylra_dtype { HYLRA_BF16 = 0, HYLRA_F32 = 1 };

/* Device error-flag bits (written into the workspace flag word, see
 * hylra_read_flags). Set by kernels; cleared by hylra_clear_flags. */
enum hylra_flag {
  HYLRA_FLAG_INDEX_OUT_OF_RANGE = 1, /* a REUSE index >= n_valid  (attention.py:256-259) */
  HYLRA_FLAG_NON_FINITE_SCORE = 2,   /* a NaN/inf score or output (attention.py:43-44)   */
  HYLRA_FLAG_REFINE_SKIPPED = 4,     /* a row's f64 refinement window exceeded 1024
                                        scores: its k-th boundary follows fp32 order     */
  HYLRA_FLAG_INTERNAL = 8,           /* a kernel invariant failed (selection size != k)  */
  HYLRA_FLAG_NON_FINITE_CACHE = 16   /* a NaN/inf K/V entry (hylra_check_cache, appended
                                        rows; attention.py:38-46,61-71)                 */
};

/*
 * Shapes and strides of one KV cache + query tensor set (GQA).
 *   q   : element [layer][b][qh][i]  at q   + layer*q_stride_layer  + b*q_stride_batch  + qh*d + i
 *   k,v : element [layer][b][kh][n][i] at k + layer*kv_stride_layer + b*kv_stride_batch + kh*kv_stride_head + n*d + i
 *   out : fp32 element [layer][b][qh][i] at out + layer*out_stride_layer + b*out_stride_batch + qh*d + i
 * Query head qh reads KV head qh / (q_heads / kv_heads). All strides are in
 * elements and must keep every (layer, b, kh) block 16-byte aligned.
 */
typedef struct hylra_geometry {
  int32_t batch;      /* B                                        */
  int32_t q_heads;    /* Hq                                       */
  int32_t kv_heads;   /* Hkv; Hq % Hkv == 0; G = Hq / Hkv <= 16   */
  int32_t head_dim;   /* d in {32, 64, 128}                       */
  int32_t capacity;   /* N_cap rows allocated per (layer, b, kh)  */
  int32_t dtype;      /* enum hylra_dtype (q, k and v share it)   */
  int32_t num_layers; /* L addressable through the strides        */
  int32_t reserved;
  int64_t q_stride_layer, q_stride_batch;
  int64_t kv_stride_layer, kv_stride_batch, kv_stride_head;
  int64_t out_stride_layer, out_stride_batch;
} hylra_geometry;

int hylra_abi_version(void);
const char* hylra_status_string(int status);
/* Detail message of the last non-OK status returned on the calling thread. */
const char* hylra_last_error(void);
/* Host-side count of kernels this library has launched (not graph replays). */
uint64_t hylra_launch_count(void);
/* Process-wide tuning overrides (ABI 7; value -1 restores the default rule):
 *   "rowsel"         1/0: token rows that fit a CTA cluster's shared memory are selected by
 *                    the shared-memory-resident select (default 1; env HYLRA_ROWSEL);
 *   "select_threads" 128/256/512/1024: CTA width of the streaming select kernel (default:
 *                    by row count; env HYLRA_SELECT_THREADS).
 *   "rowsel_cluster" 1/2/4/8: CTAs per row of the shared-memory-resident select (default:
 *                    the fewest that hold the row, doubled while the launch stays within
 *                    one wave of SMs).
 *   "gather_tma"     1/0: standalone REUSE launches gather rows with TMA tile::gather4
 *                    (UTMALDG.2D.GATHER4) instead of cp.async, for contiguous caches
 *                    (default 0: measured 1.5x slower, profiles/r02_gather_tma_ab.txt).
 *   "bulk_merge"     1/0: the split-K final merge pulls a pair's partials into shared
 *                    memory with cp.async.bulk (default 1; env HYLRA_BULK_MERGE).
 *   "cluster_merge"  1/0: a REUSE launch split 2-16 ways within one CTA per SM runs each pair's
 *                    splits as one CTA cluster and merges them through distributed shared
 *                    memory (default 1; env HYLRA_CLUSTER_MERGE).
 *   "reuse_prefetch" REUSE L2 prefetch distance in tiles (default 0, the best measured).
 *   "fused_fine_splits" 1: FULL launches with fused selects over <= 64 pairs take finer
 *                    split-K partitions (faster at small batch; outputs then differ from
 *                    the other schedules' at bf16 level). Default 0.
 * Index sets never depend on them; outputs neither, except under "fused_fine_splits". */
int hylra_set_tuning(const char* name, int value);

/* Bytes of zero-filled workspace the attention ops need for `n_layers` layer
 * slots processed in one call over `rows` rows (n_valid for FULL, k for REUSE). */
size_t hylra_attention_workspace_bytes(const hylra_geometry* g, int n_layers, int rows);
/* Bytes of workspace hylra_topk_select needs for n_slots * B * (Hkv/sel_group) rows. */
size_t hylra_select_workspace_bytes(const hylra_geometry* g, int n_slots, int sel_group);

/*
 * FULL attention for layers layer_ids[0..n_layers) (host array) over rows [0, n_valid).
 * out   : written for every query head of those layers (geometry out strides).
 * scores: optional (NULL = do not emit); fp32 [n_layers][B][Hkv][capacity],
 *         scores[s][b][kh][n] = sum_{g<G} (q_{kh*G+g} . k_n) / sqrt(d).
 */
int hylra_full_decode(const hylra_geometry* g, const void* q, const void* k, const void* v,
                      int n_valid, int n_layers, const int32_t* layer_ids, float* out,
                      float* scores, void* ws, size_t ws_bytes, void* stream);

/*
 * Exact top-min(budget, n_valid) selection per (slot, b, group) row, where a group is
 * `sel_group` consecutive KV heads whose score rows are summed in head order
 * (sel_group = 1: per-KV-head sets; sel_group = Hkv: the reference's layer-wide set).
 * Ties go to the lower index; idx[s][b][grp][0..k_eff) is written ascending (int32).
 * If q and k are non-NULL (with layer_ids, host array of the scored layers), the
 * k-th boundary is re-resolved in float64 from the original q/k values, which makes
 * the set match a float64 evaluation except at float64-level ties.
 * info (optional, int32 [rows][8]): k_eff, refined candidates, mode, band size, and the
 * clock64 cycles of the sample / pass / select+refine / compaction phases.
 */
int hylra_topk_select(const hylra_geometry* g, const float* scores, int n_slots, int n_valid,
                      int budget, int sel_group, const void* q, const void* k,
                      const int32_t* layer_ids, int32_t* idx, int k_stride, int32_t* info,
                      void* ws, size_t ws_bytes, void* stream);

/* hylra_topk_select with options (ABI 7). HYLRA_SELECT_COMPACT: the select runs beside
 * other work (a side stream under a streaming launch), so the shared-memory-resident select
 * keeps each row on the fewest CTAs instead of spreading few rows over more SMs. */
#define HYLRA_SELECT_COMPACT 1
int hylra_topk_select_ex(const hylra_geometry* g, const float* scores, int n_slots,
                         int n_valid, int budget, int sel_group, const void* q, const void* k,
                         const int32_t* layer_ids, int32_t* idx, int k_stride, int32_t* info,
                         void* ws, size_t ws_bytes, void* stream, int options);

/*
 * REUSE attention for layers layer_ids[0..n_layers) (host array): layer i gathers the
 * k_eff rows idx[src_slots[i]][b][kh / sel_group][0..k_eff) of its own K/V and runs
 * the subset-renormalised softmax (attention.py:229-241). Indices >= n_valid are
 * masked and raise HYLRA_FLAG_INDEX_OUT_OF_RANGE. counts (optional, same row indexing as
 * idx) trims each selection row to its own length (block coverage).
 */
int hylra_reuse_decode(const hylra_geometry* g, const void* q, const void* k, const void* v,
                       int n_valid, int n_layers, const int32_t* layer_ids,
                       const int32_t* src_slots, const int32_t* idx, const int32_t* counts,
                       int k_stride, int k_eff, int sel_group, float* out, void* ws,
                       size_t ws_bytes, void* stream);

/*
 * One layer of a LAYER-SEQUENTIAL decode step (ABI 7): the per-layer body of the reference's
 * hybrid_decode loop (engine.py:174-194), for callers whose next layer's query depends on
 * this layer's output (a real model's decode). Launches on `stream`, in order:
 *   full = 1: FULL attention of `layer` over rows [0, n_valid) -> out; with `scores`
 *             (fp32 [B][Hkv][round_up(capacity, 8)]) the layer's selection scores; with idx
 *             as well, its top-min(budget, n_valid) selection (float64 refinement if refine)
 *             into selection slot `slot` of idx ([slot][B][Hkv/sel_group][k_stride]) by a
 *             second launch;
 *   full = 0: REUSE attention of `layer` over the selection in slot `slot` of idx.
 * prefetch = 1 lets the kernel's producer warps start loading K/V (REUSE: and the indices)
 * before the previous kernel on the stream has finished (programmatic dependent launch;
 * only the reads of q wait for it). This only matters when that previous kernel releases
 * its dependents early, as this library's kernels do; an ordinary kernel completes first.
 * The caller asserts that an early-releasing previous kernel wrote none of those: e.g. this
 * is not the first REUSE layer after the selection it reads. ws: zero-filled,
 * hylra_attention_workspace_bytes(g, 1, max(n_valid, k)) bytes, flag word first; kernels of
 * consecutive layers may overlap, so consecutive calls must alternate between two
 * workspaces.
 */
int hylra_decode_layer(const hylra_geometry* g, const void* q, const void* k, const void* v,
                       int n_valid, int layer, int full, int slot, int budget, int sel_group,
                       int refine, int prefetch, float* out, float* scores, int32_t* idx,
                       int k_stride, void* ws, size_t ws_bytes, void* stream);

/*
 * Block-level selection (paper §3.5; engine.py:212-286): per (slot, b, group) row the
 * token scores are max-pooled into ceil(n_valid / block_size) block scores
 * (attention.py:287-295), the top min(block_budget, n_blocks) blocks are selected with
 * the token rule (ties -> lower block, ascending; float64 refinement when q/k given, a
 * block's exact score being the float64 max over its tokens), written to
 * blocks[s][b][grp][bk_stride], and — if tokens != NULL — expanded to their ascending
 * token coverage tokens[..][tok_stride] (final block truncated at n_valid) with the
 * coverage length in counts[..] (attention.py:166-182). info: as hylra_topk_select.
 * ws: 256 B + 4 * n_slots * B * (Hkv/sel_group) * round_up(n_blocks, 8) bytes.
 */
int hylra_block_select(const hylra_geometry* g, const float* scores, int n_slots, int n_valid,
                       int block_budget, int block_size, int sel_group, const void* q,
                       const void* k, const int32_t* layer_ids, int32_t* blocks, int bk_stride,
                       int32_t* tokens, int tok_stride, int32_t* counts, int32_t* info,
                       void* ws, size_t ws_bytes, void* stream);

/* Workspace for hylra_decode_step (covers scores, select and attention workspaces). */
size_t hylra_decode_step_workspace_bytes(const hylra_geometry* g, const uint8_t* actions,
                                         int n_valid, int budget, int sel_group, int sinks,
                                         int recent);

/*
 * One hybrid decode step over all g->num_layers layers (Algorithm 2).
 * actions: host array of L bytes, 1 = FULL, 0 = REUSE; actions[0] must be FULL.
 * idx    : int32 [n_full][B][Hkv/sel_group][k_stride]; slot s holds the selection of
 *          the s-th FULL layer; a REUSE layer's selection is its source slot's.
 * All FULL layers are scored in one launch, all selections made in one launch and all
 * REUSE layers gathered in one launch: 3 kernels per step whatever L is. sinks / recent
 * (engine.py:122-126, off = 0) add the first `sinks` and last `recent` tokens to the sets
 * REUSE layers read (one more launch); idx keeps the FULL layers' own sets.
 */
int hylra_decode_step(const hylra_geometry* g, const void* q, const void* k, const void* v,
                      int n_valid, const uint8_t* actions, int budget, int sel_group,
                      int refine, int sinks, int recent, float* out, int32_t* idx,
                      int k_stride, void* ws, size_t ws_bytes, void* stream);

/*
 * hylra_decode_step with scheduling options (same kernels and results; NULL opt = plain
 * hylra_decode_step). Every field is optional (NULL):
 *   side_stream + fork_event, select_event, full_event, join_event: a second stream (best
 *     created with a higher priority than `stream`) that takes the latency-bound selects
 *     off the critical path. FULL layers some REUSE layer inherits from (A) are scored
 *     first, then the others (B), then the REUSE launch, all on `stream`; SELECT(A) runs on
 *     side_stream under FULL(B) and SELECT(B) under the REUSE launch; `stream` finally
 *     waits for side_stream. Ignored without REUSE layers, when every FULL layer feeds a
 *     REUSE layer, or with sinks / recent.
 *   fuse_select (with side_stream + fork_event and join_event): the selections of the FULL
 *     layers some REUSE layer inherits from are made inside the FULL kernel (the last CTA
 *     of each (layer, b, kv-head) pair selects that pair's row while other CTAs keep
 *     streaming); those layers' pairs come first in the grid. The other FULL layers'
 *     SELECT runs on side_stream under the REUSE launch. Tensor-core path, sel_group 1,
 *     no sinks / recent; otherwise the plain or side-stream schedule applies.
 *   fuse_select = 2 (no side stream needed): single-launch step. ONE kernel runs every
 *     FULL (layer, b, kv-head) split with every selection fused into the last CTA of its
 *     pair, then every REUSE split; a REUSE CTA first waits for its selection row's ready
 *     flag. CTAs claim work by an atomic ticket, so a waiting REUSE CTA only ever waits on
 *     FULL work already running (no deadlock for any dispatch order). Same split-K
 *     partitions as the plain step: outputs and selections are bit-identical to it.
 *     With sinks / recent the final CTA also writes the augmented row; with sel_group > 1
 *     the last pair of each selection group to finish selects. Tensor-core path, no
 *     layer_events (otherwise the schedules above apply);
 *     reuse_wait_event is waited on before the launch. The
 *     workspace carries the ticket / ready words and the kernel leaves them zeroed.
 *   fuse_select = 3: the single-launch step with COOPERATIVE selects (token mode, sel_group
 *     1): every split of a FULL pair classifies its own slice of the score row against the
 *     k-th value's histogram bin (published by the last split to finish streaming), and the
 *     last split to classify resolves the row. The select leaves the critical path of small
 *     batches at the cost of splits waiting on their slowest sibling; same results (ABI 6).
 *   reuse_wait_event: the REUSE launches wait on it (e.g. REUSE layers' queries arriving).
 *   layer_events: L entries (NULL allowed); layer_events[l] is recorded as soon as out[l] is
 *     final — FULL layers right after their FULL launch, REUSE layers after the REUSE
 *     launch that covers them: REUSE layers are launched in chunks ending at each REUSE
 *     layer that carries an event, so a caller can stream finished layers out while later
 *     chunks run.
 * Workspace: as hylra_decode_step.
 */
typedef struct hylra_step_options {
  int32_t fuse_select; /* 1 (with side_stream, fork_event, join_event), 2 or 3: see above */
  void* side_stream;
  void* fork_event;   /* stream -> side: FULL(A) done   */
  void* select_event; /* side -> stream: SELECT(A) done */
  void* full_event;   /* stream -> side: FULL(B) done   */
  void* join_event;   /* side -> stream: SELECT(B) done */
  void* reuse_wait_event;
  void* const* layer_events;
  /* the step's new K/V rows, [L][B][Hkv][d] in the cache dtype, device or pinned host memory
     (NULL: none), written at cache row append_pos (< n_valid) before they are read. With
     fuse_select = 2 the single-launch kernel writes them itself (no extra launch: each FULL
     pair's own row by the split that streams it, the REUSE layers' rows by the FULL pair
     whose selection they inherit); otherwise hylra_append_kv runs first. Not with
     hylra_decode_step_offload. (ABI 5) */
  const void* append_k_rows;
  const void* append_v_rows;
  int32_t append_pos;
  /* a second copy of the selections (idx / blocks, same layout and stride), in device or
     page-locked host memory (NULL: none). Written by the selecting CTAs as they write idx,
     so a caller that wants the per-layer index sets on the host needs no copy after the
     step (ABI 6). */
  void* idx_mirror;
} hylra_step_options;

int hylra_decode_step_ex(const hylra_geometry* g, const void* q, const void* k, const void* v,
                         int n_valid, const uint8_t* actions, int budget, int sel_group,
                         int refine, int sinks, int recent, float* out, int32_t* idx,
                         int k_stride, void* ws, size_t ws_bytes, void* stream,
                         const hylra_step_options* opt);

/*
 * hylra_decode_step with the cache split by action (index-guided offload). k_full/v_full:
 * [n_full][B][Hkv][cap][d] DEVICE memory holding the FULL layers in layer order; k_reuse /
 * v_reuse: [n_reuse][B][Hkv][cap][d] holding the REUSE layers in layer order, in
 * page-locked host memory (cudaHostAlloc / cudaHostRegister; read in place over the link
 * through its device mapping) or in device memory. Both use g->kv_stride_* (the layer
 * stride is per compact buffer); g->num_layers = L still sizes q and out. REUSE kernels
 * read only the selected rows, so the link carries B*Hkv*2*k_eff*d*e bytes per REUSE
 * layer. Pageable host memory -> ConfigurationError. Workspace: as hylra_decode_step.
 */
int hylra_decode_step_offload(const hylra_geometry* g, const void* q, const void* k_full,
                              const void* v_full, const void* k_reuse, const void* v_reuse,
                              int n_valid, const uint8_t* actions, int budget, int sel_group,
                              int refine, int sinks, int recent, float* out, int32_t* idx,
                              int k_stride, void* ws, size_t ws_bytes, void* stream);

/*
 * Append one decode step's new K/V rows (synthetic.py:154-187 grows the cache one row per
 * step): k_rows / v_rows are [L][B][Hkv][d] (dtype of g, contiguous) in device memory OR
 * page-locked host memory (read in place across the link: no separate H2D copy); row `pos`
 * of every (layer, b, kh) block of k / v receives them. layer_ids (host array of n_layers,
 * NULL = all g->num_layers layers) limits the append to some layers (rows stay indexed by
 * layer id), so an append can be split around the kernels that need it first.
 */
int hylra_append_kv(const hylra_geometry* g, void* k, void* v, const void* k_rows,
                    const void* v_rows, int pos, int n_layers, const int32_t* layer_ids,
                    void* stream);

/* hylra_append_kv that also validates the new rows: a NaN / inf entry sets
 * HYLRA_FLAG_NON_FINITE_CACHE in the workspace flag word ws[0] (ABI 6). The decode steps'
 * append_* options validate the same way. */
int hylra_append_kv_checked(const hylra_geometry* g, void* k, void* v, const void* k_rows,
                            const void* v_rows, int pos, int n_layers, const int32_t* layer_ids,
                            void* ws, void* stream);

/* Whole-cache validation (attention.py:38-46,61-71: the reference rejects any non-finite
 * K/V entry of every layer when it builds its float64 caches): one streaming pass over rows
 * [0, n_valid) of layers layer_ids[0..n_layers) (host array; NULL = all g->num_layers) sets
 * HYLRA_FLAG_NON_FINITE_CACHE in ws[0] if any entry is NaN or inf (ABI 6). */
int hylra_check_cache(const hylra_geometry* g, const void* k, const void* v, int n_valid,
                      int n_layers, const int32_t* layer_ids, void* ws, void* stream);

/* Sink / recent augmentation (engine.py:122-126): out[r] = sorted(idx[r][0..k_eff) |
 * [0, sinks) | [n_valid - recent, n_valid)), counts[r] its length. */
int hylra_augment_selection(const int32_t* idx, int rows, int k_eff, int k_stride, int n_valid,
                            int sinks, int recent, int32_t* out, int out_stride,
                            int32_t* counts, void* stream);

/* Block-mode decode step (engine.py:212-286): budget counts blocks of block_size tokens;
 * blocks[s][b][grp][bk_stride] receives each FULL layer's block selection. */
size_t hylra_decode_step_blocks_workspace_bytes(const hylra_geometry* g, const uint8_t* actions,
                                                int n_valid, int block_budget, int block_size,
                                                int sel_group);
int hylra_decode_step_blocks(const hylra_geometry* g, const void* q, const void* k,
                             const void* v, int n_valid, const uint8_t* actions,
                             int block_budget, int block_size, int sel_group, int refine,
                             float* out, int32_t* blocks, int bk_stride, void* ws,
                             size_t ws_bytes, void* stream);

/* hylra_decode_step_blocks with options (ABI 5): opt->fuse_select = 2 runs the block step as
 * ONE kernel. The final CTA of every FULL (layer, b, kv-head) pair pools that pair's scores
 * into blocks, selects them (block_budget, float64 refinement as above) and writes the
 * token coverage; the REUSE items gather it once their row's ready flag is set. Same
 * results as the multi-launch block step (tensor-core path, sel_group 1; otherwise the
 * multi-launch step runs). append_k_rows / append_v_rows / append_pos as for
 * hylra_decode_step_ex (written inside the single-launch kernel, else appended first).
 * Other option fields are ignored. Workspace: as above. */
int hylra_decode_step_blocks_ex(const hylra_geometry* g, const void* q, const void* k,
                                const void* v, int n_valid, const uint8_t* actions,
                                int block_budget, int block_size, int sel_group, int refine,
                                float* out, int32_t* blocks, int bk_stride, void* ws,
                                size_t ws_bytes, void* stream, const hylra_step_options* opt);

/*
 * Pairwise selection overlaps: counts[t][r][j][i] = |S(t,i,r) & S(t,j,r)| where
 * S(t,l,r) = idx[t][l][r][0..k) (ascending, distinct, each < n_tokens).
 */
int hylra_overlap_counts(const int32_t* idx, int steps, int layers, int rows, int k,
                         int k_stride, int n_tokens, int32_t* counts, void* stream);

/* Flag word helpers. The flag word is the first int32 of the attention / select / step
 * workspaces; the second int32 counts the selection rows that raised
 * HYLRA_FLAG_REFINE_SKIPPED. hylra_read_flags returns the flag word, hylra_clear_flags zeroes
 * both words. */
int hylra_read_flags(const void* ws, int32_t* flags_host, void* stream);
int hylra_clear_flags(void* ws, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HYLRA_H */
