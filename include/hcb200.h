/*
 * HeteroCache-B200: C ABI of the B200-native decode hot path.
 *
 * The reference (arXiv 2601.13684, /root/reference/pkg/src/heterocache) is a
 * pure-Python package with no FFI layer; its boundary is the Python API in
 * engine.py / metrics.py / budget.py / profiling.py.  Each entry point below
 * names the reference routine it replaces (file:line).  The Python package
 * paper_2601_13684_b200 binds these through ctypes and keeps the reference's
 * class and method names on top (see INTEGRATION.md for the binding a
 * heterocache maintainer would add).
 *
 * Conventions
 *   - plain pointers and sizes only; device pointers are marked _dev,
 *     host pointers _host; streams are cudaStream_t passed as void*.
 *   - every function returns an int status (HC_OK == 0) and never throws;
 *     hc_last_error() returns a thread-local description of the last failure.
 *   - all device work is stream ordered on the caller's stream (plus, for an
 *     engine handle, one handle-owned retrieval stream joined by events).
 *   - there is no CPU fallback: without an sm_100a device every compute
 *     entry point returns HC_ECUDA.
 */
#ifndef HCB200_H_
#define HCB200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum hc_status {
  HC_OK = 0,
  HC_EINVAL = 1,      /* malformed argument (EngineError analogue, engine.py:44)   */
  HC_EINFEASIBLE = 2, /* InfeasibleStateError analogue (engine.py:48)            */
  HC_ECUDA = 3,       /* CUDA runtime failure / no device                        */
  HC_ENOMEM = 4,      /* device or pinned-host allocation failed                 */
  HC_ESTATE = 5       /* call out of order for this handle                       */
};

#define HC_PAD_INDEX 0xFFFFFFFFu /* trace.py:34 PAD_INDEX */

const char* hc_version(void);
const char* hc_last_error(void);
/* Kernels launched by this library since load (bench evidence). */
unsigned long long hc_launch_count(void);

/* ---------------------------------------------------------------------------
 * K1 -- deterministic top-k selection.
 *
 * Replaces heterocache.metrics.top_k_indices (metrics.py:48-71): the sparse
 * branch _sparse_top_k (metrics.py:42-45; PAD entries skipped, order score
 * desc then index asc) when idx != NULL, and the dense no-pooling branch
 * _dense_top_k (metrics.py:26-39, pooled == raw, so order score desc then
 * position asc) when idx == NULL.  Called by the engine from _top_set /
 * pivot_top_set / prefill_init / the fetch loop (engine.py:229-240,
 * 263-274, 326-329).
 *
 * A job selects min(k, live) entries of one row of n candidates (scores[i],
 * token index idx[i] or i).  Selected token indices are written to out_idx
 * in candidate order (ascending positions for dense rows) and their count
 * to *out_count.  If base_bitmap != NULL, the number of selected positions
 * whose bit is set there is written to *overlap_out -- this is the
 * |top & K_base| numerator of pivot_overlap (engine.py:242-245, Eq. 9).
 * ------------------------------------------------------------------------- */
typedef struct hc_topk_job {
  const float* scores;         /* [n] fp32 scores                               */
  const uint32_t* idx;         /* [n] token indices, or NULL for a dense row    */
  uint32_t n;                  /* candidates (dense: row length)                */
  uint32_t k;                  /* requested count                               */
  uint32_t* out_idx;           /* [k] selected token indices                    */
  uint32_t* out_count;         /* selected count                                */
  const uint32_t* base_bitmap; /* optional K_base bitmap over token positions   */
  uint32_t* overlap_out;       /* optional |selected & base|                    */
} hc_topk_job;

/* jobs_dev: device array of n_jobs jobs; n_add is added to every job's n
 * (dense rows that grow by one position per decode step). */
int hc_topk_batched(const hc_topk_job* jobs_dev, int n_jobs, uint32_t n_add, void* stream);

/* Pooled dense top-k (metrics.py:26-39 with pool_kernel > 0): float64 row
 * w_dev[n], odd pool_kernel <= n; writes the first min(k, n) indices of the
 * order (zero-padded moving average desc, raw desc, index asc).  The engine
 * never pools; this backs top_k_indices(scores, k, pool_kernel) for dense
 * profiling. */
int hc_pooled_topk(const double* w_dev, uint32_t n, uint32_t pool_kernel, uint32_t k,
                   uint32_t* out_idx_dev, void* stream);

/* Single-row convenience wrapper around the same kernel. */
int hc_select_topk(const float* scores_dev, const uint32_t* idx_dev, uint32_t n, uint32_t k,
                   uint32_t* out_idx_dev, uint32_t* out_count_dev, void* stream);

/* Set bit p of bitmap_dev for every p in idx_dev[0..*count_dev) after
 * clearing the first n_words words (K_base <- current top set,
 * engine.py:357; dynamic sets for residency tests, engine.py:265-268). */
int hc_bitmap_from_indices(uint32_t* bitmap_dev, uint32_t n_words, const uint32_t* idx_dev,
                           const uint32_t* count_dev, uint32_t max_count, void* stream);

/* Drift-monitor form of K1+K2 for dense rows (pivot_overlap, engine.py:242-245):
 * for each of n_rows rows (row r at rows_dev + r*row_stride, n scores) and
 * bitmap r (kbase_dev + r*words), write the composite-key threshold of the
 * top-k set (selected <=> (score_key << 32 | ~pos) >= thr) and the overlap
 * |top_k & base|.  Synchronises the stream (test entry point). */
int hc_monitor_rows(const float* rows_dev, int64_t row_stride, int32_t n_rows, uint32_t n,
                    uint32_t k, const uint32_t* kbase_dev, int32_t words, uint64_t* thr_dev,
                    uint32_t* ovl_dev, void* stream);

/* ---------------------------------------------------------------------------
 * Trace-driven residency diagnostics (CacheView + attention_recall).
 *
 * Replaces the per-head loop of CacheEngine._measure (engine.py:276-288):
 * attention_recall (evaluation.py:41-59) over CacheView membership
 * (engine.py:98-107).  One thread per head sums the recorded scores of its
 * row in record order in float64, exactly as the reference's Python loop
 * does, so per-head recalls are bit-identical.  The cross-head mean is left
 * to the host (sum(recalls)/len, engine.py:287).
 * ------------------------------------------------------------------------- */
typedef struct hc_recall_head {
  const uint32_t* idx;      /* [K] recorded token indices (PAD suffix allowed) */
  const float* scores;      /* [K] recorded scores                             */
  const uint32_t* dynamic;  /* bitmap of the compressed head's dynamic set, or */
                            /* NULL for a full-cache head (base None)          */
} hc_recall_head;

/* heads_dev[h].idx / .scores point at the head's step-0 record; the kernel
 * reads record `step` at offset step * step_stride elements. */
int hc_trace_recall(const hc_recall_head* heads_dev, int n_heads, uint32_t K,
                    uint64_t step_stride, uint32_t prefill_len, uint32_t step,
                    uint32_t sink_count, uint32_t recency_window, double* recall_out_dev,
                    void* stream);


/* ---------------------------------------------------------------------------
 * K5 -- prefill observation-window scoring on the tcgen05 tensor cores.
 *
 * Step-0 score rows (prefill_init input, engine.py:263-268; the last prompt
 * token's GQA-mean post-softmax attention, export.ts:125-127 and
 * model.ts:274-291) generalised to an observation window of `window` prompt
 * tokens: score(t) = mean over the window*group query rows of softmax_t with
 * causal masking.  window = 1 is exactly the reference semantics.
 *   k_dev      [batch*kv_heads][L][128] bf16 keys
 *   q_obs_dev  [batch][window][kv_heads*group][128] bf16 queries
 *   rows_dev   [batch*kv_heads][row_stride] fp32 scores (first L written)
 * window*group <= 128.
 * ------------------------------------------------------------------------- */
int hc_obs_scores(const void* k_dev, const void* q_obs_dev, int32_t batch, int32_t kv_heads,
                  int32_t group, int32_t window, int32_t L, float* rows_dev, int64_t row_stride,
                  void* stream);

/* ---------------------------------------------------------------------------
 * K6 -- head-similarity profiling counts on the tcgen05 tensor cores.
 *
 * Every overlap coefficient of the taxonomy (metrics.py:74-106:
 * stability vs the prefill set, same-step peer agreement; profiling.py:286-367)
 * is |A & B| / min(|A|, |B|) over top-k index sets.  For each batch (one
 * trace x layer) this computes the full Gram matrix of the 0/1 indicator
 * matrix of its `sets` index sets (sel_dev [n_batches][sets][k_stride]
 * positions < n_positions, counts_dev [n_batches][sets] set sizes):
 *   gram_dev[batch][i][j] = |S_i & S_j|   (fp32, exact below 2^24),
 * with row pitch rows_pad = ceil(sets / 128) * 128.
 * ------------------------------------------------------------------------- */
int hc_gram_from_sets(const uint32_t* sel_dev, const uint32_t* counts_dev, int32_t n_batches,
                      int32_t sets, int32_t k_stride, int32_t n_positions, float* gram_dev,
                      void* stream);

/* ---------------------------------------------------------------------------
 * Tensor-mode engine: hierarchical KV store + per-step decode pipeline.
 *
 * Units are (batch b, layer l, kv head h), numbered u = (b*NL + l)*H + h.
 * Roles per (layer, head) come from the taxonomy (profiling.py:38-40):
 * volatile / pivot keep their full cache on the GPU; anchor / satellite keep
 * a compressed cache of their planned length l_h (budget.py:144-208) plus
 * sinks, recency tail and decode appends (CacheView, engine.py:98-115).
 * Satellites' full prefill K/V live in a pinned host pool for retrieval.
 * ------------------------------------------------------------------------- */
typedef struct hc_engine hc_engine; /* opaque handle; one host thread per handle */

enum hc_role { HC_ROLE_VOLATILE = 0, HC_ROLE_ANCHOR = 1, HC_ROLE_PIVOT = 2, HC_ROLE_SATELLITE = 3 };

typedef struct hc_engine_desc {
  int32_t batch;          /* sequences (the reference has one engine per sequence) */
  int32_t num_layers;
  int32_t kv_heads;       /* heads_per_layer of the trace manifest (trace.py:82-89) */
  int32_t group;          /* query heads per KV head (GQA), 1..8                     */
  int32_t head_dim;       /* 128                                                     */
  int32_t prefill_len;    /* L                                                       */
  int32_t max_decode;     /* capacity in decode steps                                */
  int32_t sink_count;     /* EngineConfig.sink_count (engine.py:58)                  */
  int32_t recency_window; /* EngineConfig.recency_window (engine.py:59), <= 32       */
  int32_t l_base_int;     /* BudgetPlan.l_base_int (budget.py:206)                   */
  int32_t chunk;          /* split-K rows per tile, multiple of 64 (0: 1024)         */
  int32_t monitor;        /* drift monitoring on (variant != no_retrieval)           */
  int32_t host_pool;      /* 1: satellite prefill K/V in pinned host memory          */
  int32_t obs_window;     /* prefill observation window w (0/1: last prompt token)   */
  int32_t score_material; /* pivot score material between K4 and the GQA-mean row:   */
                          /* 0 = fp32 e = 2^(x - m) (default: rows within fp32       */
                          /* rounding of the oracle's), 1 = fp16 (half the bytes,    */
                          /* ~5e-4 relative row error)                               */
  /* Device-resident boundary decisions (devdec): 1 = the window median test,
   * byte / completion accounting, fetch selection, gathers and landings run on
   * device streams (engine.py:293-357) and the host only mirrors them
   * (hc_engine_poll_decisions); the step never waits for the host.  The
   * EngineConfig knobs below are then required (engine.py:52-79). */
  int32_t device_decisions;
  int32_t window;             /* EngineConfig.window (<= 64)                      */
  int32_t update_delay_steps; /* EngineConfig.update_delay_steps                  */
  int32_t eval_every_step;    /* EngineConfig.eval_every_step (sliding window)    */
  int32_t bytes_per_kv_entry; /* transfer bytes per fetched index                 */
  int32_t pad_;
  int64_t transfer_bandwidth; /* EngineConfig.transfer_bandwidth, bytes per step  */
  double tau_drift;           /* EngineConfig.tau_drift                           */
} hc_engine_desc;

/* CacheEngine.__init__ (engine.py:156-214): allocate and lay out the store.
 * roles/lengths/cluster_pivot are [num_layers * kv_heads] host arrays;
 * lengths[i] is the planned length of a compressed head (ignored for full
 * heads); cluster_pivot[i] is the pivot head index of a satellite's cluster
 * (same layer, profiling.py:237-239), -1 otherwise. */
int hc_engine_create(const hc_engine_desc* desc, const int32_t* roles, const int32_t* lengths,
                     const int32_t* cluster_pivot, hc_engine** out);
/* Sharded store (units are (sequence, layer, cluster-or-loner
 * head)): owned is a [batch * num_layers * kv_heads] host array, unit
 * u = (b * num_layers + l) * kv_heads + h; units with owned[u] == 0 belong to
 * another rank and get no rows, no tiles, no append and no output (O rows of
 * absent units are left untouched).  A satellite must be owned together with
 * its pivot (it is refilled from the pivot's row, engine.py:326-329).  Measure
 * mode needs an unsharded engine.  owned == NULL: hc_engine_create. */
int hc_engine_create_sharded(const hc_engine_desc* desc, const int32_t* roles,
                             const int32_t* lengths, const int32_t* cluster_pivot,
                             const uint8_t* owned, hc_engine** out);
int hc_engine_destroy(hc_engine* eng);
/* device bytes, pinned host bytes, arena rows, number of pivot units */
int hc_engine_info(const hc_engine* eng, int64_t* out4);

/* prefill_init (engine.py:263-274) for one layer: k/v [B, H, L, 128] bf16 and
 * q_obs [B, w, H*G, 128] bf16 (the last w prompt tokens' queries; w = 1:
 * [B, H*G, 128]) on the device.  Scores every head with K5 (the step-0
 * record: GQA-mean attention of the last token, export.ts:125-127, or its
 * observation-window mean), selects top-l_h for compressed heads and
 * top-l_base for pivots (K_base), gathers the selected rows into the
 * compressed caches, copies full heads whole and satellites to the host pool. */
int hc_engine_prefill_layer(hc_engine* eng, int32_t layer, const void* k_dev, const void* v_dev,
                            const void* q_last_dev, void* stream);

/* decode_step (engine.py:290-311) minus host bookkeeping: append the step's
 * K/V (k_new/v_new [B, NL, H, 128]), run attention for every head of every
 * layer (q/o [B, NL, H*G, 128]), form pivot score rows and their top-l_base
 * sets with the |top & K_base| counts (Eq. 9). */
int hc_engine_decode_step(hc_engine* eng, int32_t step, const void* q_dev, const void* k_new_dev,
                          const void* v_new_dev, void* o_dev, void* stream);

/* decode_step from pinned HOST buffers (a serving runtime's per-step call):
 * q_host / o_host [B, NL, H*G, 128] and k_new_host / v_new_host [B, NL, H, 128]
 * bf16, page-locked (cudaHostAlloc / cudaHostRegister).  Steps moving more
 * than 512 KB cross H2D and D2H on engine-owned copy streams, double-buffered
 * by step parity so they overlap the neighbouring steps' decode; smaller
 * steps (launch-bound) read their inputs with one zero-copy kernel on
 * `stream` and the combine writes O straight into o_host.  Either way o_host
 * holds the step's output once `stream` has passed hc_engine_join.  The
 * caller must not rewrite the input buffers before then. */
int hc_engine_decode_step_host(hc_engine* eng, int32_t step, const void* q_host,
                               const void* k_new_host, const void* v_new_host, void* o_host,
                               void* stream);

/* decode_step in two halves (decode_step = begin(hold 0) + end), so that the
 * host's window decision of step-1 (engine.py:313-360, read with
 * hc_engine_overlaps, acted on with hc_engine_fire_batch / land_batch) runs
 * while the step's attention does:
 *   begin  appends the token and launches attention over every unit except
 *          the landing ones -- with hold_satellites != 0, except every
 *          satellite (transfers fired by the open decision may land now);
 *   end    applies the landings requested so far (landing point: wait for
 *          the gathers, swap descriptors), attends the held units, then
 *          combine, score rows and overlap counts.
 * Between the halves, overlaps and fire_batch read the previous step's
 * state on an internal side stream; land_batch is allowed only with
 * hold_satellites.  Results equal decode_step's. */
int hc_engine_decode_begin(hc_engine* eng, int32_t step, const void* q_dev,
                           const void* k_new_dev, const void* v_new_dev, void* o_dev,
                           int32_t hold_satellites, void* stream);
int hc_engine_decode_end(hc_engine* eng, int32_t step, void* stream);

/* The per-step drift monitor (overlap counts, thresholds) runs on an
 * internal stream beside the next step's attention; engine calls that read
 * its results wait for it.  hc_engine_join makes `stream` wait for the last
 * step's monitor (e.g. before timing or reading engine memory directly). */
int hc_engine_join(hc_engine* eng, void* stream);

/* Measure mode: attention-mass recall at scale (CacheEngine._measure,
 * engine.py:276-288, attention_recall evaluation.py:41-59).  Enable before
 * prefill; the engine then keeps a full-context copy of every head's K and,
 * per hc_engine_measure call (right after decode step `step`; step 0 = after
 * prefill), forms every head's dense GQA-mean row (K5 for non-pivots; pivots
 * keep their own decision rows), its top records (recall_topk per head,
 * at step 0 and for pivots max(recall_topk, l_base_int, every l_h) -- enough
 * for every selection the reference makes from them; HCTRACE1 order: score
 * descending, index ascending, PAD tail) and each head's recall of the recorded mass against its CacheView
 * resident set, in float64 in record order.  recall_out_host (optional):
 * one double per unit u = (b*NL + layer)*H + head. */
int hc_engine_enable_measure(hc_engine* eng, int32_t recall_topk);
int hc_engine_measure(hc_engine* eng, int32_t step, const void* q_dev, double* recall_out_host,
                      void* stream);
/* The records of unit u from the last hc_engine_measure (capacity >= records). */
int hc_engine_measure_records(hc_engine* eng, int32_t unit, uint32_t* idx_host,
                              float* scores_host, int32_t capacity, void* stream);

/* Copy the overlap counts of steps [first, last] (<= 64 steps back) into
 * out [(last-first+1) x n_pivots] (pivot order = ascending unit), then sync. */
int hc_engine_overlaps(hc_engine* eng, int32_t first, int32_t last, int32_t* out_host,
                       void* stream);

/* Fire a drift event for pivot unit `pivot_unit` at `step` (engine.py:322-357):
 * select top-l_s of the pivot's current row for each satellite (sorted by
 * head), restamp K_base with the current top set, and schedule the host ->
 * HBM gather of the selected rows on the retrieval stream.  Writes one
 * transfer id per satellite. */
int hc_engine_fire(hc_engine* eng, int32_t pivot_unit, int32_t step, int32_t completion_step,
                   int32_t* transfer_ids, void* stream);

/* The same for every pivot that fires at `step` (one K1 launch, one
 * restamp, one batched gather), in the given order (the reference's sorted
 * pivot order, engine.py:313).  transfer_ids receives one id per satellite
 * (pivot order, then satellite head order); if fetched_host (pinned) is not
 * NULL the fetched positions are copied there asynchronously, concatenated
 * in the same order (valid after the caller's stream has synchronised). */
int hc_engine_fire_batch(hc_engine* eng, int32_t n, const int32_t* pivot_units, int32_t step,
                         const int32_t* completion_steps, int32_t* transfer_ids,
                         uint32_t* fetched_host, void* stream);

/* Device decisions: one fire of a boundary (engine.py:322-347), as decided on
 * the device.  Fires are listed per sequence, in sorted pivot order. */
typedef struct hc_fire_record {
  int32_t trigger_step, pivot_unit, completion_step, n_satellites;
  int64_t transfer_bytes, cumulative_bytes;
  int32_t first_satellite;  /* index into hc_engine_devdec_satellites()            */
  int32_t fetched_offset;   /* the satellites' fetched sets, concatenated, at this */
                            /* offset of fetched_out (-1: not available)           */
  int32_t fetched_counts[8];
} hc_fire_record;

/* Device decisions: the next boundary not yet read, in step order.  wait = 0:
 * returns *step_out = -1 if its decision has not completed yet; wait = 1:
 * blocks on it (and returns -1 only when no boundary is outstanding).  Fills
 * fires[0 .. *n_fires_out) and the fetched sets (ascending positions) into
 * fetched_out (capacity entries; HC_EINVAL with the needed size in
 * *n_fires_out if too small).  Reports device-side faults (a satellite's
 * transfer ring overflowing, a landing wait timing out) as HC_ESTATE. */
int hc_engine_poll_decisions(hc_engine* eng, int32_t wait, int32_t* step_out,
                             hc_fire_record* fires, int32_t fire_capacity, int32_t* n_fires_out,
                             uint32_t* fetched_out, int64_t fetched_capacity);
/* Device decisions: the unit of every satellite, in the order
 * hc_fire_record.first_satellite indexes (pivot slots ascending, each pivot's
 * satellites by head). */
int hc_engine_devdec_satellites(hc_engine* eng, int32_t* units_out, int32_t capacity,
                                int32_t* n_out);

/* Block the calling host thread until the last fire batch's selection and
 * fetched-set copies (fetched_host) are done -- only those, on the engine's
 * side stream, not the work queued on the caller's stream since. */
int hc_engine_wait_fetched(hc_engine* eng);

/* Landing of a due transfer (engine.py:293-299): applied inside the next
 * decode step (or before the next call that reads engine state), where the
 * step's stream waits for the gather after attending every other unit; the
 * satellite serves the new set from that step on. */
int hc_engine_land(hc_engine* eng, int32_t transfer_id, void* stream);
/* Land several due transfers in (completion, order) order with one launch. */
int hc_engine_land_batch(hc_engine* eng, int32_t n, const int32_t* transfer_ids, void* stream);

/* Read back index sets (sorted ascending) and sync:
 *   kind 0: fetched set of a transfer, 1: a compressed unit's current
 *   dynamic set, 2: a pivot unit's current top-l_base set, 3: a compressed
 *   unit's prefix-buffer positions. */
int hc_engine_read_indices(hc_engine* eng, int32_t kind, int32_t id, uint32_t* out_host,
                           int32_t capacity, int32_t* n_out, void* stream);

/* Copy a pivot unit's probability row over [0, L + step) to dst (device). */
int hc_engine_pivot_row(hc_engine* eng, int32_t pivot_unit, int32_t step, float* dst_dev,
                        void* stream);

/* Resident K/V rows summed over all units at `step` (the algorithmic bytes of
 * the step are rows * 2 * head_dim * 2); syncs. */
int hc_engine_resident_rows(hc_engine* eng, int32_t step, int64_t* rows_out, void* stream);

/* Test hook: when set, prefill copies every layer's step-0 rows (the
 * GQA-mean probability rows over [0, L) of all B*H units of the layer,
 * unit order b*H + h) to dst [NL][B*H][L] fp32 (device). */
int hc_engine_set_prefill_dump(hc_engine* eng, float* dst_dev);

/* Per-step phase timeline for the roofline, from CUDA events on the
 * launching stream.  Reports (syncs) the summed milliseconds since the last
 * call of phase_ms[8] = {append, K4 attention, combine, pivot score rows,
 * K1/K2 monitor, overlap copy, whole step, gaps between steps} and the
 * number of steps, then
 * resets and enables (enable 1: every phase; 2: the K4 attention phase only,
 * two timed events per step, for launch-bound timed regions) or disables
 * (0) recording. */
int hc_engine_timing(hc_engine* eng, int32_t enable, double* phase_ms, int32_t* steps);

/* Retrieval statistics since the last call (timing must be enabled):
 * out4 = {bytes gathered over the host link (upper bound), gather-kernel
 * milliseconds on the retrieval stream, milliseconds the caller's stream
 * stalled waiting for due gathers at landings, gather batches}.  Syncs. */
int hc_engine_retrieval_stats(hc_engine* eng, double* out4);

/* Per-step idle gaps (ms) of the recorded timeline (does not reset). */
int hc_engine_gaps(hc_engine* eng, float* out, int32_t cap, int32_t* n);

/* Prefill scoring totals: out3 = {K5 milliseconds (CUDA events), layers, w}. */
int hc_engine_prefill_stats(hc_engine* eng, double* out3);

/* Number of attention tiles (CTAs) the step launches. */
int hc_engine_active_tiles(const hc_engine* eng, int32_t step, int32_t* n_tiles);

/* ---------------------------------------------------------------------------
 * Synthetic workload generator (bench inputs; no reference counterpart).
 *
 * out_dev[i] = N(key, offset + i) as fp32: splitmix64 of the counter, an
 * Irwin-Hall(4) normal from its four 16-bit fields, every step exact or one
 * IEEE rounding -- bit-identical to the host twin oracle/synth.c, so the CPU
 * arms of bench.py decode the same K/V/Q (workload.SyntheticKV).
 * ------------------------------------------------------------------------- */
int hc_synth_normal(float* out_dev, int64_t n, uint64_t key, int64_t offset, void* stream);

/* Read-only HBM probe (bench roofline denominator; no reference counterpart):
 * streams `bytes` (a multiple of 16) of buf_dev once with `ctas` CTAs of 256
 * threads and writes one XOR per CTA into sink_dev[ctas]. */
int hc_read_probe(const void* buf_dev, int64_t bytes, uint32_t* sink_dev, int32_t ctas,
                  void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HCB200_H_ */
