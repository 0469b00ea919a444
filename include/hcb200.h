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

/* Single-row convenience wrapper around the same kernel. */
int hc_select_topk(const float* scores_dev, const uint32_t* idx_dev, uint32_t n, uint32_t k,
                   uint32_t* out_idx_dev, uint32_t* out_count_dev, void* stream);

/* Set bit p of bitmap_dev for every p in idx_dev[0..*count_dev) after
 * clearing the first n_words words (K_base <- current top set,
 * engine.py:357; dynamic sets for residency tests, engine.py:265-268). */
int hc_bitmap_from_indices(uint32_t* bitmap_dev, uint32_t n_words, const uint32_t* idx_dev,
                           const uint32_t* count_dev, uint32_t max_count, void* stream);

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

#ifdef __cplusplus
}
#endif
#endif /* HCB200_H_ */
