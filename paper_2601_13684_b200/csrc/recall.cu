// Trace-driven residency recall (CacheEngine._measure, engine.py:276-288).
//
// One thread per head walks its recorded row in record order and keeps two
// float64 running sums, exactly as attention_recall (evaluation.py:41-59)
// does in Python: IEEE double additions in the same order give the same
// bits.  Membership follows CacheView.__contains__ (engine.py:98-107).

#include <cub/device/device_segmented_radix_sort.cuh>

#include "hc_common.cuh"

namespace hc {
namespace {

__global__ void trace_recall_kernel(const hc_recall_head* __restrict__ heads, int n_heads,
                                    uint32_t K, uint64_t stride, uint32_t L, uint32_t t,
                                    uint32_t sinks, uint32_t recency, double* __restrict__ out) {
  const int h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h >= n_heads) return;
  hc_recall_head hd = heads[h];
  hd.idx += stride * t;
  hd.scores += stride * t;
  // position >= L + t - recency  (signed: the floor may be negative)
  const long long tail_floor = (long long)L + (long long)t - (long long)recency;
  double total = 0.0, hit = 0.0;
  for (uint32_t j = 0; j < K; ++j) {
    const uint32_t p = __ldg(hd.idx + j);
    if (p == HC_PAD_INDEX) continue;
    const double s = (double)__ldg(hd.scores + j);
    total = __dadd_rn(total, s);
    bool in = (p >= L) || (hd.dynamic == nullptr) || (p < sinks) ||
              ((long long)p >= tail_floor);
    if (!in) in = (__ldg(hd.dynamic + (p >> 5)) >> (p & 31)) & 1u;
    if (in) hit = __dadd_rn(hit, s);
  }
  out[h] = (total == 0.0) ? 1.0 : __ddiv_rn(hit, total);
}

}  // namespace
// Measure mode's record order: HCTRACE1 records are sorted by score
// descending, token index ascending (trace.py invariants; the exporter's
// selectTopK order), i.e. by the composite key (score_key << 32) | ~index
// descending -- a segmented radix sort per head from the CUDA toolkit (CUB).
// temp == nullptr: *temp_bytes receives the scratch size.
int segmented_sort_desc_u64(void* temp, size_t* temp_bytes, const uint64_t* in, uint64_t* out,
                            int n_items, int n_segments, const int* offsets, cudaStream_t st) {
  size_t bytes = temp ? *temp_bytes : 0;
  cudaError_t r = cub::DeviceSegmentedRadixSort::SortKeysDescending(
      temp, bytes, in, out, n_items, n_segments, offsets, offsets + 1, 0, 64, st);
  if (r != cudaSuccess) {
    set_error("segmented sort: %s", cudaGetErrorString(r));
    return HC_ECUDA;
  }
  if (!temp) *temp_bytes = bytes;
  return HC_OK;
}

}  // namespace hc

extern "C" int hc_trace_recall(const hc_recall_head* heads_dev, int n_heads, uint32_t K,
                               uint64_t step_stride, uint32_t prefill_len, uint32_t step,
                               uint32_t sink_count,
                               uint32_t recency_window, double* recall_out_dev, void* stream) {
  HC_REQUIRE(n_heads >= 0 && (n_heads == 0 || (heads_dev && recall_out_dev)), HC_EINVAL,
             "hc_trace_recall: bad arguments");
  if (n_heads == 0) return HC_OK;
  const int threads = 128;
  hc::trace_recall_kernel<<<(n_heads + threads - 1) / threads, threads, 0,
                            (cudaStream_t)stream>>>(heads_dev, n_heads, K, step_stride, prefill_len, step,
                                                    sink_count, recency_window, recall_out_dev);
  HC_CHECK_LAUNCH();
  return HC_OK;
}
