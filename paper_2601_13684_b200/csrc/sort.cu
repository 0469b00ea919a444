// Segmented descending sort of 64-bit composite keys (measure-mode records).
//
// HCTRACE1 records are ordered by score descending, token index ascending
// (trace.py invariants; the exporter's selectTopK order), i.e. by the
// composite key (score_key << 32) | ~index descending.  The measure path
// (diagnostic, not the per-step hot path) sorts each head's records with the
// CUDA toolkit's segmented radix sort.

#include <cub/device/device_segmented_radix_sort.cuh>

#include "hc_common.cuh"

namespace hc {

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
