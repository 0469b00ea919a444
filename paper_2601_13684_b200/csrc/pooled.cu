// Pooled dense top-k (metrics.py:26-39, _dense_top_k with pool_kernel > 0):
//   pooled = zero-padded moving sum over an odd window / pool_kernel   (float64)
//   order  = pooled descending, then raw descending, then index ascending
//   top-k  = the first k of that order.
// The engine itself never pools (traces are sparse, engine.py:229-230); this is
// the dense-profiling primitive behind top_k_indices(scores, k, pool_kernel).
//
// Exactness: numpy's np.convolve(w, ones, "same") reduces each window with a
// sequential float64 dot in ascending position order (BLAS ddot for windows
// below its 16-element vector block); the kernel below adds the same values in
// the same order, then divides by pool_kernel.  The three-key order comes from
// two stable radix sorts (raw descending, then pooled descending) of
// order-preserving 64-bit keys with -0.0 folded onto +0.0, as lexsort compares.

#include <cub/device/device_radix_sort.cuh>

#include "hc_common.cuh"

namespace hc {
namespace {

__device__ __forceinline__ uint64_t f64_key(double x) {
  if (x == 0.0) x = 0.0;  // -0.0 == +0.0 for lexsort
  const uint64_t b = static_cast<uint64_t>(__double_as_longlong(x));
  return (b >> 63) ? ~b : (b | (uint64_t(1) << 63));
}

__global__ void pooled_keys_kernel(const double* __restrict__ w, uint32_t n, int half, int kern,
                                   uint64_t* __restrict__ kp, uint64_t* __restrict__ kr,
                                   uint32_t* __restrict__ idx) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t lo = int64_t(i) - half < 0 ? 0 : int64_t(i) - half;
  const int64_t hi = int64_t(i) + half >= int64_t(n) ? int64_t(n) - 1 : int64_t(i) + half;
  double s = 0.0;
  for (int64_t j = lo; j <= hi; ++j) s = __dadd_rn(s, w[j]);
  kp[i] = f64_key(__ddiv_rn(s, double(kern)));
  kr[i] = f64_key(w[i]);
  idx[i] = i;
}

__global__ void gather_keys_kernel(const uint64_t* __restrict__ kp, const uint32_t* __restrict__ idx,
                                   uint32_t n, uint64_t* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = kp[idx[i]];
}

}  // namespace
}  // namespace hc

extern "C" int hc_pooled_topk(const double* w_dev, uint32_t n, uint32_t pool_kernel, uint32_t k,
                              uint32_t* out_idx_dev, void* stream) {
  HC_REQUIRE(w_dev && out_idx_dev && n > 0, HC_EINVAL, "hc_pooled_topk: bad arguments");
  HC_REQUIRE(pool_kernel >= 1 && (pool_kernel & 1) && pool_kernel <= n, HC_EINVAL,
             "pool kernel must be odd, positive and <= n");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // scratch: kp, kr, kp2 (n x u64), idx, idx2 (n x u32), cub temp
  size_t t1 = 0, t2 = 0;
  HC_CUDA_TRY(cub::DeviceRadixSort::SortPairsDescending(nullptr, t1, (uint64_t*)nullptr,
                                                         (uint64_t*)nullptr, (uint32_t*)nullptr,
                                                         (uint32_t*)nullptr, int(n), 0, 64, st));
  t2 = t1;
  const size_t bytes = size_t(n) * 8 * 4 + size_t(n) * 4 * 2 + t2 + 256;
  char* s = nullptr;
  HC_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&s), bytes, st));
  uint64_t* kp = reinterpret_cast<uint64_t*>(s);
  uint64_t* kr = kp + n;
  uint64_t* ks = kr + n;   // sorted raw keys (discarded)
  uint64_t* kp2 = ks + n;  // pooled keys in raw order
  uint32_t* idx = reinterpret_cast<uint32_t*>(kp2 + n);
  uint32_t* idx2 = idx + n;
  void* tmp = reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(idx2 + n) + 255) & ~uintptr_t(255));
  const int threads = 256, blocks = int((n + threads - 1) / threads);
  hc::pooled_keys_kernel<<<blocks, threads, 0, st>>>(w_dev, n, int(pool_kernel / 2),
                                                     int(pool_kernel), kp, kr, idx);
  HC_CHECK_LAUNCH();
  // (1) raw descending, stable -> ties keep ascending index
  HC_CUDA_TRY(cub::DeviceRadixSort::SortPairsDescending(tmp, t1, kr, ks, idx, idx2, int(n), 0, 64,
                                                         st));
  hc::gather_keys_kernel<<<blocks, threads, 0, st>>>(kp, idx2, n, kp2);
  HC_CHECK_LAUNCH();
  // (2) pooled descending, stable -> ties keep (raw desc, index asc)
  HC_CUDA_TRY(cub::DeviceRadixSort::SortPairsDescending(tmp, t1, kp2, kp, idx2, idx, int(n), 0, 64,
                                                         st));
  const uint32_t kk = k < n ? k : n;
  if (kk)
    HC_CUDA_TRY(cudaMemcpyAsync(out_idx_dev, idx, size_t(kk) * 4, cudaMemcpyDeviceToDevice, st));
  HC_CUDA_TRY(cudaFreeAsync(s, st));
  return HC_OK;
}
