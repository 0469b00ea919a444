// K1: deterministic top-k selection (radix select on a 64-bit composite key).
//
// Reference semantics (metrics.py:42-45 sparse, metrics.py:26-39 dense with
// pool_kernel == 0): order by score descending, ties by token index
// ascending; PAD entries (trace.py:34) never compete.  We select the k
// largest composite keys  K = (score_key(score) << 32) | ~index,  which is
// exactly that order, with an MSB-first byte-radix select.  Keys are unique
// (token indices are unique within a row, trace.py:278-281), so the final
// threshold splits the row exactly: selected <=> (K & mask) >= prefix.
//
// One CTA per row; rows are independent jobs so one launch serves every
// pivot / satellite / compressed head of a step.  All integer work -- no
// fast-math, no FTZ dependence (subnormal scores from 0.9^i compare exactly).

#include "hc_common.cuh"

namespace hc {
namespace {

constexpr int kThreads = 1024;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 4;  // consecutive candidates per thread in the output pass

struct TopkShared {
  uint32_t hist[256];
  uint32_t warp_tot[kWarps];
  uint32_t bucket;
  uint32_t rem;
  uint32_t overlap;
};

__device__ __forceinline__ uint64_t composite_key(const float* __restrict__ scores,
                                                  const uint32_t* __restrict__ idx, uint32_t i,
                                                  uint32_t* token, bool* live) {
  uint32_t t = idx ? __ldg(idx + i) : i;
  *token = t;
  *live = (t != HC_PAD_INDEX);
  return (uint64_t(score_key(__ldg(scores + i))) << 32) | uint64_t(~t);
}

// Warp 0 finds the bucket b (scanning 255 -> 0) holding the rem-th largest
// key; updates s.bucket and s.rem (rem becomes the rank inside bucket b).
__device__ void find_bucket(TopkShared& s) {
  const int lane = threadIdx.x & 31;
  uint32_t c[8];
  uint32_t local = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    c[j] = s.hist[255 - (lane * 8 + j)];
    local += c[j];
  }
  uint32_t incl = local;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    uint32_t v = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += v;
  }
  const uint32_t rem = s.rem;
  const uint32_t excl = incl - local;
  const bool mine = excl < rem && rem <= incl;
  if (mine) {
    uint32_t above = excl;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (above < rem && rem <= above + c[j]) {
        s.bucket = 255 - (lane * 8 + j);
        s.rem = rem - above;
      }
      above += c[j];
    }
  }
}

__global__ void __launch_bounds__(kThreads, 1)
topk_rows_kernel(const hc_topk_job* __restrict__ jobs, uint32_t n_add) {
  __shared__ TopkShared s;
  const hc_topk_job job = jobs[blockIdx.x];
  const uint32_t n = job.n + n_add;
  const float* __restrict__ scores = job.scores;
  const uint32_t* __restrict__ idx = job.idx;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;

  // ---- live count (sparse rows carry a PAD suffix) ----
  uint32_t live_cnt = 0;
  if (idx) {
    uint32_t c = 0;
    for (uint32_t i = tid; i < n; i += kThreads) c += (__ldg(idx + i) != HC_PAD_INDEX);
    for (int off = 16; off; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
    if (lane == 0) s.warp_tot[warp] = c;
    __syncthreads();
    if (warp == 0) {
      uint32_t v = lane < kWarps ? s.warp_tot[lane] : 0;
      for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if (lane == 0) s.rem = v;
    }
    __syncthreads();
    live_cnt = s.rem;
    __syncthreads();
  } else {
    live_cnt = n;
  }
  const uint32_t k = job.k < live_cnt ? job.k : live_cnt;

  // ---- MSB-first byte radix select on the 64-bit key ----
  uint64_t prefix = 0, mask = 0;  // selected <=> (key & mask) >= prefix
  if (k > 0 && k < live_cnt) {
    if (tid == 0) s.rem = k;
    for (int byte = 7; byte >= 0; --byte) {
      const int shift = byte * 8;
      for (int j = tid; j < 256; j += kThreads) s.hist[j] = 0;
      __syncthreads();
      for (uint32_t i0 = 0; i0 < n; i0 += kThreads) {  // warp-uniform trip count
        const uint32_t i = i0 + tid;
        uint32_t tok = HC_PAD_INDEX;
        bool live = false;
        uint64_t key = 0;
        if (i < n) key = composite_key(scores, idx, i, &tok, &live);
        const bool in = live && ((key & mask) == prefix);
        const uint32_t bin = uint32_t(key >> shift) & 255u;
        // warp-aggregated increment: equal bins (ties, zeros) would serialise
        const unsigned act = __ballot_sync(0xffffffffu, in);
        if (in) {
          const unsigned peers = __match_any_sync(act, bin);
          if ((__ffs(peers) - 1) == lane) atomicAdd(&s.hist[bin], __popc(peers));
        }
      }
      __syncthreads();
      if (warp == 0) find_bucket(s);
      __syncthreads();
      const uint32_t b = s.bucket;
      prefix |= uint64_t(b) << shift;
      mask |= uint64_t(255) << shift;
      const bool whole = (s.hist[b] == s.rem);
      __syncthreads();
      if (whole) break;  // every key in this bucket is selected
    }
  }
  const bool take_all = (k == live_cnt);

  // ---- ordered compaction + overlap with K_base ----
  uint32_t base = 0;
  uint32_t ovl = 0;
  if (k > 0) {
    for (uint32_t start = 0; start < n; start += kThreads * kItems) {
      const uint32_t i0 = start + uint32_t(tid) * kItems;
      uint32_t tok[kItems];
      bool sel[kItems];
      uint32_t c = 0;
#pragma unroll
      for (int j = 0; j < kItems; ++j) {
        sel[j] = false;
        tok[j] = 0;
        const uint32_t i = i0 + j;
        if (i < n) {
          bool live;
          const uint64_t key = composite_key(scores, idx, i, &tok[j], &live);
          sel[j] = live && (take_all || (key & mask) >= prefix);
          c += sel[j];
        }
      }
      // block exclusive scan of c
      uint32_t incl = c;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        uint32_t v = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += v;
      }
      if (lane == 31) s.warp_tot[warp] = incl;
      __syncthreads();
      if (warp == 0) {
        uint32_t v = s.warp_tot[lane];
        uint32_t wi = v;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          uint32_t u = __shfl_up_sync(0xffffffffu, wi, off);
          if (lane >= off) wi += u;
        }
        s.warp_tot[lane] = wi - v;  // exclusive
      }
      __syncthreads();
      uint32_t pos = base + s.warp_tot[warp] + incl - c;
      const uint32_t chunk_total = s.warp_tot[kWarps - 1] +
                                   __shfl_sync(0xffffffffu, incl, 31);  // valid in last warp
#pragma unroll
      for (int j = 0; j < kItems; ++j) {
        if (sel[j]) {
          job.out_idx[pos++] = tok[j];
          if (job.base_bitmap) ovl += (__ldg(job.base_bitmap + (tok[j] >> 5)) >> (tok[j] & 31)) & 1u;
        }
      }
      if (warp == kWarps - 1 && lane == 0) s.bucket = chunk_total;
      __syncthreads();
      base += s.bucket;
      __syncthreads();
    }
  }
  if (job.overlap_out) {
    for (int off = 16; off; off >>= 1) ovl += __shfl_xor_sync(0xffffffffu, ovl, off);
    if (tid == 0) s.overlap = 0;
    __syncthreads();
    if (lane == 0) atomicAdd(&s.overlap, ovl);
    __syncthreads();
    if (tid == 0) *job.overlap_out = s.overlap;
  }
  if (tid == 0) *job.out_count = k;
}

__global__ void bitmap_from_indices_kernel(uint32_t* __restrict__ bm, uint32_t n_words,
                                           const uint32_t* __restrict__ idx,
                                           const uint32_t* __restrict__ count, uint32_t max_count) {
  // single CTA: clear, then set (ordering inside one block)
  for (uint32_t w = threadIdx.x; w < n_words; w += blockDim.x) bm[w] = 0u;
  __syncthreads();
  const uint32_t c = min(*count, max_count);
  for (uint32_t i = threadIdx.x; i < c; i += blockDim.x) {
    const uint32_t p = idx[i];
    if ((p >> 5) < n_words) atomicOr(bm + (p >> 5), 1u << (p & 31));
  }
}

}  // namespace

int launch_topk(const hc_topk_job* jobs_dev, int n_jobs, uint32_t n_add, cudaStream_t st) {
  if (n_jobs <= 0) return HC_OK;
  topk_rows_kernel<<<n_jobs, kThreads, 0, st>>>(jobs_dev, n_add);
  HC_CHECK_LAUNCH();
  return HC_OK;
}

}  // namespace hc

extern "C" int hc_topk_batched(const hc_topk_job* jobs_dev, int n_jobs, uint32_t n_add,
                               void* stream) {
  HC_REQUIRE(n_jobs >= 0 && (n_jobs == 0 || jobs_dev), HC_EINVAL, "hc_topk_batched: bad jobs");
  return hc::launch_topk(jobs_dev, n_jobs, n_add, (cudaStream_t)stream);
}

extern "C" int hc_select_topk(const float* scores_dev, const uint32_t* idx_dev, uint32_t n,
                              uint32_t k, uint32_t* out_idx_dev, uint32_t* out_count_dev,
                              void* stream) {
  HC_REQUIRE(scores_dev && out_idx_dev && out_count_dev, HC_EINVAL,
             "hc_select_topk: null pointer");
  cudaStream_t st = (cudaStream_t)stream;
  hc_topk_job job{scores_dev, idx_dev, n, k, out_idx_dev, out_count_dev, nullptr, nullptr};
  hc_topk_job* d = nullptr;
  HC_CUDA_TRY(cudaMallocAsync(&d, sizeof(job), st));
  HC_CUDA_TRY(cudaMemcpyAsync(d, &job, sizeof(job), cudaMemcpyHostToDevice, st));
  int rc = hc::launch_topk(d, 1, 0, st);
  HC_CUDA_TRY(cudaFreeAsync(d, st));
  HC_CUDA_TRY(cudaStreamSynchronize(st));  // job lives on this stack frame
  return rc;
}

extern "C" int hc_bitmap_from_indices(uint32_t* bitmap_dev, uint32_t n_words,
                                      const uint32_t* idx_dev, const uint32_t* count_dev,
                                      uint32_t max_count, void* stream) {
  HC_REQUIRE(bitmap_dev && idx_dev && count_dev, HC_EINVAL, "hc_bitmap_from_indices: null");
  hc::bitmap_from_indices_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(bitmap_dev, n_words,
                                                                       idx_dev, count_dev,
                                                                       max_count);
  HC_CHECK_LAUNCH();
  return HC_OK;
}
