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

#include <algorithm>
#include <vector>

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

// ---------------------------------------------------------------------------
// Drift-monitor top-k (K1 + K2 fused), dense pivot rows.
//
// The monitor needs, per pivot and step, only the size of the overlap
// |top_{l_base}(row) & K_base| (engine.py:305-311) -- not the index list --
// plus the selection threshold so that K_base can be restamped if the pivot
// fires (engine.py:357).  One CTA per row, two streaming passes:
//   1. 13-bit histogram of the score keys (smem, 8192 bins) -> bucket b1
//      holding the k-th largest composite key;
//   2. count K_base bits of every key above b1, collect the keys inside b1
//      as (score, ~index) composites into shared memory;
// then an 8-bit radix select over the candidates only (score low bits and
// the index tie-break) yields the exact composite threshold T (selected <=>
// key >= T, the same set as metrics.py:26-45), and the candidates >= T add
// their K_base bits.  If the bucket overflows shared memory the select falls
// back to streaming radix passes over the row restricted to b1.
// ---------------------------------------------------------------------------
namespace hc {
namespace {

// The monitor runs beside the next step's attention: 512 threads (<= 64
// registers) and ~97 KB of shared memory let one monitor CTA share an SM
// with one attention CTA instead of owning it.
constexpr int kMonThreads = 512;
constexpr int kSelThreads = 1024;   // fire selection (runs beside K4 on its own)
constexpr int kMonBins = 8192;      // 13-bit first digit: key32 >> 19
constexpr int kMonCand = 8192;      // shared-memory candidate capacity
constexpr int kMonSmem = kMonBins * 4 + kMonCand * 8 + 64 * 4;

__device__ __forceinline__ uint64_t ckey(uint32_t k32, uint32_t pos) {
  return (uint64_t(k32) << 32) | uint64_t(~pos);
}

// Block-wide: find the bin (scanning from the top of `hist[nb]`) that holds
// the rem-th largest entry.  Returns via sh[0] = bin, sh[1] = rank in bin,
// sh[2] = bin count.  Every thread owns nb / blockDim.x consecutive bins.
template <int NB, int NT>
__device__ void block_find_bucket(const uint32_t* hist, uint32_t rem, uint32_t* sh,
                                  uint32_t* warp_tot) {
  constexpr int per = NB / NT;
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t local = 0;
#pragma unroll
  for (int j = 0; j < per; ++j) local += hist[NB - 1 - (tid * per + j)];
  uint32_t incl = local;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += v;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const uint32_t v = lane < NW ? warp_tot[lane] : 0u;
    uint32_t wi = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, wi, off);
      if (lane >= off) wi += u;
    }
    if (lane < NW) warp_tot[lane] = wi - v;
  }
  __syncthreads();
  const uint32_t excl = warp_tot[warp] + incl - local;
  if (excl < rem && rem <= excl + local) {
    uint32_t above = excl;
    for (int j = 0; j < per; ++j) {
      const int bin = NB - 1 - (tid * per + j);
      const uint32_t c = hist[bin];
      if (above < rem && rem <= above + c) {
        sh[0] = uint32_t(bin);
        sh[1] = rem - above;
        sh[2] = c;
        break;
      }
      above += c;
    }
  }
  __syncthreads();
}

// Exact composite threshold T of a row's top set, given the 13-bit bucket b1
// holding the rem-th largest key: an 8-bit radix over bits 50..0 of the
// composite key among the bucket's keys -- the m candidates in shared memory,
// or (cand == nullptr, bucket overflowed) streamed from the row.  Selected
// <=> key >= T.  hist: >= 1024 words of shared scratch.
template <int NT>
__device__ uint64_t radix_threshold(const float* __restrict__ row, uint32_t n, uint32_t b1,
                                    uint32_t rem, const uint64_t* cand, uint32_t m,
                                    uint32_t* hist, uint32_t* sh, uint32_t* warp_tot) {
  const int tid = threadIdx.x;
  uint64_t prefix = uint64_t(b1) << 51, mask = uint64_t(0x1fff) << 51;
  for (int shift = 43; ; shift -= 8) {
    const int sh_eff = shift < 0 ? 0 : shift;
    const uint64_t dmask = shift < 0 ? ((uint64_t(1) << (shift + 8)) - 1) : uint64_t(255);
    for (int j = tid; j < 1024; j += NT) hist[j] = 0;  // 1024-bin scan below
    __syncthreads();
    if (cand) {
      for (uint32_t i = tid; i < m; i += NT) {
        const uint64_t key = cand[i];
        if ((key & mask) == prefix) atomicAdd(&hist[uint32_t((key >> sh_eff) & dmask)], 1u);
      }
    } else {
      for (uint32_t i = tid; i < n; i += NT) {
        const uint64_t key = ckey(score_key(__ldg(row + i)), i);
        if ((key & mask) == prefix) atomicAdd(&hist[uint32_t((key >> sh_eff) & dmask)], 1u);
      }
    }
    __syncthreads();
    block_find_bucket<1024, NT>(hist, rem, sh, warp_tot);  // 1024 >= 256 bins (zeros above)
    const uint32_t b = sh[0];
    rem = sh[1];
    const bool done = (sh[2] == rem) || shift <= 0;
    prefix |= uint64_t(b) << sh_eff;
    mask |= dmask << sh_eff;
    __syncthreads();
    if (done) break;
  }
  return prefix;  // bucket fully taken, or keys unique
}

__global__ void __launch_bounds__(kMonThreads, 2)
monitor_kernel(const float* __restrict__ rows, int64_t row_stride, const int32_t* __restrict__ slots,
               uint32_t n, uint32_t k, const uint32_t* __restrict__ kbase, int words,
               uint64_t* __restrict__ thr_out, uint32_t* __restrict__ ovl_out,
               uint32_t* __restrict__ hist_out) {
  extern __shared__ __align__(16) uint8_t mon_smem[];
  uint32_t* hist = reinterpret_cast<uint32_t*>(mon_smem);
  uint64_t* cand = reinterpret_cast<uint64_t*>(mon_smem + kMonBins * 4);
  uint32_t* misc = reinterpret_cast<uint32_t*>(mon_smem + kMonBins * 4 + kMonCand * 8);
  uint32_t* sh = misc;            // [0..3] results
  uint32_t* warp_tot = misc + 8;  // [32]
  const int s = slots[blockIdx.x];
  const float* __restrict__ row = rows + size_t(s) * row_stride;
  const uint32_t* __restrict__ bm = kbase + size_t(s) * words;
  const int tid = threadIdx.x, lane = tid & 31;

  // hist_out (optional): the row's first-digit histogram is published for
  // the fire selection of this step (fire_select_kernel)
  uint32_t* gh = hist_out ? hist_out + size_t(s) * kMonBins : nullptr;
  if (k >= n) {  // everything is selected
    uint32_t c = 0;
    for (uint32_t i = tid; i < n; i += kMonThreads) c += (__ldg(bm + (i >> 5)) >> (i & 31)) & 1u;
    for (int off = 16; off; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
    if (tid == 0) sh[3] = 0;
    __syncthreads();
    if (lane == 0) atomicAdd(&sh[3], c);
    __syncthreads();
    if (tid == 0) { thr_out[s] = 0; ovl_out[s] = sh[3]; }
    return;
  }
  if (tid == 0) sh[3] = 0;  // candidate count
  const uint32_t n4 = n >> 2;
  const float4* __restrict__ row4 = reinterpret_cast<const float4*>(row);
  for (int j = tid; j < kMonBins; j += kMonThreads) hist[j] = 0;
  __syncthreads();
  // pass 1: 13-bit histogram; four float4 loads in flight per thread (one
  // CTA per row: the pass is bound by bytes in flight per SM)
  constexpr int kU = 4;
  for (uint32_t i0 = tid; i0 < n4; i0 += kMonThreads * kU) {
    float4 v[kU];
#pragma unroll
    for (int q = 0; q < kU; ++q)
      if (i0 + q * kMonThreads < n4) v[q] = __ldg(row4 + i0 + q * kMonThreads);
#pragma unroll
    for (int q = 0; q < kU; ++q) {
      if (i0 + q * kMonThreads >= n4) break;
      atomicAdd(&hist[score_key(v[q].x) >> 19], 1u);
      atomicAdd(&hist[score_key(v[q].y) >> 19], 1u);
      atomicAdd(&hist[score_key(v[q].z) >> 19], 1u);
      atomicAdd(&hist[score_key(v[q].w) >> 19], 1u);
    }
  }
  for (uint32_t i = n4 * 4 + tid; i < n; i += kMonThreads)
    atomicAdd(&hist[score_key(__ldg(row + i)) >> 19], 1u);
  __syncthreads();
  if (gh)
#pragma unroll
    for (int q = 0; q < kMonBins / kMonThreads; ++q)
      gh[tid + q * kMonThreads] = hist[tid + q * kMonThreads];
  block_find_bucket<kMonBins, kMonThreads>(hist, k, sh, warp_tot);
  const uint32_t b1 = sh[0];
  uint32_t rem = sh[1];
  const bool whole = (sh[2] == rem);
  __syncthreads();

  // pass 2: K_base bits above b1, candidates inside b1
  uint32_t ovl = 0;
  auto visit = [&](uint32_t pos, float x, uint32_t word) {
    const uint32_t k32 = score_key(x);
    const uint32_t d = k32 >> 19;
    const uint32_t bit = (word >> (pos & 31)) & 1u;
    if (d > b1 || (whole && d == b1)) ovl += bit;
    else if (!whole && d == b1) {
      const uint32_t at = atomicAdd(&sh[3], 1u);
      if (at < uint32_t(kMonCand)) cand[at] = ckey(k32, pos);
    }
  };
  for (uint32_t i0 = tid; i0 < n4; i0 += kMonThreads * kU) {
    float4 v[kU];
    uint32_t wd[kU];
#pragma unroll
    for (int q = 0; q < kU; ++q) {
      const uint32_t i = i0 + q * kMonThreads;
      if (i < n4) {
        v[q] = __ldg(row4 + i);
        wd[q] = __ldg(bm + (i >> 3));  // positions 4i..4i+3 share one bitmap word
      }
    }
#pragma unroll
    for (int q = 0; q < kU; ++q) {
      const uint32_t i = i0 + q * kMonThreads;
      if (i < n4) {
        visit(4 * i, v[q].x, wd[q]);
        visit(4 * i + 1, v[q].y, wd[q]);
        visit(4 * i + 2, v[q].z, wd[q]);
        visit(4 * i + 3, v[q].w, wd[q]);
      }
    }
  }
  for (uint32_t i = n4 * 4 + tid; i < n; i += kMonThreads) visit(i, __ldg(row + i), __ldg(bm + (i >> 5)));
  __syncthreads();

  uint64_t T = uint64_t(b1) << 51;  // lowest composite key of bucket b1
  if (!whole) {
    const uint32_t m = sh[3];
    const bool in_smem = m <= uint32_t(kMonCand);
    T = radix_threshold<kMonThreads>(row, n, b1, rem, in_smem ? cand : nullptr, m, hist, sh,
                                     warp_tot);
    // candidates at or above T add their K_base bits
    if (in_smem) {
      for (uint32_t i = tid; i < m; i += kMonThreads) {
        const uint64_t key = cand[i];
        if (key >= T) {
          const uint32_t pos = ~uint32_t(key);
          ovl += (__ldg(bm + (pos >> 5)) >> (pos & 31)) & 1u;
        }
      }
    } else {
      for (uint32_t i = tid; i < n; i += kMonThreads) {
        const uint64_t key = ckey(score_key(__ldg(row + i)), i);
        if ((key >> 51) == b1 && key >= T) ovl += (__ldg(bm + (i >> 5)) >> (i & 31)) & 1u;
      }
    }
  }
  for (int off = 16; off; off >>= 1) ovl += __shfl_xor_sync(0xffffffffu, ovl, off);
  if (tid == 0) sh[3] = 0;
  __syncthreads();
  if (lane == 0) atomicAdd(&sh[3], ovl);
  __syncthreads();
  if (tid == 0) {
    thr_out[s] = T;
    ovl_out[s] = sh[3];
  }
}

// K_base <- {p : key(p) >= T} over [0, n) for the listed pivot slots
// (engine.py:357), one warp per 32-position word via ballot.
__global__ void restamp_threshold_kernel(const float* __restrict__ rows, int64_t row_stride,
                                         const int32_t* __restrict__ slots, uint32_t n,
                                         const uint64_t* __restrict__ thr, uint32_t* kbase,
                                         int words, const uint32_t* n_rows_dev) {
  if (n_rows_dev && blockIdx.y >= *n_rows_dev) return;  // device-written slot list
  const int s = slots[blockIdx.y];
  const float* row = rows + size_t(s) * row_stride;
  const uint64_t T = thr[s];
  uint32_t* bm = kbase + size_t(s) * words;
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (int w = blockIdx.x * wpb + (threadIdx.x >> 5); w < words; w += gridDim.x * wpb) {
    const uint32_t pos = uint32_t(w) * 32 + lane;
    const bool sel = pos < n && ckey(score_key(__ldg(row + pos)), pos) >= T;
    const uint32_t word = __ballot_sync(0xffffffffu, sel);
    if (lane == 0) bm[w] = word;
  }
}

// K1 for fire selection (engine.py:326-329): top-k positions of a pivot row
// whose first-digit histogram the score-row kernel already built.  One CTA
// per satellite job, two passes over the (L2-resident) row instead of up to
// nine: (A) each warp scans its contiguous segment, counting keys above the
// threshold bucket and collecting the bucket's keys as candidates; a radix
// select over the candidates gives the exact composite threshold T, and the
// candidates >= T are added to their segments' counts; (C) after one scan
// over the 32 segment counts every warp writes its selected positions in
// ascending order (warp prefix sums, no block barriers in the loop).
constexpr int kFireCand = 12288;
constexpr int kFireSmem = kFireCand * 8 + kSelThreads * 4 + 96 * 4;

__global__ void __launch_bounds__(kSelThreads, 2) fire_select_kernel(const FireJob* __restrict__ jobs,
                                                                      const uint32_t* n_jobs_dev) {
  if (n_jobs_dev && blockIdx.x >= *n_jobs_dev) return;  // device-written job list
  extern __shared__ __align__(16) uint8_t fs_smem[];
  uint64_t* cand = reinterpret_cast<uint64_t*>(fs_smem);
  uint32_t* hist = reinterpret_cast<uint32_t*>(fs_smem + kFireCand * 8);  // radix scratch
  uint32_t* sh = hist + kSelThreads;  // [0..7]
  uint32_t* warp_tot = sh + 8;        // [32]
  uint32_t* seg = sh + 40;            // [32] per-warp selected counts -> offsets
  const FireJob job = jobs[blockIdx.x];
  const uint32_t n = job.n, k = job.k;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (k >= n || k == 0) {  // everything / nothing
    const uint32_t c = k >= n ? n : 0u;
    for (uint32_t i = tid; i < c; i += kSelThreads) job.out_idx[i] = i;
    __syncthreads();
    if (tid == 0) {
      *job.out_count = c;
      if (job.state_out) {
        __threadfence_system();
        atomicExch(job.state_out, 2);
      }
    }
    return;
  }
  block_find_bucket<kMonBins, kSelThreads>(job.hist, k, sh, warp_tot);
  const uint32_t b1 = sh[0];
  const uint32_t rem = sh[1];
  const bool whole = (sh[2] == rem);
  __syncthreads();
  if (tid == 0) sh[3] = 0;
  if (tid < 32) seg[tid] = 0;
  __syncthreads();

  const float4* __restrict__ row4 = reinterpret_cast<const float4*>(job.row);
  const uint32_t nv = (n + 3) / 4;
  const uint32_t segv = (nv + 31) / 32;
  const uint32_t wbeg = min(nv, uint32_t(warp) * segv), wend = min(nv, wbeg + segv);
  constexpr int kU = 4;
  // ---- pass A: keys above bucket b1, candidates inside it ----
  uint32_t above = 0;
  for (uint32_t v0 = wbeg + lane; v0 < wend; v0 += 32 * kU) {
    float4 x[kU];
#pragma unroll
    for (int q = 0; q < kU; ++q)
      if (v0 + q * 32 < wend) x[q] = __ldg(row4 + v0 + q * 32);
#pragma unroll
    for (int q = 0; q < kU; ++q) {
      const uint32_t v = v0 + q * 32;
      if (v >= wend) break;
      const float xs[4] = {x[q].x, x[q].y, x[q].z, x[q].w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t pos = 4 * v + e;
        if (pos >= n) break;
        const uint32_t k32 = score_key(xs[e]);
        const uint32_t d = k32 >> 19;
        if (d > b1 || (whole && d == b1)) {
          ++above;
        } else if (d == b1) {
          const uint32_t at = atomicAdd(&sh[3], 1u);
          if (at < uint32_t(kFireCand)) cand[at] = ckey(k32, pos);
        }
      }
    }
  }
  for (int off = 16; off; off >>= 1) above += __shfl_xor_sync(0xffffffffu, above, off);
  if (lane == 0) atomicAdd(&seg[warp], above);
  __syncthreads();
  uint64_t T = uint64_t(b1) << 51;
  if (!whole) {
    const uint32_t m = sh[3];
    const bool in_smem = m <= uint32_t(kFireCand);
    T = radix_threshold<kSelThreads>(job.row, n, b1, rem, in_smem ? cand : nullptr, m, hist, sh,
                                     warp_tot);
    if (in_smem) {
      for (uint32_t i = tid; i < m; i += kSelThreads) {
        const uint64_t key = cand[i];
        if (key >= T) atomicAdd(&seg[min((~uint32_t(key) >> 2) / segv, 31u)], 1u);
      }
    } else {
      for (uint32_t i = tid; i < n; i += kSelThreads) {
        const uint64_t key = ckey(score_key(__ldg(job.row + i)), i);
        if ((key >> 51) == b1 && key >= T) atomicAdd(&seg[min((i >> 2) / segv, 31u)], 1u);
      }
    }
    __syncthreads();
  }
  if (warp == 0) {  // exclusive scan of the segment counts
    const uint32_t c = seg[lane];
    uint32_t incl = c;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += u;
    }
    seg[lane] = incl - c;
  }
  __syncthreads();
  // ---- pass C: ordered write of the selected positions ----
  uint32_t off = seg[warp];
  for (uint32_t v0 = wbeg; v0 < wend; v0 += 32 * kU) {
    float4 x[kU];
#pragma unroll
    for (int q = 0; q < kU; ++q) {
      const uint32_t v = v0 + q * 32 + lane;
      if (v < wend) x[q] = __ldg(row4 + v);
    }
#pragma unroll
    for (int q = 0; q < kU; ++q) {
      const uint32_t vb = v0 + q * 32;
      if (vb >= wend) break;  // warp-uniform
      const uint32_t v = vb + lane;
      const float xs[4] = {x[q].x, x[q].y, x[q].z, x[q].w};
      uint32_t selm = 0, c = 0;
      if (v < wend) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t pos = 4 * v + e;
          if (pos < n && ckey(score_key(xs[e]), pos) >= T) {
            selm |= 1u << e;
            ++c;
          }
        }
      }
      uint32_t incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
      }
      uint32_t p = off + incl - c;
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (selm & (1u << e)) job.out_idx[p++] = 4 * v + e;
      off += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
  __syncthreads();
  if (tid == 0) {
    *job.out_count = k;
    if (job.state_out) {  // device decisions: the transfer's set is complete
      __threadfence_system();
      atomicExch(job.state_out, 2);
    }
  }
}

}  // namespace

int launch_fire_select(const FireJob* jobs_dev, int n_jobs, cudaStream_t st,
                       const uint32_t* n_jobs_dev) {
  static bool configured = false;
  if (!configured) {
    HC_CUDA_TRY(cudaFuncSetAttribute(fire_select_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, kFireSmem));
    configured = true;
  }
  if (n_jobs <= 0) return HC_OK;
  fire_select_kernel<<<n_jobs, kSelThreads, kFireSmem, st>>>(jobs_dev, n_jobs_dev);
  HC_CHECK_LAUNCH();
  return HC_OK;
}

int launch_monitor(const float* rows, int64_t row_stride, const int32_t* slots, int n_rows,
                   uint32_t n, uint32_t k, const uint32_t* kbase, int words, uint64_t* thr,
                   uint32_t* ovl, cudaStream_t st, uint32_t* hist_out) {
  static bool configured = false;
  if (!configured) {
    HC_CUDA_TRY(cudaFuncSetAttribute(monitor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kMonSmem));
    configured = true;
  }
  if (n_rows <= 0) return HC_OK;
  monitor_kernel<<<n_rows, kMonThreads, kMonSmem, st>>>(rows, row_stride, slots, n, k, kbase,
                                                        words, thr, ovl, hist_out);
  HC_CHECK_LAUNCH();
  return HC_OK;
}

int launch_restamp_threshold(const float* rows, int64_t row_stride, const int32_t* slots,
                             int n_rows, uint32_t n, const uint64_t* thr, uint32_t* kbase,
                             int words, cudaStream_t st, const uint32_t* n_rows_dev) {
  if (n_rows <= 0) return HC_OK;
  const int blocks = std::min(64, (words + 7) / 8);
  restamp_threshold_kernel<<<dim3(std::max(1, blocks), n_rows), 256, 0, st>>>(
      rows, row_stride, slots, n, thr, kbase, words, n_rows_dev);
  HC_CHECK_LAUNCH();
  return HC_OK;
}

}  // namespace hc

extern "C" int hc_monitor_rows(const float* rows_dev, int64_t row_stride, int32_t n_rows,
                               uint32_t n, uint32_t k, const uint32_t* kbase_dev, int32_t words,
                               uint64_t* thr_dev, uint32_t* ovl_dev, void* stream) {
  HC_REQUIRE(rows_dev && kbase_dev && thr_dev && ovl_dev && n_rows >= 0, HC_EINVAL,
             "hc_monitor_rows: bad arguments");
  HC_REQUIRE(row_stride % 4 == 0 && int64_t(words) * 32 >= int64_t(n), HC_EINVAL,
             "hc_monitor_rows: row stride must be a multiple of 4, bitmap must cover n");
  cudaStream_t st = (cudaStream_t)stream;
  int32_t* slots = nullptr;
  HC_CUDA_TRY(cudaMallocAsync((void**)&slots, size_t(std::max(1, n_rows)) * 4, st));
  std::vector<int32_t> iota(std::max(1, n_rows));
  for (int i = 0; i < n_rows; ++i) iota[i] = i;
  HC_CUDA_TRY(cudaMemcpyAsync(slots, iota.data(), iota.size() * 4, cudaMemcpyHostToDevice, st));
  int rc = hc::launch_monitor(rows_dev, row_stride, slots, n_rows, n, k, kbase_dev, words,
                              thr_dev, ovl_dev, st, nullptr);
  HC_CUDA_TRY(cudaFreeAsync(slots, st));
  HC_CUDA_TRY(cudaStreamSynchronize(st));
  return rc;
}
