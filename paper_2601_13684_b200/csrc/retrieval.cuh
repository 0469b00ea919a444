// Shared retrieval helpers (host-issued and device-decided transfers).
#pragma once

#include <stdint.h>

namespace hc {

// Prefix position list of a landing transfer (kv_layout.cuh): the recency
// positions in [L + t_c - R, L) the fetched set does not hold (tail-only rows,
// ascending), then sinks, then the fetched positions < L (ascending; sel is
// sorted).  Fetched positions >= L are served by the append segment.  One CTA;
// meta = {rows, tail mask (R <= 32) or tail count, fetched positions >= L}.
__device__ inline void build_positions_block(const uint32_t* sel, int k, uint32_t* pos,
                                             int32_t* meta, int L, int S, int R, int t_c) {
  __shared__ int s_lo, s_hi, s_ntail;
  __shared__ uint32_t s_mask;
  const int sinks = S < L ? S : L;
  if (threadIdx.x == 0) {
    int a = 0, b = k;
    while (a < b) { const int m = (a + b) >> 1; if (int(sel[m]) < sinks) a = m + 1; else b = m; }
    const int lo = a;
    b = k;
    while (a < b) { const int m = (a + b) >> 1; if (int(sel[m]) < L) a = m + 1; else b = m; }
    const int hi = a;
    int nt = 0;
    uint32_t mask = 0;
    int first = L + t_c - R;
    if (first < sinks) first = sinks;
    for (int p = first; p < L; ++p) {
      int u = lo, v = hi;
      while (u < v) { const int m = (u + v) >> 1; if (int(sel[m]) < p) u = m + 1; else v = m; }
      if (!(u < hi && int(sel[u]) == p)) {
        pos[nt++] = uint32_t(p);
        if (R <= 32) mask |= 1u << (p - (L - R));
      }
    }
    if (R > 32) mask = uint32_t(nt);  // contiguous tail block [L - nt, L) (no dynamic set)
    s_lo = lo;
    s_hi = hi;
    s_ntail = nt;
    s_mask = mask;
  }
  __syncthreads();
  const int nt = s_ntail, lo = s_lo, hi = s_hi;
  for (int i = threadIdx.x; i < sinks; i += blockDim.x) pos[nt + i] = uint32_t(i);
  for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) pos[nt + sinks + (i - lo)] = sel[i];
  if (threadIdx.x == 0) {
    meta[0] = nt + sinks + (hi - lo);
    meta[1] = int32_t(s_mask);
    meta[2] = k - hi;
  }
  __syncthreads();
}

// Rows pos[j0 .. n) of one transfer, warp w of nw handling every nw-th group
// of kUnroll rows: lanes 0-15 move K (16 x 16 B = 256 B), 16-31 move V.
template <int kUnroll = 4>
__device__ inline void gather_rows(const uint32_t* pos, int n, const uint4* srcK,
                                   const uint4* srcV, uint4* K, uint4* V, int64_t dst_row,
                                   int gw, int nw) {
  const int lane = threadIdx.x & 31;
  for (int j0 = gw * kUnroll; j0 < n; j0 += nw * kUnroll) {
    uint4 v[kUnroll];
#pragma unroll
    for (int q = 0; q < kUnroll; ++q) {
      const int j = j0 + q;
      if (j < n) {
        const size_t p = pos[j];
        v[q] = lane < 16 ? srcK[p * 16 + lane] : srcV[p * 16 + lane - 16];
      }
    }
#pragma unroll
    for (int q = 0; q < kUnroll; ++q) {
      const int j = j0 + q;
      if (j < n) {
        const int64_t r = dst_row + j;
        if (lane < 16) K[r * 16 + lane] = v[q];
        else V[r * 16 + lane - 16] = v[q];
      }
    }
  }
}

}  // namespace hc
