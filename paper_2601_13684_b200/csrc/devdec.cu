// Device-resident boundary decisions: kernels (see devdec.cuh).
//
// Reference semantics (engine.py:293-357), restated on the device:
//   * the window test fires iff median(overlap / l_base_int) < tau_drift --
//     values and the mean of the middle pair in float64, exactly as
//     statistics.median / np.median compute them (engine.py:247-250);
//   * per sequence, fires are accounted in sorted pivot order (engine.py:313):
//     bytes = sum over satellites of min(l_s, L + t) * bytes_per_kv_entry,
//     cumulative += bytes, completion = max(t + delay, ceil(cumulative / bw))
//     with a correctly rounded float64 division (engine.py:330-337);
//   * every pending transfer with completion <= t lands at step t in
//     (completion, order) order (engine.py:293-299); a transfer followed by
//     one of the same satellite with the same completion is overwritten in
//     the same step and never served, so it is never gathered.

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "devdec.cuh"
#include "retrieval.cuh"

namespace hc {
namespace {

__device__ __forceinline__ DevXfer& xf(const DevDec& d, int sat, int64_t ring_idx) {
  return d.xfers[size_t(sat) * d.nq + size_t(ring_idx % d.nq)];
}

__device__ __forceinline__ int32_t vload(const int32_t* p) {
  return *reinterpret_cast<const volatile int32_t*>(p);
}

// median of n float64 values (insertion sort; n <= 64)
__device__ double median_of(double* v, int n) {
  for (int i = 1; i < n; ++i) {
    const double x = v[i];
    int j = i - 1;
    while (j >= 0 && v[j] > x) {
      v[j + 1] = v[j];
      --j;
    }
    v[j + 1] = x;
  }
  return (n & 1) ? v[n / 2] : (v[n / 2 - 1] + v[n / 2]) / 2.0;
}

// The same median for n <= 16 values v_j = c_j / lb (c_j: overlap counts, lb
// > 0): the division is monotone, so the two middle values are those of the
// middle counts -- found by rank counting on integers held in registers --
// and are then formed exactly as median_of forms them.
__device__ __forceinline__ double median_counts16(const uint32_t (&c)[16], int n, double lb) {
  uint32_t lo = 0, hi = 0;
  const int k0 = (n - 1) / 2, k1 = n / 2;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    int r = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) r += (j < n && (c[j] < c[i] || (c[j] == c[i] && j < i))) ? 1 : 0;
    if (i < n && r == k0) lo = c[i];
    if (i < n && r == k1) hi = c[i];
  }
  const double vlo = double(lo) / lb, vhi = double(hi) / lb;
  return (n & 1) ? vhi : (vlo + vhi) / 2.0;
}

constexpr int kMaxPiv = 8192;

// The window test of pivot slot s at boundary t (engine.py:247-250, 313-321,
// 358-360): median of the window's overlap / l_base_int values < tau.
__device__ bool window_test(const DevDec& d, int s, int t, int first, int nvals,
                            const uint32_t* __restrict__ ovl, int ring) {
  const double lb = double(d.lbase);
  if (!d.sliding) {
    if (nvals <= 16) {
      uint32_t c[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) c[j] = j < nvals ? ovl[size_t((first + j) % ring) * d.n_piv + s] : 0u;
      return nvals > 0 && median_counts16(c, nvals, lb) < d.tau;
    }
    double v[64];
    for (int j = 0; j < nvals; ++j) v[j] = double(ovl[size_t((first + j) % ring) * d.n_piv + s]) / lb;
    return nvals > 0 && median_of(v, nvals) < d.tau;
  }
  int c = d.scnt[s];
  d.svals[size_t(s) * 64 + (c % 64)] = double(ovl[size_t(t % ring) * d.n_piv + s]) / lb;
  ++c;
  bool f = false;
  if (c >= d.window) {
    double v[64];
    for (int j = 0; j < d.window; ++j) v[j] = d.svals[size_t(s) * 64 + ((c - d.window + j) % 64)];
    f = median_of(v, d.window) < d.tau;
    if (f) c = 0;  // the buffer is cleared on a fire
  }
  d.scnt[s] = c;
  return f;
}

// The decision chain's kernels are small and latency-bound and run while K4
// holds two CTAs (2 x 160 threads x 168 registers, 2 x 97 KB of shared memory)
// on every SM.  Sized to fit beside them (256 threads, <= 42 registers, <= 24 KB
// of shared memory), they start at once instead of waiting for a K4 CTA to retire.
constexpr int kChainThreads = 256;
constexpr int kChainMinBlocks = 6;  // 65536 / (256 * 6) -> at most 42 registers
constexpr int kDecideThreads = 128, kDecideMinBlocks = 8;  // <= 64 registers, 8K in all

// One CTA.  Boundary mode: the window's values are overlap ring rows first ..
// first + nvals - 1.  Sliding mode (eval_every_step): this step's value joins
// the pivot's buffer; the test runs once it holds >= window values and clears
// it on a fire (engine.py:313-321, 358-360).  Then, per sequence in order and
// per pivot in sorted order (engine.py:313), the fires' accounting.
__global__ void __launch_bounds__(kDecideThreads, kDecideMinBlocks) decide_kernel(DevDec d, int t, int first, int nvals,
                                                      int bidx, const uint32_t* __restrict__ ovl,
                                                      int ring) {
  // The serial accounting below runs while K4 saturates HBM, where every
  // dependent global access costs microseconds: its inputs are fetched up front
  // (in parallel, or by loads whose latency the window tests hide) and the ring
  // tails it advances are kept in shared memory, not re-read.
  constexpr int kSeqSm = 256, kBumpSm = 512;
  __shared__ uint8_t fired[kMaxPiv];
  __shared__ int32_t s_seq[kSeqSm + 1], s_ord[kSeqSm];
  __shared__ int64_t s_cum[kSeqSm];
  __shared__ int32_t s_bsat[kBumpSm];
  __shared__ int64_t s_btail[kBumpSm];
  int64_t host_tail = 0, head = 0;
  unsigned long long g0 = 0, g1 = 0;
  if (d.dbg && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  if (threadIdx.x == 0) {
    host_tail = *d.fetched_tail;  // one read over the host link
    head = *d.head_dev;
  }
  const bool seq_sm = d.B <= kSeqSm;
  if (seq_sm)
    for (int b = threadIdx.x; b <= d.B; b += blockDim.x) {
      s_seq[b] = d.seq_piv[b];
      if (b < d.B) {
        s_cum[b] = d.cum[b];
        s_ord[b] = d.order[b];
      }
    }
  for (int s = threadIdx.x; s < d.n_piv; s += blockDim.x) {
    const bool f = window_test(d, s, t, first, nvals, ovl, ring);
    fired[s] = f ? 1 : 0;
    if (f) {  // warm this CTA's L1 with the satellites thread 0 is about to walk
      uint32_t touch = 0;
      for (int a = d.piv_sat_begin[s]; a < d.piv_sat_begin[s + 1]; ++a) {
        const DevSat& x = d.sats[a];
        touch += uint32_t(x.k) ^ uint32_t(x.tail) ^ uint32_t(x.head) ^
                 uint32_t(reinterpret_cast<uintptr_t>(x.sel));
      }
      if (touch == 0x9e3779b9u) fired[s] = 3;  // (keeps the loads; never true in practice,
    }                                          //  and 3 still reads as fired)
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  if (d.dbg) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  BoundaryHdr* hdr = d.hdr_dev + (bidx % kLogRing);
  FireLog* log = d.log_dev + size_t(bidx % kLogRing) * d.n_piv;
  const uint32_t* hist = d.ghist + size_t(t & 1) * d.n_piv * 8192;
  int n_fires = 0;
  uint32_t n_jobs = 0, n_rest = 0;
  for (int b = 0; b < d.B; ++b) {
    int64_t cum = seq_sm ? s_cum[b] : d.cum[b];
    int32_t ord = seq_sm ? s_ord[b] : d.order[b];
    const int s_end = seq_sm ? s_seq[b + 1] : d.seq_piv[b + 1];
    for (int s = seq_sm ? s_seq[b] : d.seq_piv[b]; s < s_end; ++s) {
      if (!fired[s]) continue;
      const int a0 = d.piv_sat_begin[s], a1 = d.piv_sat_begin[s + 1];
      const int ns = a1 - a0;
      int32_t ks[8];
      int64_t n_ent = 0;
      for (int i = 0; i < ns && i < 8; ++i) {
        const int k = min(d.sats[a0 + i].k, d.L + t);
        ks[i] = k;
        n_ent += k;
      }
      if (ns > 8) atomicExch(d.error, int(kDDTooManySats));
      const int64_t nbytes = n_ent * d.bpe;
      cum += nbytes;
      const int32_t completion = max(t + d.delay, int32_t(ceil(double(cum) / double(d.bw))));
      // fetched sets for the host mirror: one contiguous span of the mapped ring
      int64_t h = head;
      int64_t phys = h % d.fetched_cap;
      if (phys + n_ent > d.fetched_cap) {  // no wrap inside a span: skip to the ring start
        h += d.fetched_cap - phys;
        phys = 0;
      }
      int32_t host_off = int32_t(phys);
      if (h + n_ent - host_tail > d.fetched_cap || n_ent > d.fetched_cap) {
        atomicExch(d.error, int(kDDHostRingFull));
        host_off = -1;
      } else {
        head = h + n_ent;
      }
      int64_t hoff = host_off;
      for (int i = 0; i < ns && i < 8; ++i) {
        DevSat& sat = d.sats[a0 + i];
        const int64_t idx = sat.tail;
        if (idx - sat.head >= d.nq) {
          atomicExch(d.error, int(kDDRingFull));
          continue;
        }
        // its tail advances once every slot is written
        if (n_jobs < uint32_t(kBumpSm)) {
          s_bsat[n_jobs] = a0 + i;
          s_btail[n_jobs] = idx + 1;
        } else {
          d.bump[n_jobs] = a0 + i;
        }
        DevXfer& x = xf(d, a0 + i, idx);
        const int slot = int(idx % d.nq);
        x.completion = completion;
        x.order = ord++;
        x.trigger = t;
        x.k = ks[i];
        x.buf = -1;
        x.host_off = host_off < 0 ? -1 : int32_t(hoff);
        x.cnt = 0;
        x.done_chunks = 0;
        x.next_chunk = 0;
        x.built = 0;
        x.state = kXAlloc;
        FireJob& jb = d.jobs[n_jobs++];
        jb.row = d.rowbuf + size_t(s) * d.row_len;
        jb.hist = hist + size_t(s) * 8192;
        jb.n = uint32_t(d.L + t);
        jb.k = uint32_t(ks[i]);
        jb.out_idx = sat.sel + size_t(slot) * sat.k;
        jb.out_count = &x.cnt;
        jb.host_out = host_off < 0 || d.no_host_copy ? nullptr : d.fetched + hoff;
        jb.state_out = &x.state;
        hoff += ks[i];
      }
      d.restamp_slots[n_rest++] = s;
      FireLog& lg = log[n_fires++];
      lg.trigger = t;
      lg.pivot_unit = d.piv_unit[s];
      lg.completion = completion;
      lg.n_sats = ns;
      lg.bytes = nbytes;
      lg.cum_after = cum;
      lg.first_sat = a0;
      lg.host_off = host_off;
      for (int i = 0; i < 8; ++i) lg.ks[i] = i < ns ? ks[i] : 0;
    }
    if (!seq_sm || cum != s_cum[b]) d.cum[b] = cum;
    if (!seq_sm || ord != s_ord[b]) d.order[b] = ord;
  }
  // one fence for every slot written above, then the new tails: a schedule pass
  // running concurrently on another stream sees a slot only once it is complete
  __threadfence();
  for (uint32_t j = 0; j < n_jobs; ++j) {
    if (j < uint32_t(kBumpSm)) d.sats[s_bsat[j]].tail = s_btail[j];
    else ++d.sats[d.bump[j]].tail;
  }
  *d.n_jobs = n_jobs;
  *d.n_restamp = n_rest;
  *d.head_dev = head;
  hdr->t = t;
  hdr->n_fires = n_fires;
  hdr->head_after = head;
  hdr->pad = 1;
  if (d.dbg) {
    unsigned long long g2;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g2));
    d.dbg[0] += g1 - g0;  // window tests (parallel part)
    d.dbg[1] += g2 - g1;  // accounting (serial part)
    d.dbg[2] += 1;
  }
}


// The same decision for up to kFastPiv pivots and kFastSeq sequences, in four
// phases so that no thread walks a chain of dependent global accesses while K4
// saturates HBM: (1) per pivot, in parallel: the window test, and for a fire
// its satellites' entry counts and ring room; (2) one thread: the per-sequence
// accounting in sorted pivot order (engine.py:313, 330-337) over shared memory
// only; (3) per fired pivot, in parallel: its transfer slots, fire-selection
// jobs and log entry; (4) after one fence per thread and a barrier, the ring
// tails.  Results equal decide_kernel's.
constexpr int kFastPiv = 512, kFastSeq = 256;

__global__ void __launch_bounds__(kDecideThreads, kDecideMinBlocks)
decide_fast_kernel(DevDec d, int t, int first, int nvals, int bidx,
                   const uint32_t* __restrict__ ovl, int ring) {
  __shared__ int32_t f_a0[kFastPiv], f_nent[kFastPiv], f_comp[kFastPiv], f_ord0[kFastPiv];
  __shared__ int32_t f_job0[kFastPiv], f_hoff[kFastPiv], f_fidx[kFastPiv];
  __shared__ int64_t f_cum[kFastPiv];
  __shared__ uint8_t f_fired[kFastPiv], f_ns[kFastPiv], f_full[kFastPiv];
  __shared__ int32_t s_seq[kFastSeq + 1], s_ord[kFastSeq];
  __shared__ int64_t s_cum[kFastSeq];
  __shared__ uint32_t s_jobs, s_fires;
  __shared__ int64_t s_head;
  const int tid = threadIdx.x;
  unsigned long long g0 = 0, g1 = 0;
  if (d.dbg && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  int64_t host_tail = 0, head = 0;
  if (tid == 0) {  // used after the window tests: their latency hides these loads
    host_tail = *d.fetched_tail;  // one read over the host link
    head = *d.head_dev;
  }
  for (int b = tid; b <= d.B; b += blockDim.x) {
    s_seq[b] = d.seq_piv[b];
    if (b < d.B) {
      s_cum[b] = d.cum[b];
      s_ord[b] = d.order[b];
    }
  }
  const int Lt = d.L + t;
  // (1) window tests; a fire's satellites: entries and ring room
  for (int s = tid; s < d.n_piv; s += blockDim.x) {
    const bool f = window_test(d, s, t, first, nvals, ovl, ring);
    f_fired[s] = f ? 1 : 0;
    if (!f) continue;
    const int a0 = d.piv_sat_begin[s], a1 = d.piv_sat_begin[s + 1];
    const int ns = min(a1 - a0, 8);
    int32_t nent = 0;
    uint32_t full = 0;
    for (int i = 0; i < ns; ++i) {
      const DevSat& x = d.sats[a0 + i];
      nent += min(x.k, Lt);
      if (x.tail - x.head >= d.nq) full |= 1u << i;
    }
    if (a1 - a0 > 8) atomicExch(d.error, int(kDDTooManySats));
    f_a0[s] = a0;
    f_ns[s] = uint8_t(a1 - a0 > 255 ? 255 : a1 - a0);
    f_nent[s] = nent;
    f_full[s] = uint8_t(full);
  }
  __syncthreads();
  if (d.dbg && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  // (2) accounting, per sequence in sorted pivot order
  if (tid == 0) {
    uint32_t n_jobs = 0, n_fires = 0;
    for (int b = 0; b < d.B; ++b) {
      int64_t cum = s_cum[b];
      int32_t ord = s_ord[b];
      for (int s = s_seq[b]; s < s_seq[b + 1]; ++s) {
        if (!f_fired[s]) continue;
        const int64_t n_ent = f_nent[s];
        cum += n_ent * d.bpe;
        const int32_t completion = max(t + d.delay, int32_t(ceil(double(cum) / double(d.bw))));
        int64_t h = head;
        int64_t phys = h % d.fetched_cap;
        if (phys + n_ent > d.fetched_cap) {  // no wrap inside a span: skip to the ring start
          h += d.fetched_cap - phys;
          phys = 0;
        }
        int32_t host_off = int32_t(phys);
        if (h + n_ent - host_tail > d.fetched_cap || n_ent > d.fetched_cap) {
          atomicExch(d.error, int(kDDHostRingFull));
          host_off = -1;
        } else {
          head = h + n_ent;
        }
        const uint32_t full = f_full[s];
        if (full) atomicExch(d.error, int(kDDRingFull));
        const int nfree = min(int(f_ns[s]), 8) - __popc(full);
        f_comp[s] = completion;
        f_ord0[s] = ord;
        f_job0[s] = int32_t(n_jobs);
        f_hoff[s] = host_off;
        f_fidx[s] = int32_t(n_fires);
        f_cum[s] = cum;
        ord += nfree;
        n_jobs += uint32_t(nfree);
        ++n_fires;
      }
      s_cum[b] = cum;
      s_ord[b] = ord;
    }
    s_jobs = n_jobs;
    s_fires = n_fires;
    s_head = head;
  }
  __syncthreads();
  // (3) slots, jobs and log entries of every fire
  FireLog* log = d.log_dev + size_t(bidx % kLogRing) * d.n_piv;
  const uint32_t* hist = d.ghist + size_t(t & 1) * d.n_piv * 8192;
  for (int b = tid; b < d.B; b += blockDim.x) {
    d.cum[b] = s_cum[b];
    d.order[b] = s_ord[b];
  }
  for (int s = tid; s < d.n_piv; s += blockDim.x) {
    if (!f_fired[s]) continue;
    const int a0 = f_a0[s], ns = min(int(f_ns[s]), 8);
    const uint32_t full = f_full[s];
    const int32_t host_off = f_hoff[s];
    int32_t ord = f_ord0[s];
    uint32_t job = uint32_t(f_job0[s]);
    int64_t hoff = host_off;
    int32_t ks[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) ks[i] = i < ns ? min(d.sats[a0 + i].k, Lt) : 0;
    for (int i = 0; i < ns; ++i) {
      if ((full >> i) & 1u) continue;
      DevSat& sat = d.sats[a0 + i];
      const int64_t idx = sat.tail;
      DevXfer& x = xf(d, a0 + i, idx);
      const int slot = int(idx % d.nq);
      x.completion = f_comp[s];
      x.order = ord++;
      x.trigger = t;
      x.k = ks[i];
      x.buf = -1;
      x.host_off = host_off < 0 ? -1 : int32_t(hoff);
      x.cnt = 0;
      x.done_chunks = 0;
      x.next_chunk = 0;
      x.built = 0;
      x.state = kXAlloc;
      FireJob& jb = d.jobs[job++];
      jb.row = d.rowbuf + size_t(s) * d.row_len;
      jb.hist = hist + size_t(s) * 8192;
      jb.n = uint32_t(Lt);
      jb.k = uint32_t(ks[i]);
      jb.out_idx = sat.sel + size_t(slot) * sat.k;
      jb.out_count = &x.cnt;
      jb.host_out = host_off < 0 || d.no_host_copy ? nullptr : d.fetched + hoff;
      jb.state_out = &x.state;
      hoff += ks[i];
    }
    const int fi = f_fidx[s];
    d.restamp_slots[fi] = s;
    FireLog& lg = log[fi];
    lg.trigger = t;
    lg.pivot_unit = d.piv_unit[s];
    lg.completion = f_comp[s];
    lg.n_sats = f_ns[s];
    lg.bytes = int64_t(f_nent[s]) * d.bpe;
    lg.cum_after = f_cum[s];
    lg.first_sat = a0;
    lg.host_off = host_off;
#pragma unroll
    for (int i = 0; i < 8; ++i) lg.ks[i] = ks[i];
  }
  // (4) every slot is written (fence, barrier): now the ring tails
  __threadfence();
  __syncthreads();
  for (int s = tid; s < d.n_piv; s += blockDim.x) {
    if (!f_fired[s]) continue;
    const int a0 = f_a0[s], ns = min(int(f_ns[s]), 8);
    const uint32_t full = f_full[s];
    for (int i = 0; i < ns; ++i)
      if (!((full >> i) & 1u)) d.sats[a0 + i].tail += 1;
  }
  if (tid == 0) {
    *d.n_jobs = s_jobs;
    *d.n_restamp = s_fires;
    *d.head_dev = s_head;
    BoundaryHdr* hdr = d.hdr_dev + (bidx % kLogRing);
    hdr->t = t;
    hdr->n_fires = int32_t(s_fires);
    hdr->head_after = s_head;
    hdr->pad = 1;
    if (d.dbg) {
      unsigned long long g2;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g2));
      d.dbg[0] += g1 - g0;
      d.dbg[1] += g2 - g1;
      d.dbg[2] += 1;
    }
  }
}

// Which selected transfers can be gathered now: the satellite's staging
// buffer is free, or the transfer holding it is superseded at the same
// completion step.  Marks them SCHEDULED (target buffer chosen); the
// retrieval stream's next build pass picks them up.  One CTA, a thread per
// satellite.
__global__ void __launch_bounds__(kChainThreads, kChainMinBlocks) schedule_kernel(DevDec d, int t_now) {
  __shared__ int urgent;
  if (threadIdx.x == 0) urgent = 0;
  __syncthreads();
  for (int si = threadIdx.x; si < d.n_sat; si += blockDim.x) {
    DevSat& sat = d.sats[si];
    const int64_t tail = *reinterpret_cast<volatile int64_t*>(&sat.tail);
    for (int64_t i = sat.head; i < tail; ++i) {
      DevXfer& x = xf(d, si, i);
      const int32_t st = vload(&x.state);
      if (st == kXAlloc) break;  // selection still pending (ring order)
      if (st != kXSelected) continue;  // scheduled / gathered / superseded
      if (i + 1 < tail && xf(d, si, i + 1).completion == x.completion) {
        x.state = kXSuperseded;  // overwritten in its landing step: never read
        continue;
      }
      int target;
      if (sat.staging_owner < 0) {
        target = 1 - sat.active;
      } else {
        DevXfer& z = xf(d, si, sat.staging_owner);
        if (vload(&z.state) == kXGathered && z.completion == x.completion) {
          target = z.buf;  // z lands in the same step and is overwritten at once
          z.state = kXSuperseded;
        } else {
          break;  // staging busy until an earlier transfer lands
        }
      }
      x.buf = target;
      x.built = 0;  // not yet built by the retrieval stream
      __threadfence();
      sat.staging_owner = int32_t(i);
      atomicExch(&x.state, int(kXScheduled));
      if (x.completion <= t_now + 1) urgent = 1;
      break;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && urgent) {  // a running gather pass yields to the next one
    __threadfence();
    atomicAdd(d.urgent_epoch, 1u);
  }
}

// Retrieval stream, one CTA per satellite: its scheduled transfer (the
// staging buffer's) gets its prefix position list if it has none yet and joins
// this pass's list -- new ones and the remainder of ones a preempted pass left
// (the list belongs to the retrieval stream: passes never overlap).
__global__ void __launch_bounds__(kChainThreads, kChainMinBlocks) build_dev_kernel(DevDec d, int t_max) {
  const int si = blockIdx.x;
  DevSat& sat = d.sats[si];
  __shared__ int64_t s_i;
  __shared__ int s_new;
  if (threadIdx.x == 0) {
    s_i = -1;
    s_new = 0;
    const int64_t tail = *reinterpret_cast<volatile int64_t*>(&sat.tail);
    for (int64_t i = sat.head; i < tail; ++i) {
      DevXfer& x = xf(d, si, i);
      if (vload(&x.state) == kXScheduled && x.built != 2) {
        if (x.completion <= t_max) {  // later passes take the later deadlines
          s_i = i;
          s_new = x.built == 0;
        }
        break;
      }
    }
  }
  __syncthreads();
  if (s_i < 0) return;
  DevXfer& x = xf(d, si, s_i);
  const int slot = int(s_i % d.nq);
  if (s_new)
    build_positions_block(sat.sel + size_t(slot) * sat.k, int(x.cnt),
                          sat.pos + size_t(x.buf) * sat.cap, x.meta, d.L, d.S, d.R,
                          x.completion);
  if (threadIdx.x == 0) {
    x.built = 1;
    const uint32_t at = atomicAdd(d.n_glist, 1u);
    d.glist[at] = GatherItem{si, slot, x.completion, x.order};
  }
}

// Earliest deadline first: rank sort of the pass's list by (completion,
// sequence, order) into glist2.
__global__ void __launch_bounds__(kChainThreads, kChainMinBlocks) order_kernel(DevDec d) {
  const uint32_t n = *d.n_glist;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    const GatherItem a = d.glist[i];
    const int sa = d.sats[a.sat].seq;
    uint32_t r = 0;
    for (uint32_t j = 0; j < n; ++j) {
      const GatherItem c = d.glist[j];
      const int sc = d.sats[c.sat].seq;
      const bool less = c.completion < a.completion ||
                        (c.completion == a.completion &&
                         (sc < sa || (sc == sa && (c.order < a.order ||
                                                   (c.order == a.order && j < i)))));
      r += less ? 1u : 0u;
    }
    d.glist2[r] = a;
  }
}

// Rows are claimed in chunks of kChunkRows, earliest deadline first, by
// whichever CTA is free; before each claim a CTA checks the urgent epoch and
// leaves if a transfer due next step was scheduled after this pass started --
// the next pass (queued behind this one) re-lists the remainders with the new
// transfer in deadline order.  A claimed chunk is always finished; the CTA
// completing a transfer's last chunk flags it GATHERED.
constexpr int kChunkRows = 256;  // default of DevDec::gather_chunk

__global__ void __launch_bounds__(kChainThreads, kChainMinBlocks) gather_dev_kernel(DevDec d, uint4* __restrict__ K,
                                                         uint4* __restrict__ V) {
  const uint32_t n = *d.n_glist;
  __shared__ uint32_t s_epoch, s_c;
  __shared__ int s_stop;
  if (threadIdx.x == 0) {
    s_epoch = *reinterpret_cast<volatile uint32_t*>(d.urgent_epoch);
    s_stop = 0;
  }
  __syncthreads();
  const int wid = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  for (uint32_t i = 0; i < n; ++i) {
    const GatherItem it = d.glist2[i];
    const DevSat& sat = d.sats[it.sat];
    DevXfer& x = d.xfers[size_t(it.sat) * d.nq + it.slot];
    const int rows = x.meta[0];
    const int chunk_rows = d.gather_chunk;
    const uint32_t n_chunks = uint32_t((rows + chunk_rows - 1) / chunk_rows);
    if (n_chunks == 0) {
      if (threadIdx.x == 0) atomicCAS(&x.state, int(kXScheduled), int(kXGathered));
      continue;
    }
    while (true) {
      if (threadIdx.x == 0) {
        if (*reinterpret_cast<volatile uint32_t*>(d.urgent_epoch) != s_epoch) s_stop = 1;
        s_c = s_stop ? n_chunks : atomicAdd(&x.next_chunk, 1u);
      }
      __syncthreads();
      const uint32_t c = s_c;
      const int stop = s_stop;
      __syncthreads();
      if (stop) return;
      if (c >= n_chunks) break;
      const int r0 = int(c) * chunk_rows;
      const int nr = min(chunk_rows, rows - r0);
      gather_rows(sat.pos + size_t(x.buf) * sat.cap + r0, nr, sat.srcK, sat.srcV, K, V,
                  sat.row0[x.buf] + r0, wid, nwarps);
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(&x.done_chunks, 1u) == n_chunks - 1) {
          __threadfence();
          atomicExch(&x.state, int(kXGathered));
        }
      }
    }
  }
}

__device__ void land_one(const DevDec& d, DevSat& sat, DevXfer& x, int64_t idx, UnitDesc* units) {
  UnitDesc& u = units[sat.unit];
  u.row0 = sat.row0[x.buf];
  u.n_prefix = x.meta[0];
  u.tail_mask = uint32_t(x.meta[1]);
  u.pad_ = x.meta[2];
  sat.active = x.buf;
  sat.cur_slot = int32_t(idx % d.nq);
  if (sat.staging_owner == int32_t(idx)) sat.staging_owner = -1;
  sat.head = idx + 1;
}

// Landing point of step t (engine.py:293-299).  One small CTA (it runs beside
// the step's main attention), a thread per satellite.
__global__ void __launch_bounds__(kChainThreads, kChainMinBlocks) land_kernel(DevDec d, int t, UnitDesc* units,
                                                    uint4* __restrict__ K,
                                                    uint4* __restrict__ V) {
  __shared__ int32_t inl_sat[2048];
  __shared__ int64_t inl_idx[2048];
  __shared__ uint32_t n_inl;
  for (int round = 0; round < 4; ++round) {
    if (threadIdx.x == 0) n_inl = 0;
    __syncthreads();
    for (int si = threadIdx.x; si < d.n_sat; si += blockDim.x) {
      DevSat& sat = d.sats[si];
      while (sat.head < sat.tail) {
        const int64_t i = sat.head;
        DevXfer& x = xf(d, si, i);
        if (x.completion > t) break;
        int32_t st = vload(&x.state);
        if (st == kXSuperseded) {
          if (sat.staging_owner == int32_t(i)) sat.staging_owner = -1;
          sat.head = i + 1;
          continue;
        }
        if (st == kXSelected && i + 1 < sat.tail && xf(d, si, i + 1).completion == x.completion) {
          x.state = kXSuperseded;
          sat.head = i + 1;
          continue;
        }
        if (st == kXScheduled) {  // in flight on the retrieval stream: wait (bounded)
          const long long t0 = clock64();
          while ((st = vload(&x.state)) == kXScheduled) {
            __nanosleep(2000);
            if (clock64() - t0 > (long long)8e9) {  // ~4 s
              atomicExch(d.error, int(kDDSpinTimeout));
              break;
            }
          }
          if (st != kXGathered) break;
        }
        if (st == kXGathered) {
          __threadfence();
          land_one(d, sat, x, i, units);
          continue;
        }
        // selected but never scheduled: its staging buffer was busy until a
        // landing of this very pass -- gather it inline below
        if (st == kXSelected) {
          x.buf = 1 - sat.active;
          x.built = 2;  // gathered here, never by a retrieval pass
          __threadfence();
          x.state = kXScheduled;
          sat.staging_owner = int32_t(i);
          const uint32_t at = atomicAdd(&n_inl, 1u);
          if (at < 2048) {
            inl_sat[at] = si;
            inl_idx[at] = i;
          }
        }
        break;
      }
    }
    __syncthreads();
    const uint32_t n = min(n_inl, 2048u);
    if (n == 0) break;
    for (uint32_t q = 0; q < n; ++q) {  // the whole CTA gathers each inline transfer
      const int si = inl_sat[q];
      DevSat& sat = d.sats[si];
      DevXfer& x = xf(d, si, inl_idx[q]);
      const int slot = int(inl_idx[q] % d.nq);
      build_positions_block(sat.sel + size_t(slot) * sat.k, int(x.cnt),
                            sat.pos + size_t(x.buf) * sat.cap, x.meta, d.L, d.S, d.R,
                            x.completion);
      gather_rows(sat.pos + size_t(x.buf) * sat.cap, x.meta[0], sat.srcK, sat.srcV, K, V,
                  sat.row0[x.buf], threadIdx.x >> 5, blockDim.x >> 5);
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        x.state = kXGathered;
      }
      __syncthreads();
    }
    // next round lands them (and anything due behind them)
  }
}

// The boundary's fetched sets to the host mirror's mapped ring: one CTA per
// fire-selection job, coalesced stores over the host link, on a low-priority
// stream after the selection -- never between a decision and its gathers.
__global__ void __launch_bounds__(256) copy_fetched_kernel(DevDec d, int bidx) {
  if (blockIdx.x == gridDim.x - 1) {  // the decision log of this boundary
    const int r = bidx % kLogRing;
    const BoundaryHdr* hs = d.hdr_dev + r;
    const int n = hs->n_fires;
    const int32_t* src = reinterpret_cast<const int32_t*>(d.log_dev + size_t(r) * d.n_piv);
    int32_t* dst = reinterpret_cast<int32_t*>(d.log + size_t(r) * d.n_piv);
    const int words = n * int(sizeof(FireLog) / 4);
    for (int i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      d.hdr[r] = *hs;
    }
    return;
  }
  if (blockIdx.x >= *d.n_jobs) return;
  const FireJob jb = d.jobs[blockIdx.x];
  if (!jb.host_out) return;
  const uint32_t n = *jb.out_count;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) jb.host_out[i] = jb.out_idx[i];
}

}  // namespace

int launch_copy_fetched(const DevDec& d, int bidx, cudaStream_t st) {
  copy_fetched_kernel<<<std::max(1, d.n_sat) + 1, 256, 0, st>>>(d, bidx);
  HC_CHECK_LAUNCH();
  return HC_OK;
}

bool getenv_serial_decide() {  // tests: force the general kernel (read per boundary)
  return getenv("HC_DECIDE_SERIAL") != nullptr;
}

int launch_decide(const DevDec& d, int t, int first, int nvals, int bidx, const uint32_t* ovl_ring,
                  int ring, cudaStream_t st) {
  HC_REQUIRE(nvals <= 64 && d.window <= 64, HC_EINVAL, "decision window > 64");
  HC_REQUIRE(d.n_piv <= kMaxPiv, HC_EINVAL, "more than %d monitored pivots", kMaxPiv);
  if (d.n_piv <= kFastPiv && d.B <= kFastSeq && !getenv_serial_decide())
    decide_fast_kernel<<<1, kDecideThreads, 0, st>>>(d, t, first, nvals, bidx, ovl_ring, ring);
  else
    decide_kernel<<<1, kDecideThreads, 0, st>>>(d, t, first, nvals, bidx, ovl_ring, ring);
  HC_CHECK_LAUNCH();
  return HC_OK;
}

int launch_schedule(const DevDec& d, int t_now, cudaStream_t st) {
  schedule_kernel<<<1, kChainThreads, 0, st>>>(d, t_now);
  HC_CHECK_LAUNCH();
  return HC_OK;
}

int launch_dev_gathers(const DevDec& d, uint4* K, uint4* V, cudaStream_t st, int t_max,
                       cudaEvent_t g0, cudaEvent_t g1) {
  HC_CUDA_TRY(cudaMemsetAsync(d.n_glist, 0, 4, st));
  build_dev_kernel<<<std::max(1, d.n_sat), kChainThreads, 0, st>>>(d, t_max);
  HC_CHECK_LAUNCH();
  order_kernel<<<1, kChainThreads, 0, st>>>(d);
  HC_CHECK_LAUNCH();
  if (g0) HC_CUDA_TRY(cudaEventRecord(g0, st));
  gather_dev_kernel<<<d.gather_ctas, kChainThreads, 0, st>>>(d, K, V);
  if (g1) HC_CUDA_TRY(cudaEventRecord(g1, st));
  HC_CHECK_LAUNCH();
  return HC_OK;
}

int launch_land(const DevDec& d, int t, UnitDesc* units, uint4* K, uint4* V, cudaStream_t st) {
  land_kernel<<<1, kChainThreads, 0, st>>>(d, t, units, K, V);
  HC_CHECK_LAUNCH();
  return HC_OK;
}

}  // namespace hc
