// Device-resident boundary decisions (engine.py:305-357 on the GPU).
//
// With device decisions on, a decode step never waits for the host: the
// window median test, the per-sequence byte accounting and completion steps,
// the fetch selection, the retrieval gathers and the landings all run on
// device streams, driven by the state below; the host mirrors the decisions
// from a mapped log afterwards (decoder.py) for its StepRows / RetrievalRecords.
//
//   decide_kernel    (monitor stream, after the monitor of a boundary step):
//                    median of the window's overlap values per pivot, fires
//                    in sorted pivot order per sequence, bytes, cumulative
//                    bytes, completion = max(t + delay, ceil(cum / bw)); one
//                    transfer slot per satellite in its ring; fire-selection
//                    jobs and the K_base restamp list; the host log
//   fire_select      (side stream) over the jobs the decide kernel wrote
//   schedule_kernel  (schedule stream, after every landing pass and every
//                    boundary's selection): which selected transfers can be
//                    gathered now (the satellite's staging buffer is free, or
//                    the staging transfer is superseded at the same
//                    completion step), in (completion, order) order
//   build/gather     (retrieval stream) over the scheduled list; each transfer
//                    is flagged GATHERED when all CTAs finished its rows
//   land_kernel      (the step's stream, before the held satellites' K4):
//                    every transfer with completion <= t lands in (completion,
//                    order) order (engine.py:293-299); a due transfer still in
//                    flight is waited for (bounded spin), one that could not be
//                    scheduled (its staging buffer was busy until this very
//                    landing) is gathered inline.
#pragma once

#include <stdint.h>

#include "hc_common.cuh"
#include "kv_layout.cuh"

namespace hc {

constexpr int kLogRing = 256;  // boundaries the mapped host log holds

enum XState : int32_t {
  kXFree = 0,
  kXAlloc = 1,       // decided, selection pending
  kXSelected = 2,    // fetched set written
  kXScheduled = 3,   // gather issued into buf
  kXGathered = 4,    // rows in buf
  kXSuperseded = 5,  // lands together with a later transfer of the same satellite: never read
};

struct DevXfer {
  int32_t completion, order, trigger, k;
  int32_t state, buf, host_off, built;  // built: 0 no, 1 positions built, 2 gathered inline
  int32_t meta[4];  // prefix rows, tail mask, positions >= L (build_positions)
  uint32_t cnt, done_chunks;
  uint32_t next_chunk, pad_;  // gather progress: chunks claimed / completed
};

struct DevSat {
  int32_t unit, pivot_slot, k, cap;  // k: planned length l_s; cap: prefix capacity
  int32_t active, staging_owner, cur_slot, seq;
  int64_t head, tail;                // ring counters (slot = counter % kQ)
  int64_t row0[2];                   // the two prefix buffers' first arena rows
  uint32_t* sel;                     // [nq][k] fetched sets of the ring's transfers
  uint32_t* pos;                     // [2][cap] prefix position lists of the two buffers
  const uint4* srcK;                 // host pool (mapped pinned) prefill K / V of the satellite
  const uint4* srcV;
};

// one fire of a boundary, as the host mirror reads it
struct FireLog {
  int32_t trigger, pivot_unit, completion, n_sats;
  int64_t bytes, cum_after;
  int32_t first_sat;   // index of the pivot's first satellite in DevSat order
  int32_t host_off;    // fetched sets, concatenated in satellite order, in the host ring
  int32_t ks[8];       // fetched counts per satellite (clusters have <= 8 satellites here)
};

struct BoundaryHdr {
  int32_t t, n_fires, overflow, pad;
  int64_t head_after;  // fetched-ring head after this boundary (host releases up to it)
};

struct GatherItem {
  int32_t sat, slot, completion, order;
};

struct DevDec {
  // static geometry
  int32_t n_sat, n_piv, B, L, S, R, lbase, window, sliding, delay;
  int32_t nq, no_host_copy;  // transfer slots per satellite ring; diagnostics switch
  int32_t gather_ctas, gather_chunk;  // retrieval gather grid and rows per claimed chunk
  double tau;
  int64_t bw, bpe;
  int32_t* seq_piv;        // [B + 1] pivot slot ranges per sequence
  int32_t* piv_sat_begin;  // [n_piv + 1] satellites of each pivot (DevSat indices)
  int32_t* piv_unit;       // [n_piv]
  const float* rowbuf;     // pivot probability rows [n_piv][row_len]
  int64_t row_len;
  const uint32_t* ghist;   // [2][n_piv][8192] the monitor's key histograms (step parity)
  DevSat* sats;            // [n_sat]
  DevXfer* xfers;          // [n_sat][nq]
  // per-sequence accounting
  int64_t* cum;            // [B]
  int32_t* order;          // [B]
  // sliding-window buffers (eval_every_step)
  double* svals;           // [n_piv][64]
  int32_t* scnt;           // [n_piv]
  // per-boundary work lists (written by decide)
  FireJob* jobs;           // [n_sat]
  int32_t* bump;           // [n_sat] the satellite of each job (its ring tail advances)
  uint32_t* n_jobs;
  int32_t* restamp_slots;  // [n_piv]
  uint32_t* n_restamp;
  uint32_t* urgent_epoch;  // bumped when a transfer due next step is scheduled: a
                           // running gather pass yields (between chunks) to the next
  GatherItem* glist;       // [n_sat] this gather pass (retrieval stream)
  GatherItem* glist2;      // [n_sat] the same, earliest deadline first
  uint32_t* n_glist;
  // the decision log: written in device memory by decide_kernel, copied to the
  // host-mapped copies by copy_fetched_kernel (low priority, off the chain to
  // the gathers); the fetched-set ring is host-mapped
  BoundaryHdr* hdr_dev;    // [kLogRing]
  FireLog* log_dev;        // [kLogRing][n_piv]
  int64_t* head_dev;       // the fetched ring's virtual head
  BoundaryHdr* hdr;        // [kLogRing] mapped
  FireLog* log;            // [kLogRing][n_piv] mapped
  uint32_t* fetched;       // [fetched_cap] host ring (mapped)
  int64_t fetched_cap;
  volatile int64_t* fetched_tail;  // host-written (mapped): entries consumed
  int32_t* error;          // mapped: 0 ok, else an error code
  unsigned long long* dbg; // diagnostics (HC_CHAIN_TRACE): decide-kernel phase times, or null
};

enum DevDecError : int32_t {
  kDDOk = 0,
  kDDRingFull = 1,     // more than nq transfers pending for one satellite
  kDDHostRingFull = 2, // the host has not consumed the fetched-set ring
  kDDSpinTimeout = 3,  // a due gather never completed
  kDDTooManySats = 4,
};

int launch_decide(const DevDec& d, int t, int first, int nvals, int bidx, const uint32_t* ovl_ring,
                  int ring, cudaStream_t st);
int launch_schedule(const DevDec& d, int t_now, cudaStream_t st);
int launch_copy_fetched(const DevDec& d, int bidx, cudaStream_t st);
int launch_dev_gathers(const DevDec& d, uint4* K, uint4* V, cudaStream_t st, int t_max,
                       cudaEvent_t g0 = nullptr, cudaEvent_t g1 = nullptr);
int launch_land(const DevDec& d, int t, UnitDesc* units, uint4* K, uint4* V, cudaStream_t st);

}  // namespace hc
