// Tensor-mode engine handle: the hierarchical KV store, the per-step decode
// pipeline (append -> K4 attention -> combine -> pivot score rows -> K1/K2
// drift monitor) and K3 retrieval from the pinned host pool.
//
// Mirrors the reference engine's lifecycle (engine.py:153-416):
//   hc_engine_create         CacheEngine.__init__ geometry / plan  (engine.py:156-214)
//   hc_engine_prefill_layer  prefill_init                          (engine.py:263-274)
//   hc_engine_decode_step    decode_step steps 2-4                 (engine.py:301-311)
//     = decode_begin + decode_end, split so the previous boundary's decision
//     can run beside the step's attention
//   hc_engine_fire[_batch]   fetch loop + K_base restamp           (engine.py:322-357)
//   hc_engine_land[_batch]   landing of due transfers              (engine.py:293-299)
//   hc_engine_measure        _measure / attention_recall           (engine.py:276-288)
// The window median / completion-step arithmetic stays in the Python mirror
// (decoder.py), exactly as the reference writes it.
//
// Streams: the caller's stream runs the step; `mon` runs each step's monitor
// beside the next step's attention; `side` runs fire selection and in-step
// readbacks; `retr` (high priority) runs the retrieval gathers.  Events
// (step_end, rows_done, selected, gather done) order every hand-off.

#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <new>
#include <optional>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "hc_common.cuh"
#include "kv_layout.cuh"
#include "retrieval.cuh"
#include "devdec.cuh"

namespace hc {

int make_kv_tensor_map(CUtensorMap* map, const void* base, int64_t rows);
int launch_combine(const AttnParams& p, cudaStream_t st);
int launch_score_rows(const AttnParams& p, const int32_t* pivot_units_dev, int n_pivots,
                      cudaStream_t st);
int launch_attn_tiles(const CUtensorMap& tmK, const CUtensorMap& tmV, const AttnParams& p,
                      int n_tiles, cudaStream_t st);
int launch_topk(const hc_topk_job* jobs_dev, int n_jobs, uint32_t n_add, cudaStream_t st);
size_t obs_scratch_bytes(int n_units, int L, int rows);
int launch_obs_scores(const void* k, const void* q_obs, int B, int H, int G, int w, int L,
                      float* out, int64_t row_stride, void* scratch, cudaStream_t st, int64_t kstride = 0);
int launch_monitor(const float* rows, int64_t row_stride, const int32_t* slots, int n_rows,
                   uint32_t n, uint32_t k, const uint32_t* kbase, int words, uint64_t* thr,
                   uint32_t* ovl, cudaStream_t st, uint32_t* hist_out = nullptr);
int launch_fire_select(const FireJob* jobs_dev, int n_jobs, cudaStream_t st,
                       const uint32_t* n_jobs_dev = nullptr);
int segmented_sort_desc_u64(void* temp, size_t* temp_bytes, const uint64_t* in, uint64_t* out,
                            int n_items, int n_segments, const int* offsets, cudaStream_t st);
int launch_restamp_threshold(const float* rows, int64_t row_stride, const int32_t* slots,
                             int n_rows, uint32_t n, const uint64_t* thr, uint32_t* kbase,
                             int words, cudaStream_t st, const uint32_t* n_rows_dev = nullptr);

namespace {

constexpr int kRing = 64;  // overlap-count ring (steps), read back at window boundaries

// ---- kernels: append, position lists, row gathers -------------------------

// Append the decode token of step t (position L+t-1) to every unit.
__global__ void append_kernel(const UnitDesc* __restrict__ units, int n_units, int L, int t,
                              const uint4* __restrict__ k_new, const uint4* __restrict__ v_new,
                              uint4* __restrict__ K, uint4* __restrict__ V,
                              uint4* __restrict__ shadow, int NL, int H, int64_t srows) {
  const int u = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (u >= n_units) return;
  const UnitDesc d = units[u];
  if (d.kind == kUnitAbsent) return;
  const int64_t row = d.kind == kUnitFull ? d.row0 + L + t - 1 : d.app_row + t - 1;
  // 256 B per row = 16 x uint4; lanes 0-15 move K, 16-31 move V
  if (lane < 16) {
    const uint4 x = k_new[size_t(u) * 16 + lane];
    K[row * 16 + lane] = x;
    if (shadow) {  // measure mode: full-context K, layout [layer][b*H + h][srows]
      const int h = u % H, l = (u / H) % NL, b = u / (NL * H);
      const int64_t B = n_units / (NL * H);
      const int64_t srow = ((int64_t(l) * B + b) * H + h) * srows + L + t - 1;
      shadow[srow * 16 + lane] = x;
    }
  } else {
    V[row * 16 + lane - 16] = v_new[size_t(u) * 16 + lane - 16];
  }
}


struct Transfer {
  int unit = -1;
  int k = 0;
  int completion = 0;
  int buf = -1;
  uint32_t* sel = nullptr;  // [k] fetched positions
  uint32_t* cnt = nullptr;  // [1]
  uint32_t* pos = nullptr;  // [prefix capacity]
  int32_t* meta = nullptr;  // [3]
  int block = -1;           // the fire batch's device allocation these point into
  bool gathered = false;
  bool landed = false;
  cudaEvent_t selected = nullptr;  // caller's stream, after selection (shared per batch)
  cudaEvent_t done = nullptr;      // retrieval stream, after the gather (shared per batch)
};


int dalloc(void** p, size_t bytes, int64_t* counter) {
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaSuccess) {
    *p = nullptr;
    set_error("cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(e));
    return HC_ENOMEM;
  }
  if (counter) *counter += int64_t(bytes);
  HC_CUDA_TRY(cudaMemset(*p, 0, bytes));
  return HC_OK;
}

}  // namespace

// Host submission profile (diagnostics: HC_HOST_PROF=1 prints, at engine
// destroy, the host time spent per decode-step section).
struct HostProf {
  static constexpr int kN = 12;
  bool on = getenv("HC_HOST_PROF") != nullptr;
  double ns[kN] = {};
  long n[kN] = {};
};
HostProf g_hprof;
const char* const kHostProfNames[HostProf::kN] = {
    "decode_begin", "append", "k4_main", "devdec_land", "schedule_gather", "k4_sats",
    "decode_end", "combine", "rows_monitor", "decide", "gc_events", "step_host"};
struct HostProfScope {
  int k;
  std::chrono::steady_clock::time_point t0;
  explicit HostProfScope(int k_) : k(g_hprof.on ? k_ : -1) {
    if (k >= 0) t0 = std::chrono::steady_clock::now();
  }
  ~HostProfScope() {
    if (k < 0) return;
    g_hprof.ns[k] += std::chrono::duration<double, std::nano>(std::chrono::steady_clock::now() - t0).count();
    ++g_hprof.n[k];
  }
};
void host_prof_report() {
  if (!g_hprof.on) return;
  for (int k = 0; k < HostProf::kN; ++k)
    if (g_hprof.n[k])
      fprintf(stderr, "hc_host_prof %-16s %8ld calls %9.2f us/call\n", kHostProfNames[k],
              g_hprof.n[k], g_hprof.ns[k] / g_hprof.n[k] * 1e-3);
}

struct EngineImpl {
  hc_engine_desc cfg{};
  int B = 0, NL = 0, H = 0, G = 0, Hq = 0, L = 0, T = 0, S = 0, R = 0, CH = 0, lbase = 0;
  int n_units = 0;
  int64_t dev_bytes = 0, host_bytes = 0;
  std::vector<int32_t> role, length, cpivot;
  std::vector<uint8_t> owned;  // per unit: 0 = absent (another shard's)
  int n_absent = 0;
  std::vector<UnitDesc> units;
  UnitDesc* d_units = nullptr;
  int64_t rows = 0;
  __nv_bfloat16 *K = nullptr, *V = nullptr;
  CUtensorMap tmK{}, tmV{};
  std::vector<uint32_t> t_act;  // sorted activation steps of the tile table
  std::vector<TileDesc> tiles_host;          // the tile table (host copy, same order)
  std::vector<std::vector<int>> unit_tiles;  // per unit: its entries in the tile table
  TileDesc* d_tiles = nullptr;
  uint8_t* d_skip = nullptr;                 // per unit: K4 tiles deferred past a landing
  // landings requested by hc_engine_land_batch, applied inside the next decode
  // step: K4 runs every other unit while the gathers finish (see decode_step)
  std::vector<int> deferred;
  cudaStream_t deferred_st = nullptr;
  // satellites: static tile list + K4 skip flags for steps whose fire
  // decision is still open (hold_satellites, see decode_begin)
  TileDesc* d_sat_tiles = nullptr;
  std::vector<uint32_t> sat_t_act;
  // pivot-first step (device decisions): the pivots' tiles, then every other
  // unit's tiles on a second stream beside them; the boundary chain (the
  // pivots' combine, score rows, monitor, decision) starts when the pivots are done
  bool pivot_first = false;
  TileDesc* d_piv_tiles = nullptr;
  TileDesc* d_rest_tiles = nullptr;
  std::vector<uint32_t> piv_t_act, rest_t_act;
  cudaStream_t kst2 = nullptr;
  cudaEvent_t ev_k4s = nullptr, ev_piv = nullptr, ev_rest = nullptr, ev_pc = nullptr;
  cudaEvent_t step_out = nullptr;  // pivot-first: the step's O complete (caller's stream)
  uint8_t* d_sat_flags = nullptr;
  // the open step between decode_begin and decode_end
  int in_step = 0;
  bool cur_hold = false;
  cudaStream_t cur_st = nullptr;
  AttnParams cur_p{};
  cudaEvent_t* cur_ev = nullptr;
  std::vector<int> cur_land;
  int32_t* d_land = nullptr;
  int n_lu = 0, n_lt = 0;
  cudaEvent_t step_end = nullptr;  // monitor of the last completed step done (rows free again,
                                   // overlap counts, thresholds and histograms valid)
  cudaEvent_t rows_done = nullptr;     // combine of the last step done (main stream)
  cudaEvent_t rows_ev[2] = {nullptr, nullptr};  // score rows of steps with parity 0 / 1 done
  cudaStream_t mon = nullptr;      // the monitor runs beside the next step's attention
  cudaStream_t side = nullptr;     // fire selection and control readbacks inside a step
  int n_slots = 0;
  float* partial = nullptr;
  // pivots
  std::vector<int32_t> piv_units, piv_slot;  // piv_slot: unit -> slot or -1
  int32_t* d_piv_units = nullptr;
  int n_piv = 0;
  int64_t row_len = 0;
  int words = 0;
  void* logits = nullptr;  // per-token pivot material (fp32, or fp16 when mat_f16)
  int mat_f16 = 0;
  size_t mat_bytes = 4;    // bytes per material element
  float *mref = nullptr, *stats = nullptr, *rowbuf = nullptr;
  uint32_t *top_idx = nullptr, *top_cnt = nullptr, *kbase = nullptr;
  uint32_t* ovl_ring = nullptr;
  uint32_t* ovl_host = nullptr;     // pinned readback of the overlap window
  uint64_t* thr = nullptr;          // per pivot slot: composite-key threshold of its top set
  uint32_t* ghist = nullptr;        // [2][pivot slot][8192] first-digit key histograms of the
                                    // rows: step t's monitor fills buffer t&1 for its fires
  int32_t* d_piv_slots = nullptr;   // iota over pivot slots
  int last_t = 0;                   // last decode step run
  // compressed units
  std::vector<int32_t> cap;               // prefix capacity per unit (0 for full)
  std::vector<int64_t> buf_row0, buf_row1;
  std::vector<int> active;
  std::vector<uint32_t*> dyn_sel;          // current dynamic set (device) per comp unit
  std::vector<uint32_t*> dyn_cnt;
  std::vector<int> dyn_owner;              // transfer id owning dyn_sel, or -1 (prefill buffer)
  std::vector<uint32_t*> pre_pos;          // prefix positions of the active buffer
  std::vector<int32_t*> pre_meta;
  std::vector<std::deque<int>> fifo;       // pending transfers per unit
  // host pool
  std::vector<int32_t> sat_slot;
  int n_sat = 0;
  __nv_bfloat16* pool = nullptr;          // [n_sat][2][L][128]
  bool pool_host = true;
  // transfers by id (ids increase monotonically); a record is dropped once a
  // later landing supersedes it, so the table holds only pending transfers and
  // the ones serving a satellite right now -- bounded over any decode length
  // one device allocation per fire batch holds every transfer's buffers (all
  // fetched sets contiguous first: one D2H copy); freed with its last transfer
  struct XferBlock {
    void* ptr;
    int refs;
  };
  std::unordered_map<int, XferBlock> blocks;
  int next_block = 0;
  struct TransferTable {
    std::unordered_map<int, Transfer> m;
    int next = 0;
    Transfer& operator[](int id) { return m.at(id); }
    const Transfer& operator[](int id) const { return m.at(id); }
    bool contains(int id) const { return m.count(id) != 0; }
    int add(const Transfer& x) { m.emplace(next, x); return next++; }
    void erase(int id) { m.erase(id); }
  } xfers;
  // owned ordering events (fires, gathers, landings), with the step that made
  // them; gc_events() retires the completed, unreferenced ones
  std::deque<std::pair<cudaEvent_t, int>> events;
  // pinned staging ring for small host->device descriptor uploads: keeps every
  // cudaMemcpyAsync truly asynchronous (pageable sources may sync the stream)
  char* stage = nullptr;
  size_t stage_cap = 0, stage_head = 0;
  std::deque<std::tuple<size_t, size_t, cudaEvent_t>> stage_busy;  // (lo, hi, copy done)
  cudaStream_t retr = nullptr;
  cudaMemPool_t mpool = nullptr;  // private stream-ordered pool (descriptors, transfer blocks)
  // decode_step_host: copy stream, double-buffered device staging, ordering events
  cudaStream_t hcopy = nullptr, hdown = nullptr;  // uploads / downloads
  void* hbuf[2] = {nullptr, nullptr};
  cudaEvent_t h_in[2] = {}, h_used[2] = {}, h_out[2] = {};
  int h_last = -1;
  bool small_io = false;  // decode_step_host moves its inputs / output by zero-copy kernels
  std::vector<std::pair<const void*, void*>> hmap;  // pinned host -> device-mapped pointer
  cudaEvent_t last_selected = nullptr;  // side stream: the last fire batch's copies are done
  // per-step phase timeline (bench roofline): 7 events per step: start |
  // append | K4 | combine (step stream) | score rows | monitor (monitor
  // stream) | end (step stream)
  static constexpr int kPhaseEvents = 7;
  bool timing = false;
  bool timing_light = false;  // only the attention phase (ev[1] -> ev[2]) is recorded
  // decision-chain trace (diagnostics, HC_CHAIN_TRACE=1): per boundary t, timed
  // events from step t's combine to step t+1's satellites
  static constexpr int kChainMarks = 11;
  bool chain_trace = getenv("HC_CHAIN_TRACE") != nullptr;
  std::vector<std::array<cudaEvent_t, kChainMarks>> ctr;
  int ctr_open = -1;    // trace of the boundary whose landing step has not run yet
  int ctr_step = -1;    // that step
  bool ctr_in_decide = false;
  std::vector<cudaEvent_t> tpool;  // timed events for gather / landing pairs, reused
  std::vector<cudaEvent_t> tev;
  size_t tev_used = 0;  // steps recorded
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> gather_ev;  // retrieval-stream gathers
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> land_ev;    // caller-stream landing waits
  int64_t gather_rows_issued = 0;
  // prefill scratch
  int W = 1;                        // observation window (prompt tokens scored)
  cudaEvent_t pf_ev0 = nullptr, pf_ev1 = nullptr;
  double pf_score_ms = 0;
  int pf_layers = 0;
  float* prefill_dump = nullptr;
  char* pf = nullptr;
  size_t pf_bytes = 0;

  // measure mode: attention-mass recall at scale (CacheEngine._measure,
  // engine.py:276-288).  Every head's dense GQA-mean row
  // per step (K5 over a full-context K copy; pivots keep their own K4 rows),
  // its top records, and recall against the resident sets, all on the GPU.
  int rec_k = 0;                       // records per head (0 = off)
  int rec_kmax = 0;                    // record capacity: max(rec_k, l_base_int, l_h)
  __nv_bfloat16* shadowK = nullptr;    // [NL][B*H][L+T][128]
  float* mrows = nullptr;              // [NL*B*H][row_len], measure index mu = (l*B + b)*H + h
  uint32_t* rec_idx = nullptr;         // [NL*B*H][rec_kmax] records (ascending position, PAD tail)
  float* rec_sc = nullptr;             // [NL*B*H][rec_kmax]
  uint32_t* rec_cnt = nullptr;         // [NL*B*H]
  uint32_t* dynbm = nullptr;           // [n_units][words] dynamic-set bitmaps
  double* rec_out = nullptr;           // [NL*B*H] per-head recall
  hc_topk_job* d_mjobs = nullptr;      // static K1 jobs over mrows (n grows with n_add);
                                       // [0, nm): steps >= 1, [nm, 2 nm): step 0
  hc_recall_head* d_rheads = nullptr;  // static recall heads
  int32_t* d_piv_mu = nullptr;         // pivot slot -> mu
  uint64_t* rec_keys = nullptr;        // [2][NL*B*H][rec_kmax] composite keys (sort in/out)
  int* rec_off = nullptr;              // [NL*B*H + 1] segment offsets
  void* sort_tmp = nullptr;
  size_t sort_tmp_bytes = 0;
  char* mscratch = nullptr;            // packed queries + K5 scratch of one layer
  size_t mscratch_bytes = 0;
  int measured_t = -1;

  // device-resident boundary decisions (devdec.cuh)
  bool devdec = false;
  DevDec dd{};
  cudaStream_t sched = nullptr;         // schedule passes (tiny, never behind a gather)
  cudaStream_t lnd = nullptr;           // landing + satellites' K4, beside the main K4
  cudaStream_t hcp = nullptr;           // low priority: fetched sets to the mapped host ring
  cudaEvent_t ev_copy = nullptr;
  bool copy_valid = false;
  cudaEvent_t ev_land = nullptr, ev_sched = nullptr, ev_sel = nullptr, ev_dec = nullptr;
  cudaEvent_t ev_app = nullptr, ev_sats = nullptr;
  bool sched_valid = false;
  bool sel_valid = false;  // a fire selection the monitor stream is not yet ordered after
  // a gather pass takes only transfers due within this many steps (0: all of
  // them, the default -- keeping the host link busy as early as possible beat
  // every horizon of 1-8 steps at cfg4; HC_DEVDEC_HORIZON overrides)
  int dd_horizon = 0;
  cudaEvent_t ev_log[kLogRing] = {};    // side stream: boundary decided and selected
  int64_t n_bound = 0, n_read = 0;      // boundaries issued / read by the host
  int dd_pending_until = 0;             // latest completion step of the read decisions
  bool dd_quiet = false;                // this step: nothing can land
  std::vector<int32_t> dd_sat_units;
  std::vector<int32_t> dd_sat_of_unit;  // unit -> DevSat index or -1
  std::vector<void*> dd_dev;            // device allocations of the devdec state
  std::vector<void*> dd_host;           // mapped pinned allocations
  BoundaryHdr* hdr_h = nullptr;
  FireLog* log_h = nullptr;
  uint32_t* fetched_h = nullptr;
  int64_t* fetched_tail_h = nullptr;
  int32_t* error_h = nullptr;

  int lh(int u) const { return u % (NL * H); }
  int mu_of(int u) const { const int b = u / (NL * H), l = (u / H) % NL, h = u % H;
                           return (l * B + b) * H + h; }
  int head(int u) const { return u % H; }
};

}  // namespace hc

struct hc_engine {
  hc::EngineImpl e;
};

namespace hc {
namespace {

void chain_report(EngineImpl& e);

int engine_destroy(EngineImpl& e) {
  cudaDeviceSynchronize();
  host_prof_report();
  chain_report(e);
  for (auto& tr : e.ctr)
    for (auto ev : tr)
      if (ev) cudaEventDestroy(ev);
  for (auto& pr : e.stage_busy) cudaEventDestroy(std::get<2>(pr));
  if (e.stage) cudaFreeHost(e.stage);
  if (e.ovl_host) cudaFreeHost(e.ovl_host);
  for (auto& ev : e.events) cudaEventDestroy(ev.first);
  if (e.step_end) cudaEventDestroy(e.step_end);
  for (cudaEvent_t x : {e.ev_k4s, e.ev_piv, e.ev_rest, e.ev_pc, e.step_out})
    if (x) cudaEventDestroy(x);
  if (e.kst2) cudaStreamDestroy(e.kst2);
  if (e.rows_done) cudaEventDestroy(e.rows_done);
  for (auto x : e.rows_ev)
    if (x) cudaEventDestroy(x);
  for (auto& kv : e.blocks) cudaFree(kv.second.ptr);
  for (size_t u = 0; u < e.dyn_sel.size(); ++u) {
    if (e.dyn_sel[u]) cudaFree(e.dyn_sel[u]);
    if (e.dyn_cnt[u]) cudaFree(e.dyn_cnt[u]);
    if (e.pre_pos[u]) cudaFree(e.pre_pos[u]);
    if (e.pre_meta[u]) cudaFree(e.pre_meta[u]);
  }
  void* ptrs[] = {e.shadowK, e.mrows, e.rec_idx, e.rec_sc, e.rec_cnt, e.dynbm, e.rec_out,
                  e.d_mjobs, e.d_rheads, e.d_piv_mu, e.mscratch, e.rec_keys, e.rec_off,
                  e.sort_tmp,
                  e.d_units, e.K, e.V, e.d_tiles, e.d_skip, e.d_sat_tiles, e.d_sat_flags,
                  e.partial, e.d_piv_units, e.logits, e.mref,
                  e.stats,
                  e.rowbuf, e.top_idx, e.top_cnt, e.kbase, e.ovl_ring,
                  e.thr, e.ghist, e.d_piv_slots,
                  e.pf};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (e.pool) {
    if (e.pool_host) cudaFreeHost(e.pool);
    else cudaFree(e.pool);
  }
  for (void* p : e.dd_dev) cudaFree(p);
  for (void* p : e.dd_host) cudaFreeHost(p);
  for (cudaEvent_t x : {e.ev_land, e.ev_sched, e.ev_sel, e.ev_dec, e.ev_app, e.ev_sats})
    if (x) cudaEventDestroy(x);
  if (e.lnd) cudaStreamDestroy(e.lnd);
  if (e.hcp) cudaStreamDestroy(e.hcp);
  if (e.ev_copy) cudaEventDestroy(e.ev_copy);
  for (cudaEvent_t x : e.ev_log)
    if (x) cudaEventDestroy(x);
  if (e.sched) cudaStreamDestroy(e.sched);
  for (int i = 0; i < 2; ++i) {
    if (e.hbuf[i]) cudaFree(e.hbuf[i]);
    for (cudaEvent_t x : {e.h_in[i], e.h_used[i], e.h_out[i]})
      if (x) cudaEventDestroy(x);
  }
  if (e.hcopy) cudaStreamDestroy(e.hcopy);
  if (e.hdown) cudaStreamDestroy(e.hdown);
  if (e.mpool) cudaMemPoolDestroy(e.mpool);  // every block above is freed by now
  if (e.retr) cudaStreamDestroy(e.retr);
  if (e.side) cudaStreamDestroy(e.side);
  if (e.mon) cudaStreamDestroy(e.mon);
  if (e.pf_ev0) cudaEventDestroy(e.pf_ev0);
  if (e.pf_ev1) cudaEventDestroy(e.pf_ev1);
  for (auto x : e.tev) cudaEventDestroy(x);
  for (auto x : e.tpool) cudaEventDestroy(x);
  for (auto& pr : e.gather_ev) cudaEventDestroy(pr.first), cudaEventDestroy(pr.second);
  for (auto& pr : e.land_ev) cudaEventDestroy(pr.first), cudaEventDestroy(pr.second);
  return HC_OK;
}

int host_io_init(EngineImpl& e);

// Device decisions: satellites in pivot-slot order, rings, mapped host log.
int devdec_create(EngineImpl& e, const hc_engine_desc& c) {
  HC_REQUIRE(c.monitor && e.n_piv > 0, HC_EINVAL, "device decisions need monitored pivots");
  HC_REQUIRE(e.n_absent == 0, HC_EINVAL, "device decisions need an unsharded engine");
  HC_REQUIRE(c.window >= 1 && c.window <= 64, HC_EINVAL, "window must be 1..64");
  HC_REQUIRE(c.transfer_bandwidth >= 1 && c.update_delay_steps >= 0 && c.bytes_per_kv_entry >= 1,
             HC_EINVAL, "bad device-decision parameters");
  DevDec& d = e.dd;
  d.n_piv = e.n_piv;
  d.B = e.B;
  d.L = e.L;
  d.S = e.S;
  d.R = e.R;
  d.lbase = e.lbase;
  d.window = c.window;
  d.sliding = c.eval_every_step ? 1 : 0;
  d.delay = c.update_delay_steps;
  d.tau = c.tau_drift;
  d.bw = c.transfer_bandwidth;
  d.bpe = c.bytes_per_kv_entry;
  d.rowbuf = e.rowbuf;
  d.row_len = e.row_len;
  d.ghist = e.ghist;
  const int LH = e.NL * e.H;
  std::vector<int32_t> seq_piv(e.B + 1, 0), psb{0}, punit(e.n_piv);
  std::vector<DevSat> sats;
  e.dd_sat_of_unit.assign(e.n_units, -1);
  auto dev = [&](size_t bytes) -> void* {
    void* p = nullptr;
    if (dalloc(&p, bytes, &e.dev_bytes) != HC_OK) return nullptr;
    e.dd_dev.push_back(p);
    return p;
  };
  for (int s = 0; s < e.n_piv; ++s) {
    const int pu = e.piv_units[s];
    punit[s] = pu;
    const int b = pu / LH, i = e.lh(pu), l = i / e.H, ph = i % e.H;
    seq_piv[b + 1]++;
    for (int h = 0; h < e.H; ++h) {
      const int j = l * e.H + h;
      if (e.role[j] != HC_ROLE_SATELLITE || e.cpivot[j] != ph) continue;
      const int u = (b * e.NL + l) * e.H + h;
      DevSat x{};
      x.unit = u;
      x.pivot_slot = s;
      x.k = e.length[j];
      x.cap = e.cap[u];
      x.active = 0;
      x.staging_owner = -1;
      x.cur_slot = -1;
      x.seq = b;
      x.row0[0] = e.buf_row0[u];
      x.row0[1] = e.buf_row1[u];
      x.pos = static_cast<uint32_t*>(dev(2 * size_t(std::max(1, x.cap)) * 4));
      HC_REQUIRE(x.pos, HC_ENOMEM, "device decisions: position lists");
      const __nv_bfloat16* sk = e.pool + size_t(e.sat_slot[u]) * 2 * e.L * kHeadDim;
      x.srcK = reinterpret_cast<const uint4*>(sk);
      x.srcV = reinterpret_cast<const uint4*>(sk + size_t(e.L) * kHeadDim);
      e.dd_sat_of_unit[u] = int32_t(sats.size());
      sats.push_back(x);
      e.dd_sat_units.push_back(u);
    }
    HC_REQUIRE(int(sats.size()) - psb.back() <= 8, HC_EINVAL,
               "device decisions: a pivot with more than 8 satellites (use host decisions)");
    psb.push_back(int32_t(sats.size()));
  }
  for (int b = 0; b < e.B; ++b) seq_piv[b + 1] += seq_piv[b];
  d.n_sat = int32_t(sats.size());
  // transfer slots per satellite: as many as ~2 GB of fetched-set storage holds
  // (8..512); a satellite with more transfers pending at once faults loudly
  {
    int64_t per_slot = 0;
    for (const DevSat& x : sats) per_slot += int64_t(std::max(1, x.k)) * 4;
    d.nq = int32_t(std::max<int64_t>(8, std::min<int64_t>(512, (int64_t(2) << 30) /
                                                                   std::max<int64_t>(1, per_slot))));
    if (const char* q = getenv("HC_DEVDEC_NQ")) d.nq = std::max(2, atoi(q));  // tests: tiny rings
    d.no_host_copy = getenv("HC_DEVDEC_NO_HOST_COPY") ? 1 : 0;  // timing diagnostics only
    d.gather_ctas = 40;
    d.gather_chunk = 256;
    if (const char* g = getenv("HC_GATHER_CTAS")) d.gather_ctas = std::max(1, atoi(g));
    if (const char* g = getenv("HC_GATHER_CHUNK")) d.gather_chunk = std::max(32, atoi(g));
    for (DevSat& x : sats) {
      x.sel = static_cast<uint32_t*>(dev(size_t(d.nq) * std::max(1, x.k) * 4));
      HC_REQUIRE(x.sel, HC_ENOMEM, "device decisions: transfer rings");
    }
  }
  const size_t ns = std::max<size_t>(1, sats.size());
  auto up = [&](const void* src, size_t bytes) -> void* {
    void* p = dev(bytes);
    if (p && bytes) cudaMemcpy(p, src, bytes, cudaMemcpyHostToDevice);
    return p;
  };
  d.seq_piv = static_cast<int32_t*>(up(seq_piv.data(), seq_piv.size() * 4));
  d.piv_sat_begin = static_cast<int32_t*>(up(psb.data(), psb.size() * 4));
  d.piv_unit = static_cast<int32_t*>(up(punit.data(), punit.size() * 4));
  d.sats = static_cast<DevSat*>(up(sats.data(), sats.size() * sizeof(DevSat)));
  d.xfers = static_cast<DevXfer*>(dev(ns * d.nq * sizeof(DevXfer)));
  d.cum = static_cast<int64_t*>(dev(size_t(e.B) * 8));
  d.order = static_cast<int32_t*>(dev(size_t(e.B) * 4));
  d.svals = static_cast<double*>(dev(size_t(e.n_piv) * 64 * 8));
  d.scnt = static_cast<int32_t*>(dev(size_t(e.n_piv) * 4));
  d.jobs = static_cast<FireJob*>(dev(ns * sizeof(FireJob)));
  d.bump = static_cast<int32_t*>(dev(ns * 4));
  if (e.chain_trace) {
    d.dbg = static_cast<unsigned long long*>(dev(64));
    HC_CUDA_TRY(cudaMemset(d.dbg, 0, 64));
  }
  d.n_jobs = static_cast<uint32_t*>(dev(4));
  d.restamp_slots = static_cast<int32_t*>(dev(size_t(e.n_piv) * 4));
  d.n_restamp = static_cast<uint32_t*>(dev(4));
  d.glist = static_cast<GatherItem*>(dev(ns * sizeof(GatherItem)));
  d.glist2 = static_cast<GatherItem*>(dev(ns * sizeof(GatherItem)));
  d.n_glist = static_cast<uint32_t*>(dev(4));
  d.urgent_epoch = static_cast<uint32_t*>(dev(4));
  d.head_dev = static_cast<int64_t*>(dev(8));
  d.hdr_dev = static_cast<BoundaryHdr*>(dev(sizeof(BoundaryHdr) * kLogRing));
  d.log_dev = static_cast<FireLog*>(dev(sizeof(FireLog) * kLogRing * std::max(1, e.n_piv)));
  HC_CUDA_TRY(cudaGetLastError());
  HC_REQUIRE(d.seq_piv && d.piv_sat_begin && d.piv_unit && d.sats && d.xfers && d.cum &&
                 d.order && d.svals && d.scnt && d.jobs && d.bump && d.n_jobs && d.restamp_slots &&
                 d.n_restamp && d.glist && d.glist2 && d.n_glist && d.urgent_epoch &&
                 d.head_dev && d.hdr_dev && d.log_dev,
             HC_ENOMEM, "device decisions: state");
  // mapped host memory: the decision log and the fetched sets the host mirrors
  int64_t ksum = 0;
  for (const DevSat& x : sats) ksum += x.k;
  // the host reads boundaries within a few of their decision (decoder.py blocks
  // beyond 4 unread): 6 boundaries of every satellite firing fit
  d.fetched_cap = std::max<int64_t>(6 * ksum + 64, int64_t(1) << 20);
  auto mapped = [&](void** h, size_t bytes) -> int {
    HC_CUDA_TRY(cudaHostAlloc(h, bytes, cudaHostAllocMapped));
    std::memset(*h, 0, bytes);
    e.dd_host.push_back(*h);
    e.host_bytes += int64_t(bytes);
    return HC_OK;
  };
  void* p = nullptr;
  HC_TRY(mapped(&p, sizeof(BoundaryHdr) * kLogRing));
  e.hdr_h = static_cast<BoundaryHdr*>(p);
  HC_TRY(mapped(&p, sizeof(FireLog) * kLogRing * std::max(1, e.n_piv)));
  e.log_h = static_cast<FireLog*>(p);
  HC_TRY(mapped(&p, size_t(d.fetched_cap) * 4));
  e.fetched_h = static_cast<uint32_t*>(p);
  HC_TRY(mapped(&p, 64));
  int64_t* ctr = static_cast<int64_t*>(p);  // [0] head (device), [1] tail (host)
  e.fetched_tail_h = ctr + 1;
  HC_TRY(mapped(&p, 64));
  e.error_h = static_cast<int32_t*>(p);
  void* dp = nullptr;
  HC_CUDA_TRY(cudaHostGetDevicePointer(&dp, e.hdr_h, 0));
  d.hdr = static_cast<BoundaryHdr*>(dp);
  HC_CUDA_TRY(cudaHostGetDevicePointer(&dp, e.log_h, 0));
  d.log = static_cast<FireLog*>(dp);
  HC_CUDA_TRY(cudaHostGetDevicePointer(&dp, e.fetched_h, 0));
  d.fetched = static_cast<uint32_t*>(dp);
  HC_CUDA_TRY(cudaHostGetDevicePointer(&dp, ctr, 0));
  d.fetched_tail = static_cast<int64_t*>(dp) + 1;
  HC_CUDA_TRY(cudaHostGetDevicePointer(&dp, e.error_h, 0));
  d.error = static_cast<int32_t*>(dp);
  int lo_prio = 0, hi_prio = 0;
  HC_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
  HC_CUDA_TRY(cudaStreamCreateWithPriority(&e.sched, cudaStreamNonBlocking, hi_prio));
  HC_CUDA_TRY(cudaStreamCreateWithPriority(&e.lnd, cudaStreamNonBlocking, hi_prio));
  HC_CUDA_TRY(cudaStreamCreateWithPriority(&e.hcp, cudaStreamNonBlocking, lo_prio));
  HC_CUDA_TRY(cudaEventCreateWithFlags(&e.ev_copy, cudaEventDisableTiming));
  for (cudaEvent_t* x : {&e.ev_land, &e.ev_sched, &e.ev_sel, &e.ev_dec, &e.ev_app, &e.ev_sats})
    HC_CUDA_TRY(cudaEventCreateWithFlags(x, cudaEventDisableTiming));
  for (auto& x : e.ev_log) HC_CUDA_TRY(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
  if (const char* h = getenv("HC_DEVDEC_HORIZON")) e.dd_horizon = atoi(h);
  if (e.dd_horizon <= 0) e.dd_horizon = 1 << 29;
  e.devdec = true;
  return HC_OK;
}

int engine_create(EngineImpl& e, const hc_engine_desc& c, const int32_t* roles,
                  const int32_t* lengths, const int32_t* cpiv, const uint8_t* owned) {
  HC_REQUIRE(c.head_dim == kHeadDim, HC_EINVAL, "head_dim must be 128");
  HC_REQUIRE(c.group >= 1 && c.group <= 8, HC_EINVAL, "group must be 1..8");
  HC_REQUIRE(c.batch >= 1 && c.num_layers >= 1 && c.kv_heads >= 1, HC_EINVAL, "bad geometry");
  HC_REQUIRE(c.prefill_len >= 1 && c.max_decode >= 1, HC_EINVAL, "bad lengths");
  HC_REQUIRE(c.recency_window >= 0, HC_EINVAL, "recency_window must be >= 0");
  HC_REQUIRE(c.sink_count >= 0, HC_EINVAL, "sink_count must be >= 0");
  HC_REQUIRE(c.l_base_int >= 1, HC_EINFEASIBLE, "l_base_int must be >= 1");
  e.cfg = c;
  e.B = c.batch, e.NL = c.num_layers, e.H = c.kv_heads, e.G = c.group, e.Hq = c.kv_heads * c.group;
  e.L = c.prefill_len, e.T = c.max_decode, e.S = c.sink_count, e.R = c.recency_window;
  e.CH = c.chunk > 0 ? c.chunk : 1024;
  HC_REQUIRE(e.CH % 64 == 0, HC_EINVAL, "chunk must be a multiple of 64");
  e.lbase = c.l_base_int;
  e.pool_host = c.host_pool != 0;
  e.W = c.obs_window > 0 ? c.obs_window : 1;
  HC_REQUIRE(e.W * e.G <= 128 && e.W <= e.L, HC_EINVAL,
             "observation window %d x group %d exceeds the 128 tcgen05 rows", e.W, e.G);
  const int LH = e.NL * e.H;
  e.role.assign(roles, roles + LH);
  e.length.assign(lengths, lengths + LH);
  e.cpivot.assign(cpiv, cpiv + LH);
  for (int i = 0; i < LH; ++i) {
    HC_REQUIRE(e.role[i] >= 0 && e.role[i] <= 3, HC_EINVAL, "bad role at %d", i);
    const bool comp = e.role[i] == HC_ROLE_ANCHOR || e.role[i] == HC_ROLE_SATELLITE;
    if (comp) HC_REQUIRE(e.length[i] >= 0 && e.length[i] <= e.L, HC_EINVAL, "bad length at %d", i);
    // recency tails longer than 32 rows are held as a contiguous block
    // (kv_layout.cuh tail_lo): only without a dynamic set (sink_window)
    if (comp && e.R > 32)
      HC_REQUIRE(e.length[i] == 0, HC_EINVAL,
                 "recency_window %d > 32 needs compressed heads without a dynamic set", e.R);
    if (e.role[i] == HC_ROLE_SATELLITE) {
      const int p = e.cpivot[i];
      HC_REQUIRE(p >= 0 && p < e.H && e.role[(i / e.H) * e.H + p] == HC_ROLE_PIVOT, HC_EINVAL,
                 "satellite %d has no pivot in its layer", i);
    }
  }
  e.n_units = e.B * LH;
  // sharded engines: units another rank owns are absent; a
  // satellite always lives with its pivot (it is refilled from the pivot's
  // row, engine.py:326-329)
  e.owned.assign(e.n_units, 1);
  if (owned) {
    for (int u = 0; u < e.n_units; ++u) e.owned[u] = owned[u] ? 1 : 0;
    for (int u = 0; u < e.n_units; ++u) {
      const int i = u % LH;
      if (e.role[i] != HC_ROLE_SATELLITE) continue;
      const int pu = (u / e.H) * e.H + e.cpivot[i];
      HC_REQUIRE(e.owned[u] == e.owned[pu], HC_EINVAL,
                 "unit %d: a satellite must be owned together with its pivot", u);
    }
  }
  e.units.resize(e.n_units);
  e.cap.assign(e.n_units, 0);
  e.buf_row0.assign(e.n_units, -1);
  e.buf_row1.assign(e.n_units, -1);
  e.active.assign(e.n_units, 0);
  e.piv_slot.assign(e.n_units, -1);
  e.sat_slot.assign(e.n_units, -1);
  e.dyn_sel.assign(e.n_units, nullptr);
  e.dyn_cnt.assign(e.n_units, nullptr);
  e.dyn_owner.assign(e.n_units, -1);
  e.pre_pos.assign(e.n_units, nullptr);
  e.pre_meta.assign(e.n_units, nullptr);
  e.fifo.assign(e.n_units, {});
  e.row_len = (int64_t(e.L) + e.T + 15) / 16 * 16;  // aligned logit / score-row stride
  e.words = int((e.row_len + 31) / 32);

  // ---- arena rows and the static tile table ----
  struct TileH { TileDesc d; };
  std::vector<TileDesc> tiles;
  int64_t row = 0;
  int slot = 0;
  for (int u = 0; u < e.n_units; ++u) {
    const int i = e.lh(u);
    const int b = u / LH, l = i / e.H, h = i % e.H;
    UnitDesc& d = e.units[u];
    d = UnitDesc{};
    d.q_row = (b * e.NL + l) * e.Hq + h * e.G;
    d.pivot_slot = -1;
    d.slot0 = slot;
    const bool full = e.role[i] == HC_ROLE_VOLATILE || e.role[i] == HC_ROLE_PIVOT;
    if (!e.owned[u]) {
      d.kind = kUnitAbsent;
      ++e.n_absent;
    } else if (full) {
      d.kind = kUnitFull;
      d.row0 = row;
      d.app_row = row + e.L;
      d.n_prefix = e.L;
      row += e.row_len;
      const int nch = int((e.row_len + e.CH - 1) / e.CH);
      for (int ch = 0; ch < nch; ++ch) {
        const int64_t first = int64_t(ch) * e.CH - e.L + 1;
        tiles.push_back(TileDesc{uint32_t(u), uint32_t(ch), uint32_t(slot + ch),
                                 uint32_t(first > 0 ? first : 0)});
      }
      slot += nch;
      if (e.role[i] == HC_ROLE_PIVOT && c.monitor) {
        d.pivot_slot = e.n_piv++;
        e.piv_slot[u] = d.pivot_slot;
        e.piv_units.push_back(u);
      }
    } else {
      d.kind = kUnitComp;
      const int capu = std::min(e.length[i], e.L) + std::min(e.S, e.L) + e.R;
      e.cap[u] = capu;
      e.buf_row0[u] = row;
      row += capu;
      if (e.role[i] == HC_ROLE_SATELLITE) {
        e.buf_row1[u] = row;
        row += capu;
        e.sat_slot[u] = e.n_sat++;
      }
      d.row0 = e.buf_row0[u];
      d.app_row = row;
      row += e.T;
      d.n_prefix = 0;
      d.n_pchunks = std::max(1, (capu + e.CH - 1) / e.CH);
      for (int ch = 0; ch < d.n_pchunks; ++ch)
        tiles.push_back(TileDesc{uint32_t(u), uint32_t(ch), uint32_t(slot + ch), 0u});
      const int nap = (e.T + e.CH - 1) / e.CH;
      for (int ch = 0; ch < nap; ++ch)
        tiles.push_back(TileDesc{uint32_t(u), 0x80000000u | uint32_t(ch),
                                 uint32_t(slot + d.n_pchunks + ch),
                                 uint32_t(int64_t(ch) * e.CH + 1)});
      slot += d.n_pchunks + nap;
    }
  }
  e.rows = row + 64;  // slack: the last sub-tile of a segment may read past it
  e.n_slots = slot;
  std::stable_sort(tiles.begin(), tiles.end(),
                   [](const TileDesc& a, const TileDesc& b) { return a.t_act < b.t_act; });
  e.t_act.resize(tiles.size());
  for (size_t i = 0; i < tiles.size(); ++i) e.t_act[i] = tiles[i].t_act;
  e.tiles_host = tiles;
  e.unit_tiles.assign(e.n_units, {});
  for (size_t i = 0; i < tiles.size(); ++i) e.unit_tiles[tiles[i].unit].push_back(int(i));
  HC_TRY(dalloc((void**)&e.d_skip, size_t(e.n_units), &e.dev_bytes));
  {
    std::vector<TileDesc> st;
    std::vector<uint8_t> fl(e.n_units, 0);
    for (int u = 0; u < e.n_units; ++u)
      if (e.units[u].kind == kUnitComp && e.role[e.lh(u)] == HC_ROLE_SATELLITE) fl[u] = 1;
    for (const TileDesc& d : tiles)
      if (fl[d.unit]) st.push_back(d);  // keeps the t_act order
    for (const TileDesc& d : st) e.sat_t_act.push_back(d.t_act);
    HC_TRY(dalloc((void**)&e.d_sat_tiles, std::max<size_t>(1, st.size()) * sizeof(TileDesc),
                  &e.dev_bytes));
    if (!st.empty())
      HC_CUDA_TRY(cudaMemcpy(e.d_sat_tiles, st.data(), st.size() * sizeof(TileDesc),
                             cudaMemcpyHostToDevice));
    HC_TRY(dalloc((void**)&e.d_sat_flags, size_t(e.n_units), &e.dev_bytes));
    HC_CUDA_TRY(cudaMemcpy(e.d_sat_flags, fl.data(), fl.size(), cudaMemcpyHostToDevice));
  }
  {  // pivot-first tile lists (each keeps the t_act order)
    std::vector<TileDesc> pt, rt;
    for (const TileDesc& d : tiles) (e.units[d.unit].pivot_slot >= 0 ? pt : rt).push_back(d);
    for (const TileDesc& d : pt) e.piv_t_act.push_back(d.t_act);
    for (const TileDesc& d : rt) e.rest_t_act.push_back(d.t_act);
    for (auto* pr : {&pt, &rt}) {
      TileDesc*& dst = pr == &pt ? e.d_piv_tiles : e.d_rest_tiles;
      HC_TRY(dalloc((void**)&dst, std::max<size_t>(1, pr->size()) * sizeof(TileDesc),
                    &e.dev_bytes));
      if (!pr->empty())
        HC_CUDA_TRY(cudaMemcpy(dst, pr->data(), pr->size() * sizeof(TileDesc),
                               cudaMemcpyHostToDevice));
    }
  }

  HC_TRY(dalloc((void**)&e.K, size_t(e.rows) * kHeadDim * 2, &e.dev_bytes));
  HC_TRY(dalloc((void**)&e.V, size_t(e.rows) * kHeadDim * 2, &e.dev_bytes));
  HC_TRY(make_kv_tensor_map(&e.tmK, e.K, e.rows));
  HC_TRY(make_kv_tensor_map(&e.tmV, e.V, e.rows));
  HC_TRY(dalloc((void**)&e.d_tiles, tiles.size() * sizeof(TileDesc), &e.dev_bytes));
  HC_CUDA_TRY(cudaMemcpy(e.d_tiles, tiles.data(), tiles.size() * sizeof(TileDesc),
                         cudaMemcpyHostToDevice));
  HC_TRY(dalloc((void**)&e.partial, size_t(e.n_slots) * e.G * kPartStride * 4, &e.dev_bytes));
  HC_TRY(dalloc((void**)&e.d_units, size_t(e.n_units) * sizeof(UnitDesc), &e.dev_bytes));
  HC_CUDA_TRY(cudaMemcpy(e.d_units, e.units.data(), size_t(e.n_units) * sizeof(UnitDesc),
                         cudaMemcpyHostToDevice));

  // ---- pivot monitoring state ----
  const int np = std::max(1, e.n_piv);
  HC_TRY(dalloc((void**)&e.d_piv_units, size_t(np) * 4, &e.dev_bytes));
  if (e.n_piv)
    HC_CUDA_TRY(cudaMemcpy(e.d_piv_units, e.piv_units.data(), size_t(e.n_piv) * 4,
                           cudaMemcpyHostToDevice));
  // pivot score material and statistics, double-buffered by step parity: the
  // score rows of step t run beside step t+1's attention
  e.mat_f16 = c.score_material == 1 ? 1 : 0;
  HC_REQUIRE(c.score_material == 0 || c.score_material == 1, HC_EINVAL,
             "score_material must be 0 (fp32) or 1 (fp16)");
  e.mat_bytes = e.mat_f16 ? 2 : 4;
  HC_TRY(dalloc((void**)&e.logits, 2 * size_t(np) * e.G * e.row_len * e.mat_bytes, &e.dev_bytes));
  HC_TRY(dalloc((void**)&e.mref, 2 * size_t(np) * e.G * (e.row_len / 16) * 4, &e.dev_bytes));
  HC_TRY(dalloc((void**)&e.stats, 2 * size_t(np) * e.G * 2 * 4, &e.dev_bytes));
  HC_TRY(dalloc((void**)&e.rowbuf, size_t(np) * e.row_len * 4, &e.dev_bytes));
  HC_TRY(dalloc((void**)&e.top_idx, size_t(np) * e.lbase * 4, &e.dev_bytes));
  HC_TRY(dalloc((void**)&e.top_cnt, size_t(np) * 4, &e.dev_bytes));
  HC_TRY(dalloc((void**)&e.kbase, size_t(np) * e.words * 4, &e.dev_bytes));
  HC_TRY(dalloc((void**)&e.ovl_ring, size_t(np) * kRing * 4, &e.dev_bytes));
  HC_TRY(dalloc((void**)&e.thr, size_t(np) * 8, &e.dev_bytes));
  HC_TRY(dalloc((void**)&e.ghist, 2 * size_t(np) * 8192 * 4, &e.dev_bytes));
  {
    std::vector<int32_t> iota(np);
    for (int i = 0; i < np; ++i) iota[i] = i;
    HC_TRY(dalloc((void**)&e.d_piv_slots, size_t(np) * 4, &e.dev_bytes));
    HC_CUDA_TRY(cudaMemcpy(e.d_piv_slots, iota.data(), size_t(np) * 4, cudaMemcpyHostToDevice));
  }

  // ---- compressed-unit bookkeeping buffers ----
  for (int u = 0; u < e.n_units; ++u) {
    if (e.units[u].kind != kUnitComp) continue;
    const int k = std::max(1, e.length[e.lh(u)]);
    HC_TRY(dalloc((void**)&e.dyn_sel[u], size_t(k) * 4, &e.dev_bytes));
    HC_TRY(dalloc((void**)&e.dyn_cnt[u], 4, &e.dev_bytes));
    HC_TRY(dalloc((void**)&e.pre_pos[u], size_t(std::max(1, e.cap[u])) * 4, &e.dev_bytes));
    HC_TRY(dalloc((void**)&e.pre_meta[u], 16, &e.dev_bytes));
  }

  // ---- host pool for satellites' prefill K/V ----
  if (e.n_sat) {
    const size_t bytes = size_t(e.n_sat) * 2 * e.L * kHeadDim * 2;
    if (e.pool_host) {
      cudaError_t r = cudaHostAlloc((void**)&e.pool, bytes, cudaHostAllocMapped | cudaHostAllocPortable);
      HC_REQUIRE(r == cudaSuccess, HC_ENOMEM, "cudaHostAlloc(%zu) failed: %s", bytes,
                 cudaGetErrorString(r));
      e.host_bytes += int64_t(bytes);
    } else {
      HC_TRY(dalloc((void**)&e.pool, bytes, &e.dev_bytes));
    }
  }
  {  // a private stream-ordered pool for the engine's fire / land descriptors and
     // transfer blocks: its settings must not leak into the process's default
     // pool (torch's cudaMallocAsync backend, other libraries); destroyed with
     // the engine
    int dev = 0;
    HC_CUDA_TRY(cudaGetDevice(&dev));
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    HC_CUDA_TRY(cudaMemPoolCreate(&e.mpool, &props));
    cudaMemPool_t pool = e.mpool;
    // keep freed blocks cached in the pool (no release back to the driver)
    uint64_t keep = ~uint64_t(0);
    HC_CUDA_TRY(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    // a block freed on one stream (a superseded transfer, on the caller's) must
    // not be handed to an allocation on another (the fire selection's side
    // stream) with an inserted wait on the free: that would hold the selection
    // -- and the gathers behind it -- until the caller's stream got there
    int no = 0;
    HC_CUDA_TRY(cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &no));
    // grow the pool once, here, for the transfer blocks of ~16 fires per
    // satellite in flight: growing it inside a decode step (a fire batch's
    // cudaMallocAsync) costs milliseconds on the boundary's critical path
    if (c.monitor && e.n_sat) {
      size_t per = 0;
      for (int u = 0; u < e.n_units; ++u)
        if (e.sat_slot[u] >= 0) per += (2 * size_t(std::max(1, e.cap[u])) + 8) * 4;
      const size_t want = std::min<size_t>(per * 16, size_t(1) << 30);
      void* tmp = nullptr;
      if (cudaMallocFromPoolAsync(&tmp, want, pool, 0) == cudaSuccess) {
        HC_CUDA_TRY(cudaFreeAsync(tmp, 0));
        HC_CUDA_TRY(cudaStreamSynchronize(0));
      } else {
        cudaGetLastError();  // no room to pre-grow: the pool grows on demand
      }
    }
  }
  HC_CUDA_TRY(cudaHostAlloc((void**)&e.ovl_host, size_t(kRing) * std::max(1, e.n_piv) * 4,
                            cudaHostAllocDefault));
  e.stage_cap = size_t(8) << 20;
  HC_CUDA_TRY(cudaHostAlloc((void**)&e.stage, e.stage_cap, cudaHostAllocDefault));
  int lo_prio = 0, hi_prio = 0;
  HC_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
  HC_CUDA_TRY(cudaStreamCreateWithPriority(&e.retr, cudaStreamNonBlocking, hi_prio));
  HC_CUDA_TRY(cudaStreamCreateWithPriority(&e.side, cudaStreamNonBlocking, hi_prio));
  HC_CUDA_TRY(cudaStreamCreateWithPriority(&e.mon, cudaStreamNonBlocking, hi_prio));
  if (c.device_decisions) HC_TRY(devdec_create(e, c));
  {
    const char* pfe = getenv("HC_PIVOT_FIRST");
    // measured (profiles/r02_chain_trace.md): +0.6% at cfg2 and +1.5% at cfg4, but
    // -2.2% at cfg3 and -0.6% at cfg5 -- off unless HC_PIVOT_FIRST=1
    e.pivot_first = e.devdec && e.n_piv > 0 && pfe && pfe[0] == '1';
  }
  if (e.pivot_first) {
    HC_CUDA_TRY(cudaStreamCreateWithFlags(&e.kst2, cudaStreamNonBlocking));
    for (cudaEvent_t* x : {&e.ev_k4s, &e.ev_piv, &e.ev_rest, &e.ev_pc, &e.step_out})
      HC_CUDA_TRY(cudaEventCreateWithFlags(x, cudaEventDisableTiming));
  }
  return host_io_init(e);  // decode_step_host staging, outside any timed step
}

AttnParams decode_params(EngineImpl& e, int t, const void* q, void* o) {
  AttnParams p{};
  p.units = e.d_units;
  p.tiles = e.d_tiles;
  p.q = q;
  p.out = o;
  p.partial = e.partial;
  const size_t np = size_t(std::max(1, e.n_piv));
  p.logits = static_cast<char*>(e.logits) + size_t(t & 1) * np * e.G * e.row_len * e.mat_bytes;
  p.mat_f16 = e.mat_f16;
  p.mref = e.mref + size_t(t & 1) * np * e.G * (e.row_len / 16);
  p.stats = e.stats + size_t(t & 1) * np * e.G * 2;
  p.rows = e.n_piv ? e.rowbuf : nullptr;
  p.logit_stride = e.row_len;
  p.row_stride = e.row_len;
  p.group = e.G;
  p.L = e.L;
  p.t = t;
  p.chunk = e.CH;
  p.recency = e.R;
  p.n_units = e.n_units;
  p.scale_log2 = float(1.4426950408889634 / 11.313708498984761);  // log2(e)/sqrt(128)
  return p;
}

int active_tiles(const EngineImpl& e, int t) {
  return int(std::upper_bound(e.t_act.begin(), e.t_act.end(), uint32_t(t)) - e.t_act.begin());
}

int new_event(EngineImpl& e, cudaEvent_t* out, bool timed = false) {
  cudaEvent_t ev;
  HC_CUDA_TRY(cudaEventCreateWithFlags(&ev, timed ? cudaEventDefault : cudaEventDisableTiming));
  e.events.emplace_back(ev, e.last_t);
  *out = ev;
  return HC_OK;
}

// Chain trace mark k of the open boundary trace on stream st (diagnostics).
int chain_mark(EngineImpl& e, int k, cudaStream_t st) {
  if (!e.chain_trace || e.ctr_open < 0) return HC_OK;
  cudaEvent_t& ev = e.ctr[e.ctr_open][k];
  if (!ev) HC_CUDA_TRY(cudaEventCreate(&ev));
  HC_CUDA_TRY(cudaEventRecord(ev, st));
  return HC_OK;
}

void chain_report(EngineImpl& e) {
  if (!e.chain_trace || e.ctr.empty()) return;
  static const char* names[EngineImpl::kChainMarks] = {
      "combine(t) done", "monitor(t)", "decide+restamp", "fire_select", "schedule",
      "gathers done", "main K4(t+1)", "landing(t+1)", "sats K4(t+1)", "step t+1 joins",
      "decide only"};
  double sum[EngineImpl::kChainMarks] = {};
  int n = 0;
  for (auto& tr : e.ctr) {
    bool ok = true;
    for (auto ev : tr) ok = ok && ev && cudaEventSynchronize(ev) == cudaSuccess;
    if (!ok) continue;
    for (int k = 1; k < EngineImpl::kChainMarks; ++k) {
      float ms = 0;
      cudaEventElapsedTime(&ms, tr[0], tr[k]);
      sum[k] += ms;
    }
    ++n;
  }
  cudaGetLastError();
  if (e.dd.dbg) {
    unsigned long long h[3] = {};
    cudaMemcpy(h, e.dd.dbg, sizeof(h), cudaMemcpyDeviceToHost);
    if (h[2])
      fprintf(stderr, "hc_chain_trace decide kernel: window tests %.1f us, accounting %.1f us (%llu)\n",
              h[0] / 1e3 / h[2], h[1] / 1e3 / h[2], h[2]);
  }
  fprintf(stderr, "hc_chain_trace %d boundaries (us after step t's combine):\n", n);
  for (int k = 1; k < EngineImpl::kChainMarks; ++k)
    fprintf(stderr, "hc_chain_trace %-18s %8.1f\n", names[k], n ? sum[k] / n * 1e3 : 0.0);
}

// A timed event for a gather / landing timing pair, from the engine's pool
// (returned by hc_engine_retrieval_stats once read): no event creation inside a step.
int timed_event(EngineImpl& e, cudaEvent_t* out) {
  if (e.tpool.empty()) {
    HC_CUDA_TRY(cudaEventCreate(out));
  } else {
    *out = e.tpool.back();
    e.tpool.pop_back();
  }
  return HC_OK;
}

// Retire ordering events older than kRing steps that have completed and that
// no pending transfer or timing record still refers to (a long decode would
// otherwise accumulate one per fire / gather / landing).
int gc_events(EngineImpl& e, int t) {
  if (t % kRing || e.events.empty()) return HC_OK;
  std::vector<cudaEvent_t> live;
  for (const auto& q : e.fifo)
    for (int id : q) {
      live.push_back(e.xfers[id].selected);
      live.push_back(e.xfers[id].done);
    }
  if (e.last_selected) live.push_back(e.last_selected);
  for (const auto& pr : e.gather_ev) live.push_back(pr.first), live.push_back(pr.second);
  for (const auto& pr : e.land_ev) live.push_back(pr.first), live.push_back(pr.second);
  std::sort(live.begin(), live.end());
  while (!e.events.empty() && e.events.front().second < t - kRing) {
    const cudaEvent_t ev = e.events.front().first;
    if (std::binary_search(live.begin(), live.end(), ev)) break;
    const cudaError_t q = cudaEventQuery(ev);
    if (q == cudaErrorNotReady) break;
    HC_CUDA_TRY(q);
    HC_CUDA_TRY(cudaEventDestroy(ev));
    e.events.pop_front();
  }
  return HC_OK;
}

int upload(EngineImpl& e, const void* src, size_t bytes, cudaStream_t st, void** dev);
int apply_landings(EngineImpl& e, const std::vector<int>& ids, cudaStream_t st);

// Apply landings requested earlier but not yet consumed by a decode step.
int flush_deferred(EngineImpl& e) {
  if (e.deferred.empty() || e.in_step) return HC_OK;  // an open step lands them itself
  std::vector<int> ids;
  ids.swap(e.deferred);
  return apply_landings(e, ids, e.deferred_st);
}

__global__ void set_flags_kernel(uint8_t* flags, const int32_t* __restrict__ idx, int n,
                                 uint8_t v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) flags[idx[i]] = v;
}

// Device decisions: landing point of step t on the step's stream, then a
// schedule pass and the gathers it frees (retrieval stream).
int devdec_land(EngineImpl& e, int t, cudaStream_t st) {
  if (e.sched_valid) HC_CUDA_TRY(cudaStreamWaitEvent(st, e.ev_sched, 0));
  HC_TRY(launch_land(e.dd, t, e.d_units, reinterpret_cast<uint4*>(e.K),
                     reinterpret_cast<uint4*>(e.V), st));
  HC_CUDA_TRY(cudaEventRecord(e.ev_land, st));
  HC_CUDA_TRY(cudaStreamWaitEvent(e.sched, e.ev_land, 0));
  return HC_OK;
}

// A schedule pass on the schedule stream and the gathers it lists.
int devdec_schedule_and_gather(EngineImpl& e, int t_max) {
  HC_TRY(launch_schedule(e.dd, t_max - e.dd_horizon, e.sched));
  HC_CUDA_TRY(cudaEventRecord(e.ev_sched, e.sched));
  if (e.ctr_in_decide) HC_TRY(chain_mark(e, 4, e.sched));
  e.sched_valid = true;
  HC_CUDA_TRY(cudaStreamWaitEvent(e.retr, e.ev_sched, 0));
  cudaEvent_t g0 = nullptr, g1 = nullptr;
  if (e.timing) {
    HC_TRY(timed_event(e, &g0));
    HC_TRY(timed_event(e, &g1));
  }
  HC_TRY(launch_dev_gathers(e.dd, reinterpret_cast<uint4*>(e.K), reinterpret_cast<uint4*>(e.V),
                            e.retr, t_max, g0, g1));
  if (e.timing) e.gather_ev.emplace_back(g0, g1);
  return HC_OK;
}

// The decision of boundary t on the monitor stream (after its monitor), the
// K_base restamp, the fetch selection (side stream), a schedule pass and the
// gathers.
int devdec_decide(EngineImpl& e, int t) {
  const bool boundary = e.dd.sliding || t % e.dd.window == 0;
  if (!boundary) return HC_OK;
  const int first = e.dd.sliding ? t : std::max(1, t - e.dd.window + 1);
  const int nvals = t - first + 1;
  const int64_t bidx = e.n_bound++;
  HC_REQUIRE(e.n_bound - e.n_read <= kLogRing, HC_ESTATE,
             "device decisions: %d boundaries unread (poll the decisions)", kLogRing);
  // the previous boundary's host copy still reads the job list the decision rewrites
  if (e.copy_valid) HC_CUDA_TRY(cudaStreamWaitEvent(e.mon, e.ev_copy, 0));
  HC_TRY(launch_decide(e.dd, t, first, nvals, int(bidx), e.ovl_ring, kRing, e.mon));
  // the fire selection needs the decision's job list, not the K_base restamp
  // (which only the next monitor reads): it starts beside the restamp
  HC_CUDA_TRY(cudaEventRecord(e.ev_dec, e.mon));
  HC_TRY(chain_mark(e, 10, e.mon));
  HC_TRY(launch_restamp_threshold(e.rowbuf, e.row_len, e.dd.restamp_slots, e.n_piv,
                                  uint32_t(e.L + t), e.thr, e.kbase, e.words, e.mon,
                                  e.dd.n_restamp));
  HC_TRY(chain_mark(e, 2, e.mon));
  HC_CUDA_TRY(cudaStreamWaitEvent(e.side, e.ev_dec, 0));
  HC_TRY(launch_fire_select(e.dd.jobs, std::max(1, e.dd.n_sat), e.side, e.dd.n_jobs));
  HC_CUDA_TRY(cudaEventRecord(e.ev_sel, e.side));
  HC_TRY(chain_mark(e, 3, e.side));
  e.sel_valid = true;
  // the host mirror's copy of the fetched sets, on a low-priority stream
  HC_CUDA_TRY(cudaStreamWaitEvent(e.hcp, e.ev_sel, 0));
  HC_TRY(launch_copy_fetched(e.dd, int(bidx), e.hcp));
  HC_CUDA_TRY(cudaEventRecord(e.ev_copy, e.hcp));
  HC_CUDA_TRY(cudaEventRecord(e.ev_log[bidx % kLogRing], e.hcp));
  e.copy_valid = true;
  HC_CUDA_TRY(cudaStreamWaitEvent(e.sched, e.ev_sel, 0));
  e.ctr_in_decide = true;
  const int rc = devdec_schedule_and_gather(e, t + e.dd_horizon);
  e.ctr_in_decide = false;
  HC_TRY(rc);
  HC_TRY(chain_mark(e, 5, e.retr));
  return HC_OK;
}

// Score rows and the K1+K2 monitor (top-l_base threshold and |top & K_base| per
// pivot, engine.py:305-311; counts land in the overlap ring row of the step)
// feed only the drift decision, so they run on their own stream beside the
// next step's attention.  Readers (overlaps, fire, measure, pivot_row) wait for
// step_end; the attention two steps later waits for this step's rows before it
// overwrites the score material of its parity.  Pivot-first: the chain starts
// when the pivots' tiles are done (ev_piv) with the pivots' own combine.
int monitor_chain(EngineImpl& e, int t, const AttnParams& p, cudaEvent_t* ev, cudaStream_t st) {
  if (e.pivot_first) {
    HC_CUDA_TRY(cudaStreamWaitEvent(e.mon, e.ev_piv, 0));
  } else {
    if (!e.rows_done)
      HC_CUDA_TRY(cudaEventCreateWithFlags(&e.rows_done, cudaEventDisableTiming));
    HC_CUDA_TRY(cudaEventRecord(e.rows_done, st));
    HC_CUDA_TRY(cudaStreamWaitEvent(e.mon, e.rows_done, 0));
  }
  // the previous boundary's fetch selection still reads the rows and histograms
  if (e.sel_valid) {  // (once per selection: the monitor stream stays ordered after it)
    HC_CUDA_TRY(cudaStreamWaitEvent(e.mon, e.ev_sel, 0));
    e.sel_valid = false;
  }
  if (e.pivot_first) {  // the pivots' O and softmax statistics
    AttnParams pc = p;
    pc.combine_sel = 1;
    pc.cunits = e.d_piv_units;
    pc.n_cunits = e.n_piv;
    HC_TRY(launch_combine(pc, e.mon));
    HC_CUDA_TRY(cudaEventRecord(e.ev_pc, e.mon));
  }
  HC_TRY(launch_score_rows(p, e.d_piv_units, e.n_piv, e.mon));
  cudaEvent_t& re = e.rows_ev[t & 1];
  if (!re) HC_CUDA_TRY(cudaEventCreateWithFlags(&re, cudaEventDisableTiming));
  HC_CUDA_TRY(cudaEventRecord(re, e.mon));
  if (ev) HC_CUDA_TRY(cudaEventRecord(ev[4], e.mon));
  HC_TRY(launch_monitor(e.rowbuf, e.row_len, e.d_piv_slots, e.n_piv, uint32_t(e.L + t),
                        uint32_t(e.lbase), e.kbase, e.words, e.thr,
                        e.ovl_ring + size_t(t % kRing) * e.n_piv, e.mon,
                        e.ghist + size_t(t & 1) * e.n_piv * 8192));
  if (e.chain_trace && e.devdec && (e.dd.sliding || t % e.dd.window == 0)) {
    e.ctr.push_back({});
    e.ctr_open = int(e.ctr.size()) - 1;
    e.ctr_step = t + 1;
    HC_TRY(chain_mark(e, 0, st));     // the chain's start on the caller's stream
    HC_TRY(chain_mark(e, 1, e.mon));  // score rows + monitor done
  }
  if (e.devdec) HC_TRY(devdec_decide(e, t));
  if (ev) HC_CUDA_TRY(cudaEventRecord(ev[5], e.mon));
  if (!e.step_end)
    HC_CUDA_TRY(cudaEventCreateWithFlags(&e.step_end, cudaEventDisableTiming));
  HC_CUDA_TRY(cudaEventRecord(e.step_end, e.mon));
  return HC_OK;
}

// Decode step t, in two halves so a host decision can overlap the attention:
//
//   decode_begin  append the token; K4 over every unit except those that may
//                 change this step (landing units, or -- hold_satellites --
//                 every satellite, when the fire decision of step t-1 is still
//                 open and may land transfers at t)
//   (host)        overlaps / fire_batch / land_batch for the open decision:
//                 they run on the side stream against step t-1's state
//   decode_end    landing point (wait for the gathers, swap descriptors), K4
//                 over the held units, combine, score rows, monitor
//
// The retrieval gathers of a landing overlap the step's main K4 instead of
// stalling it; decode_step = begin(hold 0) + end.
int engine_decode_begin(EngineImpl& e, int t, const void* q, const void* kn, const void* vn,
                        void* o, bool hold, cudaStream_t st) {
  HC_REQUIRE(t >= 1 && t <= e.T, HC_EINVAL, "step %d outside 1..%d", t, e.T);
  HC_REQUIRE(e.in_step == 0, HC_ESTATE, "decode_begin(%d) while step %d is open", t, e.in_step);
  HostProfScope prof_all(0);
  e.dd_quiet = false;
  if (e.devdec) {  // landings are decided on the device: satellites run after them ...
    HC_REQUIRE(e.deferred.empty(), HC_ESTATE, "host landings with device decisions");
    // ... unless nothing can land: every decision is read and every transfer it
    // made has landed already -- then no landing pass, no split K4
    e.dd_quiet = e.n_read == e.n_bound && t > e.dd_pending_until;
    hold = !e.dd_quiet;
  }
  if (!e.deferred.empty() && e.deferred_st != st) {  // landings requested on another stream
    std::vector<int> ids;
    ids.swap(e.deferred);
    HC_TRY(apply_landings(e, ids, e.deferred_st));
    cudaEvent_t ev;
    HC_TRY(new_event(e, &ev));
    HC_CUDA_TRY(cudaEventRecord(ev, e.deferred_st));
    HC_CUDA_TRY(cudaStreamWaitEvent(st, ev, 0));
  }
  std::vector<int> land;
  if (!hold) land.swap(e.deferred);
  e.d_land = nullptr;
  e.n_lu = e.n_lt = 0;
  if (!land.empty()) {
    std::vector<int32_t> lu;
    for (int id : land) {
      const int u = e.xfers[id].unit;
      if (std::find(lu.begin(), lu.end(), u) == lu.end()) lu.push_back(u);
    }
    e.n_lu = int(lu.size());
    const size_t off = (lu.size() * 4 + 15) & ~size_t(15);
    std::vector<char> blob(off);
    std::memcpy(blob.data(), lu.data(), lu.size() * 4);
    for (int u : lu)
      for (int i : e.unit_tiles[u])
        if (e.tiles_host[i].t_act <= uint32_t(t)) {
          blob.resize(blob.size() + sizeof(TileDesc));
          std::memcpy(blob.data() + blob.size() - sizeof(TileDesc), &e.tiles_host[i],
                      sizeof(TileDesc));
          ++e.n_lt;
        }
    HC_TRY(upload(e, blob.data(), blob.size(), st, (void**)&e.d_land));
    set_flags_kernel<<<(e.n_lu + 127) / 128, 128, 0, st>>>(e.d_skip, e.d_land, e.n_lu, 1);
    HC_CHECK_LAUNCH();
  }
  cudaEvent_t* ev = nullptr;
  if (e.timing) {
    const size_t need = (e.tev_used + 1) * EngineImpl::kPhaseEvents;
    while (e.tev.size() < need) {
      cudaEvent_t x;
      HC_CUDA_TRY(cudaEventCreate(&x));
      e.tev.push_back(x);
    }
    ev = e.tev.data() + e.tev_used * EngineImpl::kPhaseEvents;
    ++e.tev_used;
    if (!e.timing_light) HC_CUDA_TRY(cudaEventRecord(ev[0], st));
  }
  std::optional<HostProfScope> prof_sec;
  prof_sec.emplace(1);
  append_kernel<<<(e.n_units + 7) / 8, 256, 0, st>>>(
      e.d_units, e.n_units, e.L, t, reinterpret_cast<const uint4*>(kn),
      reinterpret_cast<const uint4*>(vn), reinterpret_cast<uint4*>(e.K),
      reinterpret_cast<uint4*>(e.V), reinterpret_cast<uint4*>(e.shadowK), e.NL, e.H,
      int64_t(e.L) + e.T);
  HC_CHECK_LAUNCH();
  if (ev) HC_CUDA_TRY(cudaEventRecord(ev[1], st));  // light timing: this ...
  if (e.devdec && !e.dd_quiet)  // the token is appended (the landing stream waits for it)
    HC_CUDA_TRY(cudaEventRecord(e.ev_app, st));
  AttnParams p = decode_params(e, t, q, o);
  if (e.pivot_first) HC_CUDA_TRY(cudaEventRecord(e.ev_k4s, st));  // (before the material wait below)
  // K4 overwrites the score material of parity t&1: step t-2's rows must be done
  if (e.rows_ev[t & 1]) HC_CUDA_TRY(cudaStreamWaitEvent(st, e.rows_ev[t & 1], 0));
  p.skip = hold ? e.d_sat_flags : (land.empty() ? nullptr : e.d_skip);
  prof_sec.emplace(2);
  if (e.pivot_first) {
    // the pivots' tiles on the caller's stream, every other unit's on kst2
    // beside them (the same priority: the pivots' CTAs are dispatched first)
    AttnParams pp = p;
    pp.skip = nullptr;
    pp.tiles = e.d_piv_tiles;
    const int np = int(std::upper_bound(e.piv_t_act.begin(), e.piv_t_act.end(), uint32_t(t)) -
                       e.piv_t_act.begin());
    HC_TRY(launch_attn_tiles(e.tmK, e.tmV, pp, np, st));
    HC_CUDA_TRY(cudaEventRecord(e.ev_piv, st));
    HC_CUDA_TRY(cudaStreamWaitEvent(e.kst2, e.ev_k4s, 0));
    AttnParams pr = p;
    pr.tiles = e.d_rest_tiles;
    const int nr = int(std::upper_bound(e.rest_t_act.begin(), e.rest_t_act.end(),
                                        uint32_t(t)) - e.rest_t_act.begin());
    HC_TRY(launch_attn_tiles(e.tmK, e.tmV, pr, nr, e.kst2));
    HC_CUDA_TRY(cudaEventRecord(e.ev_rest, e.kst2));
  } else {
    HC_TRY(launch_attn_tiles(e.tmK, e.tmV, p, active_tiles(e, t), st));
  }
  prof_sec.reset();
  if (e.devdec && !e.dd_quiet) {
    // landing point (device-decided transfers due at t), then the satellites'
    // K4, on their own stream beside the main K4: the landing's wait for a late
    // gather no longer serialises the step
    prof_sec.emplace(3);
    HC_CUDA_TRY(cudaStreamWaitEvent(e.lnd, e.ev_app, 0));
    HC_TRY(devdec_land(e, t, e.lnd));
    const bool traced = e.ctr_open >= 0 && e.ctr_step == t;
    if (traced) HC_TRY(chain_mark(e, 7, e.lnd));
    prof_sec.emplace(4);
    HC_TRY(devdec_schedule_and_gather(e, t + e.dd_horizon));
    prof_sec.emplace(5);
    AttnParams ps = p;
    ps.skip = nullptr;
    ps.tiles = e.d_sat_tiles;
    const int n = int(std::upper_bound(e.sat_t_act.begin(), e.sat_t_act.end(), uint32_t(t)) -
                      e.sat_t_act.begin());
    HC_TRY(launch_attn_tiles(e.tmK, e.tmV, ps, n, e.lnd));
    if (traced) {
      HC_TRY(chain_mark(e, 8, e.lnd));
      HC_TRY(chain_mark(e, 6, st));  // the main K4 was queued on st before the landing
    }
    HC_CUDA_TRY(cudaEventRecord(e.ev_sats, e.lnd));
    if (e.timing) {  // landing stall = how far the satellites' path ends after the main K4
      cudaEvent_t w0 = nullptr, w1 = nullptr;
      HC_TRY(timed_event(e, &w0));
      HC_TRY(timed_event(e, &w1));
      HC_CUDA_TRY(cudaEventRecord(w0, st));
      HC_CUDA_TRY(cudaEventRecord(w1, e.lnd));
      e.land_ev.emplace_back(w0, w1);
    }
  }
  if (e.pivot_first) {  // the boundary chain of step t, beside the other units' tiles
    prof_sec.emplace(8);
    HC_TRY(monitor_chain(e, t, p, (ev && !e.timing_light) ? ev : nullptr, st));
    prof_sec.reset();
  }
  e.in_step = t;
  e.cur_hold = hold;
  e.cur_st = st;
  e.cur_p = p;
  e.cur_ev = ev;
  e.cur_land.swap(land);
  return HC_OK;
}

int engine_decode_end(EngineImpl& e, int t, cudaStream_t st) {
  HC_REQUIRE(e.in_step == t, HC_ESTATE, "decode_end(%d) without decode_begin(%d)", t, t);
  HC_REQUIRE(st == e.cur_st, HC_EINVAL, "decode_end on another stream than decode_begin");
  HostProfScope prof_all(6);
  std::optional<HostProfScope> prof_sec;
  e.in_step = 0;  // landings below are applied for real
  AttnParams pl = e.cur_p;
  pl.skip = nullptr;
  if (e.devdec) {
    if (e.pivot_first) HC_CUDA_TRY(cudaStreamWaitEvent(st, e.ev_rest, 0));  // the other units' tiles
    if (!e.dd_quiet) HC_CUDA_TRY(cudaStreamWaitEvent(st, e.ev_sats, 0));  // satellites attended
    if (e.ctr_open >= 0 && e.ctr_step == t) {
      HC_TRY(chain_mark(e, 9, st));
      e.ctr_open = -1;
    }
  } else if (e.cur_hold) {
    std::vector<int> land;
    land.swap(e.deferred);
    if (!land.empty()) HC_TRY(apply_landings(e, land, st));
    const int n = int(std::upper_bound(e.sat_t_act.begin(), e.sat_t_act.end(), uint32_t(t)) -
                      e.sat_t_act.begin());
    pl.tiles = e.d_sat_tiles;
    HC_TRY(launch_attn_tiles(e.tmK, e.tmV, pl, n, st));
  } else if (!e.cur_land.empty()) {
    HC_TRY(apply_landings(e, e.cur_land, st));
    pl.tiles = reinterpret_cast<const TileDesc*>(reinterpret_cast<const char*>(e.d_land) +
                                                 ((size_t(e.n_lu) * 4 + 15) & ~size_t(15)));
    HC_TRY(launch_attn_tiles(e.tmK, e.tmV, pl, e.n_lt, st));
    set_flags_kernel<<<(e.n_lu + 127) / 128, 128, 0, st>>>(e.d_skip, e.d_land, e.n_lu, 0);
    HC_CHECK_LAUNCH();
    HC_CUDA_TRY(cudaFreeAsync(e.d_land, st));
    e.d_land = nullptr;
  }
  e.cur_land.clear();
  cudaEvent_t* ev = e.cur_ev;
  prof_sec.emplace(7);
  if (ev) HC_CUDA_TRY(cudaEventRecord(ev[2], st));  // ... and this one only
  if (ev && e.timing_light) ev = nullptr;
  if (e.pivot_first) {
    AttnParams pc = e.cur_p;
    pc.combine_sel = 2;  // every unit but the pivots (combined on the monitor stream)
    HC_TRY(launch_combine(pc, st));  // O: the step's output
    if (ev) HC_CUDA_TRY(cudaEventRecord(ev[3], st));
    HC_CUDA_TRY(cudaStreamWaitEvent(st, e.ev_pc, 0));  // the pivots' O
    if (ev) HC_CUDA_TRY(cudaEventRecord(ev[6], st));
    HC_CUDA_TRY(cudaEventRecord(e.step_out, st));
    e.last_t = t;
    prof_sec.emplace(10);
    return gc_events(e, t);
  }
  HC_TRY(launch_combine(e.cur_p, st));  // O: the step's output
  if (ev) HC_CUDA_TRY(cudaEventRecord(ev[3], st));
  e.last_t = t;
  if (!e.step_end)
    HC_CUDA_TRY(cudaEventCreateWithFlags(&e.step_end, cudaEventDisableTiming));
  if (e.n_piv) {
    // Score rows and the K1+K2 monitor (top-l_base threshold and |top & K_base|
    // per pivot, engine.py:305-311; counts land in the overlap ring row of the
    // step) feed only the drift decision, so they run on their own stream
    // beside the next step's attention.  Readers (overlaps, fire, measure,
    // pivot_row) wait for step_end; the attention two steps later waits for
    // this step's rows before it overwrites the score material of its parity.
    prof_sec.emplace(8);
    if (!e.rows_done)
      HC_CUDA_TRY(cudaEventCreateWithFlags(&e.rows_done, cudaEventDisableTiming));
    HC_CUDA_TRY(cudaEventRecord(e.rows_done, st));
    HC_CUDA_TRY(cudaStreamWaitEvent(e.mon, e.rows_done, 0));
    // the previous boundary's fetch selection still reads the rows and histograms
    if (e.sel_valid) {  // (once per selection: the monitor stream stays ordered after it)
      HC_CUDA_TRY(cudaStreamWaitEvent(e.mon, e.ev_sel, 0));
      e.sel_valid = false;
    }
    HC_TRY(launch_score_rows(e.cur_p, e.d_piv_units, e.n_piv, e.mon));
    cudaEvent_t& re = e.rows_ev[t & 1];
    if (!re) HC_CUDA_TRY(cudaEventCreateWithFlags(&re, cudaEventDisableTiming));
    HC_CUDA_TRY(cudaEventRecord(re, e.mon));
    if (ev) HC_CUDA_TRY(cudaEventRecord(ev[4], e.mon));
    HC_TRY(launch_monitor(e.rowbuf, e.row_len, e.d_piv_slots, e.n_piv, uint32_t(e.L + t),
                          uint32_t(e.lbase), e.kbase, e.words, e.thr,
                          e.ovl_ring + size_t(t % kRing) * e.n_piv, e.mon,
                          e.ghist + size_t(t & 1) * e.n_piv * 8192));
    prof_sec.emplace(9);
    if (e.chain_trace && e.devdec && (e.dd.sliding || t % e.dd.window == 0)) {
      e.ctr.push_back({});
      e.ctr_open = int(e.ctr.size()) - 1;
      e.ctr_step = t + 1;
      HC_TRY(chain_mark(e, 0, st));     // combine(t) done (the caller's stream)
      HC_TRY(chain_mark(e, 1, e.mon));  // score rows + monitor done
    }
    if (e.devdec) HC_TRY(devdec_decide(e, t));
    prof_sec.reset();
  } else if (ev) {
    HC_CUDA_TRY(cudaEventRecord(ev[4], st));
  }
  cudaStream_t ms = e.n_piv ? e.mon : st;
  if (ev) {
    HC_CUDA_TRY(cudaEventRecord(ev[5], ms));
    HC_CUDA_TRY(cudaEventRecord(ev[6], st));
  }
  HC_CUDA_TRY(cudaEventRecord(e.step_end, ms));
  prof_sec.emplace(10);
  return gc_events(e, t);
}

int engine_decode_step(EngineImpl& e, int t, const void* q, const void* kn, const void* vn,
                       void* o, cudaStream_t st) {
  HC_TRY(engine_decode_begin(e, t, q, kn, vn, o, false, st));
  return engine_decode_end(e, t, st);
}

// decode_step from pinned HOST buffers: the step's inputs cross H2D and its
// output D2H on engine-owned copy streams, double-buffered so step t's
// download and step t+1's upload overlap the decode (the e2e path of a
// serving runtime: one call per step, no framework on the host).
// Staging of decode_step_host, set up with the engine (not inside a timed step).
//
// Small steps (inputs + output <= 512 KB, e.g. one layer at batch 1) are
// launch-bound: their inputs are read from the caller's pinned buffers by one
// zero-copy kernel on the step's stream and the combine writes O straight into
// the caller's pinned output -- two fewer copies, events and streams per step.
// Larger steps copy on the engine's copy streams, overlapped with the decode.
constexpr size_t kSmallHostIo = size_t(512) << 10;

__global__ void stage_in_kernel(const uint4* q, const uint4* kn, const uint4* vn, uint4* dq,
                                uint4* dkn, uint4* dvn, int nq, int nk) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const uint4* src;
  uint4* dst;
  if (i < nq) src = q + i, dst = dq + i;
  else if (i < nq + nk) src = kn + (i - nq), dst = dkn + (i - nq);
  else if (i < nq + 2 * nk) src = vn + (i - nq - nk), dst = dvn + (i - nq - nk);
  else return;
  uint4 v;  // .cv: system-memory lines are fetched again, never served stale from L2
  asm volatile("ld.global.cv.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(src));
  *dst = v;
}

// Device address of a pinned (page-locked, mapped) host buffer; cached per pointer.
int mapped_ptr(EngineImpl& e, const void* h, void** d) {
  for (const auto& pr : e.hmap)
    if (pr.first == h) {
      *d = pr.second;
      return HC_OK;
    }
  const cudaError_t rc = cudaHostGetDevicePointer(d, const_cast<void*>(h), 0);
  if (rc != cudaSuccess) {
    cudaGetLastError();
    HC_REQUIRE(false, HC_EINVAL, "decode_step_host: %p is not pinned host memory", h);
  }
  if (e.hmap.size() >= 64) e.hmap.erase(e.hmap.begin());
  e.hmap.emplace_back(h, *d);
  return HC_OK;
}

int host_io_init(EngineImpl& e) {
  const size_t qb = size_t(e.B) * e.NL * e.Hq * kHeadDim * 2;
  const size_t kb = size_t(e.B) * e.NL * e.H * kHeadDim * 2;
  e.small_io = 2 * qb + 2 * kb <= kSmallHostIo && !getenv("HC_HOST_IO_COPY");
  HC_CUDA_TRY(cudaStreamCreateWithFlags(&e.hcopy, cudaStreamNonBlocking));
  HC_CUDA_TRY(cudaStreamCreateWithFlags(&e.hdown, cudaStreamNonBlocking));
  for (int i = 0; i < 2; ++i) {
    HC_TRY(dalloc(&e.hbuf[i], 2 * qb + 2 * kb, &e.dev_bytes));
    for (cudaEvent_t* x : {&e.h_in[i], &e.h_used[i], &e.h_out[i]}) {
      HC_CUDA_TRY(cudaEventCreateWithFlags(x, cudaEventDisableTiming));
      HC_CUDA_TRY(cudaEventRecord(*x, 0));
    }
  }
  return HC_OK;
}

int engine_decode_step_host(EngineImpl& e, int t, const void* q_h, const void* kn_h,
                            const void* vn_h, void* o_h, cudaStream_t st) {
  const size_t qb = size_t(e.B) * e.NL * e.Hq * kHeadDim * 2;
  const size_t kb = size_t(e.B) * e.NL * e.H * kHeadDim * 2;
  if (!e.hcopy) HC_TRY(host_io_init(e));
  HostProfScope prof_all(11);
  const int s = t & 1;
  char* d = static_cast<char*>(e.hbuf[s]);
  void *dq = d, *dkn = d + qb, *dvn = d + qb + kb, *dout = d + qb + 2 * kb;
  if (e.small_io) {
    void *mq, *mk, *mv, *mo;
    HC_TRY(mapped_ptr(e, q_h, &mq));
    HC_TRY(mapped_ptr(e, kn_h, &mk));
    HC_TRY(mapped_ptr(e, vn_h, &mv));
    HC_TRY(mapped_ptr(e, o_h, &mo));
    const int nq = int(qb / 16), nk = int(kb / 16);
    stage_in_kernel<<<(nq + 2 * nk + 255) / 256, 256, 0, st>>>(
        static_cast<const uint4*>(mq), static_cast<const uint4*>(mk),
        static_cast<const uint4*>(mv), static_cast<uint4*>(dq), static_cast<uint4*>(dkn),
        static_cast<uint4*>(dvn), nq, nk);
    HC_CHECK_LAUNCH();
    HC_TRY(engine_decode_step(e, t, dq, dkn, dvn, mo, st));  // the combine writes O to the host
    HC_CUDA_TRY(cudaEventRecord(e.h_out[s], st));
    e.h_last = s;
    return HC_OK;
  }
  HC_CUDA_TRY(cudaStreamWaitEvent(e.hcopy, e.h_used[s], 0));  // the decode that read this slot
  HC_CUDA_TRY(cudaMemcpyAsync(dq, q_h, qb, cudaMemcpyHostToDevice, e.hcopy));
  HC_CUDA_TRY(cudaMemcpyAsync(dkn, kn_h, kb, cudaMemcpyHostToDevice, e.hcopy));
  HC_CUDA_TRY(cudaMemcpyAsync(dvn, vn_h, kb, cudaMemcpyHostToDevice, e.hcopy));
  HC_CUDA_TRY(cudaEventRecord(e.h_in[s], e.hcopy));
  HC_CUDA_TRY(cudaStreamWaitEvent(st, e.h_in[s], 0));
  HC_CUDA_TRY(cudaStreamWaitEvent(st, e.h_out[s], 0));  // the previous download of this slot
  HC_TRY(engine_decode_step(e, t, dq, dkn, dvn, dout, st));
  HC_CUDA_TRY(cudaEventRecord(e.h_used[s], st));
  // the download runs on its own stream: the next step's upload must not
  // queue behind it (it waits for this decode to finish)
  HC_CUDA_TRY(cudaStreamWaitEvent(e.hdown, e.h_used[s], 0));
  HC_CUDA_TRY(cudaMemcpyAsync(o_h, dout, qb, cudaMemcpyDeviceToHost, e.hdown));
  HC_CUDA_TRY(cudaEventRecord(e.h_out[s], e.hdown));
  e.h_last = s;
  return HC_OK;
}

// Stream-ordered upload of a small host array: copy into the pinned staging
// ring, allocate a device buffer on `st` from the engine's pool and copy asynchronously.  The
// caller frees *dev with cudaFreeAsync on the same stream.
int upload(EngineImpl& e, const void* src, size_t bytes, cudaStream_t st, void** dev) {
  const size_t need = (bytes + 255) & ~size_t(255);
  HC_REQUIRE(need <= e.stage_cap, HC_EINVAL, "descriptor upload of %zu B too large", bytes);
  if (e.stage_head + need > e.stage_cap) e.stage_head = 0;  // wrap
  const size_t lo = e.stage_head, hi = lo + need;
  // a region may be rewritten only after the copy that read it has executed
  for (auto it = e.stage_busy.begin(); it != e.stage_busy.end();) {
    const bool overlap = std::get<0>(*it) < hi && lo < std::get<1>(*it);
    if (overlap || e.stage_busy.size() > 256) {
      HC_CUDA_TRY(cudaEventSynchronize(std::get<2>(*it)));
      HC_CUDA_TRY(cudaEventDestroy(std::get<2>(*it)));
      it = e.stage_busy.erase(it);
    } else {
      ++it;
    }
  }
  std::memcpy(e.stage + lo, src, bytes);
  HC_CUDA_TRY(cudaMallocFromPoolAsync(dev, need, e.mpool, st));
  HC_CUDA_TRY(cudaMemcpyAsync(*dev, e.stage + lo, bytes, cudaMemcpyHostToDevice, st));
  cudaEvent_t ev;
  HC_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  HC_CUDA_TRY(cudaEventRecord(ev, st));
  e.stage_busy.emplace_back(lo, hi, ev);
  e.stage_head = hi;
  return HC_OK;
}

// Batched retrieval plumbing: one launch builds the prefix position lists of
// many transfers, one launch gathers all their rows from the host pool.
struct XferDev {
  const uint32_t* sel;
  const uint32_t* cnt;
  uint32_t* pos;
  int32_t* meta;
  const uint4* srcK;
  const uint4* srcV;
  int64_t dst_row;
  int32_t t_c;
  int32_t pad_;
};

__global__ void build_positions_batch_kernel(const XferDev* __restrict__ xs, int L, int S, int R) {
  const XferDev x = xs[blockIdx.x];
  build_positions_block(x.sel, int(*x.cnt), x.pos, x.meta, L, S, R, x.t_c);
}

__global__ void gather_rows_batch_kernel(const XferDev* __restrict__ xs, uint4* __restrict__ K,
                                         uint4* __restrict__ V) {
  const XferDev x = xs[blockIdx.y];
  gather_rows(x.pos, x.meta[0], x.srcK, x.srcV, K, V, x.dst_row,
              blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), gridDim.x * (blockDim.x >> 5));
}

// Retrieval gather from the pinned host pool (zero-copy over the host link).
// A small fixed grid loops over all transfers of the batch: 40 CTAs of 256
// threads (4 x 16-B loads in flight per thread, 640 KB in all) hold the link
// at 47-48 GB/s, and each gather CTA that shares an SM with the attention
// slows that SM's K4.  At cfg4, where gathers run most of every step, back to
// back on one box: 128 CTAs 993 / 802 steps/s, 40 CTAs 1211 / 1188 (cfg5
// unchanged within noise; 24 CTAs: the link drops to 42 GB/s; more loads in
// flight per thread or fewer threads per CTA: slower).
constexpr int kGatherCtas = 40;

__global__ void __launch_bounds__(256) gather_host_rows_kernel(const XferDev* __restrict__ xs,
                                                               int n_x, uint4* __restrict__ K,
                                                               uint4* __restrict__ V) {
  const int nw = gridDim.x * (blockDim.x >> 5);
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  for (int xi = 0; xi < n_x; ++xi) {
    const XferDev x = xs[xi];
    gather_rows(x.pos, x.meta[0], x.srcK, x.srcV, K, V, x.dst_row, gw, nw);
  }
}

struct LandDev {
  int32_t unit;
  int32_t pad_;
  int64_t row0;
  const int32_t* meta;
};

__global__ void set_prefix_batch_kernel(UnitDesc* units, const LandDev* __restrict__ ls, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const LandDev l = ls[i];
  units[l.unit].row0 = l.row0;
  units[l.unit].n_prefix = l.meta[0];
  units[l.unit].tail_mask = uint32_t(l.meta[1]);
  units[l.unit].pad_ = l.meta[2];
}

// K_base <- current top set for several pivots (one block per bitmap).
__global__ void restamp_batch_kernel(uint32_t* kbase, const uint32_t* top_idx,
                                     const uint32_t* top_cnt, const int32_t* slots, int words,
                                     int lbase) {
  const int s = slots[blockIdx.x];
  uint32_t* bm = kbase + size_t(s) * words;
  for (int w = threadIdx.x; w < words; w += blockDim.x) bm[w] = 0u;
  __syncthreads();
  const int c = min(int(top_cnt[s]), lbase);
  const uint32_t* idx = top_idx + size_t(s) * lbase;
  for (int i = threadIdx.x; i < c; i += blockDim.x) {
    const uint32_t p = idx[i];
    if (int(p >> 5) < words) atomicOr(bm + (p >> 5), 1u << (p & 31));
  }
}

// Issue the gathers of transfers `ids` (their units' staging buffers are free)
// on the retrieval stream, after `after` (an event on the caller's stream).
int issue_gathers(EngineImpl& e, const std::vector<int>& ids_in, cudaEvent_t after) {
  if (ids_in.empty()) return HC_OK;
  // one batch per completion step (ascending): a landing then waits only for
  // the gathers that are due, not for the whole burst of a drift event
  std::vector<int> ids(ids_in);
  std::stable_sort(ids.begin(), ids.end(), [&](int a, int b) {
    return e.xfers[a].completion < e.xfers[b].completion;
  });
  HC_CUDA_TRY(cudaStreamWaitEvent(e.retr, after, 0));
  size_t lo = 0;
  while (lo < ids.size()) {
    size_t hi = lo + 1;
    while (hi < ids.size() && e.xfers[ids[hi]].completion == e.xfers[ids[lo]].completion) ++hi;
    std::vector<XferDev> xd;
    int max_cap = 1;
    int64_t rows = 0;
    for (size_t i = lo; i < hi; ++i) {
      Transfer& x = e.xfers[ids[i]];
      const int u = x.unit;
      x.buf = 1 - e.active[u];
      const int ss = e.sat_slot[u];
      const __nv_bfloat16* sk = e.pool + size_t(ss) * 2 * e.L * kHeadDim;
      xd.push_back(XferDev{x.sel, x.cnt, x.pos, x.meta, reinterpret_cast<const uint4*>(sk),
                           reinterpret_cast<const uint4*>(sk + size_t(e.L) * kHeadDim),
                           x.buf ? e.buf_row1[u] : e.buf_row0[u], x.completion, 0});
      max_cap = std::max(max_cap, e.cap[u]);
      rows += x.k + std::min(e.S, e.L) + e.R;  // upper bound of the rows moved
    }
    XferDev* d = nullptr;
    HC_TRY(upload(e, xd.data(), xd.size() * sizeof(XferDev), e.retr, (void**)&d));
    build_positions_batch_kernel<<<int(xd.size()), 256, 0, e.retr>>>(d, e.L, e.S, e.R);
    HC_CHECK_LAUNCH();
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    if (e.timing) {
      HC_TRY(timed_event(e, &t0));
      HC_TRY(timed_event(e, &t1));
      HC_CUDA_TRY(cudaEventRecord(t0, e.retr));
    }
    (void)max_cap;
    gather_host_rows_kernel<<<kGatherCtas, 256, 0, e.retr>>>(
        d, int(xd.size()), reinterpret_cast<uint4*>(e.K), reinterpret_cast<uint4*>(e.V));
    HC_CHECK_LAUNCH();
    if (e.timing) {
      HC_CUDA_TRY(cudaEventRecord(t1, e.retr));
      e.gather_ev.emplace_back(t0, t1);
    }
    if (e.timing) e.gather_rows_issued += rows;  // same window as gather_ev
    HC_CUDA_TRY(cudaFreeAsync(d, e.retr));
    cudaEvent_t done;
    HC_TRY(new_event(e, &done));
    HC_CUDA_TRY(cudaEventRecord(done, e.retr));
    for (size_t i = lo; i < hi; ++i) {
      e.xfers[ids[i]].done = done;
      e.xfers[ids[i]].gathered = true;
    }
    lo = hi;
  }
  return HC_OK;
}

int engine_prefill_layer(EngineImpl& e, int layer, const __nv_bfloat16* k,
                         const __nv_bfloat16* v, const __nv_bfloat16* q, cudaStream_t st) {
  HC_REQUIRE(layer >= 0 && layer < e.NL, HC_EINVAL, "layer out of range");
  const int nu = e.B * e.H;  // units of this layer, i = b*H + h
  const int nch = (e.L + e.CH - 1) / e.CH;
  const int64_t Lp = (int64_t(e.L) + 3) / 4 * 4;  // 16-B aligned row stride
  // scratch layout
  size_t off = 0;
  auto carve = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~size_t(255); return o; };
  const size_t o_rows = carve(size_t(nu) * Lp * 4);
  const size_t o_jobs = carve(size_t(nu) * sizeof(hc_topk_job));
  const size_t o_obs = carve(obs_scratch_bytes(nu, e.L, e.W * e.G));
  if (off > e.pf_bytes) {
    if (e.pivot_first) {
      HC_CUDA_TRY(cudaStreamSynchronize(st));
      cudaFree(e.pf);
      e.pf = nullptr;
    }
    HC_TRY(dalloc((void**)&e.pf, off, nullptr));
    e.pf_bytes = off;
  }
  char* pf = e.pf;
  float* rows = reinterpret_cast<float*>(pf + o_rows);
  (void)nch;
  // K5: step-0 score rows of every head of the layer on the tcgen05 tensor
  // cores (observation window w; w = 1 is the reference's last-token row)
  if (!e.pf_ev0) {
    HC_CUDA_TRY(cudaEventCreate(&e.pf_ev0));
    HC_CUDA_TRY(cudaEventCreate(&e.pf_ev1));
  }
  HC_CUDA_TRY(cudaEventRecord(e.pf_ev0, st));
  HC_TRY(launch_obs_scores(k, q, e.B, e.H, e.G, e.W, e.L, rows, Lp, pf + o_obs, st));
  HC_CUDA_TRY(cudaEventRecord(e.pf_ev1, st));
  HC_CUDA_TRY(cudaEventSynchronize(e.pf_ev1));
  {
    float ms = 0;
    HC_CUDA_TRY(cudaEventElapsedTime(&ms, e.pf_ev0, e.pf_ev1));
    e.pf_score_ms += ms;
    e.pf_layers += 1;
  }
  if (e.rec_k) {  // measure mode: full-context K copy and the step-0 rows
    const int64_t srows = int64_t(e.L) + e.T;
    HC_CUDA_TRY(cudaMemcpy2DAsync(e.shadowK + size_t(layer) * nu * srows * kHeadDim,
                                  size_t(srows) * kHeadDim * 2, k, size_t(e.L) * kHeadDim * 2,
                                  size_t(e.L) * kHeadDim * 2, nu, cudaMemcpyDeviceToDevice, st));
    HC_CUDA_TRY(cudaMemcpy2DAsync(e.mrows + size_t(layer) * nu * e.row_len, size_t(e.row_len) * 4,
                                  rows, size_t(Lp) * 4, size_t(e.L) * 4, nu,
                                  cudaMemcpyDeviceToDevice, st));
  }
  if (e.prefill_dump)  // test hook: step-0 rows [NL][B*H][L]
    HC_CUDA_TRY(cudaMemcpy2DAsync(e.prefill_dump + size_t(layer) * nu * e.L, size_t(e.L) * 4,
                                  rows, size_t(Lp) * 4, size_t(e.L) * 4, nu,
                                  cudaMemcpyDeviceToDevice, st));

  // K1: compressed heads select l_h (prefill_init, engine.py:265-268), pivots
  // select l_base for K_base (engine.py:269-271).
  std::vector<hc_topk_job> jobs;
  std::vector<int> job_unit;
  for (int i = 0; i < nu; ++i) {
    const int b = i / e.H, h = i % e.H;
    const int u = (b * e.NL + layer) * e.H + h;
    const int r = e.role[layer * e.H + h];
    if (!e.owned[u]) continue;
    hc_topk_job j{};
    j.scores = rows + size_t(i) * Lp;
    j.n = uint32_t(e.L);
    if (r == HC_ROLE_ANCHOR || r == HC_ROLE_SATELLITE) {
      j.k = uint32_t(e.length[layer * e.H + h]);
      j.out_idx = e.dyn_sel[u];
      j.out_count = e.dyn_cnt[u];
    } else if (r == HC_ROLE_PIVOT && e.piv_slot[u] >= 0) {
      const int s = e.piv_slot[u];
      j.k = uint32_t(e.lbase);
      j.out_idx = e.top_idx + size_t(s) * e.lbase;
      j.out_count = e.top_cnt + s;
    } else {
      continue;
    }
    jobs.push_back(j);
    job_unit.push_back(u);
  }
  if (!jobs.empty()) {
    hc_topk_job* dj = reinterpret_cast<hc_topk_job*>(pf + o_jobs);
    HC_CUDA_TRY(cudaMemcpyAsync(dj, jobs.data(), jobs.size() * sizeof(hc_topk_job),
                                cudaMemcpyHostToDevice, st));
    HC_TRY(launch_topk(dj, int(jobs.size()), 0, st));
  }
  // K_base bitmaps for pivots
  std::vector<int32_t> pslots;
  for (int u : job_unit)
    if (e.piv_slot[u] >= 0) pslots.push_back(e.piv_slot[u]);
  if (!pslots.empty()) {
    int32_t* ds = nullptr;
    HC_TRY(upload(e, pslots.data(), pslots.size() * 4, st, (void**)&ds));
    restamp_batch_kernel<<<int(pslots.size()), 1024, 0, st>>>(e.kbase, e.top_idx, e.top_cnt, ds,
                                                              e.words, e.lbase);
    HC_CHECK_LAUNCH();
    HC_CUDA_TRY(cudaFreeAsync(ds, st));
  }
  // caches: full heads whole, compressed heads gathered (batched), satellites to the host pool
  const size_t rowb = size_t(kHeadDim) * 2;
  std::vector<XferDev> xd;
  std::vector<LandDev> lds;
  for (int i = 0; i < nu; ++i) {
    const int b = i / e.H, h = i % e.H;
    const int u = (b * e.NL + layer) * e.H + h;
    const __nv_bfloat16* sk = k + size_t(i) * e.L * kHeadDim;
    const __nv_bfloat16* sv = v + size_t(i) * e.L * kHeadDim;
    const UnitDesc& d = e.units[u];
    if (d.kind == kUnitAbsent) continue;
    if (d.kind == kUnitFull) {
      HC_CUDA_TRY(cudaMemcpyAsync(e.K + size_t(d.row0) * kHeadDim, sk, rowb * e.L,
                                  cudaMemcpyDeviceToDevice, st));
      HC_CUDA_TRY(cudaMemcpyAsync(e.V + size_t(d.row0) * kHeadDim, sv, rowb * e.L,
                                  cudaMemcpyDeviceToDevice, st));
      continue;
    }
    // decode starts at step 1: the recency tail then covers [L+1-R, L)
    xd.push_back(XferDev{e.dyn_sel[u], e.dyn_cnt[u], e.pre_pos[u], e.pre_meta[u],
                         reinterpret_cast<const uint4*>(sk), reinterpret_cast<const uint4*>(sv),
                         e.buf_row0[u], 1, 0});
    lds.push_back(LandDev{u, 0, e.buf_row0[u], e.pre_meta[u]});
    e.active[u] = 0;
    const int ss = e.sat_slot[u];
    if (ss >= 0) {
      __nv_bfloat16* dk = e.pool + size_t(ss) * 2 * e.L * kHeadDim;
      __nv_bfloat16* dv = dk + size_t(e.L) * kHeadDim;
      const cudaMemcpyKind kind = e.pool_host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
      HC_CUDA_TRY(cudaMemcpyAsync(dk, sk, rowb * e.L, kind, st));
      HC_CUDA_TRY(cudaMemcpyAsync(dv, sv, rowb * e.L, kind, st));
    }
  }
  if (!xd.empty()) {
    XferDev* dx = nullptr;
    LandDev* dl = nullptr;
    int max_cap = 1;
    for (const auto& l : lds) max_cap = std::max(max_cap, e.cap[l.unit]);
    HC_TRY(upload(e, xd.data(), xd.size() * sizeof(XferDev), st, (void**)&dx));
    HC_TRY(upload(e, lds.data(), lds.size() * sizeof(LandDev), st, (void**)&dl));
    build_positions_batch_kernel<<<int(xd.size()), 256, 0, st>>>(dx, e.L, e.S, e.R);
    HC_CHECK_LAUNCH();
    const int per = std::max(1, std::min(64, (max_cap + 127) / 128));
    gather_rows_batch_kernel<<<dim3(per, int(xd.size())), 256, 0, st>>>(
        dx, reinterpret_cast<uint4*>(e.K), reinterpret_cast<uint4*>(e.V));
    HC_CHECK_LAUNCH();
    set_prefix_batch_kernel<<<int((lds.size() + 127) / 128), 128, 0, st>>>(e.d_units, dl,
                                                                           int(lds.size()));
    HC_CHECK_LAUNCH();
    HC_CUDA_TRY(cudaFreeAsync(dx, st));
    HC_CUDA_TRY(cudaFreeAsync(dl, st));
  }
  // (host vectors above were staged by cudaMemcpyAsync from pageable memory)
  return HC_OK;
}

int engine_fire_batch(EngineImpl& e, int n, const int32_t* pus, int t, const int32_t* completion,
                      int32_t* ids, uint32_t* fetched_host, cudaStream_t caller) {
  // Selection, K_base restamp and the fetched-set copies run on the side
  // stream after the rows they read: inside an open step (decode_begin) that
  // is the end of the previous step, so they overlap the step's K4; outside,
  // everything queued on the caller's stream so far.  The caller's stream
  // then waits for them (later score rows overwrite the rows, the monitor
  // reads K_base).
  cudaStream_t st = e.side;
  if (e.step_end) HC_CUDA_TRY(cudaStreamWaitEvent(st, e.step_end, 0));
  if (!e.in_step) {
    cudaEvent_t dep;
    HC_TRY(new_event(e, &dep));
    HC_CUDA_TRY(cudaEventRecord(dep, caller));
    HC_CUDA_TRY(cudaStreamWaitEvent(st, dep, 0));
  }
  std::vector<hc_topk_job> jobs;
  std::vector<FireJob> fjobs;
  // the rows of step t still have their key histograms (buffer t&1) until
  // step t+1's monitor: fast two-pass selection (fire_select_kernel)
  const bool fast = e.ghist && t >= 1 && t == e.last_t;
  std::vector<int> new_ids;
  std::vector<int32_t> slots;
  const int LH = e.NL * e.H;
  // pass 1: the transfers (one per satellite of each firing pivot) and their sizes
  struct Pending {
    Transfer x;
    int slot;
  };
  std::vector<Pending> pend;
  for (int f = 0; f < n; ++f) {
    const int pu = pus[f];
    HC_REQUIRE(pu >= 0 && pu < e.n_units && e.piv_slot[pu] >= 0, HC_EINVAL,
               "unit %d is not a monitored pivot", pu);
    const int s = e.piv_slot[pu];
    slots.push_back(s);
    const int b = pu / LH, i = e.lh(pu), l = i / e.H, ph = i % e.H;
    for (int h = 0; h < e.H; ++h) {
      const int j = l * e.H + h;
      if (e.role[j] != HC_ROLE_SATELLITE || e.cpivot[j] != ph) continue;
      Transfer x;
      x.unit = (b * e.NL + l) * e.H + h;
      x.k = std::min(e.length[j], e.L + t);
      x.completion = completion[f];
      pend.push_back({x, s});
    }
  }
  // pass 2: one allocation [sel_0 .. sel_m | cnt x m | pos_0 .. pos_m | meta x m]
  // (fetched sets contiguous in firing order: a single D2H copy below)
  size_t n_sel = 0, n_pos = 0;
  for (const Pending& q : pend) {
    n_sel += size_t(std::max(1, q.x.k));
    n_pos += (size_t(std::max(1, e.cap[q.x.unit])) + 3) & ~size_t(3);
  }
  const size_t m = pend.size();
  const size_t o_cnt = (n_sel + 3) & ~size_t(3), o_pos = o_cnt + ((m + 3) & ~size_t(3));
  const size_t o_meta = o_pos + n_pos, words_total = o_meta + 4 * m;
  uint32_t* blk = nullptr;
  const int block_id = e.next_block++;
  if (m) {
    HC_CUDA_TRY(cudaMallocFromPoolAsync((void**)&blk, words_total * 4, e.mpool, st));
    e.blocks[block_id] = EngineImpl::XferBlock{blk, int(m)};
  }
  size_t a_sel = 0, a_pos = o_pos;
  for (size_t q = 0; q < m; ++q) {
    Transfer& x = pend[q].x;
    const int s = pend[q].slot;
    x.block = block_id;
    x.sel = blk + a_sel;
    x.cnt = blk + o_cnt + q;
    x.pos = blk + a_pos;
    x.meta = reinterpret_cast<int32_t*>(blk + o_meta + 4 * q);
    a_sel += size_t(std::max(1, x.k));
    a_pos += (size_t(std::max(1, e.cap[x.unit])) + 3) & ~size_t(3);
    if (fast) {
      fjobs.push_back(FireJob{e.rowbuf + size_t(s) * e.row_len,
                              e.ghist + (size_t(t & 1) * e.n_piv + s) * 8192, uint32_t(e.L + t),
                              uint32_t(x.k), x.sel, x.cnt});
    } else {
      hc_topk_job jb{};
      jb.scores = e.rowbuf + size_t(s) * e.row_len;
      jb.n = uint32_t(e.L + t);
      jb.k = uint32_t(x.k);
      jb.out_idx = x.sel;
      jb.out_count = x.cnt;
      jobs.push_back(jb);
    }
    new_ids.push_back(e.xfers.add(x));
  }
  if (!jobs.empty()) {
    // pageable -> device copies are staged before cudaMemcpyAsync returns
    hc_topk_job* dj = nullptr;
    HC_TRY(upload(e, jobs.data(), jobs.size() * sizeof(hc_topk_job), st, (void**)&dj));
    HC_TRY(launch_topk(dj, int(jobs.size()), 0, st));
    HC_CUDA_TRY(cudaFreeAsync(dj, st));
  }
  if (!fjobs.empty()) {
    FireJob* dj = nullptr;
    HC_TRY(upload(e, fjobs.data(), fjobs.size() * sizeof(FireJob), st, (void**)&dj));
    HC_TRY(launch_fire_select(dj, int(fjobs.size()), st));
    HC_CUDA_TRY(cudaFreeAsync(dj, st));
  }
  if (n > 0) {  // K_base <- current top set (engine.py:357), from the monitor threshold
    int32_t* ds = nullptr;
    HC_TRY(upload(e, slots.data(), slots.size() * 4, st, (void**)&ds));
    HC_TRY(launch_restamp_threshold(e.rowbuf, e.row_len, ds, n, uint32_t(e.L + t), e.thr,
                                    e.kbase, e.words, st));
    HC_CUDA_TRY(cudaFreeAsync(ds, st));
  }
  // fetched sets, in firing order, packed at k per transfer (the block pads k = 0 to 1)
  size_t off = 0;
  for (size_t q = 0; q < new_ids.size(); ++q) {
    off += size_t(e.xfers[new_ids[q]].k);
    ids[q] = new_ids[q];
  }
  if (fetched_host && m) {
    bool packed = true;  // k >= 1 for every transfer: device and host layouts coincide
    for (const Pending& q : pend) packed &= q.x.k >= 1;
    if (packed) {
      HC_CUDA_TRY(cudaMemcpyAsync(fetched_host, blk, off * 4, cudaMemcpyDeviceToHost, st));
    } else {
      size_t ho = 0, dof = 0;
      for (const Pending& q : pend) {
        if (q.x.k > 0)
          HC_CUDA_TRY(cudaMemcpyAsync(fetched_host + ho, blk + dof, size_t(q.x.k) * 4,
                                      cudaMemcpyDeviceToHost, st));
        ho += size_t(q.x.k);
        dof += size_t(std::max(1, q.x.k));
      }
    }
  }
  cudaEvent_t selected;
  HC_TRY(new_event(e, &selected));
  HC_CUDA_TRY(cudaEventRecord(selected, st));
  e.last_selected = selected;  // after the fetched-set D2H copies (hc_engine_wait_fetched)
  HC_CUDA_TRY(cudaStreamWaitEvent(caller, selected, 0));
  std::vector<int> now;
  for (int id : new_ids) {
    Transfer& x = e.xfers[id];
    x.selected = selected;
    e.fifo[x.unit].push_back(id);
    if (e.fifo[x.unit].size() == 1) now.push_back(id);
  }
  return issue_gathers(e, now, selected);
}

// hc_engine_land_batch: validate now, apply inside the next decode step (or
// at the next call that reads engine state).
int engine_land_batch(EngineImpl& e, int n, const int32_t* ids, cudaStream_t st) {
  if (e.in_step) {
    HC_REQUIRE(e.cur_hold, HC_ESTATE,
               "landing inside an open step needs decode_begin(hold_satellites=1)");
    HC_REQUIRE(st == e.cur_st, HC_EINVAL, "landing on another stream than the open step");
  } else {
    HC_TRY(flush_deferred(e));
  }
  std::vector<std::pair<int, size_t>> seen;  // (unit, landings already requested)
  for (int id : e.deferred) {
    const int u = e.xfers[id].unit;
    bool found = false;
    for (auto& pr : seen)
      if (pr.first == u) ++pr.second, found = true;
    if (!found) seen.emplace_back(u, 1);
  }
  for (int q = 0; q < n; ++q) {
    const int id = ids[q];
    HC_REQUIRE(e.xfers.contains(id), HC_EINVAL, "bad transfer id %d", id);
    const Transfer& x = e.xfers[id];
    HC_REQUIRE(!x.landed, HC_ESTATE, "transfer %d already landed", id);
    HC_REQUIRE(std::find(ids, ids + q, id) == ids + q &&
                   std::find(e.deferred.begin(), e.deferred.end(), id) == e.deferred.end(),
               HC_ESTATE, "transfer %d landed twice", id);
    size_t k = 0;
    bool found = false;
    for (auto& pr : seen)
      if (pr.first == x.unit) k = pr.second++, found = true;
    if (!found) seen.emplace_back(x.unit, 1);
    HC_REQUIRE(e.fifo[x.unit].size() > k && e.fifo[x.unit][k] == id, HC_ESTATE,
               "transfer %d lands out of order", id);
  }
  e.deferred.insert(e.deferred.end(), ids, ids + n);
  e.deferred_st = st;
  return HC_OK;
}

int apply_landings(EngineImpl& e, const std::vector<int>& idv, cudaStream_t st) {
  const int n = int(idv.size());
  const int32_t* ids = idv.data();
  std::vector<LandDev> lds;
  std::vector<int> landed_units;
  cudaEvent_t last_wait = nullptr;
  auto flush = [&]() -> int {
    if (lds.empty()) return HC_OK;
    LandDev* d = nullptr;
    HC_TRY(upload(e, lds.data(), lds.size() * sizeof(LandDev), st, (void**)&d));
    set_prefix_batch_kernel<<<int((lds.size() + 127) / 128), 128, 0, st>>>(e.d_units, d,
                                                                           int(lds.size()));
    HC_CHECK_LAUNCH();
    HC_CUDA_TRY(cudaFreeAsync(d, st));
    lds.clear();
    return HC_OK;
  };
  for (int q = 0; q < n; ++q) {
    const int id = ids[q];
    HC_REQUIRE(e.xfers.contains(id), HC_EINVAL, "bad transfer id %d", id);
    Transfer& x = e.xfers[id];
    HC_REQUIRE(!x.landed, HC_ESTATE, "transfer %d already landed", id);
    const int u = x.unit;
    HC_REQUIRE(!e.fifo[u].empty() && e.fifo[u].front() == id, HC_ESTATE,
               "transfer %d lands out of order", id);
    if (!x.gathered) {
      // its unit's staging buffer was busy with an earlier transfer that
      // landed just before: apply pending descriptor updates, then gather
      HC_TRY(flush());
      cudaEvent_t ev;
      HC_TRY(new_event(e, &ev));
      HC_CUDA_TRY(cudaEventRecord(ev, st));
      HC_TRY(issue_gathers(e, {id}, ev));
    }
    if (x.done != last_wait) {
      cudaEvent_t w0 = nullptr, w1 = nullptr;
      if (e.timing) {
        HC_TRY(timed_event(e, &w0));
        HC_TRY(timed_event(e, &w1));
        HC_CUDA_TRY(cudaEventRecord(w0, st));
      }
      HC_CUDA_TRY(cudaStreamWaitEvent(st, x.done, 0));
      if (e.timing) {
        HC_CUDA_TRY(cudaEventRecord(w1, st));
        e.land_ev.emplace_back(w0, w1);
      }
      last_wait = x.done;
    }
    lds.push_back(LandDev{u, 0, x.buf ? e.buf_row1[u] : e.buf_row0[u], x.meta});
    e.active[u] = x.buf;
    if (e.dyn_owner[u] >= 0) {  // superseded records
      Transfer& old = e.xfers[e.dyn_owner[u]];
      auto bl = e.blocks.find(old.block);
      if (bl != e.blocks.end() && --bl->second.refs == 0) {
        HC_CUDA_TRY(cudaFreeAsync(bl->second.ptr, st));
        e.blocks.erase(bl);
      }
      e.xfers.erase(e.dyn_owner[u]);
    }
    e.dyn_owner[u] = id;
    x.landed = true;
    e.fifo[u].pop_front();
    landed_units.push_back(u);
  }
  HC_TRY(flush());
  // queued gathers may now overwrite the freed buffers: order them after this point
  std::vector<int> next;
  for (int u : landed_units)
    if (!e.fifo[u].empty() && !e.xfers[e.fifo[u].front()].gathered) {
      const int id = e.fifo[u].front();
      if (std::find(next.begin(), next.end(), id) == next.end()) next.push_back(id);
    }
  if (!next.empty()) {
    cudaEvent_t ev;
    HC_TRY(new_event(e, &ev));
    HC_CUDA_TRY(cudaEventRecord(ev, st));
    HC_TRY(issue_gathers(e, next, ev));
  }
  return HC_OK;
}

const uint32_t* dyn_list(const EngineImpl& e, int u, const uint32_t** cnt) {
  if (e.dyn_owner[u] >= 0) {
    *cnt = e.xfers[e.dyn_owner[u]].cnt;
    return e.xfers[e.dyn_owner[u]].sel;
  }
  *cnt = e.dyn_cnt[u];
  return e.dyn_sel[u];
}

// ---- measure mode ----------------------------------------------------------

__global__ void copy_pivot_rows_kernel(float* __restrict__ mrows, const float* __restrict__ rows,
                                       const int32_t* __restrict__ piv_mu, int64_t stride,
                                       int n) {
  const int s = blockIdx.y;
  const float4* src = reinterpret_cast<const float4*>(rows + size_t(s) * stride);
  float4* dst = reinterpret_cast<float4*>(mrows + size_t(piv_mu[s]) * stride);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < (n + 3) / 4; i += gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// records -> composite keys (score_key << 32 | ~index); 0 past the count
__global__ void record_keys_kernel(const float* __restrict__ mrows, int64_t stride,
                                   const uint32_t* __restrict__ idx,
                                   const uint32_t* __restrict__ cnt, int kmax,
                                   uint64_t* __restrict__ keys) {
  const int m = blockIdx.y;
  const uint32_t c = cnt[m];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < kmax; i += gridDim.x * blockDim.x) {
    const size_t o = size_t(m) * kmax + i;
    uint64_t k = 0;
    if (uint32_t(i) < c) {
      const uint32_t p = idx[o];
      k = (uint64_t(score_key(mrows[size_t(m) * stride + p])) << 32) | uint64_t(~p);
    }
    keys[o] = k;
  }
}

// sorted keys -> records in (score desc, index asc) order, PAD tail
__global__ void record_unpack_kernel(const float* __restrict__ mrows, int64_t stride,
                                     const uint64_t* __restrict__ keys, int kmax,
                                     uint32_t* __restrict__ idx, float* __restrict__ sc) {
  const int m = blockIdx.y;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < kmax; i += gridDim.x * blockDim.x) {
    const size_t o = size_t(m) * kmax + i;
    const uint64_t k = keys[o];
    if (k) {
      const uint32_t p = ~uint32_t(k);
      idx[o] = p;
      sc[o] = mrows[size_t(m) * stride + p];
    } else {
      idx[o] = HC_PAD_INDEX;
      sc[o] = 0.f;
    }
  }
}

struct BitmapJob {
  const uint32_t* sel;
  const uint32_t* cnt;
  uint32_t* bm;
};

__global__ void bitmaps_kernel(const BitmapJob* __restrict__ jobs, int words) {
  const BitmapJob j = jobs[blockIdx.x];
  for (int w = threadIdx.x; w < words; w += blockDim.x) j.bm[w] = 0u;
  __syncthreads();
  const uint32_t c = *j.cnt;
  for (uint32_t i = threadIdx.x; i < c; i += blockDim.x) {
    const uint32_t p = j.sel[i];
    if (int(p >> 5) < words) atomicOr(j.bm + (p >> 5), 1u << (p & 31));
  }
}

int engine_enable_measure(EngineImpl& e, int recall_topk) {
  HC_REQUIRE(e.n_absent == 0, HC_EINVAL,
             "measure mode needs every head of every sequence (unsharded engine)");
  HC_REQUIRE(recall_topk >= 1, HC_EINVAL, "recall_topk must be >= 1");
  HC_REQUIRE(!e.rec_k && e.pf_layers == 0, HC_ESTATE, "enable measure once, before prefill");
  const int nm = e.NL * e.B * e.H;
  const int64_t srows = int64_t(e.L) + e.T;
  e.rec_k = recall_topk;
  // enough records for every selection the reference makes from them: step 0
  // (all heads) feeds prefill_init's top-l_h (engine.py:263-271); pivots'
  // records feed the monitor (l_base_int) and every fetch of their
  // satellites (top-l_s of the pivot row, engine.py:326-329)
  int kmax = e.n_piv ? e.lbase : 0;
  for (int j = 0; j < e.NL * e.H; ++j)
    if (e.role[j] == HC_ROLE_ANCHOR || e.role[j] == HC_ROLE_SATELLITE)
      kmax = std::max(kmax, e.length[j]);
  e.rec_kmax = std::max(recall_topk, kmax);
  HC_TRY(dalloc((void**)&e.shadowK, size_t(nm) * srows * kHeadDim * 2, &e.dev_bytes));
  HC_TRY(dalloc((void**)&e.mrows, size_t(nm) * e.row_len * 4, &e.dev_bytes));
  HC_TRY(dalloc((void**)&e.rec_idx, size_t(nm) * e.rec_kmax * 4, &e.dev_bytes));
  HC_TRY(dalloc((void**)&e.rec_sc, size_t(nm) * e.rec_kmax * 4, &e.dev_bytes));
  HC_TRY(dalloc((void**)&e.rec_cnt, size_t(nm) * 4, &e.dev_bytes));
  HC_TRY(dalloc((void**)&e.dynbm, size_t(e.n_units) * e.words * 4, &e.dev_bytes));
  HC_TRY(dalloc((void**)&e.rec_out, size_t(nm) * 8, &e.dev_bytes));
  std::vector<hc_topk_job> jobs(2 * nm);
  std::vector<hc_recall_head> heads(nm);
  for (int u = 0; u < e.n_units; ++u) {
    const int m = e.mu_of(u);
    const bool piv = e.piv_slot[u] >= 0;
    hc_topk_job& j = jobs[m];
    j = hc_topk_job{};
    j.scores = e.mrows + size_t(m) * e.row_len;
    j.n = uint32_t(e.L);  // + step (n_add)
    j.k = uint32_t(piv ? e.rec_kmax : e.rec_k);
    j.out_idx = e.rec_idx + size_t(m) * e.rec_kmax;
    j.out_count = e.rec_cnt + m;
    jobs[nm + m] = j;
    jobs[nm + m].k = uint32_t(e.rec_kmax);
    heads[m].idx = e.rec_idx + size_t(m) * e.rec_kmax;
    heads[m].scores = e.rec_sc + size_t(m) * e.rec_kmax;
    heads[m].dynamic = e.units[u].kind == kUnitComp ? e.dynbm + size_t(u) * e.words : nullptr;
  }
  HC_TRY(dalloc((void**)&e.rec_keys, 2 * size_t(nm) * e.rec_kmax * 8, &e.dev_bytes));
  {
    std::vector<int> off(nm + 1);
    for (int m = 0; m <= nm; ++m) off[m] = m * e.rec_kmax;
    HC_REQUIRE(int64_t(nm) * e.rec_kmax < (int64_t(1) << 31), HC_EINVAL, "too many records");
    HC_TRY(dalloc((void**)&e.rec_off, off.size() * 4, &e.dev_bytes));
    HC_CUDA_TRY(cudaMemcpy(e.rec_off, off.data(), off.size() * 4, cudaMemcpyHostToDevice));
    HC_TRY(segmented_sort_desc_u64(nullptr, &e.sort_tmp_bytes, e.rec_keys,
                                   e.rec_keys + size_t(nm) * e.rec_kmax, nm * e.rec_kmax, nm,
                                   e.rec_off, 0));
    HC_TRY(dalloc(&e.sort_tmp, e.sort_tmp_bytes, &e.dev_bytes));
  }
  HC_TRY(dalloc((void**)&e.d_mjobs, jobs.size() * sizeof(hc_topk_job), &e.dev_bytes));
  HC_CUDA_TRY(cudaMemcpy(e.d_mjobs, jobs.data(), jobs.size() * sizeof(hc_topk_job),
                         cudaMemcpyHostToDevice));
  HC_TRY(dalloc((void**)&e.d_rheads, heads.size() * sizeof(hc_recall_head), &e.dev_bytes));
  HC_CUDA_TRY(cudaMemcpy(e.d_rheads, heads.data(), heads.size() * sizeof(hc_recall_head),
                         cudaMemcpyHostToDevice));
  std::vector<int32_t> pm(std::max(1, e.n_piv));
  for (int s2 = 0; s2 < e.n_piv; ++s2) pm[s2] = e.mu_of(e.piv_units[s2]);
  HC_TRY(dalloc((void**)&e.d_piv_mu, pm.size() * 4, &e.dev_bytes));
  HC_CUDA_TRY(cudaMemcpy(e.d_piv_mu, pm.data(), pm.size() * 4, cudaMemcpyHostToDevice));
  const int nu = e.B * e.H;
  size_t obs = 0;
  for (int64_t n = e.L; n <= srows; n += std::max<int64_t>(1, (srows - e.L) / 8 + 1))
    obs = std::max(obs, obs_scratch_bytes(nu, int(n), e.G));
  obs = std::max(obs, obs_scratch_bytes(nu, int(srows), e.G));
  e.mscratch_bytes = ((size_t(nu) * e.G * kHeadDim * 2 + 255) & ~size_t(255)) + obs;
  HC_TRY(dalloc((void**)&e.mscratch, e.mscratch_bytes, &e.dev_bytes));
  return HC_OK;
}

// Recall of every head at step t (after decode step t; t = 0: after prefill).
// q: the step's queries [B][NL][H*G][128] (unused at t = 0: the step-0 rows
// are the prefill rows).  recall_out (host, optional): per unit u.
int engine_measure(EngineImpl& e, int t, const void* q, double* recall_out, cudaStream_t st) {
  HC_REQUIRE(e.rec_k, HC_ESTATE, "measure mode is off (hc_engine_enable_measure)");
  HC_REQUIRE(e.in_step == 0, HC_ESTATE, "measure inside an open step");
  HC_REQUIRE(t == 0 ? e.pf_layers >= e.NL : (t == e.last_t && q), HC_EINVAL,
             "measure(%d): run it right after that step", t);
  const int nu = e.B * e.H, nm = e.NL * nu;
  const int64_t srows = int64_t(e.L) + e.T;
  const int len = e.L + t;
  if (t > 0) {
    __nv_bfloat16* qp = reinterpret_cast<__nv_bfloat16*>(e.mscratch);
    char* obs = e.mscratch + ((size_t(nu) * e.G * kHeadDim * 2 + 255) & ~size_t(255));
    HC_REQUIRE(obs_scratch_bytes(nu, len, e.G) + (obs - e.mscratch) <= e.mscratch_bytes, HC_EINVAL,
               "measure scratch too small");
    const size_t qrow = size_t(e.H) * e.G * kHeadDim * 2;  // one (b, layer) block of queries
    for (int l = 0; l < e.NL; ++l) {
      HC_CUDA_TRY(cudaMemcpy2DAsync(qp, qrow, static_cast<const char*>(q) + size_t(l) * qrow,
                                    qrow * e.NL, qrow, e.B, cudaMemcpyDeviceToDevice, st));
      HC_TRY(launch_obs_scores(e.shadowK + size_t(l) * nu * srows * kHeadDim, qp, e.B, e.H, e.G,
                               1, len, e.mrows + size_t(l) * nu * e.row_len, e.row_len, obs, st,
                               srows));
    }
    if (e.n_piv) {  // the pivots' rows are the engine's own (the decision rows)
      if (e.step_end) HC_CUDA_TRY(cudaStreamWaitEvent(st, e.step_end, 0));
      copy_pivot_rows_kernel<<<dim3(64, e.n_piv), 256, 0, st>>>(e.mrows, e.rowbuf, e.d_piv_mu,
                                                                e.row_len, len);
      HC_CHECK_LAUNCH();
    }
  }
  HC_TRY(launch_topk(e.d_mjobs + (t == 0 ? nm : 0), nm, uint32_t(t), st));
  {  // records in HCTRACE1 order: score descending, index ascending
    const dim3 g(std::max(1, std::min(64, (e.rec_kmax + 255) / 256)), nm);
    uint64_t* kin = e.rec_keys;
    uint64_t* kout = e.rec_keys + size_t(nm) * e.rec_kmax;
    record_keys_kernel<<<g, 256, 0, st>>>(e.mrows, e.row_len, e.rec_idx, e.rec_cnt, e.rec_kmax,
                                          kin);
    HC_CHECK_LAUNCH();
    HC_TRY(segmented_sort_desc_u64(e.sort_tmp, &e.sort_tmp_bytes, kin, kout, nm * e.rec_kmax, nm,
                                   e.rec_off, st));
    record_unpack_kernel<<<g, 256, 0, st>>>(e.mrows, e.row_len, kout, e.rec_kmax, e.rec_idx,
                                            e.rec_sc);
    HC_CHECK_LAUNCH();
  }
  std::vector<BitmapJob> bj;
  for (int u = 0; u < e.n_units; ++u) {
    if (e.units[u].kind != kUnitComp) continue;
    const uint32_t* cnt = nullptr;
    const uint32_t* sel = dyn_list(e, u, &cnt);
    bj.push_back(BitmapJob{sel, cnt, e.dynbm + size_t(u) * e.words});
  }
  if (!bj.empty()) {
    BitmapJob* d = nullptr;
    HC_TRY(upload(e, bj.data(), bj.size() * sizeof(BitmapJob), st, (void**)&d));
    bitmaps_kernel<<<int(bj.size()), 256, 0, st>>>(d, e.words);
    HC_CHECK_LAUNCH();
    HC_CUDA_TRY(cudaFreeAsync(d, st));
  }
  HC_TRY_RC(hc_trace_recall(e.d_rheads, nm, uint32_t(e.rec_kmax), 0, uint32_t(e.L), uint32_t(t),
                            uint32_t(e.S), uint32_t(e.R), e.rec_out, st));
  e.measured_t = t;
  if (recall_out) {
    std::vector<double> r(nm);
    HC_CUDA_TRY(cudaMemcpyAsync(r.data(), e.rec_out, size_t(nm) * 8, cudaMemcpyDeviceToHost, st));
    HC_CUDA_TRY(cudaStreamSynchronize(st));
    for (int u = 0; u < e.n_units; ++u) recall_out[u] = r[e.mu_of(u)];
  }
  return HC_OK;
}

}  // namespace
}  // namespace hc

// ============================== C ABI ======================================

extern "C" int hc_engine_create(const hc_engine_desc* desc, const int32_t* roles,
                                const int32_t* lengths, const int32_t* cluster_pivot,
                                hc_engine** out) {
  return hc_engine_create_sharded(desc, roles, lengths, cluster_pivot, nullptr, out);
}

extern "C" int hc_engine_create_sharded(const hc_engine_desc* desc, const int32_t* roles,
                                        const int32_t* lengths, const int32_t* cluster_pivot,
                                        const uint8_t* owned, hc_engine** out) {
  HC_REQUIRE(desc && roles && lengths && cluster_pivot && out, HC_EINVAL,
             "hc_engine_create: null argument");
  *out = nullptr;
  hc_engine* h = new (std::nothrow) hc_engine();
  HC_REQUIRE(h, HC_ENOMEM, "out of host memory");
  const int rc = hc::engine_create(h->e, *desc, roles, lengths, cluster_pivot, owned);
  if (rc != HC_OK) {
    hc::engine_destroy(h->e);
    delete h;
    return rc;
  }
  *out = h;
  return HC_OK;
}

extern "C" int hc_engine_destroy(hc_engine* eng) {
  if (!eng) return HC_OK;
  hc::engine_destroy(eng->e);
  delete eng;
  return HC_OK;
}

extern "C" int hc_engine_info(const hc_engine* eng, int64_t* out4) {
  HC_REQUIRE(eng && out4, HC_EINVAL, "null argument");
  out4[0] = eng->e.dev_bytes;
  out4[1] = eng->e.host_bytes;
  out4[2] = eng->e.rows;
  out4[3] = eng->e.n_piv;
  return HC_OK;
}

extern "C" int hc_engine_prefill_layer(hc_engine* eng, int32_t layer, const void* k_dev,
                                       const void* v_dev, const void* q_last_dev, void* stream) {
  HC_REQUIRE(eng && k_dev && v_dev && q_last_dev, HC_EINVAL, "null argument");
  HC_TRY(hc::flush_deferred(eng->e));  // pending landings first
  return hc::engine_prefill_layer(eng->e, layer, (const __nv_bfloat16*)k_dev,
                                  (const __nv_bfloat16*)v_dev, (const __nv_bfloat16*)q_last_dev,
                                  (cudaStream_t)stream);
}

extern "C" int hc_engine_decode_step(hc_engine* eng, int32_t step, const void* q_dev,
                                     const void* k_new_dev, const void* v_new_dev, void* o_dev,
                                     void* stream) {
  HC_REQUIRE(eng && q_dev && k_new_dev && v_new_dev && o_dev, HC_EINVAL, "null argument");
  return hc::engine_decode_step(eng->e, step, q_dev, k_new_dev, v_new_dev, o_dev,
                                (cudaStream_t)stream);
}

extern "C" int hc_engine_decode_begin(hc_engine* eng, int32_t step, const void* q_dev,
                                      const void* k_new_dev, const void* v_new_dev, void* o_dev,
                                      int32_t hold_satellites, void* stream) {
  HC_REQUIRE(eng && q_dev && k_new_dev && v_new_dev && o_dev, HC_EINVAL, "null argument");
  return hc::engine_decode_begin(eng->e, step, q_dev, k_new_dev, v_new_dev, o_dev,
                                 hold_satellites != 0, (cudaStream_t)stream);
}

extern "C" int hc_engine_decode_end(hc_engine* eng, int32_t step, void* stream) {
  HC_REQUIRE(eng, HC_EINVAL, "null argument");
  return hc::engine_decode_end(eng->e, step, (cudaStream_t)stream);
}

extern "C" int hc_engine_enable_measure(hc_engine* eng, int32_t recall_topk) {
  HC_REQUIRE(eng, HC_EINVAL, "null argument");
  HC_REQUIRE(!eng->e.devdec, HC_ESTATE, "measure mode needs host decisions");
  return hc::engine_enable_measure(eng->e, recall_topk);
}

extern "C" int hc_engine_measure(hc_engine* eng, int32_t step, const void* q_dev,
                                 double* recall_out_host, void* stream) {
  HC_REQUIRE(eng, HC_EINVAL, "null argument");
  HC_TRY(hc::flush_deferred(eng->e));
  return hc::engine_measure(eng->e, step, q_dev, recall_out_host, (cudaStream_t)stream);
}

extern "C" int hc_engine_measure_records(hc_engine* eng, int32_t unit, uint32_t* idx_host,
                                         float* scores_host, int32_t capacity, void* stream) {
  HC_REQUIRE(eng && idx_host && scores_host, HC_EINVAL, "null argument");
  auto& e = eng->e;
  HC_REQUIRE(e.rec_k && e.measured_t >= 0, HC_ESTATE, "nothing measured yet");
  HC_REQUIRE(unit >= 0 && unit < e.n_units, HC_EINVAL, "bad unit %d", unit);
  HC_REQUIRE(capacity >= e.rec_kmax, HC_EINVAL, "capacity %d < %d records", capacity, e.rec_kmax);
  cudaStream_t st = (cudaStream_t)stream;
  const size_t o = size_t(e.mu_of(unit)) * e.rec_kmax;
  HC_CUDA_TRY(cudaMemcpyAsync(idx_host, e.rec_idx + o, size_t(e.rec_kmax) * 4,
                              cudaMemcpyDeviceToHost, st));
  HC_CUDA_TRY(cudaMemcpyAsync(scores_host, e.rec_sc + o, size_t(e.rec_kmax) * 4,
                              cudaMemcpyDeviceToHost, st));
  HC_CUDA_TRY(cudaStreamSynchronize(st));
  return HC_OK;
}

extern "C" int hc_engine_join(hc_engine* eng, void* stream) {
  HC_REQUIRE(eng, HC_EINVAL, "null argument");
  if (eng->e.step_end)
    HC_CUDA_TRY(cudaStreamWaitEvent((cudaStream_t)stream, eng->e.step_end, 0));
  if (eng->e.pivot_first && eng->e.step_out)  // pivot-first: the step's O (caller's stream)
    HC_CUDA_TRY(cudaStreamWaitEvent((cudaStream_t)stream, eng->e.step_out, 0));
  if (eng->e.h_last >= 0)  // the last decode_step_host download
    HC_CUDA_TRY(cudaStreamWaitEvent((cudaStream_t)stream, eng->e.h_out[eng->e.h_last], 0));
  return HC_OK;
}

extern "C" int hc_engine_decode_step_host(hc_engine* eng, int32_t step, const void* q_host,
                                          const void* k_new_host, const void* v_new_host,
                                          void* o_host, void* stream) {
  HC_REQUIRE(eng && q_host && k_new_host && v_new_host && o_host, HC_EINVAL, "null argument");
  return hc::engine_decode_step_host(eng->e, step, q_host, k_new_host, v_new_host, o_host,
                                     (cudaStream_t)stream);
}

extern "C" int hc_engine_overlaps(hc_engine* eng, int32_t first, int32_t last, int32_t* out,
                                  void* stream) {
  HC_REQUIRE(eng && out, HC_EINVAL, "null argument");
  HC_REQUIRE(!eng->e.devdec, HC_ESTATE, "overlap readback: decisions are on the device");
  HC_TRY(hc::flush_deferred(eng->e));  // pending landings first
  auto& e = eng->e;
  HC_REQUIRE(last >= first && last - first < hc::kRing, HC_EINVAL, "overlap window too long");
  cudaStream_t st = (cudaStream_t)stream;
  if (e.in_step) {  // inside an open step: read the finished rows beside its K4
    HC_REQUIRE(last < e.in_step && e.step_end, HC_ESTATE, "overlaps of the open step %d",
               e.in_step);
    st = e.side;
  }
  if (e.step_end) HC_CUDA_TRY(cudaStreamWaitEvent(st, e.step_end, 0));  // counts written
  if (!e.ovl_host)
    HC_CUDA_TRY(cudaHostAlloc((void**)&e.ovl_host, size_t(hc::kRing) * std::max(1, e.n_piv) * 4,
                              cudaHostAllocDefault));
  // the window is at most two contiguous runs of the ring: one or two async copies, one sync
  const int n = last - first + 1;
  const int r0 = first % hc::kRing;
  const int run1 = std::min(n, hc::kRing - r0);
  const size_t row = size_t(e.n_piv) * 4;
  HC_CUDA_TRY(cudaMemcpyAsync(e.ovl_host, e.ovl_ring + size_t(r0) * e.n_piv, row * run1,
                              cudaMemcpyDeviceToHost, st));
  if (run1 < n)
    HC_CUDA_TRY(cudaMemcpyAsync(e.ovl_host + size_t(run1) * e.n_piv, e.ovl_ring,
                                row * (n - run1), cudaMemcpyDeviceToHost, st));
  HC_CUDA_TRY(cudaStreamSynchronize(st));
  std::memcpy(out, e.ovl_host, row * n);
  return HC_OK;
}

extern "C" int hc_engine_fire(hc_engine* eng, int32_t pivot_unit, int32_t step,
                              int32_t completion_step, int32_t* transfer_ids, void* stream) {
  HC_REQUIRE(eng && transfer_ids, HC_EINVAL, "null argument");
  HC_REQUIRE(!eng->e.devdec, HC_ESTATE, "host fires: decisions are on the device");
  HC_TRY(hc::flush_deferred(eng->e));  // pending landings first
  return hc::engine_fire_batch(eng->e, 1, &pivot_unit, step, &completion_step, transfer_ids,
                               nullptr, (cudaStream_t)stream);
}

extern "C" int hc_engine_fire_batch(hc_engine* eng, int32_t n, const int32_t* pivot_units,
                                    int32_t step, const int32_t* completion_steps,
                                    int32_t* transfer_ids, uint32_t* fetched_host, void* stream) {
  HC_REQUIRE(eng && (n == 0 || (pivot_units && completion_steps && transfer_ids)), HC_EINVAL,
             "null argument");
  HC_REQUIRE(!eng->e.devdec, HC_ESTATE, "host fires: decisions are on the device");
  HC_TRY(hc::flush_deferred(eng->e));  // pending landings first
  return hc::engine_fire_batch(eng->e, n, pivot_units, step, completion_steps, transfer_ids,
                               fetched_host, (cudaStream_t)stream);
}

extern "C" int hc_engine_wait_fetched(hc_engine* eng) {
  HC_REQUIRE(eng, HC_EINVAL, "null argument");
  // only the side stream's selection and fetched-set copies, not the caller's queue
  if (eng->e.last_selected) HC_CUDA_TRY(cudaEventSynchronize(eng->e.last_selected));
  return HC_OK;
}

extern "C" int hc_engine_land(hc_engine* eng, int32_t transfer_id, void* stream) {
  HC_REQUIRE(eng, HC_EINVAL, "null argument");
  HC_REQUIRE(!eng->e.devdec, HC_ESTATE, "host landings: decisions are on the device");
  return hc::engine_land_batch(eng->e, 1, &transfer_id, (cudaStream_t)stream);
}

extern "C" int hc_engine_land_batch(hc_engine* eng, int32_t n, const int32_t* transfer_ids,
                                    void* stream) {
  HC_REQUIRE(eng && (n == 0 || transfer_ids), HC_EINVAL, "null argument");
  HC_REQUIRE(!eng->e.devdec || n == 0, HC_ESTATE, "host landings: decisions are on the device");
  return hc::engine_land_batch(eng->e, n, transfer_ids, (cudaStream_t)stream);
}

extern "C" int hc_engine_read_indices(hc_engine* eng, int32_t kind, int32_t id, uint32_t* out,
                                      int32_t capacity, int32_t* n_out, void* stream) {
  HC_REQUIRE(eng && out && n_out, HC_EINVAL, "null argument");
  HC_TRY(hc::flush_deferred(eng->e));  // pending landings first
  auto& e = eng->e;
  cudaStream_t st = (cudaStream_t)stream;
  const uint32_t* list = nullptr;
  const uint32_t* cnt = nullptr;
  const int32_t* meta = nullptr;
  if (kind == 0) {
    HC_REQUIRE(e.xfers.contains(id) && e.xfers[id].sel, HC_EINVAL, "bad transfer");
    list = e.xfers[id].sel;
    cnt = e.xfers[id].cnt;
  } else if (kind == 1 || kind == 3) {
    HC_REQUIRE(id >= 0 && id < e.n_units && e.units[id].kind == hc::kUnitComp, HC_EINVAL,
               "unit %d is not compressed", id);
    hc::DevSat ds{};
    int si = e.devdec ? e.dd_sat_of_unit[id] : -1;
    if (si >= 0) {  // device decisions: the satellite's landed transfer, if any
      HC_CUDA_TRY(cudaStreamSynchronize(st));
      HC_CUDA_TRY(cudaMemcpy(&ds, e.dd.sats + si, sizeof(ds), cudaMemcpyDeviceToHost));
      if (ds.cur_slot < 0) si = -1;
    }
    if (si >= 0) {
      hc::DevXfer* x = e.dd.xfers + size_t(si) * e.dd.nq + ds.cur_slot;
      if (kind == 1) {
        list = ds.sel + size_t(ds.cur_slot) * ds.k;
        cnt = &x->cnt;
      } else {
        list = ds.pos + size_t(ds.active) * ds.cap;
        meta = x->meta;
      }
    } else if (kind == 1) {
      list = hc::dyn_list(e, id, &cnt);
    } else {
      const int ow = e.dyn_owner[id];
      list = ow >= 0 ? e.xfers[ow].pos : e.pre_pos[id];
      meta = ow >= 0 ? e.xfers[ow].meta : e.pre_meta[id];
    }
  } else if (kind == 2) {
    HC_REQUIRE(id >= 0 && id < e.n_units && e.piv_slot[id] >= 0, HC_EINVAL, "not a pivot");
    const int s = e.piv_slot[id];
    list = e.top_idx + size_t(s) * e.lbase;
    cnt = e.top_cnt + s;
    if (e.step_end) HC_CUDA_TRY(cudaStreamWaitEvent(st, e.step_end, 0));  // rows on `mon`
    if (e.last_t > 0) {  // the monitor keeps only a threshold: materialise the set
      hc_topk_job jb{};
      jb.scores = e.rowbuf + size_t(s) * e.row_len;
      jb.n = uint32_t(e.L + e.last_t);
      jb.k = uint32_t(e.lbase);
      jb.out_idx = e.top_idx + size_t(s) * e.lbase;
      jb.out_count = e.top_cnt + s;
      hc_topk_job* dj = nullptr;
      HC_TRY(hc::upload(e, &jb, sizeof(jb), st, (void**)&dj));
      HC_TRY(hc::launch_topk(dj, 1, 0, st));
      HC_CUDA_TRY(cudaFreeAsync(dj, st));
    }
  } else {
    HC_REQUIRE(false, HC_EINVAL, "bad kind %d", kind);
  }
  int32_t n = 0;
  if (meta) HC_CUDA_TRY(cudaMemcpyAsync(&n, meta, 4, cudaMemcpyDeviceToHost, st));
  else HC_CUDA_TRY(cudaMemcpyAsync(&n, cnt, 4, cudaMemcpyDeviceToHost, st));
  HC_CUDA_TRY(cudaStreamSynchronize(st));
  *n_out = n;
  HC_REQUIRE(n <= capacity, HC_EINVAL, "capacity %d < %d", capacity, n);
  if (n) HC_CUDA_TRY(cudaMemcpyAsync(out, list, size_t(n) * 4, cudaMemcpyDeviceToHost, st));
  HC_CUDA_TRY(cudaStreamSynchronize(st));
  return HC_OK;
}

extern "C" int hc_engine_pivot_row(hc_engine* eng, int32_t pivot_unit, int32_t step, float* dst,
                                   void* stream) {
  HC_REQUIRE(eng && dst, HC_EINVAL, "null argument");
  HC_TRY(hc::flush_deferred(eng->e));  // pending landings first
  auto& e = eng->e;
  HC_REQUIRE(pivot_unit >= 0 && pivot_unit < e.n_units && e.piv_slot[pivot_unit] >= 0,
             HC_EINVAL, "not a monitored pivot");
  // the rows are written on the monitor stream
  if (e.step_end) HC_CUDA_TRY(cudaStreamWaitEvent((cudaStream_t)stream, e.step_end, 0));
  HC_CUDA_TRY(cudaMemcpyAsync(dst, e.rowbuf + size_t(e.piv_slot[pivot_unit]) * e.row_len,
                              size_t(e.L + step) * 4, cudaMemcpyDeviceToDevice,
                              (cudaStream_t)stream));
  return HC_OK;
}

extern "C" int hc_engine_resident_rows(hc_engine* eng, int32_t step, int64_t* rows_out,
                                       void* stream) {
  HC_REQUIRE(eng && rows_out, HC_EINVAL, "null argument");
  HC_TRY(hc::flush_deferred(eng->e));  // pending landings first
  auto& e = eng->e;
  std::vector<hc::UnitDesc> u(e.n_units);
  cudaStream_t st = (cudaStream_t)stream;
  HC_CUDA_TRY(cudaMemcpyAsync(u.data(), e.d_units, u.size() * sizeof(hc::UnitDesc),
                              cudaMemcpyDeviceToHost, st));
  HC_CUDA_TRY(cudaStreamSynchronize(st));
  int64_t total = 0;
  for (const auto& d : u) {
    if (d.kind == hc::kUnitFull) total += int64_t(e.L) + step;
    else if (d.kind == hc::kUnitAbsent) continue;
    else total += int64_t(d.n_prefix) - hc::tail_lo(d.tail_mask, step, e.R) + step;
  }
  *rows_out = total;
  return HC_OK;
}

extern "C" int hc_engine_active_tiles(const hc_engine* eng, int32_t step, int32_t* n_tiles) {
  HC_REQUIRE(eng && n_tiles, HC_EINVAL, "null argument");
  *n_tiles = hc::active_tiles(eng->e, step);
  return HC_OK;
}

extern "C" int hc_engine_set_prefill_dump(hc_engine* eng, float* dst_dev) {
  HC_REQUIRE(eng, HC_EINVAL, "null argument");
  eng->e.prefill_dump = dst_dev;
  return HC_OK;
}

extern "C" int hc_engine_timing(hc_engine* eng, int32_t enable, double* phase_ms,
                                int32_t* steps) {
  HC_REQUIRE(eng, HC_EINVAL, "null argument");
  auto& e = eng->e;
  constexpr int P = hc::EngineImpl::kPhaseEvents;
  if (phase_ms && steps) {
    for (int k = 0; k <= P; ++k) phase_ms[k] = 0;
    for (size_t i = 0; i < e.tev_used; ++i) {
      const cudaEvent_t* ev = e.tev.data() + i * P;
      if (e.timing_light) {  // the attention phase only
        HC_CUDA_TRY(cudaEventSynchronize(ev[2]));
        float ms = 0;
        HC_CUDA_TRY(cudaEventElapsedTime(&ms, ev[1], ev[2]));
        phase_ms[1] += ms;
        continue;
      }
      HC_CUDA_TRY(cudaEventSynchronize(ev[P - 1]));
      HC_CUDA_TRY(cudaEventSynchronize(ev[5]));
      // append | attention | combine on the step's stream; score rows (ev3 ->
      // ev4) and the monitor (ev4 -> ev5) on the monitor stream beside the next
      // step; tail = the step stream after the combine (ev3 -> ev6)
      for (int k = 1; k < P; ++k) {
        float ms = 0;
        HC_CUDA_TRY(cudaEventElapsedTime(&ms, ev[k < 6 ? k - 1 : 3], ev[k]));
        phase_ms[k - 1] += ms;
      }
      float tot = 0;
      HC_CUDA_TRY(cudaEventElapsedTime(&tot, ev[0], ev[P - 1]));
      phase_ms[P - 1] += tot;
      if (i > 0) {  // idle (or landing-stall) gap between consecutive steps
        float gap = 0;
        HC_CUDA_TRY(cudaEventElapsedTime(&gap, ev[-1], ev[0]));
        phase_ms[P] += gap;
      }
    }
    *steps = int32_t(e.tev_used);
  }
  e.tev_used = 0;
  e.timing = enable != 0;
  e.timing_light = enable == 2;
  return HC_OK;
}

extern "C" int hc_engine_retrieval_stats(hc_engine* eng, double* out4) {
  HC_REQUIRE(eng && out4, HC_EINVAL, "null argument");
  auto& e = eng->e;
  double g = 0, w = 0;
  for (auto& pr : e.gather_ev) {
    HC_CUDA_TRY(cudaEventSynchronize(pr.second));
    float ms = 0;
    HC_CUDA_TRY(cudaEventElapsedTime(&ms, pr.first, pr.second));
    g += ms;
  }
  for (auto& pr : e.land_ev) {
    HC_CUDA_TRY(cudaEventSynchronize(pr.second));
    HC_CUDA_TRY(cudaEventSynchronize(pr.first));
    float ms = 0;
    HC_CUDA_TRY(cudaEventElapsedTime(&ms, pr.first, pr.second));
    w += ms > 0 ? ms : 0;  // device decisions: the pair may end in either order
  }
  out4[0] = double(e.gather_rows_issued) * 2 * hc::kHeadDim * 2;  // bytes (upper bound)
  out4[1] = g;                                                     // gather kernel ms
  out4[2] = w;                                                     // landing stall ms
  out4[3] = double(e.gather_ev.size());
  for (auto& pr : e.gather_ev) e.tpool.push_back(pr.first), e.tpool.push_back(pr.second);
  for (auto& pr : e.land_ev) e.tpool.push_back(pr.first), e.tpool.push_back(pr.second);
  e.gather_ev.clear();
  e.land_ev.clear();
  e.gather_rows_issued = 0;
  return HC_OK;
}

extern "C" int hc_engine_gaps(hc_engine* eng, float* out, int32_t cap, int32_t* n) {
  HC_REQUIRE(eng && out && n, HC_EINVAL, "null argument");
  auto& e = eng->e;
  constexpr int P = hc::EngineImpl::kPhaseEvents;
  int m = 0;
  for (size_t i = 1; !e.timing_light && i < e.tev_used && m < cap; ++i) {
    const cudaEvent_t* ev = e.tev.data() + i * P;
    HC_CUDA_TRY(cudaEventSynchronize(ev[P - 1]));
    float gap = 0;
    HC_CUDA_TRY(cudaEventElapsedTime(&gap, ev[-1], ev[0]));
    out[m++] = gap;
  }
  *n = m;
  return HC_OK;
}

extern "C" int hc_engine_prefill_stats(hc_engine* eng, double* out3) {
  HC_REQUIRE(eng && out3, HC_EINVAL, "null argument");
  auto& e = eng->e;
  out3[0] = e.pf_score_ms;
  out3[1] = e.pf_layers;
  out3[2] = e.W;
  return HC_OK;
}

extern "C" int hc_engine_poll_decisions(hc_engine* eng, int32_t wait, int32_t* step_out,
                                        hc_fire_record* fires, int32_t fire_capacity,
                                        int32_t* n_fires_out, uint32_t* fetched_out,
                                        int64_t fetched_capacity) {
  HC_REQUIRE(eng && step_out && n_fires_out, HC_EINVAL, "null argument");
  auto& e = eng->e;
  HC_REQUIRE(e.devdec, HC_ESTATE, "the engine takes its decisions on the host");
  *step_out = -1;
  *n_fires_out = 0;
  static const char* kWhy[] = {"", "a satellite's transfer ring overflowed (more than 8 pending)",
                               "the host did not consume the fetched-set ring",
                               "a due gather did not complete (landing wait timed out)",
                               "a cluster has more than 8 satellites"};
  auto fault = [&]() -> int {
    const int code = *reinterpret_cast<volatile int32_t*>(e.error_h);
    HC_REQUIRE(code == 0, HC_ESTATE, "device decisions: %s",
               kWhy[code > 0 && code < 5 ? code : 0]);
    return HC_OK;
  };
  HC_TRY(fault());
  if (e.n_read >= e.n_bound) return HC_OK;
  cudaEvent_t ev = e.ev_log[e.n_read % hc::kLogRing];
  if (wait) {
    HC_CUDA_TRY(cudaEventSynchronize(ev));
  } else {
    const cudaError_t q = cudaEventQuery(ev);
    if (q == cudaErrorNotReady) return HC_OK;
    HC_CUDA_TRY(q);
  }
  HC_TRY(fault());
  const volatile hc::BoundaryHdr* hp = e.hdr_h + (e.n_read % hc::kLogRing);
  const int n = hp->n_fires;
  const int64_t head_after = hp->head_after;
  const hc::FireLog* lg = e.log_h + size_t(e.n_read % hc::kLogRing) * std::max(1, e.n_piv);
  int64_t need = 0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < lg[i].n_sats && j < 8; ++j) need += lg[i].ks[j];
  if (n > fire_capacity || need > fetched_capacity) {
    *n_fires_out = n;
    HC_REQUIRE(false, HC_EINVAL, "poll_decisions: needs %d fire records and %lld fetched entries",
               n, (long long)need);
  }
  int64_t off = 0;
  for (int i = 0; i < n; ++i) {
    const hc::FireLog& f = lg[i];
    hc_fire_record& r = fires[i];
    r.trigger_step = f.trigger;
    r.pivot_unit = f.pivot_unit;
    r.completion_step = f.completion;
    r.n_satellites = f.n_sats;
    r.transfer_bytes = f.bytes;
    r.cumulative_bytes = f.cum_after;
    r.first_satellite = f.first_sat;
    int64_t cnt = 0;
    for (int j = 0; j < 8; ++j) {
      r.fetched_counts[j] = f.ks[j];
      cnt += f.ks[j];
    }
    r.fetched_offset = f.host_off < 0 ? -1 : int32_t(off);
    // it lands at max(completion, trigger + 1): a step's landing pass precedes its decision
    e.dd_pending_until = std::max(e.dd_pending_until, std::max(f.completion, f.trigger + 1));
    if (f.host_off >= 0 && cnt) {
      std::memcpy(fetched_out + off, e.fetched_h + f.host_off, size_t(cnt) * 4);
      if (e.timing)
        for (int j = 0; j < f.n_sats && j < 8; ++j)
          e.gather_rows_issued += f.ks[j] + std::min(e.S, e.L) + e.R;
    }
    off += cnt;
  }
  *reinterpret_cast<volatile int64_t*>(e.fetched_tail_h) = head_after;  // ring space released
  *step_out = hp->t;
  *n_fires_out = n;
  ++e.n_read;
  return HC_OK;
}

extern "C" int hc_engine_devdec_satellites(hc_engine* eng, int32_t* units_out, int32_t capacity,
                                           int32_t* n_out) {
  HC_REQUIRE(eng && n_out, HC_EINVAL, "null argument");
  auto& e = eng->e;
  *n_out = int32_t(e.dd_sat_units.size());
  HC_REQUIRE(int(e.dd_sat_units.size()) <= capacity || !units_out, HC_EINVAL, "capacity");
  if (units_out)
    std::memcpy(units_out, e.dd_sat_units.data(), e.dd_sat_units.size() * 4);
  return HC_OK;
}
