// Tensor-mode engine handle: the hierarchical KV store, the per-step decode
// pipeline (append -> K4 attention -> combine -> pivot score rows -> K1/K2
// drift monitor) and K3 retrieval from the pinned host pool.
//
// Mirrors the reference engine's lifecycle (engine.py:153-416):
//   hc_engine_create        CacheEngine.__init__ geometry / plan  (engine.py:156-214)
//   hc_engine_prefill_layer prefill_init                          (engine.py:263-274)
//   hc_engine_decode_step   decode_step steps 2-4                 (engine.py:301-311)
//   hc_engine_fire          fetch loop + K_base restamp           (engine.py:322-357)
//   hc_engine_land          landing of a due transfer             (engine.py:293-299)
// The window median / completion-step arithmetic stays in the Python mirror
// (decoder.py), exactly as the reference writes it.

#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <deque>
#include <new>
#include <vector>

#include "hc_common.cuh"
#include "kv_layout.cuh"

namespace hc {

int make_kv_tensor_map(CUtensorMap* map, const void* base, int64_t rows);
int launch_attention(const CUtensorMap& tmK, const CUtensorMap& tmV, const AttnParams& p,
                     int n_tiles, const int32_t* pivot_units_dev, int n_pivots, cudaStream_t st);
int launch_topk(const hc_topk_job* jobs_dev, int n_jobs, uint32_t n_add, cudaStream_t st);

namespace {

constexpr int kRing = 64;  // overlap-count ring (steps), read back at window boundaries

// ---- kernels: append, position lists, row gathers -------------------------

// Append the decode token of step t (position L+t-1) to every unit.
__global__ void append_kernel(const UnitDesc* __restrict__ units, int n_units, int L, int t,
                              const uint4* __restrict__ k_new, const uint4* __restrict__ v_new,
                              uint4* __restrict__ K, uint4* __restrict__ V) {
  const int u = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (u >= n_units) return;
  const UnitDesc d = units[u];
  const int64_t row = d.kind == kUnitFull ? d.row0 + L + t - 1 : d.app_row + t - 1;
  // 256 B per row = 16 x uint4; lanes 0-15 move K, 16-31 move V
  if (lane < 16) K[row * 16 + lane] = k_new[size_t(u) * 16 + lane];
  else V[row * 16 + lane - 16] = v_new[size_t(u) * 16 + lane - 16];
}

// Prefix position list of a compressed unit, valid from step t_c:
//   [tail-only positions asc][sinks U (sel & [S, L)) asc]
// `sel` is a K1 dense selection (ascending).  meta = {n_prefix, tail_mask,
// #selected positions >= L (those are served by the append segment)}.
__global__ void build_positions_kernel(const uint32_t* __restrict__ sel,
                                       const uint32_t* __restrict__ sel_count, int L, int S,
                                       int R, int t_c, uint32_t* __restrict__ pos_out,
                                       int32_t* __restrict__ meta) {
  __shared__ int s_lo, s_hi, s_ntail;
  __shared__ uint32_t s_mask;
  const int k = int(*sel_count);
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
      int x = lo, y = hi;
      while (x < y) { const int m = (x + y) >> 1; if (int(sel[m]) < p) x = m + 1; else y = m; }
      if (!(x < hi && int(sel[x]) == p)) {
        pos_out[nt++] = uint32_t(p);
        mask |= 1u << (p - (L - R));
      }
    }
    s_lo = lo;
    s_hi = hi;
    s_ntail = nt;
    s_mask = mask;
  }
  __syncthreads();
  const int nt = s_ntail, lo = s_lo, hi = s_hi;
  for (int i = threadIdx.x; i < sinks; i += blockDim.x) pos_out[nt + i] = uint32_t(i);
  for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) pos_out[nt + sinks + (i - lo)] = sel[i];
  if (threadIdx.x == 0) {
    meta[0] = nt + sinks + (hi - lo);
    meta[1] = int32_t(s_mask);
    meta[2] = k - hi;
  }
}

// Copy rows pos[j] of a [positions x 128] K/V source (device memory or
// mapped pinned host memory: zero-copy over the host link) into arena rows
// dst_row + j.  One warp moves one 512 B row pair per iteration, 4 in flight.
__global__ void gather_rows_kernel(const uint4* __restrict__ srcK, const uint4* __restrict__ srcV,
                                   const uint32_t* __restrict__ pos,
                                   const int32_t* __restrict__ meta, int64_t dst_row,
                                   uint4* __restrict__ K, uint4* __restrict__ V) {
  const int n = meta[0];
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x >> 5);
  constexpr int kUnroll = 4;
  for (int j0 = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * kUnroll; j0 < n;
       j0 += warps * kUnroll) {
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

__global__ void set_prefix_kernel(UnitDesc* units, int u, int64_t row0, const int32_t* meta) {
  units[u].row0 = row0;
  units[u].n_prefix = meta[0];
  units[u].tail_mask = uint32_t(meta[1]);
  units[u].pad_ = meta[2];
}

__global__ void iota_kernel(int32_t* p, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = i;
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
  bool gathered = false;
  bool landed = false;
  cudaEvent_t selected = nullptr;  // on the caller's stream after selection
  cudaEvent_t done = nullptr;      // on the retrieval stream after the gather
};

#define HC_TRY(x)                    \
  do {                               \
    int _rc = (x);                   \
    if (_rc != HC_OK) return _rc;    \
  } while (0)

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

struct EngineImpl {
  hc_engine_desc cfg{};
  int B = 0, NL = 0, H = 0, G = 0, Hq = 0, L = 0, T = 0, S = 0, R = 0, CH = 0, lbase = 0;
  int n_units = 0;
  int64_t dev_bytes = 0, host_bytes = 0;
  std::vector<int32_t> role, length, cpivot;
  std::vector<UnitDesc> units;
  UnitDesc* d_units = nullptr;
  int64_t rows = 0;
  __nv_bfloat16 *K = nullptr, *V = nullptr;
  CUtensorMap tmK{}, tmV{};
  std::vector<uint32_t> t_act;  // sorted activation steps of the tile table
  TileDesc* d_tiles = nullptr;
  int n_slots = 0;
  float* partial = nullptr;
  // pivots
  std::vector<int32_t> piv_units, piv_slot;  // piv_slot: unit -> slot or -1
  int32_t* d_piv_units = nullptr;
  int n_piv = 0;
  int64_t row_len = 0;
  int words = 0;
  float *logits = nullptr, *stats = nullptr, *rowbuf = nullptr;
  uint32_t *top_idx = nullptr, *top_cnt = nullptr, *kbase = nullptr;
  uint32_t *ovl_cur = nullptr, *ovl_ring = nullptr;
  hc_topk_job* d_piv_jobs = nullptr;
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
  std::vector<Transfer> xfers;
  cudaStream_t retr = nullptr;
  // prefill scratch
  float* prefill_dump = nullptr;
  char* pf = nullptr;
  size_t pf_bytes = 0;

  int lh(int u) const { return u % (NL * H); }
  int head(int u) const { return u % H; }
};

}  // namespace hc

struct hc_engine {
  hc::EngineImpl e;
};

namespace hc {
namespace {

int engine_destroy(EngineImpl& e) {
  cudaDeviceSynchronize();
  for (auto& x : e.xfers) {
    if (x.selected) cudaEventDestroy(x.selected);
    if (x.done) cudaEventDestroy(x.done);
    if (x.sel) cudaFree(x.sel);
    if (x.cnt) cudaFree(x.cnt);
    if (x.pos) cudaFree(x.pos);
    if (x.meta) cudaFree(x.meta);
  }
  for (size_t u = 0; u < e.dyn_sel.size(); ++u) {
    if (e.dyn_sel[u]) cudaFree(e.dyn_sel[u]);
    if (e.dyn_cnt[u]) cudaFree(e.dyn_cnt[u]);
    if (e.pre_pos[u]) cudaFree(e.pre_pos[u]);
    if (e.pre_meta[u]) cudaFree(e.pre_meta[u]);
  }
  void* ptrs[] = {e.d_units, e.K, e.V, e.d_tiles, e.partial, e.d_piv_units, e.logits, e.stats,
                  e.rowbuf, e.top_idx, e.top_cnt, e.kbase, e.ovl_cur, e.ovl_ring, e.d_piv_jobs,
                  e.pf};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (e.pool) {
    if (e.pool_host) cudaFreeHost(e.pool);
    else cudaFree(e.pool);
  }
  if (e.retr) cudaStreamDestroy(e.retr);
  return HC_OK;
}

int engine_create(EngineImpl& e, const hc_engine_desc& c, const int32_t* roles,
                  const int32_t* lengths, const int32_t* cpiv) {
  HC_REQUIRE(c.head_dim == kHeadDim, HC_EINVAL, "head_dim must be 128");
  HC_REQUIRE(c.group >= 1 && c.group <= 8, HC_EINVAL, "group must be 1..8");
  HC_REQUIRE(c.batch >= 1 && c.num_layers >= 1 && c.kv_heads >= 1, HC_EINVAL, "bad geometry");
  HC_REQUIRE(c.prefill_len >= 1 && c.max_decode >= 1, HC_EINVAL, "bad lengths");
  HC_REQUIRE(c.recency_window >= 0 && c.recency_window <= 32, HC_EINVAL,
             "recency_window must be in [0, 32]");
  HC_REQUIRE(c.sink_count >= 0, HC_EINVAL, "sink_count must be >= 0");
  HC_REQUIRE(c.l_base_int >= 1, HC_EINFEASIBLE, "l_base_int must be >= 1");
  e.cfg = c;
  e.B = c.batch, e.NL = c.num_layers, e.H = c.kv_heads, e.G = c.group, e.Hq = c.kv_heads * c.group;
  e.L = c.prefill_len, e.T = c.max_decode, e.S = c.sink_count, e.R = c.recency_window;
  e.CH = c.chunk > 0 ? c.chunk : 1024;
  HC_REQUIRE(e.CH % 64 == 0, HC_EINVAL, "chunk must be a multiple of 64");
  e.lbase = c.l_base_int;
  e.pool_host = c.host_pool != 0;
  const int LH = e.NL * e.H;
  e.role.assign(roles, roles + LH);
  e.length.assign(lengths, lengths + LH);
  e.cpivot.assign(cpiv, cpiv + LH);
  for (int i = 0; i < LH; ++i) {
    HC_REQUIRE(e.role[i] >= 0 && e.role[i] <= 3, HC_EINVAL, "bad role at %d", i);
    const bool comp = e.role[i] == HC_ROLE_ANCHOR || e.role[i] == HC_ROLE_SATELLITE;
    if (comp) HC_REQUIRE(e.length[i] >= 0 && e.length[i] <= e.L, HC_EINVAL, "bad length at %d", i);
    if (e.role[i] == HC_ROLE_SATELLITE) {
      const int p = e.cpivot[i];
      HC_REQUIRE(p >= 0 && p < e.H && e.role[(i / e.H) * e.H + p] == HC_ROLE_PIVOT, HC_EINVAL,
                 "satellite %d has no pivot in its layer", i);
    }
  }
  e.n_units = e.B * LH;
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
  e.row_len = int64_t(e.L) + e.T;
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
    if (full) {
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
  HC_TRY(dalloc((void**)&e.logits, size_t(np) * e.G * e.row_len * 4, &e.dev_bytes));
  HC_TRY(dalloc((void**)&e.stats, size_t(np) * e.G * 2 * 4, &e.dev_bytes));
  HC_TRY(dalloc((void**)&e.rowbuf, size_t(np) * e.row_len * 4, &e.dev_bytes));
  HC_TRY(dalloc((void**)&e.top_idx, size_t(np) * e.lbase * 4, &e.dev_bytes));
  HC_TRY(dalloc((void**)&e.top_cnt, size_t(np) * 4, &e.dev_bytes));
  HC_TRY(dalloc((void**)&e.kbase, size_t(np) * e.words * 4, &e.dev_bytes));
  HC_TRY(dalloc((void**)&e.ovl_cur, size_t(np) * 4, &e.dev_bytes));
  HC_TRY(dalloc((void**)&e.ovl_ring, size_t(np) * kRing * 4, &e.dev_bytes));
  std::vector<hc_topk_job> jobs(np);
  for (int s = 0; s < e.n_piv; ++s) {
    hc_topk_job& j = jobs[s];
    j.scores = e.rowbuf + size_t(s) * e.row_len;
    j.idx = nullptr;
    j.n = uint32_t(e.L);  // + step (n_add)
    j.k = uint32_t(e.lbase);
    j.out_idx = e.top_idx + size_t(s) * e.lbase;
    j.out_count = e.top_cnt + s;
    j.base_bitmap = e.kbase + size_t(s) * e.words;
    j.overlap_out = e.ovl_cur + s;
  }
  HC_TRY(dalloc((void**)&e.d_piv_jobs, size_t(np) * sizeof(hc_topk_job), &e.dev_bytes));
  HC_CUDA_TRY(cudaMemcpy(e.d_piv_jobs, jobs.data(), size_t(np) * sizeof(hc_topk_job),
                         cudaMemcpyHostToDevice));

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
  int lo_prio = 0, hi_prio = 0;
  HC_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
  HC_CUDA_TRY(cudaStreamCreateWithPriority(&e.retr, cudaStreamNonBlocking, hi_prio));
  return HC_OK;
}

AttnParams decode_params(EngineImpl& e, int t, const void* q, void* o) {
  AttnParams p{};
  p.units = e.d_units;
  p.tiles = e.d_tiles;
  p.q = q;
  p.out = o;
  p.partial = e.partial;
  p.logits = e.logits;
  p.stats = e.stats;
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

// Position list + gather of a compressed unit's prefix buffer `buf_row`.
int build_prefix(EngineImpl& e, int u, const uint32_t* sel, const uint32_t* cnt, int t_c,
                 uint32_t* pos, int32_t* meta, const __nv_bfloat16* srcK,
                 const __nv_bfloat16* srcV, int64_t buf_row, cudaStream_t st) {
  build_positions_kernel<<<1, 256, 0, st>>>(sel, cnt, e.L, e.S, e.R, t_c, pos, meta);
  HC_CHECK_LAUNCH();
  const int blocks = std::max(1, std::min(64, (e.cap[u] + 31) / 32));
  gather_rows_kernel<<<blocks, 256, 0, st>>>(reinterpret_cast<const uint4*>(srcK),
                                             reinterpret_cast<const uint4*>(srcV), pos, meta,
                                             buf_row, reinterpret_cast<uint4*>(e.K),
                                             reinterpret_cast<uint4*>(e.V));
  HC_CHECK_LAUNCH();
  return HC_OK;
}

int engine_prefill_layer(EngineImpl& e, int layer, const __nv_bfloat16* k,
                         const __nv_bfloat16* v, const __nv_bfloat16* q, cudaStream_t st) {
  HC_REQUIRE(layer >= 0 && layer < e.NL, HC_EINVAL, "layer out of range");
  const int nu = e.B * e.H;  // units of this layer, i = b*H + h
  const int nch = (e.L + e.CH - 1) / e.CH;
  // scratch layout
  size_t off = 0;
  auto carve = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~size_t(255); return o; };
  const size_t o_units = carve(size_t(nu) * sizeof(UnitDesc));
  const size_t o_tiles = carve(size_t(nu) * nch * sizeof(TileDesc));
  const size_t o_part = carve(size_t(nu) * nch * e.G * kPartStride * 4);
  const size_t o_logit = carve(size_t(nu) * e.G * e.L * 4);
  const size_t o_stats = carve(size_t(nu) * e.G * 2 * 4);
  const size_t o_rows = carve(size_t(nu) * e.L * 4);
  const size_t o_iota = carve(size_t(nu) * 4);
  const size_t o_jobs = carve(size_t(nu) * sizeof(hc_topk_job));
  if (off > e.pf_bytes) {
    if (e.pf) {
      HC_CUDA_TRY(cudaStreamSynchronize(st));
      cudaFree(e.pf);
      e.pf = nullptr;
    }
    HC_TRY(dalloc((void**)&e.pf, off, nullptr));
    e.pf_bytes = off;
  }
  char* pf = e.pf;
  std::vector<UnitDesc> ud(nu);
  std::vector<TileDesc> td;
  td.reserve(size_t(nu) * nch);
  for (int i = 0; i < nu; ++i) {
    const int b = i / e.H, h = i % e.H;
    UnitDesc& d = ud[i];
    d = UnitDesc{};
    d.kind = kUnitFull;
    d.row0 = int64_t(i) * e.L;
    d.app_row = d.row0 + e.L;
    d.n_prefix = e.L;
    d.q_row = b * e.Hq + h * e.G;
    d.pivot_slot = i;
    d.slot0 = i * nch;
    for (int ch = 0; ch < nch; ++ch)
      td.push_back(TileDesc{uint32_t(i), uint32_t(ch), uint32_t(i * nch + ch), 0u});
  }
  // the prefill descriptors must stay valid until the kernels ran: copy on stream
  HC_CUDA_TRY(cudaMemcpyAsync(pf + o_units, ud.data(), ud.size() * sizeof(UnitDesc),
                              cudaMemcpyHostToDevice, st));
  HC_CUDA_TRY(cudaMemcpyAsync(pf + o_tiles, td.data(), td.size() * sizeof(TileDesc),
                              cudaMemcpyHostToDevice, st));
  iota_kernel<<<(nu + 255) / 256, 256, 0, st>>>(reinterpret_cast<int32_t*>(pf + o_iota), nu);
  HC_CHECK_LAUNCH();
  CUtensorMap mk, mv;
  HC_TRY(make_kv_tensor_map(&mk, k, int64_t(nu) * e.L));
  HC_TRY(make_kv_tensor_map(&mv, v, int64_t(nu) * e.L));
  AttnParams p{};
  p.units = reinterpret_cast<UnitDesc*>(pf + o_units);
  p.tiles = reinterpret_cast<TileDesc*>(pf + o_tiles);
  p.q = q;
  p.out = nullptr;
  p.partial = reinterpret_cast<float*>(pf + o_part);
  p.logits = reinterpret_cast<float*>(pf + o_logit);
  p.stats = reinterpret_cast<float*>(pf + o_stats);
  p.rows = reinterpret_cast<float*>(pf + o_rows);
  p.logit_stride = e.L;
  p.row_stride = e.L;
  p.group = e.G;
  p.L = e.L;
  p.t = 0;
  p.chunk = e.CH;
  p.recency = e.R;
  p.n_units = nu;
  p.scale_log2 = float(1.4426950408889634 / 11.313708498984761);
  HC_TRY(launch_attention(mk, mv, p, int(td.size()),
                          reinterpret_cast<int32_t*>(pf + o_iota), nu, st));
  if (e.prefill_dump)  // test hook: step-0 rows [NL][B*H][L]
    HC_CUDA_TRY(cudaMemcpyAsync(e.prefill_dump + size_t(layer) * nu * e.L, p.rows,
                                size_t(nu) * e.L * 4, cudaMemcpyDeviceToDevice, st));

  // K1: compressed heads select l_h (prefill_init, engine.py:265-268), pivots
  // select l_base for K_base (engine.py:269-271).
  std::vector<hc_topk_job> jobs;
  std::vector<int> job_unit;
  for (int i = 0; i < nu; ++i) {
    const int b = i / e.H, h = i % e.H;
    const int u = (b * e.NL + layer) * e.H + h;
    const int r = e.role[layer * e.H + h];
    hc_topk_job j{};
    j.scores = p.rows + size_t(i) * e.L;
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
  for (int u : job_unit) {
    const int s = e.piv_slot[u];
    if (s < 0) continue;
    HC_REQUIRE(hc_bitmap_from_indices(e.kbase + size_t(s) * e.words, uint32_t(e.words),
                                      e.top_idx + size_t(s) * e.lbase, e.top_cnt + s,
                                      uint32_t(e.lbase), st) == HC_OK,
               HC_ECUDA, "K_base bitmap failed");
  }
  // caches: full heads whole, compressed heads gathered, satellites to the host pool
  const size_t rowb = size_t(kHeadDim) * 2;
  for (int i = 0; i < nu; ++i) {
    const int b = i / e.H, h = i % e.H;
    const int u = (b * e.NL + layer) * e.H + h;
    const __nv_bfloat16* sk = k + size_t(i) * e.L * kHeadDim;
    const __nv_bfloat16* sv = v + size_t(i) * e.L * kHeadDim;
    const UnitDesc& d = e.units[u];
    if (d.kind == kUnitFull) {
      HC_CUDA_TRY(cudaMemcpyAsync(e.K + size_t(d.row0) * kHeadDim, sk, rowb * e.L,
                                  cudaMemcpyDeviceToDevice, st));
      HC_CUDA_TRY(cudaMemcpyAsync(e.V + size_t(d.row0) * kHeadDim, sv, rowb * e.L,
                                  cudaMemcpyDeviceToDevice, st));
      continue;
    }
    HC_TRY(build_prefix(e, u, e.dyn_sel[u], e.dyn_cnt[u], 1, e.pre_pos[u], e.pre_meta[u], sk, sv,
                        e.buf_row0[u], st));
    set_prefix_kernel<<<1, 1, 0, st>>>(e.d_units, u, e.buf_row0[u], e.pre_meta[u]);
    HC_CHECK_LAUNCH();
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
  // prefill descriptors/jobs were uploaded from host vectors on `st`: make the
  // uploads complete before those vectors go out of scope.
  HC_CUDA_TRY(cudaStreamSynchronize(st));
  return HC_OK;
}

int engine_decode_step(EngineImpl& e, int t, const void* q, const void* kn, const void* vn,
                       void* o, cudaStream_t st) {
  HC_REQUIRE(t >= 1 && t <= e.T, HC_EINVAL, "step %d outside 1..%d", t, e.T);
  append_kernel<<<(e.n_units + 7) / 8, 256, 0, st>>>(
      e.d_units, e.n_units, e.L, t, reinterpret_cast<const uint4*>(kn),
      reinterpret_cast<const uint4*>(vn), reinterpret_cast<uint4*>(e.K),
      reinterpret_cast<uint4*>(e.V));
  HC_CHECK_LAUNCH();
  AttnParams p = decode_params(e, t, q, o);
  HC_TRY(launch_attention(e.tmK, e.tmV, p, active_tiles(e, t), e.d_piv_units, e.n_piv, st));
  if (e.n_piv) {
    HC_TRY(launch_topk(e.d_piv_jobs, e.n_piv, uint32_t(t), st));
    HC_CUDA_TRY(cudaMemcpyAsync(e.ovl_ring + size_t(t % kRing) * e.n_piv, e.ovl_cur,
                                size_t(e.n_piv) * 4, cudaMemcpyDeviceToDevice, st));
  }
  return HC_OK;
}

int issue_gather(EngineImpl& e, int id) {
  Transfer& x = e.xfers[id];
  const int u = x.unit;
  x.buf = 1 - e.active[u];
  const int64_t dst = x.buf ? e.buf_row1[u] : e.buf_row0[u];
  const int ss = e.sat_slot[u];
  const __nv_bfloat16* sk = e.pool + size_t(ss) * 2 * e.L * kHeadDim;
  const __nv_bfloat16* sv = sk + size_t(e.L) * kHeadDim;
  HC_CUDA_TRY(cudaStreamWaitEvent(e.retr, x.selected, 0));
  HC_TRY(build_prefix(e, u, x.sel, x.cnt, x.completion, x.pos, x.meta, sk, sv, dst, e.retr));
  HC_CUDA_TRY(cudaEventRecord(x.done, e.retr));
  x.gathered = true;
  return HC_OK;
}

int engine_fire(EngineImpl& e, int pu, int t, int completion, int32_t* ids, cudaStream_t st) {
  HC_REQUIRE(pu >= 0 && pu < e.n_units && e.piv_slot[pu] >= 0, HC_EINVAL, "unit %d is not a monitored pivot", pu);
  const int s = e.piv_slot[pu];
  const int LH = e.NL * e.H;
  const int b = pu / LH, i = e.lh(pu), l = i / e.H, ph = i % e.H;
  std::vector<hc_topk_job> jobs;
  std::vector<int> new_ids;
  for (int h = 0; h < e.H; ++h) {
    const int j = l * e.H + h;
    if (e.role[j] != HC_ROLE_SATELLITE || e.cpivot[j] != ph) continue;
    const int u = (b * e.NL + l) * e.H + h;
    Transfer x;
    x.unit = u;
    x.k = e.length[j];
    x.completion = completion;
    HC_CUDA_TRY(cudaMallocAsync((void**)&x.sel, size_t(std::max(1, x.k)) * 4, st));
    HC_CUDA_TRY(cudaMallocAsync((void**)&x.cnt, 4, st));
    HC_CUDA_TRY(cudaMallocAsync((void**)&x.pos, size_t(std::max(1, e.cap[u])) * 4, st));
    HC_CUDA_TRY(cudaMallocAsync((void**)&x.meta, 16, st));
    HC_CUDA_TRY(cudaEventCreateWithFlags(&x.selected, cudaEventDisableTiming));
    HC_CUDA_TRY(cudaEventCreateWithFlags(&x.done, cudaEventDisableTiming));
    hc_topk_job jb{};
    jb.scores = e.rowbuf + size_t(s) * e.row_len;
    jb.n = uint32_t(e.L + t);
    jb.k = uint32_t(x.k);
    jb.out_idx = x.sel;
    jb.out_count = x.cnt;
    jobs.push_back(jb);
    new_ids.push_back(int(e.xfers.size()));
    e.xfers.push_back(x);
  }
  if (!jobs.empty()) {
    hc_topk_job* dj = nullptr;
    HC_CUDA_TRY(cudaMallocAsync((void**)&dj, jobs.size() * sizeof(hc_topk_job), st));
    HC_CUDA_TRY(cudaMemcpyAsync(dj, jobs.data(), jobs.size() * sizeof(hc_topk_job),
                                cudaMemcpyHostToDevice, st));
    HC_TRY(launch_topk(dj, int(jobs.size()), 0, st));
    HC_CUDA_TRY(cudaFreeAsync(dj, st));
    HC_CUDA_TRY(cudaStreamSynchronize(st));  // host job vector is about to go away
  }
  // K_base <- current top set (engine.py:357)
  HC_REQUIRE(hc_bitmap_from_indices(e.kbase + size_t(s) * e.words, uint32_t(e.words),
                                    e.top_idx + size_t(s) * e.lbase, e.top_cnt + s,
                                    uint32_t(e.lbase), st) == HC_OK,
             HC_ECUDA, "K_base restamp failed");
  for (size_t n = 0; n < new_ids.size(); ++n) {
    Transfer& x = e.xfers[new_ids[n]];
    HC_CUDA_TRY(cudaEventRecord(x.selected, st));
    e.fifo[x.unit].push_back(new_ids[n]);
    if (e.fifo[x.unit].size() == 1) HC_TRY(issue_gather(e, new_ids[n]));
    ids[n] = new_ids[n];
  }
  return HC_OK;
}

int engine_land(EngineImpl& e, int id, cudaStream_t st) {
  HC_REQUIRE(id >= 0 && id < int(e.xfers.size()), HC_EINVAL, "bad transfer id");
  Transfer& x = e.xfers[id];
  HC_REQUIRE(!x.landed, HC_ESTATE, "transfer %d already landed", id);
  const int u = x.unit;
  HC_REQUIRE(!e.fifo[u].empty() && e.fifo[u].front() == id, HC_ESTATE,
             "transfer %d lands out of order", id);
  if (!x.gathered) HC_TRY(issue_gather(e, id));
  HC_CUDA_TRY(cudaStreamWaitEvent(st, x.done, 0));
  const int64_t row0 = x.buf ? e.buf_row1[u] : e.buf_row0[u];
  set_prefix_kernel<<<1, 1, 0, st>>>(e.d_units, u, row0, x.meta);
  HC_CHECK_LAUNCH();
  e.active[u] = x.buf;
  // the transfer's buffers become the unit's dynamic-set / prefix records
  if (e.dyn_owner[u] >= 0) {
    Transfer& old = e.xfers[e.dyn_owner[u]];
    HC_CUDA_TRY(cudaFreeAsync(old.sel, st));
    HC_CUDA_TRY(cudaFreeAsync(old.cnt, st));
    HC_CUDA_TRY(cudaFreeAsync(old.pos, st));
    HC_CUDA_TRY(cudaFreeAsync(old.meta, st));
    old.sel = nullptr;
    old.cnt = nullptr;
    old.pos = nullptr;
    old.meta = nullptr;
  }
  e.dyn_owner[u] = id;
  x.landed = true;
  e.fifo[u].pop_front();
  if (!e.fifo[u].empty()) {
    // the next queued gather may only overwrite the old buffer once this
    // stream no longer reads it: order it after the landing point
    cudaEvent_t ev;
    HC_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    HC_CUDA_TRY(cudaEventRecord(ev, st));
    HC_CUDA_TRY(cudaStreamWaitEvent(e.retr, ev, 0));
    HC_CUDA_TRY(cudaEventDestroy(ev));
    HC_TRY(issue_gather(e, e.fifo[u].front()));
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

}  // namespace
}  // namespace hc

// ============================== C ABI ======================================

extern "C" int hc_engine_create(const hc_engine_desc* desc, const int32_t* roles,
                                const int32_t* lengths, const int32_t* cluster_pivot,
                                hc_engine** out) {
  HC_REQUIRE(desc && roles && lengths && cluster_pivot && out, HC_EINVAL,
             "hc_engine_create: null argument");
  *out = nullptr;
  hc_engine* h = new (std::nothrow) hc_engine();
  HC_REQUIRE(h, HC_ENOMEM, "out of host memory");
  const int rc = hc::engine_create(h->e, *desc, roles, lengths, cluster_pivot);
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

extern "C" int hc_engine_overlaps(hc_engine* eng, int32_t first, int32_t last, int32_t* out,
                                  void* stream) {
  HC_REQUIRE(eng && out, HC_EINVAL, "null argument");
  auto& e = eng->e;
  HC_REQUIRE(last >= first && last - first < hc::kRing, HC_EINVAL, "overlap window too long");
  cudaStream_t st = (cudaStream_t)stream;
  for (int t = first; t <= last; ++t)
    HC_CUDA_TRY(cudaMemcpyAsync(out + size_t(t - first) * e.n_piv,
                                e.ovl_ring + size_t(t % hc::kRing) * e.n_piv,
                                size_t(e.n_piv) * 4, cudaMemcpyDeviceToHost, st));
  HC_CUDA_TRY(cudaStreamSynchronize(st));
  return HC_OK;
}

extern "C" int hc_engine_fire(hc_engine* eng, int32_t pivot_unit, int32_t step,
                              int32_t completion_step, int32_t* transfer_ids, void* stream) {
  HC_REQUIRE(eng && transfer_ids, HC_EINVAL, "null argument");
  return hc::engine_fire(eng->e, pivot_unit, step, completion_step, transfer_ids,
                         (cudaStream_t)stream);
}

extern "C" int hc_engine_land(hc_engine* eng, int32_t transfer_id, void* stream) {
  HC_REQUIRE(eng, HC_EINVAL, "null argument");
  return hc::engine_land(eng->e, transfer_id, (cudaStream_t)stream);
}

extern "C" int hc_engine_read_indices(hc_engine* eng, int32_t kind, int32_t id, uint32_t* out,
                                      int32_t capacity, int32_t* n_out, void* stream) {
  HC_REQUIRE(eng && out && n_out, HC_EINVAL, "null argument");
  auto& e = eng->e;
  cudaStream_t st = (cudaStream_t)stream;
  const uint32_t* list = nullptr;
  const uint32_t* cnt = nullptr;
  const int32_t* meta = nullptr;
  if (kind == 0) {
    HC_REQUIRE(id >= 0 && id < int(e.xfers.size()) && e.xfers[id].sel, HC_EINVAL, "bad transfer");
    list = e.xfers[id].sel;
    cnt = e.xfers[id].cnt;
  } else if (kind == 1 || kind == 3) {
    HC_REQUIRE(id >= 0 && id < e.n_units && e.units[id].kind == hc::kUnitComp, HC_EINVAL,
               "unit %d is not compressed", id);
    if (kind == 1) {
      list = hc::dyn_list(e, id, &cnt);
    } else {
      const int ow = e.dyn_owner[id];
      list = ow >= 0 ? e.xfers[ow].pos : e.pre_pos[id];
      meta = ow >= 0 ? e.xfers[ow].meta : e.pre_meta[id];
    }
  } else if (kind == 2) {
    HC_REQUIRE(id >= 0 && id < e.n_units && e.piv_slot[id] >= 0, HC_EINVAL, "not a pivot");
    list = e.top_idx + size_t(e.piv_slot[id]) * e.lbase;
    cnt = e.top_cnt + e.piv_slot[id];
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
  auto& e = eng->e;
  HC_REQUIRE(pivot_unit >= 0 && pivot_unit < e.n_units && e.piv_slot[pivot_unit] >= 0,
             HC_EINVAL, "not a monitored pivot");
  HC_CUDA_TRY(cudaMemcpyAsync(dst, e.rowbuf + size_t(e.piv_slot[pivot_unit]) * e.row_len,
                              size_t(e.L + step) * 4, cudaMemcpyDeviceToDevice,
                              (cudaStream_t)stream));
  return HC_OK;
}

extern "C" int hc_engine_resident_rows(hc_engine* eng, int32_t step, int64_t* rows_out,
                                       void* stream) {
  HC_REQUIRE(eng && rows_out, HC_EINVAL, "null argument");
  auto& e = eng->e;
  std::vector<hc::UnitDesc> u(e.n_units);
  cudaStream_t st = (cudaStream_t)stream;
  HC_CUDA_TRY(cudaMemcpyAsync(u.data(), e.d_units, u.size() * sizeof(hc::UnitDesc),
                              cudaMemcpyDeviceToHost, st));
  HC_CUDA_TRY(cudaStreamSynchronize(st));
  int64_t total = 0;
  for (const auto& d : u) {
    if (d.kind == hc::kUnitFull) total += int64_t(e.L) + step;
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
