// Device-side layout of the hierarchical KV store (tensor mode).
//
// One K arena and one V arena, each a row-major [rows x 128] bf16 matrix
// (one row = one token of one KV head, 256 B), addressed by TMA as a single
// 2-D tensor.  Every (batch, layer, kv_head) "unit" owns row ranges:
//
//   full unit (volatile / pivot, keeps the whole context):
//       row0 + p holds position p, p in [0, L + T_max)
//   compressed unit (anchor / satellite, engine.py:98-115 CacheView):
//       prefix buffer  [tail-only rows asc][base rows asc]  at row0
//           base  = sinks U (dynamic & [0, L))        (sorted positions)
//           tail  = recency positions in [L-R, L) not in base; row j of the
//                   tail block is resident at step t iff its position is
//                   >= L + t - R, i.e. a suffix of the block (lo(t) below)
//       append region (decode positions L..L+T_max-1) at app_row
//     satellites own two prefix buffers (active + staging for retrieval).
//
// Attention work is cut into fixed-size chunks ("tiles") of at most
// `chunk` rows that never cross a segment; the tile table is static and
// sorted by the first decode step at which each tile is non-empty, so a
// step launches exactly the tiles it needs (no empty CTAs).
#pragma once

#include <stdint.h>

namespace hc {

constexpr int kHeadDim = 128;

// kUnitAbsent: a (sequence, layer, head) another rank owns (sharded engines,
// hc_engine_create_sharded): no rows, no tiles, no output.
enum UnitKind : int32_t { kUnitFull = 0, kUnitComp = 1, kUnitAbsent = 2 };

struct UnitDesc {
  int64_t row0;        // full: row of position 0; comp: active prefix buffer
  int64_t app_row;     // comp: row of decode position L; full: row0 + L
  int32_t kind;        // UnitKind
  int32_t n_prefix;    // comp: rows in the active prefix buffer; full: L
  uint32_t tail_mask;  // comp: bit i set <=> position L-R+i is a tail-only row (R <= 32),
                       // or the tail-only row count (R > 32, see tail_lo)
  int32_t q_row;       // first query row (of G) for this unit
  int32_t pivot_slot;  // >= 0: emit logits / score row into this slot
  int32_t slot0;       // first split-K partial slot
  int32_t n_pchunks;   // comp: static prefix-chunk count; full: unused
  int32_t pad_;
};
static_assert(sizeof(UnitDesc) == 48, "UnitDesc layout");

struct TileDesc {
  uint32_t unit;
  uint32_t seg_chunk;  // bit 31: append segment of a compressed unit; low bits: chunk
  uint32_t slot;       // split-K partial slot
  uint32_t t_act;      // first decode step at which this tile holds rows
};
static_assert(sizeof(TileDesc) == 16, "TileDesc layout");

// Row range of a tile at decode step t:  rows [row, row + n), and the
// position of its first row (valid for full units only, -1 otherwise).
struct TileRange {
  int64_t row;
  int32_t n;
  int32_t pos;
};

__host__ __device__ inline int popc32(uint32_t x) {
#ifdef __CUDA_ARCH__
  return __popc(x);
#else
  return __builtin_popcount(x);
#endif
}

// lo(t): tail-only prefix rows that left the recency window by step t.
// recency <= 32: bit i of tail_mask <=> position L-R+i is a tail-only row.
// recency > 32 (heads without a dynamic set): tail_mask = n, the tail-only
// rows are the contiguous positions [L-n, L), of which those below L+t-R left.
__host__ __device__ inline int32_t tail_lo(uint32_t tail_mask, int32_t t, int32_t recency) {
  if (recency > 32) {
    const int32_t n = int32_t(tail_mask);
    const int32_t v = n + t - recency;
    return v < 0 ? 0 : (v > n ? n : v);
  }
  const int32_t w = t < recency ? t : recency;
  const uint32_t m = w >= 32 ? 0xffffffffu : ((1u << w) - 1u);
  return popc32(tail_mask & m);
}

__host__ __device__ inline TileRange tile_range(const UnitDesc& u, uint32_t seg_chunk, int32_t t,
                                                int32_t L, int32_t recency, int32_t chunk) {
  TileRange r;
  const int32_t c = int32_t(seg_chunk & 0x7fffffffu);
  const bool app = (seg_chunk >> 31) != 0;
  int32_t lo = c * chunk, hi = lo + chunk;
  if (u.kind == kUnitFull) {
    const int32_t len = L + t;
    hi = hi < len ? hi : len;
    r.row = u.row0 + lo;
    r.pos = lo;
  } else if (!app) {
    const int32_t first = tail_lo(u.tail_mask, t, recency);
    lo = lo > first ? lo : first;
    hi = hi < u.n_prefix ? hi : u.n_prefix;
    r.row = u.row0 + lo;
    r.pos = -1;
  } else {
    hi = hi < t ? hi : t;
    r.row = u.app_row + lo;
    r.pos = -1;
  }
  r.n = hi > lo ? hi - lo : 0;
  return r;
}

// Number of split-K partial slots a unit uses at step t (combine side).
__host__ __device__ inline int32_t unit_slots(const UnitDesc& u, int32_t t, int32_t L, int32_t chunk) {
  if (u.kind == kUnitFull) return (L + t + chunk - 1) / chunk;
  if (u.kind == kUnitAbsent) return 0;
  return u.n_pchunks + (t + chunk - 1) / chunk;
}

struct AttnParams {
  const UnitDesc* units;
  const TileDesc* tiles;
  const void* q;         // bf16 [q_rows][128]
  void* out;             // bf16 [q_rows][128] (combine)
  float* partial;        // [slots][G][kPartStride]
  void* logits;          // [pivot slots][G][logit_stride] e = 2^(x - m_ref), x = log2 score
                         // (fp32, or fp16 when mat_f16)
  float* mref;           // [pivot slots][G][logit_stride / 16] m_ref per 16-position group
  float* stats;          // [pivot slots][G][2]  (M, L) after combine
  float* rows;           // [pivot slots][row_stride]  GQA-mean probability rows
  int64_t logit_stride;
  int64_t row_stride;
  int32_t group;         // G (<= 8)
  int32_t L;             // prefill length
  int32_t t;             // decode step (0 during prefill scoring)
  int32_t chunk;         // rows per tile
  int32_t recency;       // recency_window
  int32_t n_units;
  float scale_log2;      // log2(e) / sqrt(d)
  const uint8_t* skip;   // per unit: 1 = tiles deferred to a later launch (landing units), or null
  int32_t mat_f16;       // pivot score material: 0 = fp32, 1 = fp16
  int32_t combine_sel;   // combine over: 0 every unit, 1 the units listed in cunits,
                         // 2 every unit that is not a pivot
  const int32_t* cunits; // combine_sel 1: the units (grid.x = n_cunits)
  int32_t n_cunits;
  int32_t pad2_;
};

constexpr int kPartStride = 132;  // M, L, pad, pad, O[128]

}  // namespace hc
