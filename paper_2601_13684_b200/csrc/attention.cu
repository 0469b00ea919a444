// K4: fused ragged split-K flash-decoding over the hierarchical KV store.
//
// No reference implementation exists (the reference moves index sets only,
// SPEC.md:103); semantics follow the exporter's attention
// (pkg/exporter/src/model.ts:232-291): per query head softmax(q.K^T/sqrt(d))
// over the head's resident rows, then P.V; GQA groups of G query heads share
// one KV head.  Pivot heads also emit their scaled logits so the GQA-mean
// probability row (model.ts:274-291) can be formed after the split-K merge.
//
// Decode attention is a stream over K/V (arithmetic intensity ~G flop/B, far
// below the B200 ridge), so the kernel is built around HBM:
//   * one CTA per tile of <= `chunk` rows of one unit; a producer warp
//     streams 64-row K and V sub-tiles into a 3-stage shared-memory ring with
//     TMA (cp.async.bulk.tensor, 128B swizzle) and mbarrier transaction
//     counts; 2 CTAs per SM keep ~192 KB of loads in flight per SM;
//   * four consumer warps each own 16 rows of every sub-tile: QK^T and PV on
//     the tensor pipe with mma.sync m16n8k16 (bf16 in, fp32 accumulate; rows
//     G..15 of the M=16 tile are zero), online softmax in exp2 domain with
//     quad shuffles, conflict-free ldmatrix thanks to the swizzle;
//   * warps merge through shared memory; each tile writes one (M, L, O)
//     partial per query head; combine_kernel merges a unit's partials.

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "hc_common.cuh"
#include "kv_layout.cuh"

namespace hc {
namespace {

constexpr int kSub = 64;                      // rows per pipeline stage
constexpr int kConsumerWarps = 4;
constexpr int kThreadsAttn = (kConsumerWarps + 1) * 32;
constexpr int kStages = 3;
constexpr int kBoxBytes = kSub * 128;         // 64 rows x 64 bf16 (one swizzle span)
constexpr int kStageBytes = 4 * kBoxBytes;    // K lo/hi halves + V lo/hi halves
constexpr int kSmemAttn = kStages * kStageBytes + 1024 /*align*/ + 64 /*barriers*/;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int32_t c0,
                                            int32_t c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1,
                                          uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
// D += A(16x16, row) * B(16x8, col); rows 8..15 of A are zero here (a1=a3=0).
__device__ __forceinline__ void mma_bf16(float (&d)[4], uint32_t a0, uint32_t a2, uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
// Address of 16-byte chunk J (0..15, 8 bf16 each) of row r of a K or V
// sub-tile stored as two 128B-swizzled 64-column boxes.
__device__ __forceinline__ uint32_t swz(uint32_t base, int r, int J) {
  return base + (J >> 3) * kBoxBytes + r * 128 + (((J & 7) ^ (r & 7)) << 4);
}

// Pivot score material element: fp32 (default) or fp16 (compact).
template <bool F16>
struct Mat;
template <>
struct Mat<false> {
  using T = float;
  __device__ static void put2(float* dst, float a, float b) {
    *reinterpret_cast<float2*>(dst) = make_float2(a, b);
  }
  __device__ static void put1(float* dst, float a) { *dst = a; }
};
template <>
struct Mat<true> {
  using T = __half;
  __device__ static void put2(__half* dst, float a, float b) {
    *reinterpret_cast<__half2*>(dst) = __floats2half2_rn(a, b);
  }
  __device__ static void put1(__half* dst, float a) { *dst = __float2half_rn(a); }
};

template <bool F16>
__global__ void __launch_bounds__(kThreadsAttn, 2)
attn_tiles_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                  const AttnParams p) {
  using MT = typename Mat<F16>::T;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* sgen = smem_raw + (sbase - smem_u32(smem_raw));
  const uint32_t bar_full = sbase + kStages * kStageBytes;  // kStages x 8 B
  const uint32_t bar_empty = bar_full + kStages * 8;

  const TileDesc tile = p.tiles[blockIdx.x];
  if (p.skip && p.skip[tile.unit]) return;  // landing unit: its tiles run after the landing
  const UnitDesc unit = p.units[tile.unit];
  const TileRange rg = tile_range(unit, tile.seg_chunk, p.t, p.L, p.recency, p.chunk);
  const int G = p.group;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* part = p.partial + size_t(tile.slot) * G * kPartStride;

  if (rg.n <= 0) {  // nothing resident in this tile at this step
    if (threadIdx.x < G) {
      part[threadIdx.x * kPartStride + 0] = -INFINITY;
      part[threadIdx.x * kPartStride + 1] = 0.f;
    }
    return;
  }
  const int n_sub = (rg.n + kSub - 1) / kSub;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(bar_full + 8 * s, 1);
      mbar_init(bar_empty + 8 * s, kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    // ---------------- producer: TMA K/V sub-tiles into the ring ----------------
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmK)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmV)) : "memory");
      for (int s = 0; s < n_sub; ++s) {
        const int st = s % kStages;
        const uint32_t ph = (s / kStages) & 1;
        mbar_wait(bar_empty + 8 * st, ph ^ 1);
        const uint32_t dst = sbase + st * kStageBytes;
        const uint32_t fb = bar_full + 8 * st;
        mbar_expect_tx(fb, kStageBytes);
        const int32_t row = int32_t(rg.row + int64_t(s) * kSub);
        tma_load_2d(dst + 0 * kBoxBytes, &tmK, 0, row, fb);
        tma_load_2d(dst + 1 * kBoxBytes, &tmK, 64, row, fb);
        tma_load_2d(dst + 2 * kBoxBytes, &tmV, 0, row, fb);
        tma_load_2d(dst + 3 * kBoxBytes, &tmV, 64, row, fb);
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const int g = lane >> 2;   // query head row of the MMA tile
  const int c = lane & 3;    // column pair
  const bool row_ok = g < G;
  // Q A-fragments for 8 k-steps (a0: d 16kk+2c.., a2: d 16kk+8+2c..)
  uint32_t qa0[8], qa2[8];
  {
    const __nv_bfloat16* q = reinterpret_cast<const __nv_bfloat16*>(p.q) +
                             (size_t(unit.q_row) + (row_ok ? g : 0)) * kHeadDim;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const uint32_t lo = *reinterpret_cast<const uint32_t*>(q + 16 * kk + 2 * c);
      const uint32_t hi = *reinterpret_cast<const uint32_t*>(q + 16 * kk + 8 + 2 * c);
      qa0[kk] = row_ok ? lo : 0u;
      qa2[kk] = row_ok ? hi : 0u;
    }
  }
  float o[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_run = -INFINITY, l_run = 0.f;
  const int tb = warp * 16;  // this warp's 16 rows of each sub-tile
  // pivot score-row material: e = 2^(x - m) per token (m = this warp's
  // running max after the 16-token group, one fp32 per group), finalised by
  // score_rows_kernel once the global (M, L) are known.  fp32 keeps the row
  // within fp32 rounding of the oracle's; fp16 halves these bytes at ~5e-4
  // relative error
  MT* lg = nullptr;
  float* mr = nullptr;
  if (unit.pivot_slot >= 0 && rg.pos >= 0 && row_ok) {
    const size_t hg = size_t(unit.pivot_slot) * G + g;
    lg = reinterpret_cast<MT*>(p.logits) + hg * p.logit_stride + rg.pos;
    mr = p.mref + hg * (p.logit_stride / 16) + rg.pos / 16;
  }

  for (int s = 0; s < n_sub; ++s) {
    const int st = s % kStages;
    mbar_wait(bar_full + 8 * st, (s / kStages) & 1);
    const uint32_t sK = sbase + st * kStageBytes;
    const uint32_t sV = sK + 2 * kBoxBytes;

    // S = Q K^T for rows tb..tb+15 (two n-tiles of 8 rows)
    float sc[2][4];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.f;
      const int r = tb + nt * 8 + (lane & 7);
#pragma unroll
      for (int kp = 0; kp < 4; ++kp) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4(swz(sK, r, 4 * kp + (lane >> 3)), b0, b1, b2, b3);
        mma_bf16(sc[nt], qa0[2 * kp], qa2[2 * kp], b0, b1);
        mma_bf16(sc[nt], qa0[2 * kp + 1], qa2[2 * kp + 1], b2, b3);
      }
    }
    // scale, mask, emit pivot logits
    const int base_tok = s * kSub + tb;
    float x[2][2];
    float mloc = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int tok = base_tok + nt * 8 + 2 * c + e;
        const float v = sc[nt][e] * p.scale_log2;
        x[nt][e] = tok < rg.n ? v : -INFINITY;
        mloc = fmaxf(mloc, x[nt][e]);
      }
    }
    mloc = fmaxf(mloc, __shfl_xor_sync(0xffffffffu, mloc, 1));
    mloc = fmaxf(mloc, __shfl_xor_sync(0xffffffffu, mloc, 2));
    const float m_new = fmaxf(m_run, mloc);
    const float mb = (m_new == -INFINITY) ? 0.f : m_new;
    const float alpha = exp2f(m_run - mb);
    float pr[2][2];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) pr[nt][e] = exp2f(x[nt][e] - mb);
    if (lg) {
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const int tok = base_tok + nt * 8 + 2 * c;
        if (tok + 1 < rg.n) {
          Mat<F16>::put2(lg + tok, pr[nt][0], pr[nt][1]);
        } else if (tok < rg.n) {
          Mat<F16>::put1(lg + tok, pr[nt][0]);
        }
      }
      if (c == 0 && base_tok < rg.n) mr[base_tok / 16] = mb;
    }
    l_run = l_run * alpha + (pr[0][0] + pr[0][1]) + (pr[1][0] + pr[1][1]);
    m_run = m_new;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      o[i][0] *= alpha;
      o[i][1] *= alpha;
    }
    const uint32_t pa0 = pack_bf16(pr[0][0], pr[0][1]);
    const uint32_t pa2 = pack_bf16(pr[1][0], pr[1][1]);
    // O += P V over this warp's 16 rows; V fragments via transposed ldmatrix
    {
      const int r = tb + ((lane >> 3) & 1) * 8 + (lane & 7);
#pragma unroll
      for (int dp = 0; dp < 8; ++dp) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(swz(sV, r, 2 * dp + (lane >> 4)), b0, b1, b2, b3);
        mma_bf16(o[2 * dp], pa0, pa2, b0, b1);
        mma_bf16(o[2 * dp + 1], pa0, pa2, b2, b3);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(bar_empty + 8 * st);
  }

  // ---------------- merge the four warps through (reused) shared memory ----------------
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 1);
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 2);
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32) : "memory");  // ring no longer read
  float* ws = reinterpret_cast<float*>(sgen);  // [warp][8 rows][132]
  float* mine = ws + warp * 8 * kPartStride + g * kPartStride;
  if (c == 0) {
    mine[0] = m_run;
    mine[1] = l_run;
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    *reinterpret_cast<float2*>(mine + 4 + i * 8 + 2 * c) = make_float2(o[i][0], o[i][1]);
  }
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32) : "memory");
  const int d = threadIdx.x;  // 0..127
  for (int gg = 0; gg < G; ++gg) {
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kConsumerWarps; ++w) M = fmaxf(M, ws[(w * 8 + gg) * kPartStride]);
    const float mb = (M == -INFINITY) ? 0.f : M;
    float Ls = 0.f, acc = 0.f;
#pragma unroll
    for (int w = 0; w < kConsumerWarps; ++w) {
      const float* src = ws + (w * 8 + gg) * kPartStride;
      const float f = exp2f(src[0] - mb);
      Ls += src[1] * f;
      acc += src[4 + d] * f;
    }
    float* dst = part + gg * kPartStride;
    dst[4 + d] = acc;
    if (d == 0) {
      dst[0] = M;
      dst[1] = Ls;
    }
  }
}

// Merge a unit's split-K partials for one query head (block = (unit, g));
// write O (bf16) and, for pivots, (M, L).  One pass: warp w folds slots
// w, w+4, ... with an online max (lane l owns output dims 4l..4l+3, 512 B
// coalesced per slot), eight slots' loads in flight per warp; the four warp
// states meet in shared memory.
__global__ void __launch_bounds__(128) combine_kernel(const AttnParams p) {
  __shared__ float wm[4], wl[4];
  __shared__ __align__(16) float racc[4][128];
  const UnitDesc u = p.units[p.combine_sel == 1 ? p.cunits[blockIdx.x] : int(blockIdx.x)];
  if (u.kind == kUnitAbsent) return;  // owned by another shard
  if (p.combine_sel == 2 && u.pivot_slot >= 0) return;  // the pivots were combined already
  const int g = blockIdx.y;
  const int G = p.group;
  const int n = unit_slots(u, p.t, p.L, p.chunk);
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const float* base = p.partial + (size_t(u.slot0) * G + g) * kPartStride;
  const size_t sstride = size_t(G) * kPartStride;
  constexpr int kU = 8;
  float m = -INFINITY, l = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int i0 = w; i0 < n; i0 += 4 * kU) {
    float mi[kU], li[kU];
    float4 oi[kU];
#pragma unroll
    for (int q = 0; q < kU; ++q) {
      const int i = i0 + 4 * q;
      li[q] = 0.f;
      mi[q] = -INFINITY;
      if (i < n) {
        const float* src = base + i * sstride;
        mi[q] = src[0];
        li[q] = src[1];
        oi[q] = reinterpret_cast<const float4*>(src + 4)[lane];
      }
    }
#pragma unroll
    for (int q = 0; q < kU; ++q) {
      if (li[q] == 0.f) continue;  // empty tile: O never written
      const float mn = fmaxf(m, mi[q]);
      const float a = exp2f(m - mn), f = exp2f(mi[q] - mn);
      acc.x = acc.x * a + f * oi[q].x;
      acc.y = acc.y * a + f * oi[q].y;
      acc.z = acc.z * a + f * oi[q].z;
      acc.w = acc.w * a + f * oi[q].w;
      l = l * a + f * li[q];
      m = mn;
    }
  }
  reinterpret_cast<float4*>(racc[w])[lane] = acc;
  if (lane == 0) {
    wm[w] = m;
    wl[w] = l;
  }
  __syncthreads();
  const float M = fmaxf(fmaxf(wm[0], wm[1]), fmaxf(wm[2], wm[3]));
  const float mb = (M == -INFINITY) ? 0.f : M;
  float sw[4];
#pragma unroll
  for (int v = 0; v < 4; ++v) sw[v] = wl[v] == 0.f ? 0.f : exp2f(wm[v] - mb);
  const float Ls = (wl[0] * sw[0] + wl[1] * sw[1]) + (wl[2] * sw[2] + wl[3] * sw[3]);
  const float a = (racc[0][tid] * sw[0] + racc[1][tid] * sw[1]) +
                  (racc[2][tid] * sw[2] + racc[3][tid] * sw[3]);
  __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(p.out);
  if (out) out[(size_t(u.q_row) + g) * kHeadDim + tid] = __float2bfloat16_rn(a / Ls);
  if (u.pivot_slot >= 0 && tid == 0) {
    p.stats[(size_t(u.pivot_slot) * G + g) * 2 + 0] = M;
    p.stats[(size_t(u.pivot_slot) * G + g) * 2 + 1] = Ls;
  }
}

// GQA-mean probability row of every pivot over [0, L + t):
//   row[pos] = (sum_j e_j(pos) * 2^(m_j(pos/16) - M_j) * (1 / L_j)) / G
// i.e. (sum_j exp(s_j - max_j) / sum_j) / G in head order (model.ts:283-289).
// One thread per 8 consecutive positions: all G 16-B loads of fp16 material
// and G m_ref loads are issued before any is consumed (latency-bound
// otherwise), then one exp2 per head and 8 FMAs.
constexpr int kRowsThreads = 256;
constexpr int kRowsSpan = kRowsThreads * 8;  // positions per block

__device__ __forceinline__ void unpack8(const uint4 (&raw)[2], float (&f)[8], const float*) {
  const float4 a = *reinterpret_cast<const float4*>(&raw[0]);
  const float4 b = *reinterpret_cast<const float4*>(&raw[1]);
  f[0] = a.x, f[1] = a.y, f[2] = a.z, f[3] = a.w, f[4] = b.x, f[5] = b.y, f[6] = b.z, f[7] = b.w;
}
__device__ __forceinline__ void unpack8(const uint4 (&raw)[1], float (&f)[8], const __half*) {
  const uint32_t w[4] = {raw[0].x, raw[0].y, raw[0].z, raw[0].w};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float2 v = __half22float2(*reinterpret_cast<const __half2*>(&w[q]));
    f[2 * q] = v.x;
    f[2 * q + 1] = v.y;
  }
}

template <int G, bool F16>
__global__ void __launch_bounds__(kRowsThreads) score_rows_kernel(const AttnParams p,
                                                                  const int32_t* __restrict__ pivot_units) {
  using MT = typename Mat<F16>::T;
  constexpr int kV = F16 ? 1 : 2;  // 16-B vectors per 8 positions
  __shared__ float s_m[G], s_inv[G];
  const UnitDesc u = p.units[pivot_units[blockIdx.y]];
  const int slot = u.pivot_slot;
  const int len = p.L + p.t;
  const int tid = threadIdx.x;
  if (tid < G) {
    s_m[tid] = p.stats[(size_t(slot) * G + tid) * 2 + 0];
    s_inv[tid] = 1.0f / p.stats[(size_t(slot) * G + tid) * 2 + 1];
  }
  __syncthreads();
  const int pos = blockIdx.x * kRowsSpan + tid * 8;
  if (pos >= len) return;
  const MT* lg = reinterpret_cast<const MT*>(p.logits) + size_t(slot) * G * p.logit_stride;
  const float* mr = p.mref + size_t(slot) * G * (p.logit_stride / 16);
  uint4 raw[G][kV];
  float mv[G];
#pragma unroll
  for (int j = 0; j < G; ++j) {
    const uint4* src = reinterpret_cast<const uint4*>(lg + size_t(j) * p.logit_stride + pos);
#pragma unroll
    for (int v = 0; v < kV; ++v) raw[j][v] = __ldcs(src + v);
    mv[j] = __ldg(mr + size_t(j) * (p.logit_stride / 16) + pos / 16);
  }
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;
#pragma unroll
  for (int j = 0; j < G; ++j) {
    const float cj = exp2f(mv[j] - s_m[j]) * s_inv[j];
    float f[8];
    unpack8(raw[j], f, static_cast<const MT*>(nullptr));
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] += f[e] * cj;
  }
  const float rg = float(G);
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = acc[e] / rg;
  float* row = p.rows + size_t(slot) * p.row_stride;
  if (pos + 7 < len) {
    reinterpret_cast<float4*>(row + pos)[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
    reinterpret_cast<float4*>(row + pos)[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
  } else {
    for (int e = 0; pos + e < len; ++e) row[pos + e] = acc[e];
  }
}

}  // namespace

// ---- host launchers (used by engine.cu and the raw test entry point) ----

int make_kv_tensor_map_rows(CUtensorMap* map, const void* base, int64_t rows, int box_rows);
int make_bf16_tensor_map(CUtensorMap* map, const void* base, int64_t rows, int64_t cols,
                         int box_cols, int box_rows);

int make_kv_tensor_map(CUtensorMap* map, const void* base, int64_t rows) {
  return make_kv_tensor_map_rows(map, base, rows, kSub);
}

// 2-D bf16 [rows x 128] tensor map, 128B swizzle, boxes of 64 columns x box_rows rows.
int make_kv_tensor_map_rows(CUtensorMap* map, const void* base, int64_t rows, int box_rows) {
  return make_bf16_tensor_map(map, base, rows, kHeadDim, 64, box_rows);
}

// Generic 2-D bf16 [rows x cols] row-major tensor map with 128B swizzle
// (box_cols * 2 must be <= 128 B), out-of-bounds boxes zero-filled.
int make_bf16_tensor_map(CUtensorMap* map, const void* base, int64_t rows, int64_t cols,
                         int box_cols, int box_rows) {
  HC_REQUIRE(rows > 0 && rows < (int64_t(1) << 31), HC_EINVAL, "tensor rows out of TMA range");
  HC_REQUIRE((reinterpret_cast<uintptr_t>(base) & 15) == 0 && (cols * 2) % 16 == 0, HC_EINVAL,
             "tensor base / row pitch not 16-B aligned");
  HC_REQUIRE(box_cols * 2 <= 128 && box_rows <= 256, HC_EINVAL, "bad TMA box");
  // resolve the driver entry point at run time: the library must load (and
  // export its ABI) on hosts without libcuda, e.g. the CPU build container
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    HC_CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    HC_REQUIRE(fn && q == cudaDriverEntryPointSuccess, HC_ECUDA, "cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<EncodeFn>(fn);
  }
  const cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  const cuuint64_t strides[1] = {cuuint64_t(cols * 2)};
  const cuuint32_t box[2] = {cuuint32_t(box_cols), cuuint32_t(box_rows)};
  const cuuint32_t estr[2] = {1u, 1u};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                      strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  HC_REQUIRE(r == CUDA_SUCCESS, HC_ECUDA, "cuTensorMapEncodeTiled failed (%d)", int(r));
  return HC_OK;
}

static int configure_attn() {
  static bool configured = false;
  if (!configured) {
    HC_CUDA_TRY(cudaFuncSetAttribute(attn_tiles_kernel<false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemAttn));
    HC_CUDA_TRY(cudaFuncSetAttribute(attn_tiles_kernel<true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemAttn));
    configured = true;
  }
  return HC_OK;
}

// Split-K combine (O and the pivots' softmax statistics).
int launch_combine(const AttnParams& p, cudaStream_t st) {
  HC_REQUIRE(p.group >= 1 && p.group <= 8, HC_EINVAL, "GQA group must be 1..8");
  const int n = p.combine_sel == 1 ? p.n_cunits : p.n_units;
  if (n > 0) {
    combine_kernel<<<dim3(n, p.group), 128, 0, st>>>(p);
    HC_CHECK_LAUNCH();
  }
  return HC_OK;
}

// The pivots' GQA-mean probability rows (needs combine's statistics).
int launch_score_rows(const AttnParams& p, const int32_t* pivot_units_dev, int n_pivots,
                      cudaStream_t st) {
  if (n_pivots > 0 && p.rows) {
    HC_REQUIRE(p.logit_stride % 16 == 0 && p.row_stride % 8 == 0, HC_EINVAL,
               "score-row strides must be multiples of 16 / 8");
    const int len = p.L + p.t;
    dim3 grid((len + kRowsSpan - 1) / kRowsSpan, n_pivots);
    switch (p.group) {
#define HC_ROWS(GG)                                                                     \
  case GG:                                                                              \
    if (p.mat_f16) score_rows_kernel<GG, true><<<grid, kRowsThreads, 0, st>>>(p, pivot_units_dev); \
    else score_rows_kernel<GG, false><<<grid, kRowsThreads, 0, st>>>(p, pivot_units_dev);         \
    break;
      HC_ROWS(1) HC_ROWS(2) HC_ROWS(3) HC_ROWS(4) HC_ROWS(5) HC_ROWS(6) HC_ROWS(7) HC_ROWS(8)
#undef HC_ROWS
    }
    HC_CHECK_LAUNCH();
  }
  return HC_OK;
}

// K4 over an explicit tile list (p.tiles, n_tiles entries).
int launch_attn_tiles(const CUtensorMap& tmK, const CUtensorMap& tmV, const AttnParams& p,
                      int n_tiles, cudaStream_t st) {
  HC_TRY(configure_attn());
  if (n_tiles > 0) {
    if (p.mat_f16) attn_tiles_kernel<true><<<n_tiles, kThreadsAttn, kSmemAttn, st>>>(tmK, tmV, p);
    else attn_tiles_kernel<false><<<n_tiles, kThreadsAttn, kSmemAttn, st>>>(tmK, tmV, p);
    HC_CHECK_LAUNCH();
  }
  return HC_OK;
}


}  // namespace hc
