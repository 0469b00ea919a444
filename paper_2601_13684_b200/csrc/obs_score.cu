// K5: prefill observation-window scoring on the 5th-generation tensor cores.
//
// The step-0 record of a head is the last prompt token's post-softmax
// attention averaged over the G query heads of its GQA group (export.ts:125-127,
// model.ts:274-291).  Generalised to an observation window of w prompt tokens
// (w = 1 is exactly the reference semantics), the score of key t is
//     score(t) = 1/(w*G) * sum_{i<w, j<G} softmax_t(q_{i,j} . k_t / sqrt(d)),
// with query i = prompt position L-w+i seeing keys t <= L-w+i (causal).
// That is a dense contraction: the M = w*G query rows (padded to 128) of one
// KV head against all L keys, so it runs as tcgen05 GEMM tiles:
//   * warp 0: TMA producer -- Q_obs once (two 128B-swizzled 64-col boxes),
//     then 128-key x 128-d K tiles into a 4-stage shared-memory ring;
//   * warp 1: allocates 256 TMEM columns (two 128x128 fp32 accumulators) and
//     issues tcgen05.mma.cta_group::1.kind::f16 (M=128, N=128, K=16 x 8)
//     from shared-memory descriptors; tcgen05.commit frees ring slots and
//     hands accumulators to the epilogue;
//   * warps 2-5: epilogue, one thread per query row, tcgen05.ld 32x32b.x32.
// Pass 1 keeps per-row online softmax statistics (max, sum) per key chunk;
// obs_merge combines chunks; pass 2 recomputes the tiles TRANSPOSED (S^T =
// K Q^T: TMEM lane = key, column = query row), so each epilogue thread turns
// its key's 64 query-row scores into probabilities and sums them in
// registers; the two row halves meet in shared memory.  Each key
// tile's score column is owned by exactly one CTA: no atomics, deterministic.

#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>

#include "hc_common.cuh"

namespace hc {
namespace {

constexpr int kM = 128;                 // query rows per KV head (w*G padded)
constexpr int kN = 128;                 // keys per tile
constexpr int kBox = 128 * 128;         // bytes of one 64-col x 128-row swizzled box
constexpr int kTile = 2 * kBox;         // one K tile (128 keys x 128 d bf16)
constexpr int kStagesObs = 2;  // 2 CTAs per SM keep 4 K tiles in flight per SM
constexpr int kEpiWarps = 8;  // two per TMEM lane quarter: each owns half of a tile's columns
constexpr int kObsThreads = (2 + kEpiWarps) * 32;
constexpr int kSmemObs = 1024 + kTile /*Q*/ + kStagesObs * kTile + 256 /*barriers*/ +
                         4 * 4 * kN * 4 /*column partials of 4 tiles*/;

struct ObsParams {
  int L;             // keys per unit
  int64_t kstride;   // rows between consecutive units' keys (>= L)
  int rows;          // valid query rows (w * G)
  int G;
  int w;
  int tiles_per_cta; // key tiles per CTA
  int pass;          // 1: statistics, 2: scores
  float scale_log2;  // log2(e) / sqrt(d)
  float* part;       // pass 1 out: [unit][chunk][128][2] (m, l), log2 domain
  const float* stats;  // pass 2 in: [unit][128][2] (M, L)
  float* out;        // pass 2 out: [unit][row_stride]
  int64_t row_stride;
  int n_chunks;
  float* xs;         // small windows (w*G <= 16): pass 1 also keeps the raw scores
  int64_t xs_stride; // [unit][rows][xs_stride]; pass 2 then reads them instead of K
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mb_init(uint32_t b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c));
}
__device__ __forceinline__ void mb_expect(uint32_t b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mb_arrive(uint32_t b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
}
__device__ __forceinline__ void mb_wait(uint32_t b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n\t}" ::"r"(b),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma2d(uint32_t dst, const CUtensorMap* m, int c0, int c1,
                                      uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
// Shared-memory matrix descriptor (sm_100 UMMA): K-major, 128B swizzle,
// 8-row core-matrix groups 1024 B apart (SBO), version 1.
__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
  uint64_t d = 0;
  d |= uint64_t((addr >> 4) & 0x3FFF);          // start address
  d |= uint64_t(1) << 16;                        // LBO (unused for swizzled K-major)
  d |= uint64_t(1024 >> 4) << 32;                // SBO
  d |= uint64_t(1) << 46;                        // descriptor version (sm_100)
  d |= uint64_t(2) << 61;                        // SWIZZLE_128B
  return d;
}
// Instruction descriptor: D f32, A/B bf16, both K-major, M=128, N=128.
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(kN >> 3) << 17) |
                            (uint32_t(kM >> 4) << 24);

__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kIdesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   bar)
               : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// exp2 as one MUFU.EX2 (ex2.approx.ftz: max relative error 2^-22, results
// below 2^-126 flush to 0); exp2f() adds a subnormal-range fixup per call
// (FSETP + 2 FMUL), which the SFU-bound epilogues cannot afford.
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <bool kKeep>  // kKeep: small-window pass 1 also stores the raw scores (p.xs)
__global__ void __launch_bounds__(kObsThreads, 2)
obs_score_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmQ,
                 const ObsParams p) {
  extern __shared__ uint8_t sm_raw[];
  const uint32_t base = (smem_addr(sm_raw) + 1023u) & ~1023u;
  uint8_t* gbase = sm_raw + (base - smem_addr(sm_raw));
  const uint32_t sQ = base;
  const uint32_t sK = base + kTile;
  const uint32_t bars = sK + kStagesObs * kTile;
  const uint32_t full = bars, empty = bars + 8 * kStagesObs;
  const uint32_t tfull = bars + 16 * kStagesObs, tempty = tfull + 16, qfull = tempty + 16;
  const uint32_t tmem_slot = qfull + 8;
  float* colsum = reinterpret_cast<float*>(gbase + (bars - base) + 256);  // [4][4][128]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(gbase + (tmem_slot - base));

  const int unit = blockIdx.y, chunk = blockIdx.x;
  const int tile0 = chunk * p.tiles_per_cta;
  const int n_tiles_unit = (p.L + kN - 1) / kN;
  const int n_tiles = min(p.tiles_per_cta, n_tiles_unit - tile0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStagesObs; ++s) {
      mb_init(full + 8 * s, 1);
      mb_init(empty + 8 * s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mb_init(tfull + 8 * a, 1);
      mb_init(tempty + 8 * a, kEpiWarps);  // one arrive per epilogue warp
    }
    mb_init(qfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {  // TMEM: two 128-column fp32 accumulators
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
                     tmem_slot));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    if (lane == 0 && n_tiles > 0) {
      mb_expect(qfull, kTile);
      tma2d(sQ, &tmQ, 0, unit * kM, qfull);
      tma2d(sQ + kBox, &tmQ, 64, unit * kM, qfull);
      for (int i = 0; i < n_tiles; ++i) {
        const int s = i % kStagesObs;
        mb_wait(empty + 8 * s, ((i / kStagesObs) & 1) ^ 1);
        mb_expect(full + 8 * s, kTile);
        const int row = int(unit * p.kstride) + (tile0 + i) * kN;
        tma2d(sK + s * kTile, &tmK, 0, row, full + 8 * s);
        tma2d(sK + s * kTile + kBox, &tmK, 64, row, full + 8 * s);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0 && n_tiles > 0) {
      mb_wait(qfull, 0);
      for (int i = 0; i < n_tiles; ++i) {
        const int s = i % kStagesObs, a = i & 1;
        mb_wait(tempty + 8 * a, ((i >> 1) & 1) ^ 1);
        mb_wait(full + 8 * s, (i / kStagesObs) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + a * kN;
        // pass 1: S = Q K^T (TMEM lane = query row, column = key); pass 2: S^T =
        // K Q^T (lane = key, column = query row), so each thread's column sum
        // of probabilities is a plain sum over its registers -- no shuffles
        const bool tr = !kKeep && p.pass == 2;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk >> 2) * kBox + (kk & 3) * 32;
          const uint64_t qd = sdesc(sQ + off), kd = sdesc(sK + s * kTile + off);
          umma(d, tr ? kd : qd, tr ? qd : kd, kk > 0 ? 1u : 0u);
        }
        umma_commit(empty + 8 * s);  // ring slot reusable once these MMAs finish
        umma_commit(tfull + 8 * a);  // accumulator ready for the epilogue
      }
    }
    __syncwarp();
  } else {
    // ---------------- epilogue: thread = query row, warp = half of the columns ----------------
    const int q4 = warp & 3;                 // TMEM lane quarter this warp may access
    const int half = (warp - 2) >> 2;        // columns [64 * half, 64 * half + 64) of each tile
    const int r = q4 * 32 + lane;            // query row
    const bool row_ok = r < p.rows;
    const int qpos = p.L - p.w + (row_ok ? r / p.G : 0);  // causal limit of this row
    float m = -INFINITY, l = 0.f;
    const float inv_rows = 1.f / float(p.rows);
    // pass 2: per query row, exp2(x*scale - M - log2 L) = its probability;
    // rows beyond w*G or with an empty softmax get +inf (probability 0)
    float* s_off = colsum + 4 * 2 * kN;  // [128]
    if (!kKeep && p.pass == 2) {
      const int t = threadIdx.x - 64;  // 0..255
      if (t < kM) {
        float o = INFINITY;
        if (t < p.rows) {
          const float Mt = p.stats[(size_t(unit) * kM + t) * 2 + 0];
          const float Lt = p.stats[(size_t(unit) * kM + t) * 2 + 1];
          if (Lt > 0.f) o = Mt + log2f(Lt);
        }
        s_off[t] = o;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
    }
    for (int i = 0; i < n_tiles; ++i) {
      const int a = i & 1;
      mb_wait(tfull + 8 * a, (i >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int key0 = (tile0 + i) * kN;
      // this warp's two 32-column TMEM loads in flight per wait (64 registers)
      float v2[2][32];
      const int c0 = half * 2;
      tmem_ld32(tmem + (uint32_t(q4 * 32) << 16) + a * kN + c0 * 32, v2[0]);
      tmem_ld32(tmem + (uint32_t(q4 * 32) << 16) + a * kN + (c0 + 1) * 32, v2[1]);
      tmem_wait_ld();
      // the accumulator may be overwritten as soon as every warp holds its columns
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mb_arrive(tempty + 8 * a);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float (&v)[32] = v2[h];
        const int c = c0 + h;
        const int first = key0 + c * 32;
        const bool unmasked = row_ok && first + 31 <= qpos;  // common case: no causal cut
        if (p.pass == 1) {
          // common case: the row's running reference m stays (softmax is shift
          // invariant; m need not be the max, only keep exp2 finite), so no
          // per-element max -- one FFMA + EX2 + FADD; a chunk whose sum would
          // get large falls back to the exact max below
          if (!row_ok) continue;  // padding rows: no statistics
          if (kKeep && first < p.L) {  // single-read path: keep this row's raw scores
            float* dst = p.xs + (size_t(unit) * p.rows + r) * p.xs_stride + first;
            if (first + 31 < p.L) {
#pragma unroll
              for (int j = 0; j < 32; j += 4)
                *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
            } else {  // last chunk (unrolled: v must stay in registers)
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (first + j < p.L) dst[j] = v[j];
            }
          }
          if (unmasked && m != -INFINITY) {
            float s = 0.f;
#pragma unroll
            for (int j = 0; j < 32; ++j) s += fast_exp2(fmaf(v[j], p.scale_log2, -m));
            if (s <= 0x1p64f) {
              l += s;
              continue;
            }
          }
          // max on raw scores (scale > 0), then exp2(v*scale - m) as one FFMA + EX2
          float tmax = -INFINITY;
          if (unmasked) {
#pragma unroll
            for (int j = 0; j < 32; ++j) tmax = fmaxf(tmax, v[j]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              v[j] = (row_ok && first + j <= qpos) ? v[j] : -INFINITY;
              tmax = fmaxf(tmax, v[j]);
            }
          }
          const float mn = fmaxf(m, tmax * p.scale_log2);
          const float mb = mn == -INFINITY ? 0.f : mn;
          float s = 0.f;
#pragma unroll
          for (int j = 0; j < 32; ++j) s += fast_exp2(fmaf(v[j], p.scale_log2, -mb));
          l = l * exp2f(m - mb) + s;
          m = mn;
        }
      }
      if (!kKeep && p.pass == 2) {
        // transposed accumulator: this thread is key `key`, its 64 columns the
        // query rows [64*half, 64*half + 64); p = exp2(x*scale - off_row)
        const int key = key0 + q4 * 32 + lane;
        const int rb = half * 64;
        float acc = 0.f;
        if (key0 + kN - 1 <= p.L - p.w) {  // the whole tile precedes every query
#pragma unroll
          for (int h = 0; h < 2; ++h) {
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              const float4 o = *reinterpret_cast<const float4*>(s_off + rb + h * 32 + j);
              acc += fast_exp2(fmaf(v2[h][j + 0], p.scale_log2, -o.x));
              acc += fast_exp2(fmaf(v2[h][j + 1], p.scale_log2, -o.y));
              acc += fast_exp2(fmaf(v2[h][j + 2], p.scale_log2, -o.z));
              acc += fast_exp2(fmaf(v2[h][j + 3], p.scale_log2, -o.w));
            }
          }
        } else {  // causal cut: row r (window position r / G) sees keys <= L - w + r / G
#pragma unroll
          for (int h = 0; h < 2; ++h) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int r = rb + h * 32 + j;
              const bool vis = r < p.rows && key <= p.L - p.w + r / p.G;
              acc += vis ? fast_exp2(fmaf(v2[h][j], p.scale_log2, -s_off[r])) : 0.f;
            }
          }
        }
        colsum[((i & 3) * 2 + half) * kN + q4 * 32 + lane] = acc;
      }
      if (!kKeep && p.pass == 2 && ((i & 1) || i == n_tiles - 1)) {
        // one barrier per PAIR of tiles: the partials of tile i live in buffer
        // i&3, which tile i+4 overwrites only after the next pair's barrier
        // (every thread has read this pair's keys by then); the 256 epilogue
        // threads then add the two row halves of one (tile, key) each
        asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
        const int t = threadIdx.x - 64;  // 0..255
        const int ti = (i & 1) ? i - 1 + (t >> 7) : i;
        const int col = t & (kN - 1);
        if ((i & 1) || t < kN) {
          const float* cs = colsum + (ti & 3) * 2 * kN;
          const float sum = cs[col] + cs[kN + col];
          const int kt = (tile0 + ti) * kN + col;
          if (kt < p.L) p.out[size_t(unit) * p.row_stride + kt] = sum * inv_rows;
        }
      }
    }
    if (p.pass == 1) {  // one (m, l) per row and column half: 2 x n_chunks partials per row
      float* dst = p.part + ((size_t(unit) * 2 * p.n_chunks + 2 * chunk + half) * kM + r) * 2;
      dst[0] = m;
      dst[1] = l;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

// Single-read pass 2 for small windows (w*G <= 16 rows): the probabilities
// from the raw scores pass 1 kept, 4 keys per thread, rows in order --
// score(t) = sum_r exp2(x_rt*scale - M_r - log2 L_r) / rows.  K is read once.
__global__ void __launch_bounds__(256) obs_rows_from_scores_kernel(const ObsParams p) {
  __shared__ float off[16];
  const int unit = blockIdx.y;
  // each block merges its unit's pass-1 chunk statistics itself (obs_merge's
  // arithmetic; a few KB from L2) instead of a separate launch
  const int parts = 2 * p.n_chunks;
  if (threadIdx.x < p.rows) {
    const int r = threadIdx.x;
    const float* src = p.part + (size_t(unit) * parts * kM + r) * 2;
    float M = -INFINITY;
    for (int c = 0; c < parts; ++c) M = fmaxf(M, src[size_t(c) * kM * 2]);
    const float mb = M == -INFINITY ? 0.f : M;
    float Lt = 0.f;
    for (int c = 0; c < parts; ++c) {
      const float l = src[size_t(c) * kM * 2 + 1];
      if (l > 0.f) Lt += l * exp2f(src[size_t(c) * kM * 2] - mb);
    }
    off[r] = Lt > 0.f ? mb + log2f(Lt) : INFINITY;
  }
  __syncthreads();
  const int key = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (key >= p.L) return;
  const float* xs = p.xs + size_t(unit) * p.rows * p.xs_stride + key;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int r = 0; r < p.rows; ++r) {
    const float4 x = *reinterpret_cast<const float4*>(xs + size_t(r) * p.xs_stride);
    const float o = -off[r];
    const int qpos = p.L - p.w + r / p.G;  // causal limit of row r
    const float xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int e = 0; e < 4; ++e)
      acc[e] += (key + e <= qpos) ? fast_exp2(fmaf(xv[e], p.scale_log2, o)) : 0.f;
  }
  const float inv = 1.f / float(p.rows);
  float* out = p.out + size_t(unit) * p.row_stride + key;
  for (int e = 0; e < 4 && key + e < p.L; ++e) out[e] = acc[e] * inv;
}

// Combine pass-1 chunk statistics: (M, L) per query row, log2 domain.
__global__ void obs_merge_kernel(const float* __restrict__ part, int n_chunks,
                                 float* __restrict__ stats) {
  const int unit = blockIdx.x, r = threadIdx.x;
  const float* src = part + (size_t(unit) * n_chunks * kM + r) * 2;
  float M = -INFINITY;
  for (int c = 0; c < n_chunks; ++c) M = fmaxf(M, src[size_t(c) * kM * 2]);
  const float mb = M == -INFINITY ? 0.f : M;
  float L = 0.f;
  for (int c = 0; c < n_chunks; ++c) {
    const float l = src[size_t(c) * kM * 2 + 1];
    if (l > 0.f) L += l * exp2f(src[size_t(c) * kM * 2] - mb);
  }
  stats[(size_t(unit) * kM + r) * 2 + 0] = mb;
  stats[(size_t(unit) * kM + r) * 2 + 1] = L;
}

// Pack q_obs [B][w][H*G][128] into the padded [B*H][128][128] operand
// (row r = i*G + j of KV head h: query head h*G+j at window position i).
__global__ void obs_pack_q_kernel(const __nv_bfloat16* __restrict__ q, int H, int G, int w,
                                  __nv_bfloat16* __restrict__ qp) {
  const int unit = blockIdx.x, r = blockIdx.y;  // unit = b*H + h
  const int b = unit / H, h = unit % H;
  const int d = threadIdx.x;
  __nv_bfloat16 val = __float2bfloat16_rn(0.f);
  if (r < w * G) {
    const int i = r / G, j = r % G;
    val = q[((size_t(b) * w + i) * (H * G) + h * G + j) * 128 + d];
  }
  qp[(size_t(unit) * kM + r) * 128 + d] = val;
}

// Key tiles per CTA: about two waves of 2 CTAs x 148 SMs over all units.
int obs_tiles_per_cta(int n_units, int n_tiles) {
  const long total = long(n_units) * n_tiles;
  const long ctas = 2L * 2 * 148;
  return int(std::max(4L, (total + ctas - 1) / ctas));
}

}  // namespace

int make_kv_tensor_map_rows(CUtensorMap* map, const void* base, int64_t rows, int box_rows);

// Score rows for n_units KV heads whose keys are k[unit*L + t][128] and whose
// observation queries are q_obs [B][w][H*G][128] (n_units = B*H).  `scratch`
// must hold obs_scratch_bytes(); out rows have stride row_stride floats.
constexpr int kSmallRows = 16;  // w*G up to this: K read once, raw scores kept

size_t obs_scratch_bytes(int n_units, int L, int rows) {
  const int n_tiles = (L + kN - 1) / kN;
  const int tiles_per_cta = obs_tiles_per_cta(n_units, n_tiles);
  const int n_chunks = (n_tiles + tiles_per_cta - 1) / tiles_per_cta;
  const size_t xs = rows <= kSmallRows ? size_t(n_units) * rows * (size_t(L + 3) / 4 * 4) * 4 : 0;
  return size_t(n_units) * kM * 128 * 2 /*packed Q*/ +
         size_t(n_units) * 2 * n_chunks * kM * 2 * 4 /*partials*/ + size_t(n_units) * kM * 2 * 4 +
         xs + 256;
}

int launch_obs_scores(const void* k, const void* q_obs, int B, int H, int G, int w, int L,
                      float* out, int64_t row_stride, void* scratch, cudaStream_t st,
                      int64_t kstride) {
  if (kstride <= 0) kstride = L;
  HC_REQUIRE(kstride >= L && int64_t(B) * H * kstride < (int64_t(1) << 31), HC_EINVAL,
             "key stride %lld out of range", (long long)kstride);
  HC_REQUIRE(w >= 1 && w * G <= kM, HC_EINVAL, "observation window %d x group %d > 128 rows", w,
             G);
  static bool configured = false;
  if (!configured) {
    HC_CUDA_TRY(cudaFuncSetAttribute(obs_score_kernel<false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemObs));
    HC_CUDA_TRY(cudaFuncSetAttribute(obs_score_kernel<true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemObs));
    configured = true;
  }
  const int n_units = B * H;
  const int n_tiles = (L + kN - 1) / kN;
  const int tiles_per_cta = obs_tiles_per_cta(n_units, n_tiles);
  const int n_chunks = (n_tiles + tiles_per_cta - 1) / tiles_per_cta;
  char* sc = static_cast<char*>(scratch);
  __nv_bfloat16* qp = reinterpret_cast<__nv_bfloat16*>(sc);
  float* part = reinterpret_cast<float*>(sc + size_t(n_units) * kM * 128 * 2);
  float* stats = part + size_t(n_units) * 2 * n_chunks * kM * 2;
  static const int small_rows = getenv("HC_K5_SMALL_ROWS") ? atoi(getenv("HC_K5_SMALL_ROWS"))
                                                           : kSmallRows;  // A/B switch
  const bool small = w * G <= std::min(small_rows, kSmallRows);
  float* xs = nullptr;
  if (small) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(stats + size_t(n_units) * kM * 2);
    xs = reinterpret_cast<float*>((a + 15) & ~uintptr_t(15));
  }
  obs_pack_q_kernel<<<dim3(n_units, kM), 128, 0, st>>>(
      static_cast<const __nv_bfloat16*>(q_obs), H, G, w, qp);
  HC_CHECK_LAUNCH();
  CUtensorMap tk, tq;
  HC_TRY_RC(make_kv_tensor_map_rows(&tk, k, int64_t(n_units) * kstride, 128));
  HC_TRY_RC(make_kv_tensor_map_rows(&tq, qp, int64_t(n_units) * kM, 128));
  ObsParams p{};
  p.L = L;
  p.kstride = kstride;
  p.rows = w * G;
  p.G = G;
  p.w = w;
  p.tiles_per_cta = tiles_per_cta;
  p.scale_log2 = float(1.4426950408889634 / 11.313708498984761);
  p.part = part;
  p.stats = stats;
  p.out = out;
  p.row_stride = row_stride;
  p.n_chunks = n_chunks;
  p.xs = xs;
  p.xs_stride = (int64_t(L) + 3) / 4 * 4;
  dim3 grid(n_chunks, n_units);
  p.pass = 1;
  if (small) obs_score_kernel<true><<<grid, kObsThreads, kSmemObs, st>>>(tk, tq, p);
  else obs_score_kernel<false><<<grid, kObsThreads, kSmemObs, st>>>(tk, tq, p);
  HC_CHECK_LAUNCH();
  p.pass = 2;
  if (small) {  // the window's few rows: probabilities from the kept scores, K not re-read
    obs_rows_from_scores_kernel<<<dim3((L + 1023) / 1024, n_units), 256, 0, st>>>(p);
  } else {
    obs_merge_kernel<<<n_units, kM, 0, st>>>(part, 2 * n_chunks, stats);
    HC_CHECK_LAUNCH();
    obs_score_kernel<false><<<grid, kObsThreads, kSmemObs, st>>>(tk, tq, p);
  }
  HC_CHECK_LAUNCH();
  return HC_OK;
}

}  // namespace hc

extern "C" int hc_obs_scores(const void* k_dev, const void* q_obs_dev, int32_t batch,
                             int32_t kv_heads, int32_t group, int32_t window, int32_t L,
                             float* rows_dev, int64_t row_stride, void* stream) {
  HC_REQUIRE(k_dev && q_obs_dev && rows_dev && batch > 0 && kv_heads > 0 && L > 0, HC_EINVAL,
             "hc_obs_scores: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  const size_t bytes = hc::obs_scratch_bytes(batch * kv_heads, L, window * group);
  void* scratch = nullptr;
  HC_CUDA_TRY(cudaMallocAsync(&scratch, bytes, st));
  const int rc = hc::launch_obs_scores(k_dev, q_obs_dev, batch, kv_heads, group, window, L,
                                       rows_dev, row_stride, scratch, st, 0);
  HC_CUDA_TRY(cudaFreeAsync(scratch, st));
  return rc;
}
