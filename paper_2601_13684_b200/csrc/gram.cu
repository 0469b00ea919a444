// K6: head-similarity profiling counts as a tcgen05 GEMM.
//
// The taxonomy (profiling.py:286-367, metrics.py:74-106) compares top-k
// index sets: stability = |S_t & S_0| / min(|S_t|, |S_0|) per head and step,
// similarity / agreement = |S_{t,h} & S_{t,h'}| / min(...) per step and
// same-layer head pair.  All intersection sizes of a (trace, layer) are
// entries of one Gram matrix  C = X X^T  of the 0/1 indicator matrix X
// [sets = (step, head)] x [positions], a dense contraction over the
// positions: bf16 0/1 operands are exact and fp32 accumulation in TMEM is
// exact for counts < 2^24.
//
// One CTA computes a 128 x 128 block of C: warp 0 streams 128-set x 64-position
// tiles of both operands with TMA (128B swizzle), warp 1 issues
// tcgen05.mma (M=N=128, K=16 x 4 per tile) accumulating in TMEM across the
// whole position range, warps 2-5 drain TMEM with tcgen05.ld and store.

#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>

#include "hc_common.cuh"

namespace hc {

int make_bf16_tensor_map(CUtensorMap* map, const void* base, int64_t rows, int64_t cols,
                         int box_cols, int box_rows);

namespace {

constexpr int kGM = 128;
constexpr int kGK = 64;                    // positions per tile (one 128-B swizzle span)
constexpr int kGBox = 128 * 128;           // 128 rows x 128 B
constexpr int kGStages = 4;
constexpr int kGThreads = 192;
constexpr int kGSmem = 1024 + kGStages * 2 * kGBox + 128;

__device__ __forceinline__ uint32_t saddr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bar_init(uint32_t b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c));
}
__device__ __forceinline__ void bar_expect(uint32_t b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bar_wait(uint32_t b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n\t}" ::"r"(b),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap* m, int c0, int c1,
                                       uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ uint64_t kmajor_sw128(uint32_t addr) {
  return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) |
         (uint64_t(1) << 46) | (uint64_t(2) << 61);
}
constexpr uint32_t kGIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(128 >> 3) << 17) |
                             (uint32_t(128 >> 4) << 24);

__global__ void __launch_bounds__(kGThreads, 1)
gram_kernel(const __grid_constant__ CUtensorMap tmX, int rows_pad, int k_tiles,
            float* __restrict__ out) {
  extern __shared__ uint8_t gsm[];
  const uint32_t base = (saddr(gsm) + 1023u) & ~1023u;
  uint8_t* gbase = gsm + (base - saddr(gsm));
  const uint32_t bars = base + kGStages * 2 * kGBox;
  const uint32_t full = bars, empty = bars + 8 * kGStages, done = bars + 16 * kGStages;
  const uint32_t tslot = done + 8;
  uint32_t* tholder = reinterpret_cast<uint32_t*>(gbase + (tslot - base));
  const int mb = blockIdx.x, nb = blockIdx.y, batch = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rowA = batch * rows_pad + mb * kGM, rowB = batch * rows_pad + nb * kGM;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kGStages; ++s) {
      bar_init(full + 8 * s, 1);
      bar_init(empty + 8 * s, 1);
    }
    bar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(tslot));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tholder;

  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < k_tiles; ++i) {
        const int s = i % kGStages;
        bar_wait(empty + 8 * s, ((i / kGStages) & 1) ^ 1);
        bar_expect(full + 8 * s, 2 * kGBox);
        const uint32_t dst = base + s * 2 * kGBox;
        tma_2d(dst, &tmX, i * kGK, rowA, full + 8 * s);
        tma_2d(dst + kGBox, &tmX, i * kGK, rowB, full + 8 * s);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      for (int i = 0; i < k_tiles; ++i) {
        const int s = i % kGStages;
        bar_wait(full + 8 * s, (i / kGStages) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t a = base + s * 2 * kGBox, b = a + kGBox;
#pragma unroll
        for (int kk = 0; kk < kGK / 16; ++kk) {
          const uint32_t acc = (i | kk) != 0;
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
              "l"(kmajor_sw128(a + kk * 32)), "l"(kmajor_sw128(b + kk * 32)), "r"(kGIdesc),
              "r"(acc));
        }
        asm volatile(
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                empty + 8 * s)
            : "memory");
      }
      asm volatile(
          "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(done)
          : "memory");
    }
    __syncwarp();
  } else {
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;
    bar_wait(done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    float* dst = out + (size_t(batch) * rows_pad + mb * kGM + r) * rows_pad + nb * kGM;
    for (int c = 0; c < 4; ++c) {
      uint32_t v[32];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
          "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
            "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
            "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
            "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
            "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
            "=r"(v[31])
          : "r"(tmem + (uint32_t(q4 * 32) << 16) + c * 32));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        *reinterpret_cast<float4*>(dst + c * 32 + j) =
            make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]),
                        __uint_as_float(v[j + 2]), __uint_as_float(v[j + 3]));
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

// X[batch][set][pos] = 1.0 (bf16) for every selected position of the set.
__global__ void scatter_indicator_kernel(const uint32_t* __restrict__ sel,
                                         const uint32_t* __restrict__ counts, int sets,
                                         int k_stride, int rows_pad, int cols_pad,
                                         __nv_bfloat16* __restrict__ X) {
  const int set = blockIdx.x, batch = blockIdx.y;
  const uint32_t c = counts[size_t(batch) * sets + set];
  const uint32_t* src = sel + (size_t(batch) * sets + set) * k_stride;
  __nv_bfloat16* row = X + (size_t(batch) * rows_pad + set) * cols_pad;
  const __nv_bfloat16 one = __float2bfloat16_rn(1.f);
  for (uint32_t i = threadIdx.x; i < c; i += blockDim.x) {
    const uint32_t p = src[i];
    if (int(p) < cols_pad) row[p] = one;
  }
}

}  // namespace

int launch_gram(const uint32_t* sel, const uint32_t* counts, int n_batches, int sets,
                int k_stride, int n_positions, float* gram, cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    HC_CUDA_TRY(cudaFuncSetAttribute(gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kGSmem));
    configured = true;
  }
  const int rows_pad = (sets + kGM - 1) / kGM * kGM;
  const int cols_pad = (n_positions + kGK - 1) / kGK * kGK;
  const size_t xbytes = size_t(n_batches) * rows_pad * cols_pad * 2;
  __nv_bfloat16* X = nullptr;
  HC_CUDA_TRY(cudaMallocAsync((void**)&X, xbytes, st));
  HC_CUDA_TRY(cudaMemsetAsync(X, 0, xbytes, st));
  scatter_indicator_kernel<<<dim3(sets, n_batches), 256, 0, st>>>(sel, counts, sets, k_stride,
                                                                 rows_pad, cols_pad, X);
  HC_CHECK_LAUNCH();
  CUtensorMap tm;
  HC_TRY(make_bf16_tensor_map(&tm, X, int64_t(n_batches) * rows_pad, cols_pad, kGK, kGM));
  const int mt = rows_pad / kGM;
  gram_kernel<<<dim3(mt, mt, n_batches), kGThreads, kGSmem, st>>>(tm, rows_pad, cols_pad / kGK,
                                                                  gram);
  HC_CHECK_LAUNCH();
  HC_CUDA_TRY(cudaFreeAsync(X, st));
  return HC_OK;
}

}  // namespace hc

extern "C" int hc_gram_from_sets(const uint32_t* sel_dev, const uint32_t* counts_dev,
                                 int32_t n_batches, int32_t sets, int32_t k_stride,
                                 int32_t n_positions, float* gram_dev, void* stream) {
  HC_REQUIRE(sel_dev && counts_dev && gram_dev && n_batches > 0 && sets > 0 && n_positions > 0,
             HC_EINVAL, "hc_gram_from_sets: bad arguments");
  HC_REQUIRE(n_positions < (1 << 24), HC_EINVAL, "counts must stay exact in fp32 (< 2^24)");
  return hc::launch_gram(sel_dev, counts_dev, n_batches, sets, k_stride, n_positions, gram_dev,
                         (cudaStream_t)stream);
}
