// Counter-based synthetic workload generator (bench inputs).
//
// out[i] = N(key, offset + i): splitmix64 of the counter, its four 16-bit
// fields as uniforms on the 2^-16 grid, summed (exact: 18 significant bits),
// centred exactly and scaled by sqrt(3) (one fp32 rounding): an Irwin-Hall(4)
// approximation of N(0, 1).  Every operation is exact or a single IEEE
// rounding with contraction disabled, so the host twin
// (oracle/synth.c, used by the CPU arms) produces bit-identical values and
// both bench arms decode the same K/V/Q.  Any element can be generated
// independently, so a CPU sample of sequences reproduces exactly the slice of
// the GPU's batch.

#include "hc_common.cuh"

namespace hc {
namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__global__ void synth_normal_kernel(float* __restrict__ out, int64_t n, uint64_t key,
                                    int64_t offset) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t h = splitmix64(key + uint64_t(offset + i));
    const float u0 = float(uint32_t(h & 0xffffu)), u1 = float(uint32_t((h >> 16) & 0xffffu));
    const float u2 = float(uint32_t((h >> 32) & 0xffffu)), u3 = float(uint32_t(h >> 48));
    // (u0 + u1) + (u2 + u3) on the integer grid is exact; scale by 2^-16 exact
    const float s = __fmul_rn(__fadd_rn(__fadd_rn(u0, u1), __fadd_rn(u2, u3)), 1.52587890625e-05f);
    out[i] = __fmul_rn(__fsub_rn(s, 1.999969482421875f), 1.7320508075688772f);
  }
}

// Read-only streaming probe: every 16-byte word of buf once (non-coherent,
// no L1 allocation, 4 independent loads in flight per thread), folded into
// one XOR per CTA so the loads are live.  bench.py times it beside K4 as the
// read-only denominator of the roofline (the copy peak in MEASURED_PEAKS.json
// moves read+write traffic, which a read-mostly kernel can exceed).
__global__ void __launch_bounds__(256) read_probe_kernel(const uint4* __restrict__ buf, int64_t n,
                                                         uint32_t* __restrict__ sink) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  uint32_t acc = 0;
  for (; i + 3 * stride < n; i += 4 * stride) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                   : "l"(buf + i + u * stride));
#pragma unroll
    for (int u = 0; u < 4; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  for (; i < n; i += stride) {
    const uint4 v = buf[i];
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  for (int o = 16; o; o >>= 1) acc ^= __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ uint32_t red[8];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t a = 0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) a ^= red[w];
    sink[blockIdx.x] = a;
  }
}

}  // namespace
}  // namespace hc

extern "C" int hc_read_probe(const void* buf_dev, int64_t bytes, uint32_t* sink_dev,
                             int32_t ctas, void* stream) {
  HC_REQUIRE(buf_dev && sink_dev && ctas > 0 && bytes >= 0 && bytes % 16 == 0, HC_EINVAL,
             "read probe: bad arguments");
  hc::read_probe_kernel<<<ctas, 256, 0, (cudaStream_t)stream>>>((const uint4*)buf_dev,
                                                                 bytes / 16, sink_dev);
  HC_CHECK_LAUNCH();
  return HC_OK;
}

extern "C" int hc_synth_normal(float* out_dev, int64_t n, uint64_t key, int64_t offset,
                               void* stream) {
  HC_REQUIRE(out_dev || n == 0, HC_EINVAL, "null output");
  if (n <= 0) return HC_OK;
  const int64_t blocks = (n + 255) / 256;
  hc::synth_normal_kernel<<<int(blocks < 148 * 32 ? blocks : 148 * 32), 256, 0,
                            (cudaStream_t)stream>>>(out_dev, n, key, offset);
  HC_CHECK_LAUNCH();
  return HC_OK;
}
