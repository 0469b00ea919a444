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

}  // namespace
}  // namespace hc

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
