/* Host twin of the bench's counter-based generator (csrc/synth.cu).
 *
 * TEST / BASELINE INFRASTRUCTURE: used by the CPU arms of bench.py (the
 * reference arm and the cpu_baseline leg) and by tests/ to regenerate,
 * bit for bit, the synthetic K/V/Q the GPU arm decodes.  Not part of the
 * product path.  Built by oracle/build_oracle.py into oracle/liboracle.so.
 *
 * Compile with contraction off (-ffp-contract=off): every step is exact or
 * one IEEE rounding, exactly as the CUDA kernel's __fadd_rn / __fmul_rn.
 */
#include <stdint.h>

static inline uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

void oracle_synth_normal(float* out, int64_t n, uint64_t key, int64_t offset) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    const uint64_t h = splitmix64(key + (uint64_t)(offset + i));
    const float u0 = (float)(uint32_t)(h & 0xffffu), u1 = (float)(uint32_t)((h >> 16) & 0xffffu);
    const float u2 = (float)(uint32_t)((h >> 32) & 0xffffu), u3 = (float)(uint32_t)(h >> 48);
    const float a = u0 + u1, b = u2 + u3;
    const float s = (a + b) * 1.52587890625e-05f;
    const float c = s - 1.999969482421875f;
    out[i] = c * 1.7320508075688772f;
  }
}
