// Shared helpers for the HeteroCache B200 kernels (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/hcb200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "HeteroCache-B200 kernels are written for sm_100a only"
#endif

namespace hc {

// Thread-local last-error message, surfaced through hc_last_error().
void set_error(const char* fmt, ...);

#define HC_CUDA_TRY(expr)                                                      \
  do {                                                                         \
    cudaError_t _e = (expr);                                                   \
    if (_e != cudaSuccess) {                                                   \
      ::hc::set_error("%s:%d %s -> %s", __FILE__, __LINE__, #expr,             \
                      cudaGetErrorString(_e));                                 \
      return HC_ECUDA;                                                         \
    }                                                                          \
  } while (0)

// Every kernel launch is followed by HC_CHECK_LAUNCH(), which also counts it
// (hc_launch_count(): the bench reports how many of our kernels ran).
void count_launch();

#define HC_CHECK_LAUNCH()                                                      \
  do {                                                                         \
    ::hc::count_launch();                                                      \
    cudaError_t _e = cudaGetLastError();                                       \
    if (_e != cudaSuccess) {                                                   \
      ::hc::set_error("%s:%d launch -> %s", __FILE__, __LINE__,                \
                      cudaGetErrorString(_e));                                 \
      return HC_ECUDA;                                                         \
    }                                                                          \
  } while (0)

#define HC_REQUIRE(cond, code, ...)                                            \
  do {                                                                         \
    if (!(cond)) {                                                             \
      ::hc::set_error(__VA_ARGS__);                                            \
      return (code);                                                           \
    }                                                                          \
  } while (0)

#define HC_TRY(x)                                                              \
  do {                                                                         \
    int _rc = (x);                                                             \
    if (_rc != HC_OK) return _rc;                                              \
  } while (0)
#define HC_TRY_RC(x) HC_TRY(x)

// Order-preserving map of an fp32 score to uint32 (larger score -> larger
// key).  -0.0 is folded onto +0.0 so that equal scores tie exactly as they
// do under Python float comparison (metrics.py:44 sorts on -score).
__device__ __forceinline__ uint32_t score_key(float f) {
  uint32_t u = __float_as_uint(f);
  if (u == 0x80000000u) u = 0u;
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__host__ __device__ __forceinline__ uint32_t ceil_div_u32(uint32_t a, uint32_t b) {
  return (a + b - 1) / b;
}

// Fire selection job (engine fire_batch -> fire_select_kernel): top-k of a
// dense pivot row whose 13-bit first-digit key histogram is already known.
struct FireJob {
  const float* row;       // [n] probability row
  const uint32_t* hist;   // [8192] histogram of score_key(row) >> 19
  uint32_t n, k;
  uint32_t* out_idx;      // [k] selected positions, ascending
  uint32_t* out_count;
  uint32_t* host_out;     // device decisions: copy_fetched_kernel copies the selection here
                          // (mapped host ring), off the gathers' critical path
  int32_t* state_out;     // optional: set to 2 (devdec.cuh kXSelected) once written
};

}  // namespace hc
