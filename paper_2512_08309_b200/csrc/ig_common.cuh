// Shared helpers for the infigrid_b200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string>

#include "../../include/infigrid_b200.h"

namespace ig {

// thread-local error message behind ig_last_error()
void set_error(const char* fmt, ...);

// process-wide count of kernels this library launched (ig_launch_count)
void note_launch();

inline int cuda_check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return IG_ERR_CUDA;
  }
  return IG_OK;
}

#define IG_REQUIRE(cond, ...)          \
  do {                                 \
    if (!(cond)) {                     \
      ::ig::set_error(__VA_ARGS__);    \
      return IG_ERR_ARG;               \
    }                                  \
  } while (0)

constexpr int kNumSMs = 148;

// grid for a grid-stride loop over n items with `threads` per CTA:
// enough CTAs to cover n, capped at a few waves of the 148 SMs
inline int grid_for(int64_t n, int threads, int waves = 16) {
  int64_t need = (n + threads - 1) / threads;
  int64_t cap = (int64_t)kNumSMs * waves;
  if (need < 1) need = 1;
  return (int)(need < cap ? need : cap);
}

// Python floor division / modulo for a positive divisor
__host__ __device__ __forceinline__ int64_t floordiv(int64_t a, int64_t b) {
  int64_t q = a / b;
  return (q * b != a && a < 0) ? q - 1 : q;
}
__host__ __device__ __forceinline__ int64_t ceildiv(int64_t a, int64_t b) {
  return -floordiv(-a, b);
}
__host__ __device__ __forceinline__ int64_t pymod(int64_t a, int64_t b) {
  return a - floordiv(a, b) * b;
}

// exact-rounding arithmetic in the element type (no FMA contraction)
__device__ __forceinline__ float radd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float rsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float rmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float rdiv(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double radd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double rsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double rmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double rdiv(double a, double b) { return __ddiv_rn(a, b); }

}  // namespace ig
