// Shared helpers for the sm_100a ISAAC path: status plumbing and float
// arithmetic with explicit rounding (no FMA contraction where the reference's
// numpy evaluation order must be reproduced bit-for-bit).
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include <string>

#include "isaac_b200.h"

namespace isc {

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define ISC_CUDA_CHECK(expr)                         \
  do {                                               \
    cudaError_t _e = (expr);                         \
    if (_e != cudaSuccess) return isc::cuda_fail(_e, #expr); \
  } while (0)

// ---- float64 with explicit round-to-nearest (numpy semantics, no FMA) ----
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
// numpy.maximum / minimum on non-NaN inputs
__device__ __forceinline__ double dmax(double a, double b) { return a > b ? a : b; }
__device__ __forceinline__ double dmin(double a, double b) { return a < b ? a : b; }

// ---- float32 with explicit rounding (bit-exact min/max oracle) ----
__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }

__device__ __forceinline__ float4 over4(float4 f, float4 b) {
  // premultiplied over (compositing.py:25-33): C = C_f + (1 - A_f) C_b
  const float k = 1.0f - f.w;
  return make_float4(fmaf(k, b.x, f.x), fmaf(k, b.y, f.y), fmaf(k, b.z, f.z), fmaf(k, b.w, f.w));
}

}  // namespace isc
