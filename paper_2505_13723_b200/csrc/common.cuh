// Shared device helpers for the sapgp_b200 kernels (sm_100a).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/sapgp_b200.h"

namespace sap {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kSqrt3 = 1.7320508075688772f;
constexpr float kSqrt5 = 2.2360679774997896f;

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float rsqrt_approx(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Unit-variance kernel value from a squared scaled distance (kernels.py:56-66).
// The clamp at zero happens here; callers multiply by the variance once per
// output (the sum is linear in it).
template <int FAM>
__device__ __forceinline__ float kernel_value(float sq) {
  sq = fmaxf(sq, 0.0f);
  if constexpr (FAM == SAP_RBF) {
    return ex2_approx(sq * (-0.5f * kLog2e));
  } else if constexpr (FAM == SAP_MATERN32) {
    const float a = kSqrt3 * sqrt_approx(sq);
    return (1.0f + a) * ex2_approx(-a * kLog2e);
  } else {
    const float a = kSqrt5 * sqrt_approx(sq);
    return fmaf(5.0f / 3.0f, sq, 1.0f + a) * ex2_approx(-a * kLog2e);
  }
}

}  // namespace sap
