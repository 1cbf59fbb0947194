// common.cuh — shared device helpers for the janus sm_100a kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "cuda_check.hpp"

namespace janus {
namespace dev {

constexpr float kPi = 3.14159265358979323846f;

__device__ __forceinline__ float sigm(float x) { return 1.0f / (1.0f + expf(-x)); }
__device__ __forceinline__ float silu(float x) { return x * sigm(x); }
__device__ __forceinline__ float dsilu(float x) {
  const float s = sigm(x);
  return s * (1.0f + x * (1.0f - s));
}
__device__ __forceinline__ float d2silu(float x) {
  const float s = sigm(x);
  return s * (1.0f - s) * (2.0f + x * (1.0f - 2.0f * s));
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace dev

}  // namespace janus
