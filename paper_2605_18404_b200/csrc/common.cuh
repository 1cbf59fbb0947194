// common.cuh — shared device helpers for the janus sm_100a kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <utility>

#include "cuda_check.hpp"

// Programmatic dependent launch.  Every kernel of the stage chain starts with
// JANUS_GDC_WAIT() (griddepcontrol.wait: returns once the previous kernel on
// the stream has completed and its writes are visible; a no-op for a normal
// launch), and stage.cu launches them through janus::pdl(...) with
// programmatic stream serialization, so a kernel's CTAs are scheduled and
// resident when its predecessor's last CTA exits instead of after the
// predecessor's completion round trip.  The wait is the FIRST statement of
// every such kernel (before any early return), so completion stays transitive
// along the stream: nothing a kernel does precedes its predecessor's end.
// (Each micro-batch lane is a chain of ~70 dependent, latency-bound kernels.)
#if defined(__CUDA_ARCH__) && defined(JANUS_PDL_EARLY)
// (A/B variant: also release the dependent grid at once, so its CTAs are
// resident and waiting while this grid runs)
#define JANUS_GDC_WAIT() asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory")
#elif defined(__CUDA_ARCH__)
#define JANUS_GDC_WAIT() asm volatile("griddepcontrol.wait;" ::: "memory")
#else
#define JANUS_GDC_WAIT()
#endif

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

// janus::pdl(kernel, grid, block, smem, stream)(args...): the <<<>>> launch
// with programmatic stream serialization (build with -DJANUS_NO_PDL for plain
// launches).  Arguments are coerced to the kernel's parameter types exactly as
// a <<<>>> launch does (cudaLaunchKernelEx's typed overload).
template <typename... P>
struct PdlLaunch {
  void (*k)(P...);
  cudaLaunchConfig_t cfg;
  cudaLaunchAttribute at;
  template <typename... A>
  void operator()(A&&... a) {
#ifndef JANUS_NO_PDL
    at.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at.val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = &at;
    cfg.numAttrs = 1;
#else
    cfg.attrs = nullptr;
    cfg.numAttrs = 0;
#endif
    JANUS_CUDA(cudaLaunchKernelEx(&cfg, k, std::forward<A>(a)...));  // a failed launch throws (cuda_error)
  }
};
template <typename... P>
PdlLaunch<P...> pdl(void (*k)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t s) {
  PdlLaunch<P...> l{};
  l.k = k;
  l.cfg.gridDim = grid;
  l.cfg.blockDim = block;
  l.cfg.dynamicSmemBytes = smem;
  l.cfg.stream = s;
  return l;
}

}  // namespace janus
