// cuda_check.hpp — host-side CUDA error checking that throws (caught at the C ABI).
#pragma once

#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

namespace janus {

struct cuda_error : std::runtime_error {
  explicit cuda_error(const std::string& m) : std::runtime_error(m) {}
};

/// NCCL failures (executor transports); mapped to janus::kNcclError at the ABI.
struct nccl_error : std::runtime_error {
  explicit nccl_error(const std::string& m) : std::runtime_error(m) {}
};

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw cuda_error(std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace janus

#define JANUS_CUDA(x) ::janus::cuda_check((x), #x)
#define JANUS_LAUNCH_CHECK(name) ::janus::cuda_check(cudaGetLastError(), name)
