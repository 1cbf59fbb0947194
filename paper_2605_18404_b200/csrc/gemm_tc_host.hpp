// gemm_tc_host.hpp — host side of gemm_tc.cuh: SWIZZLE_128B tensor maps
// (cuTensorMapEncodeTiled through the runtime's driver entry point, so the
// library needs no -lcuda) and the launchers.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <string>

#include "../../include/janus/errors.hpp"
#include "cuda_check.hpp"
#include "gemm_tc.cuh"

namespace janus {
namespace gemm_tc {

// [rows x K] fp32 row-major at base, boxes of 32 floats x box_rows rows, SW128
inline CUtensorMap make_tmap(const float* base, int rows, int K, int box_rows) {
  using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                              const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Encode enc = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn ||
        q != cudaDriverEntryPointSuccess)
      throw cuda_error("cuTensorMapEncodeTiled is unavailable");
    return reinterpret_cast<Encode>(fn);
  }();
  if (K % kKB || rows < 1 || box_rows < 1 || box_rows > 256) throw domain_error("gemm_tc: bad tensor map shape");
  CUtensorMap m;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(K) * sizeof(float)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(kKB), static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw cuda_error("cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
  return m;
}

// D = A . W^T: A [rows or 2P x K] (map with box rows 128 plain / 16 pair),
// W [N x K] (box rows N); one 128-row tile per CTA
template <class Epi>
void launch(const CUtensorMap& tmA, const CUtensorMap& tmW, const Problem& pb, const Epi& epi, cudaStream_t s) {
  if (pb.K % kKB || (pb.N != 64 && pb.N != 128 && pb.N != 256)) throw domain_error("gemm_tc: unsupported K / N");
  const int tiles = pb.pair ? (pb.rows + 63) / 64 : (pb.rows + 127) / 128;
  if (tiles <= 0) return;
  static bool attr = false;
  if (!attr) {
    JANUS_CUDA(cudaFuncSetAttribute(gemm_nt_kernel<Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem_bytes(256, 1))));
    attr = true;
  }
  janus::pdl(gemm_nt_kernel<Epi>, tiles, kThreads, smem_bytes(pb.N, pb.split3), s)(tmA, tmW, pb, epi);
  JANUS_LAUNCH_CHECK("gemm_tc");
}

}  // namespace gemm_tc
}  // namespace janus
