// tc_probe.cu — self-test of the tcgen05 layer (tc.cuh).  Test infrastructure
// exposed through the C ABI (janus_tc_probe) so tests/test_gpu_tc.py can
// validate descriptor encodings and TMEM accumulator layouts on the B200.
// One CTA: A tile [a_rows x a_cols] and B tile [b_rows x b_cols] (row-major
// fp32 in global) are staged into core-matrix smem tiles, K/8 kind::tf32 MMAs
// run with K-major (rows = M|N, cols = K) or MN-major (rows = K, cols = M|N)
// descriptors, and the raw TMEM image (128 lanes x N columns) is returned.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "../../include/janus/errors.hpp"
#include "cuda_check.hpp"
#include "tc.cuh"
#include "gemm_tc_host.hpp"

namespace janus {
namespace {

struct ProbeArgs {
  int M, N, K, a_mn, b_mn, a_rows, a_cols, b_rows, b_cols, swap, layout;
};

__global__ void __launch_bounds__(128) tc_probe_kernel(ProbeArgs p, const float* __restrict__ A, const float* __restrict__ B,
                                                       float* __restrict__ D) {
  extern __shared__ __align__(1024) float dyn[];  // 1024 B aligned for SWIZZLE_128B
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  float* sa = dyn;
  float* sb = dyn + p.a_rows * p.a_cols;
  const int t = threadIdx.x, warp = t >> 5;
  char* pa = reinterpret_cast<char*>(sa);
  char* pb = reinterpret_cast<char*>(sb);
  const bool sw = p.layout == 2;
  if (p.layout == 3) {  // bf16 SWIZZLE_128B tiles, kind::f16 (K-step 16)
    for (int x = t; x < p.a_rows * p.a_cols; x += 128) {
      const int r = x / p.a_cols, c = x % p.a_cols;
      *reinterpret_cast<__nv_bfloat16*>(pa + tc::sw128_off_b16(r, c, p.a_rows)) = __float2bfloat16_rn(A[x]);
    }
    for (int x = t; x < p.b_rows * p.b_cols; x += 128) {
      const int r = x / p.b_cols, c = x % p.b_cols;
      *reinterpret_cast<__nv_bfloat16*>(pb + tc::sw128_off_b16(r, c, p.b_rows)) = __float2bfloat16_rn(B[x]);
    }
  }
  for (int x = t; x < p.a_rows * p.a_cols && p.layout != 3; x += 128) {
    const int r = x / p.a_cols, c = x % p.a_cols;
    *reinterpret_cast<float*>(pa + (sw ? tc::sw128_off(r, c, p.a_rows) : tc::core_off(r, c, p.a_cols))) = A[x];
  }
  for (int x = t; x < p.b_rows * p.b_cols && p.layout != 3; x += 128) {
    const int r = x / p.b_cols, c = x % p.b_cols;
    *reinterpret_cast<float*>(pb + (sw ? tc::sw128_off(r, c, p.b_rows) : tc::core_off(r, c, p.b_cols))) = B[x];
  }
  if (t == 0) tc::mbar_init(&mbar, 1);
  if (warp == 0) tc::tmem_alloc(&tmem_base, 128);
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;
  if (t == 0) {
    const uint32_t a0 = tc::smem_u32(sa), b0 = tc::smem_u32(sb);
    if (p.layout == 3) {
      // K-major: rows = M|N, K along 64-col slabs: k-step s (16) -> slab s/4, +32 B inside the row
      // MN-major: rows = K: k-step of 16 rows -> +2048 B; one 64-wide MN slab (LBO unused: rows*128)
      const uint32_t id16 = tc::idesc_bf16(p.M, p.N, p.a_mn, p.b_mn);
      const uint32_t a_slab = p.a_rows * 128, b_slab = p.b_rows * 128;
      for (int s = 0; s < p.K / 16; ++s) {
        const uint64_t da = p.a_mn ? tc::smem_desc(a0 + 2048 * s, a_slab, 1024, 2)
                                   : tc::smem_desc(a0 + (s >> 2) * a_slab + 32 * (s & 3), 16, 1024, 2);
        const uint64_t db = p.b_mn ? tc::smem_desc(b0 + 2048 * s, b_slab, 1024, 2)
                                   : tc::smem_desc(b0 + (s >> 2) * b_slab + 32 * (s & 3), 16, 1024, 2);
        tc::mma_bf16(tmem, da, db, id16, s > 0);
      }
      tc::commit(&mbar);
    }
    const uint32_t id = tc::idesc_tf32(p.M, p.N, p.a_mn, p.b_mn);
    const uint32_t a_grp = (p.a_cols / 4) * 128, b_grp = (p.b_cols / 4) * 128;
    for (int s = 0; s < p.K / 8 && p.layout != 3; ++s) {
      if (sw) {
        // K-major: rows = M|N, K along the 32-col slabs: k-step s -> slab s/4, +32 B inside the row
        // MN-major: rows = K: k-step of 8 rows -> +1024 B; MN slabs of 32 at LBO = rows*128
        const uint32_t a_slab = p.a_rows * 128, b_slab = p.b_rows * 128;
        const uint64_t da = p.a_mn ? tc::smem_desc(a0 + 1024 * s, a_slab, 1024, 2)
                                   : tc::smem_desc(a0 + (s >> 2) * a_slab + 32 * (s & 3), 16, 1024, 2);
        const uint64_t db = p.b_mn ? tc::smem_desc(b0 + 1024 * s, b_slab, 1024, 2)
                                   : tc::smem_desc(b0 + (s >> 2) * b_slab + 32 * (s & 3), 16, 1024, 2);
        tc::mma_tf32(tmem, da, db, id, s > 0);
        continue;
      }
      const uint32_t al = p.swap ? 128 : a_grp, as = p.swap ? a_grp : 128;
      const uint32_t bl = p.swap ? 128 : b_grp, bs = p.swap ? b_grp : 128;
      const uint64_t da = p.a_mn ? tc::smem_desc(a0 + a_grp * s, al, as) : tc::smem_desc(a0 + 256 * s, 128, a_grp);
      const uint64_t db = p.b_mn ? tc::smem_desc(b0 + b_grp * s, bl, bs) : tc::smem_desc(b0 + 256 * s, 128, b_grp);
      tc::mma_tf32(tmem, da, db, id, s > 0);
    }
    if (p.layout != 3) tc::commit(&mbar);
  }
  tc::mbar_wait(&mbar, 0);
  tc::fence_after();
  float v[32];
  for (int c0 = 0; c0 < p.N; c0 += 32) {
    tc::ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
    for (int i = 0; i < 32; ++i) D[t * p.N + c0 + i] = v[i];
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free(tmem, 128);
}

}  // namespace

void tc_probe(const int* args, const float* A, const float* B, float* D) {
  ProbeArgs p{args[0], args[1], args[2], args[3], args[4], args[5], args[6], args[7], args[8], args[9], args[10]};
  if (p.N % 32 || p.N > 128 || p.K % 8 || (p.M != 64 && p.M != 128)) throw domain_error("tc_probe: bad shape");
  const size_t na = static_cast<size_t>(p.a_rows) * p.a_cols, nb = static_cast<size_t>(p.b_rows) * p.b_cols;
  float *dA, *dB, *dD;
  JANUS_CUDA(cudaMalloc(&dA, na * 4));
  JANUS_CUDA(cudaMalloc(&dB, nb * 4));
  JANUS_CUDA(cudaMalloc(&dD, 128 * p.N * 4));
  JANUS_CUDA(cudaMemcpy(dA, A, na * 4, cudaMemcpyHostToDevice));
  JANUS_CUDA(cudaMemcpy(dB, B, nb * 4, cudaMemcpyHostToDevice));
  const int smem = static_cast<int>((na + nb) * 4);
  JANUS_CUDA(cudaFuncSetAttribute(tc_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  tc_probe_kernel<<<1, 128, smem>>>(p, dA, dB, dD);
  JANUS_LAUNCH_CHECK("tc_probe");
  JANUS_CUDA(cudaDeviceSynchronize());
  JANUS_CUDA(cudaMemcpy(D, dD, 128 * p.N * 4, cudaMemcpyDeviceToHost));
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
}

// gemm_tc.cuh self-test: D = A . W^T through the TMA + tcgen05 pipeline with
// the plain store epilogue.  mode bit 0 = pair (A and D stacked [2P x K] /
// [2P x N]), bit 1 = 3xTF32 split (Problem::split3).
void gemm_tc_probe(int rows, int K, int N, int mode, const float* A, const float* W, float* D) {
  const int pair = mode & 1;
  const int arows = pair ? 2 * rows : rows;
  float *dA, *dW, *dD;
  JANUS_CUDA(cudaMalloc(&dA, sizeof(float) * arows * K));
  JANUS_CUDA(cudaMalloc(&dW, sizeof(float) * N * K));
  JANUS_CUDA(cudaMalloc(&dD, sizeof(float) * arows * N));
  JANUS_CUDA(cudaMemcpy(dA, A, sizeof(float) * arows * K, cudaMemcpyHostToDevice));
  JANUS_CUDA(cudaMemcpy(dW, W, sizeof(float) * N * K, cudaMemcpyHostToDevice));
  JANUS_CUDA(cudaMemset(dD, 0, sizeof(float) * arows * N));
  const CUtensorMap ta = gemm_tc::make_tmap(dA, arows, K, pair ? 16 : 128);
  const CUtensorMap tw = gemm_tc::make_tmap(dW, N, K, N);
  gemm_tc::launch(ta, tw, gemm_tc::Problem{rows, K, N, pair, (mode >> 1) & 1}, gemm_tc::EpiStore{dD, N}, nullptr);
  JANUS_CUDA(cudaDeviceSynchronize());
  JANUS_CUDA(cudaMemcpy(D, dD, sizeof(float) * arows * N, cudaMemcpyDeviceToHost));
  cudaFree(dA);
  cudaFree(dW);
  cudaFree(dD);
}

}  // namespace janus
