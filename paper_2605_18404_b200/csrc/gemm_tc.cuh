// gemm_tc.cuh — TMA-fed tcgen05 GEMM with fused epilogues for the
// generic-width path (stage_wide.inc): D[rows x N] = A[rows x K] . W^T with
// A fp32 row-major (K-major) in global memory and W the weight as a K-major
// [N x K] fp32 matrix, tf32 tensor-core math, fp32 accumulate in TMEM.
//
// Warp roles (256 threads): warp 0 issues the TMA loads (cp.async.bulk.tensor
// with SWIZZLE_128B tensor maps: each 32-float K block of A and W lands in the
// canonical SW128 K-major slab the UMMA descriptor reads), warp 1 issues the
// MMAs (one elected thread, M=128 x N x K=8 tf32 per instruction) and frees a
// pipeline stage with tcgen05.commit, warps 4-7 are the epilogue (thread =
// tile row = TMEM lane; 32-column tcgen05.ld chunks).
//
// Pair mode.  The per-pair operands are stacked [value rows; derivative rows]
// (rows p and P + p belong to pair p).  A pair-mode tile takes 64 pairs: the
// value rows land in smem rows 0..63 and the derivative rows in 64..127 (two
// TMA boxes), so TMEM lanes l and l + 64 hold one pair's value and radial
// derivative, and the epilogue combines them through a shared-memory swap —
// the elementwise steps that need both (SiLU and SiLU'·z', the filter w, w',
// zbar) run in the GEMM's epilogue instead of a separate pass over HBM.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "tc.cuh"

namespace janus {
namespace gemm_tc {

constexpr int kThreads = 256;
constexpr int kKB = 32;  // floats per K block (one 128 B SW128 slab)

struct Problem {
  int rows;      // plain mode: rows of A / D; pair mode: pairs P (A, D have 2P rows)
  int K;         // multiple of 32
  int N;         // 64, 128 or 256 (one N tile)
  int pair;      // 1: pair-mode tiles (64 pairs = 128 rows)
};

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint64_t* mbar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(tc::smem_u32(mbar))
      : "memory");
}

// ----------------------------------------------------------------- epilogues
// Each functor sees, per 32-column chunk, this thread's accumulator row and
// (pair mode) the partner row (value <-> derivative), and writes its outputs.
// Row indices: plain: r = tile row; pair: p = pair, half = 0 value / 1 deriv.
struct EpiStore {  // D = the accumulator (pair mode: stacked like A)
  float* D;
  int ld;
  __device__ void operator()(int rows_total, int p, int half, int P, int c0, const float (&own)[32], const float (&)[32]) const {
    if (p >= rows_total) return;  // plain tiles past the last row
    const int r = half ? P + p : p;
    float4* o = reinterpret_cast<float4*>(D + static_cast<size_t>(r) * ld + c0);
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = make_float4(own[4 * j], own[4 * j + 1], own[4 * j + 2], own[4 * j + 3]);
  }
};

// [z; z'] -> a2 = [SiLU(z + alpha); SiLU'(z + alpha) z']  (+ the raw z2 when asked)
struct EpiAct2 {
  float* a2;
  float* z2;  // optional raw copy (BF needs z, z' again for zbar)
  const float* alpha;
  int ld;
  __device__ void operator()(int, int p, int half, int P, int c0, const float (&own)[32], const float (&oth)[32]) const {
    const int r = half ? P + p : p;
    float o[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float zz = (half ? oth[j] : own[j]) + __ldg(alpha + c0 + j);
      o[j] = half ? dev::dsilu(zz) * own[j] : dev::silu(zz);
    }
    float4* d = reinterpret_cast<float4*>(a2 + static_cast<size_t>(r) * ld + c0);
#pragma unroll
    for (int j = 0; j < 8; ++j) d[j] = make_float4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
    if (z2) {
      float4* z = reinterpret_cast<float4*>(z2 + static_cast<size_t>(r) * ld + c0);
#pragma unroll
      for (int j = 0; j < 8; ++j) z[j] = make_float4(own[4 * j], own[4 * j + 1], own[4 * j + 2], own[4 * j + 3]);
    }
  }
};

// [g; g'] -> w = c (g + beta), w' = c' (g + beta) + c g'   ([P][N] each)
struct EpiFilter {
  float* wf;
  float* wfp;
  const float* beta;
  const float4* pgeo;  // (d, c, c', i | u, j) per pair
  int ld;
  __device__ void operator()(int, int p, int half, int, int c0, const float (&own)[32], const float (&oth)[32]) const {
    const float4 g0 = __ldg(pgeo + 2 * p);
    float o[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float g = (half ? oth[j] : own[j]) + __ldg(beta + c0 + j);
      o[j] = half ? g0.z * g + g0.y * own[j] : g0.y * g;
    }
    float4* d = reinterpret_cast<float4*>((half ? wfp : wf) + static_cast<size_t>(p) * ld + c0);
#pragma unroll
    for (int j = 0; j < 8; ++j) d[j] = make_float4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
  }
};

// [sbar; sdotbar] (+ raw [z; z']) -> [zbar; zbar'] = [sbar SiLU'(z) + sdotbar SiLU''(z) z'; sdotbar SiLU'(z)]
struct EpiZbar {
  float* zb;
  const float* z2;
  const float* alpha;
  int ld;
  __device__ void operator()(int, int p, int half, int P, int c0, const float (&own)[32], const float (&oth)[32]) const {
    const float* zr = z2 + static_cast<size_t>(p) * ld + c0;
    const float* zpr = z2 + static_cast<size_t>(P + p) * ld + c0;
    float o[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float zz = __ldg(zr + j) + __ldg(alpha + c0 + j);
      const float ds = dev::dsilu(zz);
      o[j] = half ? own[j] * ds : own[j] * ds + oth[j] * dev::d2silu(zz) * __ldg(zpr + j);
    }
    float4* d = reinterpret_cast<float4*>(zb + static_cast<size_t>(half ? P + p : p) * ld + c0);
#pragma unroll
    for (int j = 0; j < 8; ++j) d[j] = make_float4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
  }
};

// plain: z -> a = SiLU(z + alpha) (+ raw z)
struct EpiAct1 {
  float* a;
  float* zraw;
  const float* alpha;
  int ld;
  __device__ void operator()(int rows, int r, int, int, int c0, const float (&own)[32], const float (&)[32]) const {
    if (r >= rows) return;
    float o[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) o[j] = dev::silu(own[j] + __ldg(alpha + c0 + j));
    float4* d = reinterpret_cast<float4*>(a + static_cast<size_t>(r) * ld + c0);
#pragma unroll
    for (int j = 0; j < 8; ++j) d[j] = make_float4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
    if (zraw) {
      float4* z = reinterpret_cast<float4*>(zraw + static_cast<size_t>(r) * ld + c0);
#pragma unroll
      for (int j = 0; j < 8; ++j) z[j] = make_float4(own[4 * j], own[4 * j + 1], own[4 * j + 2], own[4 * j + 3]);
    }
  }
};

// plain: sbar (+ raw z) -> zbar = sbar SiLU'(z + alpha)
struct EpiBeZbar {
  float* zb;
  const float* z;
  const float* alpha;
  int ld;
  __device__ void operator()(int rows, int r, int, int, int c0, const float (&own)[32], const float (&)[32]) const {
    if (r >= rows) return;
    const float* zr = z + static_cast<size_t>(r) * ld + c0;
    float o[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) o[j] = own[j] * dev::dsilu(__ldg(zr + j) + __ldg(alpha + c0 + j));
    float4* d = reinterpret_cast<float4*>(zb + static_cast<size_t>(r) * ld + c0);
#pragma unroll
    for (int j = 0; j < 8; ++j) d[j] = make_float4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
  }
};

// bytes of dynamic shared memory: STAGES x (A slab 16 KB + W slab N x 128 B) + swap buffer
constexpr size_t smem_bytes(int stages, int N) {
  return static_cast<size_t>(stages) * (128 * 128 + N * 128) + 128 * 33 * 4 + 1024;
}

template <int STAGES, class Epi>
__global__ void __launch_bounds__(kThreads, 1) gemm_nt_kernel(const __grid_constant__ CUtensorMap tmA,
                                                             const __grid_constant__ CUtensorMap tmW, Problem pb, Epi epi) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (tc::smem_u32(sm_raw) & 1023u)) & 1023u);
  const uint32_t slabA = 128 * 128, slabW = static_cast<uint32_t>(pb.N) * 128, stage_bytes = slabA + slabW;
  float* swap = reinterpret_cast<float*>(sm + STAGES * stage_bytes);  // [128][33]
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], accum;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KB = pb.K / kKB;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(&accum, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) tc::tmem_alloc(&tslot, static_cast<uint32_t>(pb.N < 32 ? 32 : pb.N));
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tslot;
  // tile rows: plain rows [128 t, 128 t + 128); pair: pairs [64 t, 64 t + 64) -> value rows, then P + those
  const int t = blockIdx.x;
  if (warp == 0 && lane == 0) {  // TMA producer
    for (int kb = 0; kb < KB; ++kb) {
      const int s = kb % STAGES;
      if (kb >= STAGES) tc::mbar_wait(&empty[s], ((kb / STAGES) - 1) & 1);
      tc::mbar_expect_tx(&full[s], stage_bytes);
      const uint32_t a = tc::smem_u32(sm + s * stage_bytes), w = a + slabA;
      if (pb.pair) {
        tma_load_2d(a, &tmA, kb * kKB, 64 * t, &full[s]);
        tma_load_2d(a + 64 * 128, &tmA, kb * kKB, pb.rows + 64 * t, &full[s]);
      } else {
        tma_load_2d(a, &tmA, kb * kKB, 128 * t, &full[s]);
      }
      tma_load_2d(w, &tmW, kb * kKB, 0, &full[s]);
    }
  } else if (warp == 1 && lane == 0) {  // MMA issuer
    const uint32_t idesc = tc::idesc_tf32(128, pb.N, false, false);
    for (int kb = 0; kb < KB; ++kb) {
      const int s = kb % STAGES;
      tc::mbar_wait(&full[s], (kb / STAGES) & 1);
      tc::fence_after();
      const uint32_t a = tc::smem_u32(sm + s * stage_bytes), w = a + slabA;
      const uint64_t da = tc::smem_desc(a, 16, 1024, 2), dw = tc::smem_desc(w, 16, 1024, 2);
#pragma unroll
      for (int k = 0; k < kKB / 8; ++k)  // K = 8 per instruction: +32 B inside the 128 B slab
        tc::mma_tf32(tmem, da + static_cast<uint64_t>((32 * k) >> 4), dw + static_cast<uint64_t>((32 * k) >> 4), idesc,
                     (kb > 0 || k > 0) ? 1u : 0u);
      tc::commit(&empty[s]);  // the stage is free once these MMAs have read it
    }
    tc::commit(&accum);
  } else if (warp >= 4) {  // epilogue: thread = tile row = TMEM lane
    const int row = threadIdx.x - 128;  // 0..127 (warp 4 -> lanes 0..31, ...)
    tc::mbar_wait(&accum, 0);
    tc::fence_after();
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const int half = pb.pair ? (row >> 6) : 0;
    const int p = pb.pair ? 64 * t + (row & 63) : 128 * t + row;
    const int partner = row ^ 64;
    for (int c0 = 0; c0 < pb.N; c0 += 32) {
      float own[32], oth[32];
      tc::ld32(tmem + lane_base + static_cast<uint32_t>(c0), own);
      if (pb.pair) {
        asm volatile("bar.sync 1, 128;" ::: "memory");  // the previous chunk's swap reads are done
#pragma unroll
        for (int j = 0; j < 32; ++j) swap[row * 33 + j] = own[j];
        asm volatile("bar.sync 1, 128;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 32; ++j) oth[j] = swap[partner * 33 + j];
        if (p < pb.rows) epi(pb.rows, p, half, pb.rows, c0, own, oth);
      } else {
        epi(pb.rows, p, 0, 0, c0, own, own);
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 2) tc::tmem_free(tmem, static_cast<uint32_t>(pb.N < 32 ? 32 : pb.N));
}

}  // namespace gemm_tc
}  // namespace janus
