// wgrad_tc.cuh — node-side weight gradients G = sum_i op(a_i)^T b_i
// (+ a2_i^T b2_i) of the upd / msg / readout units on 5th-gen tensor cores
// (the JANUS_PREC_TF32 path; the fp32 parity path keeps
// node_kernels.cuh wgrad_multi_kernel).  One CTA per job: 128-atom blocks of
// a and b are staged transposed ([64 features][128 atoms], SWIZZLE_128B
// K-major, the same layout as edge_tc.cuh's feature-major tiles) and
// contracted by M=64 x N=64 x K=128 kind::tf32 MMAs accumulating in TMEM in
// atom-block order — deterministic, one launch CTA instead of nine.
#pragma once

#include "edge_tc.cuh"
#include "geo_job.hpp"
#include "node_kernels.cuh"

namespace janus {
namespace edge_tc {

constexpr size_t wgrad_tc_smem() { return 2 * kTile + 1024; }

constexpr int kWgT = 512;  // threads: 4 float4 of a and of b per thread per 128-atom block

// Column sums of x1 / x2 (grid.y = 1 CTAs; they ran after the MMA loop, as
// 2 x 8 dependent L2 round trips, until round 2): thread = (matrix, row
// quarter, column), 16 loads in flight, each column summed in row order
// within its quarter and the quarters combined in a fixed order — the same
// sums as before, bit for bit.
__device__ __forceinline__ void colsums(int rows, const node::WJob& jb, float (*csp)[2][64]) {
  const int tid = static_cast<int>(threadIdx.x), w = tid >> 8, qr = (tid >> 6) & 3, c = tid & 63;
  const int r0 = (rows * qr) >> 2, r1 = (rows * (qr + 1)) >> 2;
  const float* X = w ? jb.x2 : jb.x1;
  float s = 0.f;
  if (X) {
    int i = r0;
    for (; i + 16 <= r1; i += 16) {
      float v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) v[u] = __ldg(X + (size_t)(i + u) * 64 + c);
#pragma unroll
      for (int u = 0; u < 16; ++u) s += v[u];
    }
    for (; i < r1; ++i) s += __ldg(X + (size_t)i * 64 + c);
  }
  csp[qr][w][c] = s;
  __syncthreads();
  if (tid < 128) {
    const int ww = tid >> 6, cc = tid & 63;
    float* out = ww ? jb.cs2 : jb.cs1;
    if ((ww ? jb.x2 : jb.x1) && out) out[cc] = (csp[0][ww][cc] + csp[1][ww][cc]) + (csp[2][ww][cc] + csp[3][ww][cc]);
  }
}

__global__ void __launch_bounds__(kWgT, 1) wgrad_tc_kernel(int rows, node::WJobs jobs) {
  JANUS_GDC_WAIT();
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = align1024(sm_raw);
  uint8_t* TA = sm;          // a^T [64 features][128 atoms]
  uint8_t* TB = TA + kTile;  // b^T
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tslot;
  __shared__ float csp[4][2][64];
  const node::WJob& jb = jobs.j[blockIdx.x];
  const int tid = static_cast<int>(threadIdx.x), warp = tid >> 5, lane = tid & 31;
  if (blockIdx.y == 1) {  // the job's column sums, beside the MMA CTA instead of after it
    colsums(rows, jb, csp);
    return;
  }
  if (tid == 0) tc::mbar_init(&mbar, 1);
  if (warp == 0) tc::tmem_alloc(&tslot, 64);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tslot, aA = tc::smem_u32(TA), aB = tc::smem_u32(TB);
  uint32_t phase = 0;
  bool first = true;
  // work items: (pass, 128-atom block); the next item's loads are in flight
  // while the current block is staged and contracted
  const int nblk = (rows + TE - 1) / TE, npass = jb.a2 ? 2 : 1, nit = nblk * npass;
  float4 ra[4], rb[4];
  auto fetch = [&](int it) {
    const int pass = it / nblk, i0 = (it % nblk) * TE;
    const float* A = pass ? jb.a2 : jb.a;
    const float* B = pass ? jb.b2 : jb.b;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int x = tid + kWgT * q, c4 = x >> 7, r = x & 127;
      const bool ok = i0 + r < rows;
      ra[q] = ok ? __ldg(reinterpret_cast<const float4*>(A + (size_t)(i0 + r) * 64) + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
      rb[q] = ok ? __ldg(reinterpret_cast<const float4*>(B + (size_t)(i0 + r) * 64) + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  if (nit > 0) fetch(0);
  for (int it = 0; it < nit; ++it) {
    const bool sl = it < nblk && jb.silu_a;
    const int i0 = (it % nblk) * TE;
    // thread -> (feature quad c4, atom r): a warp writes 32 consecutive atoms of one feature row
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int x = tid + kWgT * q, c4 = x >> 7, r = x & 127;
      float4 va = ra[q];
      const float4 vb = rb[q];
      if (sl && i0 + r < rows) va = make_float4(dev::silu(va.x), dev::silu(va.y), dev::silu(va.z), dev::silu(va.w));
      *reinterpret_cast<float*>(TA + off_fm(4 * c4 + 0, r)) = va.x;
      *reinterpret_cast<float*>(TA + off_fm(4 * c4 + 1, r)) = va.y;
      *reinterpret_cast<float*>(TA + off_fm(4 * c4 + 2, r)) = va.z;
      *reinterpret_cast<float*>(TA + off_fm(4 * c4 + 3, r)) = va.w;
      *reinterpret_cast<float*>(TB + off_fm(4 * c4 + 0, r)) = vb.x;
      *reinterpret_cast<float*>(TB + off_fm(4 * c4 + 1, r)) = vb.y;
      *reinterpret_cast<float*>(TB + off_fm(4 * c4 + 2, r)) = vb.z;
      *reinterpret_cast<float*>(TB + off_fm(4 * c4 + 3, r)) = vb.w;
    }
    if (it + 1 < nit) fetch(it + 1);
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (tid == 0) {
      mma_tiles<64, 64, 128, 64>(tmem, aA, aB, !first);
      tc::commit(&mbar);
    }
    tc::mbar_wait(&mbar, phase);  // the MMA has read TA / TB: they may be restaged
    phase ^= 1u;
    tc::fence_after();
    first = false;
  }
  // M=64 accumulator: row r at lane (r/16)*32 + r%16; warp w reads lanes 32w..
  if (first) {  // rows == 0
    for (int x = tid; x < 64 * 64; x += kWgT) jb.G[x] = 0.f;
  } else if (warp < 4) {
#pragma unroll
    for (int cb = 0; cb < 4; ++cb) {
      float v[16];
      tc::ld16(tmem + (static_cast<uint32_t>(32 * warp) << 16) + static_cast<uint32_t>(16 * cb), v);
      if (lane < 16) {
        float4* o = reinterpret_cast<float4*>(jb.G + (16 * warp + lane) * 64 + 16 * cb);
#pragma unroll
        for (int j = 0; j < 4; ++j) o[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free(tmem, 64);
}

}  // namespace edge_tc
}  // namespace janus
