// node_kernels.cuh — per-atom ([N,H]) kernels: small GEMMs with fused input
// transforms and epilogues, weight-gradient reductions over atoms,
// elementwise activation derivatives, energy/force loss seeds, Adam, and the
// LM geometry kernel.  All reductions are fixed-order (deterministic).
#pragma once

#include "common.cuh"
#include "geo_job.hpp"

namespace janus {
namespace node {

// --------------------------------------------------------- input transforms
struct InId {
  __device__ __forceinline__ float operator()(int, int, float x) const { return x; }
};
struct InSilu {
  __device__ __forceinline__ float operator()(int, int, float x) const { return dev::silu(x); }
};
// x * SiLU'(p[i][k])
struct InMulDsilu {
  const float* p;
  int H;
  __device__ __forceinline__ float operator()(int i, int k, float x) const { return x * dev::dsilu(p[(size_t)i * H + k]); }
};
// x * pdot[i][k] * SiLU''(p[i][k])
struct InMulPdotD2silu {
  const float* p;
  const float* pdot;
  int H;
  __device__ __forceinline__ float operator()(int i, int k, float x) const {
    const size_t o = (size_t)i * H + k;
    return x * pdot[o] * dev::d2silu(p[o]);
  }
};
// SiLU'(x) * omega[k]
struct InDsiluOmega {
  const float* omega;
  __device__ __forceinline__ float operator()(int, int k, float x) const { return dev::dsilu(x) * omega[k]; }
};

// out[i][n] = sum_k op(X[i][k]) M[k][n] (+ bias[n]) (+ add1[i][n]) (+ add2[i][n])
// One CTA = 256/H rows x H columns, one output per thread; the transformed
// input rows are staged in smem (op applied once per element), M is read
// through L1 (every CTA reads all of M: 16 KB, L2-resident).
template <int H, typename InOp>
__global__ void __launch_bounds__(256) gemm_rows_kernel(int rows, const float* __restrict__ X, const float* __restrict__ M,
                                                        const float* __restrict__ bias, const float* add1, const float* add2,
                                                        float* out, InOp op) {
  JANUS_GDC_WAIT();
  constexpr int RB = 256 / H;
  __shared__ __align__(16) float sx[RB][H];
  const int r0 = blockIdx.x * RB;
  const int r = threadIdx.x / H, c = threadIdx.x % H;
  const int i = r0 + r;
  sx[r][c] = (i < rows) ? op(i, c, X[(size_t)i * H + c]) : 0.f;
  __syncthreads();
  float acc0 = 0.f, acc1 = 0.f;
#pragma unroll 16
  for (int k = 0; k < H; k += 2) {
    acc0 = fmaf(sx[r][k], __ldg(M + (size_t)k * H + c), acc0);
    acc1 = fmaf(sx[r][k + 1], __ldg(M + (size_t)(k + 1) * H + c), acc1);
  }
  if (i >= rows) return;
  const size_t o = (size_t)i * H + c;
  float y = acc0 + acc1;
  if (bias) y += bias[c];
  if (add1) y += add1[o];
  if (add2) y += add2[o];
  out[o] = y;
}

// Weight gradients over atoms, two deterministic stages:
//  (1) wgrad_partial: CTA c reduces rows [64c, 64c+64): G_c = sum_i opA(a_i)^T b_i
//      (+ a2_i^T b2_i), plus up to two column sums cs1 = sum_i x1_i, cs2 = sum_i x2_i;
//  (2) wgrad_final: out = sum_c G_c in chunk order.
// Partial layout per chunk: [H*H | H | H].
constexpr int kWChunk = 64;

template <int H, typename InOp>
__global__ void __launch_bounds__(256) wgrad_partial_kernel(int rows, const float* __restrict__ a, const float* __restrict__ b,
                                                            const float* __restrict__ a2, const float* __restrict__ b2,
                                                            const float* __restrict__ x1, const float* __restrict__ x2,
                                                            float* __restrict__ part, InOp op) {
  JANUS_GDC_WAIT();
  static_assert(H == 64, "tile mapping assumes H = 64");
  __shared__ __align__(16) float sa[kWChunk][H + 4];
  __shared__ __align__(16) float sb[kWChunk][H + 4];
  const int i0 = blockIdx.x * kWChunk;
  const int n = min(kWChunk, rows - i0);
  const int kb = (threadIdx.x >> 4) * 4, hb = (threadIdx.x & 15) * 4;
  float acc[4][4];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) acc[x][y] = 0.f;
  for (int pass = 0; pass < (a2 ? 2 : 1); ++pass) {
    const float* A = pass ? a2 : a;
    const float* B = pass ? b2 : b;
    __syncthreads();
    {
      // all 2 x 16 loads of this thread in flight before any use (ILP), then the stores
      constexpr int PER = kWChunk * H / 256;
      float va[PER], vb[PER];
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        const int x = threadIdx.x + 256 * q, r = x / H, c = x % H;
        const bool ok = r < n;
        va[q] = ok ? __ldg(A + (size_t)(i0 + r) * H + c) : 0.f;
        vb[q] = ok ? __ldg(B + (size_t)(i0 + r) * H + c) : 0.f;
      }
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        const int x = threadIdx.x + 256 * q, r = x / H, c = x % H;
        sa[r][c] = (pass || r >= n) ? va[q] : op(i0 + r, c, va[q]);
        sb[r][c] = vb[q];
      }
    }
    __syncthreads();
#pragma unroll 4
    for (int r = 0; r < n; ++r) {
      const float4 va = *reinterpret_cast<const float4*>(&sa[r][kb]);
      const float4 vb = *reinterpret_cast<const float4*>(&sb[r][hb]);
      const float xa[4] = {va.x, va.y, va.z, va.w}, xb[4] = {vb.x, vb.y, vb.z, vb.w};
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y] = fmaf(xa[x], xb[y], acc[x][y]);
    }
  }
  float* P = part + (size_t)blockIdx.x * (H * H + 2 * H);
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) P[(kb + x) * H + hb + y] = acc[x][y];
  // column sums, staged through smem (coalesced loads, fixed row order)
  for (int q = 0; q < 2; ++q) {
    const float* X = q ? x2 : x1;
    if (!X) {
      if (threadIdx.x < H) P[H * H + q * H + threadIdx.x] = 0.f;
      continue;
    }
    __syncthreads();
    for (int x = threadIdx.x; x < kWChunk * H; x += 256) {
      const int r = x / H, c = x % H;
      sa[r][c] = r < n ? X[(size_t)(i0 + r) * H + c] : 0.f;
    }
    __syncthreads();
    if (threadIdx.x < H) {
      float s = 0.f;
      for (int r = 0; r < n; ++r) s += sa[r][threadIdx.x];
      P[H * H + q * H + threadIdx.x] = s;
    }
  }
}

// out_G (if non-null) = sum_c G_c ; cs_out1/2 = sum_c cs_c (fixed chunk order)
template <int H>
__global__ void wgrad_final_kernel(int n_chunks, const float* __restrict__ part, float* __restrict__ G,
                                   float* __restrict__ cs_out1, float* __restrict__ cs_out2) {
  JANUS_GDC_WAIT();
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  constexpr int W = H * H + 2 * H;
  if (o >= W) return;
  float* dst = o < H * H ? G : (o < H * H + H ? cs_out1 : cs_out2);
  if (!dst) return;
  float s = 0.f;
#pragma unroll 4
  for (int c = 0; c < n_chunks; ++c) s += part[(size_t)c * W + o];
  dst[o < H * H ? o : (o - H * H) % H] = s;
}

// out[z][k] = sum_{i: Z_i = z} x[i][k]  (chunked; partial [chunk][S*H]).  When
// x is null the summand is the scalar eps[struct_id[i]] (readout bias grads, k = 0).
template <int H>
__global__ void species_sum_partial_kernel(int rows, int S, const int* __restrict__ species, const float* __restrict__ x,
                                           const float* __restrict__ eps, const int* __restrict__ struct_id,
                                           float* __restrict__ part) {
  JANUS_GDC_WAIT();
  const int i0 = blockIdx.x * kWChunk;
  const int n = min(kWChunk, rows - i0);
  for (int o = threadIdx.x; o < S * H; o += blockDim.x) {
    const int z = o / H, k = o % H;
    float s = 0.f;
    for (int r = 0; r < n; ++r) {
      const int i = i0 + r;
      if (species[i] != z) continue;
      s += x ? x[(size_t)i * H + k] : (k == 0 ? eps[struct_id[i]] : 0.f);
    }
    part[(size_t)blockIdx.x * S * H + o] = s;
  }
}

template <int H>
__global__ void species_sum_final_kernel(int n_chunks, int S, int stride_out, const float* __restrict__ part,
                                         float* __restrict__ out) {
  JANUS_GDC_WAIT();
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= S * H) return;
  const int z = o / H, k = o % H;
  if (stride_out == 1 && k != 0) return;  // scalar mode: one value per species
  float s = 0.f;
  for (int c = 0; c < n_chunks; ++c) s += part[(size_t)c * S * H + o];
  out[stride_out == 1 ? z : o] = s;
}

// ------------------------------------------------------------ elementwise
// upd BF: pbar = r pdot SiLU''(p), pdbar = r SiLU'(p), u = SiLU'(p) pdot
__global__ void upd_bf_ew_kernel(int n, const float* __restrict__ r, const float* __restrict__ pdot,
                                 const float* __restrict__ p, float* __restrict__ pbar, float* __restrict__ pdbar,
                                 float* __restrict__ u) {
  JANUS_GDC_WAIT();
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= n) return;
  const float pp = p[x], ds = dev::dsilu(pp);
  pbar[x] = r[x] * pdot[x] * dev::d2silu(pp);
  pdbar[x] = r[x] * ds;
  u[x] = ds * pdot[x];
}

// upd BE: pbar = r SiLU'(p)
__global__ void upd_be_ew_kernel(int n, const float* __restrict__ r, const float* __restrict__ p, float* __restrict__ pbar) {
  JANUS_GDC_WAIT();
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= n) return;
  pbar[x] = r[x] * dev::dsilu(p[x]);
}

// readout BF: tau = tdot omega SiLU''(t), w2 = tdot SiLU'(t), sw = SiLU'(t) omega
template <int H>
__global__ void ro_bf_ew_kernel(int n, const float* __restrict__ tdot, const float* __restrict__ t,
                                const float* __restrict__ omega, float* __restrict__ tau, float* __restrict__ w2,
                                float* __restrict__ sw) {
  JANUS_GDC_WAIT();
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= n) return;
  const int k = x % H;
  const float tt = t[x], ds = dev::dsilu(tt);
  tau[x] = tdot[x] * omega[k] * dev::d2silu(tt);
  w2[x] = tdot[x] * ds;
  sw[x] = ds * omega[k];
}

// readout BE: tbar = eps_s SiLU'(t) omega, es = eps_s SiLU(t)
template <int H>
__global__ void ro_be_ew_kernel(int n, const float* __restrict__ t, const float* __restrict__ omega,
                                const float* __restrict__ eps, const int* __restrict__ struct_id, float* __restrict__ tbar,
                                float* __restrict__ es) {
  JANUS_GDC_WAIT();
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= n) return;
  const int i = x / H, k = x % H;
  const float ep = eps[struct_id[i]], tt = t[x];
  tbar[x] = ep * dev::dsilu(tt) * omega[k];
  es[x] = ep * dev::silu(tt);
}

// ------------------------------------------------------ embed / readout I/O
template <int H>
__global__ void embed_fe_kernel(int n_atoms, const int* __restrict__ species, const float* __restrict__ Emb,
                                float* __restrict__ h) {
  JANUS_GDC_WAIT();
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= n_atoms * H) return;
  const int i = x / H, k = x % H;
  h[x] = Emb[(size_t)species[i] * H + k];
}

// e_i = <SiLU(t_i), omega> + bias[Z_i]   (warp per atom)
template <int H>
__global__ void readout_energy_kernel(int n_atoms, const float* __restrict__ t, const float* __restrict__ omega,
                                      const float* __restrict__ bias, const int* __restrict__ species,
                                      float* __restrict__ e_atom) {
  JANUS_GDC_WAIT();
  const int i = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x & 31;
  if (i >= n_atoms) return;
  float s = 0.f;
  for (int k = lane; k < H; k += 32) s = fmaf(dev::silu(t[(size_t)i * H + k]), omega[k], s);
  s = dev::warp_sum(s);
  if (lane == 0) e_atom[i] = s + bias[species[i]];
}

// E_s, eps_s = 2 w_E (E_s - E*_s), loss_E = sum w_E (E - E*)^2.  One thread per
// structure for E_s (atoms contiguous: struct_ptr), thread 0 for the loss.
__global__ void energy_loss_kernel(int n_struct, const int* __restrict__ struct_ptr, const float* __restrict__ e_atom,
                                   const float* __restrict__ E_target, float w_E, float* __restrict__ E,
                                   float* __restrict__ eps, float* __restrict__ loss_E) {
  JANUS_GDC_WAIT();
  for (int s = threadIdx.x; s < n_struct; s += blockDim.x) {
    float acc = 0.f;
    for (int i = struct_ptr[s]; i < struct_ptr[s + 1]; ++i) acc += e_atom[i];
    E[s] = acc;
    eps[s] = 2.0f * w_E * (acc - E_target[s]);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float l = 0.f;
    for (int s = 0; s < n_struct; ++s) {
      const float d = E[s] - E_target[s];
      l += w_E * d * d;
    }
    *loss_E = l;
  }
}

// Fbar = 2 w_F (F - F*); loss_F = sum w_F |F - F*|^2 (single CTA, fixed tree)
__global__ void force_loss_kernel(int n3, const float* __restrict__ F, const float* __restrict__ F_target, float w_F,
                                  float* __restrict__ Fbar, float* __restrict__ loss_F) {
  JANUS_GDC_WAIT();
  __shared__ float red[1024];
  float l = 0.f;
  for (int x = threadIdx.x; x < n3; x += blockDim.x) {
    const float d = F[x] - F_target[x];
    Fbar[x] = 2.0f * w_F * d;
    l += w_F * d * d;
  }
  red[threadIdx.x] = l;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) *loss_F = red[0];
}

// ----------------------------------------------------------- optimizer
// g = sum_mb (g1[mb] + g2[mb]) in micro-batch order (schedule-independent)
__global__ void ledger_reduce_kernel(int64_t n, int n_mb, const float* __restrict__ g1, const float* __restrict__ g2,
                                     float* __restrict__ g) {
  JANUS_GDC_WAIT();
  const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= n) return;
  float s = 0.f;
  for (int m = 0; m < n_mb; ++m) {
    s += g1[(size_t)m * n + x];
    s += g2[(size_t)m * n + x];
  }
  g[x] = s;
}

__global__ void adam_tick_kernel(int* step) {
  JANUS_GDC_WAIT(); *step += 1; }

// Bias corrections from the device-side step counter and the hyperparameters
// {lr, beta1, beta2, eps} from a device buffer, so a captured step (CUDA
// graph) replays correctly when the caller changes the learning rate.
__global__ void adam_kernel(int64_t n, float* __restrict__ p, float* __restrict__ m1, float* __restrict__ m2,
                            const float* __restrict__ g, const float* __restrict__ hp,
                            const int* __restrict__ step) {
  JANUS_GDC_WAIT();
  const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= n) return;
  const float lr = hp[0], b1 = hp[1], b2 = hp[2], eps = hp[3];
  const float t = static_cast<float>(*step);
  const float c1 = 1.0f - powf(b1, t), c2 = 1.0f - powf(b2, t);
  const float gg = g[x];
  const float a = b1 * m1[x] + (1.0f - b1) * gg;
  const float b = b2 * m2[x] + (1.0f - b2) * gg * gg;
  m1[x] = a;
  m2[x] = b;
  p[x] -= lr * (a / c1) / (sqrtf(b / c2) + eps);
}

// dst[c][r] = src[r][c] for a square H x H block
template <int H>
__global__ void transpose_kernel(const float* __restrict__ src, float* __restrict__ dst) {
  JANUS_GDC_WAIT();
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= H * H) return;
  const int r = x / H, c = x % H;
  dst[(size_t)c * H + r] = src[x];
}

// ------------------------------------------------------------ LM geometry
// One thread per edge: receiver i by binary search on row_ptr, then
// r = x_j + s L - x_i in fp64 (same association as the oracle, no FMA), and
// d, u = r/d, cosine cutoff c and c' stored in fp32.
__global__ void geometry_kernel(int n_atoms, int n_edges, const int* __restrict__ row_ptr, const int* __restrict__ col,
                                const int* __restrict__ shift, const double* __restrict__ pos,
                                const int* __restrict__ struct_id, const double* __restrict__ cell, double rc,
                                int* __restrict__ src, float* __restrict__ d_out, float* __restrict__ u_out,
                                float* __restrict__ c_out, float* __restrict__ dc_out) {
  JANUS_GDC_WAIT();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_edges) return;
  int lo = 0, hi = n_atoms;  // largest i with row_ptr[i] <= e
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (row_ptr[mid] <= e) lo = mid; else hi = mid;
  }
  const int i = lo, j = col[e];
  const double L = cell[struct_id[i]];
  const double rx = __dsub_rn(__dadd_rn(pos[3 * j + 0], __dmul_rn((double)shift[3 * e + 0], L)), pos[3 * i + 0]);
  const double ry = __dsub_rn(__dadd_rn(pos[3 * j + 1], __dmul_rn((double)shift[3 * e + 1], L)), pos[3 * i + 1]);
  const double rz = __dsub_rn(__dadd_rn(pos[3 * j + 2], __dmul_rn((double)shift[3 * e + 2], L)), pos[3 * i + 2]);
  const double d = sqrt(rx * rx + ry * ry + rz * rz);
  src[e] = i;
  d_out[e] = (float)d;
  u_out[3 * e + 0] = (float)(rx / d);
  u_out[3 * e + 1] = (float)(ry / d);
  u_out[3 * e + 2] = (float)(rz / d);
  double sn, cs;  // sin / cos of pi d / r_c, one fp64 sincospi (not two calls)
  sincospi(d / rc, &sn, &cs);
  c_out[e] = d < rc ? (float)(0.5 * (cs + 1.0)) : 0.f;
  dc_out[e] = d < rc ? (float)(-0.5 * (3.14159265358979323846 / rc) * sn) : 0.f;
}

// Batched LM geometry: one launch for the micro-batches of one load.  Per
// edge: (optionally) the device-built CSR slice is copied in with col / rev
// rebased, then the same per-edge geometry as geometry_kernel.  The job table
// travels as a kernel parameter.
__global__ void geometry_batched_kernel(const __grid_constant__ GeoJobs J) {
  JANUS_GDC_WAIT();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= J.total_edges) return;
  int k = 0;
  while (k + 1 < J.n && J.j[k + 1].edge_base <= t) ++k;
  const GeoJob& jb = J.j[k];
  const int e = t - jb.edge_base;
  int j, sx, sy, sz;
  if (jb.scol) {
    j = jb.scol[jb.edge0 + e] - jb.atom0;
    jb.col[e] = j;
    jb.rev[e] = jb.srev[jb.edge0 + e] - jb.edge0;
    sx = jb.sshift[3 * (jb.edge0 + e) + 0];
    sy = jb.sshift[3 * (jb.edge0 + e) + 1];
    sz = jb.sshift[3 * (jb.edge0 + e) + 2];
    jb.shift[3 * e + 0] = sx;
    jb.shift[3 * e + 1] = sy;
    jb.shift[3 * e + 2] = sz;
  } else {
    j = jb.col[e];
    sx = jb.shift[3 * e + 0];
    sy = jb.shift[3 * e + 1];
    sz = jb.shift[3 * e + 2];
  }
  int lo = 0, hi = jb.n_atoms;  // largest i with row_ptr[i] <= e
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (jb.row_ptr[mid] <= e) lo = mid; else hi = mid;
  }
  const int i = lo;
  const double L = jb.cell[jb.struct_id[i]];
  const double* pj = jb.pos + 3 * j;
  const double* pi = jb.pos + 3 * i;
  const double rx = __dsub_rn(__dadd_rn(pj[0], __dmul_rn((double)sx, L)), pi[0]);
  const double ry = __dsub_rn(__dadd_rn(pj[1], __dmul_rn((double)sy, L)), pi[1]);
  const double rz = __dsub_rn(__dadd_rn(pj[2], __dmul_rn((double)sz, L)), pi[2]);
  const double d = sqrt(rx * rx + ry * ry + rz * rz);
  jb.src[e] = i;
  jb.d[e] = (float)d;
  jb.u[3 * e + 0] = (float)(rx / d);
  jb.u[3 * e + 1] = (float)(ry / d);
  jb.u[3 * e + 2] = (float)(rz / d);
  double sn, cs;  // sin / cos of pi d / r_c, one fp64 sincospi (not two calls)
  sincospi(d / J.rc, &sn, &cs);
  jb.c[e] = d < J.rc ? (float)(0.5 * (cs + 1.0)) : 0.f;
  jb.dc[e] = d < J.rc ? (float)(-0.5 * (3.14159265358979323846 / J.rc) * sn) : 0.f;
}

}  // namespace node
}  // namespace janus

namespace janus {
namespace node {

// ===================================================================== fused
// Row-local programs for the upd unit (p = mU + ups, y = SiLU(p) V): one CTA =
// 16 atoms x 64 features, thread (row t/16, 4 columns); row vectors staged in
// smem, weights read through L1.  Each replaces 3-5 separate launches.
// upd kernels: RB rows per CTA, 16 * RB threads (1 row x 4 columns each);
// 32 rows for large micro-batches (half the CTAs and weight staging of 16:
// C2 15515 -> 15765), 16 for small ones (more CTAs on a latency-bound chain)
constexpr int kRB = 32;
constexpr int kRBSmall = 16;
inline int upd_rows_per_cta(int n_atoms) { return n_atoms >= 256 ? kRB : kRBSmall; }

__device__ __forceinline__ void rowmm(const float (*X)[68], const float* Ms, int r, int c0, float (&o)[4]) {
  o[0] = o[1] = o[2] = o[3] = 0.f;
#pragma unroll 16
  for (int k = 0; k < 64; ++k) {
    const float a = X[r][k];
    const float4 m = *reinterpret_cast<const float4*>(Ms + k * 64 + c0);
    o[0] = fmaf(a, m.x, o[0]);
    o[1] = fmaf(a, m.y, o[1]);
    o[2] = fmaf(a, m.z, o[2]);
    o[3] = fmaf(a, m.w, o[3]);
  }
}
// Same products in gemm_rows_kernel's summation order (even / odd k chains,
// then their sum), so a fused v = h W is bit-identical to the row-GEMM launch
// it replaces (pipeline stages that cannot fuse use the launch).
__device__ __forceinline__ void rowmm_eo(const float (*X)[68], const float* Ms, int r, int c0, float (&o)[4]) {
  float e[4] = {0.f, 0.f, 0.f, 0.f}, d[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 8
  for (int k = 0; k < 64; k += 2) {
    const float a0 = X[r][k], a1 = X[r][k + 1];
    const float4 m0 = *reinterpret_cast<const float4*>(Ms + k * 64 + c0);
    const float4 m1 = *reinterpret_cast<const float4*>(Ms + (k + 1) * 64 + c0);
    e[0] = fmaf(a0, m0.x, e[0]);
    e[1] = fmaf(a0, m0.y, e[1]);
    e[2] = fmaf(a0, m0.z, e[2]);
    e[3] = fmaf(a0, m0.w, e[3]);
    d[0] = fmaf(a1, m1.x, d[0]);
    d[1] = fmaf(a1, m1.y, d[1]);
    d[2] = fmaf(a1, m1.z, d[2]);
    d[3] = fmaf(a1, m1.w, d[3]);
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) o[q] = e[q] + d[q];
}
// Stage up to 4 [64][64] weight matrices into smem with every load in flight
// at once (16 float4 per thread per matrix), then one barrier.
// (cp.async: every 16 B copy of every matrix in flight at once, no registers;
// the caller's barrier follows cp.async.wait_group 0 in stage_mats_wait)
__device__ __forceinline__ void stage_mats(float* dst, const float* const* src, int n) {
  for (int m = 0; m < n; ++m) {
    const float4* s4 = reinterpret_cast<const float4*>(src[m]);
    float4* d4 = reinterpret_cast<float4*>(dst + m * 4096);
    for (int q = static_cast<int>(threadIdx.x); q < 1024; q += static_cast<int>(blockDim.x)) {
      const uint32_t da = static_cast<uint32_t>(__cvta_generic_to_shared(d4 + q));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(da), "l"(s4 + q) : "memory");
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}
// the matrices landed (this thread's copies); a barrier then publishes them
__device__ __forceinline__ void stage_mats_wait() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
constexpr size_t upd_smem(int nmats) { return sizeof(float) * 4096 * nmats; }

template <int RB>
__device__ __forceinline__ void row_load(float (*X)[68], const float* __restrict__ src, int i0, int rows) {
  for (int x = threadIdx.x; x < RB * 16; x += blockDim.x) {
    const int r = x / 16, q = x % 16;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (i0 + r < rows) v = __ldg(reinterpret_cast<const float4*>(src + (size_t)(i0 + r) * 64) + q);
    *reinterpret_cast<float4*>(&X[r][4 * q]) = v;
  }
}
__device__ __forceinline__ void row_store(float* dst, int i, int c0, const float (&v)[4]) {
  *reinterpret_cast<float4*>(dst + (size_t)i * 64 + c0) = make_float4(v[0], v[1], v[2], v[3]);
}
__device__ __forceinline__ float4 row_get(const float* src, int i, int c0) {
  return __ldg(reinterpret_cast<const float4*>(src + (size_t)i * 64 + c0));
}

// out[i] = op(X[i]) M (+ bias) (+ add1[i]) (+ add2[i]) with RB rows per CTA
// and M staged once per CTA by cp.async (gemm_rows_kernel: 4 rows per CTA,
// each re-reading M through L1).  Same per-output arithmetic as
// gemm_rows_kernel (even / odd k chains, then bias, add1, add2): bit-identical.
template <int RB, typename InOp>
__global__ void __launch_bounds__(16 * RB) gemm_rb_kernel(int rows, const float* __restrict__ X, const float* __restrict__ M,
                                                          const float* __restrict__ bias, const float* add1, const float* add2,
                                                          float* out, InOp op) {
  JANUS_GDC_WAIT();
  __shared__ __align__(16) float Xs[RB][68];
  extern __shared__ __align__(16) float Ws[];
  const int i0 = blockIdx.x * RB, r = threadIdx.x / 16, c0 = (threadIdx.x % 16) * 4, i = i0 + r;
  {
    const float* mats[1] = {M};
    stage_mats(Ws, mats, 1);
  }
  for (int x = threadIdx.x; x < RB * 64; x += blockDim.x) {
    const int rr = x / 64, c = x % 64;
    Xs[rr][c] = i0 + rr < rows ? op(i0 + rr, c, X[(size_t)(i0 + rr) * 64 + c]) : 0.f;
  }
  stage_mats_wait();
  __syncthreads();
  float o[4];
  rowmm_eo(Xs, Ws, r, c0, o);
  if (i >= rows) return;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const size_t idx = (size_t)i * 64 + c0 + q;
    float y = o[q];
    if (bias) y += bias[c0 + q];
    if (add1) y += add1[idx];
    if (add2) y += add2[idx];
    out[idx] = y;
  }
}

// FE: p = m U + ups ; h_out = h + SiLU(p) V ; and, when the next unit is a
// msg unit on the stage, its v = h_out Wn (saves that unit's row-GEMM launch)
template <int RB>
__global__ void __launch_bounds__(16 * RB) upd_fe_fused(int rows, const float* __restrict__ m, const float* __restrict__ h,
                                                    const float* __restrict__ U, const float* __restrict__ ups,
                                                    const float* __restrict__ V, float* __restrict__ p_out,
                                                    float* __restrict__ h_out, const float* __restrict__ Wn,
                                                    float* __restrict__ v_out) {
  JANUS_GDC_WAIT();
  __shared__ __align__(16) float X[RB][68];
  extern __shared__ __align__(16) float Ws[];
  const int i0 = blockIdx.x * RB, r = threadIdx.x / 16, c0 = (threadIdx.x % 16) * 4, i = i0 + r;
  {
    const float* mats[3] = {U, V, Wn};
    stage_mats(Ws, mats, Wn ? 3 : 2);
  }
  row_load<RB>(X, m, i0, rows);
  stage_mats_wait();
  __syncthreads();
  float o[4];
  rowmm(X, Ws, r, c0, o);
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    o[q] += ups[c0 + q];
    X[r][c0 + q] = dev::silu(o[q]);
  }
  if (i < rows) row_store(p_out, i, c0, o);
  __syncthreads();
  rowmm(X, Ws + 4096, r, c0, o);
  if (i < rows) {
    const float4 hh = row_get(h, i, c0);
    o[0] += hh.x, o[1] += hh.y, o[2] += hh.z, o[3] += hh.w;
    row_store(h_out, i, c0, o);
  }
  if (Wn) {  // v = h_out Wn (padding rows: h = 0 loads, results not stored)
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) X[r][c0 + q] = o[q];
    __syncthreads();
    rowmm_eo(X, Ws + 2 * 4096, r, c0, o);
    if (i < rows) row_store(v_out, i, c0, o);
  }
}

// FF: ff_a = a' ; am = ((a' V^T) SiLU'(p)) U^T
template <int RB>
__global__ void __launch_bounds__(16 * RB) upd_ff_fused(int rows, const float* __restrict__ a, const float* __restrict__ p,
                                                    const float* __restrict__ Vt, const float* __restrict__ Ut,
                                                    float* __restrict__ ff_a, float* __restrict__ am) {
  JANUS_GDC_WAIT();
  __shared__ __align__(16) float X[RB][68];
  extern __shared__ __align__(16) float Ws[];
  const int i0 = blockIdx.x * RB, r = threadIdx.x / 16, c0 = (threadIdx.x % 16) * 4, i = i0 + r;
  {
    const float* mats[2] = {Vt, Ut};
    stage_mats(Ws, mats, 2);
  }
  row_load<RB>(X, a, i0, rows);
  stage_mats_wait();
  __syncthreads();
  if (i < rows) {
    const float v4[4] = {X[r][c0], X[r][c0 + 1], X[r][c0 + 2], X[r][c0 + 3]};
    row_store(ff_a, i, c0, v4);
  }
  float o[4];
  rowmm(X, Ws, r, c0, o);
  __syncthreads();
  if (i < rows) {
    const float4 pp = row_get(p, i, c0);
    o[0] *= dev::dsilu(pp.x), o[1] *= dev::dsilu(pp.y), o[2] *= dev::dsilu(pp.z), o[3] *= dev::dsilu(pp.w);
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) X[r][c0 + q] = o[q];
  __syncthreads();
  rowmm(X, Ws + 4096, r, c0, o);
  if (i < rows) row_store(am, i, c0, o);
}

// BF: pdot = abar_m U ; r = a' V^T ; pbar = r pdot SiLU''(p) ; pdbar = r SiLU'(p) ;
//     u = SiLU'(p) pdot ; inj = pbar U^T ; abar_h += u V
template <int RB>
__global__ void __launch_bounds__(16 * RB) upd_bf_fused(int rows, const float* __restrict__ am, const float* __restrict__ ffa,
                                                    const float* __restrict__ p, const float* __restrict__ U,
                                                    const float* __restrict__ Vt, const float* __restrict__ Ut,
                                                    const float* __restrict__ V, float* __restrict__ pbar,
                                                    float* __restrict__ pdbar, float* __restrict__ u,
                                                    float* __restrict__ inj, const float* ah, float* ah_out,
                                                    const float* __restrict__ Wn, float* __restrict__ vdot_out) {
  JANUS_GDC_WAIT();
  __shared__ __align__(16) float X[RB][68];
  __shared__ __align__(16) float Y[RB][68];
  extern __shared__ __align__(16) float Ws[];
  const int i0 = blockIdx.x * RB, r = threadIdx.x / 16, c0 = (threadIdx.x % 16) * 4, i = i0 + r;
  {
    const float* mats[5] = {U, Vt, Ut, V, Wn};
    stage_mats(Ws, mats, Wn ? 5 : 4);
  }
  row_load<RB>(X, am, i0, rows);
  stage_mats_wait();
  row_load<RB>(Y, ffa, i0, rows);
  __syncthreads();
  float pd[4], rr[4];
  rowmm(X, Ws, r, c0, pd);
  rowmm(Y, Ws + 4096, r, c0, rr);
  __syncthreads();
  float pb[4], pdb[4], uu[4];
  const float4 pp4 = i < rows ? row_get(p, i, c0) : make_float4(0.f, 0.f, 0.f, 0.f);
  const float pp[4] = {pp4.x, pp4.y, pp4.z, pp4.w};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float ds = dev::dsilu(pp[q]);
    pb[q] = rr[q] * pd[q] * dev::d2silu(pp[q]);
    pdb[q] = rr[q] * ds;
    uu[q] = ds * pd[q];
    X[r][c0 + q] = pb[q];
    Y[r][c0 + q] = uu[q];
  }
  if (i < rows) {
    row_store(pbar, i, c0, pb);
    row_store(pdbar, i, c0, pdb);
    row_store(u, i, c0, uu);
  }
  __syncthreads();
  float o[4];
  rowmm(X, Ws + 2 * 4096, r, c0, o);
  if (i < rows) row_store(inj, i, c0, o);
  rowmm(Y, Ws + 3 * 4096, r, c0, o);
  if (i < rows) {
    const float4 a4 = row_get(ah, i, c0);
    o[0] += a4.x, o[1] += a4.y, o[2] += a4.z, o[3] += a4.w;
    row_store(ah_out, i, c0, o);  // ah_out may alias ah (same element, read first)
  }
  if (Wn) {  // the next msg unit's vdot = abar_h' Wn (saves its row-GEMM launch)
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) X[r][c0 + q] = o[q];
    __syncthreads();
    rowmm_eo(X, Ws + 4 * 4096, r, c0, o);
    if (i < rows) row_store(vdot_out, i, c0, o);
  }
}

// BE: r = b' V^T ; pbar = r SiLU'(p) ; b_m = pbar U^T + inj
template <int RB>
__global__ void __launch_bounds__(16 * RB) upd_be_fused(int rows, const float* __restrict__ bh, const float* __restrict__ p,
                                                    const float* __restrict__ Vt, const float* __restrict__ Ut,
                                                    const float* __restrict__ inj, float* __restrict__ pbar,
                                                    float* __restrict__ bm) {
  JANUS_GDC_WAIT();
  __shared__ __align__(16) float X[RB][68];
  extern __shared__ __align__(16) float Ws[];
  const int i0 = blockIdx.x * RB, r = threadIdx.x / 16, c0 = (threadIdx.x % 16) * 4, i = i0 + r;
  {
    const float* mats[2] = {Vt, Ut};
    stage_mats(Ws, mats, 2);
  }
  row_load<RB>(X, bh, i0, rows);
  stage_mats_wait();
  __syncthreads();
  float o[4];
  rowmm(X, Ws, r, c0, o);
  __syncthreads();
  const float4 pp4 = i < rows ? row_get(p, i, c0) : make_float4(0.f, 0.f, 0.f, 0.f);
  const float pp[4] = {pp4.x, pp4.y, pp4.z, pp4.w};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    o[q] *= dev::dsilu(pp[q]);
    X[r][c0 + q] = o[q];
  }
  if (i < rows) row_store(pbar, i, c0, o);
  __syncthreads();
  rowmm(X, Ws + 4096, r, c0, o);
  if (i < rows) {
    const float4 j4 = row_get(inj, i, c0);
    o[0] += j4.x, o[1] += j4.y, o[2] += j4.z, o[3] += j4.w;
    row_store(bm, i, c0, o);
  }
}

// ------------------------------------------------------- multi-job wgrad
// Up to 3 independent weight-gradient jobs in one launch (grid.y = job),
// 64-row chunks (grid.x); the last CTA to finish reduces every job's chunk
// partials in chunk order (deterministic) and resets the launch counter.
struct WJob {
  const float *a, *b, *a2, *b2, *x1, *x2;
  float *G, *cs1, *cs2;
  int silu_a;
};
struct WJobs {
  WJob j[3];
  int n;
};

// Output-partitioned (no reduction pass): grid.y = job; grid.x = 8 CTAs each
// owning 8 rows of the 64x64 gradient (thread: 1 row, 2 columns), looping over
// all atoms in 64-row chunks in order, + 1 CTA for the column sums.  Every
// output is summed by one thread in atom order => deterministic.
__global__ void __launch_bounds__(256) wgrad_multi_kernel(int rows, WJobs jobs, float* __restrict__ /*part*/,
                                                          unsigned* __restrict__ /*counter*/) {
  JANUS_GDC_WAIT();
  constexpr int H = 64;
  __shared__ __align__(16) float sa[kWChunk][8];
  __shared__ __align__(16) float sb[kWChunk][H + 4];
  const WJob& jb = jobs.j[blockIdx.y];
  if (blockIdx.x == 8) {  // column sums
    const int q = threadIdx.x >> 6, c = threadIdx.x & 63;
    const float* X = q == 0 ? jb.x1 : (q == 1 ? jb.x2 : nullptr);
    float* out = q == 0 ? jb.cs1 : (q == 1 ? jb.cs2 : nullptr);
    if (!X || !out) return;
    float s0 = 0.f;
    int i = 0;
    for (; i + 8 <= rows; i += 8) {  // 8 loads in flight, summed in order
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldg(X + (size_t)(i + u) * H + c);
#pragma unroll
      for (int u = 0; u < 8; ++u) s0 += v[u];
    }
    for (; i < rows; ++i) s0 += __ldg(X + (size_t)i * H + c);
    out[c] = s0;
    return;
  }
  const int k0 = blockIdx.x * 8;
  const int kr = threadIdx.x >> 5, h = threadIdx.x & 31;
  float acc0 = 0.f, acc1 = 0.f;
  for (int pass = 0; pass < (jb.a2 ? 2 : 1); ++pass) {
    const float* A = pass ? jb.a2 : jb.a;
    const float* B = pass ? jb.b2 : jb.b;
    const bool sl = !pass && jb.silu_a;
    for (int i0 = 0; i0 < rows; i0 += kWChunk) {
      const int n = min(kWChunk, rows - i0);
      __syncthreads();
      {
        // a: 64 rows x 8 cols (2 per thread); b: 64 rows x 64 cols (4 float4 per thread)
        float va[2];
        float4 vb[4];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int x = threadIdx.x + 256 * q, r = x >> 3, c = x & 7;
          va[q] = r < n ? __ldg(A + (size_t)(i0 + r) * H + k0 + c) : 0.f;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int x = threadIdx.x + 256 * q, r = x >> 4, c4 = x & 15;
          vb[q] = r < n ? __ldg(reinterpret_cast<const float4*>(B + (size_t)(i0 + r) * H) + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int x = threadIdx.x + 256 * q, r = x >> 3, c = x & 7;
          sa[r][c] = (sl && r < n) ? dev::silu(va[q]) : va[q];
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int x = threadIdx.x + 256 * q, r = x >> 4, c4 = x & 15;
          *reinterpret_cast<float4*>(&sb[r][4 * c4]) = vb[q];
        }
      }
      __syncthreads();
#pragma unroll 8
      for (int r = 0; r < n; ++r) {
        const float a = sa[r][kr];
        acc0 = fmaf(a, sb[r][h], acc0);
        acc1 = fmaf(a, sb[r][h + 32], acc1);
      }
    }
  }
  jb.G[(k0 + kr) * H + h] = acc0;
  jb.G[(k0 + kr) * H + h + 32] = acc1;
}

}  // namespace node
}  // namespace janus
