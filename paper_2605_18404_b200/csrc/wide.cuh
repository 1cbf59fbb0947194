// wide.cuh — device kernels of the generic-width stage path (any hidden width
// H = 32·V, V in {2, 4, 8}; any basis size R): configs[2]'s deep model (L=32,
// H=256) and the cross-check of the fused H=64 kernels.
//
// The fused H=64 kernels (pair_tc.cuh, edge_tc.cuh) keep a whole 128-pair
// filter chain in shared memory and TMEM.  At H=256 a chunk's B alone is
// 256 KB, so this path splits every phase at its contractions instead:
//   * per-pair contractions of a 128..27k-pair batch are dense GEMMs on
//     stacked operands ([phi; phi'] A, [s; sdot] B, [mu; nu] B^T, and the
//     weight gradients [s; sdot]^T [mu; nu], [phi; phi']^T [zbar; zbar'] with
//     K = 2 x pairs), issued through the stage's GEMM seam (stage_wide.inc);
//   * everything between them is one streaming elementwise kernel per step
//     (coalesced, one pass over [pairs x H]);
//   * the CSR gathers / scatters (m, Y, X, mdot, Y_b, forces) are warp-per-row
//     kernels: lane l owns features [l V, l V + V) of every row, so each edge
//     moves whole node rows in single coalesced 32 x V-float transactions, and
//     the per-edge force scalars are warp reductions (fixed order).
// Math: oracle/mlip_oracle.c (the same definitions), pair form as DESIGN §3.0.
#pragma once

#include "common.cuh"

namespace janus {
namespace wide {

using dev::d2silu;
using dev::dsilu;
using dev::silu;

template <int V>
__device__ __forceinline__ void ldv(const float* __restrict__ p, float (&x)[V]) {
  if constexpr (V % 4 == 0) {
#pragma unroll
    for (int q = 0; q < V / 4; ++q) {
      const float4 t = __ldg(reinterpret_cast<const float4*>(p) + q);
      x[4 * q] = t.x;
      x[4 * q + 1] = t.y;
      x[4 * q + 2] = t.z;
      x[4 * q + 3] = t.w;
    }
  } else if constexpr (V == 2) {
    const float2 t = __ldg(reinterpret_cast<const float2*>(p));
    x[0] = t.x;
    x[1] = t.y;
  } else {
#pragma unroll
    for (int q = 0; q < V; ++q) x[q] = __ldg(p + q);
  }
}

template <int V>
__device__ __forceinline__ void stv(float* __restrict__ p, const float (&x)[V]) {
  if constexpr (V % 4 == 0) {
#pragma unroll
    for (int q = 0; q < V / 4; ++q)
      reinterpret_cast<float4*>(p)[q] = make_float4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
  } else if constexpr (V == 2) {
    *reinterpret_cast<float2*>(p) = make_float2(x[0], x[1]);
  } else {
#pragma unroll
    for (int q = 0; q < V; ++q) p[q] = x[q];
  }
}

struct PairRec {  // pgeo (pair_tc.cuh pairs_kernel): (d, c, c', i | u, j) of the canonical edge
  float d, c, dc, ux, uy, uz;
  int i, j;
};
__device__ __forceinline__ PairRec pair_rec(const float4* __restrict__ pgeo, int p) {
  const float4 a = __ldg(pgeo + 2 * p), b = __ldg(pgeo + 2 * p + 1);
  return PairRec{a.x, a.y, a.z, b.x, b.y, b.z, __float_as_int(a.w), __float_as_int(b.w)};
}

// ---------------------------------------------------------------- pairs
// phi2 = [phi; phi'] [2 P][R] (Gaussian basis of the pair length and its d/dd)
__global__ void basis2_kernel(int P, int R, const float4* __restrict__ pgeo, float rc, float* __restrict__ phi2) {
  JANUS_GDC_WAIT();
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= static_cast<int64_t>(P) * R) return;
  const int p = static_cast<int>(x / R), k = static_cast<int>(x % R);
  const float d = __ldg(pgeo + 2 * p).x;
  const float delta = rc / (R - 1);
  const float gamma = 1.0f / (2.0f * delta * delta);
  const float t = d - k * delta;
  const float e = expf(-gamma * t * t);
  phi2[x] = e;
  phi2[static_cast<int64_t>(P) * R + x] = -2.0f * gamma * t * e;
}

// FE / BF: z2 = [phi A; phi' A] -> a2 = [s; sdot] = [SiLU(z + alpha); SiLU'(z + alpha) z']
__global__ void act2_kernel(int64_t PH, int H, const float* __restrict__ z2, const float* __restrict__ alpha,
                            float* __restrict__ a2) {
  JANUS_GDC_WAIT();
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= PH) return;
  const float z = z2[x] + __ldg(alpha + x % H), zp = z2[PH + x];
  a2[x] = silu(z);
  a2[PH + x] = dsilu(z) * zp;
}

// BE: a = SiLU(z + alpha) (first half only)
__global__ void act1_kernel(int64_t PH, int H, const float* __restrict__ z, const float* __restrict__ alpha,
                            float* __restrict__ a) {
  JANUS_GDC_WAIT();
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= PH) return;
  a[x] = silu(z[x] + __ldg(alpha + x % H));
}

// FE: g2 = [s B; sdot B] -> w = c (g + beta), w' = c' (g + beta) + c g'
__global__ void filter_out_kernel(int64_t PH, int H, const float* __restrict__ g2, const float* __restrict__ beta,
                                  const float4* __restrict__ pgeo, float* __restrict__ wf, float* __restrict__ wfp) {
  JANUS_GDC_WAIT();
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= PH) return;
  const float4 r = __ldg(pgeo + 2 * (x / H));
  const float g = g2[x] + __ldg(beta + x % H), gp = g2[PH + x];
  wf[x] = r.y * g;
  wfp[x] = r.z * g + r.y * gp;
}

// BF per pair (warp per pair): rho = a_m[i] v_j + a_m[j] v_i, kappa = a_m[i] vdot_j + a_m[j] vdot_i,
// qbar = <Fbar_i - Fbar_j, u>, mu = qbar c' rho + c kappa, nu = qbar c rho -> mn = [mu; nu]
template <int V>
__global__ void __launch_bounds__(256) bf_pair_kernel(int P, const float4* __restrict__ pgeo,
                                                      const float* __restrict__ am, const float* __restrict__ v,
                                                      const float* __restrict__ vd, const float* __restrict__ Fbar,
                                                      float* __restrict__ mn) {
  JANUS_GDC_WAIT();
  constexpr int H = 32 * V;
  const int p = static_cast<int>((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5), l = threadIdx.x & 31;
  if (p >= P) return;
  const PairRec r = pair_rec(pgeo, p);
  const float qb = (__ldg(Fbar + 3 * r.i) - __ldg(Fbar + 3 * r.j)) * r.ux +
                   (__ldg(Fbar + 3 * r.i + 1) - __ldg(Fbar + 3 * r.j + 1)) * r.uy +
                   (__ldg(Fbar + 3 * r.i + 2) - __ldg(Fbar + 3 * r.j + 2)) * r.uz;
  float ai[V], aj[V], vi[V], vj[V], di[V], dj[V];
  const size_t oi = static_cast<size_t>(r.i) * H + l * V, oj = static_cast<size_t>(r.j) * H + l * V;
  ldv<V>(am + oi, ai);
  ldv<V>(am + oj, aj);
  ldv<V>(v + oi, vi);
  ldv<V>(v + oj, vj);
  ldv<V>(vd + oi, di);
  ldv<V>(vd + oj, dj);
  float mu[V], nu[V];
#pragma unroll
  for (int q = 0; q < V; ++q) {
    const float rho = ai[q] * vj[q] + aj[q] * vi[q];
    const float kap = ai[q] * dj[q] + aj[q] * di[q];
    mu[q] = qb * r.dc * rho + r.c * kap;
    nu[q] = qb * r.c * rho;
  }
  const size_t o = static_cast<size_t>(p) * H + l * V;
  stv<V>(mn + o, mu);
  stv<V>(mn + static_cast<size_t>(P) * H + o, nu);
}

// BF: sb2 = [sbar; sdotbar] = [mu B^T; nu B^T], z2 = raw [phi A; phi' A] ->
// zb2 = [zbar; zbar'] = [sbar SiLU'(z) + sdotbar SiLU''(z) z'; sdotbar SiLU'(z)]
__global__ void bf_zbar_kernel(int64_t PH, int H, const float* __restrict__ sb2, const float* __restrict__ z2,
                               const float* __restrict__ alpha, float* __restrict__ zb2) {
  JANUS_GDC_WAIT();
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= PH) return;
  const float z = z2[x] + __ldg(alpha + x % H), zp = z2[PH + x];
  const float sb = sb2[x], sdb = sb2[PH + x], ds = dsilu(z);
  zb2[x] = sb * ds + sdb * d2silu(z) * zp;
  zb2[PH + x] = sdb * ds;
}

// BE per pair (warp per pair): gbar = c (b_m[i] v_j + b_m[j] v_i)
template <int V>
__global__ void __launch_bounds__(256) be_pair_kernel(int P, const float4* __restrict__ pgeo,
                                                      const float* __restrict__ bm, const float* __restrict__ v,
                                                      float* __restrict__ gbar) {
  JANUS_GDC_WAIT();
  constexpr int H = 32 * V;
  const int p = static_cast<int>((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5), l = threadIdx.x & 31;
  if (p >= P) return;
  const PairRec r = pair_rec(pgeo, p);
  float bi[V], bj[V], vi[V], vj[V], o[V];
  const size_t oi = static_cast<size_t>(r.i) * H + l * V, oj = static_cast<size_t>(r.j) * H + l * V;
  ldv<V>(bm + oi, bi);
  ldv<V>(bm + oj, bj);
  ldv<V>(v + oi, vi);
  ldv<V>(v + oj, vj);
#pragma unroll
  for (int q = 0; q < V; ++q) o[q] = r.c * (bi[q] * vj[q] + bj[q] * vi[q]);
  stv<V>(gbar + static_cast<size_t>(p) * H + l * V, o);
}

// BE: zbar = sbar SiLU'(z + alpha)  (in place on sbar)
__global__ void be_zbar_kernel(int64_t PH, int H, float* __restrict__ sb, const float* __restrict__ z,
                               const float* __restrict__ alpha) {
  JANUS_GDC_WAIT();
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= PH) return;
  sb[x] *= dsilu(z[x] + __ldg(alpha + x % H));
}

// ------------------------------------------------------------ row kernels
// kWpr warps per CSR row i (receiver), 2 rows per 256-thread block: warp q of
// a row takes the row's edges e0 + q, e0 + q + kWpr, ...; lane l owns features
// [l V, l V + V) of every node row, so each edge moves whole rows in single
// coalesced 32 x V-float transactions.  The kWpr partials are summed in warp
// order through shared memory (deterministic; 4x the warps of one warp per
// row, which left ~3 warps per SM at 512-atom micro-batches).
constexpr int kWpr = 4;
inline int rows_grid(int N) { return (N + 256 / (32 * kWpr) - 1) / (256 / (32 * kWpr)); }

template <int V>
__device__ __forceinline__ void row_reduce_store(float (&acc)[V], float* __restrict__ out, int i, int N, bool add = false) {
  constexpr int H = 32 * V;
  __shared__ float part[8][H];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, q = w % kWpr;
#pragma unroll
  for (int k = 0; k < V; ++k) part[w][l * V + k] = acc[k];
  __syncthreads();
  if (q == 0 && i < N) {
    float o[V];
#pragma unroll
    for (int k = 0; k < V; ++k) {
      float x = part[w][l * V + k];
#pragma unroll
      for (int r = 1; r < kWpr; ++r) x += part[w + r][l * V + k];
      o[k] = x;
    }
    if (add) {
      float prev[V];
      ldv<V>(out + static_cast<size_t>(i) * H + l * V, prev);
#pragma unroll
      for (int k = 0; k < V; ++k) o[k] += prev[k];
    }
    stv<V>(out + static_cast<size_t>(i) * H + l * V, o);
  }
  __syncthreads();
}

// FE: m_i = sum_e w_p(e) v_j  (BE: Y_b,i = sum_e w_p b_m[j])
template <int V>
__global__ void __launch_bounds__(256) fe_rows_kernel(int N, const int* __restrict__ row_ptr, const int* __restrict__ col,
                                                      const int* __restrict__ pidx, const float* __restrict__ wf,
                                                      const float* __restrict__ v, float* __restrict__ m) {
  JANUS_GDC_WAIT();
  constexpr int H = 32 * V;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, q = w % kWpr;
  const int i = blockIdx.x * (8 / kWpr) + w / kWpr;
  float acc[V] = {};
  if (i < N) {
    const int e1 = __ldg(row_ptr + i + 1);
#pragma unroll 2
    for (int e = __ldg(row_ptr + i) + q; e < e1; e += kWpr) {
      float wv[V], x[V];
      ldv<V>(wf + static_cast<size_t>(__ldg(pidx + e)) * H + l * V, wv);
      ldv<V>(v + static_cast<size_t>(__ldg(col + e)) * H + l * V, x);
#pragma unroll
      for (int k = 0; k < V; ++k) acc[k] += wv[k] * x[k];
    }
  }
  row_reduce_store<V>(acc, m, i, N);
}

// FF: Y_i = sum_e w_p a_m[j];  F_i += sum_e <a_m[i] v_j + a_m[j] v_i, w'_p> u_e
template <int V>
__global__ void __launch_bounds__(256) ff_rows_kernel(int N, const int* __restrict__ row_ptr, const int* __restrict__ col,
                                                      const int* __restrict__ pidx, const float* __restrict__ u,
                                                      const float* __restrict__ wf, const float* __restrict__ wfp,
                                                      const float* __restrict__ v, const float* __restrict__ am,
                                                      float* __restrict__ Y, float* __restrict__ F) {
  JANUS_GDC_WAIT();
  constexpr int H = 32 * V;
  __shared__ float fpart[8][3];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, q = w % kWpr;
  const int i = blockIdx.x * (8 / kWpr) + w / kWpr;
  float acc[V] = {};
  float fx = 0.f, fy = 0.f, fz = 0.f;
  if (i < N) {
    float ai[V], vi[V];
    ldv<V>(am + static_cast<size_t>(i) * H + l * V, ai);
    ldv<V>(v + static_cast<size_t>(i) * H + l * V, vi);
    const int e1 = __ldg(row_ptr + i + 1);
#pragma unroll 2
    for (int e = __ldg(row_ptr + i) + q; e < e1; e += kWpr) {
      const size_t op = static_cast<size_t>(__ldg(pidx + e)) * H + l * V, oj = static_cast<size_t>(__ldg(col + e)) * H + l * V;
      float wv[V], wp[V], aj[V], vj[V];
      ldv<V>(wf + op, wv);
      ldv<V>(wfp + op, wp);
      ldv<V>(am + oj, aj);
      ldv<V>(v + oj, vj);
      float qq = 0.f;
#pragma unroll
      for (int k = 0; k < V; ++k) {
        acc[k] += wv[k] * aj[k];
        qq += (ai[k] * vj[k] + aj[k] * vi[k]) * wp[k];
      }
      qq = dev::warp_sum(qq);
      fx += qq * __ldg(u + 3 * e);
      fy += qq * __ldg(u + 3 * e + 1);
      fz += qq * __ldg(u + 3 * e + 2);
    }
  }
  if (l == 0) {
    fpart[w][0] = fx;
    fpart[w][1] = fy;
    fpart[w][2] = fz;
  }
  row_reduce_store<V>(acc, Y, i, N);  // (its barriers also publish fpart)
  if (q == 0 && l < 3 && i < N) {
    float f = fpart[w][l];
#pragma unroll
    for (int r = 1; r < kWpr; ++r) f += fpart[w + r][l];
    F[3 * i + l] += f;
  }
}

// BF: mdot_i = sum_e qbar_e w'_p v_j + w_p vdot_j;  X_i = sum_e qbar_e w'_p a_m[j]
template <int V>
__global__ void __launch_bounds__(256) bf_rows_kernel(int N, const int* __restrict__ row_ptr, const int* __restrict__ col,
                                                      const int* __restrict__ pidx, const float* __restrict__ u,
                                                      const float* __restrict__ Fbar, const float* __restrict__ wf,
                                                      const float* __restrict__ wfp, const float* __restrict__ v,
                                                      const float* __restrict__ vd, const float* __restrict__ am,
                                                      float* __restrict__ mdot, float* __restrict__ X) {
  JANUS_GDC_WAIT();
  constexpr int H = 32 * V;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, q = w % kWpr;
  const int i = blockIdx.x * (8 / kWpr) + w / kWpr;
  float md[V] = {}, xs[V] = {};
  if (i < N) {
    const float fix = __ldg(Fbar + 3 * i), fiy = __ldg(Fbar + 3 * i + 1), fiz = __ldg(Fbar + 3 * i + 2);
    const int e1 = __ldg(row_ptr + i + 1);
#pragma unroll 2
    for (int e = __ldg(row_ptr + i) + q; e < e1; e += kWpr) {
      const int j = __ldg(col + e);
      const float qb = (fix - __ldg(Fbar + 3 * j)) * __ldg(u + 3 * e) + (fiy - __ldg(Fbar + 3 * j + 1)) * __ldg(u + 3 * e + 1) +
                       (fiz - __ldg(Fbar + 3 * j + 2)) * __ldg(u + 3 * e + 2);
      const size_t op = static_cast<size_t>(__ldg(pidx + e)) * H + l * V, oj = static_cast<size_t>(j) * H + l * V;
      float wv[V], wp[V], vj[V], dj[V], aj[V];
      ldv<V>(wf + op, wv);
      ldv<V>(wfp + op, wp);
      ldv<V>(v + oj, vj);
      ldv<V>(vd + oj, dj);
      ldv<V>(am + oj, aj);
#pragma unroll
      for (int k = 0; k < V; ++k) {
        md[k] += qb * wp[k] * vj[k] + wv[k] * dj[k];
        xs[k] += qb * wp[k] * aj[k];
      }
    }
  }
  row_reduce_store<V>(md, mdot, i, N);
  row_reduce_store<V>(xs, X, i, N);
}

// (BE's Y_b,i = sum_e w_p b_m[j] is fe_rows_kernel with x = b_m)

// ------------------------------------------------------------- node kernels
__global__ void embed_kernel(int64_t NH, int H, const int* __restrict__ species, const float* __restrict__ Emb,
                             float* __restrict__ h) {
  JANUS_GDC_WAIT();
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x < NH) h[x] = __ldg(Emb + static_cast<int64_t>(__ldg(species + x / H)) * H + x % H);
}

// p += bias (per column); sp = SiLU(p)
__global__ void bias_silu_kernel(int64_t NH, int H, float* __restrict__ p, const float* __restrict__ bias,
                                 float* __restrict__ sp) {
  JANUS_GDC_WAIT();
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= NH) return;
  const float y = p[x] + __ldg(bias + x % H);
  p[x] = y;
  if (sp) sp[x] = silu(y);
}

// x *= SiLU'(p)
__global__ void mul_dsilu_kernel(int64_t NH, float* __restrict__ x, const float* __restrict__ p) {
  JANUS_GDC_WAIT();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < NH) x[i] *= dsilu(p[i]);
}

// BF upd: pb = r pdot SiLU''(p), pdb = r SiLU'(p), spd = SiLU'(p) pdot
__global__ void bf_upd_ew_kernel(int64_t NH, const float* __restrict__ r, const float* __restrict__ pdot,
                                 const float* __restrict__ p, float* __restrict__ pb, float* __restrict__ pdb,
                                 float* __restrict__ spd) {
  JANUS_GDC_WAIT();
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= NH) return;
  const float pp = p[x], pd = pdot[x], rr = r[x], ds = dsilu(pp);
  pb[x] = rr * pd * d2silu(pp);
  pdb[x] = rr * ds;
  spd[x] = ds * pd;
}

// BE upd: pb = r SiLU'(p), sp = SiLU(p)
__global__ void be_upd_ew_kernel(int64_t NH, const float* __restrict__ r, const float* __restrict__ p,
                                 float* __restrict__ pb, float* __restrict__ sp) {
  JANUS_GDC_WAIT();
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= NH) return;
  const float pp = p[x];
  pb[x] = r[x] * dsilu(pp);
  sp[x] = silu(pp);
}

// readout FE (warp per atom): t += o; e_i = bias[Z_i] + sum_k SiLU(t_k) omega_k (fixed-order warp sum)
__global__ void ro_fe_kernel(int N, int H, float* __restrict__ t, const float* __restrict__ o,
                             const float* __restrict__ om, const float* __restrict__ bias,
                             const int* __restrict__ species, float* __restrict__ e_atom) {
  JANUS_GDC_WAIT();
  const int i = static_cast<int>((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5), l = threadIdx.x & 31;
  if (i >= N) return;
  float acc = 0.f;
  for (int k = l; k < H; k += 32) {
    const float y = t[static_cast<size_t>(i) * H + k] + __ldg(o + k);
    t[static_cast<size_t>(i) * H + k] = y;
    acc += silu(y) * __ldg(om + k);
  }
  acc = dev::warp_sum(acc);
  if (l == 0) e_atom[i] = acc + __ldg(bias + __ldg(species + i));
}

// readout FF: out = SiLU'(t) omega
__global__ void ro_ff_ew_kernel(int64_t NH, int H, const float* __restrict__ t, const float* __restrict__ om,
                                float* __restrict__ out) {
  JANUS_GDC_WAIT();
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x < NH) out[x] = dsilu(t[x]) * __ldg(om + x % H);
}

// readout BF: x1 = tdot SiLU'(t) (-> domega), tau = tdot omega SiLU''(t), y = SiLU'(t) omega
__global__ void ro_bf_ew_kernel(int64_t NH, int H, const float* __restrict__ tdot, const float* __restrict__ t,
                                const float* __restrict__ om, float* __restrict__ x1, float* __restrict__ tau,
                                float* __restrict__ y) {
  JANUS_GDC_WAIT();
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= NH) return;
  const float tt = t[x], td = tdot[x], w = __ldg(om + x % H), ds = dsilu(tt);
  x1[x] = td * ds;
  tau[x] = td * w * d2silu(tt);
  y[x] = ds * w;
}

// readout BE: tb = eps_s SiLU'(t) omega, x2 = eps_s SiLU(t)
__global__ void ro_be_ew_kernel(int64_t NH, int H, const float* __restrict__ t, const float* __restrict__ om,
                                const float* __restrict__ eps, const int* __restrict__ struct_id,
                                float* __restrict__ tb, float* __restrict__ x2) {
  JANUS_GDC_WAIT();
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= NH) return;
  const float ep = __ldg(eps + __ldg(struct_id + x / H)), tt = t[x];
  tb[x] = ep * dsilu(tt) * __ldg(om + x % H);
  x2[x] = ep * silu(tt);
}

// out[z][k] += sum_{Z_i = z} x[i][k] (x != null, cols = H) or
// out[z] += sum_{Z_i = z} eps[s(i)] (x == null, cols = 1).  Block (32-column
// strip, species z), 8 warps: lane = column, warp w takes atoms i = w mod 8,
// the 8 partials are summed in warp order (deterministic).
__global__ void __launch_bounds__(256) species_sum_kernel(int N, int S, int cols, const int* __restrict__ species,
                                                          const float* __restrict__ x, const float* __restrict__ eps,
                                                          const int* __restrict__ struct_id, float* __restrict__ out) {
  JANUS_GDC_WAIT();
  __shared__ float part[8][33];
  const int z = blockIdx.y, l = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int k = blockIdx.x * 32 + l;
  float acc = 0.f;
  if (k < cols)
    for (int i = w; i < N; i += 8) {
      if (__ldg(species + i) != z) continue;
      acc += x ? __ldg(x + static_cast<size_t>(i) * cols + k) : __ldg(eps + __ldg(struct_id + i));
    }
  part[w][l] = acc;
  __syncthreads();
  if (w == 0 && k < cols) {
    float s = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += part[q][l];
    out[static_cast<size_t>(z) * cols + k] += s;
  }
}

// Column sums out[c] += sum_r X[r][c] in ONE deterministic launch: block
// (strip of 32 columns, chunk g of rows) sums its rows (8 warps interleave,
// up to kColRows / 8 independent loads in flight per thread, combined in warp
// order) into part[g][c]; the last block of a strip to finish (atomic ticket,
// counter reset by it) adds the chunks' partials — warp w the chunks w, w + 8,
// ..., then the 8 warp sums in warp order (a single thread walking all
// chunks was the long pole).  The arrival order decides only WHICH block
// sums, never the order of the sum.  256-row chunks: inside the 8-lane
// configs[2] step 64-row chunks (4x the blocks) measured 148.5 vs 152.6
// structures/s; 512 / 1024 rows are within noise of 256.
constexpr int kColChunks = 256;
constexpr int kColRows = 256;
__global__ void __launch_bounds__(256) colsum_kernel(int rows, int cols, const float* __restrict__ X,
                                                     float* __restrict__ part, unsigned* __restrict__ ticket,
                                                     float* __restrict__ out) {
  JANUS_GDC_WAIT();
  __shared__ float red[8][33];
  __shared__ bool last;
  const int l = threadIdx.x & 31, w = threadIdx.x >> 5, k = blockIdx.x * 32 + l, g = blockIdx.y;
  const int per = (rows + gridDim.y - 1) / gridDim.y, r0 = g * per, r1 = min(rows, r0 + per);
  float acc = 0.f;
  if (k < cols)
#pragma unroll 8
    for (int r = r0 + w; r < r1; r += 8) acc += __ldg(X + static_cast<size_t>(r) * cols + k);
  red[w][l] = acc;
  __syncthreads();
  if (w == 0) {
    float sum = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) sum += red[q][l];
    if (k < cols) part[static_cast<size_t>(g) * cols + k] = sum;
    __threadfence();
  }
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket + blockIdx.x, 1u) == gridDim.y - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  float sum = 0.f;
  if (k < cols)
#pragma unroll 8
    for (int q = w; q < static_cast<int>(gridDim.y); q += 8) sum += __ldcg(part + static_cast<size_t>(q) * cols + k);
  red[w][l] = sum;
  __syncthreads();
  if (w == 0) {
    float tot = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) tot += red[q][l];
    if (k < cols) out[k] += tot;
    if (l == 0) ticket[blockIdx.x] = 0u;  // ready for the next launch on this lane
  }
}

// C[x] += sum_b W[b][x] over the K slices of gemm_tn_long, in slice order
__global__ void sum_slices_kernel(int64_t n, int slices, const float* __restrict__ W, float* __restrict__ C) {
  JANUS_GDC_WAIT();
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= n) return;
  float acc = 0.f;
  for (int b = 0; b < slices; ++b) acc += W[static_cast<size_t>(b) * n + x];
  C[x] += acc;
}

// dst[c][r] = src[r][c] for a [rows x cols] matrix (weight transposes, once per optimizer step)
__global__ void transpose_any_kernel(int rows, int cols, const float* __restrict__ src, float* __restrict__ dst) {
  JANUS_GDC_WAIT();
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= rows * cols) return;
  const int r = x / cols, c = x % cols;
  dst[static_cast<size_t>(c) * rows + r] = src[x];
}

__global__ void fill_kernel(int64_t n, float* __restrict__ p, float v) {
  JANUS_GDC_WAIT();
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x < n) p[x] = v;
}

}  // namespace wide
}  // namespace janus
