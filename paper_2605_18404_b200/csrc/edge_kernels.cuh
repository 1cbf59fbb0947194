// edge_kernels.cuh — the msg unit (edge filter MLP + CSR aggregation) in all
// four phases, SIMT fp32 (the parity mode).  Math: DESIGN.md §3 / SURVEY.md
// Appendix A.2-A.3; the fp64 oracle is oracle/mlip_oracle.c (msg branches).
//
// Layout / work decomposition (B200):
//  * Edges are CSR-sorted by receiver i.  A "row tile" is a run of <= 8
//    consecutive rows holding <= TE edges (or one long row, processed in
//    TE-edge chunks).  One CTA (256 threads, 8 warps) per tile.
//  * Per chunk, per-edge vectors live in shared memory as [feature][edge]
//    (leading dim TE+1 => conflict-free column access); thread t owns edge
//    t % TE and a column quarter t / TE of every per-edge GEMM.
//  * Warp w owns row w of the tile: segmented sums over the row's edges are
//    sequential in edge order per lane (deterministic, no atomics) with the
//    per-row accumulators in registers across chunks.
//  * The neighbour list is symmetric (every (i,j,s) has (j,i,-s)) and every
//    per-edge filter depends only on |r|, so the transposed (CSC, by sender)
//    aggregations of FF/BF/BE are evaluated as CSR gathers:
//      sum_{e: j(e)=j} f_e * x[i(e)] == sum_{e in row j} f_e * x[col(e)].
//    The oracle computes them as explicit scatters (independent check).
//  * Weight gradients over edges: per-tile partials [A|alpha|B|beta] written
//    to a workspace, reduced in tile order by reduce_partials (deterministic).
#pragma once

#include "common.cuh"

namespace janus {

struct EdgeGeom {
  int n_atoms, n_edges, n_tiles;
  const int* row_ptr;   // [N+1]
  const int* col;       // [E] sender j
  const int* src;       // [E] receiver i
  const int* rev;       // [E] reverse edge
  const int* tile_row;  // [n_tiles+1]
  const float* d;       // [E]
  const float* u;       // [E*3] unit vector r/|r|
  const float* c;       // [E] cosine cutoff
  const float* dc;      // [E] its derivative
};

struct MsgParams {
  const float* A;      // [R][H]
  const float* alpha;  // [H]
  const float* B;      // [H][H]
  const float* beta;   // [H]
  const float* Bt;     // [H][H] transposed copy of B
  const float* pack;   // tensor-core image: [A^T | B^T | B] SW128 tiles, alpha, beta (edge_tc.cuh)
};

namespace edge {

constexpr int TE = 64;        // edges per chunk
constexpr int NT = 256;       // threads per CTA
constexpr int HQ = NT / TE;   // column groups per edge
constexpr int LD = TE + 1;    // smem leading dim of [feature][edge] arrays
constexpr int kRowsPerTile = NT / 32;

template <int H, int R>
struct Cfg {
  static_assert(H % (HQ * 4) == 0 && R % HQ == 0, "H must be a multiple of 16, R of 4");
  static constexpr int HC = H / HQ;  // columns per thread
  static constexpr int RC = R / HQ;  // basis rows per thread
  static constexpr int PE = R * H + H + H * H + H;  // edge-parameter partial size
};

// ---------------------------------------------------------------- helpers
template <int N>
__device__ __forceinline__ void load_smem(float* dst, const float* __restrict__ src) {
  static_assert(N % 4 == 0, "");
  const float4* s4 = reinterpret_cast<const float4*>(src);
  float4* d4 = reinterpret_cast<float4*>(dst);
  for (int i = threadIdx.x; i < N / 4; i += NT) d4[i] = s4[i];
}

// acc[j] = sum_k in[k][e] * W[k][h0 + j]   (W row-major [K][H] in smem)
template <int K, int H, int HC>
__device__ __forceinline__ void gemm_edge(const float* in, const float* W, int e, int h0, float (&acc)[HC]) {
#pragma unroll
  for (int j = 0; j < HC; ++j) acc[j] = 0.f;
#pragma unroll 4
  for (int k = 0; k < K; ++k) {
    const float a = in[k * LD + e];
    const float4* w = reinterpret_cast<const float4*>(W + k * H + h0);
#pragma unroll
    for (int q = 0; q < HC / 4; ++q) {
      const float4 x = w[q];
      acc[4 * q + 0] = fmaf(a, x.x, acc[4 * q + 0]);
      acc[4 * q + 1] = fmaf(a, x.y, acc[4 * q + 1]);
      acc[4 * q + 2] = fmaf(a, x.z, acc[4 * q + 2]);
      acc[4 * q + 3] = fmaf(a, x.w, acc[4 * q + 3]);
    }
  }
}

// Weight-gradient micro-tile: G[k][h] += sum_{e<ne} a[k][e] * b[h][e], thread
// owns a (K/16) x (H/16) block.  ne masks nothing (masked edges carry zeros).
template <int K, int H>
struct WGrad {
  static constexpr int KR = K / 16, HR = H / 16;
  float acc[KR][HR];
  __device__ void zero() {
#pragma unroll
    for (int a = 0; a < KR; ++a)
#pragma unroll
      for (int b = 0; b < HR; ++b) acc[a][b] = 0.f;
  }
  __device__ __forceinline__ void add(const float* A, const float* Bm, int ne) {
    const int kb = (threadIdx.x >> 4) * KR, hb = (threadIdx.x & 15) * HR;
    for (int e = 0; e < ne; ++e) {
      float x[KR], y[HR];
#pragma unroll
      for (int a = 0; a < KR; ++a) x[a] = A[(kb + a) * LD + e];
#pragma unroll
      for (int b = 0; b < HR; ++b) y[b] = Bm[(hb + b) * LD + e];
#pragma unroll
      for (int a = 0; a < KR; ++a)
#pragma unroll
        for (int b = 0; b < HR; ++b) acc[a][b] = fmaf(x[a], y[b], acc[a][b]);
    }
  }
  __device__ void store(float* out) const {  // out row-major [K][H]
    const int kb = (threadIdx.x >> 4) * KR, hb = (threadIdx.x & 15) * HR;
#pragma unroll
    for (int a = 0; a < KR; ++a)
#pragma unroll
      for (int b = 0; b < HR; ++b) out[(kb + a) * H + hb + b] = acc[a][b];
  }
};

struct Tile {
  int r0, r1, e0, e1;
};

__device__ __forceinline__ Tile tile_of(const EdgeGeom& g) {
  Tile t;
  t.r0 = g.tile_row[blockIdx.x];
  t.r1 = g.tile_row[blockIdx.x + 1];
  t.e0 = g.row_ptr[t.r0];
  t.e1 = g.row_ptr[t.r1];
  return t;
}

// Per-chunk edge scalars + radial basis (and derivative) into smem.
template <int R, bool kDeriv>
__device__ __forceinline__ void chunk_basis(const EdgeGeom& g, float rc, int c0, int ne, float* sC, float* sDC,
                                            float* P0, float* P1) {
  const int e = threadIdx.x % TE, hq = threadIdx.x / TE;
  const bool valid = e < ne;
  const float d = valid ? g.d[c0 + e] : 0.f;
  if (hq == 0) {
    sC[e] = valid ? g.c[c0 + e] : 0.f;
    if (sDC) sDC[e] = valid ? g.dc[c0 + e] : 0.f;
  }
  const float delta = rc / (R - 1);
  const float gamma = 1.0f / (2.0f * delta * delta);
  constexpr int RC = R / HQ;
#pragma unroll 4
  for (int k = hq * RC; k < hq * RC + RC; ++k) {
    const float x = d - k * delta;
    const float p = expf(-gamma * x * x);
    P0[k * LD + e] = p;
    if (kDeriv) P1[k * LD + e] = -2.0f * gamma * x * p;
  }
}

// ------------------------------------------------------------------- FE
// m_i = sum_{e in row i} w_e * v[col e],  w = c (SiLU(phi A + alpha) B + beta)
template <int H, int R>
__global__ void __launch_bounds__(NT) msg_fe_kernel(EdgeGeom g, MsgParams p, float rc, const float* __restrict__ v,
                                                    float* __restrict__ m_out) {
  JANUS_GDC_WAIT();
  using C = Cfg<H, R>;
  extern __shared__ __align__(16) float sm[];
  float* sA = sm;
  float* sB = sA + R * H;
  float* sAl = sB + H * H;
  float* sBe = sAl + H;
  float* P0 = sBe + H;      // phi, later w
  float* S = P0 + R * LD;   // silu(z)
  float* sC = S + H * LD;
  load_smem<R * H>(sA, p.A);
  load_smem<H * H>(sB, p.B);
  load_smem<H>(sAl, p.alpha);
  load_smem<H>(sBe, p.beta);
  const Tile t = tile_of(g);
  const int e = threadIdx.x % TE, h0 = (threadIdx.x / TE) * C::HC;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = t.r0 + warp;
  const bool has_row = row < t.r1;
  float acc_m[H / 32];
#pragma unroll
  for (int q = 0; q < H / 32; ++q) acc_m[q] = 0.f;
  __syncthreads();
  for (int c0 = t.e0; c0 < t.e1; c0 += TE) {
    const int ne = min(TE, t.e1 - c0);
    chunk_basis<R, false>(g, rc, c0, ne, sC, nullptr, P0, nullptr);
    __syncthreads();
    float acc[C::HC];
    gemm_edge<R, H, C::HC>(P0, sA, e, h0, acc);
#pragma unroll
    for (int j = 0; j < C::HC; ++j) S[(h0 + j) * LD + e] = dev::silu(acc[j] + sAl[h0 + j]);
    __syncthreads();
    gemm_edge<H, H, C::HC>(S, sB, e, h0, acc);
    __syncthreads();  // P0 (phi) fully consumed
    const float ce = sC[e];
#pragma unroll
    for (int j = 0; j < C::HC; ++j) P0[(h0 + j) * LD + e] = ce * (acc[j] + sBe[h0 + j]);
    __syncthreads();
    if (has_row) {
      const int eb = max(g.row_ptr[row], c0), ee = min(g.row_ptr[row + 1], c0 + ne);
      for (int x = eb; x < ee; ++x) {
        const int j = g.col[x], le = x - c0;
#pragma unroll
        for (int q = 0; q < H / 32; ++q) acc_m[q] = fmaf(P0[(lane + 32 * q) * LD + le], v[(size_t)j * H + lane + 32 * q], acc_m[q]);
      }
    }
    __syncthreads();
  }
  if (has_row) {
#pragma unroll
    for (int q = 0; q < H / 32; ++q) m_out[(size_t)row * H + lane + 32 * q] = acc_m[q];
  }
}

// ------------------------------------------------------------------- FF
// Y_i = sum_{e in row i} w_e * am[col e]     (transposed scatter via symmetry)
// q_e = < am[i] * v[j], w'_e >,  w' = c' g + c (SiLU'(z) z') B, and the force
// F_i += sum_{e in row i} (q_e + q_rev(e)) u_e where, w' being symmetric,
// q_rev(e) = < am[j] * v[i], w'_e > is evaluated in the same tile (no q buffer,
// no separate scatter kernel; the row's warp owns F_i => deterministic).
template <int H, int R>
__global__ void __launch_bounds__(NT) msg_ff_kernel(EdgeGeom g, MsgParams p, float rc, const float* __restrict__ v,
                                                    const float* __restrict__ am, float* __restrict__ Y_out,
                                                    float* __restrict__ F) {
  JANUS_GDC_WAIT();
  using C = Cfg<H, R>;
  extern __shared__ __align__(16) float sm[];
  float* sA = sm;
  float* sB = sA + R * H;
  float* sAl = sB + H * H;
  float* sBe = sAl + H;
  float* P0 = sBe + H;     // phi  -> w
  float* P1 = P0 + R * LD; // phi' -> w'
  float* S = P1 + R * LD;  // s
  float* Sp = S + H * LD;  // sdot
  float* sC = Sp + H * LD;
  float* sDC = sC + TE;
  load_smem<R * H>(sA, p.A);
  load_smem<H * H>(sB, p.B);
  load_smem<H>(sAl, p.alpha);
  load_smem<H>(sBe, p.beta);
  const Tile t = tile_of(g);
  const int e = threadIdx.x % TE, h0 = (threadIdx.x / TE) * C::HC;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = t.r0 + warp;
  const bool has_row = row < t.r1;
  float acc_y[H / 32];
#pragma unroll
  for (int q = 0; q < H / 32; ++q) acc_y[q] = 0.f;
  float am_i[H / 32], v_i[H / 32];
  float fx = 0.f, fy = 0.f, fz = 0.f;
  if (has_row) {
#pragma unroll
    for (int q = 0; q < H / 32; ++q) {
      am_i[q] = am[(size_t)row * H + lane + 32 * q];
      v_i[q] = v[(size_t)row * H + lane + 32 * q];
    }
  }
  __syncthreads();
  for (int c0 = t.e0; c0 < t.e1; c0 += TE) {
    const int ne = min(TE, t.e1 - c0);
    chunk_basis<R, true>(g, rc, c0, ne, sC, sDC, P0, P1);
    __syncthreads();
    {
      float z[C::HC], zp[C::HC];
      gemm_edge<R, H, C::HC>(P0, sA, e, h0, z);
      gemm_edge<R, H, C::HC>(P1, sA, e, h0, zp);
#pragma unroll
      for (int j = 0; j < C::HC; ++j) {
        const float zz = z[j] + sAl[h0 + j];
        S[(h0 + j) * LD + e] = dev::silu(zz);
        Sp[(h0 + j) * LD + e] = dev::dsilu(zz) * zp[j];
      }
    }
    __syncthreads();
    {
      float gg[C::HC], gp[C::HC];
      gemm_edge<H, H, C::HC>(S, sB, e, h0, gg);
      gemm_edge<H, H, C::HC>(Sp, sB, e, h0, gp);
      __syncthreads();
      const float ce = sC[e], dce = sDC[e];
#pragma unroll
      for (int j = 0; j < C::HC; ++j) {
        const float gb = gg[j] + sBe[h0 + j];
        P0[(h0 + j) * LD + e] = ce * gb;               // w
        P1[(h0 + j) * LD + e] = dce * gb + ce * gp[j]; // w'
      }
    }
    __syncthreads();
    if (has_row) {
      const int eb = max(g.row_ptr[row], c0), ee = min(g.row_ptr[row + 1], c0 + ne);
      for (int x = eb; x < ee; ++x) {
        const int j = g.col[x], le = x - c0;
        float part = 0.f;
#pragma unroll
        for (int q = 0; q < H / 32; ++q) {
          const int h = lane + 32 * q;
          const float amj = am[(size_t)j * H + h];
          acc_y[q] = fmaf(P0[h * LD + le], amj, acc_y[q]);
          part = fmaf(fmaf(am_i[q], v[(size_t)j * H + h], amj * v_i[q]), P1[h * LD + le], part);
        }
        part = dev::warp_sum(part);  // q_e + q_rev(e), identical in every lane
        fx = fmaf(part, g.u[3 * x + 0], fx);
        fy = fmaf(part, g.u[3 * x + 1], fy);
        fz = fmaf(part, g.u[3 * x + 2], fz);
      }
    }
    __syncthreads();
  }
  if (has_row) {
#pragma unroll
    for (int q = 0; q < H / 32; ++q) Y_out[(size_t)row * H + lane + 32 * q] = acc_y[q];
    if (lane == 0) {
      F[3 * row + 0] += fx;
      F[3 * row + 1] += fy;
      F[3 * row + 2] += fz;
    }
  }
}

// ------------------------------------------------------------------- BF
// Inputs: v = hW, vdot = abar_h W, am (FF input adjoint on m), Fbar.
// Outputs: mdot_i = sum_e qb c' ... (abar_m), X_i (for h-injection / W grad),
// per-tile partial [dA | dalpha | dB | dbeta] of the second-order term.
template <int H, int R>
__global__ void __launch_bounds__(NT, 1) msg_bf_kernel(EdgeGeom g, MsgParams p, float rc,
                                                       const float* __restrict__ v, const float* __restrict__ vdot,
                                                       const float* __restrict__ am, const float* __restrict__ Fbar,
                                                       float* __restrict__ mdot_out, float* __restrict__ X_out,
                                                       float* __restrict__ partial) {
  JANUS_GDC_WAIT();
  using C = Cfg<H, R>;
  extern __shared__ __align__(16) float sm[];
  float* sA = sm;
  float* sB = sA + R * H;
  float* sBt = sB + H * H;
  float* sAl = sBt + H * H;
  float* sBe = sAl + H;
  float* P0 = sBe + H;     // phi
  float* P1 = P0 + R * LD; // phi'
  float* Z = P1 + R * LD;  // z      -> zbar
  float* Zp = Z + H * LD;  // z'     -> zbar'
  float* S = Zp + H * LD;  // s      -> sbar
  float* Sp = S + H * LD;  // sdot   -> sdotbar
  float* G = Sp + H * LD;  // w      -> mu
  float* Gp = G + H * LD;  // w'     -> nu
  float* sC = Gp + H * LD;
  float* sDC = sC + TE;
  float* sQb = sDC + TE;
  load_smem<R * H>(sA, p.A);
  load_smem<H * H>(sB, p.B);
  load_smem<H * H>(sBt, p.Bt);
  load_smem<H>(sAl, p.alpha);
  load_smem<H>(sBe, p.beta);
  const Tile t = tile_of(g);
  const int e = threadIdx.x % TE, h0 = (threadIdx.x / TE) * C::HC;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = t.r0 + warp;
  const bool has_row = row < t.r1;
  float acc_md[H / 32], acc_x[H / 32];
#pragma unroll
  for (int q = 0; q < H / 32; ++q) acc_md[q] = acc_x[q] = 0.f;
  WGrad<R, H> gA;
  WGrad<H, H> gB;
  gA.zero();
  gB.zero();
  float gal = 0.f, gbe = 0.f;  // thread h = threadIdx.x < H owns alpha/beta column h
  __syncthreads();
  for (int c0 = t.e0; c0 < t.e1; c0 += TE) {
    const int ne = min(TE, t.e1 - c0);
    chunk_basis<R, true>(g, rc, c0, ne, sC, sDC, P0, P1);
    if (threadIdx.x < TE) {  // qbar_e = <Fbar_i - Fbar_j, u_e>
      float qb = 0.f;
      if (e < ne) {
        const int x = c0 + e, i = g.src[x], j = g.col[x];
#pragma unroll
        for (int k = 0; k < 3; ++k) qb = fmaf(Fbar[3 * i + k] - Fbar[3 * j + k], g.u[3 * x + k], qb);
      }
      sQb[e] = qb;
    }
    __syncthreads();
    {
      float z[C::HC], zp[C::HC];
      gemm_edge<R, H, C::HC>(P0, sA, e, h0, z);
      gemm_edge<R, H, C::HC>(P1, sA, e, h0, zp);
#pragma unroll
      for (int j = 0; j < C::HC; ++j) {
        const float zz = z[j] + sAl[h0 + j];
        Z[(h0 + j) * LD + e] = zz;
        Zp[(h0 + j) * LD + e] = zp[j];
        S[(h0 + j) * LD + e] = dev::silu(zz);
        Sp[(h0 + j) * LD + e] = dev::dsilu(zz) * zp[j];
      }
    }
    __syncthreads();
    {
      float gg[C::HC], gp[C::HC];
      gemm_edge<H, H, C::HC>(S, sB, e, h0, gg);
      gemm_edge<H, H, C::HC>(Sp, sB, e, h0, gp);
      const float ce = sC[e], dce = sDC[e];
#pragma unroll
      for (int j = 0; j < C::HC; ++j) {
        const float gb = gg[j] + sBe[h0 + j];
        G[(h0 + j) * LD + e] = ce * gb;               // w
        Gp[(h0 + j) * LD + e] = dce * gb + ce * gp[j]; // w'
      }
    }
    __syncthreads();
    // segmented row sums: mdot_i += qb w' v_j + w vdot_j ; X_i += qb w' am_j
    if (has_row) {
      const int eb = max(g.row_ptr[row], c0), ee = min(g.row_ptr[row + 1], c0 + ne);
      for (int x = eb; x < ee; ++x) {
        const int j = g.col[x], le = x - c0;
        const float qb = sQb[le];
#pragma unroll
        for (int q = 0; q < H / 32; ++q) {
          const int h = lane + 32 * q;
          const float wp = qb * Gp[h * LD + le];
          acc_md[q] = fmaf(wp, v[(size_t)j * H + h], fmaf(G[h * LD + le], vdot[(size_t)j * H + h], acc_md[q]));
          acc_x[q] = fmaf(wp, am[(size_t)j * H + h], acc_x[q]);
        }
      }
    }
    __syncthreads();
    // mu = qb c' rho + c kappa, nu = qb c rho with rho = am_i v_j, kappa = am_i vdot_j
    {
      const bool valid = e < ne;
      const int x = c0 + e;
      const int i = valid ? g.src[x] : 0, j = valid ? g.col[x] : 0;
      const float qb = sQb[e], ce = sC[e], dce = sDC[e];
#pragma unroll
      for (int q4 = 0; q4 < C::HC / 4; ++q4) {
        const int h = h0 + 4 * q4;
        float4 a4 = make_float4(0.f, 0.f, 0.f, 0.f), v4 = a4, vd4 = a4;
        if (valid) {
          a4 = *reinterpret_cast<const float4*>(am + (size_t)i * H + h);
          v4 = *reinterpret_cast<const float4*>(v + (size_t)j * H + h);
          vd4 = *reinterpret_cast<const float4*>(vdot + (size_t)j * H + h);
        }
        const float av[4] = {a4.x, a4.y, a4.z, a4.w}, vv[4] = {v4.x, v4.y, v4.z, v4.w},
                    vdv[4] = {vd4.x, vd4.y, vd4.z, vd4.w};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const float rho = av[r] * vv[r], kap = av[r] * vdv[r];
          G[(h + r) * LD + e] = qb * dce * rho + ce * kap;
          Gp[(h + r) * LD + e] = qb * ce * rho;
        }
      }
    }
    __syncthreads();
    gB.add(S, G, ne);
    gB.add(Sp, Gp, ne);
    if (threadIdx.x < H) {
      for (int x = 0; x < ne; ++x) gbe += G[threadIdx.x * LD + x];
    }
    __syncthreads();
    {  // sbar = mu B^T, sdotbar = nu B^T ; zbar, zbar'
      float sb[C::HC], sdb[C::HC];
      gemm_edge<H, H, C::HC>(G, sBt, e, h0, sb);
      gemm_edge<H, H, C::HC>(Gp, sBt, e, h0, sdb);
#pragma unroll
      for (int j = 0; j < C::HC; ++j) {
        const int h = h0 + j;
        const float zz = Z[h * LD + e], zp = Zp[h * LD + e];
        const float ds = dev::dsilu(zz);
        Z[h * LD + e] = sb[j] * ds + sdb[j] * dev::d2silu(zz) * zp;
        Zp[h * LD + e] = sdb[j] * ds;
      }
    }
    __syncthreads();
    gA.add(P0, Z, ne);
    gA.add(P1, Zp, ne);
    if (threadIdx.x < H) {
      for (int x = 0; x < ne; ++x) gal += Z[threadIdx.x * LD + x];
    }
    __syncthreads();
  }
  if (has_row) {
#pragma unroll
    for (int q = 0; q < H / 32; ++q) {
      mdot_out[(size_t)row * H + lane + 32 * q] = acc_md[q];
      X_out[(size_t)row * H + lane + 32 * q] = acc_x[q];
    }
  }
  float* part = partial + (size_t)blockIdx.x * C::PE;
  gA.store(part);
  gB.store(part + R * H + H);
  if (threadIdx.x < H) {
    part[R * H + threadIdx.x] = gal;
    part[R * H + H + H * H + threadIdx.x] = gbe;
  }
}

// ------------------------------------------------------------------- BE
// Yb_i = sum_{e in row i} w_e * bm[col e];  gbar = c bm_i v_j;
// dB = s^T gbar, dbeta = sum gbar, zbar = (gbar B^T) SiLU'(z), dA = phi^T zbar.
template <int H, int R>
__global__ void __launch_bounds__(NT) msg_be_kernel(EdgeGeom g, MsgParams p, float rc, const float* __restrict__ v,
                                                    const float* __restrict__ bm, float* __restrict__ Yb_out,
                                                    float* __restrict__ partial) {
  JANUS_GDC_WAIT();
  using C = Cfg<H, R>;
  extern __shared__ __align__(16) float sm[];
  float* sA = sm;
  float* sB = sA + R * H;
  float* sBt = sB + H * H;
  float* sAl = sBt + H * H;
  float* sBe = sAl + H;
  float* P0 = sBe + H;     // phi
  float* Z = P0 + R * LD;  // z -> zbar
  float* S = Z + H * LD;   // s
  float* G = S + H * LD;   // w -> gbar
  float* sC = G + H * LD;
  load_smem<R * H>(sA, p.A);
  load_smem<H * H>(sB, p.B);
  load_smem<H * H>(sBt, p.Bt);
  load_smem<H>(sAl, p.alpha);
  load_smem<H>(sBe, p.beta);
  const Tile t = tile_of(g);
  const int e = threadIdx.x % TE, h0 = (threadIdx.x / TE) * C::HC;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = t.r0 + warp;
  const bool has_row = row < t.r1;
  float acc_y[H / 32];
#pragma unroll
  for (int q = 0; q < H / 32; ++q) acc_y[q] = 0.f;
  WGrad<R, H> gA;
  WGrad<H, H> gB;
  gA.zero();
  gB.zero();
  float gal = 0.f, gbe = 0.f;
  __syncthreads();
  for (int c0 = t.e0; c0 < t.e1; c0 += TE) {
    const int ne = min(TE, t.e1 - c0);
    chunk_basis<R, false>(g, rc, c0, ne, sC, nullptr, P0, nullptr);
    __syncthreads();
    {
      float z[C::HC];
      gemm_edge<R, H, C::HC>(P0, sA, e, h0, z);
#pragma unroll
      for (int j = 0; j < C::HC; ++j) {
        const float zz = z[j] + sAl[h0 + j];
        Z[(h0 + j) * LD + e] = zz;
        S[(h0 + j) * LD + e] = dev::silu(zz);
      }
    }
    __syncthreads();
    {
      float gg[C::HC];
      gemm_edge<H, H, C::HC>(S, sB, e, h0, gg);
      const float ce = sC[e];
#pragma unroll
      for (int j = 0; j < C::HC; ++j) G[(h0 + j) * LD + e] = ce * (gg[j] + sBe[h0 + j]);
    }
    __syncthreads();
    if (has_row) {
      const int eb = max(g.row_ptr[row], c0), ee = min(g.row_ptr[row + 1], c0 + ne);
      for (int x = eb; x < ee; ++x) {
        const int j = g.col[x], le = x - c0;
#pragma unroll
        for (int q = 0; q < H / 32; ++q)
          acc_y[q] = fmaf(G[(lane + 32 * q) * LD + le], bm[(size_t)j * H + lane + 32 * q], acc_y[q]);
      }
    }
    __syncthreads();
    {  // gbar = c bm_i v_j
      const bool valid = e < ne;
      const int x = c0 + e;
      const int i = valid ? g.src[x] : 0, j = valid ? g.col[x] : 0;
      const float ce = sC[e];
#pragma unroll
      for (int q4 = 0; q4 < C::HC / 4; ++q4) {
        const int h = h0 + 4 * q4;
        float4 b4 = make_float4(0.f, 0.f, 0.f, 0.f), v4 = b4;
        if (valid) {
          b4 = *reinterpret_cast<const float4*>(bm + (size_t)i * H + h);
          v4 = *reinterpret_cast<const float4*>(v + (size_t)j * H + h);
        }
        G[(h + 0) * LD + e] = ce * b4.x * v4.x;
        G[(h + 1) * LD + e] = ce * b4.y * v4.y;
        G[(h + 2) * LD + e] = ce * b4.z * v4.z;
        G[(h + 3) * LD + e] = ce * b4.w * v4.w;
      }
    }
    __syncthreads();
    gB.add(S, G, ne);
    if (threadIdx.x < H) {
      for (int x = 0; x < ne; ++x) gbe += G[threadIdx.x * LD + x];
    }
    {
      float sb[C::HC];
      gemm_edge<H, H, C::HC>(G, sBt, e, h0, sb);
      __syncthreads();  // everyone done reading S (gB) and Z is only touched below
#pragma unroll
      for (int j = 0; j < C::HC; ++j) {
        const int h = h0 + j;
        Z[h * LD + e] = sb[j] * dev::dsilu(Z[h * LD + e]);
      }
    }
    __syncthreads();
    gA.add(P0, Z, ne);
    if (threadIdx.x < H) {
      for (int x = 0; x < ne; ++x) gal += Z[threadIdx.x * LD + x];
    }
    __syncthreads();
  }
  if (has_row) {
#pragma unroll
    for (int q = 0; q < H / 32; ++q) Yb_out[(size_t)row * H + lane + 32 * q] = acc_y[q];
  }
  float* part = partial + (size_t)blockIdx.x * C::PE;
  gA.store(part);
  gB.store(part + R * H + H);
  if (threadIdx.x < H) {
    part[R * H + threadIdx.x] = gal;
    part[R * H + H + H * H + threadIdx.x] = gbe;
  }
}

// out[p] = sum_t partial[t][p]: each CTA owns 32 columns; its 8 warps sum
// contiguous eighths of the partial list in order (coalesced 128 B rows, loads
// in flight) and warp 0 adds the eight results in order => deterministic.
constexpr int kReduceCols = 32;
inline int reduce_grid(int PE) { return (PE + kReduceCols - 1) / kReduceCols; }
__global__ void __launch_bounds__(256) reduce_partials_kernel(const float* __restrict__ partial, int n_tiles, int PE,
                                                              float* __restrict__ out) {
  JANUS_GDC_WAIT();
  __shared__ float red[8][kReduceCols + 1];
  const int c = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int p = blockIdx.x * kReduceCols + c;
  const int per = (n_tiles + 7) / 8;
  const int t0 = grp * per, t1 = min(n_tiles, t0 + per);
  float s = 0.f;
  if (p < PE) {
#pragma unroll 8
    for (int t = t0; t < t1; ++t) s += __ldg(partial + (size_t)t * PE + p);
  }
  red[grp][c] = s;
  __syncthreads();
  if (grp == 0 && p < PE) {
    float r = 0.f;
#pragma unroll
    for (int g = 0; g < 8; ++g) r += red[g][c];
    out[p] = r;
  }
}

// Few partials (the persistent pair / tile kernels' grids, <= kSeqPartials):
// one thread per column sums the partials in order, 256 columns per CTA —
// 33 CTAs for PE = 8320 instead of reduce_partials_kernel's 260.
constexpr int kSeqPartials = 48;
__global__ void __launch_bounds__(256) reduce_partials_seq_kernel(const float* __restrict__ partial, int n, int PE,
                                                                  float* __restrict__ out) {
  JANUS_GDC_WAIT();
  const int p = blockIdx.x * 256 + threadIdx.x;
  if (p >= PE) return;
  const float* src = partial + p;
  float s = 0.f;
  int t = 0;
  for (; t + 4 <= n; t += 4) {
    const float a = __ldg(src + (size_t)t * PE), b = __ldg(src + (size_t)(t + 1) * PE);
    const float c = __ldg(src + (size_t)(t + 2) * PE), d = __ldg(src + (size_t)(t + 3) * PE);
    s = (((s + a) + b) + c) + d;
  }
  for (; t < n; ++t) s += __ldg(src + (size_t)t * PE);
  out[p] = s;
}
// out = sum over the n partials, fixed order for a given n
inline void reduce_partials(const float* partial, int n, int PE, float* out, cudaStream_t s) {
  if (n <= kSeqPartials)
    janus::pdl(reduce_partials_seq_kernel, (PE + 255) / 256, 256, 0, s)(partial, n, PE, out);
  else
    janus::pdl(reduce_partials_kernel, reduce_grid(PE), 256, 0, s)(partial, n, PE, out);
}

template <int H, int R>
constexpr size_t fe_smem() { return sizeof(float) * (R * H + H * H + 2 * H + R * LD + H * LD + TE); }
template <int H, int R>
constexpr size_t ff_smem() { return sizeof(float) * (R * H + H * H + 2 * H + 2 * R * LD + 2 * H * LD + 2 * TE); }
template <int H, int R>
constexpr size_t bf_smem() { return sizeof(float) * (R * H + 2 * H * H + 2 * H + 2 * R * LD + 6 * H * LD + 3 * TE); }
template <int H, int R>
constexpr size_t be_smem() { return sizeof(float) * (R * H + 2 * H * H + 2 * H + R * LD + 3 * H * LD + TE); }

}  // namespace edge
}  // namespace janus
