// pair_tc.cuh — FE and FF of the msg unit split at the edge filter (JANUS_PREC_TF32).
//
// The filter w_e = c_e (SiLU(phi(d_e) A + alpha) B + beta) and its radial
// derivative w'_e = dw/dd depend only on the edge length and the unit's
// parameters, and d_e = d_rev(e): they are the same for an edge and its
// reverse.  So the per-edge MMAs run once per undirected PAIR, for every msg
// unit of the stage in ONE launch at the start of FE (msg_filter_tc), and the
// two phases reduce over directed edges with no MMA at all:
//
//   FE  m_i = sum_{e in row i} w_p(e) * v_j                       (msg_fe_rows)
//   FF  Y_i = sum_e w_p(e) * am_j ;  F_i += sum_e q_p(e) u_e ;  a_h += Y W^T
//       q_e + q_rev(e) = < am_i v_j + am_j v_i , w'_e >          (msg_ff_rows)
//
// (reference: the four-phase math of SURVEY.md App. A / PAPER.md:171-178;
// the directed-edge kernels in edge_tc.cuh compute the same sums).  Pair
// tables: pcanon[p] = the canonical edge (e < rev e) of pair p, pidx[e] = p
// for both directions (pairs_kernel, built at LM with the geometry).
// Filters are stored fp32 [pair][64] per (slot, msg unit): the FE -> FF
// activation the SPEC's fe_bytes accounts for.
//
// Row kernels: one warp per atom row, lane = 2 features; edges are summed in
// CSR order (deterministic, independent of tiling and lanes).
#pragma once

#include "edge_tc.cuh"
#include "geo_job.hpp"

namespace janus {
namespace edge_tc {

constexpr int kMaxFilterUnits = 16;
struct FilterJobs {
  const float* pack[kMaxFilterUnits];  // per msg unit: the tensor-core weight image (pack_msg_weights)
  float* w[kMaxFilterUnits];           // [n_pairs][64]  w
  float* wp[kMaxFilterUnits];          // [n_pairs][64]  w' = dc (g + beta) + c g'
  int n;
};

// grid (chunks, units): CTA (x, y) runs unit y over 128-pair chunks x, x + gridDim.x, ...
__global__ void __launch_bounds__(NT, JANUS_FEFF_CTAS) msg_filter_tc(EdgeGeom g, const int* __restrict__ pcanon, int n_pairs,
                                                                    const __grid_constant__ FilterJobs J, float rc) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = align1024(sm_raw);
  uint8_t* W0 = sm;            // A^T
  uint8_t* W1 = W0 + kWTile;   // B^T
  uint8_t* T0 = W1 + kWTile;   // phi -> s
  uint8_t* T1 = T0 + kTile;    // phi' -> sdot
  float* al = reinterpret_cast<float*>(T1 + kTile);
  float* be = al + 64;
  const int u = blockIdx.y;
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t wbar;
  Ctx c;
  c.sm = sm;
  c.mbar = &mbar;
  load_weights(sm, J.pack[u], 2, al, be, nullptr, &wbar);
  setup(c, &tslot, 256);
  const uint32_t aW0 = tc::smem_u32(W0), aW1 = tc::smem_u32(W1), aT0 = tc::smem_u32(T0), aT1 = tc::smem_u32(T1);
  const int f0 = FPT * c.q;
  float* const wout = J.w[u];
  float* const wpout = J.wp[u];
  for (int ch = blockIdx.x; ch * TE < n_pairs; ch += gridDim.x) {
    const int p = ch * TE + c.e;
    const bool ok = p < n_pairs;
    const int x = ok ? __ldg(pcanon + p) : 0;
    const float d = ok ? __ldg(g.d + x) : 0.f, cc = ok ? __ldg(g.c + x) : 0.f, dc = ok ? __ldg(g.dc + x) : 0.f;
    {
      float ph[FPT], dph[FPT];
      basis(d, rc, f0, ph, dph);
      st_em(T0, c.e, f0, ph);
      st_em(T1, c.e, f0, dph);
    }
    tc::mbar_wait(&wbar, 0);
    c.publish();
    if (threadIdx.x == 0) {
      mma_tiles<128, 64, 64, 128>(c.tmem + TM_Z, aT0, aW0, false);
      mma_tiles<128, 64, 64, 128>(c.tmem + TM_ZP, aT1, aW0, false);
      tc::commit(c.mbar);
    }
    c.wait_mma();
    {
      float z[FPT], zp[FPT];
      c.ld2(TM_Z, TM_ZP, z, zp);
#pragma unroll
      for (int j = 0; j < FPT; ++j) {
        const float zz = z[j] + al[f0 + j], sg1 = fsig(zz);
        z[j] = zz * sg1;
        zp[j] = sg1 * (1.0f + zz * (1.0f - sg1)) * zp[j];
      }
      st_em(T0, c.e, f0, z);
      st_em(T1, c.e, f0, zp);
    }
    c.publish();
    if (threadIdx.x == 0) {
      mma_tiles<128, 64, 64, 128>(c.tmem + TM_G, aT0, aW1, false);
      mma_tiles<128, 64, 64, 128>(c.tmem + TM_GP, aT1, aW1, false);
      tc::commit(c.mbar);
    }
    c.wait_mma();
    {
      float gg[FPT], gp[FPT];
      c.ld2(TM_G, TM_GP, gg, gp);
      if (ok) {
        float4* wo = reinterpret_cast<float4*>(wout + (size_t)p * H + f0);
        float4* wpo = reinterpret_cast<float4*>(wpout + (size_t)p * H + f0);
#pragma unroll
        for (int q = 0; q < FPT / 4; ++q) {
          float w4[4], p4[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float gb = gg[4 * q + k] + be[f0 + 4 * q + k];
            w4[k] = cc * gb;
            p4[k] = dc * gb + cc * gp[4 * q + k];
          }
          wo[q] = make_float4(w4[0], w4[1], w4[2], w4[3]);
          wpo[q] = make_float4(p4[0], p4[1], p4[2], p4[3]);
        }
      }
    }
  }
  teardown(c, 256);
}

// Pair tables of one micro-batch per CTA (1024 threads): canonical edges in
// increasing edge order by a block-wide ballot scan, so pidx is deterministic.
__global__ void __launch_bounds__(1024) pairs_kernel(const __grid_constant__ node::GeoJobs J) {
  const node::GeoJob& jb = J.j[blockIdx.x];
  __shared__ int wsum[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int base = 0;
  for (int e0 = 0; e0 < jb.n_edges; e0 += 1024) {
    const int e = e0 + static_cast<int>(threadIdx.x);
    const int r = e < jb.n_edges ? jb.rev[e] : -1;
    const bool flag = e < jb.n_edges && e < r;
    const unsigned bal = __ballot_sync(0xffffffffu, flag);
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    int excl = 0, total = 0;
#pragma unroll 8
    for (int w = 0; w < 32; ++w) {
      const int s = wsum[w];
      excl += w < warp ? s : 0;
      total += s;
    }
    if (flag) {
      const int pos = base + excl + __popc(bal & ((1u << lane) - 1u));
      jb.pcanon[pos] = e;
      jb.pidx[e] = pos;
      jb.pidx[r] = pos;
    }
    base += total;
    __syncthreads();
  }
}

// m_i = sum_e w_p(e) * v_j   (warp per row, 2 features per lane)
__global__ void __launch_bounds__(256) msg_fe_rows(int n_atoms, const int* __restrict__ row_ptr, const int* __restrict__ col,
                                                   const int* __restrict__ pidx, const float* __restrict__ w,
                                                   const float* __restrict__ v, float* __restrict__ m_out) {
  const int i = blockIdx.x * 8 + static_cast<int>(threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (i >= n_atoms) return;
  const int eb = __ldg(row_ptr + i), ee = __ldg(row_ptr + i + 1);
  float2 acc = make_float2(0.f, 0.f);
  for (int e0 = eb; e0 < ee; e0 += 32) {
    const int n = min(32, ee - e0);
    const int mp = lane < n ? __ldg(pidx + e0 + lane) : 0;
    const int mj = lane < n ? __ldg(col + e0 + lane) : 0;
    for (int k0 = 0; k0 < n; k0 += 8) {  // 8 edges' loads in flight; masked tail
      float2 a[8], b[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int pk = __shfl_sync(0xffffffffu, mp, k0 + k), jk = __shfl_sync(0xffffffffu, mj, k0 + k);
        a[k] = __ldg(reinterpret_cast<const float2*>(w + (size_t)pk * H) + lane);
        b[k] = __ldg(reinterpret_cast<const float2*>(v + (size_t)jk * H) + lane);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (k0 + k < n) {
          acc.x = fmaf(a[k].x, b[k].x, acc.x);
          acc.y = fmaf(a[k].y, b[k].y, acc.y);
        }
    }
  }
  reinterpret_cast<float2*>(m_out + (size_t)i * H)[lane] = acc;
}

// FF of a msg unit (warp per row): Y_i, F_i += sum_e (q_e + q_rev e) u_e, a_h += Y W^T.
// The per-edge scalars of 32 edges are reduced across the warp by a
// transposing butterfly (31 shuffles): lane k ends with edge k's total.
__global__ void __launch_bounds__(256) msg_ff_rows(int n_atoms, const int* __restrict__ row_ptr, const int* __restrict__ col,
                                                   const int* __restrict__ pidx, const float* __restrict__ uvec,
                                                   const float* __restrict__ w, const float* __restrict__ wp,
                                                   const float* __restrict__ v, const float* __restrict__ am,
                                                   const float* __restrict__ wt, float* __restrict__ Y_out,
                                                   float* __restrict__ F, float* ah) {
  const int i = blockIdx.x * 8 + static_cast<int>(threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (i >= n_atoms) return;
  const int eb = __ldg(row_ptr + i), ee = __ldg(row_ptr + i + 1);
  const float2 ami = __ldg(reinterpret_cast<const float2*>(am + (size_t)i * H) + lane);
  const float2 vi = __ldg(reinterpret_cast<const float2*>(v + (size_t)i * H) + lane);
  float2 Y = make_float2(0.f, 0.f);
  float fx = 0.f, fy = 0.f, fz = 0.f;
  for (int e0 = eb; e0 < ee; e0 += 32) {
    const int n = min(32, ee - e0);
    const int mp = lane < n ? __ldg(pidx + e0 + lane) : 0;
    const int mj = lane < n ? __ldg(col + e0 + lane) : 0;
    float part[32];
#pragma unroll
    for (int k0 = 0; k0 < 32; k0 += 8) {
      if (k0 < n) {  // warp-uniform
        float2 a[8], b[8], c2[8], d2[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int pk = __shfl_sync(0xffffffffu, mp, k0 + k), jk = __shfl_sync(0xffffffffu, mj, k0 + k);
          a[k] = __ldg(reinterpret_cast<const float2*>(w + (size_t)pk * H) + lane);
          b[k] = __ldg(reinterpret_cast<const float2*>(wp + (size_t)pk * H) + lane);
          c2[k] = __ldg(reinterpret_cast<const float2*>(am + (size_t)jk * H) + lane);
          d2[k] = __ldg(reinterpret_cast<const float2*>(v + (size_t)jk * H) + lane);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const bool ok = k0 + k < n;
          if (ok) {
            Y.x = fmaf(a[k].x, c2[k].x, Y.x);
            Y.y = fmaf(a[k].y, c2[k].y, Y.y);
          }
          const float px = fmaf(ami.x, d2[k].x, c2[k].x * vi.x) * b[k].x;
          const float py = fmaf(ami.y, d2[k].y, c2[k].y * vi.y) * b[k].y;
          part[k0 + k] = ok ? px + py : 0.f;
        }
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) part[k0 + k] = 0.f;
      }
    }
    // transposing butterfly: after the step of width s, lane l keeps the
    // entries whose index has bit s equal to l's
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
      const bool hi = (lane & s) != 0;
#pragma unroll
      for (int k = 0; k < s; ++k) {
        const float send = hi ? part[k] : part[k + s];
        const float keep = hi ? part[k + s] : part[k];
        part[k] = keep + __shfl_xor_sync(0xffffffffu, send, s);
      }
    }
    if (lane < n) {  // part[0] = q of edge e0 + lane
      const float* ue = uvec + 3 * (size_t)(e0 + lane);
      fx = fmaf(part[0], __ldg(ue + 0), fx);
      fy = fmaf(part[0], __ldg(ue + 1), fy);
      fz = fmaf(part[0], __ldg(ue + 2), fz);
    }
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    fx += __shfl_xor_sync(0xffffffffu, fx, o);
    fy += __shfl_xor_sync(0xffffffffu, fy, o);
    fz += __shfl_xor_sync(0xffffffffu, fz, o);
  }
  reinterpret_cast<float2*>(Y_out + (size_t)i * H)[lane] = Y;
  if (lane == 0) {
    F[3 * (size_t)i + 0] += fx;
    F[3 * (size_t)i + 1] += fy;
    F[3 * (size_t)i + 2] += fz;
  }
  if (ah) {  // a_h[i][c] += sum_q Y[q] W^T[q][c], c = 2 lane, 2 lane + 1
    float2 o0 = make_float2(0.f, 0.f), o1 = make_float2(0.f, 0.f);
#pragma unroll 8
    for (int q2 = 0; q2 < 32; ++q2) {
      const float ya = __shfl_sync(0xffffffffu, Y.x, q2), yb = __shfl_sync(0xffffffffu, Y.y, q2);
      const float2 ta = __ldg(reinterpret_cast<const float2*>(wt + (size_t)(2 * q2) * H) + lane);
      const float2 tb = __ldg(reinterpret_cast<const float2*>(wt + (size_t)(2 * q2 + 1) * H) + lane);
      o0.x = fmaf(ya, ta.x, o0.x);
      o0.y = fmaf(ya, ta.y, o0.y);
      o1.x = fmaf(yb, tb.x, o1.x);
      o1.y = fmaf(yb, tb.y, o1.y);
    }
    float2* dst = reinterpret_cast<float2*>(ah + (size_t)i * H) + lane;
    float2 x = *dst;
    x.x += o0.x + o1.x;
    x.y += o0.y + o1.y;
    *dst = x;
  }
}

constexpr size_t filter_smem() { return 2 * kWTile + 2 * kTile + kSmallBytes; }

}  // namespace edge_tc
}  // namespace janus
