// pair_tc.cuh — the msg unit's four phases per undirected edge pair
// (JANUS_PREC_TF32, the bench path).
//
// The filter w_e = c_e (SiLU(phi(d_e) A + alpha) B + beta) and its radial
// derivative w'_e = dw/dd depend only on the edge length and the unit's
// parameters, and d_e = d_rev(e): they are the same for an edge and its
// reverse.  So the per-edge MMAs run once per undirected PAIR, for every msg
// unit of the stage in ONE launch at the start of FE (msg_filter_tc, tf32),
// and FE / FF reduce over directed edges with no MMA at all:
//
//   FE  m_i = sum_{e in row i} w_p(e) * v_j                       (msg_fe_rows)
//   FF  Y_i = sum_e w_p(e) * am_j ;  F_i += sum_e q_p(e) u_e ;  a_h += Y W^T
//       q_e + q_rev(e) = < am_i v_j + am_j v_i , w'_e >          (msg_ff_rows)
//
// BF / BE: the weight gradients are linear in the per-edge adjoints with
// pair-symmetric left factors, so msg_bf_pair_tc / msg_be_pair_tc (bf16
// operands) sum both directions' adjoints and run the dB / sbar / dA MMAs once
// per pair; the per-row sums read the stored filters (msg_bf_rows /
// msg_be_rows, which also host the per-CTA partials' reduction).
//
// (reference: the four-phase math of SURVEY.md App. A / PAPER.md:171-178;
// the directed-edge kernels in edge_tc.cuh compute the same sums.)  Pair
// tables: pcanon[p] = the canonical edge (e < rev e) of pair p, pidx[e] = p
// for both directions, pgeo = the pair records (d, c, c', i | u, j)
// (pairs_count_kernel + pairs_kernel, built at LM with the geometry).
// Filters are stored fp32 [pair][64] per (slot, msg unit): the FE -> FF / BF
// / BE activation the SPEC's fe_bytes accounts for.
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
__global__ void __launch_bounds__(NT, JANUS_FEFF_CTAS) msg_filter_tc(EdgeGeom g, const float4* __restrict__ pg, int n_pairs,
                                                                    const __grid_constant__ FilterJobs J, float rc) {
  JANUS_GDC_WAIT();
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
    const float4 g0 = ok ? __ldg(pg + 2 * p) : make_float4(0.f, 0.f, 0.f, 0.f);
    const float d = g0.x, cc = g0.y, dc = g0.z;
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
    {  // w, w' into the (now free) operand tiles, swizzled plain rows (st_pl: conflict-free)
      float gg[FPT], gp[FPT];
      c.ld2(TM_G, TM_GP, gg, gp);
#pragma unroll
      for (int k = 0; k < FPT; ++k) {
        const float gb = gg[k] + be[f0 + k];
        gg[k] = cc * gb;
        gp[k] = dc * gb + cc * gp[k];
      }
      st_pl(T0, c.e, f0, gg);
      st_pl(T1, c.e, f0, gp);
    }
    __syncthreads();
    {  // coalesced copy-out: the chunk's pairs are contiguous rows of w / w' ([pair][64])
      const int np = min(TE, n_pairs - ch * TE);
      float4* wo = reinterpret_cast<float4*>(wout + (size_t)ch * TE * H);
      float4* wpo = reinterpret_cast<float4*>(wpout + (size_t)ch * TE * H);
      for (int x = threadIdx.x; x < np * 16; x += NT) {
        const uint32_t o = off_pl(x >> 4, 4 * (x & 15));
        wo[x] = *reinterpret_cast<const float4*>(T0 + o);
        wpo[x] = *reinterpret_cast<const float4*>(T1 + o);
      }
    }
    __syncthreads();  // T0 / T1 are the next chunk's operand tiles
  }
  teardown(c, 256);
}

// Pair tables, two launches over (1024-edge chunk, micro-batch) CTAs:
// pairs_count_kernel counts each chunk's canonical edges (e < rev e), then
// pairs_kernel offsets its chunk by the counts of the chunks before it and
// ranks the canonical edges with a block-wide ballot scan — canonical edges in
// increasing edge order, so pidx is deterministic (and independent of the
// chunking).  counts: [kMaxGeoJobs][chunks_cap].
__device__ __forceinline__ bool is_canonical(const node::GeoJob& jb, int e, int& r) {
  r = e < jb.n_edges ? jb.rev[e] : -1;
  return e < jb.n_edges && e < r && r < jb.n_edges;
}
__global__ void __launch_bounds__(1024) pairs_count_kernel(const __grid_constant__ node::GeoJobs J, int* __restrict__ counts,
                                                           int chunks_cap) {
  JANUS_GDC_WAIT();
  const node::GeoJob& jb = J.j[blockIdx.y];
  const int e0 = blockIdx.x * 1024;
  if (e0 >= jb.n_edges) return;
  __shared__ int wsum[32];
  int r;
  const bool flag = is_canonical(jb, e0 + static_cast<int>(threadIdx.x), r);
  const unsigned bal = __ballot_sync(0xffffffffu, flag);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = __popc(bal);
  __syncthreads();
  if (threadIdx.x < 32) {
    int v = wsum[threadIdx.x];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) counts[blockIdx.y * chunks_cap + blockIdx.x] = v;
  }
}
__global__ void __launch_bounds__(1024) pairs_kernel(const __grid_constant__ node::GeoJobs J, const int* __restrict__ counts,
                                                     int chunks_cap) {
  JANUS_GDC_WAIT();
  const node::GeoJob& jb = J.j[blockIdx.y];
  const int e0 = blockIdx.x * 1024;
  if (e0 >= jb.n_edges) return;
  __shared__ int wsum[32];
  __shared__ int base_s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < 32) {  // this chunk's offset: the counts of the chunks before it
    int v = 0;
    for (int c = lane; c < static_cast<int>(blockIdx.x); c += 32) v += counts[blockIdx.y * chunks_cap + c];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) base_s = v;
  }
  const int e = e0 + static_cast<int>(threadIdx.x);
  int r;
  const bool flag = is_canonical(jb, e, r);
  const unsigned bal = __ballot_sync(0xffffffffu, flag);
  if (lane == 0) wsum[warp] = __popc(bal);
  __syncthreads();
  int excl = base_s;
#pragma unroll 8
  for (int w = 0; w < 32; ++w) excl += w < warp ? wsum[w] : 0;
  const int pos = excl + __popc(bal & ((1u << lane) - 1u));
  if (flag && pos < (jb.n_edges >> 1)) {  // (a rev that is not an involution — host-checked at load — never writes past the tables)
    jb.pcanon[pos] = e;
    jb.pidx[e] = pos;
    jb.pidx[r] = pos;
    jb.pgeo[2 * pos] = make_float4(jb.d[e], jb.c[e], jb.dc[e], __int_as_float(jb.src[e]));
    jb.pgeo[2 * pos + 1] = make_float4(jb.u[3 * e], jb.u[3 * e + 1], jb.u[3 * e + 2], __int_as_float(jb.col[e]));
  }
}

// (Y W^T) of one row held by a warp as float2 per lane (features 2 lane, 2 lane + 1);
// wt = W^T row-major [64][64] (the pack's plain copy, read through L1)
__device__ __forceinline__ float2 row_times_wt(float2 Y, const float* __restrict__ wt, int lane) {
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
  return make_float2(o0.x + o1.x, o0.y + o1.y);
}

// m_i = sum_e w_p(e) * v_j   (warp per row, 2 features per lane)
template <int KF>  // edges whose gathers are in flight per step
__global__ void __launch_bounds__(256) msg_fe_rows(int n_atoms, const int* __restrict__ row_ptr, const int* __restrict__ col,
                                                   const int* __restrict__ pidx, const float* __restrict__ w,
                                                   const float* __restrict__ v, float* __restrict__ m_out) {
  JANUS_GDC_WAIT();
  const int i = blockIdx.x * 8 + static_cast<int>(threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (i >= n_atoms) return;
  const int eb = __ldg(row_ptr + i), ee = __ldg(row_ptr + i + 1);
  float2 acc = make_float2(0.f, 0.f);
  for (int e0 = eb; e0 < ee; e0 += 32) {
    const int n = min(32, ee - e0);
    const int mp = lane < n ? __ldg(pidx + e0 + lane) : 0;
    const int mj = lane < n ? __ldg(col + e0 + lane) : 0;
    for (int k0 = 0; k0 < n; k0 += KF) {  // KF edges' loads in flight; masked tail
      float2 a[KF], b[KF];
#pragma unroll
      for (int k = 0; k < KF; ++k) {
        const int pk = __shfl_sync(0xffffffffu, mp, k0 + k), jk = __shfl_sync(0xffffffffu, mj, k0 + k);
        a[k] = __ldg(reinterpret_cast<const float2*>(w + (size_t)pk * H) + lane);
        b[k] = __ldg(reinterpret_cast<const float2*>(v + (size_t)jk * H) + lane);
      }
#pragma unroll
      for (int k = 0; k < KF; ++k)
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
template <int KF>  // edges whose gathers are in flight per step
__global__ void __launch_bounds__(256) msg_ff_rows(int n_atoms, const int* __restrict__ row_ptr, const int* __restrict__ col,
                                                   const int* __restrict__ pidx, const float* __restrict__ uvec,
                                                   const float* __restrict__ w, const float* __restrict__ wp,
                                                   const float* __restrict__ v, const float* __restrict__ am,
                                                   const float* __restrict__ wt, float* __restrict__ Y_out,
                                                   float* __restrict__ F, float* ah) {
  JANUS_GDC_WAIT();
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
    for (int k0 = 0; k0 < 32; k0 += KF) {
      if (k0 < n) {  // warp-uniform
        float2 a[KF], b[KF], c2[KF], d2[KF];
#pragma unroll
        for (int k = 0; k < KF; ++k) {
          const int pk = __shfl_sync(0xffffffffu, mp, k0 + k), jk = __shfl_sync(0xffffffffu, mj, k0 + k);
          a[k] = __ldg(reinterpret_cast<const float2*>(w + (size_t)pk * H) + lane);
          b[k] = __ldg(reinterpret_cast<const float2*>(wp + (size_t)pk * H) + lane);
          c2[k] = __ldg(reinterpret_cast<const float2*>(am + (size_t)jk * H) + lane);
          d2[k] = __ldg(reinterpret_cast<const float2*>(v + (size_t)jk * H) + lane);
        }
#pragma unroll
        for (int k = 0; k < KF; ++k) {
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
        for (int k = 0; k < KF; ++k) part[k0 + k] = 0.f;
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
  if (ah) {  // a_h[i] += Y W^T
    const float2 o = row_times_wt(Y, wt, lane);
    float2* dst = reinterpret_cast<float2*>(ah + (size_t)i * H) + lane;
    float2 x = *dst;
    x.x += o.x;
    x.y += o.y;
    *dst = x;
  }
}

// ------------------------------------------------------------ BF / BE per pair
// Per-pair adjoints in the WARP-PER-PAIR layout: warp w builds rows 8w..8w+7
// of the chunk's bf16 adjoint tiles, lane l holding features 2l, 2l+1, so one
// 8-byte load per lane fetches a whole 256 B node row (2 L1 lines per load
// instruction).  The thread-per-edge layout the TMEM epilogues need had each
// load instruction touch 32 different rows (32 L1 wavefronts; ~12k per chunk
// for BF's six gathers, the kernels' top stall).  The arithmetic is the same
// fp32 expression per element, so the tiles are bit-identical.
struct PairRec {  // lanes 0..7: the scalars of pair 8w + lane
  int i = 0, j = 0;
  float c = 0.f, dc = 0.f, qb = 0.f;
};
__device__ __forceinline__ PairRec pair_rec(const float4* __restrict__ pg, int n_pairs, int p, const float* __restrict__ Fbar) {
  PairRec r;
  if (p < n_pairs) {
    const float4 g0 = __ldg(pg + 2 * p), g1 = __ldg(pg + 2 * p + 1);
    r.c = g0.y;
    r.dc = g0.z;
    r.i = __float_as_int(g0.w);
    r.j = __float_as_int(g1.w);
    if (Fbar)  // <Fbar_i - Fbar_j, u> (qb_rev = qb: u_rev = -u)
      r.qb = fmaf(__ldg(Fbar + 3 * r.i) - __ldg(Fbar + 3 * r.j), g1.x,
                  fmaf(__ldg(Fbar + 3 * r.i + 1) - __ldg(Fbar + 3 * r.j + 1), g1.y,
                       (__ldg(Fbar + 3 * r.i + 2) - __ldg(Fbar + 3 * r.j + 2)) * g1.z));
  }
  return r;
}
__device__ __forceinline__ float2 ldrow2(const float* __restrict__ x, int row, int lane) {
  return __ldg(reinterpret_cast<const float2*>(x + (size_t)row * H) + lane);
}
__device__ __forceinline__ void st_b16x2(uint8_t* t, int e, int f, float a, float b) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  *reinterpret_cast<uint32_t*>(t + off_b16(e, f)) = *reinterpret_cast<const uint32_t*>(&v);
}
// BF: mu -> tmu, nu -> tnu for the chunk's 128 pairs (all 16 warps)
// the record of the pair this lane (0..7) holds in chunk p0 (zeros past the end)
__device__ __forceinline__ PairRec chunk_rec(const float4* __restrict__ pg, int n_pairs, int p0, const float* __restrict__ Fbar) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  return pair_rec(pg, n_pairs, lane < 8 ? p0 + 8 * warp + lane : n_pairs, Fbar);
}
__device__ __forceinline__ void bf_adjoints_rows(const PairRec& r, const float* __restrict__ v,
                                                 const float* __restrict__ vdot, const float* __restrict__ am, uint8_t* tmu,
                                                 uint8_t* tnu) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int b = 0; b < 2; ++b) {
    float2 ai[4], aj[4], vi[4], vj[4], di[4], dj[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = __shfl_sync(0xffffffffu, r.i, 4 * b + k), j = __shfl_sync(0xffffffffu, r.j, 4 * b + k);
      ai[k] = ldrow2(am, i, lane);
      aj[k] = ldrow2(am, j, lane);
      vi[k] = ldrow2(v, i, lane);
      vj[k] = ldrow2(v, j, lane);
      di[k] = ldrow2(vdot, i, lane);
      dj[k] = ldrow2(vdot, j, lane);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float cc = __shfl_sync(0xffffffffu, r.c, 4 * b + k), dc = __shfl_sync(0xffffffffu, r.dc, 4 * b + k);
      const float qb = __shfl_sync(0xffffffffu, r.qb, 4 * b + k);
      const float rx = fmaf(ai[k].x, vj[k].x, aj[k].x * vi[k].x), ry = fmaf(ai[k].y, vj[k].y, aj[k].y * vi[k].y);
      const float kx = fmaf(ai[k].x, dj[k].x, aj[k].x * di[k].x), ky = fmaf(ai[k].y, dj[k].y, aj[k].y * di[k].y);
      const int e = 8 * warp + 4 * b + k;
      st_b16x2(tmu, e, 2 * lane, qb * dc * rx + cc * kx, qb * dc * ry + cc * ky);
      st_b16x2(tnu, e, 2 * lane, qb * cc * rx, qb * cc * ry);
    }
  }
}
// BE: gbar = c (bm_i v_j + bm_j v_i) -> tg
__device__ __forceinline__ void be_adjoint_rows(const PairRec& r, const float* __restrict__ v,
                                                const float* __restrict__ bm, uint8_t* tg) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float2 bi[8], bj[8], vi[8], vj[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int i = __shfl_sync(0xffffffffu, r.i, k), j = __shfl_sync(0xffffffffu, r.j, k);
    bi[k] = ldrow2(bm, i, lane);
    bj[k] = ldrow2(bm, j, lane);
    vi[k] = ldrow2(v, i, lane);
    vj[k] = ldrow2(v, j, lane);
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float cc = __shfl_sync(0xffffffffu, r.c, k);
    st_b16x2(tg, 8 * warp + k, 2 * lane, cc * fmaf(bi[k].x, vj[k].x, bj[k].x * vi[k].x),
             cc * fmaf(bi[k].y, vj[k].y, bj[k].y * vi[k].y));
  }
}

// The weight gradients are linear in the per-edge adjoints (mu, nu of BF;
// gbar of BE) with pair-symmetric left factors (phi, phi', s, sdot, z, z'), so
// they are accumulated once per pair on the SUMS of both directions:
//   BF  rho = am_i v_j + am_j v_i,  kappa = am_i vdot_j + am_j vdot_i,
//       mu = qb c' rho + c kappa,  nu = qb c rho   (qb_rev = qb: u_rev = -u)
//   BE  gbar = c (bm_i v_j + bm_j v_i)
// then dB = s^T mu + sdot^T nu, sbar = mu B^T, ..., exactly as the directed
// kernels (edge_tc.cuh msg_bf_tc / msg_be_tc) but with no w / w' MMAs: the
// per-row sums use the stored filters (msg_bf_rows / msg_be_rows).
// Persistent CTAs, static chunk assignment => deterministic partials.
// Register caps of the BF / BE pair kernels.  At the launch bound's 128
// registers x 512 threads a pair CTA holds the SM's whole register file, so
// nothing else (row / upd kernels of the other lanes) can share its SM while
// it waits on gathers and MMAs.  Measured (tools/ab_libs.sh, two runs each):
// 128/128 17534-17545, BF 96 / BE 64 17428-17455, 96/96 17681-17702,
// 96/80 17756-17759 structures/s (no spills; BF would spill below 96).  With
// the next chunk's records prefetched (below) BF needs 104 (ab4: 19034 vs
// 18977-19019 without the prefetch, within noise).
// With 256 TMEM columns (below) BF holds z, z' in registers across the
// second MMA group: 104 spills, 112 spills 48 B; 120 is spill-free (tools/
// ab_libs.sh, device structures/s, two runs: 512 columns at 104 registers
// 19052 / 19010; 256 columns at 112: 19114 / 19110, 120: 19097 / 19093,
// 128: 19147 / 19192 — all within ~0.5%).
#ifndef JANUS_BF_MAXNREG
#define JANUS_BF_MAXNREG 120
#endif
#ifndef JANUS_BE_MAXNREG
#define JANUS_BE_MAXNREG 80
#endif
// TMEM: 256 columns per pair CTA (JANUS_PAIR_TMEM256, the default) instead of
// 512, so a pair CTA leaves half of its SM's tensor memory to the other lanes'
// tcgen05 kernels (filter / upd / the other pair kernel), which otherwise
// spin in tcgen05.alloc beside it.  BE: z | sbar | dA | dB.  BF keeps z, z'
// in registers from epilogue 1 to epilogue 2, so sbar, sdotbar reuse z, z''s
// columns: z | z' (then sbar | sdotbar) | dA | dB.
#ifndef JANUS_PAIR_TMEM256
#define JANUS_PAIR_TMEM256 1
#endif
#if JANUS_PAIR_TMEM256
constexpr uint32_t kPairCols = 256, PT_Z = 0, PT_ZP = 64, PT_G = 0, PT_GP = 64, PT_AG = 128, PT_BG = 192;
constexpr uint32_t BT_Z = 0, BT_G = 64, BT_AG = 128, BT_BG = 192;
#else
constexpr uint32_t kPairCols = 512, PT_Z = TM_Z, PT_ZP = TM_ZP, PT_G = TM_G, PT_GP = TM_GP, PT_AG = TM_AG, PT_BG = TM_BG;
constexpr uint32_t BT_Z = TM_Z, BT_G = TM_G, BT_AG = TM_AG, BT_BG = TM_BG;
#endif
__global__ void __maxnreg__(JANUS_BF_MAXNREG) msg_bf_pair_tc(EdgeGeom g, const float4* __restrict__ pg, int n_pairs, MsgParams p,
                                                       float rc, const float* __restrict__ v, const float* __restrict__ vdot,
                                                       const float* __restrict__ am, const float* __restrict__ Fbar,
                                                       float* __restrict__ partial) {
  JANUS_GDC_WAIT();
  TC_DECL;
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = align1024(sm_raw);
  uint8_t* W2b = sm;  // bf16 weights in pack order: B | A^T | B^T
  uint8_t* W0b = W2b + kW2bBytes;  // W1b (A^T) follows W0b
  uint8_t* B0 = sm + 2 * kWTile;  // bf16: s          (write_partial scratch: B0..B2)
  uint8_t* B1 = B0 + kBTile;      //       sdot
  uint8_t* B2 = B1 + kBTile;      //       mu, then zbar
  uint8_t* B3 = B2 + kBTile;      //       nu, then zbar'
  uint8_t* B4 = B3 + kBTile;      //       phi
  uint8_t* B5 = B4 + kBTile;      //       phi'
  float* al = reinterpret_cast<float*>(B5 + kBTile);
  float* be = al + 64;
  float* csa = be + 64;
  float* csb = csa + 64;
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t wbar;
  Ctx c;
  c.sm = sm;
  c.mbar = &mbar;
  load_weights_b16(W2b, p.pack, al, be, &wbar);
  if (threadIdx.x < 128) csa[threadIdx.x] = 0.f;
  setup(c, &tslot, kPairCols);
  TC_M();
  const uint32_t aW0b = tc::smem_u32(W0b), aW2b = tc::smem_u32(W2b);
  const uint32_t aB0 = tc::smem_u32(B0), aB1 = tc::smem_u32(B1), aB2 = tc::smem_u32(B2), aB3 = tc::smem_u32(B3);
  const uint32_t aB4 = tc::smem_u32(B4), aB5 = tc::smem_u32(B5);
  bool first = true;
  const int f0 = FPT * c.q;
  // the next chunk's pair records (with qbar) and edge lengths are loaded while
  // the current chunk runs its MMAs and epilogues: two dependent L2 round
  // trips fewer at the head of every chunk (phase trace: ~2k + 3.3k cycles)
  auto edge_d = [&](int ch) { return ch * TE + c.e < n_pairs ? __ldg(&pg[2 * (ch * TE + c.e)].x) : 0.f; };
  PairRec rec = chunk_rec(pg, n_pairs, blockIdx.x * TE, Fbar);
  float d = edge_d(blockIdx.x);
  for (int ch = blockIdx.x; ch * TE < n_pairs; ch += gridDim.x) {
    {
      float ph[FPT], dph[FPT];
      basis_fast(d, rc, f0, ph, dph);
      st_b16(B4, c.e, f0, ph);
      st_b16(B5, c.e, f0, dph);
    }
    TC_M();
    bf_adjoints_rows(rec, v, vdot, am, B2, B3);  // mu (B of dB, A of sbar), nu
    rec = chunk_rec(pg, n_pairs, (ch + gridDim.x) * TE, Fbar);
    d = edge_d(ch + gridDim.x);
    TC_M();
    tc::mbar_wait(&wbar, 0);
    c.publish();
    TC_M();
    if (threadIdx.x == 0) {
      mma_kb16(c.tmem + PT_Z, aB4, aW0b);
      mma_kb16(c.tmem + PT_ZP, aB5, aW0b);
      tc::commit(c.mbar);
    }
    c.wait_mma();
    TC_M();
    float z[FPT], zp[FPT];  // raw z, z' (bias included), kept for epilogue 2
    {
      float sv[FPT], sd[FPT];
      c.ld2(PT_Z, PT_ZP, z, zp);
#pragma unroll
      for (int k = 0; k < FPT; ++k) {
        const float zz = z[k] + al[f0 + k], s1 = fsig_t(zz);
        z[k] = zz;
        sv[k] = zz * s1;
        sd[k] = s1 * (1.0f + zz * (1.0f - s1)) * zp[k];
      }
      st_b16(B0, c.e, f0, sv);  // s
      st_b16(B1, c.e, f0, sd);  // sdot
    }
    c.publish();
    if (threadIdx.x == 0) {  // dB += s^T mu + sdot^T nu; sbar = mu B^T, sdotbar = nu B^T
      mma_wg_b16(c.tmem + PT_BG, aB0, aB2, !first);
      mma_wg_b16(c.tmem + PT_BG, aB1, aB3, true);
      mma_kb16(c.tmem + PT_G, aB2, aW2b);
      mma_kb16(c.tmem + PT_GP, aB3, aW2b);
      tc::commit(c.mbar);
    }
    b16_colsum_add(B2, csb);  // dbeta += sum mu
    TC_M();
    c.wait_mma();
    TC_M();
    __syncthreads();  // column sums done: B2, B3 may be rewritten
    {
      float sb[FPT], sdb[FPT];
      c.ld2(PT_G, PT_GP, sb, sdb);
#pragma unroll
      for (int k = 0; k < FPT; ++k) {
        const float zz = z[k], s1 = fsig_t(zz);
        const float ds = s1 * (1.0f + zz * (1.0f - s1));
        const float d2s = s1 * (1.0f - s1) * (2.0f + zz * (1.0f - 2.0f * s1));
        z[k] = sb[k] * ds + sdb[k] * d2s * zp[k];  // zbar
        zp[k] = sdb[k] * ds;                       // zbar'
      }
      st_b16(B2, c.e, f0, z);
      st_b16(B3, c.e, f0, zp);
    }
    c.publish();
    if (threadIdx.x == 0) {  // dA += phi^T zbar + phi'^T zbar'
      mma_wg_b16(c.tmem + PT_AG, aB4, aB2, !first);
      mma_wg_b16(c.tmem + PT_AG, aB5, aB3, true);
      tc::commit(c.mbar);
    }
    b16_colsum_add(B2, csa);  // dalpha += sum zbar
    TC_M();
    c.wait_mma();
    TC_M();
    first = false;
    __syncthreads();
  }
  float* part = partial + (size_t)blockIdx.x * PE;
  if (first) {
    for (int x = threadIdx.x; x < PE; x += NT) part[x] = 0.f;
    teardown(c, kPairCols);
    return;
  }
  TC_M();
  write_partial(c, part, B0, csa, csb, PT_AG, PT_BG TC_PASS);
  TC_M();
  TC_DUMP("bf_pair");
  teardown(c, kPairCols);
}

__global__ void __maxnreg__(JANUS_BE_MAXNREG) msg_be_pair_tc(EdgeGeom g, const float4* __restrict__ pg, int n_pairs, MsgParams p,
                                                       float rc, const float* __restrict__ v, const float* __restrict__ bm,
                                                       float* __restrict__ partial) {
  JANUS_GDC_WAIT();
  TC_DECL;
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = align1024(sm_raw);
  uint8_t* W2b = sm;
  uint8_t* W0b = W2b + kW2bBytes;
  uint8_t* B0 = sm + 2 * kWTile;  // bf16: phi     (write_partial scratch: B0..B2)
  uint8_t* B1 = B0 + kBTile;      //       s
  uint8_t* B2 = B1 + kBTile;      //       gbar
  uint8_t* B3 = B2 + kBTile;      //       zbar
  float* al = reinterpret_cast<float*>(B3 + kBTile);
  float* be = al + 64;
  float* csa = be + 64;
  float* csb = csa + 64;
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t wbar;
  Ctx c;
  c.sm = sm;
  c.mbar = &mbar;
  load_weights_b16(W2b, p.pack, al, be, &wbar);
  if (threadIdx.x < 128) csa[threadIdx.x] = 0.f;
  setup(c, &tslot, kPairCols);
  const uint32_t aW0b = tc::smem_u32(W0b), aW2b = tc::smem_u32(W2b);
  const uint32_t aB0 = tc::smem_u32(B0), aB1 = tc::smem_u32(B1), aB2 = tc::smem_u32(B2), aB3 = tc::smem_u32(B3);
  bool first = true;
  const int f0 = FPT * c.q;
  auto edge_d = [&](int ch) { return ch * TE + c.e < n_pairs ? __ldg(&pg[2 * (ch * TE + c.e)].x) : 0.f; };
  PairRec rec = chunk_rec(pg, n_pairs, blockIdx.x * TE, nullptr);  // next chunk's: prefetched below
  float d = edge_d(blockIdx.x);
  for (int ch = blockIdx.x; ch * TE < n_pairs; ch += gridDim.x) {
    {
      float ph[FPT], dph[FPT];
      basis_fast(d, rc, f0, ph, dph);
      st_b16(B0, c.e, f0, ph);
    }
    be_adjoint_rows(rec, v, bm, B2);  // gbar (zero on padding: c = 0)
    rec = chunk_rec(pg, n_pairs, (ch + gridDim.x) * TE, nullptr);
    d = edge_d(ch + gridDim.x);
    tc::mbar_wait(&wbar, 0);
    c.publish();
    if (threadIdx.x == 0) {
      mma_kb16(c.tmem + BT_Z, aB0, aW0b);
      tc::commit(c.mbar);
    }
    c.wait_mma();
    {
      float z[FPT];
      c.ld(BT_Z, z);
#pragma unroll
      for (int k = 0; k < FPT; ++k) {
        const float zz = z[k] + al[f0 + k];
        z[k] = zz * fsig_t(zz);
      }
      st_b16(B1, c.e, f0, z);  // s
    }
    c.publish();
    if (threadIdx.x == 0) {
      mma_wg_b16(c.tmem + BT_BG, aB1, aB2, !first);  // dB += s^T gbar
      mma_kb16(c.tmem + BT_G, aB2, aW2b);            // sbar = gbar B^T
      tc::commit(c.mbar);
    }
    b16_colsum_add(B2, csb);  // dbeta += sum gbar
    c.wait_mma();
    {
      float z[FPT], sb[FPT];
      c.ld2(BT_Z, BT_G, z, sb);
#pragma unroll
      for (int k = 0; k < FPT; ++k) {
        const float zz = z[k] + al[f0 + k], s1 = fsig_t(zz);
        z[k] = sb[k] * (s1 * (1.0f + zz * (1.0f - s1)));
      }
      st_b16(B3, c.e, f0, z);  // zbar
    }
    c.publish();
    if (threadIdx.x == 0) {
      mma_wg_b16(c.tmem + BT_AG, aB0, aB3, !first);  // dA += phi^T zbar
      tc::commit(c.mbar);
    }
    b16_colsum_add(B3, csa);  // dalpha += sum zbar
    c.wait_mma();
    first = false;
    __syncthreads();
  }
  float* part = partial + (size_t)blockIdx.x * PE;
  if (first) {
    for (int x = threadIdx.x; x < PE; x += NT) part[x] = 0.f;
    teardown(c, kPairCols);
    return;
  }
  write_partial(c, part, B0, csa, csb, BT_AG, BT_BG TC_PASS);
  teardown(c, kPairCols);
}

// The BF / BE pair kernels' per-CTA partials, summed into the phase's ledger
// slice by extra CTAs of the row kernel that follows (one thread per column,
// partials in CTA order: the arithmetic of edge::reduce_partials_seq_kernel,
// one launch fewer per pair kernel and no serial tail).
struct PartialReduce {
  const float* partial = nullptr;
  int n = 0;
  float* G = nullptr;
};
__host__ __device__ constexpr int reduce_blocks(const PartialReduce& r) { return r.G ? (PE + 255) / 256 : 0; }
__device__ __forceinline__ void reduce_block(const PartialReduce& r, int blk) {
  const int p = blk * 256 + static_cast<int>(threadIdx.x);
  if (p >= PE) return;
  const float* src = r.partial + p;
  float s = 0.f;
  int t = 0;
  for (; t + 4 <= r.n; t += 4) {
    const float a = __ldg(src + (size_t)t * PE), b = __ldg(src + (size_t)(t + 1) * PE);
    const float c = __ldg(src + (size_t)(t + 2) * PE), d = __ldg(src + (size_t)(t + 3) * PE);
    s = (((s + a) + b) + c) + d;
  }
  for (; t < r.n; ++t) s += __ldg(src + (size_t)t * PE);
  r.G[p] = s;
}

// BF rows: mdot_i = sum_e qb_e w'_p v_j + w_p vdot_j ; X_i = sum_e qb_e w'_p am_j ;
// inj = X W^T (hbar^F of the unit input), qb_e = <Fbar_i - Fbar_j, u_e>
template <int KF>  // edges whose gathers are in flight per step
__global__ void __launch_bounds__(256) msg_bf_rows(int n_atoms, const int* __restrict__ row_ptr, const int* __restrict__ col,
                                                   const int* __restrict__ pidx, const float* __restrict__ uvec,
                                                   const float* __restrict__ Fbar, const float* __restrict__ w,
                                                   const float* __restrict__ wp, const float* __restrict__ v,
                                                   const float* __restrict__ vdot, const float* __restrict__ am,
                                                   const float* __restrict__ wt, float* __restrict__ mdot_out,
                                                   float* __restrict__ X_out, float* __restrict__ inj,
                                                   const __grid_constant__ PartialReduce red) {
  JANUS_GDC_WAIT();
  const int row_blocks = (n_atoms + 7) / 8;
  if (static_cast<int>(blockIdx.x) >= row_blocks) {
    reduce_block(red, static_cast<int>(blockIdx.x) - row_blocks);
    return;
  }
  const int i = blockIdx.x * 8 + static_cast<int>(threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (i >= n_atoms) return;
  const int eb = __ldg(row_ptr + i), ee = __ldg(row_ptr + i + 1);
  const float fi0 = __ldg(Fbar + 3 * i), fi1 = __ldg(Fbar + 3 * i + 1), fi2 = __ldg(Fbar + 3 * i + 2);
  float2 md = make_float2(0.f, 0.f), X = make_float2(0.f, 0.f);
  for (int e0 = eb; e0 < ee; e0 += 32) {
    const int n = min(32, ee - e0);
    int mp = 0, mj = 0;
    float mq = 0.f;
    if (lane < n) {
      const int e = e0 + lane;
      mp = __ldg(pidx + e);
      mj = __ldg(col + e);
      mq = fmaf(fi0 - __ldg(Fbar + 3 * mj), __ldg(uvec + 3 * e), 0.f);
      mq = fmaf(fi1 - __ldg(Fbar + 3 * mj + 1), __ldg(uvec + 3 * e + 1), mq);
      mq = fmaf(fi2 - __ldg(Fbar + 3 * mj + 2), __ldg(uvec + 3 * e + 2), mq);
    }
    for (int k0 = 0; k0 < n; k0 += KF) {
      float2 a[KF], b[KF], vv[KF], dv[KF], aj[KF];
      float q[KF];
#pragma unroll
      for (int k = 0; k < KF; ++k) {
        const int pk = __shfl_sync(0xffffffffu, mp, k0 + k), jk = __shfl_sync(0xffffffffu, mj, k0 + k);
        q[k] = __shfl_sync(0xffffffffu, mq, k0 + k);
        a[k] = __ldg(reinterpret_cast<const float2*>(w + (size_t)pk * H) + lane);
        b[k] = __ldg(reinterpret_cast<const float2*>(wp + (size_t)pk * H) + lane);
        vv[k] = __ldg(reinterpret_cast<const float2*>(v + (size_t)jk * H) + lane);
        dv[k] = __ldg(reinterpret_cast<const float2*>(vdot + (size_t)jk * H) + lane);
        aj[k] = __ldg(reinterpret_cast<const float2*>(am + (size_t)jk * H) + lane);
      }
#pragma unroll
      for (int k = 0; k < KF; ++k)
        if (k0 + k < n) {
          const float px = q[k] * b[k].x, py = q[k] * b[k].y;
          md.x = fmaf(px, vv[k].x, fmaf(a[k].x, dv[k].x, md.x));
          md.y = fmaf(py, vv[k].y, fmaf(a[k].y, dv[k].y, md.y));
          X.x = fmaf(px, aj[k].x, X.x);
          X.y = fmaf(py, aj[k].y, X.y);
        }
    }
  }
  reinterpret_cast<float2*>(mdot_out + (size_t)i * H)[lane] = md;
  reinterpret_cast<float2*>(X_out + (size_t)i * H)[lane] = X;
  if (inj) reinterpret_cast<float2*>(inj + (size_t)i * H)[lane] = row_times_wt(X, wt, lane);
}

// BE rows: Yb_i = sum_e w_p bm_j ; b_h += Yb W^T + inj
template <int KF>  // edges whose gathers are in flight per step
__global__ void __launch_bounds__(256) msg_be_rows(int n_atoms, const int* __restrict__ row_ptr, const int* __restrict__ col,
                                                   const int* __restrict__ pidx, const float* __restrict__ w,
                                                   const float* __restrict__ bm, const float* __restrict__ wt,
                                                   float* __restrict__ Yb_out, const float* __restrict__ inj, float* bh,
                                                   const __grid_constant__ PartialReduce red) {
  JANUS_GDC_WAIT();
  const int row_blocks = (n_atoms + 7) / 8;
  if (static_cast<int>(blockIdx.x) >= row_blocks) {
    reduce_block(red, static_cast<int>(blockIdx.x) - row_blocks);
    return;
  }
  const int i = blockIdx.x * 8 + static_cast<int>(threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (i >= n_atoms) return;
  const int eb = __ldg(row_ptr + i), ee = __ldg(row_ptr + i + 1);
  float2 acc = make_float2(0.f, 0.f);
  for (int e0 = eb; e0 < ee; e0 += 32) {
    const int n = min(32, ee - e0);
    const int mp = lane < n ? __ldg(pidx + e0 + lane) : 0;
    const int mj = lane < n ? __ldg(col + e0 + lane) : 0;
    for (int k0 = 0; k0 < n; k0 += KF) {
      float2 a[KF], b[KF];
#pragma unroll
      for (int k = 0; k < KF; ++k) {
        const int pk = __shfl_sync(0xffffffffu, mp, k0 + k), jk = __shfl_sync(0xffffffffu, mj, k0 + k);
        a[k] = __ldg(reinterpret_cast<const float2*>(w + (size_t)pk * H) + lane);
        b[k] = __ldg(reinterpret_cast<const float2*>(bm + (size_t)jk * H) + lane);
      }
#pragma unroll
      for (int k = 0; k < KF; ++k)
        if (k0 + k < n) {
          acc.x = fmaf(a[k].x, b[k].x, acc.x);
          acc.y = fmaf(a[k].y, b[k].y, acc.y);
        }
    }
  }
  reinterpret_cast<float2*>(Yb_out + (size_t)i * H)[lane] = acc;
  if (bh) {
    const float2 o = row_times_wt(acc, wt, lane);
    const float2 in = inj ? __ldg(reinterpret_cast<const float2*>(inj + (size_t)i * H) + lane) : make_float2(0.f, 0.f);
    float2* dst = reinterpret_cast<float2*>(bh + (size_t)i * H) + lane;
    float2 x = *dst;
    x.x += o.x + in.x;
    x.y += o.y + in.y;
    *dst = x;
  }
}

constexpr size_t bf_pair_smem() { return 2 * kWTile + 6 * kBTile + kSmallBytes; }
constexpr size_t be_pair_smem() { return 2 * kWTile + 4 * kBTile + kSmallBytes; }
constexpr size_t filter_smem() { return 2 * kWTile + 2 * kTile + kSmallBytes; }

}  // namespace edge_tc
}  // namespace janus
