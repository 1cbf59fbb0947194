// upd_tc.cuh — the upd unit's four phases on 5th-gen tensor cores (the
// JANUS_PREC_TF32 path; node_kernels.cuh upd_*_fused stay the fp32 path).
//
// An upd unit is a chain of [N x 64] x [64 x 64] contractions with
// elementwise steps between them (p = m U + ups, h' = h + SiLU(p) V, the
// next msg unit's v = h' W, and their derivatives).  The SIMT kernels held a
// 32-row block per 512-thread CTA and were bound by shared-memory operand
// traffic (ncu: short-scoreboard stalls on the smem weight reads, 8 CTAs x
// 10-20 us per 256-atom micro-batch ~ 20% of the step's SM time).  Here a CTA
// takes 128 atoms: every contraction of the chain is one M=128 x N=64 x K=64
// tcgen05 MMA group from SWIZZLE_128B K-major tiles (the row block is the A
// operand, the weight the B operand), the accumulators sit in TMEM, and the
// epilogues (thread = atom row = TMEM lane, 16 features per thread) stage the
// next operand straight back into the A tile.
//
// Precision: FE and FF (which carry energies and forces) run 3xTF32 —
// x = hi + lo with hi = tf32(x), x.W ~ hi.Whi + hi.Wlo + lo.Whi — fp32-level
// accuracy; BF and BE (gradient-only) run plain tf32.
//
// Weights: per upd unit one packed image of K-major B tiles, rebuilt after
// every optimizer step (pack_upd_weights) and pulled by 1-D bulk copies:
//   [U | U_lo | V | V_lo | V^T | V^T_lo | U^T | U^T_lo]  (16 KB each)
// where "M" is the B operand of X.M and "M^T" that of X.M^T; each msg unit's
// pack gets [W | W_lo] appended (kWkOff) for the fused next-v products.
#pragma once

#include "edge_tc.cuh"

namespace janus {
namespace upd_tc {

using edge_tc::Ctx;
using edge_tc::FPT;
using edge_tc::kTile;
using edge_tc::kWTile;
using edge_tc::NT;

constexpr uint32_t kUpdPackBytes = 8 * kWTile;
enum : int { kU = 0, kUlo = 1, kV = 2, kVlo = 3, kVt = 4, kVtlo = 5, kUt = 6, kUtlo = 7 };
// msg pack: [W | W_lo] after the edge kernels' image
constexpr uint32_t kWkOff = edge_tc::kPackBytes;
constexpr uint32_t kMsgPackBytes = kWkOff + 2 * kWTile;

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// B tile element (n, k) of X.M is M[k][n]; of X.M^T it is M[n][k].
__device__ __forceinline__ void put_b(uint8_t* dst, int tile, int n, int k, float v) {
  *reinterpret_cast<float*>(dst + tile * kWTile + tc::sw128_off(n, k, 64)) = v;
}

// U, V: [64][64] row-major (upd parameters); pack: kUpdPackBytes
__global__ void pack_upd_weights(const float* __restrict__ U, const float* __restrict__ V, float* __restrict__ pack) {
  JANUS_GDC_WAIT();
  uint8_t* dst = reinterpret_cast<uint8_t*>(pack);
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= 64 * 64) return;
  const int a = x / 64, b = x % 64;  // M[a][b]
  const float u = U[x], v = V[x], uh = tf32_rna(u), vh = tf32_rna(v);
  put_b(dst, kU, b, a, uh);          // X.U: (n = b, k = a)
  put_b(dst, kUlo, b, a, u - uh);
  put_b(dst, kV, b, a, vh);
  put_b(dst, kVlo, b, a, v - vh);
  put_b(dst, kVt, a, b, vh);         // X.V^T: (n = a, k = b)
  put_b(dst, kVtlo, a, b, v - vh);
  put_b(dst, kUt, a, b, uh);
  put_b(dst, kUtlo, a, b, u - uh);
}

// the msg unit's W as the B operand of X.W (hi, lo) at kWkOff of its pack
__global__ void pack_msg_w(const float* __restrict__ W, float* __restrict__ pack) {
  JANUS_GDC_WAIT();
  uint8_t* dst = reinterpret_cast<uint8_t*>(pack) + kWkOff;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= 64 * 64) return;
  const int a = x / 64, b = x % 64;
  const float w = W[x], wh = tf32_rna(w);
  put_b(dst, 0, b, a, wh);
  put_b(dst, 1, b, a, w - wh);
}

constexpr size_t upd_tc_smem(int wtiles, int atiles) { return wtiles * kWTile + atiles * kTile + 1024; }

// ------------------------------------------------------------------ helpers
struct Rows {
  int i0, rows;
};

// this thread's 16 features of row e of x (zeros past the end)
__device__ __forceinline__ void ld_row(const float* __restrict__ x, const Rows& rw, int e, int f0, float (&v)[FPT]) {
  const int i = rw.i0 + e;
  if (i < rw.rows) {
    const float4* p = reinterpret_cast<const float4*>(x + static_cast<size_t>(i) * 64 + f0);
#pragma unroll
    for (int j = 0; j < FPT / 4; ++j) {
      const float4 t = __ldg(p + j);
      v[4 * j] = t.x, v[4 * j + 1] = t.y, v[4 * j + 2] = t.z, v[4 * j + 3] = t.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < FPT; ++j) v[j] = 0.f;
  }
}
__device__ __forceinline__ void st_row(float* __restrict__ x, const Rows& rw, int e, int f0, const float (&v)[FPT]) {
  const int i = rw.i0 + e;
  if (i >= rw.rows) return;
  float4* p = reinterpret_cast<float4*>(x + static_cast<size_t>(i) * 64 + f0);
#pragma unroll
  for (int j = 0; j < FPT / 4; ++j) p[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
}
// the A operand: plain (tf32 = the hardware's truncation of fp32 operands) or split hi / lo
__device__ __forceinline__ void st_a(uint8_t* hi, uint8_t* lo, int e, int f0, const float (&v)[FPT]) {
  if (!lo) {
    edge_tc::st_em(hi, e, f0, v);
    return;
  }
  float h[FPT], l[FPT];
#pragma unroll
  for (int j = 0; j < FPT; ++j) {
    h[j] = tf32_rna(v[j]);
    l[j] = v[j] - h[j];
  }
  edge_tc::st_em(hi, e, f0, h);
  edge_tc::st_em(lo, e, f0, l);
}
// D = X.W (one thread issues): 3xTF32 when lo tiles are given
__device__ __forceinline__ void mma3(uint32_t d, uint32_t xh, uint32_t xl, uint32_t wh, uint32_t wl) {
  if (xl) {
    edge_tc::mma_tiles<128, 64, 64, 128>(d, xl, wh, false);
    edge_tc::mma_tiles<128, 64, 64, 128>(d, xh, wl, true);
    edge_tc::mma_tiles<128, 64, 64, 128>(d, xh, wh, true);
  } else {
    edge_tc::mma_tiles<128, 64, 64, 128>(d, xh, wh, false);
  }
}

__device__ __forceinline__ void load_tiles(uint8_t* dst, const float* src, uint32_t bytes, uint64_t* wbar, uint32_t total) {
  if (threadIdx.x == 0) {
    if (total) tc::mbar_expect_tx(wbar, total);
    tc::bulk_g2s(dst, src, bytes, wbar);
  }
}
__device__ __forceinline__ void init_wbar(uint64_t* wbar) {
  if (threadIdx.x == 0) {
    tc::mbar_init(wbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
}

constexpr uint32_t TA = 0, TB = 64, TC = 128;  // TMEM accumulators (64 columns each)

// ======================================================================= FE
// p = m U + ups ; h_out = h + SiLU(p) V ; v_out = h_out Wn (Wn: the next msg
// unit's pack, or null).  3xTF32.
__global__ void __launch_bounds__(NT, 1) upd_fe_tc(int rows, const float* __restrict__ m, const float* __restrict__ h,
                                                   const float* __restrict__ upack, const float* __restrict__ ups,
                                                   float* __restrict__ p_out, float* __restrict__ h_out,
                                                   const float* __restrict__ wpack, float* __restrict__ v_out) {
  JANUS_GDC_WAIT();
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = edge_tc::align1024(sm_raw);
  uint8_t* W = sm;                  // U, U_lo, V, V_lo, [Wn, Wn_lo]
  uint8_t* Xh = sm + 6 * kWTile;
  uint8_t* Xl = Xh + kTile;
  __shared__ __align__(8) uint64_t mbar, wbar;
  __shared__ uint32_t tslot;
  Ctx c;
  c.sm = sm;
  c.mbar = &mbar;
  init_wbar(&wbar);
  const uint32_t wbytes = 4 * kWTile + (wpack ? 2 * kWTile : 0u);
  load_tiles(W, upack, 4 * kWTile, &wbar, wbytes);
  if (wpack) load_tiles(W + 4 * kWTile, reinterpret_cast<const float*>(reinterpret_cast<const uint8_t*>(wpack) + kWkOff),
                        2 * kWTile, &wbar, 0);
  edge_tc::setup(c, &tslot, 256);
  const Rows rw{static_cast<int>(blockIdx.x) * 128, rows};
  const int f0 = FPT * c.q;
  const uint32_t aW = tc::smem_u32(W), aXh = tc::smem_u32(Xh), aXl = tc::smem_u32(Xl);
  float v[FPT];
  ld_row(m, rw, c.e, f0, v);
  st_a(Xh, Xl, c.e, f0, v);
  tc::mbar_wait(&wbar, 0);
  c.publish();
  if (threadIdx.x == 0) {
    mma3(c.tmem + TA, aXh, aXl, aW + kU * kWTile, aW + kUlo * kWTile);
    tc::commit(c.mbar);
  }
  c.wait_mma();
  c.ld(TA, v);
#pragma unroll
  for (int j = 0; j < FPT; ++j) v[j] += __ldg(ups + f0 + j);
  st_row(p_out, rw, c.e, f0, v);
#pragma unroll
  for (int j = 0; j < FPT; ++j) v[j] = dev::silu(v[j]);
  st_a(Xh, Xl, c.e, f0, v);  // the MMA that read X is complete
  c.publish();
  if (threadIdx.x == 0) {
    mma3(c.tmem + TB, aXh, aXl, aW + kV * kWTile, aW + kVlo * kWTile);
    tc::commit(c.mbar);
  }
  c.wait_mma();
  float hh[FPT];
  ld_row(h, rw, c.e, f0, hh);
  c.ld(TB, v);
#pragma unroll
  for (int j = 0; j < FPT; ++j) v[j] += hh[j];
  st_row(h_out, rw, c.e, f0, v);
  if (wpack) {
    st_a(Xh, Xl, c.e, f0, v);
    c.publish();
    if (threadIdx.x == 0) {
      mma3(c.tmem + TC, aXh, aXl, aW + 4 * kWTile, aW + 5 * kWTile);
      tc::commit(c.mbar);
    }
    c.wait_mma();
    c.ld(TC, v);
    st_row(v_out, rw, c.e, f0, v);
  }
  edge_tc::teardown(c, 256);
}

// ======================================================================= FF
// ff_a = a' ; am = ((a' V^T) SiLU'(p)) U^T.  3xTF32.
__global__ void __launch_bounds__(NT, 1) upd_ff_tc(int rows, const float* __restrict__ a, const float* __restrict__ p,
                                                   const float* __restrict__ upack, float* __restrict__ ff_a,
                                                   float* __restrict__ am) {
  JANUS_GDC_WAIT();
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = edge_tc::align1024(sm_raw);
  uint8_t* W = sm;  // V^T, V^T_lo, U^T, U^T_lo
  uint8_t* Xh = sm + 4 * kWTile;
  uint8_t* Xl = Xh + kTile;
  __shared__ __align__(8) uint64_t mbar, wbar;
  __shared__ uint32_t tslot;
  Ctx c;
  c.sm = sm;
  c.mbar = &mbar;
  init_wbar(&wbar);
  load_tiles(W, reinterpret_cast<const float*>(reinterpret_cast<const uint8_t*>(upack) + kVt * kWTile), 4 * kWTile, &wbar,
             4 * kWTile);
  edge_tc::setup(c, &tslot, 128);
  const Rows rw{static_cast<int>(blockIdx.x) * 128, rows};
  const int f0 = FPT * c.q;
  const uint32_t aW = tc::smem_u32(W), aXh = tc::smem_u32(Xh), aXl = tc::smem_u32(Xl);
  float v[FPT];
  ld_row(a, rw, c.e, f0, v);
  st_row(ff_a, rw, c.e, f0, v);
  st_a(Xh, Xl, c.e, f0, v);
  tc::mbar_wait(&wbar, 0);
  c.publish();
  if (threadIdx.x == 0) {
    mma3(c.tmem + TA, aXh, aXl, aW, aW + kWTile);
    tc::commit(c.mbar);
  }
  c.wait_mma();
  float pp[FPT];
  ld_row(p, rw, c.e, f0, pp);
  c.ld(TA, v);
#pragma unroll
  for (int j = 0; j < FPT; ++j) v[j] *= dev::dsilu(pp[j]);
  st_a(Xh, Xl, c.e, f0, v);
  c.publish();
  if (threadIdx.x == 0) {
    mma3(c.tmem + TB, aXh, aXl, aW + 2 * kWTile, aW + 3 * kWTile);
    tc::commit(c.mbar);
  }
  c.wait_mma();
  c.ld(TB, v);
  st_row(am, rw, c.e, f0, v);
  edge_tc::teardown(c, 128);
}

// ======================================================================= BF
// pdot = abar_m U ; r = a' V^T ; pbar = r pdot SiLU''(p) ; pdbar = r SiLU'(p) ;
// u = SiLU'(p) pdot ; inj = pbar U^T ; abar_h' = abar_h + u V ; vdot = abar_h' Wn.
// tf32 (gradient-only).
__global__ void __launch_bounds__(NT, 1) upd_bf_tc(int rows, const float* __restrict__ am, const float* __restrict__ ffa,
                                                   const float* __restrict__ p, const float* __restrict__ upack,
                                                   float* __restrict__ pbar, float* __restrict__ pdbar,
                                                   float* __restrict__ u, float* __restrict__ inj, const float* ah,
                                                   float* ah_out, const float* __restrict__ wpack,
                                                   float* __restrict__ vdot_out) {
  JANUS_GDC_WAIT();
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = edge_tc::align1024(sm_raw);
  uint8_t* W = sm;  // U, V^T, U^T, V, [Wn]
  uint8_t* X1 = sm + 5 * kWTile;
  uint8_t* X2 = X1 + kTile;
  __shared__ __align__(8) uint64_t mbar, wbar;
  __shared__ uint32_t tslot;
  Ctx c;
  c.sm = sm;
  c.mbar = &mbar;
  init_wbar(&wbar);
  const uint8_t* up = reinterpret_cast<const uint8_t*>(upack);
  if (threadIdx.x == 0) {
    tc::mbar_expect_tx(&wbar, (wpack ? 5u : 4u) * kWTile);
    tc::bulk_g2s(W, up + kU * kWTile, kWTile, &wbar);
    tc::bulk_g2s(W + kWTile, up + kVt * kWTile, kWTile, &wbar);
    tc::bulk_g2s(W + 2 * kWTile, up + kUt * kWTile, kWTile, &wbar);
    tc::bulk_g2s(W + 3 * kWTile, up + kV * kWTile, kWTile, &wbar);
    if (wpack) tc::bulk_g2s(W + 4 * kWTile, reinterpret_cast<const uint8_t*>(wpack) + kWkOff, kWTile, &wbar);
  }
  edge_tc::setup(c, &tslot, 256);
  const Rows rw{static_cast<int>(blockIdx.x) * 128, rows};
  const int f0 = FPT * c.q;
  const uint32_t aW = tc::smem_u32(W), a1 = tc::smem_u32(X1), a2 = tc::smem_u32(X2);
  float x[FPT], y[FPT];
  ld_row(am, rw, c.e, f0, x);
  ld_row(ffa, rw, c.e, f0, y);
  edge_tc::st_em(X1, c.e, f0, x);
  edge_tc::st_em(X2, c.e, f0, y);
  tc::mbar_wait(&wbar, 0);
  c.publish();
  if (threadIdx.x == 0) {
    edge_tc::mma_tiles<128, 64, 64, 128>(c.tmem + TA, a1, aW, false);            // pdot = abar_m U
    edge_tc::mma_tiles<128, 64, 64, 128>(c.tmem + TB, a2, aW + kWTile, false);   // r = a' V^T
    tc::commit(c.mbar);
  }
  float pp[FPT];
  ld_row(p, rw, c.e, f0, pp);
  c.wait_mma();
  c.ld2(TA, TB, x, y);  // x = pdot, y = r
  {
    float pb[FPT], pdb[FPT], uu[FPT];
#pragma unroll
    for (int j = 0; j < FPT; ++j) {
      const float ds = dev::dsilu(pp[j]);
      pb[j] = y[j] * x[j] * dev::d2silu(pp[j]);
      pdb[j] = y[j] * ds;
      uu[j] = ds * x[j];
    }
    st_row(pbar, rw, c.e, f0, pb);
    st_row(pdbar, rw, c.e, f0, pdb);
    st_row(u, rw, c.e, f0, uu);
    edge_tc::st_em(X1, c.e, f0, pb);
    edge_tc::st_em(X2, c.e, f0, uu);
  }
  c.publish();
  if (threadIdx.x == 0) {
    edge_tc::mma_tiles<128, 64, 64, 128>(c.tmem + TA, a1, aW + 2 * kWTile, false);  // inj = pbar U^T
    edge_tc::mma_tiles<128, 64, 64, 128>(c.tmem + TB, a2, aW + 3 * kWTile, false);  // u V
    tc::commit(c.mbar);
  }
  float a4[FPT];
  ld_row(ah, rw, c.e, f0, a4);
  c.wait_mma();
  c.ld2(TA, TB, x, y);
  st_row(inj, rw, c.e, f0, x);
#pragma unroll
  for (int j = 0; j < FPT; ++j) y[j] += a4[j];
  __syncthreads();  // every row of ah was read before ah_out (it may alias ah) is written
  st_row(ah_out, rw, c.e, f0, y);
  if (wpack) {
    edge_tc::st_em(X1, c.e, f0, y);
    c.publish();
    if (threadIdx.x == 0) {
      edge_tc::mma_tiles<128, 64, 64, 128>(c.tmem + TC, a1, aW + 4 * kWTile, false);  // vdot = abar_h' Wn
      tc::commit(c.mbar);
    }
    c.wait_mma();
    c.ld(TC, x);
    st_row(vdot_out, rw, c.e, f0, x);
  }
  edge_tc::teardown(c, 256);
}

// ======================================================================= BE
// r = b' V^T ; pbar = r SiLU'(p) ; b_m = pbar U^T + inj.  tf32 (gradient-only).
__global__ void __launch_bounds__(NT, 1) upd_be_tc(int rows, const float* __restrict__ bh, const float* __restrict__ p,
                                                   const float* __restrict__ upack, const float* __restrict__ inj,
                                                   float* __restrict__ pbar, float* __restrict__ bm) {
  JANUS_GDC_WAIT();
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = edge_tc::align1024(sm_raw);
  uint8_t* W = sm;  // V^T, U^T
  uint8_t* X = sm + 2 * kWTile;
  __shared__ __align__(8) uint64_t mbar, wbar;
  __shared__ uint32_t tslot;
  Ctx c;
  c.sm = sm;
  c.mbar = &mbar;
  init_wbar(&wbar);
  const uint8_t* up = reinterpret_cast<const uint8_t*>(upack);
  if (threadIdx.x == 0) {
    tc::mbar_expect_tx(&wbar, 2 * kWTile);
    tc::bulk_g2s(W, up + kVt * kWTile, kWTile, &wbar);
    tc::bulk_g2s(W + kWTile, up + kUt * kWTile, kWTile, &wbar);
  }
  edge_tc::setup(c, &tslot, 128);
  const Rows rw{static_cast<int>(blockIdx.x) * 128, rows};
  const int f0 = FPT * c.q;
  const uint32_t aW = tc::smem_u32(W), aX = tc::smem_u32(X);
  float v[FPT];
  ld_row(bh, rw, c.e, f0, v);
  edge_tc::st_em(X, c.e, f0, v);
  tc::mbar_wait(&wbar, 0);
  c.publish();
  if (threadIdx.x == 0) {
    edge_tc::mma_tiles<128, 64, 64, 128>(c.tmem + TA, aX, aW, false);  // r = b' V^T
    tc::commit(c.mbar);
  }
  float pp[FPT];
  ld_row(p, rw, c.e, f0, pp);
  c.wait_mma();
  c.ld(TA, v);
#pragma unroll
  for (int j = 0; j < FPT; ++j) v[j] *= dev::dsilu(pp[j]);
  st_row(pbar, rw, c.e, f0, v);
  edge_tc::st_em(X, c.e, f0, v);
  c.publish();
  if (threadIdx.x == 0) {
    edge_tc::mma_tiles<128, 64, 64, 128>(c.tmem + TB, aX, aW + kWTile, false);  // pbar U^T
    tc::commit(c.mbar);
  }
  float in[FPT];
  ld_row(inj, rw, c.e, f0, in);
  c.wait_mma();
  c.ld(TB, v);
#pragma unroll
  for (int j = 0; j < FPT; ++j) v[j] += in[j];
  st_row(bm, rw, c.e, f0, v);
  edge_tc::teardown(c, 128);
}

// ================================================================ X . W
// out = X W with the msg unit's W: the same split / MMA sequence as the fused
// next-v products of upd_fe_tc (split3: 3xTF32) and upd_bf_tc (plain tf32),
// so a msg unit whose v / vdot is not fused into the preceding upd kernel
// (first unit of a stage, after the embedding) gets the same bits — staged
// runs stay bit-identical to unstaged ones.
__global__ void __launch_bounds__(NT, 1) rows_w_tc(int rows, const float* __restrict__ X, const float* __restrict__ wpack,
                                                   int split3, float* __restrict__ out) {
  JANUS_GDC_WAIT();
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = edge_tc::align1024(sm_raw);
  uint8_t* W = sm;  // W, W_lo
  uint8_t* Xh = sm + 2 * kWTile;
  uint8_t* Xl = Xh + kTile;
  __shared__ __align__(8) uint64_t mbar, wbar;
  __shared__ uint32_t tslot;
  Ctx c;
  c.sm = sm;
  c.mbar = &mbar;
  init_wbar(&wbar);
  load_tiles(W, reinterpret_cast<const float*>(reinterpret_cast<const uint8_t*>(wpack) + kWkOff), 2 * kWTile, &wbar,
             2 * kWTile);
  edge_tc::setup(c, &tslot, 64);
  const Rows rw{static_cast<int>(blockIdx.x) * 128, rows};
  const int f0 = FPT * c.q;
  const uint32_t aW = tc::smem_u32(W), aXh = tc::smem_u32(Xh), aXl = tc::smem_u32(Xl);
  float v[FPT];
  ld_row(X, rw, c.e, f0, v);
  st_a(Xh, split3 ? Xl : nullptr, c.e, f0, v);
  tc::mbar_wait(&wbar, 0);
  c.publish();
  if (threadIdx.x == 0) {
    mma3(c.tmem, aXh, split3 ? aXl : 0u, aW, aW + kWTile);
    tc::commit(c.mbar);
  }
  c.wait_mma();
  c.ld(0, v);
  st_row(out, rw, c.e, f0, v);
  edge_tc::teardown(c, 64);
}

}  // namespace upd_tc
}  // namespace janus
