// edge_tc.cuh — the msg unit's four phases on 5th-gen tensor cores
// (tcgen05.mma kind::tf32, accumulators in TMEM), the JANUS_PREC_TF32 path.
// Same math as edge_kernels.cuh (SIMT fp32 parity path).
//
// Work decomposition (512 threads; thread t owns edge row e = t % 128 of the
// tile = TMEM lane e, and feature quarter t / 128, i.e. 16 features):
//  * an edge tile = <= 8 CSR rows with <= 128 edges (a long row is chunked);
//  * every per-edge contraction is an M=128 x N=64 x K=64 MMA from shared
//    memory: A = the tile's edge-major operand, B = a weight tile;
//  * the epilogue reads the 128x64 accumulator with tcgen05.ld (thread = edge)
//    and applies SiLU', SiLU'', cutoff, ... in registers;
//  * weight gradients sum_e X_e^T Y_e are M=64 x N=64 x K=128 MMAs over
//    feature-major (transposed) tiles, accumulated in TMEM across all tiles of
//    the CTA (BF/BE run persistent CTAs with a static tile assignment, so the
//    per-CTA partials and their ordered reduction are deterministic);
//  * all operand tiles use the SWIZZLE_128B K-major layout (tc::sw128_off): the
//    edge-major float4 stores and the feature-major scalar stores are both
//    bank-conflict-free; the tcgen05 MN-major (transpose) path was measured to
//    return zeros for kind::tf32 (tests/test_gpu_tc.py) and is not used.
#pragma once

#include "common.cuh"
#include "edge_kernels.cuh"
#include "tc.cuh"

namespace janus {
namespace edge_tc {

constexpr int TE = 128;
constexpr int NT = 512;            // 16 warps: 4 threads per edge row
constexpr int NQ = NT / TE;        // feature quarters per edge
constexpr int FPT = 64 / NQ;       // features per thread (16)
constexpr int PAIRS = 8 * 64 / NT; // (row, feature) pairs per thread in the segmented sums
constexpr int H = 64, R = 64;
constexpr int kRowsPerTile = 8;
constexpr uint32_t kTile = 128 * 64 * 4;  // 32 KB operand tile
constexpr uint32_t kWTile = 64 * 64 * 4;  // 16 KB weight tile
constexpr int PE = R * H + H + H * H + H;
// TMEM columns
constexpr uint32_t TM_Z = 0, TM_ZP = 64, TM_G = 128, TM_GP = 192, TM_AG = 256, TM_BG = 320;

__device__ __forceinline__ uint32_t off_em(int e, int f) { return tc::sw128_off(e, f, 128); }  // [128 edges][64 feat]
__device__ __forceinline__ uint32_t off_fm(int f, int e) { return tc::sw128_off(f, e, 64); }   // [64 feat][128 edges]

// D[tmem] (+)= A(rows a_rows, K) . B(rows b_rows, K)^T, K-major SWIZZLE_128B tiles.
__device__ __forceinline__ void mma_tiles(uint32_t d, uint32_t a, int a_rows, uint32_t b, int b_rows, int K, int M,
                                          bool accumulate) {
  const uint32_t id = tc::idesc_tf32(M, 64, false, false);
  const uint32_t as = static_cast<uint32_t>(a_rows) * 128u, bs = static_cast<uint32_t>(b_rows) * 128u;
#pragma unroll 1
  for (int s = 0; s < K / 8; ++s) {
    const uint64_t da = tc::smem_desc(a + (s >> 2) * as + 32u * (s & 3), 16, 1024, 2);
    const uint64_t db = tc::smem_desc(b + (s >> 2) * bs + 32u * (s & 3), 16, 1024, 2);
    tc::mma_tf32(d, da, db, id, (s > 0 || accumulate) ? 1u : 0u);
  }
}

struct Ctx {
  uint8_t* sm;
  uint64_t* mbar;
  uint32_t tmem;
  uint32_t phase;
  int e, q, warp, lane;
  __device__ uint32_t lane_base() const { return static_cast<uint32_t>((warp & 3) * 32) << 16; }
  // all threads: make smem writes visible to the tensor core, order TMEM reads, barrier
  __device__ void publish() {
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
  }
  __device__ void wait_mma() {
    tc::mbar_wait(mbar, phase);
    phase ^= 1u;
    tc::fence_after();
  }
  __device__ void ld(uint32_t col, float (&v)[FPT]) const { tc::ld16(tmem + lane_base() + col + static_cast<uint32_t>(FPT * q), v); }
};

// Weight tile for B operands: element (n, k) = src[k*64 + n] (transpose=true)
// or src[n*64 + k].
__device__ __forceinline__ void stage_weight(uint8_t* dst, const float* __restrict__ src, bool transpose) {
  for (int x = threadIdx.x; x < 64 * 64; x += NT) {
    const int a = x / 64, b = x % 64;
    const int n = transpose ? b : a, k = transpose ? a : b;
    *reinterpret_cast<float*>(dst + tc::sw128_off(n, k, 64)) = src[x];
  }
}

// Packed weight image in global memory = the exact smem image of
// [W0 = A^T | W1 = B^T | W2 = B | alpha | beta]; rebuilt after every
// optimizer step (stage.cu refresh_transposes) and pulled by each CTA with one
// TMA bulk copy.
constexpr uint32_t kPackBytes = 3 * kWTile + 2 * 64 * 4;

__global__ void pack_msg_weights(const float* __restrict__ A, const float* __restrict__ alpha, const float* __restrict__ B,
                                 const float* __restrict__ beta, float* __restrict__ pack) {
  uint8_t* dst = reinterpret_cast<uint8_t*>(pack);
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x < 64 * 64) {
    const int a = x / 64, b = x % 64;  // src[a*64 + b]
    *reinterpret_cast<float*>(dst + tc::sw128_off(b, a, 64)) = A[x];               // A^T: (n=h=b, k=r=a)
    *reinterpret_cast<float*>(dst + kWTile + tc::sw128_off(b, a, 64)) = B[x];      // B^T: (n=out=b, k=in=a)
    *reinterpret_cast<float*>(dst + 2 * kWTile + tc::sw128_off(a, b, 64)) = B[x];  // B:   (n=a, k=b)
  }
  if (x < 64) {
    pack[3 * kWTile / 4 + x] = alpha[x];
    pack[3 * kWTile / 4 + 64 + x] = beta[x];
  }
}

// All threads: bulk-load `ntiles` weight tiles (+ alpha, beta) into sm[0..).
// Returns after the copy landed (mbarrier transaction count).
__device__ __forceinline__ void load_weights(uint8_t* sm, const float* pack, int ntiles, float* al, float* be,
                                             uint64_t* wbar) {
  if (threadIdx.x == 0) {
    tc::mbar_init(wbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint32_t wbytes = static_cast<uint32_t>(ntiles) * kWTile;
    tc::mbar_expect_tx(wbar, wbytes + 512);
    tc::bulk_g2s(sm, pack, wbytes, wbar);
    tc::bulk_g2s(al, reinterpret_cast<const uint8_t*>(pack) + 3 * kWTile, 256, wbar);
    tc::bulk_g2s(be, reinterpret_cast<const uint8_t*>(pack) + 3 * kWTile + 256, 256, wbar);
  }
  __syncthreads();
  tc::mbar_wait(wbar, 0);
}

__device__ __forceinline__ void st_em(uint8_t* t, int e, int f0, const float (&v)[FPT]) {
#pragma unroll
  for (int j = 0; j < FPT / 4; ++j)
    *reinterpret_cast<float4*>(t + off_em(e, f0 + 4 * j)) = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
}
__device__ __forceinline__ void st_fm(uint8_t* t, int e, int f0, const float (&v)[FPT]) {
#pragma unroll
  for (int j = 0; j < FPT; ++j) *reinterpret_cast<float*>(t + off_fm(f0 + j, e)) = v[j];
}
__device__ __forceinline__ float ld_em(const uint8_t* t, int e, int f) {
  return *reinterpret_cast<const float*>(t + off_em(e, f));
}

// Plain [128 edges][64 features] fp32 tile for the segmented row sums: the
// 16 B chunk index is XORed with (edge & 15) so both the per-edge float4
// stores (32 consecutive edges, same feature chunk) and the per-row reads (32
// consecutive features of one edge) are bank-conflict-free.
__device__ __forceinline__ uint32_t off_pl(int e, int f) {
  return static_cast<uint32_t>(e * 256 + ((((f >> 2) ^ (e & 15))) << 4) + ((f & 3) << 2));
}
__device__ __forceinline__ void st_pl(uint8_t* t, int e, int f0, const float (&v)[FPT]) {
#pragma unroll
  for (int j = 0; j < FPT / 4; ++j)
    *reinterpret_cast<float4*>(t + off_pl(e, f0 + 4 * j)) = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
}

// Deterministic segmented row sums of NA plain tiles over this chunk: thread t
// owns (row, feature) pairs p = t and t + 256 (row = p / 64 within the tile,
// feature = p % 64) and adds the row's chunk edges in CSR order.
template <int NA>
__device__ __forceinline__ void seg_rows(const EdgeGeom& g, int r0, int r1, int c0, int ne, const uint8_t* const (&tiles)[NA],
                                         float (&acc)[NA][PAIRS]) {
#pragma unroll
  for (int k = 0; k < PAIRS; ++k) {
    const int pidx = threadIdx.x + NT * k;
    const int r = r0 + (pidx >> 6), f = pidx & 63;
    if (r >= r1) continue;
    const int eb = max(g.row_ptr[r], c0), ee = min(g.row_ptr[r + 1], c0 + ne);
    for (int x = eb; x < ee; ++x) {
      const uint32_t o = off_pl(x - c0, f);
#pragma unroll
      for (int a = 0; a < NA; ++a) acc[a][k] += *reinterpret_cast<const float*>(tiles[a] + o);
    }
  }
}

template <int NA>
__device__ __forceinline__ void seg_write(int r0, int r1, float* const (&out)[NA], const float (&acc)[NA][PAIRS]) {
#pragma unroll
  for (int k = 0; k < PAIRS; ++k) {
    const int pidx = threadIdx.x + NT * k;
    const int r = r0 + (pidx >> 6), f = pidx & 63;
    if (r >= r1) continue;
#pragma unroll
    for (int a = 0; a < NA; ++a) out[a][(size_t)r * H + f] = acc[a][k];
  }
}

// Row epilogue fused into the edge kernels: the tile's finished rows R (from
// the segmented sums) times W^T:  out[r] = (base ? base[r] : 0) + R[r] W^T
// (+ add[r]).  Rows staged in smem (rs[8][64]), W^T ([64][64] row-major) via L1.
__device__ __forceinline__ void rows_times_wt(int r0, int r1, const float (&acc)[PAIRS], float* rs, const float* __restrict__ Wt,
                                              const float* base, const float* __restrict__ add, float* out) {
#pragma unroll
  for (int k = 0; k < PAIRS; ++k) {
    const int pidx = threadIdx.x + NT * k;
    rs[(pidx >> 6) * 64 + (pidx & 63)] = (r0 + (pidx >> 6) < r1) ? acc[k] : 0.f;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < PAIRS; ++k) {
    const int pidx = threadIdx.x + NT * k;
    const int rl = pidx >> 6, c = pidx & 63, r = r0 + rl;
    if (r >= r1) continue;
    float o0 = 0.f, o1 = 0.f;
#pragma unroll 8
    for (int q = 0; q < 64; q += 2) {
      o0 = fmaf(rs[rl * 64 + q], __ldg(Wt + q * 64 + c), o0);
      o1 = fmaf(rs[rl * 64 + q + 1], __ldg(Wt + (q + 1) * 64 + c), o1);
    }
    float y = o0 + o1;
    if (base) y += base[(size_t)r * H + c];
    if (add) y += add[(size_t)r * H + c];
    out[(size_t)r * H + c] = y;
  }
  __syncthreads();
}

// 32 consecutive features of row `row` of an [N][64] array (8 float4 loads in flight)
__device__ __forceinline__ void gather32(const float* __restrict__ x, int row, int f0, float (&v)[FPT]) {
  const float4* p = reinterpret_cast<const float4*>(x + (size_t)row * H + f0);
  float4 t[FPT / 4];
#pragma unroll
  for (int q = 0; q < FPT / 4; ++q) t[q] = __ldg(p + q);
#pragma unroll
  for (int q = 0; q < FPT / 4; ++q) {
    v[4 * q] = t[q].x;
    v[4 * q + 1] = t[q].y;
    v[4 * q + 2] = t[q].z;
    v[4 * q + 3] = t[q].w;
  }
}

// radial basis (and derivative) of this thread's edge for its 32 features
__device__ __forceinline__ void basis(float d, float rc, int f0, float (&p)[FPT], float (&dp)[FPT]) {
  const float delta = rc / (R - 1);
  const float gamma = 1.0f / (2.0f * delta * delta);
#pragma unroll
  for (int j = 0; j < FPT; ++j) {
    const float x = d - (f0 + j) * delta;
    p[j] = expf(-gamma * x * x);
    dp[j] = -2.0f * gamma * x * p[j];
  }
}

struct TileRange {
  int r0, r1, e0, e1;
};
__device__ __forceinline__ TileRange tile_range(const EdgeGeom& g, const int* tile_row, int t) {
  TileRange r;
  r.r0 = tile_row[t];
  r.r1 = tile_row[t + 1];
  r.e0 = g.row_ptr[r.r0];
  r.e1 = g.row_ptr[r.r1];
  return r;
}

__device__ __forceinline__ void setup(Ctx& c, uint32_t* tmem_slot, uint32_t ncols) {
  c.e = threadIdx.x & 127;
  c.q = threadIdx.x >> 7;
  c.warp = threadIdx.x >> 5;
  c.lane = threadIdx.x & 31;
  c.phase = 0;
  if (threadIdx.x == 0) tc::mbar_init(c.mbar, 1);
  if (c.warp == 0) tc::tmem_alloc(tmem_slot, ncols);
  c.publish();
  c.tmem = *tmem_slot;
}

__device__ __forceinline__ void teardown(Ctx& c, uint32_t ncols) {
  tc::fence_before();
  __syncthreads();
  if (c.warp == 0) tc::tmem_free(c.tmem, ncols);
}

// per-chunk edge scalars into smem (threads 0..127)
struct Scal {
  float *d, *c, *dc, *qb;
  int *src, *col;
};
__device__ __forceinline__ void load_scalars(const EdgeGeom& g, Scal& s, int c0, int ne, const float* Fbar) {
  const int t = threadIdx.x;
  if (t < TE) {
    const bool ok = t < ne;
    const int x = c0 + t;
    s.d[t] = ok ? g.d[x] : 0.f;
    s.c[t] = ok ? g.c[x] : 0.f;
    if (s.dc) s.dc[t] = ok ? g.dc[x] : 0.f;
    const int i = ok ? g.src[x] : 0, j = ok ? g.col[x] : 0;
    s.src[t] = i;
    s.col[t] = j;
    if (s.qb) {
      float q = 0.f;
      if (ok)
#pragma unroll
        for (int k = 0; k < 3; ++k) q = fmaf(Fbar[3 * i + k] - Fbar[3 * j + k], g.u[3 * x + k], q);
      s.qb[t] = q;
    }
  }
}

// ----------------------------------------------------------------------- FE
// m_i = sum_{e in row i} w_e * v[col e], w = c (SiLU(phi A + alpha) B + beta)
__global__ void __launch_bounds__(NT) msg_fe_tc(EdgeGeom g, const int* __restrict__ tiles, int n_tiles, MsgParams p,
                                               float rc, const float* __restrict__ v, float* __restrict__ m_out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* W0 = sm;               // A^T  (n = h, k = r)
  uint8_t* W1 = W0 + kWTile;      // B^T  (n = out, k = in)
  uint8_t* T0 = W1 + kWTile;      // phi -> s
  uint8_t* T1 = T0 + kTile;       // w (edge-major)
  float* fsm = reinterpret_cast<float*>(T1 + kTile);
  float* al = fsm;
  float* be = al + 64;
  Scal sc{be + 64, be + 64 + TE, nullptr, nullptr, reinterpret_cast<int*>(be + 64 + 2 * TE), reinterpret_cast<int*>(be + 64 + 3 * TE)};
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tslot;
  Ctx c;
  c.sm = sm;
  c.mbar = &mbar;
  __shared__ __align__(8) uint64_t wbar;
  load_weights(sm, p.pack, 2, al, be, &wbar);
  setup(c, &tslot, 128);
  const uint32_t aW0 = tc::smem_u32(W0), aW1 = tc::smem_u32(W1), aT0 = tc::smem_u32(T0);
  for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const TileRange tr = tile_range(g, tiles, t);
    float acc[1][PAIRS] = {};
    for (int c0 = tr.e0; c0 < tr.e1; c0 += TE) {
      const int ne = min(TE, tr.e1 - c0);
      load_scalars(g, sc, c0, ne, nullptr);
      __syncthreads();
      {
        float ph[FPT], dph[FPT];
        basis(sc.d[c.e], rc, FPT * c.q, ph, dph);
        st_em(T0, c.e, FPT * c.q, ph);
      }
      c.publish();
      if (threadIdx.x == 0) {
        mma_tiles(c.tmem + TM_Z, aT0, 128, aW0, 64, 64, 128, false);
        tc::commit(c.mbar);
      }
      c.wait_mma();
      {
        float z[FPT];
        c.ld(TM_Z, z);
#pragma unroll
        for (int j = 0; j < FPT; ++j) z[j] = dev::silu(z[j] + al[FPT * c.q + j]);
        st_em(T0, c.e, FPT * c.q, z);
      }
      c.publish();
      if (threadIdx.x == 0) {
        mma_tiles(c.tmem + TM_G, aT0, 128, aW1, 64, 64, 128, false);
        tc::commit(c.mbar);
      }
      c.wait_mma();
      {
        float gg[FPT], vj[FPT];
        gather32(v, sc.col[c.e], FPT * c.q, vj);
        c.ld(TM_G, gg);
        const float ce = sc.c[c.e];
#pragma unroll
        for (int j = 0; j < FPT; ++j) gg[j] = ce * (gg[j] + be[FPT * c.q + j]) * vj[j];  // w_e * v_j
        st_pl(T1, c.e, FPT * c.q, gg);
      }
      tc::fence_before();
      __syncthreads();
      {
        const uint8_t* const tl[1] = {T1};
        seg_rows<1>(g, tr.r0, tr.r1, c0, ne, tl, acc);
      }
      __syncthreads();
    }
    float* const outs[1] = {m_out};
    seg_write<1>(tr.r0, tr.r1, outs, acc);
  }
  teardown(c, 128);
}

// ----------------------------------------------------------------------- FF
// Y_i = sum w_e * am[col e];  F_i += sum_e (q_e + q_rev(e)) u_e with
// q_e + q_rev(e) = < am_i v_j + am_j v_i , w'_e >  (w' symmetric in e <-> rev e)
__global__ void __launch_bounds__(NT) msg_ff_tc(EdgeGeom g, const int* __restrict__ tiles, int n_tiles, MsgParams p,
                                               float rc, const float* __restrict__ v, const float* __restrict__ am,
                                               float* __restrict__ Y_out, float* __restrict__ F, const float* __restrict__ Wt,
                                               float* ah) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* W0 = sm;
  uint8_t* W1 = W0 + kWTile;
  uint8_t* T0 = W1 + kWTile;  // phi -> s -> (plain) w * am_j
  uint8_t* T1 = T0 + kTile;   // phi' -> sdot
  float* fsm = reinterpret_cast<float*>(T1 + kTile);
  float* al = fsm;
  float* be = al + 64;
  Scal sc{be + 64, be + 64 + TE, be + 64 + 2 * TE, nullptr, reinterpret_cast<int*>(be + 64 + 3 * TE),
          reinterpret_cast<int*>(be + 64 + 4 * TE)};
  float* sq = be + 64 + 5 * TE;  // [NQ][TE] per-quarter force scalars
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tslot;
  Ctx c;
  c.sm = sm;
  c.mbar = &mbar;
  __shared__ __align__(8) uint64_t wbar;
  load_weights(sm, p.pack, 2, al, be, &wbar);
  setup(c, &tslot, 256);
  const uint32_t aW0 = tc::smem_u32(W0), aW1 = tc::smem_u32(W1), aT0 = tc::smem_u32(T0), aT1 = tc::smem_u32(T1);
  const int f0 = FPT * c.q;
  for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const TileRange tr = tile_range(g, tiles, t);
    float acc[1][PAIRS] = {};
    float fsum = 0.f;  // threads < 24: (row t/3, component t%3)
    for (int c0 = tr.e0; c0 < tr.e1; c0 += TE) {
      const int ne = min(TE, tr.e1 - c0);
      load_scalars(g, sc, c0, ne, nullptr);
      __syncthreads();
      {
        float ph[FPT], dph[FPT];
        basis(sc.d[c.e], rc, f0, ph, dph);
        st_em(T0, c.e, f0, ph);
        st_em(T1, c.e, f0, dph);
      }
      c.publish();
      if (threadIdx.x == 0) {
        mma_tiles(c.tmem + TM_Z, aT0, 128, aW0, 64, 64, 128, false);
        mma_tiles(c.tmem + TM_ZP, aT1, 128, aW0, 64, 64, 128, false);
        tc::commit(c.mbar);
      }
      c.wait_mma();
      {
        float z[FPT], zp[FPT];
        c.ld(TM_Z, z);
        c.ld(TM_ZP, zp);
#pragma unroll
        for (int j = 0; j < FPT; ++j) {
          const float zz = z[j] + al[f0 + j];
          z[j] = dev::silu(zz);
          zp[j] = dev::dsilu(zz) * zp[j];
        }
        st_em(T0, c.e, f0, z);
        st_em(T1, c.e, f0, zp);
      }
      c.publish();
      if (threadIdx.x == 0) {
        mma_tiles(c.tmem + TM_G, aT0, 128, aW1, 64, 64, 128, false);
        mma_tiles(c.tmem + TM_GP, aT1, 128, aW1, 64, 64, 128, false);
        tc::commit(c.mbar);
      }
      c.wait_mma();
      {
        const int i = sc.src[c.e], j = sc.col[c.e];
        const float ce = sc.c[c.e], dce = sc.dc[c.e];
        float gg[FPT], gp[FPT];
        c.ld(TM_G, gg);
        c.ld(TM_GP, gp);
        float pq = 0.f;
        float amj[FPT];
        gather32(am, j, f0, amj);
        {
          float vj[FPT], ami[FPT], vi[FPT];
          gather32(v, j, f0, vj);
          gather32(am, i, f0, ami);
          gather32(v, i, f0, vi);
#pragma unroll
          for (int q = 0; q < FPT; ++q) {
            const float gb = gg[q] + be[f0 + q];
            const float wp = dce * gb + ce * gp[q];
            pq = fmaf(fmaf(ami[q], vj[q], amj[q] * vi[q]), wp, pq);
            gg[q] = ce * gb * amj[q];  // w_e * am_j
          }
        }
        st_pl(T0, c.e, f0, gg);
        sq[c.q * TE + c.e] = pq;
      }
      tc::fence_before();
      __syncthreads();
      {
        const uint8_t* const tl[1] = {T0};
        seg_rows<1>(g, tr.r0, tr.r1, c0, ne, tl, acc);
        if (threadIdx.x < 3 * kRowsPerTile) {
          const int r = tr.r0 + threadIdx.x / 3, comp = threadIdx.x % 3;
          if (r < tr.r1) {
            const int eb = max(g.row_ptr[r], c0), ee = min(g.row_ptr[r + 1], c0 + ne);
            for (int x = eb; x < ee; ++x)
              fsum = fmaf((sq[x - c0] + sq[TE + x - c0]) + (sq[2 * TE + x - c0] + sq[3 * TE + x - c0]), g.u[3 * x + comp], fsum);
          }
        }
      }
      __syncthreads();
    }
    float* const outs[1] = {Y_out};
    seg_write<1>(tr.r0, tr.r1, outs, acc);
    if (threadIdx.x < 3 * kRowsPerTile) {
      const int r = tr.r0 + threadIdx.x / 3;
      if (r < tr.r1) F[3 * r + threadIdx.x % 3] += fsum;
    }
    if (ah) rows_times_wt(tr.r0, tr.r1, acc[0], reinterpret_cast<float*>(T1), Wt, ah, nullptr, ah);  // a_h += Y W^T
  }
  teardown(c, 256);
}

// Write the CTA's weight-gradient partial [dA | dalpha | dB | dbeta] from the
// M=64 TMEM accumulators (row r at lane (r/16)*32 + r%16) and the per-thread
// column sums (reduced over the 128 edge threads in order through smem).
__device__ __forceinline__ void write_partial(Ctx& c, float* part, uint8_t* scratch, const float (&cs_a)[FPT],
                                              const float (&cs_b)[FPT]) {
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  {
    const int q = c.warp & 3;
    float va[FPT], vb[FPT];
    c.ld(TM_AG, va);
    c.ld(TM_BG, vb);
    if (c.lane < 16) {
      const int r = 16 * q + c.lane;
#pragma unroll
      for (int j = 0; j < FPT; ++j) {
        part[r * H + FPT * c.q + j] = va[j];              // dA[r][h]
        part[R * H + H + r * H + FPT * c.q + j] = vb[j];  // dB[k][h]
      }
    }
  }
  float* red = reinterpret_cast<float*>(scratch);  // [128][64]
  for (int pass = 0; pass < 2; ++pass) {
    const float(&cs)[FPT] = pass ? cs_b : cs_a;
#pragma unroll
    for (int j = 0; j < FPT; ++j) red[c.e * 64 + FPT * c.q + j] = cs[j];
    __syncthreads();
    if (threadIdx.x < 64) {
      float s = 0.f;
      for (int e = 0; e < TE; ++e) s += red[e * 64 + threadIdx.x];
      part[(pass ? R * H + H + H * H : R * H) + threadIdx.x] = s;
    }
    __syncthreads();
  }
}

// ----------------------------------------------------------------------- BE
// Yb_i = sum w_e * bm[col e]; gbar = c bm_i v_j; dB = s^T gbar; dbeta = sum gbar;
// zbar = (gbar B^T) SiLU'(z); dA = phi^T zbar; dalpha = sum zbar.
__global__ void __launch_bounds__(NT, 1) msg_be_tc(EdgeGeom g, const int* __restrict__ tiles, int n_tiles, MsgParams p,
                                                  float rc, const float* __restrict__ v, const float* __restrict__ bm,
                                                  float* __restrict__ Yb_out, float* __restrict__ partial,
                                                  const float* __restrict__ Wt, const float* __restrict__ inj, float* bh) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* W0 = sm;           // A^T
  uint8_t* W1 = W0 + kWTile;  // B^T
  uint8_t* W2 = W1 + kWTile;  // B
  uint8_t* T0 = W2 + kWTile;
  uint8_t* T1 = T0 + kTile;
  uint8_t* T2 = T1 + kTile;
  uint8_t* T3 = T2 + kTile;
  float* fsm = reinterpret_cast<float*>(T3 + kTile);
  float* al = fsm;
  float* be = al + 64;
  Scal sc{be + 64, be + 64 + TE, nullptr, nullptr, reinterpret_cast<int*>(be + 64 + 2 * TE),
          reinterpret_cast<int*>(be + 64 + 3 * TE)};
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tslot;
  Ctx c;
  c.sm = sm;
  c.mbar = &mbar;
  __shared__ __align__(8) uint64_t wbar;
  load_weights(sm, p.pack, 3, al, be, &wbar);
  setup(c, &tslot, 512);
  const uint32_t aW0 = tc::smem_u32(W0), aW1 = tc::smem_u32(W1), aW2 = tc::smem_u32(W2);
  const uint32_t aT0 = tc::smem_u32(T0), aT1 = tc::smem_u32(T1), aT2 = tc::smem_u32(T2), aT3 = tc::smem_u32(T3);
  float cs_a[FPT], cs_b[FPT];
#pragma unroll
  for (int j = 0; j < FPT; ++j) cs_a[j] = cs_b[j] = 0.f;
  bool first = true;
  const int f0 = FPT * c.q;
  for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const TileRange tr = tile_range(g, tiles, t);
    float acc[1][PAIRS] = {};
    for (int c0 = tr.e0; c0 < tr.e1; c0 += TE) {
      const int ne = min(TE, tr.e1 - c0);
      load_scalars(g, sc, c0, ne, nullptr);
      __syncthreads();
      {
        float ph[FPT], dph[FPT];
        basis(sc.d[c.e], rc, f0, ph, dph);
        st_em(T0, c.e, f0, ph);
      }
      c.publish();
      if (threadIdx.x == 0) {
        mma_tiles(c.tmem + TM_Z, aT0, 128, aW0, 64, 64, 128, false);
        tc::commit(c.mbar);
      }
      c.wait_mma();
      {
        float z[FPT];
        c.ld(TM_Z, z);
#pragma unroll
        for (int j = 0; j < FPT; ++j) z[j] = dev::silu(z[j] + al[f0 + j]);
        st_em(T0, c.e, f0, z);  // s, edge-major (A of g = s B)
        st_fm(T1, c.e, f0, z);  // s^T (A of dB = s^T gbar)
      }
      c.publish();
      if (threadIdx.x == 0) {
        mma_tiles(c.tmem + TM_G, aT0, 128, aW1, 64, 64, 128, false);
        tc::commit(c.mbar);
      }
      c.wait_mma();
      float gb[FPT];
      {
        const int i = sc.src[c.e], j = sc.col[c.e];
        const float ce = sc.c[c.e];
        float gg[FPT], bj[FPT];
        c.ld(TM_G, gg);
        gather32(bm, j, f0, bj);
#pragma unroll
        for (int q = 0; q < FPT; ++q) gg[q] = ce * (gg[q] + be[f0 + q]) * bj[q];  // w_e * bm_j
        st_pl(T0, c.e, f0, gg);
        float bi[FPT], vj[FPT];
        gather32(bm, i, f0, bi);
        gather32(v, j, f0, vj);
#pragma unroll
        for (int q = 0; q < FPT; ++q) {
          gb[q] = ce * bi[q] * vj[q];  // gbar (zero on padding edges: c = 0)
          cs_b[q] += gb[q];
        }
      }
      st_fm(T2, c.e, f0, gb);  // gbar^T (B of dB)
      st_em(T3, c.e, f0, gb);  // gbar   (A of sbar = gbar B^T)
      c.publish();
      if (threadIdx.x == 0) {
        mma_tiles(c.tmem + TM_BG, aT1, 64, aT2, 64, 128, 64, !first);
        mma_tiles(c.tmem + TM_G, aT3, 128, aW2, 64, 64, 128, false);
        tc::commit(c.mbar);
      }
      {  // row sums overlap the MMAs (they read T1..T3, this reads T0)
        const uint8_t* const tl[1] = {T0};
        seg_rows<1>(g, tr.r0, tr.r1, c0, ne, tl, acc);
      }
      c.wait_mma();
      __syncthreads();  // T0 reads done before it is rewritten
      {
        float z[FPT], sb[FPT];
        c.ld(TM_Z, z);
        c.ld(TM_G, sb);
#pragma unroll
        for (int j = 0; j < FPT; ++j) {
          z[j] = sb[j] * dev::dsilu(z[j] + al[f0 + j]);
          cs_a[j] += z[j];
        }
        st_fm(T2, c.e, f0, z);  // zbar^T
        float ph[FPT], dph[FPT];
        basis(sc.d[c.e], rc, f0, ph, dph);
        st_fm(T0, c.e, f0, ph);  // phi^T
      }
      c.publish();
      if (threadIdx.x == 0) {
        mma_tiles(c.tmem + TM_AG, aT0, 64, aT2, 64, 128, 64, !first);
        tc::commit(c.mbar);
      }
      c.wait_mma();
      first = false;
      __syncthreads();
    }
    float* const outs[1] = {Yb_out};
    seg_write<1>(tr.r0, tr.r1, outs, acc);
    if (bh) rows_times_wt(tr.r0, tr.r1, acc[0], reinterpret_cast<float*>(T1), Wt, bh, inj, bh);  // b_h += Yb W^T + inj
  }
  float* part = partial + (size_t)blockIdx.x * PE;
  if (first) {  // CTA without tiles: zero partial (TMEM accumulators never written)
    for (int x = threadIdx.x; x < PE; x += NT) part[x] = 0.f;
    teardown(c, 512);
    return;
  }
  write_partial(c, part, T0, cs_a, cs_b);
  teardown(c, 512);
}

// ----------------------------------------------------------------------- BF
// Second-order term.  Outputs: mdot_i = sum_e qb w'_e v_j + w_e vdot_j,
// X_i = sum_e qb w'_e am_j, and the partial [dA | dalpha | dB | dbeta].
__global__ void __launch_bounds__(NT, 1) msg_bf_tc(EdgeGeom g, const int* __restrict__ tiles, int n_tiles, MsgParams p,
                                                  float rc, const float* __restrict__ v, const float* __restrict__ vdot,
                                                  const float* __restrict__ am, const float* __restrict__ Fbar,
                                                  float* __restrict__ mdot_out, float* __restrict__ X_out,
                                                  float* __restrict__ partial, const float* __restrict__ Wt,
                                                  float* __restrict__ inj) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* W0 = sm;
  uint8_t* W1 = W0 + kWTile;
  uint8_t* W2 = W1 + kWTile;
  uint8_t* T0 = W2 + kWTile;
  uint8_t* T1 = T0 + kTile;
  uint8_t* T2 = T1 + kTile;
  uint8_t* T3 = T2 + kTile;
  float* fsm = reinterpret_cast<float*>(T3 + kTile);
  float* al = fsm;
  float* be = al + 64;
  Scal sc{be + 64, be + 64 + TE, be + 64 + 2 * TE, be + 64 + 3 * TE, reinterpret_cast<int*>(be + 64 + 4 * TE),
          reinterpret_cast<int*>(be + 64 + 5 * TE)};
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tslot;
  Ctx c;
  c.sm = sm;
  c.mbar = &mbar;
  __shared__ __align__(8) uint64_t wbar;
  load_weights(sm, p.pack, 3, al, be, &wbar);
  setup(c, &tslot, 512);
  const uint32_t aW0 = tc::smem_u32(W0), aW1 = tc::smem_u32(W1), aW2 = tc::smem_u32(W2);
  const uint32_t aT0 = tc::smem_u32(T0), aT1 = tc::smem_u32(T1), aT2 = tc::smem_u32(T2), aT3 = tc::smem_u32(T3);
  float cs_a[FPT], cs_b[FPT];
#pragma unroll
  for (int j = 0; j < FPT; ++j) cs_a[j] = cs_b[j] = 0.f;
  bool first = true;
  const int f0 = FPT * c.q;
  for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const TileRange tr = tile_range(g, tiles, t);
    float acc[2][PAIRS] = {};
    for (int c0 = tr.e0; c0 < tr.e1; c0 += TE) {
      const int ne = min(TE, tr.e1 - c0);
      load_scalars(g, sc, c0, ne, Fbar);
      __syncthreads();
      {
        float ph[FPT], dph[FPT];
        basis(sc.d[c.e], rc, f0, ph, dph);
        st_em(T0, c.e, f0, ph);
        st_em(T1, c.e, f0, dph);
      }
      c.publish();
      if (threadIdx.x == 0) {
        mma_tiles(c.tmem + TM_Z, aT0, 128, aW0, 64, 64, 128, false);
        mma_tiles(c.tmem + TM_ZP, aT1, 128, aW0, 64, 64, 128, false);
        tc::commit(c.mbar);
      }
      c.wait_mma();
      {
        float z[FPT], zp[FPT];
        c.ld(TM_Z, z);
        c.ld(TM_ZP, zp);
#pragma unroll
        for (int j = 0; j < FPT; ++j) {
          const float zz = z[j] + al[f0 + j];
          z[j] = dev::silu(zz);
          zp[j] = dev::dsilu(zz) * zp[j];
        }
        st_em(T0, c.e, f0, z);   // s
        st_em(T1, c.e, f0, zp);  // sdot
        st_fm(T2, c.e, f0, z);   // s^T
        st_fm(T3, c.e, f0, zp);  // sdot^T
      }
      c.publish();
      if (threadIdx.x == 0) {
        mma_tiles(c.tmem + TM_G, aT0, 128, aW1, 64, 64, 128, false);
        mma_tiles(c.tmem + TM_GP, aT1, 128, aW1, 64, 64, 128, false);
        tc::commit(c.mbar);
      }
      c.wait_mma();
      float mu[FPT], nu[FPT];
      {
        const int i = sc.src[c.e], j = sc.col[c.e];
        const float qb = sc.qb[c.e], ce = sc.c[c.e], dce = sc.dc[c.e];
        float gg[FPT], gp[FPT];
        c.ld(TM_G, gg);
        c.ld(TM_GP, gp);
        float pm[FPT], px[FPT];
#pragma unroll
        for (int q = 0; q < FPT / 4; ++q) {
          const float4 a4 = __ldg(reinterpret_cast<const float4*>(am + (size_t)i * H + f0) + q);
          const float4 aj4 = __ldg(reinterpret_cast<const float4*>(am + (size_t)j * H + f0) + q);
          const float4 v4 = __ldg(reinterpret_cast<const float4*>(v + (size_t)j * H + f0) + q);
          const float4 d4 = __ldg(reinterpret_cast<const float4*>(vdot + (size_t)j * H + f0) + q);
          const float ai[4] = {a4.x, a4.y, a4.z, a4.w}, aj[4] = {aj4.x, aj4.y, aj4.z, aj4.w};
          const float vv[4] = {v4.x, v4.y, v4.z, v4.w}, dv[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int k = 4 * q + r;
            const float gb = gg[k] + be[f0 + k];
            const float w = ce * gb, wp = qb * (dce * gb + ce * gp[k]);
            pm[k] = fmaf(wp, vv[r], w * dv[r]);  // qb w' v_j + w vdot_j
            px[k] = wp * aj[r];                  // qb w' am_j
            const float rho = ai[r] * vv[r], kap = ai[r] * dv[r];
            mu[k] = qb * dce * rho + ce * kap;
            nu[k] = qb * ce * rho;
          }
        }
        st_pl(T0, c.e, f0, pm);
        st_pl(T1, c.e, f0, px);
#pragma unroll
        for (int q = 0; q < FPT; ++q) cs_b[q] += mu[q];
      }
      tc::fence_before();
      __syncthreads();
      {
        const uint8_t* const tl[2] = {T0, T1};
        seg_rows<2>(g, tr.r0, tr.r1, c0, ne, tl, acc);
      }
      __syncthreads();         // row sums done with T0/T1
      st_fm(T0, c.e, f0, mu);  // mu^T
      st_fm(T1, c.e, f0, nu);  // nu^T
      c.publish();
      if (threadIdx.x == 0) {  // dB += s^T mu + sdot^T nu
        mma_tiles(c.tmem + TM_BG, aT2, 64, aT0, 64, 128, 64, !first);
        mma_tiles(c.tmem + TM_BG, aT3, 64, aT1, 64, 128, 64, true);
        tc::commit(c.mbar);
      }
      c.wait_mma();
      st_em(T2, c.e, f0, mu);  // mu (A of sbar = mu B^T)
      st_em(T3, c.e, f0, nu);  // nu
      c.publish();
      if (threadIdx.x == 0) {
        mma_tiles(c.tmem + TM_G, aT2, 128, aW2, 64, 64, 128, false);   // sbar
        mma_tiles(c.tmem + TM_GP, aT3, 128, aW2, 64, 64, 128, false);  // sdotbar
        tc::commit(c.mbar);
      }
      c.wait_mma();
      {
        float z[FPT], zp[FPT], sb[FPT], sdb[FPT];
        c.ld(TM_Z, z);
        c.ld(TM_ZP, zp);
        c.ld(TM_G, sb);
        c.ld(TM_GP, sdb);
#pragma unroll
        for (int j = 0; j < FPT; ++j) {
          const float zz = z[j] + al[f0 + j];
          const float ds = dev::dsilu(zz);
          z[j] = sb[j] * ds + sdb[j] * dev::d2silu(zz) * zp[j];  // zbar
          zp[j] = sdb[j] * ds;                                   // zbar'
          cs_a[j] += z[j];
        }
        st_fm(T2, c.e, f0, z);
        st_fm(T3, c.e, f0, zp);
        float ph[FPT], dph[FPT];
        basis(sc.d[c.e], rc, f0, ph, dph);
        st_fm(T0, c.e, f0, ph);   // phi^T
        st_fm(T1, c.e, f0, dph);  // phi'^T
      }
      c.publish();
      if (threadIdx.x == 0) {  // dA += phi^T zbar + phi'^T zbar'
        mma_tiles(c.tmem + TM_AG, aT0, 64, aT2, 64, 128, 64, !first);
        mma_tiles(c.tmem + TM_AG, aT1, 64, aT3, 64, 128, 64, true);
        tc::commit(c.mbar);
      }
      c.wait_mma();
      first = false;
      __syncthreads();
    }
    float* const outs[2] = {mdot_out, X_out};
    seg_write<2>(tr.r0, tr.r1, outs, acc);
    if (inj) rows_times_wt(tr.r0, tr.r1, acc[1], reinterpret_cast<float*>(T1), Wt, nullptr, nullptr, inj);  // hbar^F = X W^T
  }
  float* part = partial + (size_t)blockIdx.x * PE;
  if (first) {
    for (int x = threadIdx.x; x < PE; x += NT) part[x] = 0.f;
    teardown(c, 512);
    return;
  }
  write_partial(c, part, T0, cs_a, cs_b);
  teardown(c, 512);
}

constexpr size_t kSmallBytes = sizeof(float) * (128 + 10 * TE);
constexpr size_t fe_smem() { return 2 * kWTile + 2 * kTile + kSmallBytes; }
constexpr size_t ff_smem() { return 2 * kWTile + 2 * kTile + kSmallBytes; }
constexpr size_t be_smem() { return 3 * kWTile + 4 * kTile + kSmallBytes; }
constexpr size_t bf_smem() { return 3 * kWTile + 4 * kTile + kSmallBytes; }

}  // namespace edge_tc
}  // namespace janus
