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

#include <cuda_bf16.h>

#include "common.cuh"
#include "edge_kernels.cuh"
#include "tc.cuh"

namespace janus {
namespace edge_tc {

constexpr int TE = 128;
#ifndef JANUS_TC_NT
#define JANUS_TC_NT 512
#endif
constexpr int NT = JANUS_TC_NT;
#ifndef JANUS_FEFF_CTAS
#define JANUS_FEFF_CTAS 2  // FE / FF CTAs per SM (64 registers per thread at 2)
#endif    // 512: 16 warps, 4 threads per edge row (1024: 8 per row)
constexpr int NQ = NT / TE;        // feature quarters per edge
constexpr int FPT = 64 / NQ;       // features per thread (16)
constexpr int H = 64, R = 64;
constexpr int kRowsPerTile = 8;
constexpr uint32_t kTile = 128 * 64 * 4;  // 32 KB operand tile
constexpr uint32_t kWTile = 64 * 64 * 4;  // 16 KB weight tile
constexpr int PE = R * H + H + H * H + H;
static_assert(PE == 4 * 2080, "write_partial copy-out assumes H = R = 64");

// Phase tracing (profiling builds only: make TRACE=1): thread 0 of CTAs 0 and
// gridDim/2 prints clock64 deltas between the marks of one kernel.
#ifdef JANUS_TC_TRACE
#define TC_DECL long long trc[32] = {}; int ntr = 0
#define TC_M()                                                   \
  do {                                                           \
    if (threadIdx.x == 0 && ntr < 32) trc[ntr] = clock64();      \
    ++ntr;                                                       \
  } while (0)
#define TC_DUMP(name)                                                                                          \
  if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x / 2)) {                                   \
    long long d[30] = {};                                                                                      \
    for (int k = 1; k < ntr && k < 31; ++k) d[k - 1] = trc[k] - trc[k - 1];                                    \
    printf("TRACE %s cta %d marks %d total %lld: %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld\n", \
           name, blockIdx.x, ntr, trc[min(ntr, 32) - 1] - trc[0], d[0], d[1], d[2], d[3], d[4], d[5], d[6], d[7], d[8], \
           d[9], d[10], d[11], d[12], d[13], d[14]);                                                           \
    printf("TRACE+ %s cta %d: %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld\n", name, blockIdx.x, \
           d[15], d[16], d[17], d[18], d[19], d[20], d[21], d[22], d[23], d[24], d[25], d[26], d[27], d[28], d[29]); \
  }
#define TC_ARGS , long long *trc, int &ntr
#define TC_GT(v) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v))
#define TC_SPAN_BEGIN unsigned long long gt0 = 0; if (threadIdx.x == 0) TC_GT(gt0)
#define TC_SPAN_END(name)                                                                          \
  if (threadIdx.x == 0) {                                                                          \
    unsigned long long gt1; TC_GT(gt1); unsigned smid; asm volatile("mov.u32 %0, %%smid;" : "=r"(smid)); \
    printf("SPAN %s cta %d sm %u t0 %llu t1 %llu\n", name, blockIdx.x, smid, gt0, gt1);              \
  }
#define TC_PASS , trc, ntr
#else
#define TC_ARGS
#define TC_PASS
#define TC_SPAN_BEGIN
#define TC_SPAN_END(name)
#define TC_DECL
#define TC_M()
#define TC_DUMP(name)
#endif
// TMEM columns
constexpr uint32_t TM_Z = 0, TM_ZP = 64, TM_G = 128, TM_GP = 192, TM_AG = 256, TM_BG = 320;

__device__ __forceinline__ uint32_t off_em(int e, int f) { return tc::sw128_off(e, f, 128); }  // [128 edges][64 feat]
__device__ __forceinline__ uint32_t off_fm(int f, int e) { return tc::sw128_off(f, e, 64); }   // [64 feat][128 edges]

// D[tmem] (+)= A(rows A_ROWS, K) . B(rows B_ROWS, K)^T, K-major SWIZZLE_128B
// tiles.  Fully unrolled: the base descriptors are built once and each K-step
// of 8 adds a compile-time offset to the 14-bit start-address field (32 B
// inside a 128 B slab row, A_ROWS * 128 B between slabs), so the issuing
// thread emits the UTCHMMAs back to back.
template <int A_ROWS, int B_ROWS, int K, int M>
__device__ __forceinline__ void mma_tiles(uint32_t d, uint32_t a, uint32_t b, bool accumulate) {
  constexpr uint32_t id = tc::idesc_tf32(M, 64, false, false);
  const uint64_t da0 = tc::smem_desc(a, 16, 1024, 2), db0 = tc::smem_desc(b, 16, 1024, 2);
#pragma unroll
  for (int s = 0; s < K / 8; ++s) {
    const uint64_t oa = static_cast<uint64_t>(((s >> 2) * A_ROWS * 128 + 32 * (s & 3)) >> 4);
    const uint64_t ob = static_cast<uint64_t>(((s >> 2) * B_ROWS * 128 + 32 * (s & 3)) >> 4);
    tc::mma_tf32(d, da0 + oa, db0 + ob, id, (s > 0 || accumulate) ? 1u : 0u);
  }
}

// SWIZZLE_128B tiles need a 1024 B-aligned base; a second co-resident CTA's
// dynamic window is not guaranteed to start on one (smem sizes carry +1 KB).
__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  const uint32_t a = tc::smem_u32(p);
  return p + ((1024u - (a & 1023u)) & 1023u);
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
  __device__ void ld(uint32_t col, float (&v)[FPT]) const { tc::ldv(tmem + lane_base() + col + static_cast<uint32_t>(FPT * q), v); }
  // two accumulators, both loads in flight before one wait
  __device__ void ld2(uint32_t ca, uint32_t cb, float (&a)[FPT], float (&b)[FPT]) const {
    const uint32_t base = tmem + lane_base() + static_cast<uint32_t>(FPT * q);
    tc::ldv2(base + ca, base + cb, a, b);
  }
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
// [W0 = A^T | W1 = B^T | W2 = B | alpha | beta | W^T (plain row-major, for
// the fused row epilogue)]; rebuilt after every optimizer step (stage.cu
// refresh_transposes) and pulled by each CTA with TMA bulk copies.
constexpr uint32_t kWtOff = 3 * kWTile + 2 * 64 * 4;
// + B as a bf16 K-major SWIZZLE_128B tile (n = out, k = in; 8 KB): the B operand
// of BF / BE's sbar = mu B^T MMAs, which feed only the parameter gradients
constexpr uint32_t kW2bOff = kWtOff + kWTile;
constexpr uint32_t kW2bBytes = 64 * 64 * 2;
// + A^T and B^T as bf16 K-major tiles (8 KB each): BF and BE compute only
// parameter gradients, so all their per-edge contractions run on bf16
constexpr uint32_t kW0bOff = kW2bOff + kW2bBytes;
constexpr uint32_t kW1bOff = kW0bOff + kW2bBytes;
constexpr uint32_t kPackBytes = kW1bOff + kW2bBytes;

__global__ void pack_msg_weights(const float* __restrict__ A, const float* __restrict__ alpha, const float* __restrict__ B,
                                 const float* __restrict__ beta, const float* __restrict__ W, float* __restrict__ pack) {
  JANUS_GDC_WAIT();
  uint8_t* dst = reinterpret_cast<uint8_t*>(pack);
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x < 64 * 64) {
    const int a = x / 64, b = x % 64;  // src[a*64 + b]
    *reinterpret_cast<float*>(dst + tc::sw128_off(b, a, 64)) = A[x];               // A^T: (n=h=b, k=r=a)
    *reinterpret_cast<float*>(dst + kWTile + tc::sw128_off(b, a, 64)) = B[x];      // B^T: (n=out=b, k=in=a)
    *reinterpret_cast<float*>(dst + 2 * kWTile + tc::sw128_off(a, b, 64)) = B[x];  // B:   (n=a, k=b)
    pack[kWtOff / 4 + b * 64 + a] = W[x];                                           // W^T[b][a] = W[a][b]
    *reinterpret_cast<__nv_bfloat16*>(dst + kW2bOff + tc::sw128_off_b16(a, b, 64)) = __float2bfloat16_rn(B[x]);  // B bf16: (n=a, k=b)
    *reinterpret_cast<__nv_bfloat16*>(dst + kW0bOff + tc::sw128_off_b16(b, a, 64)) = __float2bfloat16_rn(A[x]);  // A^T bf16
    *reinterpret_cast<__nv_bfloat16*>(dst + kW1bOff + tc::sw128_off_b16(b, a, 64)) = __float2bfloat16_rn(B[x]);  // B^T bf16
  }
  if (x < 64) {
    pack[3 * kWTile / 4 + x] = alpha[x];
    pack[3 * kWTile / 4 + 64 + x] = beta[x];
  }
}

// BF / BE: the three bf16 weight tiles [A^T | B^T | B] (contiguous in the
// pack, 24 KB) + alpha, beta with one TMA bulk copy each.
__device__ __forceinline__ void load_weights_b16(uint8_t* w0b, const float* pack, float* al, float* be, uint64_t* wbar) {
  if (threadIdx.x == 0) {
    tc::mbar_init(wbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint8_t* src = reinterpret_cast<const uint8_t*>(pack);
    tc::mbar_expect_tx(wbar, 3 * kW2bBytes + 512);
    tc::bulk_g2s(w0b, src + kW2bOff, 3 * kW2bBytes, wbar);  // order in the pack: B, A^T, B^T
    tc::bulk_g2s(al, src + 3 * kWTile, 256, wbar);
    tc::bulk_g2s(be, src + 3 * kWTile + 256, 256, wbar);
  }
  __syncthreads();
}

// Thread 0 arms `wbar` and bulk-loads `ntiles` weight tiles (+ alpha, beta,
// and W^T when wts != nullptr); ends with a CTA barrier so every thread may
// wait on `wbar` (tc::mbar_wait(wbar, 0)) — done just before the first MMA so
// the copy overlaps the TMEM allocation and the first chunk's basis.
__device__ __forceinline__ void load_weights(uint8_t* sm, const float* pack, int ntiles, float* al, float* be, float* wts,
                                             uint64_t* wbar, uint8_t* w2b = nullptr) {
  if (threadIdx.x == 0) {
    tc::mbar_init(wbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint32_t wbytes = static_cast<uint32_t>(ntiles) * kWTile;
    const uint8_t* src = reinterpret_cast<const uint8_t*>(pack);
    tc::mbar_expect_tx(wbar, wbytes + 512 + (wts ? kWTile : 0u) + (w2b ? kW2bBytes : 0u));
    tc::bulk_g2s(sm, pack, wbytes, wbar);
    tc::bulk_g2s(al, src + 3 * kWTile, 256, wbar);
    tc::bulk_g2s(be, src + 3 * kWTile + 256, 256, wbar);
    if (wts) tc::bulk_g2s(wts, src + kWtOff, kWTile, wbar);
    if (w2b) tc::bulk_g2s(w2b, src + kW2bOff, kW2bBytes, wbar);
  }
  __syncthreads();
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

struct TileRange {
  int r0, r1, e0, e1;
};
__device__ __forceinline__ TileRange tile_range(const int4* __restrict__ tiles, int t) {
  const int4 v = __ldg(tiles + t);
  return TileRange{v.x, v.y, v.z, v.w};
}

// Deterministic segmented row sums of NA plain tiles over one chunk.  The
// tile's nr rows x 64 features are spread over the CTA with `split` threads
// per (row, feature) pair (split = 8 / nr rounded down to a power of two):
// consecutive lanes share a pair and take interleaved edges of the row, so
// each partial is a short dependent chain; the partials stay per-thread across
// the tile's chunks and are combined once by an xor butterfly (seg_finish),
// which leaves the bit-identical total in every lane of the group.
struct SegMap {
  int split, span, pair, part;
  int rb, re;  // this pair's row: CSR edge range (loaded once per tile, off the chunk's critical path)
  bool active;
};
__device__ __forceinline__ SegMap seg_map(const EdgeGeom& g, const TileRange& tr) {
  SegMap m;
  const int nr = tr.r1 - tr.r0;
  constexpr int S1 = NT / 64;  // threads per (row, feature) pair for a one-row tile
  m.split = nr <= 1 ? S1 : nr <= 2 ? S1 / 2 : nr <= 4 ? S1 / 4 : S1 / 8;
  m.span = nr * 64;
  m.part = static_cast<int>(threadIdx.x) & (m.split - 1);
  m.pair = static_cast<int>(threadIdx.x) / m.split;
  m.active = m.pair < m.span;
  const int r = tr.r0 + (m.active ? (m.pair >> 6) : 0);
  m.rb = __ldg(g.row_ptr + r);
  m.re = __ldg(g.row_ptr + r + 1);
  return m;
}

template <int NA>
__device__ __forceinline__ void seg_rows(const EdgeGeom& g, int r0, int c0, int ne, const uint8_t* const (&tiles)[NA],
                                         const SegMap& m, float (&acc)[NA]) {
  if (!m.active) return;
  const int f = m.pair & 63;
  const int eb = max(m.rb, c0), ee = min(m.re, c0 + ne);
  for (int x = eb + m.part; x < ee; x += m.split) {
    const uint32_t o = off_pl(x - c0, f);
#pragma unroll
    for (int a = 0; a < NA; ++a) acc[a] += *reinterpret_cast<const float*>(tiles[a] + o);
  }
}

// all threads (warp-uniform split): combine the interleaved partials
template <int NA>
__device__ __forceinline__ void seg_finish(const SegMap& m, float (&acc)[NA]) {
  for (int o = 1; o < m.split; o <<= 1)
#pragma unroll
    for (int a = 0; a < NA; ++a) acc[a] += __shfl_xor_sync(0xffffffffu, acc[a], o);
}

template <int NA>
__device__ __forceinline__ void seg_write(int r0, const SegMap& m, float* const (&out)[NA], const float (&acc)[NA]) {
  if (!m.active || m.part != 0) return;
  const int r = r0 + (m.pair >> 6), f = m.pair & 63;
#pragma unroll
  for (int a = 0; a < NA; ++a) out[a][(size_t)r * H + f] = acc[a];
}

// Row epilogue fused into the edge kernels: the tile's finished rows R (from
// the segmented sums) times W^T:  out[r] = (base ? base[r] : 0) + R[r] W^T
// (+ add[r]).  Rows staged in smem (rs[8][64]); W^T ([64][64] row-major) was
// bulk-loaded into smem with the weight image.
__device__ __forceinline__ void rows_times_wt(int r0, int r1, const SegMap& m, float accv, float* rs,
                                              const float* Wts, const float* base, const float* __restrict__ add,
                                              float* out) {
  if (m.active && m.part == 0) rs[m.pair] = accv;
  __syncthreads();
  const int pidx = threadIdx.x;
  const int rl = pidx >> 6, c = pidx & 63, r = r0 + rl;
  if (r < r1) {
    float o[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int q = 0; q < 64; q += 4) {
      const float4 x = *reinterpret_cast<const float4*>(rs + rl * 64 + q);
      o[0] = fmaf(x.x, Wts[q * 64 + c], o[0]);
      o[1] = fmaf(x.y, Wts[(q + 1) * 64 + c], o[1]);
      o[2] = fmaf(x.z, Wts[(q + 2) * 64 + c], o[2]);
      o[3] = fmaf(x.w, Wts[(q + 3) * 64 + c], o[3]);
    }
    float y = (o[0] + o[1]) + (o[2] + o[3]);
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
    p[j] = __expf(-gamma * x * x);
    dp[j] = -2.0f * gamma * x * p[j];
  }
}

// The same basis with 3 exponentials instead of FPT: in units of delta,
// x_j = d / delta - (f0 + j) and phi_j = exp(-x_j^2 / 2), so neighbouring
// features differ by the factor phi_{j+1} / phi_j = exp(x_j - 1/2) (and
// phi_{j-1} / phi_j = exp(-x_j - 1/2)), which itself shrinks by e^-1 per
// step.  Starting at the feature nearest the peak every factor is <= 1, so
// the recurrence never overflows and underflows only where the basis is ~0.
// Error: ~FPT^2/2 ulp relative (< 1e-5), far below the bf16 / tf32 operand
// rounding these values get.  (ncu: the per-element __expf of basis() were
// ~10% of the pair kernels' stall samples, all on the MUFU pipe.)
__device__ __forceinline__ void basis_fast(float d, float rc, int f0, float (&p)[FPT], float (&dp)[FPT]) {
  const float delta = rc / (R - 1);
  const float gamma = 1.0f / (2.0f * delta * delta);
  const float u = d / delta - static_cast<float>(f0);
  const int js = min(max(__float2int_rn(u), 0), FPT - 1);
  const float xs = u - static_cast<float>(js);
  const float ps = __expf(-0.5f * xs * xs);
  float up = __expf(xs - 0.5f), dn = __expf(-xs - 0.5f);
  constexpr float kE1 = 0.36787944117144233f;  // e^-1
#pragma unroll
  for (int j = 0; j < FPT; ++j) {
    if (j == js) p[j] = ps;
    if (j > js) {
      p[j] = p[j - 1] * up;
      up *= kE1;
    }
  }
#pragma unroll
  for (int j = FPT - 2; j >= 0; --j)
    if (j < js) {
      p[j] = p[j + 1] * dn;
      dn *= kE1;
    }
#pragma unroll
  for (int j = 0; j < FPT; ++j) dp[j] = -2.0f * gamma * (d - (f0 + j) * delta) * p[j];
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

// This thread's edge scalars (the 4 threads of an edge read the same values
// through L1; padding edges get c = dc = 0, which zeroes all their terms).
struct ES {
  float d, c, dc;
  int i, j, x;
  bool ok;
};
__device__ __forceinline__ ES edge_sc(const EdgeGeom& g, int c0, int ne, int e) {
  ES s;
  s.ok = e < ne;
  s.x = c0 + (s.ok ? e : 0);
  s.d = s.ok ? __ldg(g.d + s.x) : 0.f;
  s.c = s.ok ? __ldg(g.c + s.x) : 0.f;
  s.dc = s.ok ? __ldg(g.dc + s.x) : 0.f;
  s.i = s.ok ? __ldg(g.src + s.x) : 0;
  s.j = s.ok ? __ldg(g.col + s.x) : 0;
  return s;
}
// qbar_e = < Fbar_i - Fbar_j, u_e >
__device__ __forceinline__ float edge_qbar(const EdgeGeom& g, const ES& s, const float* __restrict__ Fbar) {
  float q = 0.f;
  if (s.ok)
#pragma unroll
    for (int k = 0; k < 3; ++k) q = fmaf(__ldg(Fbar + 3 * s.i + k) - __ldg(Fbar + 3 * s.j + k), __ldg(g.u + 3 * s.x + k), q);
  return q;
}

// fast sigmoid for the tf32 path; SiLU and its derivatives derive from one s
__device__ __forceinline__ float fsig(float x) { return __fdividef(1.0f, 1.0f + __expf(-x)); }
// one-MUFU sigmoid for the gradient-only BF / BE pair kernels, whose results
// become bf16 operands: sigma(x) = (1 + tanh(x / 2)) / 2 with tanh.approx
// (abs error ~2^-12 in sigma, below bf16's 2^-9 relative rounding) instead of
// ex2 + rcp — the pair kernels' epilogues were MUFU-throttled (ncu: mio stalls).
__device__ __forceinline__ float fsig_t(float x) {
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(0.5f * x));
  return fmaf(0.5f, t, 0.5f);
}

// ----------------------------------------------------------------------- FE
// m_i = sum_{e in row i} w_e * v[col e], w = c (SiLU(phi A + alpha) B + beta)
__global__ void __launch_bounds__(NT, JANUS_FEFF_CTAS) msg_fe_tc(EdgeGeom g, const int4* __restrict__ tiles, int n_tiles, MsgParams p,
                                               float rc, const float* __restrict__ v, float* __restrict__ m_out) {
  JANUS_GDC_WAIT();
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = align1024(sm_raw);
  TC_DECL;
  TC_SPAN_BEGIN;
  TC_M();
  uint8_t* W0 = sm;               // A^T  (n = h, k = r)
  uint8_t* W1 = W0 + kWTile;      // B^T  (n = out, k = in)
  uint8_t* T0 = W1 + kWTile;      // phi -> s
  uint8_t* T1 = T0 + kTile;       // w (edge-major)
  float* al = reinterpret_cast<float*>(T1 + kTile);
  float* be = al + 64;
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tslot;
  Ctx c;
  c.sm = sm;
  c.mbar = &mbar;
  __shared__ __align__(8) uint64_t wbar;
  load_weights(sm, p.pack, 2, al, be, nullptr, &wbar);
  TC_M();
  setup(c, &tslot, 128);
  TC_M();
  const uint32_t aW0 = tc::smem_u32(W0), aW1 = tc::smem_u32(W1), aT0 = tc::smem_u32(T0);
  const int f0 = FPT * c.q;
  for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const TileRange tr = tile_range(tiles, t);
    const SegMap sg = seg_map(g, tr);
    float acc[1] = {};
    for (int c0 = tr.e0; c0 < tr.e1; c0 += TE) {
      const int ne = min(TE, tr.e1 - c0);
      const ES es = edge_sc(g, c0, ne, c.e);
#ifdef JANUS_TC_TRACE
      {
        float dmy;
        asm volatile("mov.b32 %0, %1;" : "=f"(dmy) : "f"(es.d));
        TC_M();
      }
#endif
      {
        float ph[FPT], dph[FPT];
        basis(es.d, rc, f0, ph, dph);
        st_em(T0, c.e, f0, ph);
      }
      tc::mbar_wait(&wbar, 0);  // weights landed (immediate after the first chunk)
      c.publish();
      if (threadIdx.x == 0) {
        mma_tiles<128, 64, 64, 128>(c.tmem + TM_Z, aT0, aW0, false);
        tc::commit(c.mbar);
      }
      TC_M();
      c.wait_mma();
      TC_M();
      {
        float z[FPT];
        c.ld(TM_Z, z);
#pragma unroll
        for (int j = 0; j < FPT; ++j) {
          const float zz = z[j] + al[f0 + j];
          z[j] = zz * fsig(zz);
        }
        st_em(T0, c.e, f0, z);
      }
      c.publish();
      if (threadIdx.x == 0) {
        mma_tiles<128, 64, 64, 128>(c.tmem + TM_ZP, aT0, aW1, false);
        tc::commit(c.mbar);
      }
      TC_M();
      c.wait_mma();
      TC_M();
      {
        float gg[FPT], vj[FPT];
        gather32(v, es.j, f0, vj);
        c.ld(TM_ZP, gg);
#pragma unroll
        for (int j = 0; j < FPT; ++j) gg[j] = es.c * (gg[j] + be[f0 + j]) * vj[j];  // w_e * v_j
        st_pl(T1, c.e, f0, gg);
      }
      tc::fence_before();
      __syncthreads();
      {
        const uint8_t* const tl[1] = {T1};
        TC_M();
        seg_rows<1>(g, tr.r0, c0, ne, tl, sg, acc);
      }
      TC_M();
      __syncthreads();
    }
    seg_finish<1>(sg, acc);
    float* const outs[1] = {m_out};
    seg_write<1>(tr.r0, sg, outs, acc);
  }
  TC_M();
  teardown(c, 128);
  TC_M();
  TC_SPAN_END("fe");
  TC_DUMP("fe");
}

// ----------------------------------------------------------------------- FF
// Y_i = sum w_e * am[col e];  F_i += sum_e (q_e + q_rev(e)) u_e with
// q_e + q_rev(e) = < am_i v_j + am_j v_i , w'_e >  (w' symmetric in e <-> rev e)
__global__ void __launch_bounds__(NT, JANUS_FEFF_CTAS) msg_ff_tc(EdgeGeom g, const int4* __restrict__ tiles, int n_tiles, MsgParams p,
                                               float rc, const float* __restrict__ v, const float* __restrict__ am,
                                               float* __restrict__ Y_out, float* __restrict__ F,
                                               float* ah) {
  JANUS_GDC_WAIT();
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = align1024(sm_raw);
  uint8_t* W0 = sm;
  uint8_t* W1 = W0 + kWTile;
  uint8_t* T0 = W1 + kWTile;  // phi -> s -> (plain) w * am_j
  uint8_t* T1 = T0 + kTile;   // phi' -> sdot
  float* al = reinterpret_cast<float*>(T1 + kTile);
  float* be = al + 64;
  // W^T for the fused row epilogue is read through L1 from the packed image in
  // global memory (not staged): without its 16 KB two FF CTAs fit an SM
  const float* wts = p.pack + kWtOff / sizeof(float);
  float* sq = be + 64;  // [NQ][TE] per-quarter force scalars
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tslot;
  Ctx c;
  c.sm = sm;
  c.mbar = &mbar;
  __shared__ __align__(8) uint64_t wbar;
  load_weights(sm, p.pack, 2, al, be, nullptr, &wbar);
  setup(c, &tslot, 256);
  const uint32_t aW0 = tc::smem_u32(W0), aW1 = tc::smem_u32(W1), aT0 = tc::smem_u32(T0), aT1 = tc::smem_u32(T1);
  const int f0 = FPT * c.q;
  // force sums: 8 lanes per (row, component), interleaved edges
  const int fr = threadIdx.x >> 3, fpart = threadIdx.x & 7;
  for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const TileRange tr = tile_range(tiles, t);
    const SegMap sg = seg_map(g, tr);
    float acc[1] = {};
    float fsum = 0.f;
    const bool frow = fr < 3 * (tr.r1 - tr.r0);
    const int fb = frow ? __ldg(g.row_ptr + tr.r0 + fr / 3) : 0, fe = frow ? __ldg(g.row_ptr + tr.r0 + fr / 3 + 1) : 0;
    for (int c0 = tr.e0; c0 < tr.e1; c0 += TE) {
      const int ne = min(TE, tr.e1 - c0);
      const ES es = edge_sc(g, c0, ne, c.e);
      {
        float ph[FPT], dph[FPT];
        basis(es.d, rc, f0, ph, dph);
        st_em(T0, c.e, f0, ph);
        st_em(T1, c.e, f0, dph);
      }
      tc::mbar_wait(&wbar, 0);  // weights landed (immediate after the first chunk)
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
        float pq = 0.f;
        float amj[FPT], vj[FPT], ami[FPT], vi[FPT];
        gather32(am, es.j, f0, amj);
        gather32(v, es.j, f0, vj);
        gather32(am, es.i, f0, ami);
        gather32(v, es.i, f0, vi);
        c.ld2(TM_G, TM_GP, gg, gp);
#pragma unroll
        for (int q = 0; q < FPT; ++q) {
          const float gb = gg[q] + be[f0 + q];
          const float wp = es.dc * gb + es.c * gp[q];
          pq = fmaf(fmaf(ami[q], vj[q], amj[q] * vi[q]), wp, pq);
          gg[q] = es.c * gb * amj[q];  // w_e * am_j
        }
        st_pl(T0, c.e, f0, gg);
        sq[c.q * TE + c.e] = pq;
      }
      tc::fence_before();
      __syncthreads();
      {
        const uint8_t* const tl[1] = {T0};
        seg_rows<1>(g, tr.r0, c0, ne, tl, sg, acc);
        if (frow) {
          const int comp = fr % 3;
          const int eb = max(fb, c0), ee = min(fe, c0 + ne);
          for (int x = eb + fpart; x < ee; x += 8)
          {
            float qs = 0.f;
#pragma unroll
            for (int k = 0; k < NQ; ++k) qs += sq[k * TE + x - c0];
            fsum = fmaf(qs, g.u[3 * x + comp], fsum);
          }
        }
      }
      __syncthreads();
    }
    seg_finish<1>(sg, acc);
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) fsum += __shfl_xor_sync(0xffffffffu, fsum, o);
    float* const outs[1] = {Y_out};
    seg_write<1>(tr.r0, sg, outs, acc);
    if (fpart == 0 && frow) F[3 * tr.r0 + fr] += fsum;
    if (ah) rows_times_wt(tr.r0, tr.r1, sg, acc[0], reinterpret_cast<float*>(T1), wts, ah, nullptr, ah);  // a_h += Y W^T
  }
  teardown(c, 256);
}

// Weight-gradient operands in bf16 (kind::f16): an edge-major [128 edges][64
// features] bf16 tile (one 128 B SWIZZLE_128B row per edge, 16 KB) is an
// MN-major operand of sum_e X_e^T Y_e (M|N = features, K = edges), so no
// transposed copy is written (tcgen05 MN-major returns zeros for kind::tf32,
// tests/test_gpu_tc.py).  Per-edge contractions stay tf32.
constexpr uint32_t kBTile = 128 * 64 * 2;
__device__ __forceinline__ uint32_t off_b16(int e, int f) { return tc::sw128_off_b16(e, f, 128); }
__device__ __forceinline__ void st_b16(uint8_t* t, int e, int f0, const float (&v)[FPT]) {
#pragma unroll
  for (int j = 0; j < FPT / 8; ++j) {
    const __nv_bfloat162 a = __floats2bfloat162_rn(v[8 * j], v[8 * j + 1]), b = __floats2bfloat162_rn(v[8 * j + 2], v[8 * j + 3]);
    const __nv_bfloat162 c = __floats2bfloat162_rn(v[8 * j + 4], v[8 * j + 5]), d = __floats2bfloat162_rn(v[8 * j + 6], v[8 * j + 7]);
    uint4 w;
    w.x = *reinterpret_cast<const uint32_t*>(&a);
    w.y = *reinterpret_cast<const uint32_t*>(&b);
    w.z = *reinterpret_cast<const uint32_t*>(&c);
    w.w = *reinterpret_cast<const uint32_t*>(&d);
    *reinterpret_cast<uint4*>(t + off_b16(e, f0 + 8 * j)) = w;
  }
}
// D[64][64] (+)= sum_e A[e][m] B[e][n] over the 128 edges of two bf16 tiles
// (MN-major SWIZZLE_128B: K-step of 16 edges = 2048 B; one 64-wide MN slab).
__device__ __forceinline__ void mma_wg_b16(uint32_t d, uint32_t a, uint32_t b, bool accumulate) {
  constexpr uint32_t id = tc::idesc_bf16(64, 64, true, true);
  const uint64_t da0 = tc::smem_desc(a, kBTile, 1024, 2), db0 = tc::smem_desc(b, kBTile, 1024, 2);
#pragma unroll
  for (int s = 0; s < TE / 16; ++s) {
    const uint64_t o = static_cast<uint64_t>((2048 * s) >> 4);
    tc::mma_bf16(d, da0 + o, db0 + o, id, (s > 0 || accumulate) ? 1u : 0u);
  }
}
// D[128 edges][64] = A[128][64] . B[64][64]^T on bf16 K-major SWIZZLE_128B
// tiles (one 128 B row per edge / output; K-step of 16 = +32 B in the row).
__device__ __forceinline__ void mma_kb16(uint32_t d, uint32_t a, uint32_t b) {
  constexpr uint32_t id = tc::idesc_bf16(128, 64, false, false);
  const uint64_t da0 = tc::smem_desc(a, 16, 1024, 2), db0 = tc::smem_desc(b, 16, 1024, 2);
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const uint64_t o = static_cast<uint64_t>((32 * s) >> 4);
    tc::mma_bf16(d, da0 + o, db0 + o, id, s > 0 ? 1u : 0u);
  }
}
// Column sums of an edge-major bf16 tile (same mapping as em_colsum_add; the
// four features of a warp share a 16 B chunk, so the loads broadcast).
__device__ __forceinline__ void b16_colsum_add(const uint8_t* t, float* acc) {
  if (threadIdx.x < 512) {
    const int f = static_cast<int>(threadIdx.x) >> 3, p = static_cast<int>(threadIdx.x) & 7;
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < TE / 8; ++k) s += __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(t + off_b16(p + 8 * k, f)));
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    if (p == 0) acc[f] += s;
  }
}
// Column sums (over the chunk's edges) of an edge-major fp32 SWIZZLE_128B tile
// [128 edges][64 features], added to acc[64] (shared memory): 8 threads per
// feature take edges p, p+8, ... (conflict-free scalar loads), an xor
// butterfly combines them, one thread adds — a fixed order, deterministic.
__device__ __forceinline__ void em_colsum_add(const uint8_t* t, float* acc) {
  if (threadIdx.x < 512) {
    const int f = static_cast<int>(threadIdx.x) >> 3, p = static_cast<int>(threadIdx.x) & 7;
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < TE / 8; ++k) s += *reinterpret_cast<const float*>(t + off_em(p + 8 * k, f));
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    if (p == 0) acc[f] += s;
  }
}

// Column sums (over the chunk's edges) of a feature-major SWIZZLE_128B tile
// [64 features][128 edges], added to the CTA accumulator acc[64] in shared
// memory: 8 threads per feature read 16 edges each (4 conflict-free LDS.128),
// an xor butterfly combines them and one thread adds — a fixed order per
// feature, so the sums are deterministic.  Runs while the tensor core reads
// the same tile (both are reads).  Padding edges hold zeros.
__device__ __forceinline__ void fm_colsum_add(const uint8_t* t, float* acc) {
  if (threadIdx.x < 512) {
    const int f = static_cast<int>(threadIdx.x) >> 3, p = static_cast<int>(threadIdx.x) & 7;
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float4 v = *reinterpret_cast<const float4*>(t + off_fm(f, 16 * p + 4 * k));
      s += (v.x + v.y) + (v.z + v.w);
    }
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    if (p == 0) acc[f] += s;
  }
}

// Write the CTA's weight-gradient partial [dA | dalpha | dB | dbeta] from the
// M=64 TMEM accumulators (row r at lane (r/16)*32 + r%16) and the per-thread
// column sums.  Everything is staged in smem (`scratch` = the four operand
// tiles, free by now) and leaves with coalesced float4 stores.
// Write the CTA's weight-gradient partial [dA | dalpha | dB | dbeta] from the
// M=64 TMEM accumulators (row r at lane (r/16)*32 + r%16) and the CTA's
// column-sum accumulators csa/csb (shared memory).  The rows are staged in
// smem (`scratch` = the operand tiles, free by now) and leave with coalesced
// float4 stores.
__device__ __forceinline__ void write_partial(Ctx& c, float* part, uint8_t* scratch, const float* csa,
                                              const float* csb, uint32_t tm_ag, uint32_t tm_bg TC_ARGS) {
  constexpr int LDP = 68;  // padded row: the 8 rows of an STS.128 phase hit distinct banks
  float* stg = reinterpret_cast<float*>(scratch);  // [2][64][LDP] dA, dB rows
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  TC_M();
  {
    float va[FPT], vb[FPT];
    c.ld2(tm_ag, tm_bg, va, vb);
    if (c.lane < 16) {
      const int r = 16 * (c.warp & 3) + c.lane;
      float4* pa = reinterpret_cast<float4*>(stg + r * LDP + FPT * c.q);
      float4* pb = reinterpret_cast<float4*>(stg + 64 * LDP + r * LDP + FPT * c.q);
#pragma unroll
      for (int j = 0; j < FPT / 4; ++j) {
        pa[j] = make_float4(va[4 * j], va[4 * j + 1], va[4 * j + 2], va[4 * j + 3]);
        pb[j] = make_float4(vb[4 * j], vb[4 * j + 1], vb[4 * j + 2], vb[4 * j + 3]);
      }
    }
  }
  __syncthreads();
  TC_M();
  // coalesced copy-out: PE / 4 = 2080 float4 in global order
  float4* out = reinterpret_cast<float4*>(part);
  for (int k = threadIdx.x; k < PE / 4; k += NT) {
    float4 v;
    if (k < 1024) {
      v = *reinterpret_cast<const float4*>(stg + (k >> 4) * LDP + 4 * (k & 15));
    } else if (k < 1040) {
      v = *reinterpret_cast<const float4*>(csa + 4 * (k - 1024));
    } else if (k < 2064) {
      const int kk = k - 1040;
      v = *reinterpret_cast<const float4*>(stg + 64 * LDP + (kk >> 4) * LDP + 4 * (kk & 15));
    } else {
      v = *reinterpret_cast<const float4*>(csb + 4 * (k - 2064));
    }
    out[k] = v;
  }
}

// ----------------------------------------------------------------------- BE
// Yb_i = sum w_e * bm[col e]; gbar = c bm_i v_j; dB = s^T gbar; dbeta = sum gbar;
// zbar = (gbar B^T) SiLU'(z); dA = phi^T zbar; dalpha = sum zbar.
// Per chunk: fp32 tiles T0 (phi -> s -> w bm_j rows -> zbar) and T1 (gbar,
// A of sbar); bf16 tiles B0..B3 = phi, s, gbar, zbar for the weight gradients.
__global__ void __launch_bounds__(NT, 1) msg_be_tc(EdgeGeom g, const int4* __restrict__ tiles, int n_tiles, MsgParams p,
                                                  float rc, const float* __restrict__ v, const float* __restrict__ bm,
                                                  float* __restrict__ Yb_out, float* __restrict__ partial,
                                                  const float* __restrict__ inj, float* bh) {
  JANUS_GDC_WAIT();
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = align1024(sm_raw);
  TC_DECL;
  TC_M();
  uint8_t* W2b = sm;                // bf16 weights in pack order: B | A^T | B^T
  uint8_t* W0b = W2b + kW2bBytes;
  uint8_t* W1b = W0b + kW2bBytes;
  uint8_t* T0 = sm + 2 * kWTile;    // 1024 B aligned after the 24 KB of weights
  uint8_t* T1 = T0 + kTile;   // write_partial / row-epilogue scratch
  uint8_t* B0 = T1 + kTile;   // bf16: phi
  uint8_t* B1 = B0 + kBTile;  //       s
  uint8_t* B2 = B1 + kBTile;  //       gbar
  uint8_t* B3 = B2 + kBTile;  //       zbar
  float* al = reinterpret_cast<float*>(B3 + kBTile);
  float* be = al + 64;
  float* csa = be + 64;  // CTA column sums: dalpha, dbeta
  float* csb = csa + 64;
  const float* wts = p.pack + kWtOff / sizeof(float);  // W^T (row epilogue) through L1
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tslot;
  Ctx c;
  c.sm = sm;
  c.mbar = &mbar;
  __shared__ __align__(8) uint64_t wbar;
  load_weights_b16(W2b, p.pack, al, be, &wbar);
  if (threadIdx.x < 128) csa[threadIdx.x] = 0.f;  // csa, csb (published by setup's barrier)
  TC_M();
  setup(c, &tslot, 512);
  TC_M();
  const uint32_t aW0b = tc::smem_u32(W0b), aW1b = tc::smem_u32(W1b), aW2b = tc::smem_u32(W2b);
  const uint32_t aB0 = tc::smem_u32(B0), aB1 = tc::smem_u32(B1), aB2 = tc::smem_u32(B2), aB3 = tc::smem_u32(B3);
  bool first = true;
  const int f0 = FPT * c.q;
  for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const TileRange tr = tile_range(tiles, t);
    const SegMap sg = seg_map(g, tr);
    float acc[1] = {};
    for (int c0 = tr.e0; c0 < tr.e1; c0 += TE) {
      const int ne = min(TE, tr.e1 - c0);
      const ES es = edge_sc(g, c0, ne, c.e);
      {
        float ph[FPT], dph[FPT];
        basis(es.d, rc, f0, ph, dph);
        st_b16(B0, c.e, f0, ph);  // phi (A of z = phi A and of dA)
      }
      tc::mbar_wait(&wbar, 0);  // weights landed (immediate after the first chunk)
      c.publish();
      if (threadIdx.x == 0) {
        mma_kb16(c.tmem + TM_Z, aB0, aW0b);
        tc::commit(c.mbar);
      }
      TC_M();
      c.wait_mma();
      TC_M();
      {
        float z[FPT];
        c.ld(TM_Z, z);
#pragma unroll
        for (int j = 0; j < FPT; ++j) {
          const float zz = z[j] + al[f0 + j];
          z[j] = zz * fsig(zz);
        }
        st_b16(B1, c.e, f0, z);  // s (A of g = s B and of dB = s^T gbar)
      }
      c.publish();
      if (threadIdx.x == 0) {
        mma_kb16(c.tmem + TM_G, aB1, aW1b);
        tc::commit(c.mbar);
      }
      TC_M();
      c.wait_mma();
      TC_M();
      {
        float gb[FPT];
        {
          float gg[FPT], bj[FPT], bi[FPT], vj[FPT];
          gather32(bm, es.j, f0, bj);
          gather32(bm, es.i, f0, bi);
          gather32(v, es.j, f0, vj);
          c.ld(TM_G, gg);
          TC_M();
#pragma unroll
          for (int q = 0; q < FPT; ++q) {
            gg[q] = es.c * (gg[q] + be[f0 + q]) * bj[q];  // w_e * bm_j
            gb[q] = es.c * bi[q] * vj[q];                 // gbar (zero on padding edges: c = 0)
          }
          TC_M();
          st_pl(T0, c.e, f0, gg);
        }
        st_b16(B2, c.e, f0, gb);  // gbar: B of dB, A of sbar = gbar B^T (bf16: feeds dA only)
      }
      TC_M();
      c.publish();
      TC_M();
      if (threadIdx.x == 0) {
        mma_wg_b16(c.tmem + TM_BG, aB1, aB2, !first);  // dB += s^T gbar
        mma_kb16(c.tmem + TM_G, aB2, aW2b);            // sbar
        tc::commit(c.mbar);
      }
      TC_M();
      {  // row sums and dbeta overlap the MMAs (reads of T0 / T1)
        const uint8_t* const tl[1] = {T0};
        seg_rows<1>(g, tr.r0, c0, ne, tl, sg, acc);
      }
      b16_colsum_add(B2, csb);  // dbeta += sum_e gbar_e
      TC_M();
      c.wait_mma();
      __syncthreads();  // T0 / T1 reads done before T0 is rewritten
      TC_M();
      {
        float z[FPT], sb[FPT];
        c.ld2(TM_Z, TM_G, z, sb);
#pragma unroll
        for (int j = 0; j < FPT; ++j) {
          const float zz = z[j] + al[f0 + j], s1 = fsig(zz);
          z[j] = sb[j] * (s1 * (1.0f + zz * (1.0f - s1)));
        }
        st_b16(B3, c.e, f0, z);  // zbar (B of dA; its column sums)
      }
      c.publish();
      if (threadIdx.x == 0) {
        mma_wg_b16(c.tmem + TM_AG, aB0, aB3, !first);  // dA += phi^T zbar
        tc::commit(c.mbar);
      }
      b16_colsum_add(B3, csa);  // dalpha += sum_e zbar_e (beside the dA MMA)
      TC_M();
      c.wait_mma();
      TC_M();
      first = false;
      __syncthreads();
    }
    seg_finish<1>(sg, acc);
    float* const outs[1] = {Yb_out};
    seg_write<1>(tr.r0, sg, outs, acc);
    TC_M();
    if (bh) rows_times_wt(tr.r0, tr.r1, sg, acc[0], reinterpret_cast<float*>(T1), wts, bh, inj, bh);  // b_h += Yb W^T + inj
    TC_M();
  }
  float* part = partial + (size_t)blockIdx.x * PE;
  if (first) {  // CTA without tiles: zero partial (TMEM accumulators never written)
    for (int x = threadIdx.x; x < PE; x += NT) part[x] = 0.f;
    teardown(c, 512);
    return;
  }
  write_partial(c, part, T0, csa, csb, TM_AG, TM_BG TC_PASS);
  TC_M();
  teardown(c, 512);
  TC_M();
  TC_DUMP("be");
}

// ----------------------------------------------------------------------- BF
// Second-order term.  Outputs: mdot_i = sum_e qb w'_e v_j + w_e vdot_j,
// X_i = sum_e qb w'_e am_j, and the partial [dA | dalpha | dB | dbeta].
// Per chunk: fp32 tiles T0/T1 (phi, phi' -> s, sdot -> row terms -> mu, nu;
// zbar for its column sums) and bf16 tiles B0..B5 = s, sdot, mu|zbar,
// nu|zbar', phi, phi' for the weight gradients (phi kept: no second basis).
__global__ void __launch_bounds__(NT, 1) msg_bf_tc(EdgeGeom g, const int4* __restrict__ tiles, int n_tiles, MsgParams p,
                                                  float rc, const float* __restrict__ v, const float* __restrict__ vdot,
                                                  const float* __restrict__ am, const float* __restrict__ Fbar,
                                                  float* __restrict__ mdot_out, float* __restrict__ X_out,
                                                  float* __restrict__ partial,
                                                  float* __restrict__ inj) {
  JANUS_GDC_WAIT();
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = align1024(sm_raw);
  TC_DECL;
  TC_SPAN_BEGIN;
  TC_M();
  uint8_t* W2b = sm;                // bf16 weights in pack order: B | A^T | B^T
  uint8_t* W0b = W2b + kW2bBytes;
  uint8_t* W1b = W0b + kW2bBytes;
  uint8_t* T0 = sm + 2 * kWTile;    // 1024 B aligned after the 24 KB of weights
  uint8_t* T1 = T0 + kTile;
  uint8_t* B0 = T1 + kTile;   // bf16: s
  uint8_t* B1 = B0 + kBTile;  //       sdot
  uint8_t* B2 = B1 + kBTile;  //       mu, then zbar
  uint8_t* B3 = B2 + kBTile;  //       nu, then zbar'
  uint8_t* B4 = B3 + kBTile;  //       phi
  uint8_t* B5 = B4 + kBTile;  //       phi'
  float* al = reinterpret_cast<float*>(B5 + kBTile);
  float* be = al + 64;
  float* csa = be + 64;  // CTA column sums: dalpha, dbeta
  float* csb = csa + 64;
  const float* wts = p.pack + kWtOff / sizeof(float);  // W^T (row epilogue) through L1
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tslot;
  Ctx c;
  c.sm = sm;
  c.mbar = &mbar;
  __shared__ __align__(8) uint64_t wbar;
  load_weights_b16(W2b, p.pack, al, be, &wbar);
  if (threadIdx.x < 128) csa[threadIdx.x] = 0.f;  // csa, csb (published by setup's barrier)
  TC_M();
  setup(c, &tslot, 512);
  TC_M();
  const uint32_t aW0b = tc::smem_u32(W0b), aW1b = tc::smem_u32(W1b), aW2b = tc::smem_u32(W2b);
  const uint32_t aB0 = tc::smem_u32(B0), aB1 = tc::smem_u32(B1), aB2 = tc::smem_u32(B2), aB3 = tc::smem_u32(B3);
  const uint32_t aB4 = tc::smem_u32(B4), aB5 = tc::smem_u32(B5);
  bool first = true;
  const int f0 = FPT * c.q;
  for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const TileRange tr = tile_range(tiles, t);
    const SegMap sg = seg_map(g, tr);
    float acc[2] = {};
    for (int c0 = tr.e0; c0 < tr.e1; c0 += TE) {
      const int ne = min(TE, tr.e1 - c0);
      const ES es = edge_sc(g, c0, ne, c.e);
#ifdef JANUS_TC_TRACE
      {
        float dmy;
        asm volatile("mov.b32 %0, %1;" : "=f"(dmy) : "f"(es.d));
        TC_M();
      }
#endif
      {
        float ph[FPT], dph[FPT];
        basis(es.d, rc, f0, ph, dph);
        TC_M();
        st_b16(B4, c.e, f0, ph);   // phi  (A of z = phi A and of dA)
        st_b16(B5, c.e, f0, dph);  // phi' (A of z' = phi' A and of dA)
      }
      TC_M();
      tc::mbar_wait(&wbar, 0);
      TC_M();  // weights landed (immediate after the first chunk)
      c.publish();
      if (threadIdx.x == 0) {
        mma_kb16(c.tmem + TM_Z, aB4, aW0b);
        mma_kb16(c.tmem + TM_ZP, aB5, aW0b);
        tc::commit(c.mbar);
      }
      TC_M();
      const float qb = edge_qbar(g, es, Fbar);  // its loads overlap the MMAs
      c.wait_mma();
      TC_M();
      {
        float z[FPT], zp[FPT];
        c.ld2(TM_Z, TM_ZP, z, zp);
#pragma unroll
        for (int j = 0; j < FPT; ++j) {
          const float zz = z[j] + al[f0 + j], s1 = fsig(zz);
          z[j] = zz * s1;
          zp[j] = s1 * (1.0f + zz * (1.0f - s1)) * zp[j];
        }
        st_b16(B0, c.e, f0, z);  // s    (A of g = s B and of dB)
        st_b16(B1, c.e, f0, zp); // sdot (A of g' = sdot B and of dB)
      }
      c.publish();
      if (threadIdx.x == 0) {
        mma_kb16(c.tmem + TM_G, aB0, aW1b);
        mma_kb16(c.tmem + TM_GP, aB1, aW1b);
        tc::commit(c.mbar);
      }
      TC_M();
      c.wait_mma();
      TC_M();
      {
        float mu[FPT], nu[FPT];
        float gg[FPT], gp[FPT];
        float pm[FPT], px[FPT];
        float4 a4[FPT / 4], aj4[FPT / 4], v4[FPT / 4], d4[FPT / 4];
#pragma unroll
        for (int q = 0; q < FPT / 4; ++q) {
          a4[q] = __ldg(reinterpret_cast<const float4*>(am + (size_t)es.i * H + f0) + q);
          aj4[q] = __ldg(reinterpret_cast<const float4*>(am + (size_t)es.j * H + f0) + q);
          v4[q] = __ldg(reinterpret_cast<const float4*>(v + (size_t)es.j * H + f0) + q);
          d4[q] = __ldg(reinterpret_cast<const float4*>(vdot + (size_t)es.j * H + f0) + q);
        }
        c.ld2(TM_G, TM_GP, gg, gp);
        TC_M();
#pragma unroll
        for (int q = 0; q < FPT / 4; ++q) {
          const float ai[4] = {a4[q].x, a4[q].y, a4[q].z, a4[q].w}, aj[4] = {aj4[q].x, aj4[q].y, aj4[q].z, aj4[q].w};
          const float vv[4] = {v4[q].x, v4[q].y, v4[q].z, v4[q].w}, dv[4] = {d4[q].x, d4[q].y, d4[q].z, d4[q].w};
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int k = 4 * q + r;
            const float gb = gg[k] + be[f0 + k];
            const float w = es.c * gb, wp = qb * (es.dc * gb + es.c * gp[k]);
            pm[k] = fmaf(wp, vv[r], w * dv[r]);  // qb w' v_j + w vdot_j
            px[k] = wp * aj[r];                  // qb w' am_j
            const float rho = ai[r] * vv[r], kap = ai[r] * dv[r];
            mu[k] = qb * es.dc * rho + es.c * kap;
            nu[k] = qb * es.c * rho;
          }
        }
        TC_M();
        st_pl(T0, c.e, f0, pm);
        st_pl(T1, c.e, f0, px);
        st_b16(B2, c.e, f0, mu);  // mu (B of dB)
        st_b16(B3, c.e, f0, nu);  // nu (B of dB)
      }
      TC_M();
      c.publish();
      if (threadIdx.x == 0) {  // dB += s^T mu + sdot^T nu; sbar = mu B^T, sdotbar = nu B^T (bf16: feed dA only)
        mma_wg_b16(c.tmem + TM_BG, aB0, aB2, !first);
        mma_wg_b16(c.tmem + TM_BG, aB1, aB3, true);
        mma_kb16(c.tmem + TM_G, aB2, aW2b);
        mma_kb16(c.tmem + TM_GP, aB3, aW2b);
        tc::commit(c.mbar);
      }
      TC_M();
      {  // row sums and dbeta under the MMAs
        const uint8_t* const tl[2] = {T0, T1};
        seg_rows<2>(g, tr.r0, c0, ne, tl, sg, acc);
      }
      b16_colsum_add(B2, csb);  // dbeta += sum_e mu_e
      TC_M();
      c.wait_mma();  // dB and sbar done
      __syncthreads();  // row sums and column sums done: T1, B2, B3 may be rewritten
      TC_M();
      {
        float z[FPT], zp[FPT], sb[FPT], sdb[FPT];
        c.ld2(TM_Z, TM_ZP, z, zp);
        c.ld2(TM_G, TM_GP, sb, sdb);
#pragma unroll
        for (int j = 0; j < FPT; ++j) {
          const float zz = z[j] + al[f0 + j], s1 = fsig(zz);
          const float ds = s1 * (1.0f + zz * (1.0f - s1));
          const float d2s = s1 * (1.0f - s1) * (2.0f + zz * (1.0f - 2.0f * s1));
          z[j] = sb[j] * ds + sdb[j] * d2s * zp[j];  // zbar
          zp[j] = sdb[j] * ds;                       // zbar'
        }
        st_b16(B2, c.e, f0, z);   // zbar  (B of dA; its column sums)
        st_b16(B3, c.e, f0, zp);  // zbar' (B of dA)
      }
      c.publish();
      if (threadIdx.x == 0) {  // dA += phi^T zbar + phi'^T zbar'
        mma_wg_b16(c.tmem + TM_AG, aB4, aB2, !first);
        mma_wg_b16(c.tmem + TM_AG, aB5, aB3, true);
        tc::commit(c.mbar);
      }
      b16_colsum_add(B2, csa);  // dalpha += sum_e zbar_e (beside the dA MMA)
      TC_M();
      c.wait_mma();
      TC_M();
      first = false;
      __syncthreads();
    }
    seg_finish<2>(sg, acc);
    float* const outs[2] = {mdot_out, X_out};
    seg_write<2>(tr.r0, sg, outs, acc);
    TC_M();
    if (inj) rows_times_wt(tr.r0, tr.r1, sg, acc[1], reinterpret_cast<float*>(T1), wts, nullptr, nullptr, inj);  // hbar^F = X W^T
    TC_M();
  }
  float* part = partial + (size_t)blockIdx.x * PE;
  if (first) {
    for (int x = threadIdx.x; x < PE; x += NT) part[x] = 0.f;
    teardown(c, 512);
    return;
  }
  write_partial(c, part, T0, csa, csb, TM_AG, TM_BG TC_PASS);
  TC_M();
  teardown(c, 512);
  TC_M();
  TC_SPAN_END("bf");
  TC_DUMP("bf");
}

constexpr size_t kSmallBytes = sizeof(float) * (128 + NQ * TE) + 1024;  // alpha, beta, FF force scalars, 1 KB alignment slack
constexpr size_t fe_smem() { return 2 * kWTile + 2 * kTile + kSmallBytes; }
constexpr size_t ff_smem() { return 2 * kWTile + 2 * kTile + kSmallBytes; }
constexpr size_t be_smem() { return 2 * kWTile + 2 * kTile + 4 * kBTile + kSmallBytes; }  // 24 KB bf16 weights in 32
constexpr size_t bf_smem() { return 2 * kWTile + 2 * kTile + 6 * kBTile + kSmallBytes; }

}  // namespace edge_tc
}  // namespace janus
