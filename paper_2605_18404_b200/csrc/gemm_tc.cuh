// gemm_tc.cuh — TMA-fed tcgen05 GEMM with fused epilogues for the
// generic-width path (stage_wide.inc): D[rows x N] = A[rows x K] . W^T with
// A fp32 row-major (K-major) in global memory and W the weight as a K-major
// [N x K] fp32 matrix, tf32 tensor-core math, fp32 accumulate in TMEM.
//
// Warp roles (256 threads): warp 0 issues the TMA loads (cp.async.bulk.tensor
// with SWIZZLE_128B tensor maps: each 32-float K block of A and W lands in the
// canonical SW128 K-major slab the UMMA descriptor reads), warp 1 issues the
// MMAs (one elected thread, M=128 x N x K=8 tf32 per instruction) and frees a
// pipeline stage with tcgen05.commit; then all 8 warps run the epilogue
// (thread = tile row = TMEM lane; 32-column tcgen05.ld chunks).
//
// Pair mode.  The per-pair operands are stacked [value rows; derivative rows]
// (rows p and P + p belong to pair p).  A pair-mode tile takes 64 pairs,
// arranged so a pair's value and radial-derivative rows sit in lanes l and
// l + 16 of the same TMEM lane quarter (gemm_nt_kernel); the epilogue swaps
// them with one warp shuffle, so the elementwise steps that need both (SiLU
// and SiLU'·z', the filter w, w', zbar) run in the GEMM's epilogue instead of
// a separate pass over HBM.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "tc.cuh"

namespace janus {
namespace gemm_tc {

constexpr int kKB = 32;  // floats per K block (one 128 B SW128 slab)

struct Problem {
  int rows;        // plain mode: rows of A / D; pair mode: pairs P (A, D have 2P rows)
  int K;           // multiple of 32
  int N;           // 64, 128 or 256 (one N tile)
  int pair;        // 1: pair-mode tiles (64 pairs = 128 rows)
  int split3 = 0;  // 1: 3xTF32 (fp32-accurate): x = hi + lo split in shared memory, D = lo.Whi + hi.Wlo + hi.Whi
};

__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint64_t* mbar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(tc::smem_u32(mbar))
      : "memory");
}

// ----------------------------------------------------------------- epilogues
// The accumulator arrives row-per-thread (thread = TMEM lane = tile row), so a
// thread's 32 output columns are one 128 B row segment.  Stored straight from
// registers, each warp-wide float4 store would touch 32 rows; instead each warp
// stages its 32 x 32 chunk in shared memory (4 KB, XOR-swizzled 16 B slots:
// conflict-free both ways) and writes it back as eight fully coalesced float4
// stores of four 128 B rows each.  Row pointers travel by shuffle; a null
// pointer skips the row (tiles past the last pair).  wload is the mirror image
// for epilogues that read a row-major operand (the raw z of the zbar steps).
__device__ __forceinline__ float* shfl_ptr(float* p, int src) {
  const uint64_t v = reinterpret_cast<uint64_t>(p);
  const uint32_t lo = __shfl_sync(0xffffffffu, static_cast<uint32_t>(v), src);
  const uint32_t hi = __shfl_sync(0xffffffffu, static_cast<uint32_t>(v >> 32), src);
  return reinterpret_cast<float*>((static_cast<uint64_t>(hi) << 32) | lo);
}

__device__ __forceinline__ void wstore(float* dst, const float (&v)[32], float4* stg) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 8; ++j) stg[lane * 8 + (j ^ (lane & 7))] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = 4 * i + (lane >> 3), c = lane & 7;
    float* d = shfl_ptr(dst, r);
    if (d) reinterpret_cast<float4*>(d)[c] = stg[r * 8 + (c ^ (r & 7))];
  }
}

__device__ __forceinline__ void wload(const float* src, float (&v)[32], float4* stg) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = 4 * i + (lane >> 3), c = lane & 7;
    const float* s = shfl_ptr(const_cast<float*>(src), r);
    stg[r * 8 + (c ^ (r & 7))] = s ? __ldg(reinterpret_cast<const float4*>(s) + c) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float4 x = stg[lane * 8 + (j ^ (lane & 7))];
    v[4 * j] = x.x;
    v[4 * j + 1] = x.y;
    v[4 * j + 2] = x.z;
    v[4 * j + 3] = x.w;
  }
}

// Elementwise math of the tf32 epilogues: one fast sigmoid per element
// (__expf + __fdividef, ~1e-6 relative: far below tf32's 2^-11) shared by
// SiLU, SiLU' and SiLU'', and branch-free value / derivative selects (the two
// halves of a warp take different formulas).  Per-column bias vectors are
// read as 8 warp-uniform float4s per chunk.
__device__ __forceinline__ float sig_fast(float x) { return __fdividef(1.0f, 1.0f + __expf(-x)); }
// the 3xTF32 (fp32-tolerance) launches use the accurate sigmoid
__device__ __forceinline__ float sig_sel(float x, int exact) { return exact ? 1.0f / (1.0f + expf(-x)) : sig_fast(x); }
__device__ __forceinline__ void load_cols(const float* v, int c0, float (&o)[32]) {
  const float4* v4 = reinterpret_cast<const float4*>(v + c0);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float4 x = __ldg(v4 + j);
    o[4 * j] = x.x;
    o[4 * j + 1] = x.y;
    o[4 * j + 2] = x.z;
    o[4 * j + 3] = x.w;
  }
}

// Each functor sees, per 32-column chunk, this thread's accumulator row and
// (pair mode) the partner row (value <-> derivative), and writes its outputs
// through wstore (warp-collective: every lane calls, ok = row exists).
// Row indices: plain: r = tile row; pair: p = pair, half = 0 value / 1 deriv.
struct EpiStore {  // D = the accumulator (pair mode: stacked like A)
  float* D;
  int ld;
  __device__ void operator()(int p, int half, int P, bool ok, int c0, const float (&own)[32], const float (&)[32],
                             float4* stg) const {
    wstore(ok ? D + static_cast<size_t>(half ? P + p : p) * ld + c0 : nullptr, own, stg);
  }
};

// [z; z'] -> a2 = [SiLU(z + alpha); SiLU'(z + alpha) z']  (+ the raw z2 when asked)
struct EpiAct2 {
  float* a2;
  float* z2;  // optional raw copy (BF needs z, z' again for zbar)
  const float* alpha;
  int ld;
  int exact = 0;
  __device__ void operator()(int p, int half, int P, bool ok, int c0, const float (&own)[32], const float (&oth)[32],
                             float4* stg) const {
    const size_t off = static_cast<size_t>(half ? P + p : p) * ld + c0;
    float o[32];
    load_cols(alpha, c0, o);
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float zz = (half ? oth[j] : own[j]) + o[j];
      const float sg = sig_sel(zz, exact), zs = zz * sg;
      o[j] = half ? (sg + zs * (1.0f - sg)) * own[j] : zs;  // SiLU'(z) z' : SiLU(z)
    }
    wstore(ok ? a2 + off : nullptr, o, stg);
    if (z2) wstore(ok ? z2 + off : nullptr, own, stg);
  }
};

// [g; g'] -> w = c (g + beta), w' = c' (g + beta) + c g'   ([P][N] each)
struct EpiFilter {
  float* wf;
  float* wfp;
  const float* beta;
  const float4* pgeo;  // (d, c, c', i | u, j) per pair
  int ld;
  __device__ void operator()(int p, int half, int, bool ok, int c0, const float (&own)[32], const float (&oth)[32],
                             float4* stg) const {
    const float4 g0 = ok ? __ldg(pgeo + 2 * p) : make_float4(0.f, 0.f, 0.f, 0.f);
    const float cg = half ? g0.z : g0.y, cd = half ? g0.y : 0.0f;  // w' = c' g + c g'; w = c g
    float o[32];
    load_cols(beta, c0, o);
#pragma unroll
    for (int j = 0; j < 32; ++j) o[j] = cg * ((half ? oth[j] : own[j]) + o[j]) + cd * own[j];
    wstore(ok ? (half ? wfp : wf) + static_cast<size_t>(p) * ld + c0 : nullptr, o, stg);
  }
};

// [sbar; sdotbar] (+ raw [z; z']) -> [zbar; zbar'] = [sbar SiLU'(z) + sdotbar SiLU''(z) z'; sdotbar SiLU'(z)]
struct EpiZbar {
  float* zb;
  const float* z2;
  const float* alpha;
  int ld;
  int exact = 0;
  __device__ void operator()(int p, int half, int P, bool ok, int c0, const float (&own)[32], const float (&oth)[32],
                             float4* stg) const {
    const size_t off = static_cast<size_t>(half ? P + p : p) * ld + c0;
    float zo[32];  // value lanes: z; derivative lanes: z'
    wload(ok ? z2 + off : nullptr, zo, stg);
    float o[32];
    load_cols(alpha, c0, o);
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float zx = __shfl_xor_sync(0xffffffffu, zo[j], 16);
      const float zz = (half ? zx : zo[j]) + o[j];
      const float sg = sig_sel(zz, exact), u = 1.0f - sg;
      const float ds = sg * (1.0f + zz * u);                                          // SiLU'
      const float d2 = half ? 0.0f : sg * u * (2.0f + zz * (1.0f - 2.0f * sg)) * zx;  // SiLU'' z' (value rows)
      o[j] = own[j] * ds + oth[j] * d2;
    }
    wstore(ok ? zb + off : nullptr, o, stg);
  }
};

// plain: z -> a = SiLU(z + alpha) (+ raw z)
struct EpiAct1 {
  float* a;
  float* zraw;
  const float* alpha;
  int ld;
  int exact = 0;
  __device__ void operator()(int r, int, int, bool ok, int c0, const float (&own)[32], const float (&)[32],
                             float4* stg) const {
    const size_t off = static_cast<size_t>(r) * ld + c0;
    float o[32];
    load_cols(alpha, c0, o);
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float zz = own[j] + o[j];
      o[j] = zz * sig_sel(zz, exact);
    }
    wstore(ok ? a + off : nullptr, o, stg);
    if (zraw) wstore(ok ? zraw + off : nullptr, own, stg);
  }
};

// plain: sbar (+ raw z) -> zbar = sbar SiLU'(z + alpha)
struct EpiBeZbar {
  float* zb;
  const float* z;
  const float* alpha;
  int ld;
  int exact = 0;
  __device__ void operator()(int r, int, int, bool ok, int c0, const float (&own)[32], const float (&)[32],
                             float4* stg) const {
    const size_t off = static_cast<size_t>(r) * ld + c0;
    float zr[32];
    wload(ok ? z + off : nullptr, zr, stg);
    float o[32];
    load_cols(alpha, c0, o);
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float zz = zr[j] + o[j], sg = sig_sel(zz, exact);
      o[j] = own[j] * sg * (1.0f + zz * (1.0f - sg));
    }
    wstore(ok ? zb + off : nullptr, o, stg);
  }
};

// One tile per CTA, 256 threads: warp 0 lane 0 = TMA producer, warp 1 lane 0
// = MMA issuer, 2 streamed stages (A 16 KB + W N x 128 B per 32-float K
// block), then all 8 warps run the epilogue once the accumulator is complete
// (the drained stages hold the transposes).  ~100 KB of smem: two CTAs per
// SM, so one tile's epilogue overlaps the other's loads and MMAs.  (A
// persistent variant — 148 CTAs, double-buffered TMEM accumulator, resident W
// for K = R, 4 + 8 warps — measured slower inside the 8-lane step: 146 vs
// 151 structures/s at configs[2], P = 1; 136 vs 140 at P = 8.)
//
// Pair tiles put each pair's value and derivative rows in the SAME 32-row TMEM
// lane quarter: quarter q holds the value rows of pairs 64 t + 16 q .. + 15 in
// its lanes 0..15 and their derivative rows in lanes 16..31, so the epilogue
// exchanges partners with one __shfl_xor(., 16) (eight 16-row TMA boxes per
// K block).  Warp w reads lane quarter w % 4 (the TMEM access rule) and
// column half w / 4.
constexpr int kThreads = 256;
constexpr int kStages = 2;
// per stage: A slab (128 rows x 128 B) + W slab (N x 128 B); 3xTF32 adds their lo parts
constexpr size_t smem_bytes(int N, int split3 = 0) {
  return static_cast<size_t>(kStages) * (128 * 128 + N * 128) * (split3 ? 2 : 1) + 1024;
}

template <class Epi>
__global__ void __launch_bounds__(kThreads, 1) gemm_nt_kernel(const __grid_constant__ CUtensorMap tmA,
                                                                      const __grid_constant__ CUtensorMap tmW, Problem pb,
                                                                      Epi epi) {
  JANUS_GDC_WAIT();
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (tc::smem_u32(sm_raw) & 1023u)) & 1023u);
  const uint32_t slabA = 128 * 128, slabW = static_cast<uint32_t>(pb.N) * 128, sbytes = slabA + slabW;
  const uint32_t lo_off = kStages * sbytes;  // 3xTF32: the lo parts of stage s at lo_off + s * sbytes
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages], split[kStages], accum;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KB = pb.K / kKB;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
      tc::mbar_init(&split[s], 6);  // 3xTF32: one arrive per split warp (warps 2..7)
    }
    tc::mbar_init(&accum, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) tc::tmem_alloc(&tslot, static_cast<uint32_t>(pb.N));
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tslot;
  const int t = blockIdx.x;
  if (warp == 0 && lane == 0) {
    for (int kb = 0; kb < KB; ++kb) {
      const int s = kb % kStages;
      if (kb >= kStages) tc::mbar_wait(&empty[s], ((kb / kStages) - 1) & 1);
      tc::mbar_expect_tx(&full[s], sbytes);
      const uint32_t a = tc::smem_u32(sm + s * sbytes);
      if (pb.pair) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          tma_load_2d(a + (32 * q) * 128, &tmA, kb * kKB, 64 * t + 16 * q, &full[s]);
          tma_load_2d(a + (32 * q + 16) * 128, &tmA, kb * kKB, pb.rows + 64 * t + 16 * q, &full[s]);
        }
      } else {
        tma_load_2d(a, &tmA, kb * kKB, 128 * t, &full[s]);
      }
      tma_load_2d(a + slabA, &tmW, kb * kKB, 0, &full[s]);
    }
  } else if (warp == 1 && lane == 0) {
    const uint32_t idesc = tc::idesc_tf32(128, pb.N, false, false);
    for (int kb = 0; kb < KB; ++kb) {
      const int s = kb % kStages;
      tc::mbar_wait(pb.split3 ? &split[s] : &full[s], (kb / kStages) & 1);
      tc::fence_after();
      const uint32_t a = tc::smem_u32(sm + s * sbytes);
      const uint64_t da = tc::smem_desc(a, 16, 1024, 2), dw = tc::smem_desc(a + slabA, 16, 1024, 2);
      if (pb.split3) {  // lo.Whi + hi.Wlo + hi.Whi (small terms first)
        const uint64_t dal = tc::smem_desc(a + lo_off, 16, 1024, 2), dwl = tc::smem_desc(a + lo_off + slabA, 16, 1024, 2);
#pragma unroll
        for (int k = 0; k < kKB / 8; ++k) {
          const uint64_t o = static_cast<uint64_t>((32 * k) >> 4);
          tc::mma_tf32(tmem, dal + o, dw + o, idesc, (kb > 0 || k > 0) ? 1u : 0u);
          tc::mma_tf32(tmem, da + o, dwl + o, idesc, 1u);
          tc::mma_tf32(tmem, da + o, dw + o, idesc, 1u);
        }
      } else {
#pragma unroll
        for (int k = 0; k < kKB / 8; ++k)
          tc::mma_tf32(tmem, da + static_cast<uint64_t>((32 * k) >> 4), dw + static_cast<uint64_t>((32 * k) >> 4), idesc,
                       (kb > 0 || k > 0) ? 1u : 0u);
      }
      tc::commit(&empty[s]);
    }
    tc::commit(&accum);
  } else if (warp >= 2 && pb.split3) {
    // 3xTF32 split of each landed stage: hi = rna_tf32(x) in place, lo = x - hi into the lo slabs
    // (elementwise, so the SW128 layout carries over); then visible to the tensor core
    const int st = static_cast<int>(threadIdx.x) - 64;  // 0..191
    for (int kb = 0; kb < KB; ++kb) {
      const int s = kb % kStages;
      tc::mbar_wait(&full[s], (kb / kStages) & 1);
      float4* hi = reinterpret_cast<float4*>(sm + s * sbytes);
      float4* lo = reinterpret_cast<float4*>(sm + lo_off + s * sbytes);
      const int n4 = static_cast<int>(sbytes / 16);
      for (int x = st; x < n4; x += 192) {
        const float4 v = hi[x];
        const float4 h = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
        hi[x] = h;
        lo[x] = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
      }
      tc::fence_async_smem();
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(&split[s])) : "memory");
    }
  }
  __syncwarp();
  tc::mbar_wait(&accum, 0);
  tc::fence_after();
  const int q = warp & 3, row = 32 * q + lane;
  const uint32_t lane_base = static_cast<uint32_t>(32 * q) << 16;
  const int half = pb.pair ? (lane >> 4) : 0;
  const int p = pb.pair ? 64 * t + 16 * q + (lane & 15) : 128 * t + row;
  const bool ok = p < pb.rows;
  const int n_half = pb.N / 2, cb = (warp >> 2) * n_half;
  float4* stg = reinterpret_cast<float4*>(sm) + warp * 256;  // the stages are drained
  for (int c0 = cb; c0 < cb + n_half; c0 += 32) {
    float own[32], oth[32];
    tc::ld32(tmem + lane_base + static_cast<uint32_t>(c0), own);
    if (pb.pair) {
#pragma unroll
      for (int j = 0; j < 32; ++j) oth[j] = __shfl_xor_sync(0xffffffffu, own[j], 16);
      epi(p, half, pb.rows, ok, c0, own, oth, stg);
    } else {
      epi(p, 0, 0, ok, c0, own, own, stg);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 2) tc::tmem_free(tmem, static_cast<uint32_t>(pb.N));
}

}  // namespace gemm_tc
}  // namespace janus
