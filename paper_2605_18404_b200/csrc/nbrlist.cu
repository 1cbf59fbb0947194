// nbrlist.cu — device-side LM: periodic cell-list neighbour build on the GPU
// (the LM instruction of reference ir.hpp:25 /
// graph.hpp:124 feeds the first FE).  Output is the CSR-by-receiver the stage
// consumes, BIT-IDENTICAL to the host build (host.cpp nbrlist_build) and the
// oracle (oracle/mlip_oracle.c mo_build_nbrlist):
//   * row i holds every (j, s) of i's structure with |s|_inf <= ceil(r_c / L),
//     (i, 0) excluded, and d2 = ((xj+sxL)-xi)^2 + (..)^2 + (..)^2 < r_c^2 in
//     fp64 with no FMA contraction (explicit __d*_rn, the host is compiled
//     with -ffp-contract=off);
//   * rows sorted by (j, sx, sy, sz); rev[e] = index of (j -> i, -s).
//
// Integer / byte work, HBM- and latency-bound (no tensor cores):
//   bin      : atom -> (structure, cell) with a wrap index; counting sort of
//              atoms by cell (positions copied cell-major so a stencil walk
//              reads contiguous memory)
//   walk_pad : one warp per atom walks the (2m+1)^3 stencil of cells once,
//              counts its row and keeps the 64-bit keys (j, s) of rows up to
//              kPadCap rank-sorted in a padded per-atom buffer (keys are
//              unique, so rank = #smaller keys is a permutation) — the cell
//              order inside a bin (from atomics) never reaches the output
//   scan     : row_ptr (single CTA, deterministic)
//   compact  : padded rows -> CSR (a row over kPadCap is walked again)
//   rev      : binary search of (i, -s) in row j's sorted keys
// Cells are >= r_c (1 + 1e-6) / kSub wide and the stencil reaches kSub cells
// each way, so the rounding of the binning can move a pair by at most one cell
// and the (2 kSub + 1)^3 stencil still covers it; boxes smaller than r_c /
// kSub get one cell and a stencil of ceil(r_c / L) images.  kSub = 2 (half-
// cutoff cells, 5x5x5 stencil) visits ~2.3x fewer candidates than 3x3x3 of
// r_c cells (stencil volume 125 (r_c/2)^3 vs 27 r_c^3, against the cutoff
// sphere's 4.2 r_c^3).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/janus/errors.hpp"
#include "../../include/janus_cuda.h"
#include "common.cuh"
#include "cuda_check.hpp"
#include "nbrlist.hpp"

namespace janus {
namespace nbr {

struct StructMeta {  // per structure, built on the host from the box lengths
  double L;
  int nc;      // cells per dimension
  int m;       // stencil half-width (cells)
  int nimg;    // host image range ceil(r_c / L)
  int cell0;   // first global cell id
};

constexpr int kWarps = 8;        // warps per CTA in the row kernels
#ifndef JANUS_NBR_SUB
#define JANUS_NBR_SUB 2
#endif
constexpr int kSub = JANUS_NBR_SUB;  // cells per cutoff length
constexpr int kSortCap = 512;    // keys per warp staged in shared memory
constexpr int kPadCap = 128;     // sorted keys per atom kept by the single-walk pass (denser rows re-walk)

__device__ __forceinline__ int floordiv(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

__device__ __forceinline__ unsigned long long make_key(int j, int sx, int sy, int sz) {
  return (static_cast<unsigned long long>(static_cast<unsigned>(j)) << 24) |
         (static_cast<unsigned long long>(sx + 128) << 16) | (static_cast<unsigned long long>(sy + 128) << 8) |
         static_cast<unsigned long long>(sz + 128);
}

// atom -> wrapped cell coordinates + wrap index, per-cell counts
__global__ void bin_kernel(int n, const double* __restrict__ pos, const int* __restrict__ struct_id,
                           const StructMeta* __restrict__ meta, int* __restrict__ cell_of, int4* __restrict__ cw,
                           int* __restrict__ cell_count) {
  JANUS_GDC_WAIT();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const StructMeta sm = meta[struct_id[i]];
  int c[3], w[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double x = pos[3 * i + k];
    const double wf = floor(x / sm.L);
    const double xw = x - wf * sm.L;
    int ck = static_cast<int>(floor(xw * sm.nc / sm.L));
    c[k] = min(max(ck, 0), sm.nc - 1);
    w[k] = static_cast<int>(wf);
  }
  const int cid = sm.cell0 + (c[0] * sm.nc + c[1]) * sm.nc + c[2];
  cell_of[i] = cid;
  cw[i] = make_int4(w[0], w[1], w[2], 0);
  atomicAdd(cell_count + cid, 1);
}

// exclusive scan of n ints into out[0..n] (out[n] = total), one CTA of 1024
__global__ void scan_kernel(int n, const int* __restrict__ in, int* __restrict__ out) {
  JANUS_GDC_WAIT();
  __shared__ int warp_tot[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int base = 0; base < n; base += blockDim.x) {
    const int idx = base + threadIdx.x;
    const int v = idx < n ? in[idx] : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int t = lane < static_cast<int>(blockDim.x >> 5) ? warp_tot[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      warp_tot[lane] = t;  // inclusive over warps
    }
    __syncthreads();
    const int excl = carry + (wid > 0 ? warp_tot[wid - 1] : 0) + x - v;
    if (idx < n) out[idx] = excl;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) out[n] = carry;
}

// counting sort of atoms by cell: cell-major copies of index, position and wrap
__global__ void scatter_kernel(int n, const double* __restrict__ pos, const int* __restrict__ cell_of,
                               const int4* __restrict__ cw, const int* __restrict__ cell_start,
                               int* __restrict__ cursor, int* __restrict__ c_atom, double* __restrict__ c_pos,
                               int4* __restrict__ c_w) {
  JANUS_GDC_WAIT();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int cid = cell_of[i];
  const int slot = cell_start[cid] + atomicAdd(cursor + cid, 1);
  c_atom[slot] = i;
  c_pos[3 * slot + 0] = pos[3 * i + 0];
  c_pos[3 * slot + 1] = pos[3 * i + 1];
  c_pos[3 * slot + 2] = pos[3 * i + 2];
  c_w[slot] = cw[i];
}

// Walk atom i's stencil in warp-uniform strips of 32 candidates: every lane
// calls f(hit, key) once per strip (hit = lane's candidate is a neighbour), so
// the callee may ballot.  The candidates of up to 32 stencil cells are packed
// into dense strips: lane c of a group owns cell c (its start, size and image
// shift), a warp scan of the sizes gives each cell's offset, and lane l of a
// strip finds the cell owning candidate v0 + l by a 5-step shuffle search.
// One strip per cell (~12 candidates at C2 densities) left ~60% of the lanes
// idle; packed, a 27-cell stencil of ~330 candidates takes ~11 strips instead
// of 27.  The candidate set, and each candidate's d2, are unchanged, and the
// row order comes from the rank sort: the output stays bit-identical.
template <typename F>
__device__ __forceinline__ void walk(int i, const double* __restrict__ pos, const int* __restrict__ struct_id,
                                     const StructMeta* __restrict__ meta, const int* __restrict__ cell_of,
                                     const int4* __restrict__ cw, const int* __restrict__ cell_start,
                                     const int* __restrict__ c_atom, const double* __restrict__ c_pos,
                                     const int4* __restrict__ c_w, double rc2, int lane, F&& f) {
  const StructMeta sm = meta[struct_id[i]];
  const int local = cell_of[i] - sm.cell0;
  const int ci[3] = {local / (sm.nc * sm.nc), (local / sm.nc) % sm.nc, local % sm.nc};
  const int4 wi = cw[i];
  const double xi = pos[3 * i + 0], yi = pos[3 * i + 1], zi = pos[3 * i + 2];
  const double L = sm.L;
  const int side = 2 * sm.m + 1, ncell = side * side * side;
  for (int g0 = 0; g0 < ncell; g0 += 32) {
    // this lane's stencil cell of the group: candidate range and image shift
    const int c = g0 + lane;
    int beg = 0, cnt = 0, tx = 0, ty = 0, tz = 0;
    if (c < ncell) {
      const int dx = c / (side * side) - sm.m, dy = (c / side) % side - sm.m, dz = c % side - sm.m;
      const int ux = ci[0] + dx, uy = ci[1] + dy, uz = ci[2] + dz;
      tx = floordiv(ux, sm.nc);
      ty = floordiv(uy, sm.nc);
      tz = floordiv(uz, sm.nc);
      const int cid = sm.cell0 + ((ux - tx * sm.nc) * sm.nc + (uy - ty * sm.nc)) * sm.nc + (uz - tz * sm.nc);
      beg = cell_start[cid];
      cnt = cell_start[cid + 1] - beg;
    }
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int excl = incl - cnt, total = __shfl_sync(0xffffffffu, incl, 31);
    for (int v0 = 0; v0 < total; v0 += 32) {
      const int v = v0 + lane;
      // owner = the highest lane whose range starts at or before v (excl is non-decreasing)
      int own = 0;
#pragma unroll
      for (int st = 16; st > 0; st >>= 1) {
        const int pe = __shfl_sync(0xffffffffu, excl, own + st);
        if (pe <= v) own += st;
      }
      const int obeg = __shfl_sync(0xffffffffu, beg, own), oexcl = __shfl_sync(0xffffffffu, excl, own);
      const int otx = __shfl_sync(0xffffffffu, tx, own), oty = __shfl_sync(0xffffffffu, ty, own),
                otz = __shfl_sync(0xffffffffu, tz, own);
      bool hit = false;
      unsigned long long key = 0;
      if (v < total) {
        const int q = obeg + (v - oexcl);
        const int4 wj = c_w[q];
        // image of j in i's original frame: s = t - w_j + w_i (exact integers)
        const int sx = otx - wj.x + wi.x, sy = oty - wj.y + wi.y, sz = otz - wj.z + wi.z;
        const int j = c_atom[q];
        if (abs(sx) <= sm.nimg && abs(sy) <= sm.nimg && abs(sz) <= sm.nimg && !(j == i && sx == 0 && sy == 0 && sz == 0)) {
          const double rx = __dsub_rn(__dadd_rn(c_pos[3 * q + 0], __dmul_rn(static_cast<double>(sx), L)), xi);
          const double ry = __dsub_rn(__dadd_rn(c_pos[3 * q + 1], __dmul_rn(static_cast<double>(sy), L)), yi);
          const double rz = __dsub_rn(__dadd_rn(c_pos[3 * q + 2], __dmul_rn(static_cast<double>(sz), L)), zi);
          const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(rx, rx), __dmul_rn(ry, ry)), __dmul_rn(rz, rz));
          hit = d2 < rc2;
          key = make_key(j, sx, sy, sz);
        }
      }
      f(hit, key);
    }
  }
}

#define NBR_WALK_ARGS pos, struct_id, meta, cell_of, cw, cell_start, c_atom, c_pos, c_w, rc2
#define NBR_WALK_PARAMS                                                                                        \
  const double *__restrict__ pos, const int *__restrict__ struct_id, const StructMeta *__restrict__ meta,      \
      const int *__restrict__ cell_of, const int4 *__restrict__ cw, const int *__restrict__ cell_start,         \
      const int *__restrict__ c_atom, const double *__restrict__ c_pos, const int4 *__restrict__ c_w, double rc2

// rank-sort the warp's n keys in buf (unique) and emit them at row offset base
__device__ __forceinline__ void emit_sorted(const unsigned long long* buf, int deg, int base, int lane,
                                            unsigned long long* __restrict__ skey, int* __restrict__ col,
                                            int* __restrict__ shift) {
  for (int k = lane; k < deg; k += 32) {
    const unsigned long long key = buf[k];
    int rank = 0;
    for (int q = 0; q < deg; ++q) rank += buf[q] < key;
    const int e = base + rank;
    skey[e] = key;
    col[e] = static_cast<int>(key >> 24);
    shift[3 * e + 0] = static_cast<int>((key >> 16) & 0xff) - 128;
    shift[3 * e + 1] = static_cast<int>((key >> 8) & 0xff) - 128;
    shift[3 * e + 2] = static_cast<int>(key & 0xff) - 128;
  }
}

// Single walk per atom: count the row and, when it has <= kPadCap neighbours
// (every row at the configs' densities), keep its keys sorted in a padded
// per-atom buffer, so the CSR needs no second walk (compact_kernel).  Rows
// above kPadCap are only counted here and re-walked by compact_kernel.
__global__ void __launch_bounds__(kWarps * 32) walk_pad_kernel(int n, NBR_WALK_PARAMS, int* __restrict__ deg,
                                                               unsigned long long* __restrict__ pad) {
  JANUS_GDC_WAIT();
  __shared__ unsigned long long sk[kWarps][kPadCap];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int i = blockIdx.x * kWarps + w;
  if (i >= n) return;
  int cnt = 0;
  walk(i, NBR_WALK_ARGS, lane, [&](bool hit, unsigned long long key) {
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    const int slot = cnt + __popc(m & ((1u << lane) - 1u));
    if (hit && slot < kPadCap) sk[w][slot] = key;
    cnt += __popc(m);
  });
  __syncwarp();
  if (lane == 0) deg[i] = cnt;
  if (cnt > kPadCap) return;
  for (int k = lane; k < cnt; k += 32) {
    const unsigned long long key = sk[w][k];
    int rank = 0;
    for (int q = 0; q < cnt; ++q) rank += sk[w][q] < key;
    pad[static_cast<size_t>(i) * kPadCap + rank] = key;
  }
}

// CSR from the padded rows (rows over kPadCap: walk again, sort through tmp)
__global__ void __launch_bounds__(kWarps * 32) compact_kernel(int n, NBR_WALK_PARAMS, const int* __restrict__ row_ptr,
                                                              int max_edges, const unsigned long long* __restrict__ pad,
                                                              unsigned long long* __restrict__ tmp,
                                                              unsigned long long* __restrict__ skey,
                                                              int* __restrict__ col, int* __restrict__ shift) {
  JANUS_GDC_WAIT();
  __shared__ unsigned long long sk[kWarps][kSortCap];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int i = blockIdx.x * kWarps + w;
  if (i >= n || row_ptr[n] > max_edges) return;
  const int base = row_ptr[i], deg = row_ptr[i + 1] - base;
  if (deg <= kPadCap) {
    for (int k = lane; k < deg; k += 32) {
      const unsigned long long key = pad[static_cast<size_t>(i) * kPadCap + k];
      const int e = base + k;
      skey[e] = key;
      col[e] = static_cast<int>(key >> 24);
      shift[3 * e + 0] = static_cast<int>((key >> 16) & 0xff) - 128;
      shift[3 * e + 1] = static_cast<int>((key >> 8) & 0xff) - 128;
      shift[3 * e + 2] = static_cast<int>(key & 0xff) - 128;
    }
    return;
  }
  unsigned long long* buf = deg <= kSortCap ? sk[w] : tmp + base;
  int cnt = 0;  // warp-uniform running count
  walk(i, NBR_WALK_ARGS, lane, [&](bool hit, unsigned long long key) {
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (hit) buf[cnt + __popc(m & ((1u << lane) - 1u))] = key;
    cnt += __popc(m);
  });
  __syncwarp();
  emit_sorted(buf, deg, base, lane, skey, col, shift);
}

__global__ void __launch_bounds__(kWarps * 32) rev_kernel(int n, const int* __restrict__ row_ptr, int max_edges,
                                                          const unsigned long long* __restrict__ skey,
                                                          int* __restrict__ rev, int* __restrict__ err) {
  JANUS_GDC_WAIT();
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (i >= n || row_ptr[n] > max_edges) return;
  for (int e = row_ptr[i] + lane; e < row_ptr[i + 1]; e += 32) {
    const unsigned long long k = skey[e];
    const int j = static_cast<int>(k >> 24);
    const int sx = static_cast<int>((k >> 16) & 0xff) - 128, sy = static_cast<int>((k >> 8) & 0xff) - 128,
              sz = static_cast<int>(k & 0xff) - 128;
    const unsigned long long want = make_key(i, -sx, -sy, -sz);
    int lo = row_ptr[j], hi = row_ptr[j + 1];
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (skey[mid] < want) lo = mid + 1; else hi = mid;
    }
    if (lo < row_ptr[j + 1] && skey[lo] == want) {
      rev[e] = lo;
    } else {
      rev[e] = -1;
      atomicExch(err, 1);
    }
  }
}

// copy the CSR slice of one micro-batch out of a concatenated build:
// col -= atom0, rev -= edge0 (rows of a batch only reach atoms of its own
// structures, so the slice is self-contained)
__global__ void slice_kernel(int E, int atom0, int edge0, const int* __restrict__ col, const int* __restrict__ rev,
                             const int* __restrict__ shift, int* __restrict__ col_o, int* __restrict__ rev_o,
                             int* __restrict__ shift_o) {
  JANUS_GDC_WAIT();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  col_o[e] = col[edge0 + e] - atom0;
  rev_o[e] = rev[edge0 + e] - edge0;
  shift_o[3 * e + 0] = shift[3 * (edge0 + e) + 0];
  shift_o[3 * e + 1] = shift[3 * (edge0 + e) + 1];
  shift_o[3 * e + 2] = shift[3 * (edge0 + e) + 2];
}

}  // namespace nbr
}  // namespace janus

// ================================================================== host side
struct janus_nbrlist {
  int max_atoms = 0, max_struct = 0, max_edges = 0, device = 0;
  int cell_cap = 0;
  janus::nbr::StructMeta* meta = nullptr;  // device [max_struct]
  janus::nbr::StructMeta* h_meta = nullptr;  // pinned
  int *cell_count = nullptr, *cursor = nullptr, *cell_start = nullptr;
  int *cell_of = nullptr, *c_atom = nullptr, *deg = nullptr, *err = nullptr;
  int4 *cw = nullptr, *c_w = nullptr;
  double* c_pos = nullptr;
  unsigned long long *tmp = nullptr, *skey = nullptr, *pad = nullptr;  // pad: [atoms][kPadCap] sorted rows (walk_pad)
  int* h_small = nullptr;  // pinned: [0] = E, [1] = err
  bool pending = false;    // enqueued, not yet finished
};

namespace janus {

namespace {
template <typename T>
T* dev_alloc(size_t n) {
  void* p = nullptr;
  JANUS_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
  return static_cast<T*>(p);
}
int nblk(int n, int b) { return std::max(1, (n + b - 1) / b); }
}  // namespace

janus_nbrlist* nbrlist_create(int max_atoms, int max_struct, int max_edges, int device) {
  if (max_atoms < 1 || max_struct < 1 || max_edges < 0) throw domain_error("nbrlist: bad capacities");
  JANUS_CUDA(cudaSetDevice(device));
  auto* nl = new janus_nbrlist;
  nl->max_atoms = max_atoms;
  nl->max_struct = max_struct;
  nl->max_edges = max_edges;
  nl->device = device;
  try {
    nl->meta = dev_alloc<nbr::StructMeta>(max_struct);
    JANUS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&nl->h_meta), sizeof(nbr::StructMeta) * max_struct, 0));
    JANUS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&nl->h_small), sizeof(int) * 2, 0));
    nl->cell_of = dev_alloc<int>(max_atoms);
    nl->c_atom = dev_alloc<int>(max_atoms);
    nl->deg = dev_alloc<int>(max_atoms);
    nl->err = dev_alloc<int>(1);
    nl->cw = dev_alloc<int4>(max_atoms);
    nl->c_w = dev_alloc<int4>(max_atoms);
    nl->c_pos = dev_alloc<double>(3 * static_cast<size_t>(max_atoms));
    nl->tmp = dev_alloc<unsigned long long>(max_edges);
    nl->skey = dev_alloc<unsigned long long>(max_edges);
    nl->pad = dev_alloc<unsigned long long>(static_cast<size_t>(max_atoms) * nbr::kPadCap);
  } catch (...) {
    nbrlist_destroy(nl);
    throw;
  }
  return nl;
}

void nbrlist_destroy(janus_nbrlist* nl) {
  if (!nl) return;
  cudaSetDevice(nl->device);
  cudaDeviceSynchronize();
  for (void* p : {static_cast<void*>(nl->meta), static_cast<void*>(nl->cell_count), static_cast<void*>(nl->cursor),
                  static_cast<void*>(nl->cell_start), static_cast<void*>(nl->cell_of), static_cast<void*>(nl->c_atom),
                  static_cast<void*>(nl->deg), static_cast<void*>(nl->err), static_cast<void*>(nl->cw),
                  static_cast<void*>(nl->c_w), static_cast<void*>(nl->c_pos), static_cast<void*>(nl->tmp),
                  static_cast<void*>(nl->skey), static_cast<void*>(nl->pad)})
    if (p) cudaFree(p);
  if (nl->h_meta) cudaFreeHost(nl->h_meta);
  if (nl->h_small) cudaFreeHost(nl->h_small);
  delete nl;
}

void nbrlist_enqueue(janus_nbrlist* nl, int n, int n_struct, const double* pos, const int* struct_id,
                     const double* cell_host, double rc, int* row_ptr, int* col, int* shift, int* rev,
                     cudaStream_t s) {
  if (n < 1 || n > nl->max_atoms) throw domain_error("nbrlist: n_atoms exceeds capacity");
  if (n_struct < 1 || n_struct > nl->max_struct) throw domain_error("nbrlist: n_struct exceeds capacity");
  if (!(rc > 0)) throw domain_error("r_c must be > 0");
  JANUS_CUDA(cudaSetDevice(nl->device));
  // h_meta may still feed the previous run's copy until nbrlist_finish
  if (nl->pending) throw state_error("nbrlist: previous build not finished");
  int cells = 0;
  for (int x = 0; x < n_struct; ++x) {
    const double L = cell_host[x];
    if (!(L > 0) || !std::isfinite(L)) throw domain_error("nbrlist: box length must be > 0");
    const int nimg = static_cast<int>(std::ceil(rc / L));  // host.cpp: the image range it scans
    if (nimg > 127) throw domain_error("nbrlist: box too small for r_c (more than 127 images)");
    int nc = static_cast<int>(std::floor(nbr::kSub * L / (rc * (1.0 + 1e-6))));
    nc = std::min(std::max(nc, 1), 64);
    const double a = L / nc;
    // a >= r_c (1 + 1e-6) / kSub when nc >= 2 -> m = kSub; one cell: ceil(r_c / L) images (+ margin)
    const int m = nc >= 2 ? nbr::kSub : static_cast<int>(std::ceil(rc / a * (1.0 + 1e-9) + 1e-9));
    nl->h_meta[x] = nbr::StructMeta{L, nc, m, nimg, cells};
    cells += nc * nc * nc;
  }
  if (cells > nl->cell_cap) {
    cudaFree(nl->cell_count);
    cudaFree(nl->cursor);
    cudaFree(nl->cell_start);
    nl->cell_count = nl->cursor = nl->cell_start = nullptr;
    nl->cell_count = dev_alloc<int>(cells);
    nl->cursor = dev_alloc<int>(cells);
    nl->cell_start = dev_alloc<int>(cells + 1);
    nl->cell_cap = cells;
  }
  JANUS_CUDA(cudaMemcpyAsync(nl->meta, nl->h_meta, sizeof(nbr::StructMeta) * n_struct, cudaMemcpyHostToDevice, s));
  JANUS_CUDA(cudaMemsetAsync(nl->cell_count, 0, sizeof(int) * cells, s));
  JANUS_CUDA(cudaMemsetAsync(nl->cursor, 0, sizeof(int) * cells, s));
  JANUS_CUDA(cudaMemsetAsync(nl->err, 0, sizeof(int), s));
  const double rc2 = rc * rc;
  janus::pdl(nbr::bin_kernel, nblk(n, 256), 256, 0, s)(n, pos, struct_id, nl->meta, nl->cell_of, nl->cw, nl->cell_count);
  janus::pdl(nbr::scan_kernel, 1, 1024, 0, s)(cells, nl->cell_count, nl->cell_start);
  janus::pdl(nbr::scatter_kernel, nblk(n, 256), 256, 0, s)(n, pos, nl->cell_of, nl->cw, nl->cell_start, nl->cursor,
                                                    nl->c_atom, nl->c_pos, nl->c_w);
  const int rb = nblk(n, nbr::kWarps), rt = nbr::kWarps * 32;
#define NBR_ARGS pos, struct_id, nl->meta, nl->cell_of, nl->cw, nl->cell_start, nl->c_atom, nl->c_pos, nl->c_w, rc2
  janus::pdl(nbr::walk_pad_kernel, rb, rt, 0, s)(n, NBR_ARGS, nl->deg, nl->pad);
  janus::pdl(nbr::scan_kernel, 1, 1024, 0, s)(n, nl->deg, row_ptr);
  janus::pdl(nbr::compact_kernel, rb, rt, 0, s)(n, NBR_ARGS, row_ptr, nl->max_edges, nl->pad, nl->tmp, nl->skey, col, shift);
#undef NBR_ARGS
  janus::pdl(nbr::rev_kernel, rb, rt, 0, s)(n, row_ptr, nl->max_edges, nl->skey, rev, nl->err);
  JANUS_LAUNCH_CHECK("nbrlist");
  JANUS_CUDA(cudaMemcpyAsync(nl->h_small, row_ptr + n, sizeof(int), cudaMemcpyDeviceToHost, s));
  JANUS_CUDA(cudaMemcpyAsync(nl->h_small + 1, nl->err, sizeof(int), cudaMemcpyDeviceToHost, s));
  nl->pending = true;
}

int nbrlist_finish(janus_nbrlist* nl, cudaStream_t s) {
  JANUS_CUDA(cudaStreamSynchronize(s));
  nl->pending = false;
  const int E = nl->h_small[0];
  if (E > nl->max_edges) throw domain_error("neighbour list exceeds max_edges");
  if (nl->h_small[1]) throw state_error("neighbour list is not symmetric");
  return E;
}

}  // namespace janus

namespace janus {

LmBuilder::LmBuilder(int max_atoms, int max_struct, int max_edges, int device, int n_bufs)
    : max_atoms_(max_atoms), max_struct_(max_struct), max_edges_(max_edges), device_(device) {
  JANUS_CUDA(cudaSetDevice(device));
  try {
    nl_ = nbrlist_create(max_atoms, max_struct, max_edges, device);
    const size_t per = sizeof(int) * (static_cast<size_t>(max_atoms) + 1 + 5 * static_cast<size_t>(max_edges));
    for (int b = 0; b < n_bufs; ++b) {
      void* p = nullptr;
      JANUS_CUDA(cudaMalloc(&p, per));
      dev_.push_back(p);
      int* q = static_cast<int*>(p);
      DevCsr d;
      d.row_ptr = q;
      d.col = q + max_atoms + 1;
      d.rev = d.col + max_edges;
      d.shift = d.rev + max_edges;
      bufs_.push_back(d);
      cudaEvent_t e;
      JANUS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      done_.push_back(e);
    }
    void* p = nullptr;
    JANUS_CUDA(cudaMalloc(&p, sizeof(double) * 3 * max_atoms));
    dev_.push_back(p);
    d_pos_ = static_cast<double*>(p);
    JANUS_CUDA(cudaMalloc(&p, sizeof(int) * max_atoms));
    dev_.push_back(p);
    d_sid_ = static_cast<int*>(p);
    JANUS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h_in_), (sizeof(double) * 3 + sizeof(int)) * max_atoms, 0));
    JANUS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&hrow_), sizeof(int) * (max_atoms + 1), 0));
  } catch (...) {
    this->~LmBuilder();
    throw;
  }
}

LmBuilder::~LmBuilder() {
  cudaSetDevice(device_);
  cudaDeviceSynchronize();
  if (nl_) nbrlist_destroy(nl_);
  nl_ = nullptr;
  for (void* p : dev_) cudaFree(p);
  dev_.clear();
  for (cudaEvent_t e : done_) cudaEventDestroy(e);
  done_.clear();
  if (h_in_) cudaFreeHost(h_in_);
  if (hrow_) cudaFreeHost(hrow_);
  h_in_ = nullptr;
  hrow_ = nullptr;
}

int LmBuilder::build(const janus_host_batch* hbs, int nb, double rc, int b, cudaStream_t s) {
  if (b < 0 || b >= static_cast<int>(bufs_.size())) throw domain_error("LM buffer index out of range");
  if (nb < 1) throw domain_error("LM: no batches");
  // concatenate the micro-batches: structures are independent, so one build
  // over all of them is the per-batch builds side by side (atoms and structure
  // ids offset); slices are cut out again by csr_slice_copy
  int n = 0, ns = 0;
  atom0_.assign(static_cast<size_t>(nb) + 1, 0);
  for (int k = 0; k < nb; ++k) {
    const janus_host_batch& hb = hbs[k];
    if (hb.n_atoms < 1) throw domain_error("n_atoms must be >= 1");
    if (hb.n_struct < 1) throw domain_error("n_struct must be >= 1");
    if (!hb.pos || !hb.struct_id || !hb.cell) throw domain_error("batch without pos / struct_id / cell");
    n += hb.n_atoms;
    ns += hb.n_struct;
    atom0_[static_cast<size_t>(k) + 1] = n;
  }
  if (n > max_atoms_) throw domain_error("n_atoms exceeds stage capacity");
  if (ns > max_struct_) throw domain_error("n_struct exceeds stage capacity");
  JANUS_CUDA(cudaSetDevice(device_));
  // h_in_ / hrow_ are free: the previous build ended with a sync of its stream
  double* hp = reinterpret_cast<double*>(h_in_);
  int* hs = reinterpret_cast<int*>(h_in_ + sizeof(double) * 3 * max_atoms_);
  cell_.resize(static_cast<size_t>(ns));
  for (int k = 0, so = 0; k < nb; ++k) {
    const janus_host_batch& hb = hbs[k];
    const int a = atom0_[static_cast<size_t>(k)];
    std::memcpy(hp + 3 * static_cast<size_t>(a), hb.pos, sizeof(double) * 3 * hb.n_atoms);
    for (int i = 0; i < hb.n_atoms; ++i) {
      const int sid = hb.struct_id[i];
      if (sid < 0 || sid >= hb.n_struct) throw domain_error("struct_id out of range");
      hs[a + i] = so + sid;
    }
    std::memcpy(cell_.data() + so, hb.cell, sizeof(double) * hb.n_struct);
    so += hb.n_struct;
  }
  JANUS_CUDA(cudaMemcpyAsync(d_pos_, hp, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, s));
  JANUS_CUDA(cudaMemcpyAsync(d_sid_, hs, sizeof(int) * n, cudaMemcpyHostToDevice, s));
  JANUS_CUDA(cudaStreamWaitEvent(s, done_[static_cast<size_t>(b)], 0));  // last consumer of buffer b
  const DevCsr& d = bufs_[static_cast<size_t>(b)];
  nbrlist_enqueue(nl_, n, ns, d_pos_, d_sid_, cell_.data(), rc, d.row_ptr, d.col, d.shift, d.rev, s);
  JANUS_CUDA(cudaMemcpyAsync(hrow_, d.row_ptr, sizeof(int) * (n + 1), cudaMemcpyDeviceToHost, s));
  return nbrlist_finish(nl_, s);
}

void csr_slice_copy(const DevCsr& src, int atom0, int edge0, int E, int* col, int* rev, int* shift, cudaStream_t s) {
  if (E <= 0) return;
  janus::pdl(nbr::slice_kernel, nblk(E, 256), 256, 0, s)(E, atom0, edge0, src.col, src.rev, src.shift, col, rev, shift);
  JANUS_LAUNCH_CHECK("csr slice");
}

void LmBuilder::release(int b, cudaStream_t consumer) {
  JANUS_CUDA(cudaEventRecord(done_[static_cast<size_t>(b)], consumer));
}

}  // namespace janus
