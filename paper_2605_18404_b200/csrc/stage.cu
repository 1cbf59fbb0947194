// stage.cu — the four phases of one pipeline stage, as kernel sequences.
//
// Phase semantics per unit, in the stage's unit order:
//   FE  units ascending : carrier (h[,m]) up
//   FF  units descending: adjoint a = dE/d(carrier) down, force F accumulated
//   BF  units ascending : tangent abar = dL_F/da up, BF->BE injections kept
//                         on this device (Eq. 2 merged first-order routing,
//                         graph.hpp:151), second-order grads -> ledger g2
//   BE  units descending: adjoint b = dL/d(carrier) down, grads -> ledger g1
// Kernels: edge_kernels.cuh (msg unit), node_kernels.cuh (everything else).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <initializer_list>
#include <limits>
#include <stdexcept>
#include <utility>
#include <vector>

#include <cublas_v2.h>
#include <dlfcn.h>

#include "../../include/janus/errors.hpp"

#include "edge_kernels.cuh"
#include "edge_tc.cuh"
#include "pair_tc.cuh"

// fused upd kernels by micro-batch size (node_kernels.cuh upd_rows_per_cta)
#define JANUS_UPD(KERN, SMEM, S, ...)                                                                 \
  do {                                                                                               \
    if (node::upd_rows_per_cta(N) == node::kRB)                                                      \
      janus::pdl(node::KERN<node::kRB>, blocks(N, node::kRB), 16 * node::kRB, (SMEM), (S))(__VA_ARGS__);     \
    else                                                                                             \
      janus::pdl(node::KERN<node::kRBSmall>, blocks(N, node::kRBSmall), 16 * node::kRBSmall, (SMEM), (S))(__VA_ARGS__); \
  } while (0)

// row kernels (pair_tc.cuh) by the stage's gathers-in-flight setting
#define JANUS_ROWS(KERN, GRID, S, ...)                                          \
  do {                                                                          \
    if (st->rows_kf == 4)                                                       \
      janus::pdl(edge_tc::KERN<4>, (GRID), 256, 0, (S))(__VA_ARGS__);                   \
    else                                                                        \
      janus::pdl(edge_tc::KERN<8>, (GRID), 256, 0, (S))(__VA_ARGS__);                   \
  } while (0)
#include "node_kernels.cuh"
#include "wide.cuh"
#include "wgrad_tc.cuh"
#include "upd_tc.cuh"
#include "gemm_tc_host.hpp"
#ifndef JANUS_UPD_TC
#define JANUS_UPD_TC 1  // tf32 mode: upd units on tcgen05 (upd_tc.cuh); 0 = the SIMT kernels (A/B builds)
#endif
#include "stage.cuh"
#include "stage_api.hpp"
#include "nbrlist.hpp"

namespace janus {

int64_t unit_param_count(const janus_model_desc& m, int u) {
  const int64_t H = m.H, R = m.R, S = m.n_species;
  switch (unit_kind(u, m.L)) {
    case kEmbed: return S * H;
    case kReadout: return H * H + 2 * H + S;
    case kMsg: return R * H + H + H * H + H + H * H;
    default: return H * H + H + H * H;
  }
}

int64_t unit_param_offset(const janus_model_desc& m, int u) {
  int64_t o = 0;
  for (int x = 0; x < u; ++x) o += unit_param_count(m, x);
  return o;
}

namespace {

#define JANUS_BLAS(x)                                                                                   \
  do {                                                                                                  \
    const cublasStatus_t st_ = (x);                                                                     \
    if (st_ != CUBLAS_STATUS_SUCCESS) throw cuda_error(std::string(#x) + ": cuBLAS status " + std::to_string(static_cast<int>(st_))); \
  } while (0)

constexpr int kH = 64;
constexpr int kR = 64;
using EC = edge::Cfg<kH, kR>;

template <typename T>
T* dalloc(janus_stage* st, size_t n, bool count_static) {
  void* p = nullptr;
  const size_t bytes = std::max<size_t>(n, 1) * sizeof(T);
  JANUS_CUDA(cudaMalloc(&p, bytes));
  JANUS_CUDA(cudaMemset(p, 0, bytes));
  st->allocs.push_back(p);
  (count_static ? st->static_bytes : st->arena_bytes) += static_cast<int64_t>(bytes);
  return static_cast<T*>(p);
}

inline int blocks(int64_t n, int t) { return static_cast<int>((n + t - 1) / t); }

size_t geo_index(const janus_stage* st, int mb, int par) {
  return static_cast<size_t>(par) * static_cast<size_t>(st->desc.n_micro_batches) + static_cast<size_t>(mb);
}
DevGeo& geo_of(janus_stage* st, int mb) { return st->geo[geo_index(st, mb, st->gpar[static_cast<size_t>(mb)])]; }
const DevGeo& geo_of(const janus_stage* st, int mb) { return st->geo[geo_index(st, mb, st->gpar[static_cast<size_t>(mb)])]; }

// Attribution switch, compiled into profiling builds ONLY (`make PROFILE=1`;
// numerically invalid when set): JANUS_PROF_SKIP bitmask drops launches — 1
// FE, 2 FF, 4 BF, 8 BE tensor-core edge kernels, 16 wgrad_multi, 32 fused upd
// kernels, 64 gemm_rows, 128 reduce_partials — so the step-time drop measures
// each family's share of the concurrent step.  The product build is constant 0.
#ifdef JANUS_PROFILING
int prof_skip() {
  static const int v = [] {
    const char* e = std::getenv("JANUS_PROF_SKIP");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}
#else
constexpr int prof_skip() { return 0; }
#endif

template <typename Op = node::InId>
void gemm(cudaStream_t s, int rows, const float* X, const float* M, const float* bias, const float* add1,
          const float* add2, float* out, Op op = Op{}) {
  if (rows <= 0 || (prof_skip() & 64)) return;
  static const bool rows4 = std::getenv("JANUS_GEMM_ROWS4") != nullptr;  // A/B: the 4-rows-per-CTA kernel
  if (rows4)
    janus::pdl(node::gemm_rows_kernel<kH, Op>, blocks(rows, 256 / kH), 256, 0, s)(rows, X, M, bias, add1, add2, out, op);
  else if (rows >= 256)
    janus::pdl(node::gemm_rb_kernel<node::kRB, Op>, blocks(rows, node::kRB), 16 * node::kRB, node::upd_smem(1), s)(rows, X, M, bias, add1, add2, out, op);
  else
    janus::pdl(node::gemm_rb_kernel<node::kRBSmall, Op>, blocks(rows, node::kRBSmall), 16 * node::kRBSmall, node::upd_smem(1), s)(rows, X, M, bias, add1,
                                                                                                                 add2, out, op);
  JANUS_LAUNCH_CHECK("gemm_rows");
}

// G = sum_i op(a_i)^T b_i (+ a2_i^T b2_i) over atoms, optional column sums
// cs_out1 = sum_i x1_i, cs_out2 = sum_i x2_i — two deterministic stages.
struct Colsums {
  const float* x1 = nullptr;
  float* out1 = nullptr;
  const float* x2 = nullptr;
  float* out2 = nullptr;
};

template <typename Op = node::InId>
void wgrad(Scratch& sc, cudaStream_t s, int rows, const float* a, const float* b, const float* a2, const float* b2,
           float* G, Op op = Op{}, Colsums cs = {}) {
  const int chunks = blocks(rows, node::kWChunk);
  janus::pdl(node::wgrad_partial_kernel<kH, Op>, chunks, 256, 0, s)(rows, a, b, a2, b2, cs.x1, cs.x2, sc.wpart, op);
  janus::pdl(node::wgrad_final_kernel<kH>, blocks(kH * kH + 2 * kH, 256), 256, 0, s)(chunks, sc.wpart, G, cs.out1, cs.out2);
  JANUS_LAUNCH_CHECK("wgrad");
}

// Up to three weight-gradient jobs in one launch (last CTA reduces, fixed order).
node::WJob wjob(const float* a, const float* b, float* G, const float* a2 = nullptr, const float* b2 = nullptr,
                bool silu_a = false, const float* x1 = nullptr, float* cs1 = nullptr, const float* x2 = nullptr,
                float* cs2 = nullptr) {
  node::WJob j;
  j.a = a;
  j.b = b;
  j.a2 = a2;
  j.b2 = b2;
  j.x1 = x1;
  j.x2 = x2;
  j.G = G;
  j.cs1 = cs1;
  j.cs2 = cs2;
  j.silu_a = silu_a ? 1 : 0;
  return j;
}

bool use_tc(const janus_stage* st);

// Node weight gradients of one phase (up to 3 jobs per launch): tcgen05 in
// the tensor-core mode (wgrad_tc.cuh, one CTA per job), the output-partitioned
// SIMT kernel in the fp32 parity mode.
void wjobs(const janus_stage* st, Scratch& sc, cudaStream_t s, int rows, std::initializer_list<node::WJob> list) {
  if (prof_skip() & 16) return;
  node::WJobs J{};
  J.n = static_cast<int>(list.size());
  int k = 0;
  for (const auto& j : list) J.j[k++] = j;
  static const bool simt_only = std::getenv("JANUS_WGRAD_SIMT") != nullptr;  // comparison runs
  if (use_tc(st) && !simt_only) {
    bool cs = false;
    for (int q = 0; q < J.n; ++q) cs = cs || J.j[q].x1 || J.j[q].x2;
    janus::pdl(edge_tc::wgrad_tc_kernel, dim3(static_cast<unsigned>(J.n), cs ? 2u : 1u), edge_tc::kWgT, edge_tc::wgrad_tc_smem(), s)(rows, J);
  } else {
    const dim3 grid(9u, static_cast<unsigned>(J.n));  // 8 row blocks of the gradient + 1 column-sum block
    janus::pdl(node::wgrad_multi_kernel, grid, 256, 0, s)(rows, J, sc.wpart, sc.counter);
  }
  JANUS_LAUNCH_CHECK("wgrad");
}

// out[z][k] = sum_{Z_i = z} x[i][k]; x == null: out[z] = sum_{Z_i = z} eps[s(i)]
void species_sum(janus_stage* st, Scratch& sc, cudaStream_t s, const DevGeo& g, const float* x, const float* eps, float* out) {
  const int chunks = blocks(g.n_atoms, node::kWChunk), S = st->m.n_species;
  janus::pdl(node::species_sum_partial_kernel<kH>, chunks, 256, 0, s)(g.n_atoms, S, g.species, x, eps, g.struct_id, sc.wpart);
  janus::pdl(node::species_sum_final_kernel<kH>, blocks(S * kH, 256), 256, 0, s)(chunks, S, x ? kH : 1, sc.wpart, out);
  JANUS_LAUNCH_CHECK("species_sum");
}

void copy(cudaStream_t s, float* dst, const float* src, size_t n) {
  if (n) JANUS_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(float), cudaMemcpyDeviceToDevice, s));
}

EdgeGeom edge_geom(const DevGeo& g) {
  EdgeGeom e;
  e.n_atoms = g.n_atoms;
  e.n_edges = g.n_edges;
  e.n_tiles = g.n_tiles;
  e.row_ptr = g.row_ptr;
  e.col = g.col;
  e.src = g.src;
  e.rev = g.rev;
  e.tile_row = g.tile_row;
  e.d = g.d;
  e.u = g.u;
  e.c = g.c;
  e.dc = g.dc;
  return e;
}

MsgParams msg_params(const janus_stage* st, int u) {
  const int H = kH, R = kR;
  MsgParams p;
  p.A = st->P(u);
  p.alpha = p.A + R * H;
  p.B = p.alpha + H;
  p.beta = p.B + H * H;
  p.Bt = st->tw[static_cast<size_t>(u - st->u0)];
  p.pack = p.Bt + 2 * H * H;
  return p;
}

// transposed copies: msg [Bt|Wt], upd [Ut|Vt], readout [Ot]
void refresh_transposes(janus_stage* st, cudaStream_t s) {
  if (st->wide) {  // generic width: only the tf32 GEMMs' K-major weights (A^T, B^T) of msg units
    if (!st->wide_tc) return;
    const int H = st->m.H, R = st->m.R;
    for (int u = st->u0; u < st->u1; ++u) {
      if (unit_kind(u, st->m.L) != kMsg) continue;
      float* t = st->tw[static_cast<size_t>(u - st->u0)];
      const float* P = st->P(u);
      janus::pdl(wide::transpose_any_kernel, blocks(static_cast<int64_t>(R) * H, 256), 256, 0, s)(R, H, P, t);
      janus::pdl(wide::transpose_any_kernel, blocks(static_cast<int64_t>(H) * H, 256), 256, 0, s)(H, H, P + R * H + H, t + H * R);
    }
    JANUS_LAUNCH_CHECK("transpose_wide");
    return;
  }
  const int H = kH, R = kR;
  for (int u = st->u0; u < st->u1; ++u) {
    float* t = st->tw[static_cast<size_t>(u - st->u0)];
    const float* P = st->P(u);
    const int b = blocks(H * H, 256);
    switch (unit_kind(u, st->m.L)) {
      case kMsg:
        janus::pdl(node::transpose_kernel<kH>, b, 256, 0, s)(P + R * H + H, t);
        janus::pdl(node::transpose_kernel<kH>, b, 256, 0, s)(P + R * H + H + H * H + H, t + H * H);
        janus::pdl(edge_tc::pack_msg_weights, b, 256, 0, s)(P, P + R * H, P + R * H + H, P + R * H + H + H * H,
                                                     P + R * H + H + H * H + H, t + 2 * H * H);
        janus::pdl(upd_tc::pack_msg_w, b, 256, 0, s)(P + R * H + H + H * H + H, t + 2 * H * H);
        break;
      case kUpd:
        janus::pdl(node::transpose_kernel<kH>, b, 256, 0, s)(P, t);
        janus::pdl(node::transpose_kernel<kH>, b, 256, 0, s)(P + H * H + H, t + H * H);
        janus::pdl(upd_tc::pack_upd_weights, b, 256, 0, s)(P, P + H * H + H, t + 2 * H * H);
        break;
      case kReadout:
        janus::pdl(node::transpose_kernel<kH>, b, 256, 0, s)(P, t);
        break;
      default:
        break;
    }
  }
  JANUS_LAUNCH_CHECK("transpose");
}

// pointer into a port for the actual atom count n
float* port_h(const Port& p, int) { return p.buf; }
float* port_m(const Port& p, int n) { return p.buf + static_cast<size_t>(n) * p.H; }
float* port_v(const Port& p, int n) { return p.buf + static_cast<size_t>(n) * p.H * (p.has_m ? 2 : 1); }

const float* in_h(const janus_stage* st, const Slot& sl, int u, int n) {
  if (u == st->u0) return port_h(sl.ports[JANUS_PORT_ACT_IN], n);
  const int prev = u - 1;
  const UnitKind k = unit_kind(prev, st->m.L);
  if (k == kEmbed || k == kUpd) return sl.units[static_cast<size_t>(prev - st->u0)].out_h;
  return in_h(st, sl, prev, n);  // msg passes h through
}
const float* in_m(const janus_stage* st, const Slot& sl, int u, int n) {
  if (u == st->u0) return port_m(sl.ports[JANUS_PORT_ACT_IN], n);
  return sl.units[static_cast<size_t>(u - 1 - st->u0)].out_m;
}

float* ledger(janus_stage* st, float* base, int mb, int u) {
  return base + static_cast<size_t>(mb) * st->n_params + st->uoff[static_cast<size_t>(u - st->u0)];
}

bool use_tc(const janus_stage* st) { return st->m.precision == JANUS_PREC_TF32; }
// tf32 mode: the upd units (and unfused msg v / vdot) on tcgen05 from 128-atom
// micro-batches; below one full 128-row CTA the SIMT kernels' 16-row CTAs win
// the latency-bound chain (C1, 64-atom cells: 7100 vs 6630 structures/s;
// C2 17630 vs 18990).  A function of the micro-batch only, so every stage of
// a staged run picks the same kernels (bit-identical to unstaged).
bool upd_on_tc(const janus_stage* st, int N) { return use_tc(st) && JANUS_UPD_TC && N >= 128; }
// undirected edge-pair tables (pair_tc.cuh): the tensor-core H=64 kernels and the generic-width path
bool needs_pairs(const janus_stage* st) { return use_tc(st) || st->wide; }
// Tensor-core edge grids.  CTAs loop over tiles (static assignment), so a CTA
// may take several: its fixed costs (weight TMA, TMEM alloc, first dependent
// loads and, for BF/BE, the weight-gradient partial write-out and its share of
// the ordered reduction) are paid once per CTA.  Throughput runs (several
// lanes: the step is bound by SM-time) use tpc tiles per CTA; a latency-bound
// pipeline (1 lane) keeps one tile per CTA.
int tc_grid_tpc(const DevGeo& g, int tpc) { return std::max(1, std::min((g.n_tiles_tc + tpc - 1) / tpc, 148)); }
int tc_grid(const janus_stage* st, const DevGeo& g) { return tc_grid_tpc(g, st->tpc_wg); }
// BF / BE per pair: persistent CTAs, tpc_wg 128-pair chunks each
int pair_grid(const janus_stage* st, const DevGeo& g) {
  const int chunks = (g.n_pairs + edge_tc::TE - 1) / edge_tc::TE;
  return std::max(1, std::min((chunks + st->tpc_wg - 1) / st->tpc_wg, 148));
}
int fe_grid(const janus_stage* st, const DevGeo& g) {
  return std::max(1, (g.n_tiles_tc + st->tpc_fe - 1) / st->tpc_fe);
}

Scratch& lane_of(janus_stage* st, int lane) {
  if (lane < 0 || lane >= static_cast<int>(st->lanes.size())) throw domain_error("lane index out of range");
  return st->lanes[static_cast<size_t>(lane)];
}

void check_mb_slot(const janus_stage* st, int mb, int slot) {
  if (mb < 0 || mb >= st->desc.n_micro_batches) throw domain_error("micro-batch index out of range");
  if (slot < 0 || slot >= st->desc.n_slots) throw domain_error("slot index out of range");
  if (geo_of(st, mb).n_atoms <= 0) throw state_error("micro-batch not loaded (LM missing)");
}

}  // namespace

// ============================================================= creation
// upload block layout: capacity-sized fields, 256 B aligned
LoadLayout load_layout(const janus_stage_desc& d) {
  const size_t NA = static_cast<size_t>(d.max_atoms), NE = static_cast<size_t>(std::max(d.max_edges, 1));
  const size_t MS = static_cast<size_t>(d.max_struct);
  const size_t sz[LoadLayout::kN] = {
      4 * (NA + 1), 4 * NA, 4 * NA, 4 * (MS + 1), 4 * (NA + 1), 16 * NA, 8 * 3 * NA, 8 * MS, 4 * MS, 4 * 3 * NA,
      4 * NE,       4 * NE, 4 * 3 * NE};
  LoadLayout L;
  size_t o = 0;
  for (int k = 0; k < LoadLayout::kN; ++k) {
    L.off[k] = o;
    o += (sz[k] + 255) & ~static_cast<size_t>(255);
  }
  L.bytes = o;
  return L;
}

janus_stage* stage_create(const janus_stage_desc& d, const float* unit_params) {
  const janus_model_desc& m = d.model;
  const bool wide = d.kernels == 1 || m.H != kH || m.R != kR || m.precision == JANUS_PREC_FP32_EMU;
  if (d.kernels < 0 || d.kernels > 1) throw config_error("kernels must be 0 (auto) or 1 (generic width)");
  if (wide && m.H != 64 && m.H != 128 && m.H != 256)
    throw config_error("hidden width H must be 64, 128 or 256 (got H=" + std::to_string(m.H) + ")");
  if (wide && (m.R < 2 || m.R > 1024)) throw config_error("basis size R must be in [2, 1024]");
  if (m.L < 1 || m.n_species < 1 || m.n_species > 256) throw config_error("bad model shape");
  if (m.precision != JANUS_PREC_FP32 && m.precision != JANUS_PREC_TF32 && m.precision != JANUS_PREC_FP32_EMU)
    throw config_error("unknown precision");
  const int U = 2 * m.L + 2;
  if (d.unit_begin < 0 || d.unit_end > U || d.unit_begin >= d.unit_end) throw domain_error("bad unit range");
  if (d.max_atoms < 1 || d.max_edges < 0 || d.max_struct < 1 || d.n_micro_batches < 1 || d.n_slots < 1)
    throw domain_error("bad stage capacity");
  JANUS_CUDA(cudaSetDevice(d.device));
  auto* st = new janus_stage();
  try {
    st->desc = d;
    st->m = m;
    st->wide = wide;
#ifndef JANUS_WIDE_SPLIT3
#define JANUS_WIDE_SPLIT3 1  // plain fp32 generic path: per-pair GEMMs as 3xTF32 on gemm_tc (0: cuBLAS fp32 SIMT)
#endif
    st->wide_split3 = (JANUS_WIDE_SPLIT3 && wide && m.precision == JANUS_PREC_FP32) ? 1 : 0;
    st->wide_tc = wide && (m.precision == JANUS_PREC_TF32 || st->wide_split3);
    st->u0 = d.unit_begin;
    st->u1 = d.unit_end;
    st->U = U;
    st->has_embed = st->u0 == 0;
    st->has_readout = st->u1 == U;
    st->in_has_m = st->u0 > 0 && unit_kind(st->u0 - 1, m.L) == kMsg;
    st->out_has_m = st->u1 < U && unit_kind(st->u1 - 1, m.L) == kMsg;
    int64_t off = 0;
    for (int u = st->u0; u < st->u1; ++u) {
      st->uoff.push_back(off);
      off += unit_param_count(m, u);
    }
    st->n_params = off;
    const size_t NP = static_cast<size_t>(off), NMB = static_cast<size_t>(d.n_micro_batches);
    const size_t NA = static_cast<size_t>(d.max_atoms), NE = static_cast<size_t>(d.max_edges);
    const size_t NH = NA * static_cast<size_t>(m.H);
    st->params = dalloc<float>(st, NP, true);
    st->grad = dalloc<float>(st, NP, true);
    st->m1 = dalloc<float>(st, NP, true);
    st->m2 = dalloc<float>(st, NP, true);
    st->dstep = dalloc<int>(st, 1, true);
    st->dopt = dalloc<float>(st, 4, true);
    st->g1 = dalloc<float>(st, NP * NMB, true);
    st->g2 = dalloc<float>(st, NP * NMB, true);
    JANUS_CUDA(cudaMemcpy(st->params, unit_params, NP * sizeof(float), cudaMemcpyHostToDevice));
    for (int u = st->u0; u < st->u1; ++u) {
      const UnitKind k = unit_kind(u, m.L);
      // msg: [Bt | Wt | tensor-core pack]; upd: [Ut | Vt]; readout: [Ot]
      // + the tensor-core node images: msg [W | W_lo] after its pack, upd the 8-tile image (upd_tc.cuh)
      const size_t n = k == kMsg    ? 2 * kH * kH + upd_tc::kMsgPackBytes / sizeof(float)
                       : k == kUpd  ? 2 * kH * kH + upd_tc::kUpdPackBytes / sizeof(float)
                                    : static_cast<size_t>(kH) * kH;
      if (wide) {  // tf32: msg units keep [A^T (H x R) | B^T (H x H)] for the TMA-fed GEMMs
        const bool tcw = k == kMsg && st->wide_tc;  // (tf32, or the 3xTF32 fp32 path)
        st->tw.push_back(tcw ? dalloc<float>(st, static_cast<size_t>(m.H) * (m.R + m.H), true) : nullptr);
        continue;
      }
      st->tw.push_back(k == kEmbed ? nullptr : dalloc<float>(st, n, true));
    }
    // geometry per micro-batch
    st->geo.resize(2 * NMB);
    st->gpar.assign(NMB, 0);
    for (auto& g : st->geo) {
      st->lay = load_layout(d);
      const LoadLayout& L = st->lay;
      g.d_block = dalloc<uint8_t>(st, L.bytes, false);
      auto at = [&](int k) { return g.d_block + L.off[k]; };
      g.row_ptr = reinterpret_cast<int*>(at(LoadLayout::kRowPtr));
      g.col = reinterpret_cast<int*>(at(LoadLayout::kCol));
      g.rev = reinterpret_cast<int*>(at(LoadLayout::kRev));
      g.shift = reinterpret_cast<int*>(at(LoadLayout::kShift));
      g.species = reinterpret_cast<int*>(at(LoadLayout::kSpecies));
      g.struct_id = reinterpret_cast<int*>(at(LoadLayout::kStructId));
      g.struct_ptr = reinterpret_cast<int*>(at(LoadLayout::kStructPtr));
      g.tile_row = reinterpret_cast<int*>(at(LoadLayout::kTileRow));
      g.tile_tc = reinterpret_cast<int4*>(at(LoadLayout::kTileTc));
      g.pos = reinterpret_cast<double*>(at(LoadLayout::kPos));
      g.cell = reinterpret_cast<double*>(at(LoadLayout::kCell));
      g.E_target = reinterpret_cast<float*>(at(LoadLayout::kETarget));
      g.F_target = reinterpret_cast<float*>(at(LoadLayout::kFTarget));
      for (int par = 0; par < 2; ++par) {
        void* hp = nullptr;
        JANUS_CUDA(cudaHostAlloc(&hp, L.bytes, cudaHostAllocDefault));
        std::memset(hp, 0, L.bytes);
        st->host_allocs.push_back(hp);
        g.h_pin[par] = static_cast<uint8_t*>(hp);
      }
      g.src = dalloc<int>(st, NE, false);
      g.d = dalloc<float>(st, NE, false);
      g.u = dalloc<float>(st, 3 * NE, false);
      g.c = dalloc<float>(st, NE, false);
      g.dc = dalloc<float>(st, NE, false);
      g.pidx = dalloc<int>(st, NE, false);
      g.pcanon = dalloc<int>(st, NE / 2 + 1, false);
      g.pgeo = dalloc<float4>(st, 2 * (NE / 2 + 1), false);
    }
    // activation slot pool (the executor sizes it by the schedule's in-flight
    // micro-batches, include/janus/slots.hpp)
    const int64_t arena0 = st->arena_bytes;
    st->slots.resize(static_cast<size_t>(d.n_slots));
    for (auto& sl : st->slots) {
      sl.units.resize(static_cast<size_t>(st->u1 - st->u0));
      for (int u = st->u0; u < st->u1; ++u) {
        UnitBufs& b = sl.units[static_cast<size_t>(u - st->u0)];
        switch (unit_kind(u, m.L)) {
          case kEmbed: b.out_h = dalloc<float>(st, NH, false); break;
          case kMsg:
            b.out_m = dalloc<float>(st, NH, false);
            b.v = dalloc<float>(st, NH, false);
            b.ff_a = dalloc<float>(st, NH, false);
            b.ff_Y = dalloc<float>(st, NH, false);
            b.inj = dalloc<float>(st, NH, false);
            if (m.precision == JANUS_PREC_TF32 || wide) {
              b.wf = dalloc<float>(st, (NE / 2 + 1) * m.H, false);
              b.wfp = dalloc<float>(st, (NE / 2 + 1) * m.H, false);
            }
            break;
          case kUpd:
            b.out_h = dalloc<float>(st, NH, false);
            b.p = dalloc<float>(st, NH, false);
            b.ff_a = dalloc<float>(st, NH, false);
            b.inj = dalloc<float>(st, NH, false);
            break;
          case kReadout:
            b.p = dalloc<float>(st, NH, false);
            b.inj = dalloc<float>(st, NH, false);
            break;
        }
      }
      const bool in_b = st->u0 > 0, out_b = st->u1 < U;
      for (int p = 0; p < 8; ++p) {
        const bool at_input = (p == JANUS_PORT_ACT_IN || p == JANUS_PORT_ADJ_OUT || p == JANUS_PORT_TAN_IN || p == JANUS_PORT_BADJ_OUT);
        if (at_input ? !in_b : !out_b) continue;
        Port& port = sl.ports[p];
        port.has_m = at_input ? st->in_has_m : st->out_has_m;
        port.has_vec = (p >= JANUS_PORT_ADJ_IN && p <= JANUS_PORT_TAN_OUT);
        port.H = m.H;
        port.buf = dalloc<float>(st, NH * (port.has_m ? 2 : 1) + (port.has_vec ? 3 * NA : 0), false);
      }
    }
    st->pool_bytes = st->arena_bytes - arena0;
    st->outs.resize(NMB);
    for (MbOut& mo : st->outs) {
      mo.F = dalloc<float>(st, 3 * NA, false);
      mo.Fbar = dalloc<float>(st, 3 * NA, false);
      mo.e_atom = dalloc<float>(st, NA, false);
      mo.E = dalloc<float>(st, static_cast<size_t>(d.max_struct), false);
      mo.eps = dalloc<float>(st, static_cast<size_t>(d.max_struct), false);
    }
    st->losses = dalloc<float>(st, 2 * NMB, false);
    st->pair_chunks_cap = static_cast<int>((NE + 1023) / 1024) + 1;
    st->pair_counts = dalloc<int>(st, static_cast<size_t>(node::kMaxGeoJobs) * st->pair_chunks_cap, false);
    for (size_t x = 0; x < NMB; ++x) st->outs[x].loss = st->losses + 2 * x;
    st->lanes.resize(static_cast<size_t>(std::max(1, d.n_lanes)));
    // measured on the C2 bench (16 lanes): 128-edge tiles 1/1 -> 4735, 4/8 -> 5765;
    // multi-chunk tiles (~2 chunks) 2/4 -> 6363, 2/3 -> 6467 structures/s
    // FE / FF run two CTAs per SM: one tile per CTA once every micro-batch has
    // its own lane (32 lanes: 1 -> 7760 vs 2 -> 7648; 16 lanes: 2 -> 7089 vs 1 -> 7066)
    st->tpc_fe = d.n_lanes >= 32 ? 1 : std::max(1, std::min(2, d.n_lanes / 8));
    st->tpc_wg = std::max(1, std::min(3, d.n_lanes / 5));
    // pair mode at 32 lanes (one hardware queue per lane): 3 filter chunks and
    // 5 BF / BE pair chunks per CTA (C2: 15182 -> 15527-15548 structures/s)
    st->tpc_filter = d.n_lanes >= 32 ? 3 : st->tpc_fe;
    if (d.n_lanes >= 32) st->tpc_wg = 5;
    // tensor-core tiles: runs of <= 8 rows with <= tc_tile_edges edges, cut into
    // 128-edge chunks (rows may straddle chunk boundaries: the segmented sums
    // and force sums carry across the chunks of a tile)
    st->tc_tile_edges = 0;  // 0: best-fill tiles (stage_load); > 0: greedy runs of <= that many edges (tuning)
    if (const char* e = std::getenv("JANUS_TC_TILE_EDGES")) st->tc_tile_edges = std::max(0, std::atoi(e));
    if (const char* e = std::getenv("JANUS_TC_TILE_MAXCH")) st->tc_tile_max_chunks = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("JANUS_TC_TILE_OVH")) st->tc_tile_ovh = std::atof(e);
    if (const char* e = std::getenv("JANUS_TPC_FE")) st->tpc_fe = st->tpc_filter = std::max(1, std::atoi(e));  // tuning runs only
    if (const char* e = std::getenv("JANUS_TPC_WG")) st->tpc_wg = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("JANUS_FEFF_PAIR")) st->pair_feff = std::atoi(e) != 0;  // A/B runs only
    st->pair_bfbe = st->pair_feff;
    if (const char* e = std::getenv("JANUS_ROWS_KF")) st->rows_kf = std::atoi(e) == 4 ? 4 : 8;
    if (const char* e = std::getenv("JANUS_BFBE_PAIR")) st->pair_bfbe = st->pair_feff && std::atoi(e) != 0;
    for (Scratch& sc : st->lanes) {
      sc.wh = dalloc<float>(st, NH, false);
      sc.wh2 = dalloc<float>(st, NH, false);
      sc.wm = dalloc<float>(st, NH, false);
      sc.s1 = dalloc<float>(st, NH, false);
      sc.s2 = dalloc<float>(st, NH, false);
      sc.s3 = dalloc<float>(st, NH, false);
      sc.s4 = dalloc<float>(st, NH, false);
      sc.s5 = dalloc<float>(st, NH, false);
      if (wide) {  // per-pair operand stacks + this lane's cuBLAS handle (fixed workspace: graph-capture safe)
        const size_t P2 = NE + 2;
        sc.phi2 = dalloc<float>(st, P2 * static_cast<size_t>(m.R), false);
        sc.z2 = dalloc<float>(st, P2 * static_cast<size_t>(m.H), false);
        sc.a2 = dalloc<float>(st, P2 * static_cast<size_t>(m.H), false);
        sc.b2 = dalloc<float>(st, P2 * static_cast<size_t>(m.H), false);
        sc.cspart = dalloc<float>(st, static_cast<size_t>(wide::kColChunks) * m.H, false);
        sc.cstick = dalloc<unsigned>(st, static_cast<size_t>(m.H / 32), false);  // dalloc zeroes
        sc.wslices = dalloc<float>(st, (P2 / 2048 + 2) * static_cast<size_t>(std::max(m.H, m.R)) * m.H, false);
        constexpr size_t kWs = 32u << 20;
        sc.blas_ws = dalloc<uint8_t>(st, kWs, false);
        cublasHandle_t h = nullptr;
        JANUS_BLAS(cublasCreate(&h));
        sc.blas = h;
        JANUS_BLAS(cublasSetWorkspace(h, sc.blas_ws, kWs));
        JANUS_BLAS(cublasSetPointerMode(h, CUBLAS_POINTER_MODE_HOST));
        if (st->wide_tc) {  // tensor maps of the lane's operand stacks (capacity rows; OOB rows read as zero)
          auto put = [](TMap& d, const CUtensorMap& m) { std::memcpy(d.bytes, &m, sizeof(m)); };
          const int rows = static_cast<int>(P2);
          put(sc.tm_phi2_pair, gemm_tc::make_tmap(sc.phi2, rows, m.R, 16));
          put(sc.tm_phi2_plain, gemm_tc::make_tmap(sc.phi2, rows, m.R, 128));
          put(sc.tm_a2_pair, gemm_tc::make_tmap(sc.a2, rows, m.H, 16));
          put(sc.tm_b2_pair, gemm_tc::make_tmap(sc.b2, rows, m.H, 16));
          put(sc.tm_b2_plain, gemm_tc::make_tmap(sc.b2, rows, m.H, 128));
        }
        if (m.precision == JANUS_PREC_FP32_EMU) {
          // cuBLAS >= 12.9 only; resolved at run time, since a host that loads
          // an older libcublas first (e.g. torch's bundled 12.8) must still load us
          using SetEmu = cublasStatus_t (*)(cublasHandle_t, cublasEmulationStrategy_t);
          auto fn = reinterpret_cast<SetEmu>(dlsym(RTLD_DEFAULT, "cublasSetEmulationStrategy"));
          if (!fn) throw config_error("JANUS_PREC_FP32_EMU needs cuBLAS >= 12.9 (BF16x9 emulation)");
          JANUS_BLAS(fn(h, CUBLAS_EMULATION_STRATEGY_EAGER));
        }
        continue;
      }
      sc.partial = dalloc<float>(st, NA * static_cast<size_t>(EC::PE), false);
      const size_t chunks = (NA + node::kWChunk - 1) / node::kWChunk;
      sc.wpart = dalloc<float>(st, 3 * chunks * std::max<size_t>(kH * kH + 2 * kH, static_cast<size_t>(m.n_species) * kH), false);
      sc.counter = dalloc<unsigned>(st, 1, false);
    }
    JANUS_CUDA(cudaFuncSetAttribute(edge_tc::wgrad_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)edge_tc::wgrad_tc_smem()));
    JANUS_CUDA(cudaFuncSetAttribute(edge::msg_fe_kernel<kH, kR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)edge::fe_smem<kH, kR>()));
    JANUS_CUDA(cudaFuncSetAttribute(edge::msg_ff_kernel<kH, kR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)edge::ff_smem<kH, kR>()));
    JANUS_CUDA(cudaFuncSetAttribute(edge::msg_bf_kernel<kH, kR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)edge::bf_smem<kH, kR>()));
    JANUS_CUDA(cudaFuncSetAttribute(edge::msg_be_kernel<kH, kR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)edge::be_smem<kH, kR>()));
    JANUS_CUDA(cudaFuncSetAttribute(node::upd_bf_fused<node::kRB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)node::upd_smem(5)));
    JANUS_CUDA(cudaFuncSetAttribute(node::upd_fe_fused<node::kRB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)node::upd_smem(3)));
    JANUS_CUDA(cudaFuncSetAttribute(node::upd_bf_fused<node::kRBSmall>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)node::upd_smem(5)));
    JANUS_CUDA(cudaFuncSetAttribute(node::upd_fe_fused<node::kRBSmall>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)node::upd_smem(3)));
    JANUS_CUDA(cudaFuncSetAttribute(edge_tc::msg_fe_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)edge_tc::fe_smem()));
    JANUS_CUDA(cudaFuncSetAttribute(edge_tc::msg_ff_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)edge_tc::ff_smem()));
    JANUS_CUDA(cudaFuncSetAttribute(edge_tc::msg_filter_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)edge_tc::filter_smem()));
    JANUS_CUDA(cudaFuncSetAttribute(edge_tc::msg_bf_pair_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)edge_tc::bf_pair_smem()));
    JANUS_CUDA(cudaFuncSetAttribute(edge_tc::msg_be_pair_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)edge_tc::be_pair_smem()));
    JANUS_CUDA(cudaFuncSetAttribute(edge_tc::msg_bf_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)edge_tc::bf_smem()));
    JANUS_CUDA(cudaFuncSetAttribute(edge_tc::msg_be_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)edge_tc::be_smem()));
    JANUS_CUDA(cudaFuncSetAttribute(upd_tc::upd_fe_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)upd_tc::upd_tc_smem(6, 2)));
    JANUS_CUDA(cudaFuncSetAttribute(upd_tc::upd_ff_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)upd_tc::upd_tc_smem(4, 2)));
    JANUS_CUDA(cudaFuncSetAttribute(upd_tc::upd_bf_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)upd_tc::upd_tc_smem(5, 2)));
    JANUS_CUDA(cudaFuncSetAttribute(upd_tc::upd_be_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)upd_tc::upd_tc_smem(2, 1)));
    JANUS_CUDA(cudaFuncSetAttribute(upd_tc::rows_w_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)upd_tc::upd_tc_smem(2, 2)));
    if (st->wide_tc) {  // weight maps: A^T and B^T (transposed copies) and B itself, per msg unit
      st->tm_w.resize(3 * static_cast<size_t>(st->u1 - st->u0));
      for (int u = st->u0; u < st->u1; ++u) {
        if (unit_kind(u, m.L) != kMsg) continue;
        const float* t = st->tw[static_cast<size_t>(u - st->u0)];
        const float* B = st->P(u) + m.R * m.H + m.H;
        TMap* w = &st->tm_w[3 * static_cast<size_t>(u - st->u0)];
        const CUtensorMap at = gemm_tc::make_tmap(t, m.H, m.R, m.H), bt = gemm_tc::make_tmap(t + m.H * m.R, m.H, m.H, m.H),
                          bb = gemm_tc::make_tmap(B, m.H, m.H, m.H);
        std::memcpy(w[0].bytes, &at, sizeof(at));
        std::memcpy(w[1].bytes, &bt, sizeof(bt));
        std::memcpy(w[2].bytes, &bb, sizeof(bb));
      }
    }
    refresh_transposes(st, nullptr);
    JANUS_CUDA(cudaDeviceSynchronize());
  } catch (...) {
    for (auto& sc : st->lanes)
      if (sc.blas) cublasDestroy(static_cast<cublasHandle_t>(sc.blas));
    for (void* p : st->allocs) cudaFree(p);
    for (void* p : st->host_allocs) cudaFreeHost(p);
    delete st;
    throw;
  }
  return st;
}

void stage_destroy(janus_stage* st) {
  if (!st) return;
  cudaSetDevice(st->desc.device);
  cudaDeviceSynchronize();
  delete st->lm;
  for (auto& sc : st->lanes)
    if (sc.blas) cublasDestroy(static_cast<cublasHandle_t>(sc.blas));
  for (void* p : st->allocs) cudaFree(p);
  for (void* p : st->host_allocs) cudaFreeHost(p);
  delete st;
}

size_t port_elems(const janus_stage* st, int port, int n) {
  const Port& p = st->slots[0].ports[port];
  if (!p.buf) return 0;
  return static_cast<size_t>(n) * p.H * (p.has_m ? 2 : 1) + (p.has_vec ? 3 * static_cast<size_t>(n) : 0);
}

// ================================================================== LM
// Edge-pair tables of the jobs' micro-batches (pair_tc.cuh): chunk counts, then ranks
void launch_pairs(janus_stage* st, const node::GeoJobs& J, int max_edges_job, cudaStream_t s) {
  const int chunks = (max_edges_job + 1023) / 1024;
  if (chunks <= 0) return;
  const dim3 grid(static_cast<unsigned>(chunks), static_cast<unsigned>(J.n));
  janus::pdl(edge_tc::pairs_count_kernel, grid, 1024, 0, s)(J, st->pair_counts, st->pair_chunks_cap);
  janus::pdl(edge_tc::pairs_kernel, grid, 1024, 0, s)(J, st->pair_counts, st->pair_chunks_cap);
  JANUS_LAUNCH_CHECK("pairs");
}

void stage_load(janus_stage* st, int mb, const janus_host_batch& hb, cudaStream_t s, bool sync,
                const DevCsrSlice* dcsr, std::vector<node::GeoJob>* defer, int par) {
  if (mb < 0 || mb >= st->desc.n_micro_batches) throw domain_error("micro-batch index out of range");
  if (!hb.row_ptr && !dcsr) {  // no neighbour list in the batch: build it on the device (nbrlist.cu)
    if (!st->lm) st->lm = new LmBuilder(st->desc.max_atoms, st->desc.max_struct, st->desc.max_edges, st->desc.device, 1);
    janus_host_batch hb2 = hb;
    hb2.n_edges = st->lm->build(&hb, 1, static_cast<double>(st->m.r_c), 0, s);
    hb2.row_ptr = st->lm->host_row_ptr();
    const DevCsrSlice sl{&st->lm->buf(0), 0, 0};
    stage_load(st, mb, hb2, s, sync, &sl, nullptr, par);
    st->lm->release(0, s);
    return;
  }
  if (par < 0) par = st->gpar[static_cast<size_t>(mb)];
  if (hb.n_atoms < 1 || hb.n_atoms > st->desc.max_atoms) throw domain_error("n_atoms exceeds stage capacity");
  if (hb.n_edges < 0 || hb.n_edges > st->desc.max_edges) throw domain_error("n_edges exceeds stage capacity");
  if (hb.n_struct < 1 || hb.n_struct > st->desc.max_struct) throw domain_error("n_struct exceeds stage capacity");
  JANUS_CUDA(cudaSetDevice(st->desc.device));
  DevGeo& g = st->geo[geo_index(st, mb, par)];
  const int N = hb.n_atoms, E = hb.n_edges;
  // host-side row tiles (<= 8 rows and <= te edges, or one long row) and struct offsets
  auto build_tiles = [&](int te) {
    std::vector<int> tiles{0};
    int rows = 0, edges = 0;
    for (int i = 0; i < N; ++i) {
      const int deg = hb.row_ptr[i + 1] - hb.row_ptr[i];
      if (rows > 0 && (rows == edge::kRowsPerTile || edges + deg > te)) {
        tiles.push_back(i);
        rows = 0;
        edges = 0;
      }
      ++rows;
      edges += deg;
    }
    tiles.push_back(N);
    return tiles;
  };
  // Tensor-core tiles: runs of <= 8 rows cut into 128-edge chunks (rows may
  // straddle chunk boundaries; the segmented and force sums carry across a
  // tile's chunks).  A chunk costs the same whatever its fill (a thread per
  // edge row) and a tile adds a fixed epilogue (row sums, row GEMM), so each
  // tile takes the run of 1..8 rows (<= max_chunks chunks; a longer single
  // row alone) minimising (chunks + ovh) / edges, ties to the longer run.
  auto build_tiles_cost = [&](int max_chunks, double ovh) {
    std::vector<int> tiles{0};
    for (int i = 0; i < N;) {
      int best_k = 1, e = 0;
      double best = std::numeric_limits<double>::infinity();
      for (int k = 1; k <= edge_tc::kRowsPerTile && i + k <= N; ++k) {
        e += hb.row_ptr[i + k] - hb.row_ptr[i + k - 1];
        const int chunks = (e + edge_tc::TE - 1) / edge_tc::TE;
        if (k > 1 && chunks > max_chunks) break;
        const double cost = e > 0 ? (chunks + ovh) / e : std::numeric_limits<double>::max();
        if (cost <= best * (1.0 + 1e-12)) {
          best = cost;
          best_k = k;
        }
      }
      i += best_k;
      tiles.push_back(i);
    }
    return tiles;
  };
  DevGeo& gg = g;
  gg.h_tiles = build_tiles(edge::TE);
  // up to 2 chunks per tile at ~50 neighbours, 4 in dense cells (measured:
  // C2 2 -> 6456 vs 3 -> 6070 structures/s; C5 2 -> 204 vs 4 -> 240)
  // one lane (a latency-bound pipeline stage issuing one kernel at a time):
  // single-chunk tiles, the most CTAs per launch
  const int max_chunks = st->tc_tile_max_chunks > 0 ? st->tc_tile_max_chunks
                         : st->desc.n_lanes <= 1   ? 1
                                                   : (E >= 80 * N ? 4 : 2);
  gg.h_tiles_tc = st->tc_tile_edges > 0 ? build_tiles(st->tc_tile_edges) : build_tiles_cost(max_chunks, st->tc_tile_ovh);
  const std::vector<int>& tiles = gg.h_tiles;
  const std::vector<int>& tiles_tc = gg.h_tiles_tc;
  std::vector<int>& sptr = gg.h_sptr;
  sptr.assign(static_cast<size_t>(hb.n_struct) + 1, 0);
  for (int i = 0; i < N; ++i) {
    const int sid = hb.struct_id[i];
    if (sid < 0 || sid >= hb.n_struct || (i > 0 && sid < hb.struct_id[i - 1])) throw domain_error("struct_id must be non-decreasing in [0, n_struct)");
    sptr[static_cast<size_t>(sid) + 1] = i + 1;
  }
  for (int x = 1; x <= hb.n_struct; ++x) sptr[static_cast<size_t>(x)] = std::max(sptr[static_cast<size_t>(x)], sptr[static_cast<size_t>(x) - 1]);
  if (hb.row_ptr[0] != 0 || hb.row_ptr[N] != E) throw domain_error("row_ptr inconsistent with n_edges");
  g.n_atoms = N;
  g.n_edges = E;
  g.n_struct = hb.n_struct;
  g.n_tiles = static_cast<int>(tiles.size()) - 1;
  g.n_tiles_tc = static_cast<int>(tiles_tc.size()) - 1;
  if (needs_pairs(st) && E % 2) throw domain_error("odd edge count: every edge needs a distinct reverse edge");
  if (needs_pairs(st) && !dcsr)  // host CSR: the pair tables need rev to be a fixed-point-free involution
    for (int e = 0; e < E; ++e) {
      const int r = hb.rev[e];
      if (r < 0 || r >= E || r == e || hb.rev[r] != e) throw domain_error("rev must pair every edge with a distinct reverse edge");
    }
  g.n_pairs = E / 2;
  // one pinned image per load (alternating halves: the other may still feed
  // a queued copy), one host->device copy
  const LoadLayout& L = st->lay;
  uint8_t* hp = g.h_pin[g.h_par];
  g.h_par ^= 1;
  auto put = [&](int k, const void* src, size_t bytes) {
    if (bytes) std::memcpy(hp + L.off[k], src, bytes);
  };
  put(LoadLayout::kRowPtr, hb.row_ptr, sizeof(int) * (N + 1));
  if (!dcsr) {
    put(LoadLayout::kCol, hb.col, sizeof(int) * E);
    put(LoadLayout::kRev, hb.rev, sizeof(int) * E);
    put(LoadLayout::kShift, hb.shift, sizeof(int) * 3 * E);
  }
  put(LoadLayout::kSpecies, hb.species, sizeof(int) * N);
  put(LoadLayout::kStructId, hb.struct_id, sizeof(int) * N);
  put(LoadLayout::kStructPtr, sptr.data(), sizeof(int) * sptr.size());
  put(LoadLayout::kTileRow, tiles.data(), sizeof(int) * tiles.size());
  {
    int* t4 = reinterpret_cast<int*>(hp + L.off[LoadLayout::kTileTc]);  // edge ranges resolved on the host
    for (int t = 0; t < g.n_tiles_tc; ++t) {
      t4[4 * t] = tiles_tc[t];
      t4[4 * t + 1] = tiles_tc[t + 1];
      t4[4 * t + 2] = hb.row_ptr[tiles_tc[t]];
      t4[4 * t + 3] = hb.row_ptr[tiles_tc[t + 1]];
    }
  }
  put(LoadLayout::kPos, hb.pos, sizeof(double) * 3 * N);
  put(LoadLayout::kCell, hb.cell, sizeof(double) * hb.n_struct);
  put(LoadLayout::kETarget, hb.E_target, sizeof(float) * hb.n_struct);
  put(LoadLayout::kFTarget, hb.F_target, sizeof(float) * 3 * N);
  const size_t extent = L.off[LoadLayout::kFTarget] + sizeof(float) * 3 * N;
  JANUS_CUDA(cudaMemcpyAsync(g.d_block, hp, extent, cudaMemcpyHostToDevice, s));
  if (!dcsr && E > 0) {  // host-built CSR: col | rev | shift (capacity gaps between them included)
    const size_t a = L.off[LoadLayout::kCol], b = L.off[LoadLayout::kShift] + sizeof(int) * 3 * E;
    JANUS_CUDA(cudaMemcpyAsync(g.d_block + a, hp + a, b - a, cudaMemcpyHostToDevice, s));
  }
  if (defer) {  // batched load: slice + geometry of all its micro-batches in one launch (stage_geometry_flush)
    if (E > 0) {
      node::GeoJob j{};
      j.n_atoms = N;
      j.n_edges = E;
      j.row_ptr = g.row_ptr;
      j.col = g.col;
      j.rev = g.rev;
      j.shift = g.shift;
      if (dcsr) {
        j.scol = dcsr->csr->col;
        j.srev = dcsr->csr->rev;
        j.sshift = dcsr->csr->shift;
        j.atom0 = dcsr->atom0;
        j.edge0 = dcsr->edge0;
      }
      j.pos = g.pos;
      j.struct_id = g.struct_id;
      j.cell = g.cell;
      j.src = g.src;
      j.d = g.d;
      j.u = g.u;
      j.c = g.c;
      j.dc = g.dc;
      j.pcanon = g.pcanon;
      j.pgeo = g.pgeo;
      j.pidx = g.pidx;
      defer->push_back(j);
    }
    return;
  }
  if (dcsr)  // the device-built CSR replaces the (unused) host regions of the block
    csr_slice_copy(*dcsr->csr, dcsr->atom0, dcsr->edge0, E, g.col, g.rev, g.shift, s);
  if (E > 0)
    janus::pdl(node::geometry_kernel, blocks(E, 256), 256, 0, s)(N, E, g.row_ptr, g.col, g.shift, g.pos, g.struct_id, g.cell,
                                                         static_cast<double>(st->m.r_c), g.src, g.d, g.u, g.c, g.dc);
  if (E > 0 && needs_pairs(st)) {
    node::GeoJobs J{};
    J.n = 1;
    J.j[0].n_edges = E;
    J.j[0].rev = g.rev;
    J.j[0].pcanon = g.pcanon;
    J.j[0].pgeo = g.pgeo;
    J.j[0].src = g.src;
    J.j[0].col = g.col;
    J.j[0].d = g.d;
    J.j[0].u = g.u;
    J.j[0].c = g.c;
    J.j[0].dc = g.dc;
    J.j[0].pidx = g.pidx;
    launch_pairs(st, J, E, s);
  }
  JANUS_LAUNCH_CHECK("geometry");
  // host arrays of the caller must stay valid until the stream reaches the
  // copies (pageable sources are staged by the driver before return)
  if (sync) JANUS_CUDA(cudaStreamSynchronize(s));
}

void stage_set_parity(janus_stage* st, int mb, int par) {
  if (mb < 0 || mb >= st->desc.n_micro_batches || par < 0 || par > 1) throw domain_error("bad geometry parity");
  st->gpar[static_cast<size_t>(mb)] = par;
}
const DevGeo& stage_geo(const janus_stage* st, int mb, int par) { return st->geo[geo_index(st, mb, par)]; }

void stage_geometry_flush(janus_stage* st, std::vector<node::GeoJob>& jobs, cudaStream_t s) {
  for (size_t b = 0; b < jobs.size(); b += node::kMaxGeoJobs) {
    node::GeoJobs J{};
    J.n = static_cast<int>(std::min<size_t>(node::kMaxGeoJobs, jobs.size() - b));
    J.rc = static_cast<double>(st->m.r_c);
    int base = 0;
    for (int k = 0; k < J.n; ++k) {
      J.j[k] = jobs[b + static_cast<size_t>(k)];
      J.j[k].edge_base = base;
      base += J.j[k].n_edges;
    }
    J.total_edges = base;
    if (base > 0) janus::pdl(node::geometry_batched_kernel, blocks(base, 256), 256, 0, s)(J);
    if (base > 0 && needs_pairs(st)) {
      int emax = 0;
      for (int k = 0; k < J.n; ++k) emax = std::max(emax, J.j[k].n_edges);
      launch_pairs(st, J, emax, s);
    }
    JANUS_LAUNCH_CHECK("geometry_batched");
  }
  jobs.clear();
}

// Filters w, w' of the stage's msg units (u_only < 0: all of them) for the
// slot's micro-batch, one launch (pair_tc.cuh msg_filter_tc).
void launch_filter(janus_stage* st, const DevGeo& g, Slot& sl, int u_only, cudaStream_t s, int grid_x = 0) {
  edge_tc::FilterJobs J{};
  for (int u = st->u0; u < st->u1; ++u) {
    if (unit_kind(u, st->m.L) != kMsg || (u_only >= 0 && u != u_only)) continue;
    if (J.n == edge_tc::kMaxFilterUnits) throw config_error("too many msg units on one stage for the filter launch");
    UnitBufs& b = sl.units[static_cast<size_t>(u - st->u0)];
    J.pack[J.n] = msg_params(st, u).pack;
    J.w[J.n] = b.wf;
    J.wp[J.n] = b.wfp;
    ++J.n;
  }
  if (J.n == 0 || g.n_pairs == 0) return;
  const int chunks = (g.n_pairs + edge_tc::TE - 1) / edge_tc::TE;
  const int gx = grid_x > 0 ? std::min(grid_x, chunks) : std::max(1, std::min(chunks, (chunks + st->tpc_filter - 1) / st->tpc_filter));
  janus::pdl(edge_tc::msg_filter_tc, dim3(gx, J.n), edge_tc::NT, edge_tc::filter_smem(), s)(edge_geom(g), g.pgeo, g.n_pairs, J,
                                                                                     st->m.r_c);
  JANUS_LAUNCH_CHECK("msg_filter_tc");
}

#include "stage_wide.inc"

// ================================================================== FE
void stage_fe(janus_stage* st, int mb, int slot, cudaStream_t s, int lane) {
  check_mb_slot(st, mb, slot);
  if (st->wide) return wide_fe(st, mb, slot, s, lane);
  Scratch& sc = lane_of(st, lane);
  const DevGeo& g = geo_of(st, mb);
  Slot& sl = st->slots[static_cast<size_t>(slot)];
  MbOut& mo = st->outs[static_cast<size_t>(mb)];
  sl.mb = mb;
  const int N = g.n_atoms, H = kH, R = kR, L = st->m.L;
  const EdgeGeom eg = edge_geom(g);
  const float* cur_h = st->u0 > 0 ? port_h(sl.ports[JANUS_PORT_ACT_IN], N) : nullptr;
  const float* cur_m = st->in_has_m ? port_m(sl.ports[JANUS_PORT_ACT_IN], N) : nullptr;
  const bool pairs = use_tc(st) && st->pair_feff;
  bool v_ready = false;  // the upd kernel before a msg unit already wrote its v
  if (pairs && g.n_pairs > 0 && !(prof_skip() & 1)) launch_filter(st, g, sl, -1, s);  // w, w' of every msg unit
  for (int u = st->u0; u < st->u1; ++u) {
    UnitBufs& b = sl.units[static_cast<size_t>(u - st->u0)];
    const float* P = st->P(u);
    switch (unit_kind(u, L)) {
      case kEmbed:
        janus::pdl(node::embed_fe_kernel<kH>, blocks(N * H, 256), 256, 0, s)(N, g.species, P, b.out_h);
        cur_h = b.out_h;
        break;
      case kMsg: {
        const float* W = P + R * H + H + H * H + H;
        if (v_ready) {
        } else if (upd_on_tc(st, N)) {  // the fused next-v product's bits (upd_tc.cuh rows_w_tc)
          janus::pdl(upd_tc::rows_w_tc, blocks(N, 128), edge_tc::NT, upd_tc::upd_tc_smem(2, 2), s)(N, cur_h, msg_params(st, u).pack,
                                                                                         1, b.v);
        } else {
          gemm(s, N, cur_h, W, nullptr, nullptr, nullptr, b.v);
        }
        v_ready = false;
        if (pairs) {
          if (!(prof_skip() & 1))
            JANUS_ROWS(msg_fe_rows, blocks(N, 8), s, N, g.row_ptr, g.col, g.pidx, b.wf, b.v, b.out_m);
        } else if (g.n_tiles > 0 && use_tc(st)) {
          if (!(prof_skip() & 1)) janus::pdl(edge_tc::msg_fe_tc, fe_grid(st, g), edge_tc::NT, edge_tc::fe_smem(), s)(eg, g.tile_tc, g.n_tiles_tc, msg_params(st, u),
                                                                                 st->m.r_c, b.v, b.out_m);
        } else if (g.n_tiles > 0)
          janus::pdl(edge::msg_fe_kernel<kH, kR>, g.n_tiles, edge::NT, edge::fe_smem<kH, kR>(), s)(eg, msg_params(st, u), st->m.r_c, b.v, b.out_m);
        cur_m = b.out_m;
        break;
      }
      case kUpd: {
        const float *Um = P, *ups = P + H * H, *V = P + H * H + H;
        // the next msg unit's v = h' W computed in the same kernel
        const bool fuse = u + 1 < st->u1 && unit_kind(u + 1, L) == kMsg;
        const float* Wn = fuse ? st->P(u + 1) + R * H + H + H * H + H : nullptr;
        float* vn = fuse ? sl.units[static_cast<size_t>(u + 1 - st->u0)].v : nullptr;
        if (prof_skip() & 32) {
        } else if (upd_on_tc(st, N)) {  // upd_tc.cuh: 128 atoms per CTA, 3xTF32 tcgen05 chain
          const float* T = st->tw[static_cast<size_t>(u - st->u0)];
          janus::pdl(upd_tc::upd_fe_tc, blocks(N, 128), edge_tc::NT, upd_tc::upd_tc_smem(6, 2), s)(
              N, cur_m, cur_h, T + 2 * H * H, ups, b.p, b.out_h, fuse ? msg_params(st, u + 1).pack : nullptr, vn);
        } else {
          JANUS_UPD(upd_fe_fused, node::upd_smem(fuse ? 3 : 2), s, N, cur_m, cur_h, Um, ups, V, b.p, b.out_h, Wn, vn);
        }
        v_ready = fuse;
        cur_h = b.out_h;
        cur_m = nullptr;
        break;
      }
      case kReadout: {
        const float *O = P, *o = P + H * H, *om = P + H * H + H, *bias = P + H * H + 2 * H;
        gemm(s, N, cur_h, O, o, nullptr, nullptr, b.p);
        janus::pdl(node::readout_energy_kernel<kH>, blocks(N, 8), 256, 0, s)(N, b.p, om, bias, g.species, mo.e_atom);
        janus::pdl(node::energy_loss_kernel, 1, 128, 0, s)(g.n_struct, g.struct_ptr, mo.e_atom, g.E_target, st->m.w_E, mo.E,
                                                   mo.eps, mo.loss);
        break;
      }
    }
    JANUS_LAUNCH_CHECK("stage_fe");
  }
  if (st->u1 < st->U) {
    const Port& out = sl.ports[JANUS_PORT_ACT_OUT];
    copy(s, port_h(out, N), cur_h, static_cast<size_t>(N) * H);
    if (out.has_m) copy(s, port_m(out, N), cur_m, static_cast<size_t>(N) * H);
  }
}

// ================================================================== FF
void stage_ff(janus_stage* st, int mb, int slot, cudaStream_t s, int lane) {
  check_mb_slot(st, mb, slot);
  if (st->wide) return wide_ff(st, mb, slot, s, lane);
  Scratch& sc = lane_of(st, lane);
  const DevGeo& g = geo_of(st, mb);
  Slot& sl = st->slots[static_cast<size_t>(slot)];
  MbOut& mo = st->outs[static_cast<size_t>(mb)];
  const int N = g.n_atoms, H = kH, R = kR, L = st->m.L;
  const size_t NH = static_cast<size_t>(N) * H;
  const EdgeGeom eg = edge_geom(g);
  float* wh = sc.wh;
  float* wm = sc.wm;
  if (st->has_readout) {
    JANUS_CUDA(cudaMemsetAsync(mo.F, 0, sizeof(float) * 3 * N, s));
  } else {
    const Port& in = sl.ports[JANUS_PORT_ADJ_IN];
    copy(s, wh, port_h(in, N), NH);
    if (in.has_m) copy(s, wm, port_m(in, N), NH);
    copy(s, mo.F, port_v(in, N), 3 * static_cast<size_t>(N));
  }
  for (int u = st->u1 - 1; u >= st->u0; --u) {
    UnitBufs& b = sl.units[static_cast<size_t>(u - st->u0)];
    const float* P = st->P(u);
    const float* T = st->tw[static_cast<size_t>(u - st->u0)];
    switch (unit_kind(u, L)) {
      case kReadout: {  // a_h = (SiLU'(t) omega) O^T
        const float* om = P + H * H + H;
        gemm(s, N, b.p, T, nullptr, nullptr, nullptr, wh, node::InDsiluOmega{om});
        break;
      }
      case kUpd: {  // ff_a = a'; a_m = ((a' V^T) SiLU'(p)) U^T, written straight into the
                    // preceding msg unit's saved FF input when it is on this stage
        float* am_dst = (u - 1 >= st->u0) ? sl.units[static_cast<size_t>(u - 1 - st->u0)].ff_a : wm;
        if (prof_skip() & 32) {
        } else if (upd_on_tc(st, N)) {
          janus::pdl(upd_tc::upd_ff_tc, blocks(N, 128), edge_tc::NT, upd_tc::upd_tc_smem(4, 2), s)(N, wh, b.p, T + 2 * H * H, b.ff_a,
                                                                                         am_dst);
        } else {
          JANUS_UPD(upd_ff_fused, node::upd_smem(2), s, N, wh, b.p, T + H * H, T, b.ff_a, am_dst);
        }
        break;
      }
      case kMsg: {
        if (u == st->u1 - 1) copy(s, b.ff_a, wm, NH);  // a_m arrived through the ADJ_IN port
        if (use_tc(st) && st->pair_feff) {  // a_h += Y W^T fused into the row kernel
          if (!(prof_skip() & 2))
            JANUS_ROWS(msg_ff_rows, blocks(N, 8), s, N, g.row_ptr, g.col, g.pidx, g.u, b.wf, b.wfp, b.v, b.ff_a,
                                                               msg_params(st, u).pack + edge_tc::kWtOff / sizeof(float),
                                                               b.ff_Y, mo.F, wh);
        } else if (g.n_tiles > 0 && use_tc(st)) {  // a_h += Y W^T fused into the tile epilogue
          if (!(prof_skip() & 2)) janus::pdl(edge_tc::msg_ff_tc, fe_grid(st, g), edge_tc::NT, edge_tc::ff_smem(), s)(eg, g.tile_tc, g.n_tiles_tc, msg_params(st, u),
                                                                                 st->m.r_c, b.v, b.ff_a, b.ff_Y, mo.F, wh);
        } else {
          if (g.n_tiles > 0)
            janus::pdl(edge::msg_ff_kernel<kH, kR>, g.n_tiles, edge::NT, edge::ff_smem<kH, kR>(), s)(eg, msg_params(st, u), st->m.r_c, b.v, b.ff_a, b.ff_Y, mo.F);
          else
            JANUS_CUDA(cudaMemsetAsync(b.ff_Y, 0, sizeof(float) * NH, s));
          gemm(s, N, b.ff_Y, T + H * H, nullptr, wh, nullptr, wh);  // a_h += Y W^T
        }
        break;
      }
      case kEmbed:
        break;
    }
    JANUS_LAUNCH_CHECK("stage_ff");
    (void)R;
  }
  if (st->u0 > 0) {
    const Port& out = sl.ports[JANUS_PORT_ADJ_OUT];
    copy(s, port_h(out, N), wh, NH);
    if (out.has_m) copy(s, port_m(out, N), wm, NH);
    copy(s, port_v(out, N), mo.F, 3 * static_cast<size_t>(N));
  } else {  // forces complete on stage 0: L_F seed
    janus::pdl(node::force_loss_kernel, 1, 1024, 0, s)(3 * N, mo.F, g.F_target, st->m.w_F, mo.Fbar, mo.loss + 1);
    JANUS_LAUNCH_CHECK("force_loss");
  }
}

// ================================================================== BF
void stage_bf(janus_stage* st, int mb, int slot, cudaStream_t s, int lane) {
  check_mb_slot(st, mb, slot);
  if (st->wide) return wide_bf(st, mb, slot, s, lane);
  Scratch& sc = lane_of(st, lane);
  const DevGeo& g = geo_of(st, mb);
  Slot& sl = st->slots[static_cast<size_t>(slot)];
  MbOut& mo = st->outs[static_cast<size_t>(mb)];
  const int N = g.n_atoms, H = kH, R = kR, L = st->m.L;
  const size_t NH = static_cast<size_t>(N) * H;
  const EdgeGeom eg = edge_geom(g);
  float* ah = sc.wh;
  float* am = sc.wm;
  const float* Fbar = mo.Fbar;
  JANUS_CUDA(cudaMemsetAsync(st->g2 + static_cast<size_t>(mb) * st->n_params, 0, sizeof(float) * st->n_params, s));
  if (st->u0 == 0) {
    JANUS_CUDA(cudaMemsetAsync(ah, 0, sizeof(float) * NH, s));
  } else {
    const Port& in = sl.ports[JANUS_PORT_TAN_IN];
    copy(s, ah, port_h(in, N), NH);
    if (in.has_m) copy(s, am, port_m(in, N), NH);
    Fbar = port_v(in, N);
  }
  // a_h ping-pongs between wh and wh2 at every upd unit, so a msg unit's
  // weight-gradient job (which reads a_h at msg time) can wait for the next
  // upd unit's launch
  float* ah_alt = sc.wh2;
  node::WJob pend{};
  bool has_pend = false;
  auto flush = [&] {
    if (has_pend) wjobs(st, sc, s, N, {pend});
    has_pend = false;
  };
  bool vdot_ready = false;  // the upd kernel before a msg unit already wrote its vdot
  for (int u = st->u0; u < st->u1; ++u) {
    UnitBufs& b = sl.units[static_cast<size_t>(u - st->u0)];
    const float* P = st->P(u);
    const float* T = st->tw[static_cast<size_t>(u - st->u0)];
    float* G2 = ledger(st, st->g2, mb, u);
    switch (unit_kind(u, L)) {
      case kEmbed:
        flush();
        break;
      case kMsg: {
        const float* W = P + R * H + H + H * H + H;
        if (vdot_ready) {
        } else if (upd_on_tc(st, N)) {  // vdot with the fused product's bits
          janus::pdl(upd_tc::rows_w_tc, blocks(N, 128), edge_tc::NT, upd_tc::upd_tc_smem(2, 2), s)(N, ah, msg_params(st, u).pack,
                                                                                         0, sc.s1);
        } else {
          gemm(s, N, ah, W, nullptr, nullptr, nullptr, sc.s1);  // vdot
        }
        vdot_ready = false;
        const bool pairs = use_tc(st) && st->pair_bfbe;
        if (pairs) {  // weight gradients once per pair + row sums from the stored filters (+ hbar^F = X W^T)
          const int grid = pair_grid(st, g);
          const MsgParams mp = msg_params(st, u);
          if (g.n_pairs > 0 && !(prof_skip() & 4)) {
            janus::pdl(edge_tc::msg_bf_pair_tc, grid, edge_tc::NT, edge_tc::bf_pair_smem(), s)(eg, g.pgeo, g.n_pairs, mp, st->m.r_c, b.v,
                                                                                       sc.s1, b.ff_a, Fbar, sc.partial);
            JANUS_LAUNCH_CHECK("msg_bf_pair_tc");
          }
          edge_tc::PartialReduce red;  // the partials' reduction rides in the row kernel's launch
          if (g.n_pairs > 0 && !(prof_skip() & 128)) red = {sc.partial, grid, G2};
          if (!(prof_skip() & 4))
            JANUS_ROWS(msg_bf_rows, blocks(N, 8) + edge_tc::reduce_blocks(red), s, N, g.row_ptr, g.col, g.pidx, g.u, Fbar, b.wf,
                       b.wfp, b.v, sc.s1, b.ff_a, mp.pack + edge_tc::kWtOff / sizeof(float), am, sc.s2, b.inj, red);
          else if (red.G)
            edge::reduce_partials(sc.partial, grid, EC::PE, G2, s);
        } else if (g.n_tiles > 0 && use_tc(st)) {
          const int grid = tc_grid(st, g);
          if (!(prof_skip() & 4)) janus::pdl(edge_tc::msg_bf_tc, grid, edge_tc::NT, edge_tc::bf_smem(), s)(eg, g.tile_tc, g.n_tiles_tc, msg_params(st, u),
                                                                          st->m.r_c, b.v, sc.s1, b.ff_a, Fbar, am, sc.s2,
                                                                          sc.partial, b.inj);  // + hbar^F = X W^T
          JANUS_LAUNCH_CHECK("msg_bf_tc");
          if (!(prof_skip() & 128)) edge::reduce_partials(sc.partial, grid, EC::PE, G2, s);
        } else if (g.n_tiles > 0) {
          janus::pdl(edge::msg_bf_kernel<kH, kR>, g.n_tiles, edge::NT, edge::bf_smem<kH, kR>(), s)(
              eg, msg_params(st, u), st->m.r_c, b.v, sc.s1, b.ff_a, Fbar, am, sc.s2, sc.partial);
          JANUS_LAUNCH_CHECK("msg_bf");
          janus::pdl(edge::reduce_partials_kernel, edge::reduce_grid(EC::PE), 256, 0, s)(sc.partial, g.n_tiles, EC::PE, G2);
        } else {
          JANUS_CUDA(cudaMemsetAsync(am, 0, sizeof(float) * NH, s));
          JANUS_CUDA(cudaMemsetAsync(sc.s2, 0, sizeof(float) * NH, s));
        }
        if (!pairs && !(g.n_tiles > 0 && use_tc(st))) gemm(s, N, sc.s2, T + H * H, nullptr, nullptr, nullptr, b.inj);  // hbar^F = X W^T
        flush();
        pend = wjob(in_h(st, sl, u, N), sc.s2, G2 + EC::PE, ah, b.ff_Y);  // dW2 = h^T X + abar^T Y (with the next upd's jobs)
        has_pend = true;
        break;
      }
      case kUpd: {
        const float *Um = P, *V = P + H * H + H;
        float *dU = G2, *dups = G2 + H * H, *dV = G2 + H * H + H;
        // pdot, r, pbar (s3), pdbar (s4), u (s5), mbar^F = pbar U^T, abar' = abar_h + u V
        // + the next msg unit's vdot = abar_h' W in the same kernel
        const bool fuse = u + 1 < st->u1 && unit_kind(u + 1, L) == kMsg;
        const float* Wn = fuse ? st->P(u + 1) + R * H + H + H * H + H : nullptr;
        if (prof_skip() & 32) {
        } else if (upd_on_tc(st, N)) {
          janus::pdl(upd_tc::upd_bf_tc, blocks(N, 128), edge_tc::NT, upd_tc::upd_tc_smem(5, 2), s)(
              N, am, b.ff_a, b.p, T + 2 * H * H, sc.s3, sc.s4, sc.s5, b.inj, ah, ah_alt,
              fuse ? msg_params(st, u + 1).pack : nullptr, fuse ? sc.s1 : nullptr);
        } else {
          JANUS_UPD(upd_bf_fused, node::upd_smem(fuse ? 5 : 4), s, N, am, b.ff_a, b.p, Um, T + H * H, T, V, sc.s3, sc.s4,
                    sc.s5, b.inj, ah, ah_alt, Wn, fuse ? sc.s1 : nullptr);
        }
        vdot_ready = fuse;
        std::swap(ah, ah_alt);
        const node::WJob jv = wjob(sc.s5, b.ff_a, dV);                                       // dV2 = u^T a'
        const node::WJob ju = wjob(in_m(st, sl, u, N), sc.s3, dU, am, sc.s4, false, sc.s3, dups);  // dU2, dups2
        if (has_pend)
          wjobs(st, sc, s, N, {pend, jv, ju});
        else
          wjobs(st, sc, s, N, {jv, ju});
        has_pend = false;
        break;
      }
      case kReadout: {
        flush();  // (its kernels rewrite s2)
        const float *O = P, *om = P + H * H + H;
        float *dO = G2, *dob = G2 + H * H, *dom = G2 + H * H + H;
        gemm(s, N, ah, O, nullptr, nullptr, nullptr, sc.s1);  // tdot
        janus::pdl(node::ro_bf_ew_kernel<kH>, blocks(NH, 256), 256, 0, s)(static_cast<int>(NH), sc.s1, b.p, om, sc.s2,
                                                                  sc.s3, sc.s4);
        gemm(s, N, sc.s2, T, nullptr, nullptr, nullptr, b.inj);  // hbar^F = tau O^T
        wjobs(st, sc, s, N, {wjob(ah, sc.s4, dO, in_h(st, sl, u, N), sc.s2, false, sc.s3, dom, sc.s2, dob)});
        break;
      }
    }
    JANUS_LAUNCH_CHECK("stage_bf");
  }
  flush();
  if (st->u1 < st->U) {
    const Port& out = sl.ports[JANUS_PORT_TAN_OUT];
    copy(s, port_h(out, N), ah, NH);
    if (out.has_m) copy(s, port_m(out, N), am, NH);
    copy(s, port_v(out, N), Fbar, 3 * static_cast<size_t>(N));
  }
}

// ================================================================== BE
void stage_be(janus_stage* st, int mb, int slot, cudaStream_t s, bool inj_only, int lane) {
  check_mb_slot(st, mb, slot);
  if (st->wide) return wide_be(st, mb, slot, s, inj_only, lane);
  Scratch& sc = lane_of(st, lane);
  const DevGeo& g = geo_of(st, mb);
  Slot& sl = st->slots[static_cast<size_t>(slot)];
  MbOut& mo = st->outs[static_cast<size_t>(mb)];
  const int N = g.n_atoms, H = kH, R = kR, L = st->m.L;
  const size_t NH = static_cast<size_t>(N) * H;
  const EdgeGeom eg = edge_geom(g);
  float* bh = sc.wh;
  float* bm = sc.wm;
  JANUS_CUDA(cudaMemsetAsync(st->g1 + static_cast<size_t>(mb) * st->n_params, 0, sizeof(float) * st->n_params, s));
  if (inj_only) {
    // 1F1B-2nd force replica: propagate only the BF->BE injections (b_out = 0,
    // no L_E seed); the energy device adds the result at its block input.
    JANUS_CUDA(cudaMemsetAsync(bh, 0, sizeof(float) * NH, s));
    JANUS_CUDA(cudaMemsetAsync(bm, 0, sizeof(float) * NH, s));
  } else if (!st->has_readout) {
    const Port& in = sl.ports[JANUS_PORT_BADJ_IN];
    copy(s, bh, port_h(in, N), NH);
    if (in.has_m) copy(s, bm, port_m(in, N), NH);
  }
  // a msg unit's dW1 job waits for the next (upd) unit's launch: its inputs
  // (in_h, Yb in s1) are not touched by upd_be_fused, so one launch serves both
  node::WJob pend{};
  bool has_pend = false;
  auto flush = [&] {
    if (has_pend) wjobs(st, sc, s, N, {pend});
    has_pend = false;
  };
  for (int u = st->u1 - 1; u >= st->u0; --u) {
    UnitBufs& b = sl.units[static_cast<size_t>(u - st->u0)];
    const float* P = st->P(u);
    const float* T = st->tw[static_cast<size_t>(u - st->u0)];
    float* G1 = ledger(st, st->g1, mb, u);
    switch (unit_kind(u, L)) {
      case kReadout: {
        if (inj_only) {  // no energy seed: b_h = hbar^F, readout first-order grads are zero
          copy(s, bh, b.inj, NH);
          break;
        }
        const float* om = P + H * H + H;
        float *dO = G1, *dob = G1 + H * H, *dom = G1 + H * H + H, *dbias = G1 + H * H + 2 * H;
        janus::pdl(node::ro_be_ew_kernel<kH>, blocks(NH, 256), 256, 0, s)(static_cast<int>(NH), b.p, om, mo.eps, g.struct_id,
                                                                  sc.s1, sc.s2);
        gemm(s, N, sc.s1, T, nullptr, b.inj, nullptr, bh);  // b_h = tbar O^T + hbar^F
        wjobs(st, sc, s, N, {wjob(in_h(st, sl, u, N), sc.s1, dO, nullptr, nullptr, false, sc.s1, dob, sc.s2, dom)});
        species_sum(st, sc, s, g, nullptr, mo.eps, dbias);
        break;
      }
      case kUpd: {
        float *dU = G1, *dups = G1 + H * H, *dV = G1 + H * H + H;
        // pbar (s2) = (b' V^T) SiLU'(p); b_m = pbar U^T + mbar^F
        if (prof_skip() & 32) {
        } else if (upd_on_tc(st, N)) {
          janus::pdl(upd_tc::upd_be_tc, blocks(N, 128), edge_tc::NT, upd_tc::upd_tc_smem(2, 1), s)(N, bh, b.p, T + 2 * H * H, b.inj,
                                                                                          sc.s2, bm);
        } else {
          JANUS_UPD(upd_be_fused, node::upd_smem(2), s, N, bh, b.p, T + H * H, T, b.inj, sc.s2, bm);
        }
        const node::WJob jv = wjob(b.p, bh, dV, nullptr, nullptr, true);                           // dV1 = SiLU(p)^T b'
        const node::WJob ju = wjob(in_m(st, sl, u, N), sc.s2, dU, nullptr, nullptr, false, sc.s2, dups);  // dU1, dups1
        if (has_pend)
          wjobs(st, sc, s, N, {pend, jv, ju});
        else
          wjobs(st, sc, s, N, {jv, ju});
        has_pend = false;
        break;
      }
      case kMsg: {
        const bool pairs = use_tc(st) && st->pair_bfbe;
        if (pairs) {
          const int grid = pair_grid(st, g);
          const MsgParams mp = msg_params(st, u);
          if (g.n_pairs > 0 && !(prof_skip() & 8)) {
            janus::pdl(edge_tc::msg_be_pair_tc, grid, edge_tc::NT, edge_tc::be_pair_smem(), s)(eg, g.pgeo, g.n_pairs, mp, st->m.r_c, b.v, bm,
                                                                                       sc.partial);
            JANUS_LAUNCH_CHECK("msg_be_pair_tc");
          }
          edge_tc::PartialReduce red;  // the partials' reduction rides in the row kernel's launch
          if (g.n_pairs > 0 && !(prof_skip() & 128)) red = {sc.partial, grid, G1};
          if (!(prof_skip() & 8))  // Yb; b_h += Yb W^T + hbar^F
            JANUS_ROWS(msg_be_rows, blocks(N, 8) + edge_tc::reduce_blocks(red), s, N, g.row_ptr, g.col, g.pidx, b.wf, bm,
                       mp.pack + edge_tc::kWtOff / sizeof(float), sc.s1, b.inj, bh, red);
          else if (red.G)
            edge::reduce_partials(sc.partial, grid, EC::PE, G1, s);
        } else if (g.n_tiles > 0 && use_tc(st)) {
          const int grid = tc_grid(st, g);
          if (!(prof_skip() & 8)) janus::pdl(edge_tc::msg_be_tc, grid, edge_tc::NT, edge_tc::be_smem(), s)(eg, g.tile_tc, g.n_tiles_tc, msg_params(st, u),
                                                                          st->m.r_c, b.v, bm, sc.s1, sc.partial,
                                                                          b.inj, bh);  // + b_h += Yb W^T + hbar^F
          JANUS_LAUNCH_CHECK("msg_be_tc");
          if (!(prof_skip() & 128)) edge::reduce_partials(sc.partial, grid, EC::PE, G1, s);
        } else if (g.n_tiles > 0) {
          janus::pdl(edge::msg_be_kernel<kH, kR>, g.n_tiles, edge::NT, edge::be_smem<kH, kR>(), s)(
              eg, msg_params(st, u), st->m.r_c, b.v, bm, sc.s1, sc.partial);
          JANUS_LAUNCH_CHECK("msg_be");
          janus::pdl(edge::reduce_partials_kernel, edge::reduce_grid(EC::PE), 256, 0, s)(sc.partial, g.n_tiles, EC::PE, G1);
        } else {
          JANUS_CUDA(cudaMemsetAsync(sc.s1, 0, sizeof(float) * NH, s));
        }
        flush();
        pend = wjob(in_h(st, sl, u, N), sc.s1, G1 + EC::PE);  // dW1 = h^T Yb (launched with the next upd's jobs)
        has_pend = true;
        if (!pairs && !(g.n_tiles > 0 && use_tc(st))) gemm(s, N, sc.s1, T + H * H, nullptr, bh, b.inj, bh);  // b_h += Yb W^T + hbar^F
        break;
      }
      case kEmbed:
        flush();
        species_sum(st, sc, s, g, bh, nullptr, G1);
        break;
    }
    JANUS_LAUNCH_CHECK("stage_be");
    (void)R;
  }
  flush();
  if (st->u0 > 0) {
    const Port& out = sl.ports[JANUS_PORT_BADJ_OUT];
    copy(s, port_h(out, N), bh, NH);
    if (out.has_m) copy(s, port_m(out, N), bm, NH);
  }
}

// dst[x] += src[x]
__global__ void add_kernel(int64_t n, float* __restrict__ dst, const float* __restrict__ src) {
  JANUS_GDC_WAIT();
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x < n) dst[x] += src[x];
}

void add_into(float* dst, const float* src, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  janus::pdl(add_kernel, blocks(n, 256), 256, 0, s)(n, dst, src);
  JANUS_LAUNCH_CHECK("add");
}

// ============================================================ grads / OS
void stage_reduce_grads(janus_stage* st, cudaStream_t s) {
  janus::pdl(node::ledger_reduce_kernel, blocks(st->n_params, 256), 256, 0, s)(st->n_params, st->desc.n_micro_batches, st->g1,
                                                                       st->g2, st->grad);
  JANUS_LAUNCH_CHECK("ledger_reduce");
}

void stage_optimizer(janus_stage* st, const janus_opt& o, cudaStream_t s, const float* dhp) {
  ++st->adam_step;
  if (!dhp) {  // direct (uncaptured) call: the hyperparameters go through the stage's own buffer
    JANUS_CUDA(cudaMemcpyAsync(st->dopt, &o, sizeof(janus_opt), cudaMemcpyHostToDevice, s));
    dhp = st->dopt;
  }
  janus::pdl(node::adam_tick_kernel, 1, 1, 0, s)(st->dstep);
  janus::pdl(node::adam_kernel, blocks(st->n_params, 256), 256, 0, s)(st->n_params, st->params, st->m1, st->m2, st->grad, dhp,
                                                              st->dstep);
  JANUS_LAUNCH_CHECK("adam");
  refresh_transposes(st, s);
}

void stage_port(janus_stage* st, int mb, int slot, int port, void** dptr, size_t* bytes) {
  if (port < 0 || port > 7) throw domain_error("bad port");
  if (slot < 0 || slot >= st->desc.n_slots) throw domain_error("slot index out of range");
  if (mb < 0 || mb >= st->desc.n_micro_batches) throw domain_error("micro-batch index out of range");
  const Port& p = st->slots[static_cast<size_t>(slot)].ports[port];
  if (!p.buf) {
    *dptr = nullptr;
    *bytes = 0;
    return;
  }
  *dptr = p.buf;
  *bytes = port_elems(st, port, geo_of(st, mb).n_atoms) * sizeof(float);
}

// ============================================================ kernel timing
// Algorithmic FLOPs per edge of each msg-unit edge kernel (multiply-adds x 2),
// counting the per-edge contractions only:
//   FE: z=phi A, g=s B                                  -> RH + H^2
//   FF: z, z', g, g' (+ q dot)                          -> 2RH + 2H^2 + H
//   BF: z, z', g, g', sbar, sdotbar, dB(2), dA(2)       -> 4RH + 6H^2
//   BE: z, g, sbar, dB, dA                              -> 2RH + 3H^2
// Pair mode (tensor-core FE / FF, pair_tc.cuh): "FE" = the filter launch (FE's
// and FF's per-edge MMAs once per pair, i.e. half of FF's per-edge flops per
// directed edge) + FE's row sums; "FF" = the row kernel (Y, force scalar, and
// the a_h += Y W^T row GEMM counted per edge at ~50 edges per row is < 3%: omitted).
// BF / BE per pair: z, z', dB(2), sbar, sdotbar, dA(2) = 4RH + 4H^2 and
// z, dB, sbar, dA = 2RH + 2H^2 per PAIR (half per directed edge) + row sums.
double pair_flops_per_edge(int which, int H, int R) {
  const double RH = static_cast<double>(R) * H, HH = static_cast<double>(H) * H;
  switch (which) {
    case 0: return 0.5 * 2.0 * (2 * RH + 2 * HH + H) + 2.0 * H;
    case 1: return 2.0 * (3 * H);
    case 2: return 0.5 * 2.0 * (4 * RH + 4 * HH) + 2.0 * (3 * H);
    default: return 0.5 * 2.0 * (2 * RH + 2 * HH) + 2.0 * H;
  }
}

double edge_kernel_flops_per_edge(int which, int H, int R) {
  const double RH = static_cast<double>(R) * H, HH = static_cast<double>(H) * H;
  switch (which) {
    case 0: return 2.0 * (RH + HH);
    case 1: return 2.0 * (2 * RH + 2 * HH + H);
    case 2: return 2.0 * (4 * RH + 6 * HH);
    default: return 2.0 * (2 * RH + 3 * HH);
  }
}

// One launch of a msg unit's edge kernel for (mb, slot) on `s` with scratch
// lane `lane`: step_grid = the grid the step uses (tiles per CTA), else one
// tile per CTA on the full grid.  Inputs must exist (run the step first).
void launch_edge_kernel(janus_stage* st, int u, int which, int mb, int slot, int lane, cudaStream_t s, bool step_grid) {
  if (st->wide) throw config_error("edge-kernel timing hooks cover the fused H=64 kernels only");
  const DevGeo& g = geo_of(st, mb);
  Slot& sl = st->slots[static_cast<size_t>(slot)];
  MbOut& mo = st->outs[static_cast<size_t>(mb)];
  UnitBufs& b = sl.units[static_cast<size_t>(u - st->u0)];
  const EdgeGeom eg = edge_geom(g);
  const MsgParams mp = msg_params(st, u);
  Scratch& sc = lane_of(st, lane);
  if (use_tc(st) && st->pair_feff && which < 2) {
    const int N = g.n_atoms;
    if (which == 0) {  // the filters of this unit (pair MMAs of FE and FF) + FE's row sums
      launch_filter(st, g, sl, u, s, step_grid ? 0 : (g.n_pairs + edge_tc::TE - 1) / edge_tc::TE);
      JANUS_ROWS(msg_fe_rows, blocks(N, 8), s, N, g.row_ptr, g.col, g.pidx, b.wf, b.v, sc.s3);
    } else {
      JANUS_ROWS(msg_ff_rows, blocks(N, 8), s, N, g.row_ptr, g.col, g.pidx, g.u, b.wf, b.wfp, b.v, b.ff_a,
                                                         mp.pack + edge_tc::kWtOff / sizeof(float), sc.s3, sc.s5, sc.s4);
    }
    return;
  }
  if (use_tc(st) && st->pair_bfbe) {  // which 2 / 3: pair kernel (weight gradients) + row kernel; 4 / 5: pair kernel alone
    const int N = g.n_atoms;
    const int grid = step_grid ? pair_grid(st, g) : std::max(1, std::min((g.n_pairs + edge_tc::TE - 1) / edge_tc::TE, 148));
    const float* wt = mp.pack + edge_tc::kWtOff / sizeof(float);
    if (which == 4 && g.n_pairs > 0)
      janus::pdl(edge_tc::msg_bf_pair_tc, grid, edge_tc::NT, edge_tc::bf_pair_smem(), s)(eg, g.pgeo, g.n_pairs, mp, st->m.r_c, b.v, sc.s1,
                                                                                 b.ff_a, mo.Fbar, sc.partial);
    if (which == 5 && g.n_pairs > 0)
      janus::pdl(edge_tc::msg_be_pair_tc, grid, edge_tc::NT, edge_tc::be_pair_smem(), s)(eg, g.pgeo, g.n_pairs, mp, st->m.r_c, b.v, sc.s2,
                                                                                 sc.partial);
    if (which >= 4) return;
    if (which == 2) {
      if (g.n_pairs > 0)
        janus::pdl(edge_tc::msg_bf_pair_tc, grid, edge_tc::NT, edge_tc::bf_pair_smem(), s)(eg, g.pgeo, g.n_pairs, mp, st->m.r_c, b.v, sc.s1,
                                                                                   b.ff_a, mo.Fbar, sc.partial);
      JANUS_ROWS(msg_bf_rows, blocks(N, 8), s, N, g.row_ptr, g.col, g.pidx, g.u, mo.Fbar, b.wf, b.wfp, b.v, sc.s1, b.ff_a, wt,
                                                         sc.s3, sc.s4, nullptr, edge_tc::PartialReduce{});
    } else {
      if (g.n_pairs > 0)
        janus::pdl(edge_tc::msg_be_pair_tc, grid, edge_tc::NT, edge_tc::be_pair_smem(), s)(eg, g.pgeo, g.n_pairs, mp, st->m.r_c, b.v, sc.s2,
                                                                                   sc.partial);
      JANUS_ROWS(msg_be_rows, blocks(N, 8), s, N, g.row_ptr, g.col, g.pidx, b.wf, sc.s2, wt, sc.s3, nullptr, nullptr,
                 edge_tc::PartialReduce{});
    }
    return;
  }
  if (use_tc(st)) {
    const int grid = step_grid ? tc_grid(st, g) : tc_grid_tpc(g, 1);
    const int fgrid = step_grid ? fe_grid(st, g) : g.n_tiles_tc;
    switch (which) {
      case 0:
        janus::pdl(edge_tc::msg_fe_tc, fgrid, edge_tc::NT, edge_tc::fe_smem(), s)(eg, g.tile_tc, g.n_tiles_tc, mp, st->m.r_c, b.v, sc.s3);
        break;
      case 1:
        janus::pdl(edge_tc::msg_ff_tc, fgrid, edge_tc::NT, edge_tc::ff_smem(), s)(eg, g.tile_tc, g.n_tiles_tc, mp, st->m.r_c, b.v, b.ff_a, sc.s3, sc.s5, nullptr);
        break;
      case 2:
        janus::pdl(edge_tc::msg_bf_tc, grid, edge_tc::NT, edge_tc::bf_smem(), s)(eg, g.tile_tc, g.n_tiles_tc, mp, st->m.r_c, b.v, sc.s1, b.ff_a,
                                                                        mo.Fbar, sc.s3, sc.s4, sc.partial, nullptr);
        break;
      default:
        janus::pdl(edge_tc::msg_be_tc, grid, edge_tc::NT, edge_tc::be_smem(), s)(eg, g.tile_tc, g.n_tiles_tc, mp, st->m.r_c, b.v, sc.s2, sc.s3, sc.partial, nullptr, nullptr);
        break;
    }
    return;
  }
  switch (which) {
    case 0:
      janus::pdl(edge::msg_fe_kernel<kH, kR>, g.n_tiles, edge::NT, edge::fe_smem<kH, kR>(), s)(eg, mp, st->m.r_c, b.v, sc.s3);
      break;
    case 1:
      janus::pdl(edge::msg_ff_kernel<kH, kR>, g.n_tiles, edge::NT, edge::ff_smem<kH, kR>(), s)(eg, mp, st->m.r_c, b.v, b.ff_a, sc.s3, sc.s5);
      break;
    case 2:
      janus::pdl(edge::msg_bf_kernel<kH, kR>, g.n_tiles, edge::NT, edge::bf_smem<kH, kR>(), s)(eg, mp, st->m.r_c, b.v, sc.s1, b.ff_a,
                                                                                     mo.Fbar, sc.s3, sc.s4, sc.partial);
      break;
    default:
      janus::pdl(edge::msg_be_kernel<kH, kR>, g.n_tiles, edge::NT, edge::be_smem<kH, kR>(), s)(eg, mp, st->m.r_c, b.v, sc.s2, sc.s3, sc.partial);
      break;
  }
}

double kernel_flops_per_edge(const janus_stage* st, int which) {
  const double RH = static_cast<double>(kR) * kH, HH = static_cast<double>(kH) * kH;
  if (which == 4) return 0.5 * 2.0 * (4 * RH + 4 * HH);  // BF pair kernel: MMAs per pair, per directed edge
  if (which == 5) return 0.5 * 2.0 * (2 * RH + 2 * HH);  // BE pair kernel
  const bool pairs = use_tc(st) && (which < 2 ? st->pair_feff : st->pair_bfbe);
  return pairs ? pair_flops_per_edge(which, kH, kR) : edge_kernel_flops_per_edge(which, kH, kR);
}

int first_msg_unit(const janus_stage* st) {
  for (int x = st->u0; x < st->u1; ++x)
    if (unit_kind(x, st->m.L) == kMsg) return x;
  throw state_error("stage has no msg unit");
}

void stage_time_edge_kernel(janus_stage* st, int which, int mb, int slot, int iters, cudaStream_t s, float* avg_ms,
                            int64_t* edges, double* flops) {
  if (iters < 1 || which < 0 || which > 5 || (which > 3 && !(use_tc(st) && st->pair_bfbe))) throw domain_error("bad timing request");
  const int u = first_msg_unit(st);
  cudaEvent_t a, z;
  JANUS_CUDA(cudaEventCreate(&a));
  JANUS_CUDA(cudaEventCreate(&z));
  if (mb >= 0) {  // one micro-batch, back-to-back launches, full grid
    check_mb_slot(st, mb, slot);
    const DevGeo& g = geo_of(st, mb);
    launch_edge_kernel(st, u, which, mb, slot, 0, s, false);
    JANUS_LAUNCH_CHECK("time_edge_kernel");
    JANUS_CUDA(cudaEventRecord(a, s));
    for (int i = 0; i < iters; ++i) launch_edge_kernel(st, u, which, mb, slot, 0, s, false);
    JANUS_CUDA(cudaEventRecord(z, s));
    JANUS_CUDA(cudaEventSynchronize(z));
    float ms = 0.f;
    JANUS_CUDA(cudaEventElapsedTime(&ms, a, z));
    *avg_ms = ms / iters;
    *edges = g.n_edges;
    *flops = kernel_flops_per_edge(st, which) * g.n_edges;
  } else {
    // the step's concurrency: every micro-batch (slot = mb) on lane mb % lanes,
    // each launch with the step grid (tiles per CTA); time per round of all of them
    const int L = static_cast<int>(st->lanes.size()), n_mb = st->desc.n_micro_batches;
    std::vector<cudaStream_t> ls(static_cast<size_t>(L));
    std::vector<cudaEvent_t> ev(static_cast<size_t>(L) + 1);
    for (auto& x : ls) JANUS_CUDA(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
    for (auto& x : ev) JANUS_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
    int64_t E = 0;
    for (int m = 0; m < n_mb; ++m) E += geo_of(st, m).n_edges;
    auto round = [&] {
      JANUS_CUDA(cudaEventRecord(ev[0], s));
      for (int l = 0; l < L; ++l) JANUS_CUDA(cudaStreamWaitEvent(ls[static_cast<size_t>(l)], ev[0], 0));
      for (int m = 0; m < n_mb; ++m) launch_edge_kernel(st, u, which, m, m % static_cast<int>(st->slots.size()), m % L, ls[static_cast<size_t>(m % L)], true);
      for (int l = 0; l < L; ++l) {
        JANUS_CUDA(cudaEventRecord(ev[static_cast<size_t>(l) + 1], ls[static_cast<size_t>(l)]));
        JANUS_CUDA(cudaStreamWaitEvent(s, ev[static_cast<size_t>(l) + 1], 0));
      }
    };
    round();
    JANUS_LAUNCH_CHECK("time_edge_kernel");
    JANUS_CUDA(cudaEventRecord(a, s));
    for (int i = 0; i < iters; ++i) round();
    JANUS_CUDA(cudaEventRecord(z, s));
    JANUS_CUDA(cudaEventSynchronize(z));
    float ms = 0.f;
    JANUS_CUDA(cudaEventElapsedTime(&ms, a, z));
    for (auto& x : ls) cudaStreamDestroy(x);
    for (auto& x : ev) cudaEventDestroy(x);
    *avg_ms = ms / iters;  // one round: all micro-batches
    *edges = E;
    *flops = kernel_flops_per_edge(st, which) * static_cast<double>(E);
  }
  cudaEventDestroy(a);
  cudaEventDestroy(z);
}

// ============================================================ read-back
int stage_slot_of_mb(const janus_stage* st, int mb) {
  for (size_t x = 0; x < st->slots.size(); ++x)
    if (st->slots[x].mb == mb) return static_cast<int>(x);
  throw state_error("micro-batch has no live slot (FE not run)");
}

void stage_energy(janus_stage* st, int mb, float* E_host, float* loss_E, cudaStream_t s) {
  if (!st->has_readout) throw state_error("energies live on the stage holding the readout unit");
  const MbOut& mo = st->outs[static_cast<size_t>(mb)];
  const int ns = geo_of(st, mb).n_struct;
  if (E_host) JANUS_CUDA(cudaMemcpyAsync(E_host, mo.E, sizeof(float) * ns, cudaMemcpyDeviceToHost, s));
  if (loss_E) JANUS_CUDA(cudaMemcpyAsync(loss_E, mo.loss, sizeof(float), cudaMemcpyDeviceToHost, s));
  JANUS_CUDA(cudaStreamSynchronize(s));
}

void stage_forces(janus_stage* st, int mb, float* F_host, float* loss_F, cudaStream_t s) {
  if (!st->has_embed) throw state_error("complete forces live on stage 0");
  const MbOut& mo = st->outs[static_cast<size_t>(mb)];
  const int n = geo_of(st, mb).n_atoms;
  if (F_host) JANUS_CUDA(cudaMemcpyAsync(F_host, mo.F, sizeof(float) * 3 * n, cudaMemcpyDeviceToHost, s));
  if (loss_F) JANUS_CUDA(cudaMemcpyAsync(loss_F, mo.loss + 1, sizeof(float), cudaMemcpyDeviceToHost, s));
  JANUS_CUDA(cudaStreamSynchronize(s));
}

void stage_grads(janus_stage* st, int which, int mb, float* host_out, cudaStream_t s) {
  if (which < 0 || which > 2) throw domain_error("which must be 0, 1 or 2");
  const size_t NP = static_cast<size_t>(st->n_params), NMB = static_cast<size_t>(st->desc.n_micro_batches);
  std::vector<float> a(NP * NMB), b(NP * NMB);
  JANUS_CUDA(cudaMemcpyAsync(a.data(), st->g1, sizeof(float) * NP * NMB, cudaMemcpyDeviceToHost, s));
  JANUS_CUDA(cudaMemcpyAsync(b.data(), st->g2, sizeof(float) * NP * NMB, cudaMemcpyDeviceToHost, s));
  JANUS_CUDA(cudaStreamSynchronize(s));
  const size_t m0 = mb < 0 ? 0 : static_cast<size_t>(mb), m1 = mb < 0 ? NMB : static_cast<size_t>(mb) + 1;
  if (mb >= static_cast<int>(NMB)) throw domain_error("micro-batch index out of range");
  for (size_t x = 0; x < NP; ++x) {
    float acc = 0.f;  // same order as ledger_reduce_kernel
    for (size_t m = m0; m < m1; ++m) {
      if (which != 2) acc += a[m * NP + x];
      if (which != 1) acc += b[m * NP + x];
    }
    host_out[x] = acc;
  }
}

void stage_params(janus_stage* st, float* host_out, cudaStream_t s) {
  JANUS_CUDA(cudaMemcpyAsync(host_out, st->params, sizeof(float) * st->n_params, cudaMemcpyDeviceToHost, s));
  JANUS_CUDA(cudaStreamSynchronize(s));
}

int64_t stage_param_count(const janus_stage* st) { return st->n_params; }

void stage_grad_buffer(janus_stage* st, float** dptr, int64_t* count) {
  *dptr = st->grad;
  *count = st->n_params;
}

void stage_memory(const janus_stage* st, int64_t* static_bytes, int64_t* arena_bytes) {
  if (static_bytes) *static_bytes = st->static_bytes;
  if (arena_bytes) *arena_bytes = st->arena_bytes;
}

}  // namespace janus
