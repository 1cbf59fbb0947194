// stage.cuh — janus_stage: one pipeline stage (a contiguous unit range) on
// one GPU.  Owns the parameter slice, Adam state, per-micro-batch gradient
// ledgers (BE merged-first-order g1 / BF second-order g2, Eq. (2)), the
// per-micro-batch geometry, and per-slot activation storage + mailboxes.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/janus_cuda.h"

namespace janus {

class LmBuilder;

enum UnitKind { kEmbed = 0, kMsg = 1, kUpd = 2, kReadout = 3 };

inline UnitKind unit_kind(int u, int L) {
  if (u == 0) return kEmbed;
  if (u == 2 * L + 1) return kReadout;
  return (u % 2 == 1) ? kMsg : kUpd;
}

int64_t unit_param_count(const janus_model_desc& m, int u);
int64_t unit_param_offset(const janus_model_desc& m, int u);

// Upload block of one micro-batch: the caller's arrays and the host-built
// tables at fixed capacity offsets, so one LM is ONE host->device copy into a
// device block with the same layout (the device pointers below point into it).
struct LoadLayout {
  // the per-edge CSR arrays come last: a device-LM load (CSR built on the GPU)
  // uploads only the prefix up to the force targets
  enum { kRowPtr, kSpecies, kStructId, kStructPtr, kTileRow, kTileTc, kPos, kCell, kETarget, kFTarget, kCol, kRev, kShift, kN };
  size_t off[kN] = {};
  size_t bytes = 0;
};

struct DevGeo {
  int n_atoms = 0, n_edges = 0, n_struct = 0, n_tiles = 0;
  int n_tiles_tc = 0;
  int *row_ptr = nullptr, *col = nullptr, *src = nullptr, *rev = nullptr, *tile_row = nullptr, *shift = nullptr;
  int4* tile_tc = nullptr;  // tensor-core tiles (<= 8 rows, <= 128 edges): {row0, row1, edge0, edge1}
  std::vector<int> h_tiles, h_tiles_tc, h_sptr;  // host-side tile / struct tables (built at LM)
  // pinned host image of the upload block, double-buffered: a load may be
  // issued while the previous load's copy of this micro-batch is still queued
  // (the trainer pipelines step k+1's uploads behind step k)
  uint8_t* h_pin[2] = {nullptr, nullptr};
  uint8_t* d_block = nullptr;
  int h_par = 0;
  int *species = nullptr, *struct_id = nullptr, *struct_ptr = nullptr;
  double *pos = nullptr, *cell = nullptr;
  float *d = nullptr, *u = nullptr, *c = nullptr, *dc = nullptr, *E_target = nullptr, *F_target = nullptr;
  // undirected edge pairs (tensor-core FE / FF, pair_tc.cuh): canonical edge of
  // pair p, and pair of every directed edge
  int *pcanon = nullptr, *pidx = nullptr;
  float4* pgeo = nullptr;  // per pair two float4: (d, c, c', bits of i), (u, bits of j) of the canonical edge
  int n_pairs = 0;
};

struct UnitBufs {  // per slot, per unit
  float* out_h = nullptr;  // embed / upd output h
  float* out_m = nullptr;  // msg output m
  float* v = nullptr;      // msg: h W
  float* p = nullptr;      // upd: m U + ups ; readout: t
  float* ff_a = nullptr;   // upd: FF input a' ; msg: FF input a_m
  float* ff_Y = nullptr;   // msg: Y
  float *wf = nullptr, *wfp = nullptr;  // msg, tensor-core path: per-pair filter w and w' [pairs][64] (FE -> FF)
  float* inj = nullptr;    // BF -> BE injection at the unit input (h for msg/readout, m for upd)
  const float* in_h = nullptr;  // where this unit's input h lives (static)
  const float* in_m = nullptr;  // upd: input m
};

struct Port {
  float* buf = nullptr;  // [h | m | vec3] packed for the actual n_atoms
  bool has_m = false, has_vec = false;
  int H = 64;            // row width of h / m
};

// a CUtensorMap (128 B, 64 B aligned) kept opaque here (gemm_tc_host.hpp encodes it)
struct alignas(64) TMap {
  unsigned char bytes[128];
};

// Per-lane scratch: phases of different micro-batches may run concurrently on
// different streams ("lanes") of one device; all transient buffers are per lane.
struct Scratch {
  float *wh = nullptr, *wh2 = nullptr, *wm = nullptr, *s1 = nullptr, *s2 = nullptr, *s3 = nullptr, *s4 = nullptr, *s5 = nullptr;
  float *partial = nullptr, *wpart = nullptr;
  unsigned* counter = nullptr;  // last-CTA-reduces launch counter (one launch at a time per lane)
  // generic-width path (stage_wide.inc): [2 pairs][R] basis stack, three
  // [2 pairs][H] operand stacks, and the lane's cuBLAS handle + workspace
  float *phi2 = nullptr, *z2 = nullptr, *a2 = nullptr, *b2 = nullptr, *cspart = nullptr;
  unsigned* cstick = nullptr;  // column-sum tickets (one per 32-column strip, zero between launches)
  float* wslices = nullptr;    // K-slice products of the long weight-gradient GEMMs (gemm_tn_long)
  // tf32: tensor maps of this lane's operand stacks for the TMA-fed GEMMs (gemm_tc.cuh):
  // phi2 / a2 / b2 with 16-row boxes (pair tiles) and phi2 / b2 with 128-row boxes (plain tiles)
  TMap tm_phi2_pair, tm_a2_pair, tm_b2_pair, tm_phi2_plain, tm_b2_plain;
  void* blas = nullptr;
  void* blas_ws = nullptr;
};

struct Slot {
  std::vector<UnitBufs> units;
  Port ports[8];
  int mb = -1;             // latest occupant
};

// Per-micro-batch outputs (not pooled: small, and read back after the step)
struct MbOut {
  float* F = nullptr;      // running force [N*3]
  float* Fbar = nullptr;   // stage 0: force-loss seed
  float* e_atom = nullptr; // readout per-atom energies
  float* E = nullptr;      // [n_struct]
  float* eps = nullptr;    // [n_struct]
  float* loss = nullptr;   // [2] loss_E, loss_F
};

}  // namespace janus

struct janus_stage {
  janus_stage_desc desc{};
  janus_model_desc m{};
  int u0 = 0, u1 = 0, U = 0;
  bool has_embed = false, has_readout = false, in_has_m = false, out_has_m = false;
  int64_t n_params = 0;
  std::vector<int64_t> uoff;  // unit -> offset within the stage slice
  float *params = nullptr, *grad = nullptr, *m1 = nullptr, *m2 = nullptr;
  float *g1 = nullptr, *g2 = nullptr;  // [n_mb][n_params]
  std::vector<float*> tw;              // per unit: transposed weights block
  int adam_step = 0;
  int* dstep = nullptr;  // device-side Adam step (graph-replayable bias correction)
  float* dopt = nullptr; // device-side {lr, beta1, beta2, eps} for direct optimizer calls
  // geometry per micro-batch, double-buffered: geo[par * n_mb + mb]; the
  // phases read parity gpar[mb] while a trainer load may fill the other one
  // (a step in flight keeps reading its own copy)
  std::vector<janus::DevGeo> geo;
  std::vector<int> gpar;
  std::vector<janus::Slot> slots;   // activation slot pool (n_slots; include/janus/slots.hpp)
  std::vector<janus::MbOut> outs;   // per micro-batch outputs
  std::vector<janus::Scratch> lanes;
  float* losses = nullptr;  // [n_mb][2] loss_E, loss_F (outs[mb].loss points here)
  std::vector<void*> allocs;
  std::vector<void*> host_allocs;  // pinned (cudaHostAlloc)
  janus::LoadLayout lay;           // upload block layout (capacity offsets)
  int64_t static_bytes = 0, arena_bytes = 0;  // parameters / optimizer / ledgers; everything else
  int64_t pool_bytes = 0;                     // of arena_bytes: the activation slot pool
  int tpc_fe = 1, tpc_wg = 1;        // TC edge tiles per CTA: FE/FF, BF/BE (stage_create)
  int tpc_filter = 1;                // pair mode: 128-pair chunks per filter CTA
  int tc_tile_edges = 0;             // TC tiles: 0 cost-chosen runs, > 0 greedy edge budget (tuning)
  int tc_tile_max_chunks = 0;        // cost-chosen tiles: max 128-edge chunks (0: by mean degree)
  double tc_tile_ovh = 0.3;          // per-tile epilogue cost in chunk units
  bool pair_feff = true;             // TC FE / FF: filters once per edge pair (pair_tc.cuh); JANUS_FEFF_PAIR=0 -> directed-edge kernels
  int rows_kf = 8;                   // row kernels: edges' gathers in flight per warp (JANUS_ROWS_KF=4 for A/B)
  bool pair_bfbe = true;             // TC BF / BE: weight gradients once per edge pair (needs pair_feff); JANUS_BFBE_PAIR=0 -> directed
  int* pair_counts = nullptr;      // pair tables: canonical edges per (job, 1024-edge chunk)
  int pair_chunks_cap = 0;
  janus::LmBuilder* lm = nullptr;  // device neighbour-list builder (lazy, janus_stage_load without a CSR)
  bool wide = false;               // generic-width phases (stage_wide.inc) instead of the fused H=64 kernels
  bool wide_tc = false;            // wide + tf32 (or fp32, 3xTF32): per-pair GEMMs on gemm_tc.cuh with fused epilogues
  int wide_split3 = 0;             // wide + plain fp32: those GEMMs in 3xTF32 (fp32-tolerance) with exact sigmoids
  std::vector<janus::TMap> tm_w;   // wide_tc, per unit (msg: 3 maps): A^T [H x R], B^T [H x H], B [H x H]

  float* P(int u) const { return params + uoff[static_cast<size_t>(u - u0)]; }

};
