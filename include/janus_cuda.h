/* include/janus_cuda.h — the C ABI between the janus C++ host (schedule
 * executor, include/janus/train.hpp) and the sm_100a kernels.
 *
 * The reference has no compute interface at all: its seam is "Schedule in ->
 * per-instruction cost" (graph.hpp:168 replay(g, durations)
 * instr_duration).  Each entry point below is what EXECUTES one instruction
 * kind of reference ir.hpp:21-26 instead of looking up its duration:
 *   LM  -> janus_stage_load                (ir.hpp:25, graph.hpp:124)
 *   FE/FF/BF/BE -> janus_stage_{fe,ff,bf,be} (ir.hpp:22, phases PAPER.md:171-178)
 *   SA./RA./SG./RG. payloads -> janus_stage_port (ir.hpp:23-24; pairing graph.hpp:87-118)
 *   AR  -> janus_stage_grad_buffer + NCCL  (ir.hpp:25)
 *   OS  -> janus_stage_reduce_grads + janus_stage_optimizer_step (ir.hpp:25)
 * plus the transports (janus_comm_*) used by the executor for sends, receives and AR.
 *
 * Conventions: plain pointers and sizes, no C++/torch types.  Every function
 * returns 0 on success or a janus::Status code (include/janus/errors.hpp:47)
 * and records a thread-local message readable with janus_last_error().
 * Nothing throws across the ABI.  Streams are cudaStream_t passed as void*.
 */
#ifndef JANUS_CUDA_H
#define JANUS_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define JANUS_ABI_VERSION 1

/* precision of the per-edge contractions */
/* FP32: fp32 arithmetic throughout (SIMT kernels / fp32 GEMMs); TF32: tf32
 * tensor-core contractions (bf16 operands in the gradient-only BF/BE pair
 * kernels), fp32 accumulate; FP32_EMU: fp32 accuracy on the tensor cores
 * (BF16x9 emulated fp32 GEMMs, generic-width path only). */
enum { JANUS_PREC_FP32 = 0, JANUS_PREC_TF32 = 1, JANUS_PREC_FP32_EMU = 2 };

typedef struct {
  int32_t L, H, R, n_species;
  float r_c, w_E, w_F;
  int32_t precision; /* JANUS_PREC_* */
} janus_model_desc;

/* Units: 0 embed, 1+2l msg_l, 2+2l upd_l, 2L+1 readout. */
typedef struct {
  janus_model_desc model;
  int32_t unit_begin, unit_end; /* contiguous unit range [begin, end) */
  int32_t max_atoms, max_edges, max_struct; /* per micro-batch capacity */
  int32_t n_micro_batches;                  /* geometry + gradient-ledger slots */
  int32_t n_slots;                          /* in-flight activation slots */
  int32_t device;                           /* CUDA ordinal */
  int32_t n_lanes;                          /* concurrent micro-batch lanes (scratch sets), >= 1 */
  int32_t kernels;                          /* 0 = auto: the fused H=64 kernels when H = R = 64, else the
                                               generic-width GEMM path (any H in {64,128,256}, any R);
                                               1 = the generic-width path at any width */
} janus_stage_desc;

/* Host-side micro-batch: the LM payload.  Neighbour list in CSR by receiver
 * (janus_nbrlist_build), atoms of one structure contiguous. */
typedef struct {
  int32_t n_atoms, n_struct, n_edges;
  const double* pos;        /* [n_atoms*3] */
  const int32_t* species;   /* [n_atoms] */
  const int32_t* struct_id; /* [n_atoms] */
  const double* cell;       /* [n_struct] cubic box length */
  const float* E_target;    /* [n_struct] */
  const float* F_target;    /* [n_atoms*3] */
  const int32_t* row_ptr;   /* [n_atoms+1] */
  const int32_t* col;       /* [n_edges] */
  const int32_t* shift;     /* [n_edges*3] */
  const int32_t* rev;       /* [n_edges] */
} janus_host_batch;

typedef struct {
  float lr, beta1, beta2, eps;
} janus_opt;

typedef struct janus_stage janus_stage;
typedef struct janus_comm janus_comm;

/* ---- errors / info ---- */
const char* janus_last_error(void);
int janus_abi_version(void);
int janus_device_count(int* n);

/* ---- model / host data (no device needed) ---- */
int64_t janus_param_count(const janus_model_desc* m);
int64_t janus_unit_param_offset(const janus_model_desc* m, int unit);
int janus_num_units(const janus_model_desc* m);
/* Synthetic parameters ~ N(0, 1/fan_in) from SplitMix64(seed ^ tag*phi). */
int janus_synth_params(const janus_model_desc* m, uint64_t seed, float* out);
/* Synthetic cubic cell: n_atoms on a jittered sc/fcc lattice at density rho,
 * species, targets.  pos[n*3], species[n]; returns box length in *cell. */
int janus_synth_cell(int32_t n_atoms, double rho, int32_t n_species, uint64_t seed, double* pos,
                     int32_t* species, double* cell, float* E_target, float* F_target);
/* Periodic neighbour list, bit-exact with the oracle (oracle/mlip_oracle.c).
 * Returns the edge count in *n_edges; kDomainError if max_edges is exceeded. */
int janus_nbrlist_build(int32_t n_atoms, const double* pos, const int32_t* struct_id, const double* cell,
                        double r_c, int32_t max_edges, int32_t* row_ptr, int32_t* col, int32_t* shift,
                        int32_t* rev, int32_t* n_edges);

/* Device neighbour list (LM on the GPU).  A cell-list
 * build whose CSR (row_ptr, col, shift, rev) is bit-identical to
 * janus_nbrlist_build.  pos [n_atoms*3] and struct_id are DEVICE pointers,
 * cell [n_struct] (box lengths, which size the cell grid) is HOST; the outputs
 * are device buffers with room for max_edges edges.  Runs on `stream` and
 * synchronizes it once to return *n_edges; kDomainError if max_edges is
 * exceeded (same message as the host build).  Replaces the reference's LM
 * duration slot (ir.hpp:25, graph.hpp:124).
 *
 * The stage and trainer loads use it when a batch carries no neighbour list:
 * janus_stage_load / janus_trainer_load with hb->row_ptr == NULL build the CSR
 * on the device from hb->pos (col / shift / rev / n_edges are ignored). */
typedef struct janus_nbrlist janus_nbrlist;
int janus_nbrlist_create(int32_t max_atoms, int32_t max_struct, int32_t max_edges, int32_t device,
                         janus_nbrlist** out);
int janus_nbrlist_destroy(janus_nbrlist* nl);
int janus_nbrlist_build_device(janus_nbrlist* nl, int32_t n_atoms, int32_t n_struct, const double* pos,
                               const int32_t* struct_id, const double* cell, double r_c, int32_t* row_ptr,
                               int32_t* col, int32_t* shift, int32_t* rev, int32_t* n_edges, void* stream);

/* Stage plan without a device: the trainer's min-max contiguous partition of
 * the 2L+2 units into P blocks (include/janus/model.hpp partition_units).
 * unit_ranges[P][2] = [begin, end). */
int janus_plan_stages(const janus_model_desc* m, int32_t P, int32_t* unit_ranges);

/* ---- stages ---- */
int janus_stage_create(const janus_stage_desc* desc, const float* unit_params, janus_stage** out);
int janus_stage_destroy(janus_stage* st);
int janus_stage_load(janus_stage* st, int mb, const janus_host_batch* hb, void* stream);
int janus_stage_fe(janus_stage* st, int mb, int slot, void* stream);
int janus_stage_ff(janus_stage* st, int mb, int slot, void* stream);
int janus_stage_bf(janus_stage* st, int mb, int slot, void* stream);
int janus_stage_be(janus_stage* st, int mb, int slot, void* stream);

/* Boundary mailboxes (payloads of the send / receive instructions). */
enum {
  JANUS_PORT_ACT_IN = 0,  /* FE input  (RAE): h [, m]        */
  JANUS_PORT_ACT_OUT = 1, /* FE output (SAE): h [, m]        */
  JANUS_PORT_ADJ_IN = 2,  /* FF input  (RAF): a_h [, a_m], F */
  JANUS_PORT_ADJ_OUT = 3, /* FF output (SAF): a_h [, a_m], F */
  JANUS_PORT_TAN_IN = 4,  /* BF input  (RGF): abar [,], Fbar */
  JANUS_PORT_TAN_OUT = 5, /* BF output (SGF): abar [,], Fbar */
  JANUS_PORT_BADJ_IN = 6, /* BE input  (RGE): b_h [, b_m]    */
  JANUS_PORT_BADJ_OUT = 7 /* BE output (SGE): b_h [, b_m]    */
};
int janus_stage_port(janus_stage* st, int mb, int slot, int port, void** dptr, size_t* bytes);

/* Outputs for tests and the executor. */
int janus_stage_energy(janus_stage* st, int mb, float* E_host, float* loss_E_host, void* stream);
int janus_stage_forces(janus_stage* st, int mb, float* F_host, float* loss_F_host, void* stream);
/* which: 0 = total, 1 = BE merged first-order term, 2 = BF second-order term;
 * mb < 0 sums all micro-batches in index order. */
int janus_stage_grads(janus_stage* st, int which, int mb, float* host_out, void* stream);
int janus_stage_params(janus_stage* st, float* host_out, void* stream);
int64_t janus_stage_param_count(janus_stage* st);

/* OS = reduce per-micro-batch ledgers (fixed order) then Adam; AR between. */
int janus_stage_reduce_grads(janus_stage* st, void* stream);
int janus_stage_grad_buffer(janus_stage* st, float** dptr, int64_t* count);
int janus_stage_optimizer_step(janus_stage* st, const janus_opt* opt, void* stream);
/* Time one edge kernel of the stage's first msg unit in isolation (CUDA
 * events on `stream`, back-to-back launches after one warm-up): which = 0 FE,
 * 1 FF, 2 BF, 3 BE (tensor-core pair mode: 0 = filter + FE rows, 1 = FF rows,
 * 2 / 3 = pair weight-gradient kernel + row kernel), 4 / 5 = the BF / BE pair
 * weight-gradient kernel alone (pair mode only).  Requires the phase's inputs to exist (run the step once
 * first).  Returns the mean launch time, the launch's edge count and
 * algorithmic FLOPs (DESIGN.md §4 per-edge counts).  mb < 0: the step's
 * concurrency instead — every micro-batch (slot = mb) launched on lane
 * mb % n_lanes with the step's grid (tiles per CTA); *avg_ms is then the time
 * of one round of all of them and edges / flops their totals. */
int janus_stage_time_edge_kernel(janus_stage* st, int which, int mb, int slot, int iters, void* stream,
                                 float* avg_ms, int64_t* edges, double* flops);
/* Peak device bytes held by the stage (static + activation arena). */
int janus_stage_memory(janus_stage* st, int64_t* static_bytes, int64_t* arena_bytes);

/* ---- transports ---- */
/* NCCL: one base communicator per process group (id from rank 0 via any
 * channel); a trainer splits one 2-rank communicator per transfer channel
 * (flow, from, to) plus the 1F1B pair / data-parallel groups. */
int janus_nccl_unique_id(void* id_out /* 128 bytes */);
int janus_comm_init_nccl(const void* id, int nranks, int rank, int device, janus_comm** out);
/* Same-GPU multi-process transport (the test harness for the per-rank path on
 * one GPU): N processes on ONE device exchange CUDA-IPC regions through files
 * in `dir` (one exchange per trainer) and run NCCL's blocking-rendezvous
 * semantics with stream memory operations (csrc/transport.hpp).  The trainer
 * treats it exactly like an NCCL comm. */
int janus_comm_init_ipc(const char* dir, int nranks, int rank, int device, janus_comm** out);
/* The same transport for N ranks that are THREADS of one process on one
 * device (one CUDA context: the ranks' kernels run concurrently; separate
 * processes on one GPU are time-sliced, csrc/transport.hpp).  The test harness
 * of the per-rank path: every rank still builds its own per-rank trainer. */
int janus_comm_init_threads(const char* dir, int nranks, int rank, int device, janus_comm** out);
int janus_comm_destroy(janus_comm* c);
int janus_comm_send(janus_comm* c, const void* buf, size_t bytes, int peer, void* stream);
int janus_comm_recv(janus_comm* c, void* buf, size_t bytes, int peer, void* stream);
int janus_comm_group_start(void);
int janus_comm_group_end(void);
int janus_comm_allreduce_sum(janus_comm* c, float* buf, int64_t count, void* stream);

/* ---- whole-step executor (C++ train_step behind a C entry) ----
 * Walks Schedule::device_lists[d] (ir.hpp:147) in seq order (the sole
 * intra-device order, ir.hpp:131) and executes every instruction.  Local mode
 * runs all P stages in this process on one GPU with one stream set per
 * virtual device and device-to-device copies as the transport; NCCL mode runs
 * the stage(s) of rank r over janus_comm (P2P per flow + allreduce). */
typedef struct {
  int32_t n_stages;        /* P */
  int32_t method;          /* 0 SymFold, 1 WaveK, 2 1F1B-2nd, 4 Hanayo-2nd */
  int32_t wavek_k;
  int32_t n_micro_batches; /* per replica */
  int32_t local_stages;    /* 1 = all P stages in this process on one GPU */
  int32_t use_graphs;      /* capture the step once as a CUDA graph, replay it */
  int32_t dp_degree;       /* data-parallel replicas (NCCL mode), >= 1 */
  int32_t record_timeline; /* per-instruction CUDA events (disables graphs) */
  int32_t lanes;           /* compute streams per device; micro-batch m runs on lane m % lanes.
                              1 = strict list order (pipeline/bubble studies); >1 overlaps
                              independent micro-batches (throughput at P=1) */
  int32_t unfolded_slots;  /* 0 (default) = activation slots pooled per stage by the schedule's
                              live micro-batches (include/janus/slots.hpp); 1 = one slot per
                              micro-batch (the unfolded baseline for memory studies) */
  double phase_us[4];      /* WaveK's list-schedule cost model: measured per-stage phase times
                              {FE, FF, BE, BF} (e.g. a timeline step's means); all 0 = the
                              paper's UMA-1.2B ratios */
} janus_exec_desc;

typedef struct {
  double makespan_ms;      /* device time of the last step (anchor -> end) */
  double bubble_ratio;     /* sum idle / (P makespan), SPEC.md:436 (timeline only) */
  double busy_ms[64];      /* per (virtual) device compute time (timeline only) */
  int64_t p2p_bytes;       /* bytes moved between stages in the last step */
  int64_t kernel_launches; /* kernels issued by the last step */
  int64_t peak_bytes[64];  /* per device: static + arena bytes of its stages */
  double loss;             /* sum of loss_E + loss_F held by this process */
  int64_t act_bytes[64];   /* per device: activation slot pool bytes (part of peak_bytes) */
  int32_t act_slots[64];   /* per device: slots of its largest pool (live micro-batches) */
} janus_step_stats;

typedef struct janus_trainer janus_trainer;
int janus_trainer_create(const janus_exec_desc* ed, const janus_stage_desc* sd, const float* all_params,
                         janus_comm* comm, int rank, janus_trainer** out);
/* The same trainer executing a caller's schedule (the reference text format,
 * ir.hpp:253-359; e.g. one built with transform::priority_topo_order): a
 * validated second-order schedule over ed->n_stages devices and
 * ed->n_micro_batches micro-batches; its stage map selects the folded
 * (SymFold / WaveK / Hanayo) or the 1F1B-2nd layout, ed->method is ignored.
 * Used by include/janus/train.hpp's train_step. */
int janus_trainer_create_from_text(const janus_exec_desc* ed, const janus_stage_desc* sd, const float* all_params,
                                   const char* schedule_text, janus_comm* comm, int rank, janus_trainer** out);
int janus_trainer_destroy(janus_trainer* t);
int janus_trainer_load(janus_trainer* t, int mb, const janus_host_batch* hb);
/* LM of n micro-batches (mbs[k] <- hbs[k]).  Each micro-batch's geometry is
 * double-buffered: a load fills the copy the step in flight does not read, on
 * the trainer's load stream, and the next janus_trainer_step[_async] switches
 * to it (root waits for the loads).  Batches without a neighbour list
 * (row_ptr == NULL) get ONE device cell-list build over all of them (their
 * structures side by side) and one host sync for the row-tile tables.
 * janus_trainer_load == n = 1. */
int janus_trainer_load_many(janus_trainer* t, int n, const int32_t* mbs, const janus_host_batch* hbs);
int janus_trainer_step(janus_trainer* t, const janus_opt* opt, janus_step_stats* stats);
/* janus_trainer_step split in two: issue the step and return; then wait for it
 * and fill stats (loss read back).  Loads issued in between run beside the
 * step in flight (into the other geometry copy), so the next step's uploads,
 * neighbour lists and geometry overlap this step's device time (input
 * pipelining).  Up to two steps may be in flight: janus_trainer_wait
 * returns the oldest one (its loss terms are snapshotted on the device when
 * the step ends), so a training loop can issue step k+1 before reading step k
 * back.  janus_trainer_step == step_async + wait. */
int janus_trainer_step_async(janus_trainer* t, const janus_opt* opt);
int janus_trainer_wait(janus_trainer* t, janus_step_stats* stats);
/* per compute instruction of the last timed step: [n][5] = device, kind, mb, start_us, end_us */
int janus_trainer_timeline(janus_trainer* t, double* out, int32_t cap, int32_t* n);
int janus_trainer_stage(janus_trainer* t, int block, int force_replica, janus_stage** out);
int janus_trainer_schedule_text(janus_trainer* t, char* buf, int64_t cap, int64_t* len);
int janus_trainer_plan(janus_trainer* t, int32_t* unit_ranges /* [P][2] */);

/* ---- diagnostics ---- */
/* tcgen05 layer self-test (tests/test_gpu_tc.py).  args = {M, N, K, a_mn, b_mn,
 * a_rows, a_cols, b_rows, b_cols}; tiles are row-major fp32; K-major tiles are
 * [M|N rows][K cols], MN-major tiles [K rows][M|N cols].  D = raw TMEM image,
 * 128 lanes x N fp32 columns. */
int janus_tc_probe(const int32_t* args, const float* A, const float* B, float* D);
/* gemm_tc.cuh self-test (tests/test_gpu_tc.py): D = A . W^T through the TMA-fed
 * tcgen05 GEMM.  pair bit 0 = 1: A [2 rows x K] and D [2 rows x N] are the
 * stacked [value; derivative] layout of the generic-width path; bit 1 = 1:
 * 3xTF32 (fp32-accurate) instead of tf32. */
int janus_gemm_tc_probe(int32_t rows, int32_t K, int32_t N, int32_t pair, const float* A, const float* W, float* D);

/* ---- GARS micro-batch packing (host only; include/janus/gars.hpp) ----
 * SPEC.md:496-562, Algorithm 1.  Graph i has atoms[i] atoms and id i.
 * order[M]: graph ids grouped by micro-batch (in shuffled order), mb_ptr[n_mb+1]
 * the group offsets, tags[n_mb]: 0 comm_free / 1 dist (max size * d_gp <= total). */
int janus_gars_pack(const int32_t* atoms, int32_t M, int32_t n_mb, int32_t d_gp, uint64_t seed, int32_t* order,
                    int32_t* mb_ptr, int32_t* tags);
/* Baseline: greedy sequential fixed-atom packing in dataset order. */
int janus_gars_greedy(const int32_t* atoms, int32_t M, int32_t n_mb, int32_t d_gp, int32_t* order,
                      int32_t* mb_ptr, int32_t* tags);
/* Second-level GP bins of one comm_free micro-batch (atoms in its order): bin_of[n];
 * kStateError for a dist micro-batch. */
int janus_gars_assign_bins(const int32_t* atoms, int32_t n, int32_t d_gp, int32_t* bin_of);
/* Synthetic long-tailed sizes: stats = {mean, P50, P90, P99, max} or NULL for
 * the mixed preset (85, 53, 213, 427, 905); edges = 20 * atoms^1.3. */
int janus_gars_synth_sizes(const double* stats, int32_t n, uint64_t seed, int32_t* atoms, int64_t* edges);

/* ---- cost model + WaveK tuner (host only; include/janus/tuner.hpp) ----
 * SPEC.md:387-395 (lifetime-rule peak memory), 578-637 (tuner).  t[4] =
 * measured per-stage phase times {FE, FF, BE, BF}; mem[6] = {M_GPU,
 * M_reserve, M_static, fe_bytes, ff_bytes, stage0_mult} in bytes (fe/ff =
 * activation bytes one micro-batch keeps live FE->BE / FF->BF per device).
 * table[n][5] = {k, makespan, bubble_ratio, peak_max_bytes, feasible}. */
int janus_tune_wavek(int32_t P, int32_t n_mb, const double* t, const double* mem, int32_t divisors_only,
                     int32_t* k_star, int32_t* tuned, double* table, int32_t cap, int32_t* n);
/* Lifetime-rule peak bytes per device of any schedule text replayed under
 * t[4]; static_bytes[n_static] per device (n_static = 1: all devices),
 * act[4] = {fe_bytes, ff_bytes, stage0_mult, replicate}.  FF with the
 * recompute flag holds fe_bytes until its BF; with replicate != 0,
 * replicated-parameter devices (AR flag) count static twice (the SPEC's
 * uniform-static rule); 0 = static_bytes are exact per device.
 * peaks[num devices]. */
int janus_schedule_memory(const char* text, const double* t, const double* static_bytes, int32_t n_static,
                          const double* act, double* peaks, int32_t cap, int32_t* n_devices);

/* ---- timeline rendering (host only; include/janus/render.hpp) ----
 * recs[n][5] = {device, phase (0 FE 1 FF 2 BE 3 BF), mb, start, end}, e.g. the
 * executor timeline (janus_trainer_timeline) or a replay (text != NULL: the
 * schedule is replayed under t[4] and recs is ignored).  fmt 0 = ASCII (one
 * column per `quantum`), 1 = SVG (`quantum` = pixels per time unit). */
int janus_render_timeline(const double* recs, int32_t n, const char* text, const double* t, int32_t fmt,
                          double quantum, char* buf, int64_t cap, int64_t* len);

/* ---- schedule generation (host only) ---- */
/* method: 0 SymFold, 1 WaveK(k), 2 1F1B-2nd, 3 first-order Pass 0, 4 Hanayo-2nd */
int janus_schedule_generate(int method, int P, int n_mb, int k, char* buf, int64_t cap, int64_t* len);
int janus_schedule_validate(const char* text, int32_t* n_errors);
/* Replay (graph.hpp:168) a schedule under phase times t[4] = {FE, FF, BE, BF}
 * (FF with the recompute flag costs FF + FE): makespan and bubble ratio
 * sum idle / (devices * makespan). */
int janus_schedule_replay(const char* text, const double* t, double* makespan, double* bubble_ratio);

/* Blocking-rendezvous check of the multi-process (one process per GPU)
 * issue program of a schedule (include/janus/rendezvous.hpp): each rank's
 * lanes (micro-batch m on lane m % lanes) and transfer streams are simulated
 * with NCCL semantics (a send and its receive complete together, only when
 * both are at the heads of their streams; collectives complete when the
 * whole group is at them).  layout 0 = the executor's per-channel streams,
 * 1 = one shared send and one shared receive stream per rank (round 1's
 * layout, kept to show it deadlocks).  *ok = 1 when every op completes;
 * stuck (may be NULL) receives the blocked stream heads otherwise.  Replaces
 * nothing in the reference: its DepGraph (graph.hpp:87-118) assumes
 * non-blocking channels. */
int janus_schedule_check_rendezvous(const char* text, int32_t onef1b, int32_t lanes, int32_t dp, int32_t layout,
                                    int32_t* ok, int64_t* completed, int64_t* total, char* stuck, int64_t cap);

/* Activation slot pool per device of a schedule (include/janus/slots.hpp):
 * the most micro-batches live at once on one of the device's stage objects
 * under the SPEC lifetime rule, in the executor's issue
 * order (local = all stages in one process, else each device's own list),
 * at least min(lanes, micro-batches) per pool (concurrent lanes);
 * unfolded = 1 gives one slot per micro-batch.  slots[n_devices]. */
int janus_schedule_slot_pool(const char* text, int32_t onef1b, int32_t local, int32_t unfolded, int32_t lanes,
                             int32_t* slots, int32_t cap, int32_t* n_devices);

#ifdef __cplusplus
}
#endif
#endif
