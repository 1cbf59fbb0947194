// executor.cpp — janus_trainer: executes a SymFold / WaveK / 1F1B-2nd
// schedule (include/janus/schedule_gen.hpp) instruction by instruction.
//
// Replaces the reference's "look up a duration" seam (graph.hpp:168 replay,
// SPEC.md:377-385 instr_duration) with "execute the instruction":
//   FE/FF/BF/BE -> stage phase kernels on the device's compute stream
//   S*  -> payload leaves the stage's out-port on a side stream
//   R*  -> payload lands in the peer stage's in-port; the compute stream waits
//   OS  -> ledger reduce (+ AR) + Adam;  LM -> geometry is uploaded by load()
// Channels follow the DepGraph pairing key (graph.hpp:95-97): one transport
// channel per flow (act / adj / tan / badj / mirror), so per-channel order is
// the micro-batch order of the device lists on both ends (checked at create).
//
// Transports:
//   local: all P virtual devices in this process on one GPU, each with its own
//          compute/send streams; a send is an async D2D copy into the peer's
//          port followed by an event the receiver's compute stream waits on.
//   per-rank (one process per GPU, transport.hpp): every channel (flow, from,
//          to) has its own communicator and its own stream at each end, so a
//          blocking send / receive only ever waits for its own channel's
//          FIFO (include/janus/rendezvous.hpp proves the program deadlock-free
//          at create).  NCCL over NVLink, or the same-GPU IPC transport that
//          lets N processes exercise this path on one GPU.
// 1F1B-2nd runs the force half on
// replicated parameters: FF recomputes FE from the block input (mirror
// transfer), BF is followed by an injection-only BE whose block-input
// cotangent is sent back to the energy device, and OS all-reduces the pair.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <mutex>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <numeric>
#include <string>
#include <tuple>
#include <array>
#include <vector>

#include "../../include/janus/errors.hpp"
#include "../../include/janus/graph.hpp"
#include "../../include/janus/model.hpp"
#include "../../include/janus/schedule_gen.hpp"
#include "../../include/janus/slots.hpp"
#include "../../include/janus_cuda.h"
#include "cuda_check.hpp"
#include "stage.cuh"
#include "stage_api.hpp"
#include "nbrlist.hpp"
#include "transport.hpp"

namespace janus {
namespace {

// Channels (include/janus/rendezvous.hpp): flows act / adj / tan / badj plus
// the 1F1B-2nd mirror flows, which pair two blocks per device pair and are
// split by block parity to keep per-channel order = micro-batch order.

inline void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw nccl_error(std::string(what) + ": " + ncclGetErrorString(r));
}
#define JANUS_NCCL(x) nccl_check((x), #x)

}  // namespace
}  // namespace janus

namespace janus {
namespace {

struct VDev {
  int id = 0;                          // schedule device index
  cudaStream_t compute = nullptr;      // lane 0; OS runs here after joining the lanes
  std::vector<cudaStream_t> lane;      // compute streams; micro-batch m -> lane m % size
  cudaStream_t send = nullptr, recv = nullptr;
};

struct Rec {
  int device, kind, mb;
  cudaEvent_t a, b;
};

// A transfer endpoint: which stage object and which port.
struct End {
  janus_stage* st = nullptr;
  int port = -1;
};

}  // namespace
}  // namespace janus

struct janus_trainer {
  janus_exec_desc ed{};
  janus_stage_desc sd{};
  janus::Schedule sched;
  janus::StagePlan plan;
  int P = 1, method = 0;
  bool local = true, onef1b = false;
  janus_comm* comm = nullptr;
  int rank = 0, replica = 0, my_dev = 0;
  std::vector<janus::VDev> devs;                 // local virtual devices (local: P, NCCL: 1)
  std::vector<janus_stage*> E, F;                // per block (nullptr if not on this process)
  std::vector<int> E_dev, F_dev;                 // schedule device that holds E_b / F_b
  std::vector<janus_stage*> owned;
  std::vector<float*> mirror_buf;                // 1F1B: [block*n_mb + mb] cotangent from F_b
  std::vector<janus::ChannelKey> chans;          // per-rank mode: every channel of the schedule
  std::vector<cudaStream_t> chan_stream;         // per channel: this rank's end (nullptr: not a member)
  std::unique_ptr<janus::Transport> xport;       // per-rank mode: NCCL or same-GPU IPC
  std::vector<void*> allocs;
  cudaStream_t root = nullptr;
  cudaEvent_t anchor = nullptr, finish = nullptr;
  std::vector<cudaEvent_t> pool;
  size_t pool_next = 0;
  std::map<std::tuple<int, int, int, int>, cudaEvent_t> delivered;  // (flow, mb, from_block, to_block)
  std::vector<int> order;                        // local mode: global issue order (flat indices)
  janus::DepGraph graph;
  std::vector<janus::Rec> recs;
  bool recording = false;
  // steps issued by trainer_step_async and not yet waited for (at most two: the
  // host may issue step k+1 before reading step k back, so the GPU never idles
  // on the host between steps); per issue parity: anchor / finish events and a
  // device snapshot of the loss terms taken right after the step
  int inflight = 0;
  cudaEvent_t anchor_q[2] = {nullptr, nullptr}, finish_q[2] = {nullptr, nullptr}, done_q[2] = {nullptr, nullptr};
  float* loss_snap[2] = {nullptr, nullptr};
  float* dopt = nullptr;                         // device {lr, beta1, beta2, eps}: written on root before every step
  int64_t p2p_bytes = 0;
  int64_t kernel_count = -1;
  cudaGraphExec_t gexec = nullptr;               // instantiated step graph for key gkey (geometry parities)
  std::vector<int> gkey;
  cudaGraphExec_t gexec_alt = nullptr;           // the other cached graph (loads alternate the parities)
  std::vector<int> gkey_alt;
  int64_t kernel_count_alt = -1;
  janus_step_stats last{};
  // activation slot pool (include/janus/slots.hpp): slot per (object, mb),
  // release events, and per step which streams already waited on a release
  janus::SlotPlan slotplan;
  std::map<janus_stage*, int> obj_of;
  std::map<std::pair<int, int>, cudaEvent_t> rel_ev;
  std::map<std::pair<int, int>, std::vector<cudaStream_t>> slot_waited;
  std::map<std::pair<int, int>, cudaStream_t> slot_last;
  int reserved_streams = 0;                      // per-rank mode: streams counted against the process's hardware queues
  std::vector<int> n_atoms;                      // per mb (for port sizes on the receive side)
  std::vector<std::array<int, 5>> shape;         // per (parity, mb): atoms, edges, structs, tiles, TC tiles (graph validity)
  // double-buffered geometry: a load fills the copy the step in flight does not
  // read, on the load stream, so uploads / neighbour lists / geometry overlap it
  std::vector<int> step_par;                     // per mb: copy the last issued step read (-1: none)
  std::vector<int> load_par;                     // per mb: copy filled by a load not yet used by a step (-1: none)
  cudaStream_t load_stream = nullptr;
  cudaEvent_t load_done = nullptr;               // end of the latest loads on load_stream
  cudaEvent_t step_end[2] = {nullptr, nullptr};  // end of steps with even / odd index
  int64_t nsteps = 0;
  janus::LmBuilder* lm = nullptr;                // device neighbour lists (loads without a CSR)
  int lm_par = 0;                                 // CSR buffer of the next device LM build
  // hang diagnostics (JANUS_HANG_REPORT=<seconds>, debugging aid, off by default):
  // an event after every issued instruction; trainer_wait reports the first
  // unfinished instruction per stream instead of blocking forever
  double hang_s = 0;
  cudaStream_t last_comm = nullptr;
  struct Probe {
    int kind, mb, dev;
    cudaStream_t s;
    cudaEvent_t e;
  };
  std::vector<Probe> probes;
  std::mutex probe_mu;
  std::atomic<int64_t> waited{0};
  std::atomic<int64_t> issued{0};
  std::string last_issued;
  std::shared_ptr<std::atomic<bool>> alive = std::make_shared<std::atomic<bool>>(true);  // for the watchdog threads
};

namespace janus {
namespace {

cudaEvent_t next_event(janus_trainer* t) {
  if (t->pool_next == t->pool.size()) {
    cudaEvent_t e;
    JANUS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    t->pool.push_back(e);
  }
  return t->pool[t->pool_next++];
}

VDev& vdev(janus_trainer* t, int d) {
  if (t->local) return t->devs[static_cast<size_t>(d)];
  if (d != t->my_dev) throw state_error("instruction for a device this process does not own");
  return t->devs[0];
}

int peer_rank(const janus_trainer* t, int dev) { return t->replica * t->P + dev; }

int block_of(const janus_trainer* t, int vs) { return vs < t->P ? vs : 2 * t->P - 1 - vs; }

// Map a comm instruction to (flow, sender end, receiver end, from-block, to-block).
// Returns false for the fold-point pair of 1F1B-2nd (carried by the mirror flow).
bool route(janus_trainer* t, const Instruction& in, int* flow, End* src, End* dst, int* from_b, int* to_b) {
  const int P = t->P, vs = in.virtual_stage;
  const CommClass c = comm_class(in.kind);
  const bool send = is_send(in.kind);
  // normalise to the sending stage
  const int s_vs = send ? vs : comm_peer_stage(in.kind, vs);
  const int r_vs = send ? comm_peer_stage(in.kind, vs) : vs;
  const bool act = (c == CommClass::SA || c == CommClass::RA);
  if (act) {
    if (s_vs == P - 1 && r_vs == P) return false;  // fold point (1F1B-2nd only)
    if (r_vs < P) {                                 // FE chain up: SAE
      *flow = kFlowAct;
      *src = {t->E[static_cast<size_t>(s_vs)], JANUS_PORT_ACT_OUT};
      *dst = {t->E[static_cast<size_t>(r_vs)], JANUS_PORT_ACT_IN};
    } else {  // FF chain: force stage s_vs -> s_vs+1 = block b -> b-1
      *flow = kFlowAdj;
      *src = {t->F[static_cast<size_t>(block_of(t, s_vs))], JANUS_PORT_ADJ_OUT};
      *dst = {t->F[static_cast<size_t>(block_of(t, r_vs))], JANUS_PORT_ADJ_IN};
    }
  } else {
    if (s_vs == P && r_vs == P - 1) return false;  // fold point (1F1B-2nd only)
    if (r_vs >= P) {                                // BF chain: block b -> b+1
      *flow = kFlowTan;
      *src = {t->F[static_cast<size_t>(block_of(t, s_vs))], JANUS_PORT_TAN_OUT};
      *dst = {t->F[static_cast<size_t>(block_of(t, r_vs))], JANUS_PORT_TAN_IN};
    } else {  // BE chain down
      *flow = kFlowBadj;
      *src = {t->E[static_cast<size_t>(s_vs)], JANUS_PORT_BADJ_OUT};
      *dst = {t->E[static_cast<size_t>(r_vs)], JANUS_PORT_BADJ_IN};
    }
  }
  *from_b = block_of(t, s_vs);
  *to_b = block_of(t, r_vs);
  return true;
}

// The activation slot of (stage object, micro-batch) for a use on stream s.
// A reused slot makes every stream that touches it wait once for the previous
// occupant's release (recorded after that occupant's last use).
int slot_of(janus_trainer* t, janus_stage* st, int mb, cudaStream_t s) {
  const auto o = t->obj_of.find(st);
  if (o == t->obj_of.end()) throw state_error("stage object without a slot plan");
  const std::pair<int, int> k{o->second, mb};
  const auto it = t->slotplan.slot.find(k);
  if (it == t->slotplan.slot.end()) throw state_error("slot plan misses a use of micro-batch " + std::to_string(mb));
  const int prev = t->slotplan.prev.at(k);
  if (prev >= 0) {
    std::vector<cudaStream_t>& w = t->slot_waited[k];
    if (std::find(w.begin(), w.end(), s) == w.end()) {
      JANUS_CUDA(cudaStreamWaitEvent(s, t->rel_ev.at({k.first, prev}), 0));
      w.push_back(s);
    }
  }
  t->slot_last[k] = s;
  return it->second;
}

void port_ptr(janus_trainer* t, janus_stage* st, int mb, int port, cudaStream_t s, float** p, size_t* bytes) {
  void* d = nullptr;
  stage_port(st, mb, slot_of(t, st, mb, s), port, &d, bytes);
  *p = static_cast<float*>(d);
}

size_t port_bytes_for(const janus_trainer* t, int block, int port, int mb) {
  // both ends of a channel use identical layouts; compute from the model
  const int H = t->sd.model.H, n = t->n_atoms[static_cast<size_t>(mb)];
  const bool at_input = (port == JANUS_PORT_ACT_IN || port == JANUS_PORT_ADJ_OUT || port == JANUS_PORT_TAN_IN ||
                         port == JANUS_PORT_BADJ_OUT);
  const int u = at_input ? t->plan.blocks[static_cast<size_t>(block)].first : t->plan.blocks[static_cast<size_t>(block)].second;
  const bool has_m = (u - 1 >= 1) && (u - 1 <= 2 * t->sd.model.L) && ((u - 1) % 2 == 1);
  const bool has_vec = port >= JANUS_PORT_ADJ_IN && port <= JANUS_PORT_TAN_OUT;
  return sizeof(float) * (static_cast<size_t>(n) * H * (has_m ? 2 : 1) + (has_vec ? 3 * static_cast<size_t>(n) : 0));
}

// ------------------------------------------------------------- transfers
cudaStream_t lane_stream(const janus_trainer* t, const VDev& dv, int mb) {
  (void)t;
  return dv.lane[static_cast<size_t>(mb < 0 ? 0 : mb) % dv.lane.size()];
}
int lane_index(const VDev& dv, int mb) { return (mb < 0 ? 0 : mb) % static_cast<int>(dv.lane.size()); }

// per-rank mode: a payload leaves on its channel's own stream once the lane
// that produced it got there
void chan_send(janus_trainer* t, VDev& dv, int flow, int mb, const float* sp, size_t sb, int peer_dev) {
  const int c = channel_index(t->chans, {flow, dv.id, peer_dev});
  cudaStream_t cs = t->chan_stream[static_cast<size_t>(c)];
  cudaEvent_t ready = next_event(t);
  JANUS_CUDA(cudaEventRecord(ready, lane_stream(t, dv, mb)));
  JANUS_CUDA(cudaStreamWaitEvent(cs, ready, 0));
  t->p2p_bytes += static_cast<int64_t>(sb);
  t->xport->send(c, sp, sb, peer_rank(t, peer_dev), cs);
  t->last_comm = cs;
}
// ... and lands on its channel's stream; the lane waits for it
void chan_recv(janus_trainer* t, VDev& dv, int flow, int mb, float* dp, size_t db, int peer_dev) {
  const int c = channel_index(t->chans, {flow, peer_dev, dv.id});
  cudaStream_t cs = t->chan_stream[static_cast<size_t>(c)];
  t->xport->recv(c, dp, db, peer_rank(t, peer_dev), cs);
  t->last_comm = cs;
  cudaEvent_t done = next_event(t);
  JANUS_CUDA(cudaEventRecord(done, cs));
  JANUS_CUDA(cudaStreamWaitEvent(lane_stream(t, dv, mb), done, 0));
}

void do_send(janus_trainer* t, VDev& dv, int flow, int mb, janus_stage* src, int sport, janus_stage* dst, int dport,
             int from_b, int to_b, int peer_dev) {
  float* sp;
  size_t sb;
  if (!t->local) {
    port_ptr(t, src, mb, sport, t->chan_stream[static_cast<size_t>(channel_index(t->chans, {flow, dv.id, peer_dev}))], &sp, &sb);
    return chan_send(t, dv, flow, mb, sp, sb, peer_dev);
  }
  // local: the copy runs on this channel's own stream, so a copy waiting for
  // the receiver's slot (slots.hpp) never holds up another channel's copies
  cudaStream_t cs = t->chan_stream[static_cast<size_t>(channel_index(t->chans, {flow, dv.id, peer_dev}))];
  port_ptr(t, src, mb, sport, cs, &sp, &sb);
  cudaEvent_t ready = next_event(t);
  JANUS_CUDA(cudaEventRecord(ready, lane_stream(t, dv, mb)));
  JANUS_CUDA(cudaStreamWaitEvent(cs, ready, 0));
  t->p2p_bytes += static_cast<int64_t>(sb);
  float* dp;
  size_t db;
  port_ptr(t, dst, mb, dport, cs, &dp, &db);
  if (db != sb) throw state_error("port size mismatch between channel ends");
  JANUS_CUDA(cudaMemcpyAsync(dp, sp, sb, cudaMemcpyDeviceToDevice, cs));
  cudaEvent_t done = next_event(t);
  JANUS_CUDA(cudaEventRecord(done, cs));
  t->delivered[{flow, mb, from_b, to_b}] = done;
}

void do_recv(janus_trainer* t, VDev& dv, int flow, int mb, janus_stage* dst, int dport, int from_b, int to_b,
             int peer_dev, size_t bytes) {
  if (t->local) {
    const auto it = t->delivered.find({flow, mb, from_b, to_b});
    if (it == t->delivered.end()) throw deadlock_error("receive issued before its send (issue order)");
    JANUS_CUDA(cudaStreamWaitEvent(lane_stream(t, dv, mb), it->second, 0));
    t->delivered.erase(it);
  } else {
    float* dp;
    size_t db;
    port_ptr(t, dst, mb, dport, t->chan_stream[static_cast<size_t>(channel_index(t->chans, {flow, peer_dev, dv.id}))], &dp, &db);
    if (db != bytes) throw state_error("port size mismatch between channel ends");
    chan_recv(t, dv, flow, mb, dp, db, peer_dev);
  }
}

// 1F1B-2nd mirror transfers (not IR instructions: implied by recompute /
// replicated parameters).  Act: E_b block input -> F_b.
void mirror_act_send(janus_trainer* t, VDev& dv, int b, int mb) {
  if (b == 0) return;  // block 0 starts at the embedding: no input
  do_send(t, dv, kFlowMirror + (b & 1), mb, t->E[static_cast<size_t>(b)], JANUS_PORT_ACT_IN, t->F[static_cast<size_t>(b)],
          JANUS_PORT_ACT_IN, b, b, t->F_dev[static_cast<size_t>(b)]);
}
void mirror_act_recv(janus_trainer* t, VDev& dv, int b, int mb) {
  if (b == 0) return;
  do_recv(t, dv, kFlowMirror + (b & 1), mb, t->F[static_cast<size_t>(b)], JANUS_PORT_ACT_IN, b, b, t->E_dev[static_cast<size_t>(b)],
          port_bytes_for(t, b, JANUS_PORT_ACT_IN, mb));
}

// Back: F_b's injection-only block-input cotangent -> E_b (added after its BE).
void mirror_back_send(janus_trainer* t, VDev& dv, int b, int mb) {
  if (b == 0) return;
  janus_stage* f = t->F[static_cast<size_t>(b)];
  float* sp;
  size_t sb;
  if (!t->local) {
    const int c = channel_index(t->chans, {kFlowMirrorBack + (b & 1), dv.id, t->E_dev[static_cast<size_t>(b)]});
    port_ptr(t, f, mb, JANUS_PORT_BADJ_OUT, t->chan_stream[static_cast<size_t>(c)], &sp, &sb);
    return chan_send(t, dv, kFlowMirrorBack + (b & 1), mb, sp, sb, t->E_dev[static_cast<size_t>(b)]);
  }
  cudaStream_t cs = t->chan_stream[static_cast<size_t>(
      channel_index(t->chans, {kFlowMirrorBack + (b & 1), dv.id, t->E_dev[static_cast<size_t>(b)]}))];
  port_ptr(t, f, mb, JANUS_PORT_BADJ_OUT, cs, &sp, &sb);
  cudaEvent_t ready = next_event(t);
  JANUS_CUDA(cudaEventRecord(ready, lane_stream(t, dv, mb)));
  JANUS_CUDA(cudaStreamWaitEvent(cs, ready, 0));
  t->p2p_bytes += static_cast<int64_t>(sb);
  float* buf = t->mirror_buf[static_cast<size_t>(b) * t->ed.n_micro_batches + mb];
  JANUS_CUDA(cudaMemcpyAsync(buf, sp, sb, cudaMemcpyDeviceToDevice, cs));
  cudaEvent_t done = next_event(t);
  JANUS_CUDA(cudaEventRecord(done, cs));
  t->delivered[{kFlowMirrorBack, mb, b, b}] = done;
}
void mirror_back_recv_add(janus_trainer* t, VDev& dv, int b, int mb) {
  if (b == 0) return;
  janus_stage* e = t->E[static_cast<size_t>(b)];
  float* dp;
  size_t db;
  port_ptr(t, e, mb, JANUS_PORT_BADJ_OUT, lane_stream(t, dv, mb), &dp, &db);
  float* buf = t->mirror_buf[static_cast<size_t>(b) * t->ed.n_micro_batches + mb];
  if (t->local) {
    const auto it = t->delivered.find({kFlowMirrorBack, mb, b, b});
    if (it == t->delivered.end()) throw deadlock_error("mirror cotangent not sent before BE");
    JANUS_CUDA(cudaStreamWaitEvent(lane_stream(t, dv, mb), it->second, 0));
    t->delivered.erase(it);
  } else {
    chan_recv(t, dv, kFlowMirrorBack + (b & 1), mb, buf, db, t->F_dev[static_cast<size_t>(b)]);
  }
  add_into(dp, buf, static_cast<int64_t>(db / sizeof(float)), lane_stream(t, dv, mb));
}

// Pass 3 pruned the comm pair between adjacent virtual stages that share a
// device (transform.hpp:124-136).  When they are different stage objects
// (1F1B-2nd: two blocks per device) the payload still has to move: a local
// port copy on the compute stream, in list order.
void local_handoff(janus_trainer* t, VDev& dv, int mb, int from_vs, int to_vs) {
  const int P = t->P, S = 2 * P;
  if (to_vs < 0 || to_vs >= S) return;
  if (t->sched.stage_map[static_cast<size_t>(from_vs)] != t->sched.stage_map[static_cast<size_t>(to_vs)]) return;
  if ((from_vs == P - 1 && to_vs == P) || (from_vs == P && to_vs == P - 1)) return;  // fold point: same block
  const bool fwd = to_vs == from_vs + 1;
  janus_stage *src, *dst;
  int sp, dp;
  if (fwd && to_vs < P) {  // FE chain
    src = t->E[static_cast<size_t>(from_vs)], dst = t->E[static_cast<size_t>(to_vs)], sp = JANUS_PORT_ACT_OUT, dp = JANUS_PORT_ACT_IN;
  } else if (fwd) {  // FF chain (blocks descending)
    src = t->F[static_cast<size_t>(block_of(t, from_vs))], dst = t->F[static_cast<size_t>(block_of(t, to_vs))];
    sp = JANUS_PORT_ADJ_OUT, dp = JANUS_PORT_ADJ_IN;
  } else if (to_vs >= P) {  // BF chain (blocks ascending)
    src = t->F[static_cast<size_t>(block_of(t, from_vs))], dst = t->F[static_cast<size_t>(block_of(t, to_vs))];
    sp = JANUS_PORT_TAN_OUT, dp = JANUS_PORT_TAN_IN;
  } else {  // BE chain
    src = t->E[static_cast<size_t>(from_vs)], dst = t->E[static_cast<size_t>(to_vs)], sp = JANUS_PORT_BADJ_OUT, dp = JANUS_PORT_BADJ_IN;
  }
  if (src == dst) return;
  float *a, *b;
  size_t na, nb;
  port_ptr(t, src, mb, sp, lane_stream(t, dv, mb), &a, &na);
  port_ptr(t, dst, mb, dp, lane_stream(t, dv, mb), &b, &nb);
  if (na != nb) throw state_error("local hand-off size mismatch");
  JANUS_CUDA(cudaMemcpyAsync(b, a, na, cudaMemcpyDeviceToDevice, lane_stream(t, dv, mb)));
}

// ------------------------------------------------------------ one instruction
void timed(janus_trainer* t, VDev& dv, const Instruction& in, auto&& body) {
  if (!t->recording) {
    body();
    return;
  }
  Rec r{in.device, static_cast<int>(in.kind), in.micro_batch, nullptr, nullptr};
  JANUS_CUDA(cudaEventCreate(&r.a));
  JANUS_CUDA(cudaEventCreate(&r.b));
  cudaStream_t cs = lane_stream(t, dv, in.micro_batch);
  JANUS_CUDA(cudaEventRecord(r.a, cs));
  body();
  JANUS_CUDA(cudaEventRecord(r.b, cs));
  t->recs.push_back(r);
}

void execute(janus_trainer* t, const Instruction& in, const janus_opt& opt) {
  VDev& dv = vdev(t, in.device);
  const int mb = in.micro_batch;
  cudaStream_t cs = lane_stream(t, dv, mb);
  const int ln = lane_index(dv, mb);
  switch (in.kind) {
    case InstrKind::LM:
      return;  // geometry is uploaded to every stage by janus_trainer_load
    case InstrKind::FE: {
      const int b = block_of(t, in.virtual_stage);
      janus_stage* e = t->E[static_cast<size_t>(b)];
      timed(t, dv, in, [&] { stage_fe(e, mb, slot_of(t, e, mb, cs), cs, ln); });
      local_handoff(t, dv, mb, in.virtual_stage, in.virtual_stage + 1);
      if (t->onef1b) mirror_act_send(t, dv, b, mb);
      return;
    }
    case InstrKind::FF: {
      const int b = block_of(t, in.virtual_stage);
      janus_stage* f = t->F[static_cast<size_t>(b)];
      if (t->onef1b) mirror_act_recv(t, dv, b, mb);
      timed(t, dv, in, [&] {
        const int sl = slot_of(t, f, mb, cs);
        if (in.has_flag(kFlagRecompute)) stage_fe(f, mb, sl, cs, ln);  // regenerate FE activations
        stage_ff(f, mb, sl, cs, ln);
      });
      local_handoff(t, dv, mb, in.virtual_stage, in.virtual_stage + 1);
      return;
    }
    case InstrKind::BF: {
      const int b = block_of(t, in.virtual_stage);
      janus_stage* f = t->F[static_cast<size_t>(b)];
      timed(t, dv, in, [&] {
        const int sl = slot_of(t, f, mb, cs);
        stage_bf(f, mb, sl, cs, ln);
        if (t->onef1b) stage_be(f, mb, sl, cs, /*inj_only=*/true, ln);
      });
      if (t->onef1b) mirror_back_send(t, dv, b, mb);
      local_handoff(t, dv, mb, in.virtual_stage, in.virtual_stage - 1);
      return;
    }
    case InstrKind::BE: {
      const int b = block_of(t, in.virtual_stage);
      timed(t, dv, in, [&] {
        janus_stage* e = t->E[static_cast<size_t>(b)];
        stage_be(e, mb, slot_of(t, e, mb, cs), cs, false, ln);
        if (t->onef1b) mirror_back_recv_add(t, dv, b, mb);
      });
      local_handoff(t, dv, mb, in.virtual_stage, in.virtual_stage - 1);
      return;
    }
    case InstrKind::OS: {
      if (t->local) return;  // local mode: optimizer runs after the join (finalize_local)
      for (size_t l = 1; l < dv.lane.size(); ++l) {  // all micro-batch lanes must be done
        cudaEvent_t e = next_event(t);
        JANUS_CUDA(cudaEventRecord(e, dv.lane[l]));
        JANUS_CUDA(cudaStreamWaitEvent(dv.compute, e, 0));
      }
      timed(t, dv, in, [&] {
        std::vector<janus_stage*> mine;  // this rank's objects, block order
        for (int b = 0; b < t->P; ++b) {
          if (t->E[static_cast<size_t>(b)]) mine.push_back(t->E[static_cast<size_t>(b)]);
          if (t->onef1b && t->F[static_cast<size_t>(b)]) mine.push_back(t->F[static_cast<size_t>(b)]);
        }
        for (janus_stage* st : mine) stage_reduce_grads(st, dv.compute);
        if (t->onef1b)  // replicated parameters: energy and force copies sum their grads
          for (janus_stage* st : mine) t->xport->allreduce(0, st->grad, static_cast<size_t>(st->n_params), dv.compute);
        if (t->ed.dp_degree > 1)  // PP x DP: replicas of this stage sum their grads (AR before OS)
          for (janus_stage* st : mine) t->xport->allreduce(1, st->grad, static_cast<size_t>(st->n_params), dv.compute);
        for (janus_stage* st : mine) stage_optimizer(st, opt, dv.compute, t->dopt);
      });
      return;
    }
    case InstrKind::AR:
      return;  // pairwise / DP all-reduce is part of OS (both ends participate)
    default:
      break;
  }
  // point-to-point
  int flow, fb, tb;
  End src, dst;
  if (!route(t, in, &flow, &src, &dst, &fb, &tb)) return;
  if (is_send(in.kind)) {
    do_send(t, dv, flow, mb, src.st, src.port, dst.st, dst.port, fb, tb, in.peer_device);
  } else {
    do_recv(t, dv, flow, mb, dst.st, dst.port, fb, tb, in.peer_device, port_bytes_for(t, tb, dst.port, mb));
  }
}

// Issue one full step on the streams (no host synchronisation inside).
void issue_step(janus_trainer* t, const janus_opt& opt) {
  t->pool_next = 0;
  t->delivered.clear();
  t->p2p_bytes = 0;
  t->slot_waited.clear();
  t->slot_last.clear();
  size_t pos = 0;
  auto release = [&] {  // occupants whose last use was this instruction hand their slot on
    for (const auto& k : t->slotplan.release_after[pos])
      JANUS_CUDA(cudaEventRecord(t->rel_ev.at(k), t->slot_last.at(k)));
    ++pos;
  };
  if (t->local) {
    for (int idx : t->order) {
      execute(t, *t->graph.flat[static_cast<size_t>(idx)], opt);
      release();
    }
  } else {
    for (const Instruction& in : t->sched.device_lists[static_cast<size_t>(t->my_dev)]) {
      t->last_comm = nullptr;
      if (t->hang_s > 0) {
        std::lock_guard<std::mutex> g(t->probe_mu);
        t->last_issued = std::string(to_string(in.kind)) + " mb " + std::to_string(in.micro_batch) + " (list index " +
                         std::to_string(t->issued.load()) + ")";
      }
      execute(t, in, opt);
      release();
      ++t->issued;
      if (t->hang_s > 0) {
        cudaStream_t s = t->last_comm ? t->last_comm : lane_stream(t, t->devs[0], in.micro_batch);
        cudaEvent_t e;
        JANUS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        JANUS_CUDA(cudaEventRecord(e, s));
        std::lock_guard<std::mutex> g(t->probe_mu);
        t->probes.push_back({static_cast<int>(in.kind), in.micro_batch, in.device, s, e});
      }
    }
  }
}

// JANUS_HANG_REPORT: the first issued instruction per stream that has not finished
std::string hang_report(janus_trainer* t) {
  std::lock_guard<std::mutex> g(t->probe_mu);
  std::string rep = "rank " + std::to_string(t->rank) + ": step did not finish (" + std::to_string(t->probes.size()) +
                    " instructions issued); first unfinished instruction per stream:\n";
  std::map<cudaStream_t, bool> seen;
  for (size_t x = 0; x < t->probes.size(); ++x) {
    const auto& p = t->probes[x];
    if (seen[p.s] || cudaEventQuery(p.e) == cudaSuccess) continue;
    seen[p.s] = true;
    std::string sname = "?";
    for (size_t l = 0; l < t->devs[0].lane.size(); ++l)
      if (t->devs[0].lane[l] == p.s) sname = "lane" + std::to_string(l);
    for (size_t c = 0; c < t->chan_stream.size(); ++c)
      if (t->chan_stream[c] == p.s) sname = "chan" + std::to_string(c);
    rep += "  #" + std::to_string(x) + " " + std::string(to_string(static_cast<InstrKind>(p.kind))) + " mb " +
           std::to_string(p.mb) + " dev " + std::to_string(p.dev) + " on " + sname + "\n";
  }
  return rep;
}

// A watchdog per step (the host itself may block inside the issue loop once
// the device stops draining its queues): after hang_s seconds without the
// step being waited for, print the report and end the process.
void hang_watchdog(janus_trainer* t, int64_t step) {
  std::shared_ptr<std::atomic<bool>> alive = t->alive;  // the trainer may be destroyed before this wakes
  const double hang_s = t->hang_s;
  std::thread([t, step, alive, hang_s] {
    std::this_thread::sleep_for(std::chrono::duration<double>(hang_s));
    if (!alive->load() || t->waited.load() > step) return;
    {  // host-side facts first: CUDA calls below may block behind a stuck launch
      const int64_t n = t->issued.load();
      std::fprintf(stderr, "rank %d: step %lld not done after %.0f s; %lld instructions issued, last: %s\n", t->rank,
                   static_cast<long long>(step), t->hang_s, static_cast<long long>(n), t->last_issued.c_str());
      std::fflush(stderr);
    }
    if (t->xport) {
      const std::string x = t->xport->debug_state();  // host-only in same-process mode
      std::fprintf(stderr, "rank %d transport:\n%s", t->rank, x.c_str());
      std::fflush(stderr);
    }
    const std::string rep = hang_report(t);
    std::fprintf(stderr, "%s", rep.c_str());
    std::fflush(stderr);
    std::this_thread::sleep_for(std::chrono::seconds(3));  // let the other ranks of this process report too
    std::_Exit(3);
  }).detach();
}

void hang_wait(janus_trainer* t, cudaEvent_t ev) {
  JANUS_CUDA(cudaEventSynchronize(ev));
  if (t->hang_s <= 0) return;
  ++t->waited;
  std::lock_guard<std::mutex> g(t->probe_mu);
  for (auto& p : t->probes) cudaEventDestroy(p.e);
  t->probes.clear();
}

void fork_join_begin(janus_trainer* t) {
  JANUS_CUDA(cudaEventRecord(t->anchor, t->root));
  for (auto& d : t->devs) {
    for (cudaStream_t l : d.lane) JANUS_CUDA(cudaStreamWaitEvent(l, t->anchor, 0));
    JANUS_CUDA(cudaStreamWaitEvent(d.send, t->anchor, 0));
    JANUS_CUDA(cudaStreamWaitEvent(d.recv, t->anchor, 0));
  }
  for (cudaStream_t s : t->chan_stream)
    if (s) JANUS_CUDA(cudaStreamWaitEvent(s, t->anchor, 0));
}

void fork_join_end(janus_trainer* t) {
  for (auto& d : t->devs) {
    std::vector<cudaStream_t> all = d.lane;
    all.push_back(d.send);
    all.push_back(d.recv);
    for (cudaStream_t s : t->chan_stream)
      if (s) all.push_back(s);
    for (cudaStream_t s : all) {
      cudaEvent_t e = next_event(t);
      JANUS_CUDA(cudaEventRecord(e, s));
      JANUS_CUDA(cudaStreamWaitEvent(t->root, e, 0));
    }
  }
}

// Local mode OS for every block after all streams joined on root: ledger
// reduce, 1F1B-2nd pairwise sum of the replicated copies, Adam.
void finalize_local(janus_trainer* t, const janus_opt& opt) {
  for (int b = 0; b < t->P; ++b) {
    janus_stage* e = t->E[static_cast<size_t>(b)];
    janus_stage* f = t->F[static_cast<size_t>(b)];
    stage_reduce_grads(e, t->root);
    if (f != e) {
      stage_reduce_grads(f, t->root);
      add_into(e->grad, f->grad, e->n_params, t->root);
      JANUS_CUDA(cudaMemcpyAsync(f->grad, e->grad, sizeof(float) * e->n_params, cudaMemcpyDeviceToDevice, t->root));
      stage_optimizer(f, opt, t->root, t->dopt);
    }
    stage_optimizer(e, opt, t->root, t->dopt);
  }
}

// The per-rank path blocks streams on peers (NCCL P2P kernels, or the IPC
// transport's waits), which is only safe when (a) every kernel is loaded
// before the first step — lazy module loading (CUDA 12 default) loads a
// kernel at its first launch and can wait for a running peer-blocked kernel:
// the first step then deadlocks — and (b) each stream of this rank owns a
// hardware work queue: a stream waiting on a peer at the head of a shared
// queue stalls the unrelated streams behind it, which may be what the peer
// waits for.  Both are process-wide settings read at context creation, so
// the application sets them; the trainer refuses to run without them.
// streams held by the per-rank trainers of this process: ranks run as threads
// of one process share its context's hardware queues
std::atomic<int> g_peer_streams{0};

void check_per_rank_runtime(const janus_trainer* t, int n_streams) {
  using GetMode = CUresult (*)(CUmoduleLoadingMode*);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuModuleGetLoadingMode", &fn, cudaEnableDefault, &q) == cudaSuccess && fn &&
      q == cudaDriverEntryPointSuccess) {
    CUmoduleLoadingMode mode;
    if (reinterpret_cast<GetMode>(fn)(&mode) == CUDA_SUCCESS && mode == CU_MODULE_LAZY_LOADING)
      throw config_error("per-rank mode needs eager kernel loading: set CUDA_MODULE_LOADING=EAGER before the first "
                         "CUDA call of the process (lazy loading can deadlock the first step against a blocked peer)");
  }
  const char* e = std::getenv("CUDA_DEVICE_MAX_CONNECTIONS");
  const int conn = e ? std::atoi(e) : 8;
  if (conn < n_streams)
    throw config_error("per-rank mode: rank " + std::to_string(t->rank) + " uses " + std::to_string(n_streams) +
                       " streams but CUDA_DEVICE_MAX_CONNECTIONS=" + std::to_string(conn) +
                       " hardware queues; set it to >= " + std::to_string(n_streams) +
                       " (max 32) before the first CUDA call, or use fewer lanes");
  const int before = g_peer_streams.fetch_add(n_streams);
  if (before + n_streams > conn) {
    g_peer_streams.fetch_sub(n_streams);
    throw config_error("per-rank mode: the ranks of this process use " + std::to_string(before + n_streams) +
                       " streams in one CUDA context but CUDA_DEVICE_MAX_CONNECTIONS=" + std::to_string(conn) +
                       " hardware queues (a peer-blocked stream would stall the streams sharing its queue); run "
                       "fewer ranks per process or fewer lanes");
  }
}

}  // namespace

// ================================================================ create
janus_trainer* trainer_create(const janus_exec_desc& ed, const janus_stage_desc& sd, const float* all_params,
                              janus_comm* comm, int rank, const char* schedule_text) {
  auto t = std::make_unique<janus_trainer>();
  t->ed = ed;
  t->sd = sd;
  if (const char* h = std::getenv("JANUS_HANG_REPORT")) t->hang_s = std::atof(h);
  t->P = ed.n_stages;
  t->method = ed.method;
  t->local = ed.local_stages != 0;
  t->onef1b = ed.method == 2;
  Schedule given;
  if (schedule_text) {  // a caller's schedule (train.hpp): its stage map decides the layout
    given = deserialize(schedule_text);
    if (given.pipeline_degree != ed.n_stages || given.num_micro_batches != ed.n_micro_batches)
      throw config_error("schedule text: P / micro-batches differ from the exec desc");
    if (given.order != ScheduleOrder::second_order) throw config_error("schedule text: a second-order schedule is required");
    bool folded = true;
    for (int b = 0; b < t->P; ++b)
      folded = folded && given.stage_map[static_cast<size_t>(b)] == given.stage_map[static_cast<size_t>(2 * t->P - 1 - b)];
    t->onef1b = !folded;
  }
  if (ed.dp_degree < 1) t->ed.dp_degree = 1;
  if (ed.lanes < 1) t->ed.lanes = 1;
  if (ed.n_micro_batches < 1) throw domain_error("n_micro_batches must be >= 1");
  {  // lanes share the device's hardware work queues (CUDA default 8); the library
     // leaves the environment to the application and only says so
    const char* e = std::getenv("CUDA_DEVICE_MAX_CONNECTIONS");
    const int conn = e ? std::atoi(e) : 8;
    static bool warned = false;
    if (t->ed.lanes > conn && !warned) {
      warned = true;
      std::fprintf(stderr, "janus: %d compute lanes share %d hardware work queues (set CUDA_DEVICE_MAX_CONNECTIONS=%d "
                   "before the first CUDA context for one queue per lane)\n", t->ed.lanes, conn, std::min(32, t->ed.lanes));
    }
  }
  if (!t->local && !comm) throw config_error("NCCL mode needs a janus_comm");
  if (t->local && t->ed.dp_degree != 1) throw config_error("data parallelism needs NCCL mode");
  switch (schedule_text ? -1 : ed.method) {
    case -1: t->sched = std::move(given); break;
    case 0: t->sched = symfold(t->P, ed.n_micro_batches); break;
    case 1: {
      WaveKOptions wo;  // measured phase times when the caller has them (SPEC.md:578-637 tuner input)
      if (ed.phase_us[0] > 0 || ed.phase_us[1] > 0 || ed.phase_us[2] > 0 || ed.phase_us[3] > 0)
        wo.times = PhaseTimes{ed.phase_us[0], ed.phase_us[1], ed.phase_us[2], ed.phase_us[3]};
      t->sched = wavek(t->P, ed.n_micro_batches, ed.wavek_k, wo);
      break;
    }
    case 2: t->sched = onef1b_2nd(t->P, ed.n_micro_batches); break;
    case 4: t->sched = hanayo_2nd(t->P, ed.n_micro_batches); break;  // V-shape + wave order, FF recompute
    default: throw domain_error("unknown method");
  }
  const ValidationReport vr = validate_schedule(t->sched);
  if (!vr.ok()) throw state_error("generated schedule failed validation");
  // per-channel order must agree on both ends (NCCL pairs sends/receives in issue order)
  {
    std::map<std::tuple<int, char, int, int>, std::vector<int>> snd, rcv;
    for (const auto& dl : t->sched.device_lists)
      for (const Instruction& in : dl) {
        if (!is_comm(in.kind)) continue;
        const int pay = is_activation_comm(in.kind) ? 0 : 1;
        const int from = is_send(in.kind) ? in.device : in.peer_device, to = is_send(in.kind) ? in.peer_device : in.device;
        (is_send(in.kind) ? snd : rcv)[{pay, comm_suffix(in.kind), from, to}].push_back(in.micro_batch);
      }
    if (snd != rcv) throw deadlock_error("channel micro-batch order differs between send and receive ends");
  }
  ModelConfig mc;
  mc.L = sd.model.L;
  mc.H = sd.model.H;
  mc.R = sd.model.R;
  mc.n_species = sd.model.n_species;
  t->plan = partition_units(mc, t->P);
  t->E.assign(static_cast<size_t>(t->P), nullptr);
  t->F.assign(static_cast<size_t>(t->P), nullptr);
  t->E_dev.resize(static_cast<size_t>(t->P));
  t->F_dev.resize(static_cast<size_t>(t->P));
  for (int b = 0; b < t->P; ++b) {
    t->E_dev[static_cast<size_t>(b)] = t->sched.stage_map[static_cast<size_t>(b)];
    t->F_dev[static_cast<size_t>(b)] = t->sched.stage_map[static_cast<size_t>(2 * t->P - 1 - b)];
  }
  if (!t->local) {
    t->comm = comm;
    t->rank = rank;
    t->replica = rank / t->P;
    t->my_dev = rank % t->P;
    if (comm->nranks != t->P * t->ed.dp_degree) throw config_error("communicator size != P * dp_degree");
  }
  JANUS_CUDA(cudaSetDevice(sd.device));
  const int nd = t->local ? t->P : 1;
  t->devs.resize(static_cast<size_t>(nd));
  for (int d = 0; d < nd; ++d) {
    VDev& v = t->devs[static_cast<size_t>(d)];
    v.id = t->local ? d : t->my_dev;
    v.lane.resize(static_cast<size_t>(std::max(1, t->ed.lanes)));
    for (auto& l : v.lane) JANUS_CUDA(cudaStreamCreateWithFlags(&l, cudaStreamNonBlocking));
    v.compute = v.lane[0];
    JANUS_CUDA(cudaStreamCreateWithFlags(&v.send, cudaStreamNonBlocking));
    JANUS_CUDA(cudaStreamCreateWithFlags(&v.recv, cudaStreamNonBlocking));
  }
  JANUS_CUDA(cudaStreamCreateWithFlags(&t->root, cudaStreamNonBlocking));
  JANUS_CUDA(cudaEventCreate(&t->anchor));
  JANUS_CUDA(cudaEventCreate(&t->finish));
  for (int q = 0; q < 2; ++q) {
    JANUS_CUDA(cudaEventCreate(&t->anchor_q[q]));
    JANUS_CUDA(cudaEventCreate(&t->finish_q[q]));
    JANUS_CUDA(cudaEventCreateWithFlags(&t->done_q[q], cudaEventDisableTiming));
    JANUS_CUDA(cudaMalloc(&t->loss_snap[q], sizeof(float) * 4 * static_cast<size_t>(std::max(1, ed.n_micro_batches))));
  }
  JANUS_CUDA(cudaMalloc(&t->dopt, sizeof(janus_opt)));
  // local issue order: a topological order of the full DAG (seq + data edges),
  // so every send is issued before its receive.
  t->graph = build_dependencies(t->sched);
  if (t->local) {
    t->order = local_issue_order(t->graph);
    t->chans = schedule_channels(t->sched, t->P, t->onef1b);  // one copy stream per channel (do_send)
    t->chan_stream.assign(t->chans.size(), nullptr);
    for (auto& cs : t->chan_stream) JANUS_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  }
  // activation slot pools: sized by the micro-batches live at once on each
  // stage object in this process's issue order (include/janus/slots.hpp)
  {
    std::vector<const Instruction*> ord;
    if (t->local)
      for (int idx : t->order) ord.push_back(t->graph.flat[static_cast<size_t>(idx)]);
    else
      for (const Instruction& in : t->sched.device_lists[static_cast<size_t>(t->my_dev)]) ord.push_back(&in);
    const int P = t->P;
    auto held = [&](int obj) {
      if (t->local) return true;
      const int b = obj < P ? obj : obj - P;
      return obj < P ? t->E_dev[static_cast<size_t>(b)] == t->my_dev : t->F_dev[static_cast<size_t>(b)] == t->my_dev;
    };
    t->slotplan = plan_slots(ord, t->sched, P, t->onef1b, t->local, ed.n_micro_batches, ed.unfolded_slots != 0, held,
                             t->ed.lanes);
  }
  auto make = [&](int b, int obj) {
    janus_stage_desc d = sd;
    d.unit_begin = t->plan.blocks[static_cast<size_t>(b)].first;
    d.unit_end = t->plan.blocks[static_cast<size_t>(b)].second;
    d.n_micro_batches = ed.n_micro_batches;
    d.n_slots = std::max(1, t->slotplan.n_slots[static_cast<size_t>(obj)]);
    d.n_lanes = std::max(1, t->ed.lanes);
    const int64_t off = mc.unit_param_offset(d.unit_begin);
    janus_stage* st = stage_create(d, all_params + off);
    t->owned.push_back(st);
    t->obj_of[st] = obj;
    return st;
  };
  for (int b = 0; b < t->P; ++b) {
    const bool e_here = t->local || t->E_dev[static_cast<size_t>(b)] == t->my_dev;
    const bool f_here = t->local || t->F_dev[static_cast<size_t>(b)] == t->my_dev;
    if (e_here) t->E[static_cast<size_t>(b)] = make(b, slot_obj_energy(b, t->P, t->onef1b));
    if (f_here) t->F[static_cast<size_t>(b)] = (t->onef1b ? make(b, slot_obj_force(b, t->P, t->onef1b)) : t->E[static_cast<size_t>(b)]);
  }
  for (const auto& kv : t->slotplan.prev)
    if (kv.second >= 0 && !t->rel_ev.count({kv.first.first, kv.second})) {
      cudaEvent_t e;
      JANUS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      t->rel_ev[{kv.first.first, kv.second}] = e;
    }
  if (t->onef1b) {
    t->mirror_buf.assign(static_cast<size_t>(t->P) * ed.n_micro_batches, nullptr);
    const size_t bytes = sizeof(float) * static_cast<size_t>(sd.max_atoms) * sd.model.H * 2;
    for (int b = 1; b < t->P; ++b) {
      if (!(t->local || t->E_dev[static_cast<size_t>(b)] == t->my_dev)) continue;
      for (int m = 0; m < ed.n_micro_batches; ++m) {
        void* p;
        JANUS_CUDA(cudaMalloc(&p, bytes));
        t->allocs.push_back(p);
        t->mirror_buf[static_cast<size_t>(b) * ed.n_micro_batches + m] = static_cast<float*>(p);
      }
    }
  }
  if (!t->local) {
    // the per-rank program must be deadlock-free under blocking P2P before anything is issued
    const auto progs = build_programs(t->sched, t->P, t->onef1b, t->ed.lanes, t->ed.dp_degree, StreamLayout::kPerChannel);
    const RendezvousReport rr = simulate(progs, t->P, t->sched, t->onef1b);
    if (!rr.ok) throw deadlock_error("per-rank issue program cannot complete under blocking P2P:\n" + rr.stuck);
    TransportPlan tp;
    tp.chans = schedule_channels(t->sched, t->P, t->onef1b);
    tp.P = t->P;
    tp.dp = t->ed.dp_degree;
    tp.rank = rank;
    tp.pair_group = t->onef1b;
    const int d = t->my_dev, base = t->replica * t->P;
    if (t->onef1b) {  // ranks holding the two copies of this rank's blocks
      for (int b = 0; b < t->P; ++b)
        if (t->E_dev[static_cast<size_t>(b)] == d || t->F_dev[static_cast<size_t>(b)] == d) {
          tp.pair_members.push_back(base + t->E_dev[static_cast<size_t>(b)]);
          tp.pair_members.push_back(base + t->F_dev[static_cast<size_t>(b)]);
        }
      std::sort(tp.pair_members.begin(), tp.pair_members.end());
      tp.pair_members.erase(std::unique(tp.pair_members.begin(), tp.pair_members.end()), tp.pair_members.end());
      if (tp.pair_members.size() != 2) throw config_error("1F1B-2nd: a device must pair with exactly one other");
    }
    for (int q = 0; q < t->ed.dp_degree; ++q) tp.dp_members.push_back(q * t->P + d);
    tp.max_payload = sizeof(float) * (static_cast<size_t>(sd.max_atoms) * sd.model.H * 2 + 3 * static_cast<size_t>(sd.max_atoms));
    // the IPC region layout must agree on every rank, so size the all-reduce
    // staging from the whole partition, not from the blocks this rank holds
    for (const auto& blk : t->plan.blocks)
      tp.max_allreduce = std::max(tp.max_allreduce, sizeof(float) * static_cast<size_t>(mc.unit_param_offset(blk.second) - mc.unit_param_offset(blk.first)));
    t->chans = tp.chans;
    t->chan_stream.assign(t->chans.size(), nullptr);
    for (size_t c = 0; c < t->chans.size(); ++c)
      if (t->chans[c].from == d || t->chans[c].to == d) JANUS_CUDA(cudaStreamCreateWithFlags(&t->chan_stream[c], cudaStreamNonBlocking));
    int n_streams = static_cast<int>(t->devs[0].lane.size()) + 4;  // lanes, send, recv, root, load
    for (cudaStream_t cs : t->chan_stream) n_streams += cs ? 1 : 0;
    check_per_rank_runtime(t.get(), n_streams);
    t->reserved_streams = n_streams;
    t->xport = make_transport(comm, tp);
  }
  t->n_atoms.assign(static_cast<size_t>(ed.n_micro_batches), 0);
  JANUS_CUDA(cudaDeviceSynchronize());
  return t.release();
}

void trainer_destroy(janus_trainer* t) {
  if (!t) return;
  t->alive->store(false);
  if (t->reserved_streams) g_peer_streams.fetch_sub(t->reserved_streams);
  cudaSetDevice(t->sd.device);
  cudaDeviceSynchronize();
  if (t->gexec) cudaGraphExecDestroy(t->gexec);
  if (t->gexec_alt) cudaGraphExecDestroy(t->gexec_alt);
  if (t->load_stream) cudaStreamDestroy(t->load_stream);
  if (t->load_done) cudaEventDestroy(t->load_done);
  for (cudaEvent_t e : t->step_end)
    if (e) cudaEventDestroy(e);
  t->xport.reset();
  for (cudaStream_t s : t->chan_stream)
    if (s) cudaStreamDestroy(s);
  for (janus_stage* s : t->owned) stage_destroy(s);
  for (void* p : t->allocs) cudaFree(p);
  for (cudaEvent_t e : t->pool) cudaEventDestroy(e);
  for (auto& kv : t->rel_ev) cudaEventDestroy(kv.second);
  for (auto& r : t->recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto& d : t->devs) {
    for (cudaStream_t l : d.lane) cudaStreamDestroy(l);
    cudaStreamDestroy(d.send);
    cudaStreamDestroy(d.recv);
  }
  delete t->lm;
  if (t->root) cudaStreamDestroy(t->root);
  if (t->anchor) cudaEventDestroy(t->anchor);
  if (t->finish) cudaEventDestroy(t->finish);
  for (int q = 0; q < 2; ++q) {
    if (t->anchor_q[q]) cudaEventDestroy(t->anchor_q[q]);
    if (t->finish_q[q]) cudaEventDestroy(t->finish_q[q]);
    if (t->done_q[q]) cudaEventDestroy(t->done_q[q]);
    if (t->loss_snap[q]) cudaFree(t->loss_snap[q]);
  }
  if (t->dopt) cudaFree(t->dopt);
  delete t;
}

void trainer_note_shape(janus_trainer* t, int mb, const janus_host_batch& hb, int par);
void trainer_load_many(janus_trainer* t, int n, const int* mbs, const janus_host_batch* hbs);

void trainer_load(janus_trainer* t, int mb, const janus_host_batch& hb) { trainer_load_many(t, 1, &mb, &hb); }

void trainer_load_many(janus_trainer* t, int n, const int* mbs, const janus_host_batch* hbs) {
  for (int k = 0; k < n; ++k)
    if (mbs[k] < 0 || mbs[k] >= t->ed.n_micro_batches) throw domain_error("micro-batch index out of range");
  const size_t NMB = static_cast<size_t>(t->ed.n_micro_batches);
  if (t->step_par.size() != NMB) {
    t->step_par.assign(NMB, -1);
    t->load_par.assign(NMB, -1);
  }
  if (!t->load_stream) {
    // highest priority: the neighbour-list build and geometry take SMs ahead of
    // the step in flight, so the host's one sync for the tile tables stays short
    int lo = 0, hi = 0;
    JANUS_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    JANUS_CUDA(cudaStreamCreateWithPriority(&t->load_stream, cudaStreamNonBlocking, hi));
    JANUS_CUDA(cudaEventCreateWithFlags(&t->load_done, cudaEventDisableTiming));
    for (cudaEvent_t& e : t->step_end) JANUS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  // Loads fill the geometry copy the latest step did NOT read.  Its last reader
  // is at most the step before that one, which must be done first (steps
  // complete in order on root).
  if (t->nsteps >= 2) JANUS_CUDA(cudaStreamWaitEvent(t->load_stream, t->step_end[(t->nsteps - 2) & 1], 0));
  auto par_of = [&](int mb) {
    const int sp = t->step_par[static_cast<size_t>(mb)];
    return sp < 0 ? 0 : sp ^ 1;
  };
  cudaStream_t ls = t->load_stream;
  // asynchronous on the load stream, into the geometry copies the step in
  // flight does not read (the next step_async switches to them and makes root
  // wait for the loads).  The caller's arrays must stay valid until the copies
  // run (pinned memory) or are staged by the driver (pageable memory); the
  // host-built tile tables go through the stage's double-buffered pinned staging
  std::vector<janus_host_batch> dev;
  std::vector<int> dev_mb;
  std::vector<std::vector<node::GeoJob>> jobs(t->owned.size());  // per stage: one batched geometry launch
  for (int k = 0; k < n; ++k) {
    if (hbs[k].row_ptr) {
      const int q = par_of(mbs[k]);
      for (size_t x = 0; x < t->owned.size(); ++x)
        stage_load(t->owned[x], mbs[k], hbs[k], ls, /*sync=*/false, nullptr, &jobs[x], q);
      t->load_par[static_cast<size_t>(mbs[k])] = q;
      trainer_note_shape(t, mbs[k], hbs[k], q);
    } else {
      dev.push_back(hbs[k]);
      dev_mb.push_back(mbs[k]);
    }
  }
  if (dev.empty()) {
    for (size_t x = 0; x < t->owned.size(); ++x) stage_geometry_flush(t->owned[x], jobs[x], ls);
    JANUS_CUDA(cudaEventRecord(t->load_done, ls));
    return;
  }
  // LM with the neighbour lists built on the device: ONE cell-list build over
  // all these micro-batches (their structures side by side) on the load
  // stream, beside a step in flight; each stage then cuts its batch's slice
  // into the free geometry copy on the same stream.
  if (!t->lm) {
    const int nm = t->ed.n_micro_batches;
    t->lm = new LmBuilder(nm * t->sd.max_atoms, nm * t->sd.max_struct, nm * t->sd.max_edges, t->sd.device, 2);
  }
  const int b = t->lm_par;
  t->lm_par ^= 1;
  t->lm->build(dev.data(), static_cast<int>(dev.size()), static_cast<double>(t->sd.model.r_c), b, ls);
  const int* hrow = t->lm->host_row_ptr();
  std::vector<int> rp;
  for (size_t k = 0; k < dev.size(); ++k) {
    const int a0 = t->lm->atom0(static_cast<int>(k)), N = dev[k].n_atoms;
    rp.resize(static_cast<size_t>(N) + 1);
    for (int i = 0; i <= N; ++i) rp[static_cast<size_t>(i)] = hrow[a0 + i] - hrow[a0];
    janus_host_batch hb2 = dev[k];
    hb2.row_ptr = rp.data();
    hb2.n_edges = rp[static_cast<size_t>(N)];
    hb2.col = hb2.shift = hb2.rev = nullptr;
    const DevCsrSlice sl{&t->lm->buf(b), a0, hrow[a0]};
    const int q = par_of(dev_mb[k]);
    for (size_t x = 0; x < t->owned.size(); ++x)
      stage_load(t->owned[x], dev_mb[k], hb2, ls, /*sync=*/false, &sl, &jobs[x], q);
    t->load_par[static_cast<size_t>(dev_mb[k])] = q;
    trainer_note_shape(t, dev_mb[k], hb2, q);
  }
  for (size_t x = 0; x < t->owned.size(); ++x) stage_geometry_flush(t->owned[x], jobs[x], ls);
  t->lm->release(b, ls);
  JANUS_CUDA(cudaEventRecord(t->load_done, ls));
}

void trainer_note_shape(janus_trainer* t, int mb, const janus_host_batch& hb, int par) {
  t->n_atoms[static_cast<size_t>(mb)] = hb.n_atoms;
  // a captured step graph bakes in grid sizes and copy lengths: a batch of a
  // different shape in this geometry copy drops the cached graphs
  const size_t NMB = t->n_atoms.size();
  if (t->shape.size() != 2 * NMB) t->shape.assign(2 * NMB, {-1, -1, -1, -1, -1});
  const DevGeo& g = stage_geo(t->owned.front(), mb, par);
  const std::array<int, 5> sh{hb.n_atoms, hb.n_edges, hb.n_struct, g.n_tiles, g.n_tiles_tc};
  std::array<int, 5>& cur = t->shape[static_cast<size_t>(par) * NMB + static_cast<size_t>(mb)];
  if (cur != sh) {
    cur = sh;
    if (t->gexec || t->gexec_alt) {
      if (t->inflight) JANUS_CUDA(cudaStreamSynchronize(t->root));  // the old graphs may still be running
      if (t->gexec) JANUS_CUDA(cudaGraphExecDestroy(t->gexec));
      if (t->gexec_alt) JANUS_CUDA(cudaGraphExecDestroy(t->gexec_alt));
      t->gexec = t->gexec_alt = nullptr;
      t->gkey.clear();
      t->gkey_alt.clear();
      t->kernel_count = t->kernel_count_alt = -1;
    }
  }
}

// count kernel nodes of one captured step (the gpu_launches evidence)
// Capture one step (nothing runs); instantiate it when graphs are on.  *nk =
// kernel nodes (the gpu_launches evidence).
cudaGraphExec_t capture_step(janus_trainer* t, const janus_opt& opt, int64_t* nk) {
  cudaGraph_t g;
  JANUS_CUDA(cudaStreamBeginCapture(t->root, cudaStreamCaptureModeThreadLocal));
  try {
    fork_join_begin(t);
    issue_step(t, opt);
    fork_join_end(t);
    if (t->local) finalize_local(t, opt);
  } catch (...) {
    cudaStreamEndCapture(t->root, &g);
    throw;
  }
  JANUS_CUDA(cudaStreamEndCapture(t->root, &g));
  size_t n = 0;
  JANUS_CUDA(cudaGraphGetNodes(g, nullptr, &n));
  std::vector<cudaGraphNode_t> nodes(n);
  JANUS_CUDA(cudaGraphGetNodes(g, nodes.data(), &n));
  int64_t k = 0;
  int by_type[16] = {};
  for (auto nd : nodes) {
    cudaGraphNodeType ty;
    JANUS_CUDA(cudaGraphNodeGetType(nd, &ty));
    if (ty == cudaGraphNodeTypeKernel) ++k;
    by_type[static_cast<int>(ty) & 15]++;
  }
  if (std::getenv("JANUS_GRAPH_STATS")) {  // profiling: node census of the captured step
    size_t ne = 0;
    JANUS_CUDA(cudaGraphGetEdges(g, nullptr, nullptr, &ne));
    std::fprintf(stderr, "graph nodes %zu edges %zu: kernel %d memcpy %d memset %d host %d empty %d event_wait %d event_record %d\n",
                 n, ne, by_type[cudaGraphNodeTypeKernel], by_type[cudaGraphNodeTypeMemcpy],
                 by_type[cudaGraphNodeTypeMemset], by_type[cudaGraphNodeTypeHost], by_type[cudaGraphNodeTypeEmpty],
                 by_type[cudaGraphNodeTypeWaitEvent & 15], by_type[cudaGraphNodeTypeEventRecord & 15]);
  }
  cudaGraphExec_t exec = nullptr;
  if (t->ed.use_graphs && !t->ed.record_timeline) JANUS_CUDA(cudaGraphInstantiate(&exec, g, 0));
  JANUS_CUDA(cudaGraphDestroy(g));
  *nk = k;
  return exec;
}

// Issue one step on the root stream and return without waiting: the caller may
// queue the next step's uploads (janus_trainer_load) behind it, which overlaps
// their host-side cost with this step's device time.
void trainer_step_async(janus_trainer* t, const janus_opt& opt) {
  JANUS_CUDA(cudaSetDevice(t->sd.device));
  if (t->inflight >= 2) throw state_error("two steps are already in flight (call janus_trainer_wait)");
  if (t->inflight && t->ed.record_timeline) throw state_error("a timed step is in flight (call janus_trainer_wait)");
  for (int m = 0; m < t->ed.n_micro_batches; ++m)
    if (t->n_atoms[static_cast<size_t>(m)] <= 0) throw state_error("micro-batch " + std::to_string(m) + " not loaded");
  // loads since the last step: the phases switch to the geometry copies they
  // filled, and root waits for the load stream
  bool loaded = false;
  for (size_t m = 0; m < t->load_par.size(); ++m) {
    const int q = t->load_par[m];
    if (q < 0) continue;
    for (janus_stage* st : t->owned) stage_set_parity(st, static_cast<int>(m), q);
    t->step_par[m] = q;
    t->load_par[m] = -1;
    loaded = true;
  }
  if (loaded) JANUS_CUDA(cudaStreamWaitEvent(t->root, t->load_done, 0));
  t->recording = false;  // a capture below must not record timeline events
  cudaGraphExec_t exec = nullptr;
  const bool graphs = t->ed.use_graphs && !t->ed.record_timeline;
  if (t->local && !graphs) {
    if (t->kernel_count < 0) capture_step(t, opt, &t->kernel_count);  // count only, nothing runs
  } else if (t->local) {
    // one instantiated graph per geometry-parity vector (two alternate in steady state)
    std::vector<int> key(t->step_par.begin(), t->step_par.end());
    if (t->gexec && key == t->gkey) {
      exec = t->gexec;
    } else if (t->gexec_alt && key == t->gkey_alt) {
      std::swap(t->gexec, t->gexec_alt);
      std::swap(t->gkey, t->gkey_alt);
      std::swap(t->kernel_count, t->kernel_count_alt);
      exec = t->gexec;
    } else {
      int64_t nk = 0;
      cudaGraphExec_t e = capture_step(t, opt, &nk);  // capture only, nothing runs
      if (t->gexec_alt) JANUS_CUDA(cudaGraphExecDestroy(t->gexec_alt));
      t->gexec_alt = t->gexec;
      t->gkey_alt = t->gkey;
      t->kernel_count_alt = t->kernel_count;
      t->gexec = e;
      t->gkey = key;
      t->kernel_count = nk;
      exec = e;
    }
  }
  for (auto& r : t->recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  t->recs.clear();
  t->recording = t->ed.record_timeline != 0;
  if (t->hang_s > 0) {
    t->issued = 0;
    hang_watchdog(t, t->nsteps);
  }
  const int q = static_cast<int>(t->nsteps & 1);
  // this step's optimizer hyperparameters: captured graphs read them from the
  // device buffer (pageable source: staged by the driver before the call returns)
  JANUS_CUDA(cudaMemcpyAsync(t->dopt, &opt, sizeof(janus_opt), cudaMemcpyHostToDevice, t->root));
  JANUS_CUDA(cudaEventRecord(t->anchor_q[q], t->root));
  if (exec) {
    JANUS_CUDA(cudaEventRecord(t->anchor, t->root));
    JANUS_CUDA(cudaGraphLaunch(exec, t->root));
  } else {
    fork_join_begin(t);
    issue_step(t, opt);
    fork_join_end(t);
    if (t->local) finalize_local(t, opt);
  }
  JANUS_CUDA(cudaEventRecord(t->finish, t->root));
  JANUS_CUDA(cudaEventRecord(t->finish_q[q], t->root));  // (the device time ends here)
  {  // the loss terms of this step, before the next step may overwrite them
    const size_t n2 = 2 * static_cast<size_t>(t->ed.n_micro_batches);
    janus_stage* top = t->E[static_cast<size_t>(t->P - 1)];
    janus_stage* bot = t->F[0];
    if (top) JANUS_CUDA(cudaMemcpyAsync(t->loss_snap[q], top->losses, sizeof(float) * n2, cudaMemcpyDeviceToDevice, t->root));
    if (bot) JANUS_CUDA(cudaMemcpyAsync(t->loss_snap[q] + n2, bot->losses, sizeof(float) * n2, cudaMemcpyDeviceToDevice, t->root));
  }
  JANUS_CUDA(cudaEventRecord(t->done_q[q], t->root));
  if (t->step_end[0]) JANUS_CUDA(cudaEventRecord(t->step_end[t->nsteps & 1], t->root));
  ++t->nsteps;
  ++t->inflight;
}

// Wait for the step in flight and report it (device time, bubbles, loss: the
// per-micro-batch loss terms are read back here).
void trainer_wait(janus_trainer* t, janus_step_stats* stats) {
  JANUS_CUDA(cudaSetDevice(t->sd.device));
  if (t->inflight <= 0) throw state_error("no step in flight");
  const int q = static_cast<int>((t->nsteps - t->inflight) & 1);  // the oldest step in flight
  --t->inflight;
  hang_wait(t, t->done_q[q]);
  if (t->inflight == 0) t->recording = false;
  float ms = 0.f;
  JANUS_CUDA(cudaEventElapsedTime(&ms, t->anchor_q[q], t->finish_q[q]));
  janus_step_stats s{};
  s.makespan_ms = ms;
  s.p2p_bytes = t->p2p_bytes;
  s.kernel_launches = t->kernel_count;
  if (!t->recs.empty()) {
    std::vector<double> busy(static_cast<size_t>(t->P), 0.0);
    for (auto& r : t->recs) {
      float a = 0.f;
      JANUS_CUDA(cudaEventElapsedTime(&a, r.a, r.b));
      busy[static_cast<size_t>(r.device)] += a;
    }
    double idle = 0;
    for (int d = 0; d < t->P && d < 64; ++d) {
      s.busy_ms[d] = busy[static_cast<size_t>(d)];
      idle += ms - busy[static_cast<size_t>(d)];
    }
    s.bubble_ratio = t->local ? idle / (t->P * static_cast<double>(ms)) : (ms - busy[static_cast<size_t>(t->my_dev)]) / ms;
  }
  for (size_t x = 0; x < t->owned.size(); ++x) {
    janus_stage* st = t->owned[x];
    int dev = t->local ? 0 : t->my_dev;
    for (int b = 0; b < t->P; ++b) {
      if (t->E[static_cast<size_t>(b)] == st) dev = t->E_dev[static_cast<size_t>(b)];
      else if (t->F[static_cast<size_t>(b)] == st) dev = t->F_dev[static_cast<size_t>(b)];
    }
    if (dev < 64) {
      s.peak_bytes[dev] += st->static_bytes + st->arena_bytes;
      s.act_bytes[dev] += st->pool_bytes;
      s.act_slots[dev] = std::max<int32_t>(s.act_slots[dev], static_cast<int32_t>(st->slots.size()));
    }
  }
  // losses held here: L_E on the readout stage, L_F on the stage holding block 0's force replica
  // (slot == micro-batch; one contiguous copy per stage, summed in micro-batch order)
  double loss = 0;
  {
    const int n = t->ed.n_micro_batches;
    std::vector<float> buf(4 * static_cast<size_t>(n));
    janus_stage* top = t->E[static_cast<size_t>(t->P - 1)];
    janus_stage* bot = t->F[0];
    std::vector<float> lE(static_cast<size_t>(n), 0.f), lF(static_cast<size_t>(n), 0.f);
    JANUS_CUDA(cudaMemcpy(buf.data(), t->loss_snap[q], sizeof(float) * 4 * n, cudaMemcpyDeviceToHost));
    if (top)
      for (int m = 0; m < n; ++m) lE[static_cast<size_t>(m)] = buf[2 * static_cast<size_t>(m)];
    if (bot)
      for (int m = 0; m < n; ++m) lF[static_cast<size_t>(m)] = buf[2 * static_cast<size_t>(n) + 2 * static_cast<size_t>(m) + 1];
    for (int m = 0; m < n; ++m) loss += static_cast<double>(lE[static_cast<size_t>(m)]) + lF[static_cast<size_t>(m)];
  }
  s.loss = loss;
  t->last = s;
  if (stats) *stats = s;
}

void trainer_step(janus_trainer* t, const janus_opt& opt, janus_step_stats* stats) {
  trainer_step_async(t, opt);
  trainer_wait(t, stats);
}

}  // namespace janus

namespace janus {

void trainer_timeline(janus_trainer* t, double* out, int cap, int* n) {
  *n = static_cast<int>(t->recs.size());
  for (int x = 0; x < *n && x < cap; ++x) {
    const Rec& r = t->recs[static_cast<size_t>(x)];
    float a = 0.f, b = 0.f;
    JANUS_CUDA(cudaEventElapsedTime(&a, t->anchor, r.a));
    JANUS_CUDA(cudaEventElapsedTime(&b, t->anchor, r.b));
    out[5 * x + 0] = r.device;
    out[5 * x + 1] = r.kind;
    out[5 * x + 2] = r.mb;
    out[5 * x + 3] = 1000.0 * a;
    out[5 * x + 4] = 1000.0 * b;
  }
}

janus_stage* trainer_stage(janus_trainer* t, int block, int force_replica) {
  if (block < 0 || block >= t->P) throw domain_error("block out of range");
  janus_stage* s = force_replica ? t->F[static_cast<size_t>(block)] : t->E[static_cast<size_t>(block)];
  if (!s) throw state_error("block is not held by this process");
  return s;
}

std::string trainer_schedule_text(janus_trainer* t) { return serialize(t->sched); }

void trainer_plan(janus_trainer* t, int32_t* out) {
  for (int b = 0; b < t->P; ++b) {
    out[2 * b] = t->plan.blocks[static_cast<size_t>(b)].first;
    out[2 * b + 1] = t->plan.blocks[static_cast<size_t>(b)].second;
  }
}

// ------------------------------------------------------------------ NCCL
void nccl_unique_id(void* out) {
  ncclUniqueId id;
  JANUS_NCCL(ncclGetUniqueId(&id));
  std::memcpy(out, &id, sizeof(id));
}

janus_comm* comm_init_nccl(const void* id, int nranks, int rank, int device) {
  JANUS_CUDA(cudaSetDevice(device));
  auto c = std::make_unique<janus_comm>();
  c->kind = 0;
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  JANUS_NCCL(ncclCommInitRank(&c->base, nranks, uid, rank));
  return c.release();
}

janus_comm* comm_init_ipc(const char* dir, int nranks, int rank, int device, bool same_process) {
  if (!dir || !*dir) throw domain_error("IPC comm needs a rendezvous directory");
  if (nranks < 1 || rank < 0 || rank >= nranks) throw domain_error("bad rank / nranks");
  JANUS_CUDA(cudaSetDevice(device));
  auto c = std::make_unique<janus_comm>();
  c->kind = same_process ? 2 : 1;
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  c->dir = dir;
  return c.release();
}

void comm_destroy(janus_comm* c) {
  if (!c) return;
  if (c->base) ncclCommDestroy(c->base);
  delete c;
}

void comm_send(janus_comm* c, const void* buf, size_t bytes, int peer, cudaStream_t s) {
  if (c->kind != 0) throw config_error("generic send needs an NCCL comm");
  JANUS_NCCL(ncclSend(buf, bytes, ncclChar, peer, c->base, s));
}
void comm_recv(janus_comm* c, void* buf, size_t bytes, int peer, cudaStream_t s) {
  if (c->kind != 0) throw config_error("generic receive needs an NCCL comm");
  JANUS_NCCL(ncclRecv(buf, bytes, ncclChar, peer, c->base, s));
}
void comm_group_start() { JANUS_NCCL(ncclGroupStart()); }
void comm_group_end() { JANUS_NCCL(ncclGroupEnd()); }
void comm_allreduce_sum(janus_comm* c, float* buf, int64_t count, cudaStream_t s) {
  if (c->kind != 0) throw config_error("generic all-reduce needs an NCCL comm");
  JANUS_NCCL(ncclAllReduce(buf, buf, static_cast<size_t>(count), ncclFloat, ncclSum, c->base, s));
}

}  // namespace janus
