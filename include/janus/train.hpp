// janus/train.hpp — the C++ train-step entry of the drop-in boundary
// (SURVEY.md §8(b)):
//
//   StepReport train_step(const ModelConfig&, const StagePlan&, const Schedule&,
//                         const MicroBatches&, TrainState&);
//
// in the reference's style (namespace janus, value types, exceptions).  The
// reference only replays a Schedule with a per-instruction duration
// (graph.hpp:168); train_step EXECUTES it: every FE / FF /
// BF / BE on the sm_100a kernels, every S* / R* as a transfer, LM as the
// (device) neighbour-list build, OS as the ledger reduction + Adam.  The
// schedule may come from any generator (include/janus/schedule_gen.hpp) or
// from the reference's own transforms (transform.hpp), as long as it
// validates.  Header-only over the C ABI (janus_cuda.h): a
// maintainer switches by adding this include path and linking
// libjanus_b200.so.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "janus/errors.hpp"
#include "janus/ir.hpp"
#include "janus/model.hpp"
#include "janus_cuda.h"

namespace janus {

/// One micro-batch: structures concatenated (struct_id non-decreasing).  An
/// empty row_ptr means "build the neighbour list on the device" (the LM
/// instruction on the GPU); otherwise row_ptr / col / shift / rev are a
/// host CSR by receiver.
struct MicroBatch {
  std::vector<double> pos;           // [n_atoms * 3]
  std::vector<std::int32_t> species;  // [n_atoms]
  std::vector<std::int32_t> struct_id;
  std::vector<double> cell;           // [n_struct] cubic box lengths
  std::vector<float> E_target;        // [n_struct]
  std::vector<float> F_target;        // [n_atoms * 3]
  std::vector<std::int32_t> row_ptr, col, shift, rev;

  int n_atoms() const { return static_cast<int>(species.size()); }
  int n_struct() const { return static_cast<int>(cell.size()); }
  janus_host_batch view() const {
    janus_host_batch h{};
    h.n_atoms = n_atoms();
    h.n_struct = n_struct();
    h.n_edges = row_ptr.empty() ? 0 : row_ptr.back();
    h.pos = pos.data();
    h.species = species.data();
    h.struct_id = struct_id.data();
    h.cell = cell.data();
    h.E_target = E_target.data();
    h.F_target = F_target.data();
    h.row_ptr = row_ptr.empty() ? nullptr : row_ptr.data();
    h.col = col.empty() ? nullptr : col.data();
    h.shift = shift.empty() ? nullptr : shift.data();
    h.rev = rev.empty() ? nullptr : rev.data();
    return h;
  }
};
using MicroBatches = std::vector<MicroBatch>;

/// What one executed step reports (the SimReport fields the executor can
/// measure on the device).
struct StepReport {
  double loss = 0;               // sum over micro-batches of L_E + L_F
  double makespan_ms = 0;        // device time of the step
  double bubble_ratio = 0;       // sum idle / (P makespan), with record_timeline
  std::int64_t p2p_bytes = 0;
  std::int64_t kernel_launches = 0;
  std::vector<std::int64_t> peak_bytes;  // per device: static + arena
  std::vector<std::int64_t> act_bytes;   // per device: activation slot pool
  std::vector<int> act_slots;            // per device: live micro-batches
};

/// Everything that persists across steps: parameters, Adam state, the
/// activation pools, streams and cached step graphs.  Built by the first
/// train_step for its (model, plan, schedule); later steps must pass the same.
class TrainState {
 public:
  struct Options {
    int precision = JANUS_PREC_TF32;
    int lanes = 1;           // compute streams per device (micro-batch m on lane m % lanes)
    bool use_graphs = true;  // capture the step once, replay it
    bool record_timeline = false;
    int max_atoms = 256, max_edges = 256 * 120, max_struct = 8;
    int device = 0;
    janus_opt opt{1e-3f, 0.9f, 0.999f, 1e-8f};
  };

  TrainState(std::vector<float> params, Options o) : params_(std::move(params)), o_(o) {}
  ~TrainState() {
    if (t_) janus_trainer_destroy(t_);
  }
  TrainState(const TrainState&) = delete;
  TrainState& operator=(const TrainState&) = delete;

  janus_trainer* handle() const { return t_; }
  const Options& options() const { return o_; }
  Options& options() { return o_; }

  /// Parameters of block b (device copy; after the last step's Adam update).
  std::vector<float> block_params(int b) const {
    janus_stage* st = nullptr;
    check_status(janus_trainer_stage(t_, b, 0, &st), janus_last_error());
    const std::int64_t n = janus_stage_param_count(st);
    std::vector<float> out(static_cast<std::size_t>(n));
    check_status(janus_stage_params(st, out.data(), nullptr), janus_last_error());
    return out;
  }

 private:
  friend StepReport train_step(const ModelConfig&, const StagePlan&, const Schedule&, const MicroBatches&, TrainState&);
  std::vector<float> params_;
  Options o_;
  janus_trainer* t_ = nullptr;
  std::string text_;  // the schedule the trainer was built for
};

inline StepReport train_step(const ModelConfig& mc, const StagePlan& plan, const Schedule& s, const MicroBatches& mbs,
                             TrainState& st) {
  const int P = s.pipeline_degree;
  if (plan.P != P) throw config_error("train_step: plan and schedule disagree on P");
  if (static_cast<int>(mbs.size()) != s.num_micro_batches) throw domain_error("train_step: one MicroBatch per micro-batch");
  const StagePlan canon = partition_units(mc, P);
  if (canon.blocks != plan.blocks) throw config_error("train_step: the executor partitions units by partition_units()");
  const std::string text = serialize(s);
  if (!st.t_) {
    janus_model_desc md{mc.L, mc.H, mc.R, mc.n_species, static_cast<float>(mc.r_c), static_cast<float>(mc.w_E),
                        static_cast<float>(mc.w_F), st.o_.precision};
    if (static_cast<std::int64_t>(st.params_.size()) != mc.param_count()) throw domain_error("train_step: parameter count");
    janus_stage_desc sd{};
    sd.model = md;
    sd.unit_begin = 0;
    sd.unit_end = mc.num_units();
    sd.max_atoms = st.o_.max_atoms;
    sd.max_edges = st.o_.max_edges;
    sd.max_struct = st.o_.max_struct;
    sd.n_micro_batches = s.num_micro_batches;
    sd.n_slots = s.num_micro_batches;
    sd.device = st.o_.device;
    sd.n_lanes = st.o_.lanes;
    janus_exec_desc ed{};
    ed.n_stages = P;
    ed.n_micro_batches = s.num_micro_batches;
    ed.local_stages = 1;
    ed.use_graphs = st.o_.use_graphs ? 1 : 0;
    ed.dp_degree = 1;
    ed.record_timeline = st.o_.record_timeline ? 1 : 0;
    ed.lanes = st.o_.lanes;
    check_status(janus_trainer_create_from_text(&ed, &sd, st.params_.data(), text.c_str(), nullptr, 0, &st.t_),
                 janus_last_error());
    st.text_ = text;
  } else if (text != st.text_) {
    throw state_error("train_step: a TrainState executes the schedule it was built for");
  }
  std::vector<janus_host_batch> hb;
  std::vector<std::int32_t> ids;
  for (std::size_t m = 0; m < mbs.size(); ++m) {
    hb.push_back(mbs[m].view());
    ids.push_back(static_cast<std::int32_t>(m));
  }
  check_status(janus_trainer_load_many(st.t_, static_cast<int>(hb.size()), ids.data(), hb.data()), janus_last_error());
  janus_step_stats ss{};
  check_status(janus_trainer_step(st.t_, &st.o_.opt, &ss), janus_last_error());
  StepReport r;
  r.loss = ss.loss;
  r.makespan_ms = ss.makespan_ms;
  r.bubble_ratio = ss.bubble_ratio;
  r.p2p_bytes = ss.p2p_bytes;
  r.kernel_launches = ss.kernel_launches;
  for (int d = 0; d < s.num_devices() && d < 64; ++d) {
    r.peak_bytes.push_back(ss.peak_bytes[d]);
    r.act_bytes.push_back(ss.act_bytes[d]);
    r.act_slots.push_back(ss.act_slots[d]);
  }
  return r;
}

}  // namespace janus
