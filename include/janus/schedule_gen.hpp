// janus/schedule_gen.hpp — schedule generators and the schedule validator.
//
// The reference ships only Passes 1-3 (transform.hpp); the generators it
// specifies are SPEC-only and are implemented here in the same style:
//   gen_first_order (Pass 0) ............ SPEC.md:129-137
//   onef1b_2nd baseline ................. SPEC.md:139-158
//   symfold = prune(fold(remap(pass0))) . SPEC.md:216-220
//   wavek Passes 4-6 .................... SPEC.md:269-307 (greedy earliest-feasible)
//   analytic_bubble ..................... SPEC.md:309-317
//   validate_schedule ................... SPEC.md:73-81
// All generators are pure and deterministic.
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <limits>
#include <map>
#include <set>
#include <string>
#include <tuple>
#include <vector>

#include "janus/errors.hpp"
#include "janus/graph.hpp"
#include "janus/ir.hpp"
#include "janus/transform.hpp"

namespace janus {

// ---------------------------------------------------------------------------
// Pass 0: 1F1B over 2P virtual stages, one list per virtual stage.
// ---------------------------------------------------------------------------
inline Schedule gen_first_order(int P, int N_mb) {
  if (P < 1) throw domain_error("gen_first_order: P must be >= 1");
  if (N_mb < 1) throw domain_error("gen_first_order: N_mb must be >= 1");
  const int S = 2 * P;
  Schedule s;
  s.pipeline_degree = P;
  s.num_micro_batches = N_mb;
  s.order = ScheduleOrder::first_order;
  s.device_lists.resize(static_cast<std::size_t>(S));
  s.stage_map.resize(static_cast<std::size_t>(S));
  for (int v = 0; v < S; ++v) s.stage_map[static_cast<std::size_t>(v)] = v;

  auto mk = [](InstrKind k, int mb, int vs, int dev, int peer, std::uint8_t flags) {
    Instruction in;
    in.kind = k;
    in.micro_batch = mb;
    in.virtual_stage = vs;
    in.device = dev;
    in.peer_device = peer;
    in.flags = flags;
    return in;
  };
  for (int v = 0; v < S; ++v) {
    auto& dl = s.device_lists[static_cast<std::size_t>(v)];
    auto fw = [&](int m) {
      if (v == 0) dl.push_back(mk(InstrKind::LM, m, 0, 0, -1, 0));
      if (v > 0) dl.push_back(mk(InstrKind::RAE, m, v, v, v - 1, kFlagUnlabeled));
      dl.push_back(mk(InstrKind::FE, m, v, v, -1, kFlagUnlabeled));
      if (v < S - 1) dl.push_back(mk(InstrKind::SAE, m, v, v, v + 1, kFlagUnlabeled));
    };
    auto bw = [&](int m) {
      if (v < S - 1) dl.push_back(mk(InstrKind::RGE, m, v, v, v + 1, kFlagUnlabeled));
      dl.push_back(mk(InstrKind::BE, m, v, v, -1, kFlagUnlabeled));
      if (v > 0) dl.push_back(mk(InstrKind::SGE, m, v, v, v - 1, kFlagUnlabeled));
    };
    const int warm = std::min(S - 1 - v, N_mb);
    int next_f = 0, next_b = 0;
    for (; next_f < warm; ++next_f) fw(next_f);
    while (next_f < N_mb) {  // steady state: one forward, one backward
      fw(next_f++);
      bw(next_b++);
    }
    while (next_b < N_mb) bw(next_b++);  // cool-down
    Instruction os;
    os.kind = InstrKind::OS;
    os.device = v;
    dl.push_back(os);
  }
  renumber_seq(s);
  return s;
}

inline std::vector<int> symfold_stage_map(int P) {
  std::vector<int> m(static_cast<std::size_t>(2 * P));
  for (int v = 0; v < 2 * P; ++v) m[static_cast<std::size_t>(v)] = fold_map(v, P);
  return m;
}

/// SymFold: Passes 0-3.  `pruned` (optional) receives Pass 3's count (= 4 N_mb).
inline Schedule symfold(int P, int N_mb, int* pruned = nullptr) {
  const Schedule remapped = transform::remap_second_order(gen_first_order(P, N_mb));
  auto [out, n] = transform::prune_intra_device(transform::fold_with_map(remapped, symfold_stage_map(P)));
  if (pruned) *pruned = n;
  return out;
}

/// 1F1B-2nd baseline: linear map floor(s_v/2) — energy stages on devices
/// [0,P/2), force stages on [P/2,P); every FF recomputes FE (flag), force
/// devices hold replicated parameters and sync them with an AR before OS.
inline Schedule onef1b_2nd(int P, int N_mb) {
  if (P < 2 || P % 2 != 0) throw config_error("onef1b_2nd: P must be even and >= 2");
  std::vector<int> lin(static_cast<std::size_t>(2 * P));
  for (int v = 0; v < 2 * P; ++v) lin[static_cast<std::size_t>(v)] = v / 2;
  const Schedule remapped = transform::remap_second_order(gen_first_order(P, N_mb));
  Schedule out = transform::prune_intra_device(transform::fold_with_map(remapped, lin)).first;
  for (int d = 0; d < out.num_devices(); ++d) {
    auto& dl = out.device_lists[static_cast<std::size_t>(d)];
    for (auto& in : dl)
      if (in.kind == InstrKind::FF) in.flags |= kFlagRecompute;
    if (d >= P / 2) {
      Instruction ar;
      ar.kind = InstrKind::AR;
      ar.device = d;
      ar.flags = kFlagReplicatedParams;
      dl.insert(dl.end() - 1, ar);  // before the trailing OS
    }
  }
  renumber_seq(out);
  return out;
}

/// Hanayo-2nd baseline (§5.1 "single wave
/// (W=1, S=2P)"): the V-shape placement of fold_map (virtual stage s_v on
/// device fold_map(s_v), intra-device hand-offs pruned) with wave-style
/// ordering instead of SymFold's folded 1F1B: every instruction of micro-batch
/// m belongs to the synchronous wave step at which m reaches its virtual stage
/// (forward s_v: m + s_v; backward s_v: m + 4P - 1 - s_v), and each device
/// issues in (step, backward first, micro-batch) order — the projection of one
/// global topological order, so deadlock-free.  Every FF carries the
/// recompute flag: the baseline lacks SymFold's FE-activation reuse, so the
/// executor re-runs the block's FE before its FF.
inline Schedule hanayo_2nd(int P, int N_mb) {
  if (P < 1) throw domain_error("hanayo_2nd: P must be >= 1");
  const Schedule v = symfold(P, N_mb);
  Schedule out = transform::priority_topo_order(v, [P](const Instruction& in) {
    if (in.micro_batch < 0) return std::tuple<int, int, int>{std::numeric_limits<int>::max(), 0, 0};  // OS / AR last
    const bool fwd = is_forward_flow(in.kind);
    const int vs = in.virtual_stage < 0 ? 0 : in.virtual_stage;
    const int step = fwd ? in.micro_batch + vs : in.micro_batch + 4 * P - 1 - vs;
    return std::tuple<int, int, int>{step, fwd ? 1 : 0, in.micro_batch};
  });
  for (auto& dl : out.device_lists)
    for (auto& in : dl)
      if (in.kind == InstrKind::FF) in.flags |= kFlagRecompute;
  renumber_seq(out);
  return out;
}

// ---------------------------------------------------------------------------
// Phase times (costmodel PhaseTimes).
// ---------------------------------------------------------------------------
struct PhaseTimes {
  double t_FE = 1, t_FF = 2, t_BE = 3, t_BF = 4;

  void check() const {
    const std::array<double, 4> v{t_FE, t_FF, t_BE, t_BF};
    for (double x : v)
      if (!(x > 0) || !std::isfinite(x)) throw domain_error("PhaseTimes: times must be positive and finite");
    if (!(t_FE < t_FF && t_FF < t_BE && t_BE < t_BF))
      throw domain_error("PhaseTimes: partial order t_FE < t_FF < t_BE < t_BF violated");
  }
  /// Measured phase times (a timeline's means) need not follow the paper's
  /// partial order; a cost model only needs them positive.
  void check_positive() const {
    const std::array<double, 4> v{t_FE, t_FF, t_BE, t_BF};
    for (double x : v)
      if (!(x > 0) || !std::isfinite(x)) throw domain_error("PhaseTimes: times must be positive and finite");
  }
  double of(InstrKind k) const {
    switch (k) {
      case InstrKind::FE: return t_FE;
      case InstrKind::FF: return t_FF;
      case InstrKind::BE: return t_BE;
      case InstrKind::BF: return t_BF;
      default: return 0.0;
    }
  }
  PhaseTimes halved() const { return PhaseTimes{t_FE / 2, t_FF / 2, t_BE / 2, t_BF / 2}; }
};

/// Table 4 presets, P=8 per-micro-batch times in ms.
inline PhaseTimes preset_phase_times(const std::string& name) {
  if (name == "uma-1.2b") return {26.25, 37.51, 43.59, 82.03};
  if (name == "uma-2.3b") return {58.41, 87.22, 98.15, 190.73};
  if (name == "esen-100m") return {52.98, 84.88, 85.29, 175.67};
  if (name == "esen-220m") return {24.96, 57.67, 64.30, 118.92};
  if (name == "uniform") return {1, 2, 3, 4};
  throw domain_error("unknown phase-time preset '" + name + "'");
}

/// Durations for a replay: compute = phase time, everything else 0.
inline std::vector<double> phase_durations(const DepGraph& g, const PhaseTimes& t, double recompute_r = 1.0) {
  std::vector<double> d(static_cast<std::size_t>(g.size()), 0.0);
  for (int i = 0; i < g.size(); ++i) {
    const Instruction& in = *g.flat[static_cast<std::size_t>(i)];
    double x = t.of(in.kind);
    if (in.kind == InstrKind::FF && in.has_flag(kFlagRecompute)) x += recompute_r * t.t_FE;
    d[static_cast<std::size_t>(i)] = x;
  }
  return d;
}

struct BubbleEstimate {
  double intra_total = 0, inter_total = 0, combined_B = 0;
};

/// SPEC.md:309-317.  k must divide N_mb for the exact formulas; otherwise the
/// unit count is ceil(N_mb/k) (trailing partial unit, documented).
inline BubbleEstimate analytic_bubble(const PhaseTimes& t, int P, int N_mb, int k) {
  t.check();
  if (P < 1 || N_mb < 1 || k < 1 || k > N_mb) throw domain_error("analytic_bubble: bad P/N_mb/k");
  const double units = (N_mb % k == 0) ? static_cast<double>(N_mb / k) : std::ceil(static_cast<double>(N_mb) / k);
  BubbleEstimate b;
  b.intra_total = (t.t_BE - t.t_FF) * P * units;
  b.inter_total = (t.t_BF - t.t_FE) * P * (units - 1.0);
  // combined form is stated on the base (P-scale) times T = 2 t
  const double TFE = 2 * t.t_FE, TFF = 2 * t.t_FF, TBE = 2 * t.t_BE, TBF = 2 * t.t_BF;
  b.combined_B = (TBF + TBE - TFF - TFE) * P * units / 2.0 - (P / 2.0) * (TBF - TFE);
  return b;
}

// ---------------------------------------------------------------------------
// WaveK (Passes 4-6).
// ---------------------------------------------------------------------------
struct WaveKUnit {
  int index = 0;
  std::vector<int> micro_batches;
};

/// Pass 4 decomposition: ceil(N_mb/k) units of consecutive micro-batches.
inline std::vector<WaveKUnit> pass4_decompose(int N_mb, int k) {
  if (k < 1 || k > N_mb) throw domain_error("wavek: k must be in [1, N_mb]");
  std::vector<WaveKUnit> units;
  for (int b = 0, u = 0; b < N_mb; b += k, ++u) {
    WaveKUnit w;
    w.index = u;
    for (int m = b; m < std::min(N_mb, b + k); ++m) w.micro_batches.push_back(m);
    units.push_back(std::move(w));
  }
  return units;
}

struct WaveKOptions {
  PhaseTimes times = PhaseTimes{26.25, 37.51, 43.59, 82.03};  // uma-1.2b ratios
  int lookahead_units = 2;  // max units admitted beyond the oldest unfinished one
  int policy = -1;          // -1: search; 0: (unit, phase rank); 1: (unit, -bottom level); 2: -bottom level
};

namespace detail {

/// One dispatchable group of a second-order schedule: a compute plus its
/// comm instructions, with group-level predecessors.
struct SchedGroup {
  InstrGroup g;
  std::vector<int> preds;
  int unit = 0;
};

inline int wavek_phase_rank(InstrKind k) {
  // Within a unit the backward wave drains first (bounds live activations);
  // the forward wave fills whatever is left (Passes 5-6 overlap).
  switch (k) {
    case InstrKind::BE: return 0;
    case InstrKind::BF: return 1;
    case InstrKind::FF: return 2;
    default: return 3;  // FE
  }
}

}  // namespace detail

/// WaveK(P, N_mb, k): re-orders the SymFold groups by a work-conserving list
/// schedule over phase-time estimates (greedy earliest-feasible).
///  * Pass 4: micro-batches are grouped into units of k;
///  * Pass 5: inside a unit the forward residue (FF) fills the backward
///    wave's ramp-up because any ready group may run when a device idles;
///  * Pass 6: the next unit's forward wave (FE/FF) is admitted while the
///    current unit drains, filling the tail bubble of size ~t_BE.
/// Admission is limited to `lookahead_units` units past the oldest unit with
/// unfinished work on that device, which bounds in-flight activations to
/// about (1 + lookahead) k micro-batches.  The per-device order is the start
/// order of that simulation, so it is a projection of one topological order
/// (deadlock-free); the emitted text uses the SymFold instruction set.
inline Schedule wavek_with_policy(int P, int N_mb, int k, const WaveKOptions& opt) {
  opt.times.check_positive();  // measured times may break the paper's partial order
  const std::vector<WaveKUnit> units = pass4_decompose(N_mb, k);
  const Schedule base = symfold(P, N_mb);
  GroupedSchedule grouped = collect_groups(base);
  const int G = static_cast<int>(grouped.groups.size());

  // Group-level dependencies from the data DAG (no seq edges).
  const DepGraph dg = build_dependencies(base, /*include_seq_edges=*/false);
  std::map<std::tuple<int, int, int>, int> gid;  // (mb, vs, slot) -> group
  for (int i = 0; i < G; ++i) {
    const Instruction& c = grouped.groups[static_cast<std::size_t>(i)].compute;
    gid[{c.micro_batch, c.virtual_stage, detail::compute_slot(c.kind)}] = i;
  }
  auto group_of_instr = [&](const Instruction& in) -> int {
    if (is_compute(in.kind)) return gid.at({in.micro_batch, in.virtual_stage, detail::compute_slot(in.kind)});
    if (in.kind == InstrKind::LM) return gid.at({in.micro_batch, 0, detail::kSlotFwdCompute});
    return gid.at({in.micro_batch, in.virtual_stage, detail::comm_compute_slot(comm_class(in.kind))});
  };
  std::vector<detail::SchedGroup> sg(static_cast<std::size_t>(G));
  for (int i = 0; i < G; ++i) {
    sg[static_cast<std::size_t>(i)].g = grouped.groups[static_cast<std::size_t>(i)];
    sg[static_cast<std::size_t>(i)].unit = grouped.groups[static_cast<std::size_t>(i)].compute.micro_batch / k;
  }
  for (int i = 0; i < dg.size(); ++i) {
    const Instruction& in = *dg.flat[static_cast<std::size_t>(i)];
    if (in.kind == InstrKind::OS || in.kind == InstrKind::AR) continue;
    const int to = group_of_instr(in);
    for (int p : dg.preds[static_cast<std::size_t>(i)]) {
      const Instruction& pi = *dg.flat[static_cast<std::size_t>(p)];
      if (pi.kind == InstrKind::OS || pi.kind == InstrKind::AR) continue;
      const int from = group_of_instr(pi);
      if (from != to) sg[static_cast<std::size_t>(to)].preds.push_back(from);
    }
  }
  for (auto& x : sg) {
    std::sort(x.preds.begin(), x.preds.end());
    x.preds.erase(std::unique(x.preds.begin(), x.preds.end()), x.preds.end());
  }

  // bottom level: longest remaining path (phase-time weighted) to the end
  std::vector<double> blevel(static_cast<std::size_t>(G), 0.0);
  {
    std::vector<std::vector<int>> succ(static_cast<std::size_t>(G));
    std::vector<int> outdeg(static_cast<std::size_t>(G), 0);
    for (int i = 0; i < G; ++i)
      for (int p : sg[static_cast<std::size_t>(i)].preds) {
        succ[static_cast<std::size_t>(p)].push_back(i);
        ++outdeg[static_cast<std::size_t>(p)];
      }
    std::vector<int> q;
    for (int i = 0; i < G; ++i)
      if (outdeg[static_cast<std::size_t>(i)] == 0) q.push_back(i);
    for (std::size_t h = 0; h < q.size(); ++h) {
      const int i = q[h];
      double best = 0;
      for (int x : succ[static_cast<std::size_t>(i)]) best = std::max(best, blevel[static_cast<std::size_t>(x)]);
      blevel[static_cast<std::size_t>(i)] = opt.times.of(sg[static_cast<std::size_t>(i)].g.compute.kind) + best;
      for (int p : sg[static_cast<std::size_t>(i)].preds)
        if (--outdeg[static_cast<std::size_t>(p)] == 0) q.push_back(p);
    }
  }
  auto prio = [&](int i) {
    const auto& x = sg[static_cast<std::size_t>(i)];
    const long bl = std::lround(-blevel[static_cast<std::size_t>(i)] * 1024.0);
    switch (opt.policy) {
      case 0: return std::make_tuple(static_cast<long>(x.unit), static_cast<long>(detail::wavek_phase_rank(x.g.compute.kind)), static_cast<long>(x.g.compute.micro_batch), static_cast<long>(x.g.compute.virtual_stage));
      case 1: return std::make_tuple(static_cast<long>(x.unit), bl, static_cast<long>(x.g.compute.micro_batch), static_cast<long>(x.g.compute.virtual_stage));
      default: return std::make_tuple(0L, bl, static_cast<long>(x.g.compute.micro_batch), static_cast<long>(x.g.compute.virtual_stage));
    }
  };
  const int D = base.num_devices();
  const int U = static_cast<int>(units.size());
  std::vector<double> end(static_cast<std::size_t>(G), -1.0);
  std::vector<char> placed(static_cast<std::size_t>(G), 0);
  std::vector<double> dev_free(static_cast<std::size_t>(D), 0.0);
  std::vector<std::vector<int>> left(static_cast<std::size_t>(D), std::vector<int>(static_cast<std::size_t>(U), 0));
  for (int i = 0; i < G; ++i) ++left[static_cast<std::size_t>(sg[static_cast<std::size_t>(i)].g.compute.device)][static_cast<std::size_t>(sg[static_cast<std::size_t>(i)].unit)];
  std::vector<std::vector<int>> order(static_cast<std::size_t>(D));

  for (int step = 0; step < G; ++step) {
    int best = -1, best_dev = -1;
    double best_t = std::numeric_limits<double>::infinity();
    std::tuple<long, long, long, long> best_key{};
    for (int d = 0; d < D; ++d) {
      int oldest = 0;
      while (oldest < U && left[static_cast<std::size_t>(d)][static_cast<std::size_t>(oldest)] == 0) ++oldest;
      const int admit = oldest + opt.lookahead_units;
      // earliest start on d and, among groups starting then, the best key
      int cand = -1;
      double cand_t = std::numeric_limits<double>::infinity();
      std::tuple<long, long, long, long> cand_key{};
      for (int i = 0; i < G; ++i) {
        const auto& x = sg[static_cast<std::size_t>(i)];
        if (placed[static_cast<std::size_t>(i)] || x.g.compute.device != d || x.unit > admit) continue;
        double ready = dev_free[static_cast<std::size_t>(d)];
        bool ok = true;
        for (int p : x.preds) {
          if (!placed[static_cast<std::size_t>(p)]) {
            ok = false;
            break;
          }
          ready = std::max(ready, end[static_cast<std::size_t>(p)]);
        }
        if (!ok) continue;
        const auto key = prio(i);
        if (ready < cand_t - 1e-12 || (std::abs(ready - cand_t) <= 1e-12 && key < cand_key)) {
          cand = i;
          cand_t = ready;
          cand_key = key;
        }
      }
      if (cand >= 0 && (cand_t < best_t - 1e-12 || (std::abs(cand_t - best_t) <= 1e-12 && d < best_dev))) {
        best = cand;
        best_dev = d;
        best_t = cand_t;
        best_key = cand_key;
      }
    }
    if (best < 0) throw deadlock_error("wavek: no admissible group (internal error)");
    auto& x = sg[static_cast<std::size_t>(best)];
    placed[static_cast<std::size_t>(best)] = 1;
    end[static_cast<std::size_t>(best)] = best_t + opt.times.of(x.g.compute.kind);
    dev_free[static_cast<std::size_t>(best_dev)] = end[static_cast<std::size_t>(best)];
    --left[static_cast<std::size_t>(best_dev)][static_cast<std::size_t>(x.unit)];
    order[static_cast<std::size_t>(best_dev)].push_back(best);
  }

  Schedule out;
  out.pipeline_degree = base.pipeline_degree;
  out.num_micro_batches = base.num_micro_batches;
  out.order = base.order;
  out.stage_map = base.stage_map;
  out.device_lists.resize(static_cast<std::size_t>(D));
  for (int d = 0; d < D; ++d) {
    for (int i : order[static_cast<std::size_t>(d)]) append_group(out.device_lists[static_cast<std::size_t>(d)], sg[static_cast<std::size_t>(i)].g);
    for (const Instruction& c : grouped.control)
      if (c.device == d) out.device_lists[static_cast<std::size_t>(d)].push_back(c);
  }
  renumber_seq(out);
  return out;
}

/// Makespan of a schedule replayed under phase-time estimates.
inline double predicted_makespan(const Schedule& s, const PhaseTimes& t) {
  const DepGraph g = build_dependencies(s);
  const ReplayResult r = replay(g, phase_durations(g, t));
  if (!r.ok) throw deadlock_error("predicted_makespan: " + r.blocked);
  return r.makespan;
}

/// WaveK with the offline selection step: the list-scheduling priority
/// (phase rank vs. critical-path bottom level) and the look-ahead window
/// (0..opt.lookahead_units) are chosen by replayed makespan; ties keep the
/// smaller window (less activation memory).  policy < 0 in `opt` requests the
/// search; a fixed policy >= 0 is used as given.
inline Schedule wavek(int P, int N_mb, int k, const WaveKOptions& opt = WaveKOptions{}) {
  if (opt.policy >= 0) return wavek_with_policy(P, N_mb, k, opt);
  Schedule best;
  double best_t = std::numeric_limits<double>::infinity();
  for (int la = 0; la <= opt.lookahead_units; ++la) {
    for (int pol = 0; pol <= 1; ++pol) {
      WaveKOptions o = opt;
      o.policy = pol;
      o.lookahead_units = la;
      Schedule s = wavek_with_policy(P, N_mb, k, o);
      const double t = predicted_makespan(s, opt.times);
      if (t < best_t - 1e-9) {
        best_t = t;
        best = std::move(s);
      }
    }
  }
  return best;
}

// ---------------------------------------------------------------------------
// Validator.  Never throws on bad schedules; reports instead.
// ---------------------------------------------------------------------------
inline ValidationReport validate_schedule(const Schedule& s) {
  ValidationReport rep;
  const int P = s.pipeline_degree;
  const int S = 2 * P;
  const bool second = s.order == ScheduleOrder::second_order;
  auto issue = [](std::vector<ValidationIssue>& v, int d, int seq, std::string what) {
    v.push_back(ValidationIssue{d, seq, std::move(what)});
  };
  if (P < 1 || s.num_micro_batches < 1 || static_cast<int>(s.stage_map.size()) != S) {
    issue(rep.coverage_errors, -1, -1, "malformed header (P, N_mb or stage_map size)");
    return rep;
  }
  for (int v = 0; v < S; ++v) {
    const int dv = s.stage_map[static_cast<std::size_t>(v)];
    if (dv < 0 || dv >= s.num_devices()) {
      issue(rep.coverage_errors, -1, -1, "stage_map[" + std::to_string(v) + "] out of range");
      return rep;
    }
  }

  // (1) coverage + structural sanity
  std::map<std::tuple<int, int, int>, int> count;  // (mb, vs, fwd/bwd) -> #computes
  for (int d = 0; d < s.num_devices(); ++d) {
    const auto& dl = s.device_lists[static_cast<std::size_t>(d)];
    int os = 0;
    for (std::size_t p = 0; p < dl.size(); ++p) {
      const Instruction& in = dl[p];
      if (in.device != d) issue(rep.coverage_errors, d, in.seq, "device field does not match its list");
      if (p > 0 && in.seq <= dl[p - 1].seq) issue(rep.coverage_errors, d, in.seq, "seq not strictly increasing");
      if (in.kind == InstrKind::OS) ++os;
      if (!is_compute(in.kind)) continue;
      if (in.micro_batch < 0 || in.micro_batch >= s.num_micro_batches || in.virtual_stage < 0 || in.virtual_stage >= S) {
        issue(rep.coverage_errors, d, in.seq, "compute with micro-batch/stage out of range");
        continue;
      }
      if (s.stage_map[static_cast<std::size_t>(in.virtual_stage)] != d)
        issue(rep.coverage_errors, d, in.seq, "compute placed off its stage_map device");
      if (second) {
        const bool energy = in.virtual_stage < P;
        const bool fwd = is_forward_flow(in.kind);
        const InstrKind want = energy ? (fwd ? InstrKind::FE : InstrKind::BE) : (fwd ? InstrKind::FF : InstrKind::BF);
        if (in.kind != want) issue(rep.coverage_errors, d, in.seq, std::string("phase ") + std::string(to_string(in.kind)) + " on the wrong virtual stage");
      }
      ++count[{in.micro_batch, in.virtual_stage, detail::compute_slot(in.kind)}];
    }
    if (os != 1) issue(rep.coverage_errors, d, -1, "device must run exactly one OS, has " + std::to_string(os));
  }
  for (int m = 0; m < s.num_micro_batches; ++m) {
    for (int v = 0; v < S; ++v) {
      for (int slot = 0; slot < 2; ++slot) {
        const auto it = count.find({m, v, slot});
        const int c = it == count.end() ? 0 : it->second;
        if (c != 1) {
          issue(rep.coverage_errors, s.stage_map[static_cast<std::size_t>(v)], -1,
                "mb " + std::to_string(m) + " vs " + std::to_string(v) + (slot == 0 ? " forward" : " backward") +
                    " compute count " + std::to_string(c) + " != 1");
        }
      }
    }
  }

  // (2) matching: per channel, sends and receives pair one-to-one and the
  // peer is where stage_map puts the neighbouring stage.
  std::map<std::tuple<int, char, int, int, int>, std::pair<int, int>> chan;
  for (int d = 0; d < s.num_devices(); ++d) {
    for (const Instruction& in : s.device_lists[static_cast<std::size_t>(d)]) {
      if (!is_comm(in.kind)) continue;
      if (in.virtual_stage < 0 || in.virtual_stage >= S || in.micro_batch < 0) {
        issue(rep.matching_errors, d, in.seq, "comm with stage/micro-batch out of range");
        continue;
      }
      const int ps = comm_peer_stage(in.kind, in.virtual_stage);
      if (ps < 0 || ps >= S) {
        issue(rep.matching_errors, d, in.seq, "comm towards a non-existent stage");
        continue;
      }
      if (in.peer_device != s.stage_map[static_cast<std::size_t>(ps)])
        issue(rep.matching_errors, d, in.seq, "comm peer does not host the neighbouring stage");
      if (in.peer_device == in.device) issue(rep.matching_errors, d, in.seq, "intra-device comm left unpruned");
      if (second) {
        const CommClass c = comm_class(in.kind);
        const int consumer = c == CommClass::SA ? in.virtual_stage + 1 : (c == CommClass::SG ? in.virtual_stage - 1 : in.virtual_stage);
        if (comm_suffix(in.kind) != (consumer < P ? 'E' : 'F'))
          issue(rep.matching_errors, d, in.seq, "comm suffix does not name the consuming phase");
      }
      const bool send = is_send(in.kind);
      auto& e = chan[{is_activation_comm(in.kind) ? 0 : 1, comm_suffix(in.kind), in.micro_batch,
                      send ? in.device : in.peer_device, send ? in.peer_device : in.device}];
      (send ? e.first : e.second) += 1;
    }
  }
  for (const auto& kv : chan) {
    if (kv.second.first != 1 || kv.second.second != 1) {
      const auto& k = kv.first;
      issue(rep.matching_errors, std::get<3>(k), -1,
            "channel mb " + std::to_string(std::get<2>(k)) + " D" + std::to_string(std::get<3>(k)) + "->D" +
                std::to_string(std::get<4>(k)) + " has " + std::to_string(kv.second.first) + " sends / " +
                std::to_string(kv.second.second) + " receives");
    }
  }
  // every cross-device stage boundary needs its transfer
  for (int m = 0; m < s.num_micro_batches; ++m) {
    for (int v = 0; v + 1 < S; ++v) {
      const int a = s.stage_map[static_cast<std::size_t>(v)], b = s.stage_map[static_cast<std::size_t>(v + 1)];
      if (a == b) continue;
      const char up = second ? (v + 1 < P ? 'E' : 'F') : 'E';   // SA v -> v+1, consumed on v+1
      const char down = second ? (v < P ? 'E' : 'F') : 'E';     // SG v+1 -> v, consumed on v
      if (!chan.count({0, up, m, a, b}))
        issue(rep.matching_errors, a, -1, "missing activation transfer mb " + std::to_string(m) + " vs " + std::to_string(v));
      if (!chan.count({1, down, m, b, a}))
        issue(rep.matching_errors, b, -1, "missing gradient transfer mb " + std::to_string(m) + " vs " + std::to_string(v + 1));
    }
  }

  // (3) realizability: replay in seq order with the full DAG.
  const DepGraph g = build_dependencies(s);
  const ReplayResult r = replay(g, unit_durations(g));
  if (!r.ok) issue(rep.dependency_errors, -1, -1, "not replayable: " + r.blocked);

  // (4) gradient ledger (Eq. 2): every BE carries the merged first-order tag,
  // every BF the second-order tag, P of each per micro-batch.
  if (second) {
    std::vector<int> merged(static_cast<std::size_t>(s.num_micro_batches), 0), second_o(static_cast<std::size_t>(s.num_micro_batches), 0);
    for (int d = 0; d < s.num_devices(); ++d) {
      for (const Instruction& in : s.device_lists[static_cast<std::size_t>(d)]) {
        if (in.kind == InstrKind::BE) {
          if (!in.has_flag(kFlagMergedFirstOrder) || in.has_flag(kFlagSecondOrder))
            issue(rep.gradient_ledger_errors, d, in.seq, "BE without the merged first-order tag");
          else if (in.micro_batch >= 0 && in.micro_batch < s.num_micro_batches)
            ++merged[static_cast<std::size_t>(in.micro_batch)];
        } else if (in.kind == InstrKind::BF) {
          if (!in.has_flag(kFlagSecondOrder) || in.has_flag(kFlagMergedFirstOrder))
            issue(rep.gradient_ledger_errors, d, in.seq, "BF without the second-order tag");
          else if (in.micro_batch >= 0 && in.micro_batch < s.num_micro_batches)
            ++second_o[static_cast<std::size_t>(in.micro_batch)];
        }
      }
    }
    for (int m = 0; m < s.num_micro_batches; ++m) {
      if (merged[static_cast<std::size_t>(m)] != P || second_o[static_cast<std::size_t>(m)] != P)
        issue(rep.gradient_ledger_errors, -1, -1, "mb " + std::to_string(m) + " ledger " +
                                                      std::to_string(merged[static_cast<std::size_t>(m)]) + " merged / " +
                                                      std::to_string(second_o[static_cast<std::size_t>(m)]) + " second-order, want " + std::to_string(P));
    }
  }
  return rep;
}

/// Measured / predicted bubble bookkeeping (SimReport fields).
struct BubbleReport {
  double makespan = 0;
  std::vector<double> busy, bubble;
  double bubble_ratio = 0;
};

/// Bubble of a replay: per device idle within [0, makespan].
inline BubbleReport bubble_of(const DepGraph& g, const ReplayResult& r, const std::vector<double>& durations) {
  BubbleReport b;
  b.makespan = r.makespan;
  const Schedule& s = *g.schedule;
  b.busy.assign(static_cast<std::size_t>(s.num_devices()), 0.0);
  for (int i = 0; i < g.size(); ++i) b.busy[static_cast<std::size_t>(g.flat[static_cast<std::size_t>(i)]->device)] += durations[static_cast<std::size_t>(i)];
  double idle = 0;
  for (double x : b.busy) {
    b.bubble.push_back(r.makespan - x);
    idle += r.makespan - x;
  }
  b.bubble_ratio = r.makespan > 0 ? idle / (s.num_devices() * r.makespan) : 0.0;
  return b;
}

}  // namespace janus
