// janus/tuner.hpp — cost model (peak memory by the SPEC lifetime rule) and the
// offline WaveK unit-size search, fed with MEASURED phase times and
// per-micro-batch activation bytes from the device.
//
// SPEC-only in the reference: costmodel peak_memory and the
// tuner module (§4.2 Steps 1-3).  Same style as the
// reference headers: value types, pure deterministic functions,
// janus::domain_error on bad input.  Pinned choices:
//   * M_activation = simulated peak at k = P+1 minus k = P (finite difference);
//   * k_max = floor((M_mem - M_static) / M_activation), k_min = P;
//   * candidates = divisors of N_mb in [P, min(k_max, N_mb)] (divisors_only),
//     each re-checked against its own simulated peak;
//   * k* = argmax throughput over the feasible ones, ties -> smaller k;
//   * nothing feasible -> k = P, flagged untuned.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <string>
#include <utility>
#include <vector>

#include "janus/errors.hpp"
#include "janus/graph.hpp"
#include "janus/ir.hpp"
#include "janus/schedule_gen.hpp"

namespace janus {
namespace tuner {

/// MemoryParams, in bytes.  fe_bytes / ff_bytes: activation
/// bytes one micro-batch (MB_max) keeps live on a device from FE start to BE
/// end / from FF start to BF end.  static_bytes[d]: parameters,
/// gradients, optimizer state and ledgers of device d (one entry = all devices).
struct MemoryParams {
  double m_gpu = 0, m_reserve = 0;
  std::vector<double> static_bytes{0.0};
  double fe_bytes = 0, ff_bytes = 0;
  double stage0_mult = 1.0;
  bool replicate_static = true;  // SPEC rule: replicated-parameter devices count static twice
  double m_mem() const { return m_gpu - m_reserve; }
  double static_of(int d) const {
    return static_bytes.size() == 1 ? static_bytes[0] : static_bytes.at(static_cast<std::size_t>(d));
  }
};

/// peak_memory of a replayed schedule: per device, static +
/// max over time of the live FE activations (FE(m) start .. BE(m) end) and FF
/// intermediates (FF(m) start .. BF(m) end).  A release at the same instant
/// as an allocation is applied first.
inline std::vector<double> peak_memory(const DepGraph& g, const ReplayResult& r, const MemoryParams& mp) {
  const Schedule& s = *g.schedule;
  const int D = s.num_devices();
  std::vector<std::vector<std::pair<double, double>>> ev(static_cast<std::size_t>(D));
  std::vector<std::vector<std::pair<int, double>>> recomputed(static_cast<std::size_t>(D));  // (mb, FF start)
  std::vector<bool> replicated(static_cast<std::size_t>(D), false);
  for (int i = 0; i < g.size(); ++i) {
    const Instruction& in = *g.flat[static_cast<std::size_t>(i)];
    const int d = in.device;
    const double mult = d == 0 ? mp.stage0_mult : 1.0;
    auto& e = ev[static_cast<std::size_t>(d)];
    const double a = r.start[static_cast<std::size_t>(i)], z = r.end[static_cast<std::size_t>(i)];
    switch (in.kind) {
      case InstrKind::FE: e.push_back({a, mult * mp.fe_bytes}); break;
      case InstrKind::BE: e.push_back({z, -mult * mp.fe_bytes}); break;
      case InstrKind::FF:
        e.push_back({a, mult * mp.ff_bytes});
        if (in.has_flag(kFlagRecompute)) recomputed[static_cast<std::size_t>(d)].push_back({in.micro_batch, a});
        break;
      case InstrKind::BF: e.push_back({z, -mult * mp.ff_bytes}); break;
      default: break;
    }
    if (in.kind == InstrKind::AR && in.has_flag(kFlagReplicatedParams)) replicated[static_cast<std::size_t>(d)] = true;
  }
  // baselines: an FF that recomputes FE holds those activations until the
  // block's BF on that device ends; replicated parameters add the static
  // bytes once more
  for (int i = 0; i < g.size(); ++i) {
    const Instruction& in = *g.flat[static_cast<std::size_t>(i)];
    if (in.kind != InstrKind::BF) continue;
    const int d = in.device;
    for (const auto& [mb, t0] : recomputed[static_cast<std::size_t>(d)])
      if (mb == in.micro_batch) {
        const double mult = d == 0 ? mp.stage0_mult : 1.0;
        ev[static_cast<std::size_t>(d)].push_back({t0, mult * mp.fe_bytes});
        ev[static_cast<std::size_t>(d)].push_back({r.end[static_cast<std::size_t>(i)], -mult * mp.fe_bytes});
      }
  }
  std::vector<double> peak(static_cast<std::size_t>(D), 0.0);
  for (int d = 0; d < D; ++d) {
    auto& e = ev[static_cast<std::size_t>(d)];
    std::sort(e.begin(), e.end());  // (time, delta): releases (negative) first at equal times
    double live = 0, best = 0;
    for (const auto& x : e) {
      live += x.second;
      best = std::max(best, live);
    }
    const bool twice = mp.replicate_static && replicated[static_cast<std::size_t>(d)];
    peak[static_cast<std::size_t>(d)] = mp.static_of(d) * (twice ? 2.0 : 1.0) + best;
  }
  return peak;
}

struct Candidate {
  int k = 0;
  double makespan = 0, throughput = 0, bubble_ratio = 0, peak_max = 0;
  std::vector<double> peak;
  bool feasible = false;
};

struct TuneResult {
  int k_star = 0;
  bool tuned = false;
  double m_activation = 0;
  int k_max = 0;
  std::vector<Candidate> table;
  std::string rationale;
};

/// One simulated WaveK(P, N_mb, k) under the phase times: makespan, bubble,
/// throughput (micro-batches per time unit of t) and per-device peak memory.
inline Candidate simulate_wavek(int P, int N_mb, int k, const PhaseTimes& t, const MemoryParams& mp) {
  WaveKOptions opt;
  opt.times = t;
  const Schedule s = wavek(P, N_mb, k, opt);
  const DepGraph g = build_dependencies(s);
  const std::vector<double> d = phase_durations(g, t);
  const ReplayResult r = replay(g, d);
  if (!r.ok) throw deadlock_error("tuner: wavek replay stalled: " + r.blocked);
  Candidate c;
  c.k = k;
  c.makespan = r.makespan;
  c.throughput = r.makespan > 0 ? N_mb / r.makespan : 0.0;
  c.bubble_ratio = bubble_of(g, r, d).bubble_ratio;
  c.peak = peak_memory(g, r, mp);
  c.peak_max = *std::max_element(c.peak.begin(), c.peak.end());
  return c;
}

/// tune with feasible_k.
inline TuneResult tune(int P, int N_mb, const PhaseTimes& t, const MemoryParams& mp, bool divisors_only = true) {
  if (P < 1 || N_mb < P) throw domain_error("tune: need P >= 1 and N_mb >= P");
  t.check();
  TuneResult res;
  double st_max = 0;
  for (int d = 0; d < P; ++d) st_max = std::max(st_max, mp.static_of(mp.static_bytes.size() == 1 ? 0 : d));
  const double budget = mp.m_mem() - st_max;
  if (!(budget > 0)) {
    res.k_star = P;
    res.rationale = "no activation budget: M_static >= M_mem; default k = P (untuned)";
    return res;
  }
  // M_activation: marginal simulated peak per unit of k (k = P+1 minus k = P)
  const Candidate base = simulate_wavek(P, N_mb, P, t, mp);
  const Candidate next = P + 1 <= N_mb ? simulate_wavek(P, N_mb, P + 1, t, mp) : base;
  res.m_activation = std::max(next.peak_max - base.peak_max, 0.0);
  if (res.m_activation <= 0) {  // no marginal growth: every k fits as far as the formula can tell
    const double per = mp.stage0_mult * (mp.fe_bytes + mp.ff_bytes);
    res.m_activation = per > 0 ? per : 1.0;
  }
  res.k_max = static_cast<int>(std::floor(budget / res.m_activation));
  const int hi = std::min(N_mb, res.k_max);
  for (int k = P; k <= hi; ++k) {
    if (divisors_only && N_mb % k != 0) continue;
    Candidate c = k == P ? base : (k == P + 1 ? next : simulate_wavek(P, N_mb, k, t, mp));
    c.feasible = c.peak_max <= mp.m_mem();
    res.table.push_back(std::move(c));
  }
  const Candidate* best = nullptr;
  for (const Candidate& c : res.table)
    if (c.feasible && (!best || c.throughput > best->throughput * (1.0 + 1e-12))) best = &c;
  if (!best) {
    res.k_star = P;
    res.rationale = res.k_max < P ? "k_max < P: no feasible k; default k = P (untuned)"
                                  : "no candidate within the memory budget; default k = P (untuned)";
    return res;
  }
  res.k_star = best->k;
  res.tuned = true;
  res.rationale = "argmax simulated throughput over " + std::to_string(res.table.size()) +
                  " memory-feasible candidates (ties -> smaller k)";
  return res;
}

}  // namespace tuner
}  // namespace janus
