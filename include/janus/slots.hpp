// janus/slots.hpp — activation slot pool: the SymFold memory fold realised in
// the executor.
//
// A stage object keeps one activation slot (every unit's saved tensors, the
// per-pair filters and the transfer ports) per micro-batch that is live on it.
// The SPEC lifetime rule makes a micro-batch live on a stage
// from its first use (FE, or the receive that feeds it) to its last (BE, or
// the send that drains it); PAPER.md:334-340 is why SymFold wins: the fold
// co-locates E_b and F_b, so a micro-batch's FE->BE span on device d is short
// and few slots suffice.  The executor therefore sizes each stage object's
// pool by the maximum number of micro-batches whose [first, last] use
// intervals overlap in its issue order, and hands a slot to the next
// micro-batch when the previous occupant is done with it:
//   * the release is an event recorded after the occupant's last use (on the
//     stream that last used it: its lane, or the send stream draining it);
//   * every use of a reused slot by a new occupant waits for that event.
// Slots are chosen lowest-free-first in issue order, so the assignment is a
// deterministic function of the schedule (graph capture / replay safe, and
// identical on every rank).  Results do not depend on it: a slot holds no
// state across micro-batches.
//
// Objects: E_b (energy half of block b) is object b; F_b is object b too when
// it is the same stage object (SymFold, WaveK, Hanayo: the fold), P + b for
// 1F1B-2nd's replicated force copy.
#pragma once

#include <algorithm>
#include <map>
#include <utility>
#include <vector>

#include "janus/graph.hpp"
#include "janus/ir.hpp"

namespace janus {

inline int slot_obj_energy(int b, int /*P*/, bool /*onef1b*/) { return b; }
inline int slot_obj_force(int b, int P, bool onef1b) { return onef1b ? P + b : b; }

/// Objects whose activation slot of `in.micro_batch` an instruction touches,
/// following executor.cpp execute() exactly: the phase's own stage, the
/// same-device hand-off after a phase (1F1B-2nd: two blocks per device), the
/// 1F1B-2nd mirror transfers, and the transfer ports.  `local`: all stages in
/// one process (a send writes the receiver's port); per-rank: a receive
/// writes it.  Fold-point pairs of 1F1B-2nd carry nothing.
inline void slot_touches(const Instruction& in, const Schedule& s, int P, bool onef1b, bool local,
                         std::vector<int>* objs) {
  objs->clear();
  const int vs = in.virtual_stage, S = 2 * P;
  auto block = [&](int v) { return v < P ? v : S - 1 - v; };
  auto obj_of_vs = [&](int v) { return v < P ? slot_obj_energy(v, P, onef1b) : slot_obj_force(block(v), P, onef1b); };
  auto handoff = [&](int from, int to) {
    if (to < 0 || to >= S) return;
    if (s.stage_map[static_cast<size_t>(from)] != s.stage_map[static_cast<size_t>(to)]) return;
    if ((from == P - 1 && to == P) || (from == P && to == P - 1)) return;
    const int a = obj_of_vs(from), b = obj_of_vs(to);
    if (a != b) objs->push_back(b);
  };
  const int b = block(vs);
  switch (in.kind) {
    case InstrKind::FE:
      objs->push_back(slot_obj_energy(b, P, onef1b));
      handoff(vs, vs + 1);
      if (onef1b && b > 0 && local) objs->push_back(slot_obj_force(b, P, onef1b));  // mirror act written into F_b
      return;
    case InstrKind::FF:
      objs->push_back(slot_obj_force(b, P, onef1b));
      handoff(vs, vs + 1);
      return;
    case InstrKind::BF:
      objs->push_back(slot_obj_force(b, P, onef1b));
      handoff(vs, vs - 1);
      return;
    case InstrKind::BE:
      objs->push_back(slot_obj_energy(b, P, onef1b));
      handoff(vs, vs - 1);
      return;
    default:
      break;
  }
  if (!is_comm(in.kind)) return;
  const bool send = is_send(in.kind);
  const int s_vs = send ? vs : comm_peer_stage(in.kind, vs);
  const int r_vs = send ? comm_peer_stage(in.kind, vs) : vs;
  if ((s_vs == P - 1 && r_vs == P) || (s_vs == P && r_vs == P - 1)) return;  // fold point
  if (send) {
    objs->push_back(obj_of_vs(s_vs));
    if (local) objs->push_back(obj_of_vs(r_vs));
  } else if (!local) {
    objs->push_back(obj_of_vs(r_vs));
  }
}

/// Slot assignment over one issue order (local mode: the global topological
/// order; per-rank: this device's list).  `held(obj)` filters the objects
/// this process owns.  `lanes`: micro-batches the executor overlaps on one
/// device (micro-batch m on compute stream m % lanes); a pool holds at least
/// min(lanes, micro-batches) slots so concurrent lanes never queue on one
/// another's releases, and a freed slot is reused oldest-release-first.
struct SlotPlan {
  int n_obj = 0;
  std::vector<int> n_slots;                         // per object (0: not held / untouched)
  std::map<std::pair<int, int>, int> slot;          // (obj, mb) -> slot
  std::map<std::pair<int, int>, int> prev;          // (obj, mb) -> previous occupant's mb (-1: first)
  std::vector<std::vector<std::pair<int, int>>> release_after;  // per issue index: (obj, mb) last used there
  std::map<std::pair<int, int>, int> first, last;   // (obj, mb) -> issue index of first / last use
};

template <class Held>
SlotPlan plan_slots(const std::vector<const Instruction*>& order, const Schedule& s, int P, bool onef1b, bool local,
                    int n_mb, bool unfolded, Held&& held, int lanes = 1) {
  SlotPlan sp;
  sp.n_obj = onef1b ? 2 * P : P;
  sp.n_slots.assign(static_cast<size_t>(sp.n_obj), 0);
  sp.release_after.assign(order.size(), {});
  std::vector<int> objs;
  for (size_t i = 0; i < order.size(); ++i) {
    slot_touches(*order[i], s, P, onef1b, local, &objs);
    for (int o : objs) {
      if (!held(o)) continue;
      const std::pair<int, int> k{o, order[i]->micro_batch};
      if (!sp.first.count(k)) sp.first[k] = static_cast<int>(i);
      sp.last[k] = static_cast<int>(i);
    }
  }
  if (unfolded) {  // one slot per micro-batch: slot = mb, nothing is ever reused
    for (const auto& kv : sp.first) {
      sp.slot[kv.first] = kv.first.second;
      sp.prev[kv.first] = -1;
      sp.n_slots[static_cast<size_t>(kv.first.first)] = n_mb;
    }
    return sp;
  }
  // in order of first use: a new slot while the pool is below the lane floor,
  // else the free slot released longest ago (a slot is free once its
  // occupant's last use was issued before this first use), else a new slot
  std::vector<std::vector<std::pair<int, int>>> occ(static_cast<size_t>(sp.n_obj));  // per obj, slot -> (mb, last)
  std::vector<std::pair<int, std::pair<int, int>>> starts;
  std::map<int, int> mbs_of;
  for (const auto& kv : sp.first) {
    starts.push_back({kv.second, kv.first});
    ++mbs_of[kv.first.first];
  }
  std::sort(starts.begin(), starts.end());
  for (const auto& st : starts) {
    const std::pair<int, int> k = st.second;
    auto& pool = occ[static_cast<size_t>(k.first)];
    const int floor = std::min(std::max(1, lanes), mbs_of[k.first]);
    int pick = -1;
    if (static_cast<int>(pool.size()) >= floor)
      for (size_t x = 0; x < pool.size(); ++x)
        if (pool[x].second < st.first && (pick < 0 || pool[x].second < pool[static_cast<size_t>(pick)].second))
          pick = static_cast<int>(x);
    if (pick < 0) {
      pick = static_cast<int>(pool.size());
      pool.push_back({-1, -1});
    }
    sp.prev[k] = pool[static_cast<size_t>(pick)].first;
    pool[static_cast<size_t>(pick)] = {k.second, sp.last[k]};
    sp.slot[k] = pick;
  }
  for (size_t o = 0; o < occ.size(); ++o) sp.n_slots[o] = static_cast<int>(occ[o].size());
  for (const auto& kv : sp.prev)  // occupants that hand their slot on release it after their last use
    if (kv.second >= 0) {
      const std::pair<int, int> p{kv.first.first, kv.second};
      sp.release_after[static_cast<size_t>(sp.last.at(p))].push_back(p);
    }
  return sp;
}

/// Local-mode issue order (all P virtual devices in one process): Kahn's
/// FIFO topological order of the full DAG (seq + data edges), so every send is
/// issued before its receive.  Flat instruction indices.
inline std::vector<int> local_issue_order(const DepGraph& g) {
  const int n = g.size();
  std::vector<int> indeg(static_cast<size_t>(n));
  std::vector<std::vector<int>> succ(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) {
    indeg[static_cast<size_t>(i)] = static_cast<int>(g.preds[static_cast<size_t>(i)].size());
    for (int p : g.preds[static_cast<size_t>(i)]) succ[static_cast<size_t>(p)].push_back(i);
  }
  std::vector<int> q;
  for (int i = 0; i < n; ++i)
    if (indeg[static_cast<size_t>(i)] == 0) q.push_back(i);
  for (size_t h = 0; h < q.size(); ++h)
    for (int x : succ[static_cast<size_t>(q[h])])
      if (--indeg[static_cast<size_t>(x)] == 0) q.push_back(x);
  if (static_cast<int>(q.size()) != n) throw deadlock_error("schedule dependency graph has a cycle");
  return q;
}

/// Pool size per device of a schedule: the largest pool among the stage
/// objects each device holds (local: one process issuing the global order;
/// per-rank: each device issuing its own list).
inline std::vector<int> slot_pool_sizes(const Schedule& s, int P, bool onef1b, bool local, bool unfolded, int n_mb,
                                        int lanes = 1) {
  const int D = s.num_devices();
  std::vector<int> out(static_cast<size_t>(D), 0);
  auto dev_of = [&](int obj) {
    return obj < P ? s.stage_map[static_cast<size_t>(obj)] : s.stage_map[static_cast<size_t>(2 * P - 1 - (obj - P))];
  };
  if (local) {
    const DepGraph g = build_dependencies(s);
    std::vector<const Instruction*> ord;
    for (int idx : local_issue_order(g)) ord.push_back(g.flat[static_cast<size_t>(idx)]);
    const SlotPlan sp = plan_slots(ord, s, P, onef1b, true, n_mb, unfolded, [](int) { return true; }, lanes);
    for (int o = 0; o < sp.n_obj; ++o) {
      int& v = out[static_cast<size_t>(dev_of(o))];
      v = std::max(v, sp.n_slots[static_cast<size_t>(o)]);
    }
    return out;
  }
  for (int d = 0; d < D; ++d) {
    std::vector<const Instruction*> ord;
    for (const Instruction& in : s.device_lists[static_cast<size_t>(d)]) ord.push_back(&in);
    const SlotPlan sp = plan_slots(ord, s, P, onef1b, false, n_mb, unfolded, [&](int o) { return dev_of(o) == d; }, lanes);
    for (int o = 0; o < sp.n_obj; ++o) out[static_cast<size_t>(d)] = std::max(out[static_cast<size_t>(d)], sp.n_slots[static_cast<size_t>(o)]);
  }
  return out;
}

}  // namespace janus
