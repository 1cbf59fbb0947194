// janus/rendezvous.hpp — transfer channels of a multi-process (one process per
// GPU) pipeline, the executor's per-rank stream program, and a blocking-
// rendezvous simulator that proves a program cannot deadlock under NCCL
// semantics before anything is issued.
//
// Channels.  The reference pairs a send with a receive by the key (payload,
// suffix, micro-batch, from, to) (graph.hpp:87-118): activation and gradient
// traffic pair up independently.  The executor names a channel (flow, from
// device, to device): flow = act (FE chain up), adj (FF chain down), tan (BF
// chain up), badj (BE chain down), plus the 1F1B-2nd mirror flows (block
// input to the force replica and its cotangent back, split by block parity).
// Every channel carries one payload per micro-batch, in device-list order on
// both ends (checked by the trainer).
//
// Why channels get their own streams.  ncclSend / ncclRecv block their stream
// until the peer's matching operation runs ("blocking for the GPU"), and ops
// of one communicator are serialised in issue order.  If all of a rank's
// sends share one stream (and all receives another), the cross-flow order of
// the device lists must agree end to end, which SymFold does not satisfy: at
// P=2 device 0 sends [SAE mb3, SGF mb0] while device 1 receives [RGF mb0,
// RAE mb3] — a circular wait.  With one communicator and one stream per
// channel end, each channel is a FIFO on both sides; the only waits left are
// the DepGraph's own edges plus per-channel FIFO order, which follow
// device-list order, so the union stays acyclic (simulate() checks it).
#pragma once

#include <algorithm>
#include <cstdint>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "janus/ir.hpp"
#include "janus/slots.hpp"

namespace janus {

enum Flow : int { kFlowAct = 0, kFlowAdj = 1, kFlowTan = 2, kFlowBadj = 3, kFlowMirror = 4, kFlowMirrorBack = 6, kNumFlows = 8 };

/// Flow of a comm instruction under a 2P-virtual-stage layout; -1 for the
/// fold-point pair of 1F1B-2nd (FE top -> FF top on the same block; carried by
/// the mirror flow instead).
inline int comm_flow(const Instruction& in, int P) {
  const int vs = in.virtual_stage;
  const bool send = is_send(in.kind);
  const int s_vs = send ? vs : comm_peer_stage(in.kind, vs);
  const int r_vs = send ? comm_peer_stage(in.kind, vs) : vs;
  const CommClass c = comm_class(in.kind);
  if (c == CommClass::SA || c == CommClass::RA) {
    if (s_vs == P - 1 && r_vs == P) return -1;
    return r_vs < P ? kFlowAct : kFlowAdj;
  }
  if (s_vs == P && r_vs == P - 1) return -1;
  return r_vs >= P ? kFlowTan : kFlowBadj;
}

struct ChannelKey {
  int flow = 0, from = 0, to = 0;  // schedule devices
  bool operator<(const ChannelKey& o) const { return std::tie(flow, from, to) < std::tie(o.flow, o.from, o.to); }
  bool operator==(const ChannelKey& o) const { return flow == o.flow && from == o.from && to == o.to; }
};

/// Device of block b's energy half (E_b) and force half (F_b).
inline int energy_device(const Schedule& s, int b) { return s.stage_map[static_cast<size_t>(b)]; }
inline int force_device(const Schedule& s, int P, int b) { return s.stage_map[static_cast<size_t>(2 * P - 1 - b)]; }

/// Every channel of a schedule (deterministic order: all ranks number them
/// identically).  onef1b adds the mirror channels of blocks >= 1.
inline std::vector<ChannelKey> schedule_channels(const Schedule& s, int P, bool onef1b) {
  std::map<ChannelKey, int> seen;
  for (const auto& dl : s.device_lists)
    for (const Instruction& in : dl) {
      if (!is_comm(in.kind)) continue;
      const int f = comm_flow(in, P);
      if (f < 0) continue;
      const int from = is_send(in.kind) ? in.device : in.peer_device;
      const int to = is_send(in.kind) ? in.peer_device : in.device;
      seen[{f, from, to}] = 1;
    }
  if (onef1b)
    for (int b = 1; b < P; ++b) {
      seen[{kFlowMirror + (b & 1), energy_device(s, b), force_device(s, P, b)}] = 1;
      seen[{kFlowMirrorBack + (b & 1), force_device(s, P, b), energy_device(s, b)}] = 1;
    }
  std::vector<ChannelKey> out;
  for (const auto& kv : seen) out.push_back(kv.first);
  return out;
}

inline int channel_index(const std::vector<ChannelKey>& chans, const ChannelKey& k) {
  const auto it = std::lower_bound(chans.begin(), chans.end(), k);
  if (it == chans.end() || !(*it == k)) throw state_error("transfer on an unknown channel");
  return static_cast<int>(it - chans.begin());
}

// ------------------------------------------------------------------ program
/// One GPU-side operation of a rank's issue program.
struct StreamOp {
  enum Kind : std::uint8_t { kWork, kSend, kRecv, kCollective } kind = kWork;
  int channel = -1;  // kSend / kRecv: channel index; kCollective: group id
  int mb = -1;
  std::vector<std::pair<int, int>> deps;  // (stream, op index) that must have completed
  std::string what;
};

struct RankProgram {
  int rank = 0;
  std::vector<std::vector<StreamOp>> streams;  // stream 0..lanes-1 = compute lanes
};

/// How the executor maps transfers onto streams.
enum class StreamLayout {
  kPerChannel,  // the executor's layout: one send / recv stream per channel end
  kSharedPair   // round 1: one send stream and one recv stream per rank (deadlocks)
};

/// The per-rank stream program the NCCL-mode executor issues for one step of
/// `s` (mirrors executor.cpp execute(): micro-batch m computes on lane
/// m % lanes; a send waits for its lane, a receive's lane waits for it; 1F1B
/// mirror transfers at FE / FF / BF / BE; OS joins the lanes on lane 0 and
/// runs the group all-reduces: group 0 = 1F1B pair, 1 = data-parallel).
inline std::vector<RankProgram> build_programs(const Schedule& s, int P, bool onef1b, int lanes, int dp,
                                               StreamLayout layout, bool pooled_slots = true) {
  const std::vector<ChannelKey> chans = schedule_channels(s, P, onef1b);
  const int nch = static_cast<int>(chans.size());
  std::vector<RankProgram> progs;
  for (int r = 0; r < dp; ++r)
    for (int d = 0; d < P; ++d) {
      RankProgram pg;
      pg.rank = r * P + d;
      const int n_streams = lanes + (layout == StreamLayout::kPerChannel ? 2 * nch : 2);
      pg.streams.assign(static_cast<size_t>(n_streams), {});
      auto lane = [&](int mb) { return (mb < 0 ? 0 : mb) % lanes; };
      auto send_stream = [&](int ch) { return layout == StreamLayout::kPerChannel ? lanes + 2 * ch : lanes; };
      auto recv_stream = [&](int ch) { return layout == StreamLayout::kPerChannel ? lanes + 2 * ch + 1 : lanes + 1; };
      auto tail = [&](int st) { return std::make_pair(st, static_cast<int>(pg.streams[static_cast<size_t>(st)].size()) - 1); };
      auto push = [&](int st, StreamOp op) { pg.streams[static_cast<size_t>(st)].push_back(std::move(op)); };
      auto send = [&](const ChannelKey& k, int mb, const std::string& what) {
        const int ch = channel_index(chans, k);
        StreamOp op{StreamOp::kSend, ch, mb, {}, what};
        if (!pg.streams[static_cast<size_t>(lane(mb))].empty()) op.deps.push_back(tail(lane(mb)));
        push(send_stream(ch), op);
      };
      auto recv = [&](const ChannelKey& k, int mb, const std::string& what) {
        const int ch = channel_index(chans, k);
        push(recv_stream(ch), StreamOp{StreamOp::kRecv, ch, mb, {}, what});
        push(lane(mb), StreamOp{StreamOp::kWork, -1, mb, {tail(recv_stream(ch))}, "wait " + what});
      };
      auto work = [&](int mb, const std::string& what) { push(lane(mb), StreamOp{StreamOp::kWork, -1, mb, {}, what}); };
      // ops each instruction pushed (for the activation slot pool's waits below)
      const auto& dl = s.device_lists[static_cast<size_t>(d)];
      std::vector<std::vector<std::pair<int, int>>> pushed(dl.size());
      auto sizes = [&] {
        std::vector<int> z;
        for (const auto& st : pg.streams) z.push_back(static_cast<int>(st.size()));
        return z;
      };
      for (size_t ii = 0; ii < dl.size(); ++ii) {
        const Instruction& in = dl[ii];
        const std::vector<int> before = sizes();
        const int mb = in.micro_batch;
        const int b = in.virtual_stage < P ? in.virtual_stage : 2 * P - 1 - in.virtual_stage;
        const std::string tag = std::string(to_string(in.kind)) + " mb" + std::to_string(mb) + " vs" + std::to_string(in.virtual_stage);
        switch (in.kind) {
          case InstrKind::FE:
            work(mb, tag);
            if (onef1b && b > 0) send({kFlowMirror + (b & 1), d, force_device(s, P, b)}, mb, "mirror-act " + tag);
            break;
          case InstrKind::FF:
            if (onef1b && b > 0) recv({kFlowMirror + (b & 1), energy_device(s, b), d}, mb, "mirror-act " + tag);
            work(mb, tag);
            break;
          case InstrKind::BF:
            work(mb, tag);
            if (onef1b && b > 0) send({kFlowMirrorBack + (b & 1), d, energy_device(s, b)}, mb, "mirror-back " + tag);
            break;
          case InstrKind::BE:
            work(mb, tag);
            if (onef1b && b > 0) recv({kFlowMirrorBack + (b & 1), force_device(s, P, b), d}, mb, "mirror-back " + tag);
            break;
          case InstrKind::OS: {
            StreamOp join{StreamOp::kWork, -1, -1, {}, "OS join"};
            for (int l = 1; l < lanes; ++l)
              if (!pg.streams[static_cast<size_t>(l)].empty()) join.deps.push_back(tail(l));
            push(0, join);
            if (onef1b) push(0, StreamOp{StreamOp::kCollective, 0, -1, {}, "pair all-reduce"});
            if (dp > 1) push(0, StreamOp{StreamOp::kCollective, 1, -1, {}, "dp all-reduce"});
            work(-1, "Adam");
            break;
          }
          default:
            if (!is_comm(in.kind)) break;
            {
              const int f = comm_flow(in, P);
              if (f < 0) break;
              const int from = is_send(in.kind) ? in.device : in.peer_device;
              const int to = is_send(in.kind) ? in.peer_device : in.device;
              if (is_send(in.kind)) send({f, from, to}, mb, tag);
              else recv({f, from, to}, mb, tag);
            }
        }
        for (size_t st = 0; st < pg.streams.size(); ++st)
          for (int x = before[st]; x < static_cast<int>(pg.streams[st].size()); ++x) pushed[ii].push_back({static_cast<int>(st), x});
      }
      if (pooled_slots) {
        // slot reuse (executor.cpp slot_of): every op of an instruction that
        // uses a reused slot waits for the previous occupant's release, the
        // last op of its last instruction (a superset of the executor's waits)
        std::vector<const Instruction*> ord;
        for (const Instruction& in : dl) ord.push_back(&in);
        auto held = [&](int obj) {
          return obj < P ? energy_device(s, obj) == d : force_device(s, P, obj - P) == d;
        };
        const SlotPlan sp = plan_slots(ord, s, P, onef1b, false, 0, false, held, lanes);
        std::vector<int> objs;
        for (size_t ii = 0; ii < dl.size(); ++ii) {
          slot_touches(dl[ii], s, P, onef1b, false, &objs);
          for (int o : objs) {
            if (!held(o)) continue;
            const int prev = sp.prev.at({o, dl[ii].micro_batch});
            if (prev < 0) continue;
            const auto& rel = pushed[static_cast<size_t>(sp.last.at({o, prev}))];
            if (rel.empty()) continue;
            for (const auto& op : pushed[ii]) {
              auto& deps = pg.streams[static_cast<size_t>(op.first)][static_cast<size_t>(op.second)].deps;
              if (op.first != rel.back().first) deps.push_back(rel.back());
            }
          }
        }
      }
      progs.push_back(std::move(pg));
    }
  return progs;
}

/// Result of a blocking-rendezvous simulation.
struct RendezvousReport {
  bool ok = true;
  int64_t ops = 0, completed = 0;
  std::string stuck;  // heads of the blocked streams when no op can progress
};

/// Executes the programs with NCCL semantics: a stream runs its ops in order;
/// an op starts once its deps completed; a send and the receive with the same
/// channel and sequence number (n-th send pairs with n-th receive of the
/// channel) complete TOGETHER, only when both are at the head of their streams
/// (blocking rendezvous, no buffering); a collective completes when every
/// member of its group (group 0: ranks r and r' holding one block's two
/// copies, 1F1B; group 1: ranks of one device across replicas) is at it.
inline RendezvousReport simulate(const std::vector<RankProgram>& progs, int P, const Schedule& s, bool onef1b) {
  RendezvousReport rep;
  const size_t R = progs.size();
  std::vector<std::vector<int>> head(R), done_upto(R);  // per stream: next op; ops [0, done) completed
  for (size_t r = 0; r < R; ++r) {
    head[r].assign(progs[r].streams.size(), 0);
    for (const auto& st : progs[r].streams) rep.ops += static_cast<int64_t>(st.size());
  }
  // sequence number of each send / recv op on its channel (per rank pair)
  std::vector<std::vector<std::vector<int>>> seq(R);
  std::map<std::tuple<size_t, int, int>, int> counter;  // (rank, channel, kind) -> count
  for (size_t r = 0; r < R; ++r) {
    seq[r].resize(progs[r].streams.size());
    for (size_t st = 0; st < progs[r].streams.size(); ++st)
      for (const StreamOp& op : progs[r].streams[st]) {
        int q = -1;
        if (op.kind == StreamOp::kSend || op.kind == StreamOp::kRecv) q = counter[{r, op.channel, op.kind}]++;
        seq[r][st].push_back(q);
      }
  }
  const std::vector<ChannelKey> chans = schedule_channels(s, P, onef1b);
  auto deps_done = [&](size_t r, const StreamOp& op) {
    for (const auto& dp : op.deps)
      if (head[r][static_cast<size_t>(dp.first)] <= dp.second) return false;
    return true;
  };
  // find the op at the head of some stream of rank rr that matches (kind, channel, seq)
  auto find_head = [&](size_t rr, StreamOp::Kind k, int ch, int q, size_t* st_out) {
    for (size_t st = 0; st < progs[rr].streams.size(); ++st) {
      const int h = head[rr][st];
      if (h >= static_cast<int>(progs[rr].streams[st].size())) continue;
      const StreamOp& op = progs[rr].streams[st][static_cast<size_t>(h)];
      if (op.kind == k && op.channel == ch && seq[rr][st][static_cast<size_t>(h)] == q && deps_done(rr, op)) {
        *st_out = st;
        return true;
      }
    }
    return false;
  };
  const int dp = static_cast<int>(R) / P;
  bool progress = true;
  while (progress) {
    progress = false;
    for (size_t r = 0; r < R; ++r)
      for (size_t st = 0; st < progs[r].streams.size(); ++st) {
        const int h = head[r][st];
        if (h >= static_cast<int>(progs[r].streams[st].size())) continue;
        const StreamOp& op = progs[r].streams[st][static_cast<size_t>(h)];
        if (!deps_done(r, op)) continue;
        const int replica = static_cast<int>(r) / P;
        if (op.kind == StreamOp::kWork) {
          ++head[r][st];
          progress = true;
        } else if (op.kind == StreamOp::kSend) {
          const size_t peer = static_cast<size_t>(replica * P + chans[static_cast<size_t>(op.channel)].to);
          size_t pst = 0;
          if (find_head(peer, StreamOp::kRecv, op.channel, seq[r][st][static_cast<size_t>(h)], &pst)) {
            ++head[r][st];
            ++head[peer][pst];
            progress = true;
          }
        } else if (op.kind == StreamOp::kCollective) {
          std::vector<size_t> members;
          const int d = static_cast<int>(r) % P;
          if (op.channel == 0) {  // 1F1B pair: devices holding block b's energy and force copies
            for (int b = 0; b < P; ++b)
              if (energy_device(s, b) == d || force_device(s, P, b) == d) {
                members.push_back(static_cast<size_t>(replica * P + energy_device(s, b)));
                members.push_back(static_cast<size_t>(replica * P + force_device(s, P, b)));
              }
          } else {
            for (int q = 0; q < dp; ++q) members.push_back(static_cast<size_t>(q * P + d));
          }
          std::sort(members.begin(), members.end());
          members.erase(std::unique(members.begin(), members.end()), members.end());
          std::vector<std::pair<size_t, size_t>> at;
          bool all = true;
          for (size_t m : members) {
            size_t pst = 0;
            bool found = false;
            for (size_t x = 0; x < progs[m].streams.size() && !found; ++x) {
              const int hh = head[m][x];
              if (hh >= static_cast<int>(progs[m].streams[x].size())) continue;
              const StreamOp& o2 = progs[m].streams[x][static_cast<size_t>(hh)];
              if (o2.kind == StreamOp::kCollective && o2.channel == op.channel && deps_done(m, o2)) {
                pst = x;
                found = true;
              }
            }
            if (!found) {
              all = false;
              break;
            }
            at.emplace_back(m, pst);
          }
          if (all) {
            for (const auto& a : at) ++head[a.first][a.second];
            progress = true;
          }
        }
      }
  }
  for (size_t r = 0; r < R; ++r)
    for (size_t st = 0; st < progs[r].streams.size(); ++st) {
      rep.completed += head[r][st];
      const int h = head[r][st];
      if (h < static_cast<int>(progs[r].streams[st].size()) && rep.stuck.size() < 2000)
        rep.stuck += "rank " + std::to_string(progs[r].rank) + " stream " + std::to_string(st) + ": " +
                     progs[r].streams[st][static_cast<size_t>(h)].what + "\n";
    }
  rep.ok = rep.completed == rep.ops;
  return rep;
}

}  // namespace janus
