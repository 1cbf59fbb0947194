// janus/gars.hpp — GARS (graph-aware re-scheduling): pack-and-shuffle
// micro-batching, comm-free / dist tagging, second-level GP bin assignment,
// the synthetic long-tailed size distribution and balance statistics.
//
// SPEC-only in the reference (module "gars"; PAPER.md
// Appendix A, Algorithm 1 at PAPER.md:708-733, complexity PAPER.md:737-744),
// implemented here in the style of the reference headers: value types, pure
// deterministic functions, janus::domain_error / state_error on bad input.
// Pinned choices: sort by atoms descending with ties by id
// ascending; min-load argmin with ties to the lowest index (a heap keyed by
// (load, index): O(M log M + M log N_mb)); ONE SplitMix64(seed) stream
// shuffles micro-batch 0, 1, ... in turn with the descending Fisher-Yates of
// rng.hpp:29-34; inverse-CDF sampling through the percentile anchors.
// GARS only regroups graphs: the step gradient is a sum over graphs, so it
// is unchanged — the executor's fixed-order ledger
// reduction makes that exact for a given grouping.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <functional>
#include <queue>
#include <utility>
#include <vector>

#include "janus/errors.hpp"
#include "janus/rng.hpp"

namespace janus {
namespace gars {

/// One atomic graph (structure): SPEC.md:498-502.
struct AtomGraph {
  std::int64_t id = 0;
  int atoms = 1;            // size(g), the cost proxy
  std::int64_t edges = 0;   // statistics only
};

enum class MbTag : std::uint8_t { comm_free = 0, dist = 1 };

/// SPEC.md:504-509.
struct PackedMicroBatch {
  std::vector<AtomGraph> graphs;                 // shuffled order
  MbTag tag = MbTag::comm_free;
  std::vector<std::vector<std::int64_t>> gp_bins;  // graph ids per GP bin (comm_free, on request)
  std::int64_t total_atoms = 0;
};

/// Tagging rule of Algorithm 1: comm_free iff
/// max size <= C_rank = total / d_gp (compared exactly: max * d_gp <= total).
inline MbTag tag_of(const std::vector<AtomGraph>& g, int d_gp) {
  std::int64_t total = 0;
  int mx = 0;
  for (const auto& x : g) {
    total += x.atoms;
    mx = std::max(mx, x.atoms);
  }
  return static_cast<std::int64_t>(mx) * d_gp <= total ? MbTag::comm_free : MbTag::dist;
}

/// pack_and_shuffle (Algorithm 1).
inline std::vector<PackedMicroBatch> pack_and_shuffle(const std::vector<AtomGraph>& batch, int N_mb, int d_gp,
                                                      std::uint64_t seed) {
  if (batch.empty()) throw domain_error("pack_and_shuffle: empty batch");
  if (N_mb < 1) throw domain_error("pack_and_shuffle: N_mb must be >= 1");
  if (d_gp < 1) throw domain_error("pack_and_shuffle: d_gp must be >= 1");
  for (const auto& g : batch)
    if (g.atoms < 1) throw domain_error("pack_and_shuffle: graph with atoms < 1");
  std::vector<AtomGraph> sorted = batch;
  std::stable_sort(sorted.begin(), sorted.end(), [](const AtomGraph& a, const AtomGraph& b) {
    return a.atoms != b.atoms ? a.atoms > b.atoms : a.id < b.id;
  });
  std::vector<PackedMicroBatch> out(static_cast<std::size_t>(N_mb));
  using Load = std::pair<std::int64_t, int>;  // (current total, index): min-heap = argmin, ties -> lowest index
  std::priority_queue<Load, std::vector<Load>, std::greater<Load>> heap;
  for (int j = 0; j < N_mb; ++j) heap.push({0, j});
  for (const auto& g : sorted) {
    const auto [load, j] = heap.top();
    heap.pop();
    out[static_cast<std::size_t>(j)].graphs.push_back(g);
    heap.push({load + g.atoms, j});
  }
  SplitMix64 rng(seed);
  for (auto& mb : out) {
    rng.shuffle(mb.graphs);
    mb.total_atoms = 0;
    for (const auto& g : mb.graphs) mb.total_atoms += g.atoms;
    mb.tag = mb.graphs.empty() ? MbTag::comm_free : tag_of(mb.graphs, d_gp);
  }
  return out;
}

/// assign_gp_bins: graphs in the (shuffled) order to the bin
/// with the minimum atom load, ties to the lowest bin.
inline PackedMicroBatch assign_gp_bins(PackedMicroBatch mb, int d_gp) {
  if (d_gp < 1) throw domain_error("assign_gp_bins: d_gp must be >= 1");
  if (mb.tag != MbTag::comm_free) throw state_error("assign_gp_bins: dist micro-batches have no local bins");
  mb.gp_bins.assign(static_cast<std::size_t>(d_gp), {});
  std::vector<std::int64_t> load(static_cast<std::size_t>(d_gp), 0);
  for (const auto& g : mb.graphs) {
    const auto b = static_cast<std::size_t>(std::min_element(load.begin(), load.end()) - load.begin());
    mb.gp_bins[b].push_back(g.id);
    load[b] += g.atoms;
  }
  return mb;
}

/// Baseline packing: greedy sequential construction of
/// micro-batches in dataset order at a fixed atom budget ceil(total / N_mb),
/// without repacking or shuffling; the last micro-batch takes the rest.
inline std::vector<PackedMicroBatch> greedy_sequential(const std::vector<AtomGraph>& batch, int N_mb) {
  if (batch.empty()) throw domain_error("greedy_sequential: empty batch");
  if (N_mb < 1) throw domain_error("greedy_sequential: N_mb must be >= 1");
  std::int64_t total = 0;
  for (const auto& g : batch) total += g.atoms;
  const std::int64_t budget = (total + N_mb - 1) / N_mb;
  std::vector<PackedMicroBatch> out(static_cast<std::size_t>(N_mb));
  std::size_t j = 0;
  for (const auto& g : batch) {
    if (j + 1 < out.size() && !out[j].graphs.empty() && out[j].total_atoms + g.atoms > budget) ++j;
    out[j].graphs.push_back(g);
    out[j].total_atoms += g.atoms;
  }
  return out;
}

/// Percentile anchors of a size distribution (Table 3).
struct SizeStats {
  double mean = 85, p50 = 53, p90 = 213, p99 = 427, max = 905;
};
inline SizeStats mixed_preset() { return SizeStats{}; }

/// synth_dataset: atom counts by piecewise-linear inverse
/// CDF through (0,1) (0.5,P50) (0.9,P90) (0.99,P99) (1,max), one draw per
/// graph, rounded and clipped to [1, max]; edges = c * atoms^exponent.
inline std::vector<AtomGraph> synth_dataset(const SizeStats& s, int n, std::uint64_t seed, double c = 20.0,
                                            double exponent = 1.3) {
  if (n < 1) throw domain_error("synth_dataset: n must be >= 1");
  if (!(1.0 <= s.p50 && s.p50 <= s.p90 && s.p90 <= s.p99 && s.p99 <= s.max))
    throw domain_error("synth_dataset: percentiles must be non-decreasing");
  const double q[5] = {0.0, 0.5, 0.9, 0.99, 1.0};
  const double v[5] = {1.0, s.p50, s.p90, s.p99, s.max};
  SplitMix64 rng(seed);
  std::vector<AtomGraph> out(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) {
    const double u = rng.next_double();
    int k = 0;
    while (k < 3 && u >= q[k + 1]) ++k;
    const double t = (u - q[k]) / (q[k + 1] - q[k]);
    const double x = v[k] + t * (v[k + 1] - v[k]);
    const int atoms = static_cast<int>(std::min(s.max, std::max(1.0, std::nearbyint(x))));
    out[static_cast<std::size_t>(i)] =
        AtomGraph{i, atoms, static_cast<std::int64_t>(std::llround(c * std::pow(static_cast<double>(atoms), exponent)))};
  }
  return out;
}

/// balance_stats: mean and population std of totals.
inline std::pair<double, double> balance_stats(const std::vector<PackedMicroBatch>& mbs) {
  if (mbs.empty()) throw domain_error("balance_stats: empty list");
  double mean = 0;
  for (const auto& m : mbs) mean += static_cast<double>(m.total_atoms);
  mean /= static_cast<double>(mbs.size());
  double var = 0;
  for (const auto& m : mbs) var += (static_cast<double>(m.total_atoms) - mean) * (static_cast<double>(m.total_atoms) - mean);
  return {mean, std::sqrt(var / static_cast<double>(mbs.size()))};
}

}  // namespace gars
}  // namespace janus
