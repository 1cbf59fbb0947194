// janus/model.hpp — model and stage description (new header in the style of
// the reference's janus API; the reference has no model description, see
// SURVEY.md §8b).
//
// The canonical conservative MLIP is a chain of
// 2L+2 "units": embed, (msg_l, upd_l) for each interaction layer, readout.
// A pipeline of P energy stages partitions the units into P contiguous
// blocks; SymFold (fold_map, ir.hpp:161) puts energy block b and its mirrored
// force stage 2P-1-b on device b, so FE/FF/BF/BE of block b share one
// parameter copy and one activation store.
#pragma once

#include <algorithm>
#include <cstdint>
#include <limits>
#include <string>
#include <utility>
#include <vector>

#include "janus/errors.hpp"

namespace janus {

enum class UnitType : std::uint8_t { embed, msg, upd, readout };

struct ModelConfig {
  int L = 4;            // interaction layers
  int H = 64;           // hidden width
  int R = 64;           // radial basis size
  int n_species = 4;
  double r_c = 5.0;     // cutoff (Angstrom)
  double w_E = 1.0, w_F = 10.0;
  std::uint64_t seed = 7;

  int num_units() const { return 2 * L + 2; }
  UnitType unit_type(int u) const {
    if (u < 0 || u >= num_units()) throw domain_error("unit index out of range");
    if (u == 0) return UnitType::embed;
    if (u == num_units() - 1) return UnitType::readout;
    return (u % 2 == 1) ? UnitType::msg : UnitType::upd;
  }
  std::int64_t unit_param_count(int u) const {
    const std::int64_t h = H, r = R, s = n_species;
    switch (unit_type(u)) {
      case UnitType::embed: return s * h;
      case UnitType::msg: return r * h + h + h * h + h + h * h;
      case UnitType::upd: return h * h + h + h * h;
      default: return h * h + 2 * h + s;
    }
  }
  std::int64_t unit_param_offset(int u) const {
    std::int64_t o = 0;
    for (int x = 0; x < u; ++x) o += unit_param_count(x);
    return o;
  }
  std::int64_t param_count() const { return unit_param_offset(num_units()); }

  /// Relative FE cost of a unit for `avg_degree` neighbours per atom (FLOPs per
  /// atom; the four phases scale it by ~7.5x uniformly).
  double unit_cost(int u, double avg_degree) const {
    const double h = H, r = R;
    switch (unit_type(u)) {
      case UnitType::embed: return 1.0;
      case UnitType::msg: return 2.0 * avg_degree * (r * h + h * h) + 2.0 * h * h;
      case UnitType::upd: return 4.0 * h * h;
      default: return 2.0 * h * h;
    }
  }
};

/// Contiguous unit ranges, one per energy stage (block).
struct StagePlan {
  int P = 1;
  std::vector<std::pair<int, int>> blocks;  // [u_begin, u_end) per block

  int block_of_unit(int u) const {
    for (int b = 0; b < P; ++b)
      if (u >= blocks[static_cast<std::size_t>(b)].first && u < blocks[static_cast<std::size_t>(b)].second) return b;
    throw domain_error("unit not covered by the plan");
  }
};

/// Deterministic min-max contiguous partition of the units into P blocks
/// (integer DP over prefix sums; ties resolved toward earlier cuts).
inline StagePlan partition_units(const ModelConfig& m, int P, double avg_degree = 50.0) {
  const int U = m.num_units();
  if (P < 1 || P > U) throw config_error("P must be in [1, " + std::to_string(U) + "] for L=" + std::to_string(m.L));
  std::vector<double> pre(static_cast<std::size_t>(U) + 1, 0.0);
  for (int u = 0; u < U; ++u) pre[static_cast<std::size_t>(u) + 1] = pre[static_cast<std::size_t>(u)] + m.unit_cost(u, avg_degree);
  const double inf = std::numeric_limits<double>::infinity();
  // best[p][u] = min over partitions of units [0,u) into p blocks of the max block cost
  std::vector<std::vector<double>> best(static_cast<std::size_t>(P) + 1, std::vector<double>(static_cast<std::size_t>(U) + 1, inf));
  std::vector<std::vector<int>> cut(static_cast<std::size_t>(P) + 1, std::vector<int>(static_cast<std::size_t>(U) + 1, -1));
  best[0][0] = 0.0;
  for (int p = 1; p <= P; ++p) {
    for (int u = p; u <= U; ++u) {
      for (int c = p - 1; c < u; ++c) {
        const double v = std::max(best[static_cast<std::size_t>(p) - 1][static_cast<std::size_t>(c)], pre[static_cast<std::size_t>(u)] - pre[static_cast<std::size_t>(c)]);
        if (v < best[static_cast<std::size_t>(p)][static_cast<std::size_t>(u)] * (1.0 - 1e-12)) {
          best[static_cast<std::size_t>(p)][static_cast<std::size_t>(u)] = v;
          cut[static_cast<std::size_t>(p)][static_cast<std::size_t>(u)] = c;
        }
      }
    }
  }
  StagePlan plan;
  plan.P = P;
  plan.blocks.resize(static_cast<std::size_t>(P));
  int u = U;
  for (int p = P; p >= 1; --p) {
    const int c = cut[static_cast<std::size_t>(p)][static_cast<std::size_t>(u)];
    plan.blocks[static_cast<std::size_t>(p) - 1] = {c, u};
    u = c;
  }
  return plan;
}

}  // namespace janus
