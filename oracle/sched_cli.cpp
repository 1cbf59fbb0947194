// oracle/sched_cli.cpp — TEST INFRASTRUCTURE (schedule checker), not product.
//
// One source, compiled twice by oracle/Makefile:
//   * against the reference headers in /root/reference/proj/include
//     -> oracle/_ref/sched_ref   (the compiled reference: the schedule oracle)
//   * against this repo's include/janus -> oracle/_ref/sched_mine
// Every mode below only uses API the reference ships (ir/graph/transform), so
// both binaries run the same code; tests/test_schedule_golden.py diffs them
// and freezes the reference outputs under tests/golden/.
// Generator modes (first/symfold/onef1b/wavek) exist only in the repo build
// (-DJANUS_HAVE_GENERATORS) because the reference has no generators.
//
// Usage:
//   sched_cli passes <file> fold|lin        Pass1+2+3 on a first-order text
//   sched_cli roundtrip <file>              deserialize+serialize
//   sched_cli replay <file> tFE tFF tBE tBF  replay + longest path (%.17g)
//   sched_cli topo <file> slot|mbmajor      priority_topo_order with a key
//   sched_cli deps <file>                   sorted predecessor lists
//   sched_cli first|symfold|onef1b P N      (repo build only)
//   sched_cli wavek P N k                   (repo build only)
#include <algorithm>  // must precede janus/ir.hpp for the reference build (ir.hpp:355)
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <tuple>
#include <vector>

#include "janus/graph.hpp"
#include "janus/ir.hpp"
#include "janus/transform.hpp"
#ifdef JANUS_HAVE_GENERATORS
#include "janus/schedule_gen.hpp"
#endif

namespace {

std::string slurp(const char* path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error(std::string("cannot open ") + path);
  std::ostringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

int usage() {
  std::fprintf(stderr, "usage: sched_cli passes|roundtrip|replay|topo|deps|first|symfold|onef1b|wavek ...\n");
  return 2;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 3) return usage();
  const std::string mode = argv[1];
  try {
    if (mode == "passes" && argc == 4) {
      const janus::Schedule first = janus::deserialize(slurp(argv[2]));
      const int P = first.pipeline_degree;
      std::vector<int> map(static_cast<std::size_t>(2 * P));
      const bool lin = std::string(argv[3]) == "lin";
      for (int v = 0; v < 2 * P; ++v) map[static_cast<std::size_t>(v)] = lin ? v / 2 : janus::fold_map(v, P);
      const auto pr = janus::transform::prune_intra_device(
          janus::transform::fold_with_map(janus::transform::remap_second_order(first), map));
      std::cout << "# pruned " << pr.second << "\n" << janus::serialize(pr.first);
      return 0;
    }
    if (mode == "roundtrip" && argc == 3) {
      std::cout << janus::serialize(janus::deserialize(slurp(argv[2])));
      return 0;
    }
    if (mode == "replay" && argc == 7) {
      const janus::Schedule s = janus::deserialize(slurp(argv[2]));
      const double t[4] = {std::stod(argv[3]), std::stod(argv[4]), std::stod(argv[5]), std::stod(argv[6])};
      const janus::DepGraph g = janus::build_dependencies(s);
      std::vector<double> d(static_cast<std::size_t>(g.size()), 0.0);
      for (int i = 0; i < g.size(); ++i) {
        const auto k = g.flat[static_cast<std::size_t>(i)]->kind;
        if (janus::is_compute(k)) d[static_cast<std::size_t>(i)] = t[static_cast<int>(janus::phase_of(k))];
      }
      const janus::ReplayResult r = janus::replay(g, d);
      std::printf("ok %d makespan %.17g", r.ok ? 1 : 0, r.makespan);
      if (r.ok) std::printf(" oracle %.17g", janus::longest_path_makespan(g, d));
      std::printf("\n");
      if (r.ok) {
        for (int i = 0; i < g.size(); ++i) std::printf("%d %.17g %.17g\n", i, r.start[static_cast<std::size_t>(i)], r.end[static_cast<std::size_t>(i)]);
      } else {
        std::printf("blocked %s\n", r.blocked.c_str());
      }
      return 0;
    }
    if (mode == "topo" && argc == 4) {
      const janus::Schedule s = janus::deserialize(slurp(argv[2]));
      const std::string key = argv[3];
      const int P = s.pipeline_degree;
      janus::Schedule out;
      if (key == "mbmajor") {
        out = janus::transform::priority_topo_order(s, [](const janus::Instruction& i) {
          return std::make_tuple(i.micro_batch, i.virtual_stage, static_cast<int>(i.kind));
        });
      } else {
        // slot key: forward work of mb m at stage v precedes backward work
        out = janus::transform::priority_topo_order(s, [P](const janus::Instruction& i) {
          const int v = i.virtual_stage < 0 ? 0 : i.virtual_stage;
          const int pos = janus::is_forward_flow(i.kind) ? v : 4 * P - v;
          return std::make_tuple(i.micro_batch + pos, static_cast<int>(i.kind), i.micro_batch);
        });
      }
      std::cout << janus::serialize(out);
      return 0;
    }
    if (mode == "deps" && argc == 3) {
      const janus::Schedule s = janus::deserialize(slurp(argv[2]));
      const janus::DepGraph g = janus::build_dependencies(s);
      for (int i = 0; i < g.size(); ++i) {
        std::vector<int> p = g.preds[static_cast<std::size_t>(i)];
        std::sort(p.begin(), p.end());
        p.erase(std::unique(p.begin(), p.end()), p.end());
        std::printf("%d%s:", i, g.unsatisfiable[static_cast<std::size_t>(i)] ? "!" : "");
        for (int x : p) std::printf(" %d", x);
        std::printf("\n");
      }
      return 0;
    }
#ifdef JANUS_HAVE_GENERATORS
    if ((mode == "first" || mode == "symfold" || mode == "onef1b") && argc == 4) {
      const int P = std::stoi(argv[2]), N = std::stoi(argv[3]);
      if (mode == "first") std::cout << janus::serialize(janus::gen_first_order(P, N));
      if (mode == "symfold") std::cout << janus::serialize(janus::symfold(P, N));
      if (mode == "onef1b") std::cout << janus::serialize(janus::onef1b_2nd(P, N));
      return 0;
    }
    if (mode == "wavek" && argc == 5) {
      std::cout << janus::serialize(janus::wavek(std::stoi(argv[2]), std::stoi(argv[3]), std::stoi(argv[4])));
      return 0;
    }
    if (mode == "validate" && argc == 3) {
      const janus::ValidationReport r = janus::validate_schedule(janus::deserialize(slurp(argv[2])));
      std::printf("ok %d coverage %zu matching %zu dependency %zu ledger %zu\n", r.ok() ? 1 : 0, r.coverage_errors.size(),
                  r.matching_errors.size(), r.dependency_errors.size(), r.gradient_ledger_errors.size());
      for (const auto* v : {&r.coverage_errors, &r.matching_errors, &r.dependency_errors, &r.gradient_ledger_errors})
        for (std::size_t i = 0; i < v->size() && i < 5; ++i) std::printf("  D%d seq %d: %s\n", (*v)[i].device, (*v)[i].seq, (*v)[i].description.c_str());
      return r.ok() ? 0 : 1;
    }
    if (mode == "compare" && argc == 5) {
      // compare P N preset: makespan / bubble of 1F1B-2nd, SymFold, WaveK(k)
      const int P = std::stoi(argv[2]), N = std::stoi(argv[3]);
      const janus::PhaseTimes t = janus::preset_phase_times(argv[4]);
      auto report = [&](const char* name, const janus::Schedule& s) {
        const janus::DepGraph g = janus::build_dependencies(s);
        const auto d = janus::phase_durations(g, t);
        const auto r = janus::replay(g, d);
        const auto b = janus::bubble_of(g, r, d);
        std::printf("%-14s makespan %10.2f bubble %.4f valid %d\n", name, r.makespan, b.bubble_ratio,
                    janus::validate_schedule(s).ok() ? 1 : 0);
        return r.makespan;
      };
      if (P % 2 == 0) report("onef1b_2nd", janus::onef1b_2nd(P, N));
      report("symfold", janus::symfold(P, N));
      for (int k = 1; k <= N; ++k) {
        janus::WaveKOptions o;
        o.times = t;
        if (const char* pol = std::getenv("WAVEK_POLICY")) o.policy = std::atoi(pol);
        if (const char* la = std::getenv("WAVEK_LOOKAHEAD")) o.lookahead_units = std::atoi(la);
        char name[32];
        std::snprintf(name, sizeof name, "wavek k=%d", k);
        report(name, janus::wavek(P, N, k, o));
      }
      return 0;
    }
#endif
  } catch (const janus::parse_error& e) {
    std::printf("parse_error line %d: %s\n", e.line, e.what());
    return 3;
  } catch (const std::exception& e) {
    std::printf("error: %s\n", e.what());
    return 1;
  }
  return usage();
}
