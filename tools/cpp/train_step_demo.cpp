// A C++ host program against the drop-in boundary alone (no Python, no
// PyTorch): build a schedule with the reference-API generators, synthesise
// micro-batches, and run janus::train_step (include/janus/train.hpp) on the
// GPU.  Prints one JSON line per step.  Built and run by
// tests/test_gpu_cpp_api.py:
//   g++ -std=c++20 -O2 -Iinclude -I/usr/local/cuda/include tools/cpp/train_step_demo.cpp
//       -Lpaper_2605_18404_b200 -ljanus_b200 -Wl,-rpath,$PWD/paper_2605_18404_b200 -o train_step_demo
//   ./train_step_demo <P> <method: symfold|wavek|onef1b|hanayo> <n_mb> <steps> <precision: tf32|fp32>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "janus/schedule_gen.hpp"
#include "janus/train.hpp"

int main(int argc, char** argv) {
  const int P = argc > 1 ? std::atoi(argv[1]) : 2;
  const std::string method = argc > 2 ? argv[2] : "symfold";
  const int n_mb = argc > 3 ? std::atoi(argv[3]) : 4;
  const int steps = argc > 4 ? std::atoi(argv[4]) : 2;
  const std::string prec = argc > 5 ? argv[5] : "tf32";
  try {
    janus::ModelConfig mc;  // L=4, H=64, R=64, r_c=5 (configs[0/1])
    mc.L = 2;
    const janus::StagePlan plan = janus::partition_units(mc, P);
    janus::Schedule s = method == "wavek"    ? janus::wavek(P, n_mb, std::min(n_mb, 2 * P))
                        : method == "onef1b" ? janus::onef1b_2nd(P, n_mb)
                        : method == "hanayo" ? janus::hanayo_2nd(P, n_mb)
                                             : janus::symfold(P, n_mb);
    // parameters and cells from the library's seeded synthesiser (SplitMix64)
    janus_model_desc md{mc.L, mc.H, mc.R, mc.n_species, 5.f, 1.f, 10.f, prec == "fp32" ? JANUS_PREC_FP32 : JANUS_PREC_TF32};
    std::vector<float> params(static_cast<size_t>(janus_param_count(&md)));
    janus::check_status(janus_synth_params(&md, 7, params.data()), janus_last_error());
    janus::MicroBatches mbs(static_cast<size_t>(n_mb));
    for (int m = 0; m < n_mb; ++m) {
      const int n = 32 + 4 * (m % 3);
      auto& b = mbs[static_cast<size_t>(m)];
      b.pos.resize(3 * static_cast<size_t>(n));
      b.species.resize(static_cast<size_t>(n));
      b.struct_id.assign(static_cast<size_t>(n), 0);
      b.cell.resize(1);
      b.E_target.resize(1);
      b.F_target.resize(3 * static_cast<size_t>(n));
      janus::check_status(janus_synth_cell(n, 0.095, mc.n_species, (100 + static_cast<uint64_t>(m)) * 1000003ULL, b.pos.data(),
                                           b.species.data(), b.cell.data(), b.E_target.data(), b.F_target.data()),
                          janus_last_error());  // row_ptr empty: the neighbour list is built on the GPU
    }
    janus::TrainState::Options o;
    o.precision = md.precision;
    o.max_atoms = 64;
    o.max_edges = 64 * 120;
    o.max_struct = 1;
    janus::TrainState st(params, o);
    for (int k = 0; k < steps; ++k) {
      const janus::StepReport r = janus::train_step(mc, plan, s, mbs, st);
      std::printf("{\"step\": %d, \"loss\": %.17g, \"makespan_ms\": %.4f, \"p2p_bytes\": %lld, \"act_slots0\": %d}\n", k, r.loss,
                  r.makespan_ms, static_cast<long long>(r.p2p_bytes), r.act_slots.empty() ? 0 : r.act_slots[0]);
    }
    const std::vector<float> p0 = st.block_params(0);
    double sum = 0;
    for (float x : p0) sum += x;
    std::printf("{\"block0_param_sum\": %.17g, \"block0_params\": %zu}\n", sum, p0.size());
  } catch (const std::exception& ex) {
    std::fprintf(stderr, "train_step_demo: %s\n", ex.what());
    return 1;
  }
  return 0;
}
