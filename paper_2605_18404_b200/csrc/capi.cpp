// capi.cpp — the extern "C" boundary (include/janus_cuda.h).  Every entry
// point catches C++ exceptions and maps them onto janus::Status codes
// (include/janus/errors.hpp) with a thread-local message; nothing throws
// across the ABI.
#include <cuda_runtime.h>

#include <cstring>
#include <new>
#include <string>

#include "../../include/janus/errors.hpp"
#include "../../include/janus/gars.hpp"
#include "../../include/janus/model.hpp"
#include "../../include/janus/render.hpp"
#include "../../include/janus/rendezvous.hpp"
#include "../../include/janus/schedule_gen.hpp"
#include "../../include/janus/tuner.hpp"

#include <cstdlib>
#include "../../include/janus_cuda.h"
#include "cuda_check.hpp"
#include "executor.hpp"
#include "host.hpp"
#include "nbrlist.hpp"
#include "stage_api.hpp"

namespace {

thread_local std::string g_last_error;

template <typename F>
int guard(F&& f) {
  try {
    f();
    g_last_error.clear();
    return janus::kOk;
  } catch (const janus::domain_error& e) {
    g_last_error = e.what();
    return janus::kDomainError;
  } catch (const janus::config_error& e) {
    g_last_error = e.what();
    return janus::kConfigError;
  } catch (const janus::parse_error& e) {
    g_last_error = e.what();
    return janus::kParseError;
  } catch (const janus::deadlock_error& e) {
    g_last_error = e.what();
    return janus::kDeadlockError;
  } catch (const janus::state_error& e) {
    g_last_error = e.what();
    return janus::kStateError;
  } catch (const janus::cuda_error& e) {
    g_last_error = e.what();
    return janus::kCudaError;
  } catch (const janus::nccl_error& e) {
    g_last_error = e.what();
    return janus::kNcclError;
  } catch (const std::bad_alloc&) {
    g_last_error = "out of host memory";
    return janus::kOutOfMemory;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return janus::kInternalError;
  } catch (...) {
    g_last_error = "unknown exception";
    return janus::kInternalError;
  }
}

cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

void need(const void* p, const char* what) {
  if (!p) throw janus::domain_error(std::string(what) + " is null");
}

void check_model(const janus_model_desc* m) {
  need(m, "model");
  if (m->L < 1 || m->H < 1 || m->R < 2 || m->n_species < 1) throw janus::config_error("bad model shape");
}

}  // namespace

extern "C" {

const char* janus_last_error(void) { return g_last_error.c_str(); }
int janus_abi_version(void) { return JANUS_ABI_VERSION; }

int janus_device_count(int* n) {
  return guard([&] {
    need(n, "n");
    const cudaError_t e = cudaGetDeviceCount(n);
    if (e != cudaSuccess) {
      *n = 0;
      cudaGetLastError();
    }
  });
}

int64_t janus_param_count(const janus_model_desc* m) {
  if (!m) return -1;
  return janus::host_unit_param_offset(*m, 2 * m->L + 2);
}
int64_t janus_unit_param_offset(const janus_model_desc* m, int unit) {
  if (!m || unit < 0 || unit > 2 * m->L + 2) return -1;
  return janus::host_unit_param_offset(*m, unit);
}
int janus_num_units(const janus_model_desc* m) { return m ? 2 * m->L + 2 : -1; }

int janus_synth_params(const janus_model_desc* m, uint64_t seed, float* out) {
  return guard([&] {
    check_model(m);
    need(out, "out");
    janus::synth_params(*m, seed, out);
  });
}

int janus_synth_cell(int32_t n_atoms, double rho, int32_t n_species, uint64_t seed, double* pos, int32_t* species,
                     double* cell, float* E_target, float* F_target) {
  return guard([&] {
    need(pos, "pos");
    need(species, "species");
    need(cell, "cell");
    need(E_target, "E_target");
    need(F_target, "F_target");
    *cell = janus::synth_cell(n_atoms, rho, n_species, seed, pos, species, E_target, F_target);
  });
}

int janus_nbrlist_build(int32_t n_atoms, const double* pos, const int32_t* struct_id, const double* cell, double r_c,
                        int32_t max_edges, int32_t* row_ptr, int32_t* col, int32_t* shift, int32_t* rev,
                        int32_t* n_edges) {
  return guard([&] {
    need(pos, "pos");
    need(struct_id, "struct_id");
    need(cell, "cell");
    need(row_ptr, "row_ptr");
    need(n_edges, "n_edges");
    if (n_atoms < 1) throw janus::domain_error("n_atoms must be >= 1");
    if (!(r_c > 0)) throw janus::domain_error("r_c must be > 0");
    *n_edges = janus::nbrlist_build(n_atoms, pos, struct_id, cell, r_c, max_edges, row_ptr, col, shift, rev);
  });
}

int janus_nbrlist_create(int32_t max_atoms, int32_t max_struct, int32_t max_edges, int32_t device,
                         janus_nbrlist** out) {
  return guard([&] {
    need(out, "out");
    *out = nullptr;
    *out = janus::nbrlist_create(max_atoms, max_struct, max_edges, device);
  });
}
int janus_nbrlist_destroy(janus_nbrlist* nl) {
  return guard([&] { janus::nbrlist_destroy(nl); });
}
int janus_nbrlist_build_device(janus_nbrlist* nl, int32_t n_atoms, int32_t n_struct, const double* pos,
                               const int32_t* struct_id, const double* cell, double r_c, int32_t* row_ptr,
                               int32_t* col, int32_t* shift, int32_t* rev, int32_t* n_edges, void* stream) {
  return guard([&] {
    need(nl, "nbrlist");
    need(pos, "pos");
    need(struct_id, "struct_id");
    need(cell, "cell");
    need(row_ptr, "row_ptr");
    need(col, "col");
    need(shift, "shift");
    need(rev, "rev");
    need(n_edges, "n_edges");
    janus::nbrlist_enqueue(nl, n_atoms, n_struct, pos, struct_id, cell, r_c, row_ptr, col, shift, rev, S(stream));
    *n_edges = janus::nbrlist_finish(nl, S(stream));
  });
}

int janus_plan_stages(const janus_model_desc* m, int32_t P, int32_t* unit_ranges) {
  return guard([&] {
    check_model(m);
    need(unit_ranges, "unit_ranges");
    janus::ModelConfig mc;
    mc.L = m->L;
    mc.H = m->H;
    mc.R = m->R;
    mc.n_species = m->n_species;
    mc.r_c = m->r_c;
    const janus::StagePlan plan = janus::partition_units(mc, P);
    for (int b = 0; b < P; ++b) {
      unit_ranges[2 * b] = plan.blocks[static_cast<size_t>(b)].first;
      unit_ranges[2 * b + 1] = plan.blocks[static_cast<size_t>(b)].second;
    }
  });
}

// ------------------------------------------------------------------ stages
int janus_stage_create(const janus_stage_desc* desc, const float* unit_params, janus_stage** out) {
  return guard([&] {
    need(desc, "desc");
    need(unit_params, "unit_params");
    need(out, "out");
    *out = nullptr;
    *out = janus::stage_create(*desc, unit_params);
  });
}
int janus_stage_destroy(janus_stage* st) {
  return guard([&] { janus::stage_destroy(st); });
}
int janus_stage_load(janus_stage* st, int mb, const janus_host_batch* hb, void* stream) {
  return guard([&] {
    need(st, "stage");
    need(hb, "batch");
    janus::stage_load(st, mb, *hb, S(stream));
  });
}
int janus_stage_fe(janus_stage* st, int mb, int slot, void* stream) {
  return guard([&] { need(st, "stage"); janus::stage_fe(st, mb, slot, S(stream)); });
}
int janus_stage_ff(janus_stage* st, int mb, int slot, void* stream) {
  return guard([&] { need(st, "stage"); janus::stage_ff(st, mb, slot, S(stream)); });
}
int janus_stage_bf(janus_stage* st, int mb, int slot, void* stream) {
  return guard([&] { need(st, "stage"); janus::stage_bf(st, mb, slot, S(stream)); });
}
int janus_stage_be(janus_stage* st, int mb, int slot, void* stream) {
  return guard([&] { need(st, "stage"); janus::stage_be(st, mb, slot, S(stream)); });
}
int janus_stage_port(janus_stage* st, int mb, int slot, int port, void** dptr, size_t* bytes) {
  return guard([&] {
    need(st, "stage");
    need(dptr, "dptr");
    need(bytes, "bytes");
    janus::stage_port(st, mb, slot, port, dptr, bytes);
  });
}
int janus_stage_energy(janus_stage* st, int mb, float* E_host, float* loss_E_host, void* stream) {
  return guard([&] { need(st, "stage"); janus::stage_energy(st, mb, E_host, loss_E_host, S(stream)); });
}
int janus_stage_forces(janus_stage* st, int mb, float* F_host, float* loss_F_host, void* stream) {
  return guard([&] { need(st, "stage"); janus::stage_forces(st, mb, F_host, loss_F_host, S(stream)); });
}
int janus_stage_grads(janus_stage* st, int which, int mb, float* host_out, void* stream) {
  return guard([&] {
    need(st, "stage");
    need(host_out, "host_out");
    janus::stage_grads(st, which, mb, host_out, S(stream));
  });
}
int janus_stage_params(janus_stage* st, float* host_out, void* stream) {
  return guard([&] {
    need(st, "stage");
    need(host_out, "host_out");
    janus::stage_params(st, host_out, S(stream));
  });
}
int64_t janus_stage_param_count(janus_stage* st) { return st ? janus::stage_param_count(st) : -1; }
int janus_stage_reduce_grads(janus_stage* st, void* stream) {
  return guard([&] { need(st, "stage"); janus::stage_reduce_grads(st, S(stream)); });
}
int janus_stage_grad_buffer(janus_stage* st, float** dptr, int64_t* count) {
  return guard([&] {
    need(st, "stage");
    need(dptr, "dptr");
    need(count, "count");
    janus::stage_grad_buffer(st, dptr, count);
  });
}
int janus_stage_optimizer_step(janus_stage* st, const janus_opt* opt, void* stream) {
  return guard([&] {
    need(st, "stage");
    need(opt, "opt");
    janus::stage_optimizer(st, *opt, S(stream));
  });
}
int janus_stage_time_edge_kernel(janus_stage* st, int which, int mb, int slot, int iters, void* stream,
                                 float* avg_ms, int64_t* edges, double* flops) {
  return guard([&] {
    need(st, "stage");
    need(avg_ms, "avg_ms");
    need(edges, "edges");
    need(flops, "flops");
    janus::stage_time_edge_kernel(st, which, mb, slot, iters, S(stream), avg_ms, edges, flops);
  });
}
int janus_stage_memory(janus_stage* st, int64_t* static_bytes, int64_t* arena_bytes) {
  return guard([&] { need(st, "stage"); janus::stage_memory(st, static_bytes, arena_bytes); });
}

// -------------------------------------------------------------- transports
int janus_nccl_unique_id(void* id_out) {
  return guard([&] {
    need(id_out, "id_out");
    janus::nccl_unique_id(id_out);
  });
}
int janus_comm_init_nccl(const void* id, int nranks, int rank, int device, janus_comm** out) {
  return guard([&] {
    need(id, "id");
    need(out, "out");
    *out = nullptr;
    if (nranks < 1 || rank < 0 || rank >= nranks) throw janus::domain_error("bad rank / nranks");
    *out = janus::comm_init_nccl(id, nranks, rank, device);
  });
}
int janus_comm_init_ipc(const char* dir, int nranks, int rank, int device, janus_comm** out) {
  return guard([&] {
    need(out, "out");
    *out = janus::comm_init_ipc(dir, nranks, rank, device, false);
  });
}
int janus_comm_init_threads(const char* dir, int nranks, int rank, int device, janus_comm** out) {
  return guard([&] {
    need(out, "out");
    *out = janus::comm_init_ipc(dir, nranks, rank, device, true);
  });
}
int janus_comm_destroy(janus_comm* c) {
  return guard([&] { janus::comm_destroy(c); });
}
int janus_comm_send(janus_comm* c, const void* buf, size_t bytes, int peer, void* stream) {
  return guard([&] { need(c, "comm"); janus::comm_send(c, buf, bytes, peer, S(stream)); });
}
int janus_comm_recv(janus_comm* c, void* buf, size_t bytes, int peer, void* stream) {
  return guard([&] { need(c, "comm"); janus::comm_recv(c, buf, bytes, peer, S(stream)); });
}
int janus_comm_group_start(void) {
  return guard([&] { janus::comm_group_start(); });
}
int janus_comm_group_end(void) {
  return guard([&] { janus::comm_group_end(); });
}
int janus_comm_allreduce_sum(janus_comm* c, float* buf, int64_t count, void* stream) {
  return guard([&] { need(c, "comm"); janus::comm_allreduce_sum(c, buf, count, S(stream)); });
}

// ---------------------------------------------------------------- trainer
int janus_trainer_create(const janus_exec_desc* ed, const janus_stage_desc* sd, const float* all_params,
                         janus_comm* comm, int rank, janus_trainer** out) {
  return guard([&] {
    need(ed, "exec desc");
    need(sd, "stage desc");
    need(all_params, "all_params");
    need(out, "out");
    *out = nullptr;
    *out = janus::trainer_create(*ed, *sd, all_params, comm, rank);
  });
}
int janus_trainer_create_from_text(const janus_exec_desc* ed, const janus_stage_desc* sd, const float* all_params,
                                   const char* schedule_text, janus_comm* comm, int rank, janus_trainer** out) {
  return guard([&] {
    need(ed, "exec desc");
    need(sd, "stage desc");
    need(all_params, "all_params");
    need(schedule_text, "schedule text");
    need(out, "out");
    *out = nullptr;
    *out = janus::trainer_create(*ed, *sd, all_params, comm, rank, schedule_text);
  });
}
int janus_trainer_destroy(janus_trainer* t) {
  return guard([&] { janus::trainer_destroy(t); });
}
int janus_trainer_load(janus_trainer* t, int mb, const janus_host_batch* hb) {
  return guard([&] {
    need(t, "trainer");
    need(hb, "batch");
    janus::trainer_load(t, mb, *hb);
  });
}
int janus_trainer_load_many(janus_trainer* t, int n, const int32_t* mbs, const janus_host_batch* hbs) {
  return guard([&] {
    need(t, "trainer");
    if (n < 0) throw janus::domain_error("n must be >= 0");
    if (n > 0) {
      need(mbs, "mbs");
      need(hbs, "hbs");
      janus::trainer_load_many(t, n, mbs, hbs);
    }
  });
}
int janus_trainer_step(janus_trainer* t, const janus_opt* opt, janus_step_stats* stats) {
  return guard([&] {
    need(t, "trainer");
    need(opt, "opt");
    janus::trainer_step(t, *opt, stats);
  });
}
int janus_trainer_step_async(janus_trainer* t, const janus_opt* opt) {
  return guard([&] {
    need(t, "trainer");
    need(opt, "opt");
    janus::trainer_step_async(t, *opt);
  });
}
int janus_trainer_wait(janus_trainer* t, janus_step_stats* stats) {
  return guard([&] {
    need(t, "trainer");
    janus::trainer_wait(t, stats);
  });
}
int janus_trainer_timeline(janus_trainer* t, double* out, int32_t cap, int32_t* n) {
  return guard([&] {
    need(t, "trainer");
    need(n, "n");
    int nn = 0;
    janus::trainer_timeline(t, out, out ? cap : 0, &nn);
    *n = nn;
  });
}
int janus_trainer_stage(janus_trainer* t, int block, int force_replica, janus_stage** out) {
  return guard([&] {
    need(t, "trainer");
    need(out, "out");
    *out = janus::trainer_stage(t, block, force_replica);
  });
}
int janus_trainer_schedule_text(janus_trainer* t, char* buf, int64_t cap, int64_t* len) {
  return guard([&] {
    need(t, "trainer");
    need(len, "len");
    const std::string text = janus::trainer_schedule_text(t);
    *len = static_cast<int64_t>(text.size());
    if (buf && cap > 0) {
      const size_t n = std::min<size_t>(text.size(), static_cast<size_t>(cap - 1));
      std::memcpy(buf, text.data(), n);
      buf[n] = '\0';
    }
  });
}
int janus_trainer_plan(janus_trainer* t, int32_t* unit_ranges) {
  return guard([&] {
    need(t, "trainer");
    need(unit_ranges, "unit_ranges");
    janus::trainer_plan(t, unit_ranges);
  });
}

// ------------------------------------------------------------ diagnostics
int janus_gemm_tc_probe(int32_t rows, int32_t K, int32_t N, int32_t pair, const float* A, const float* W, float* D) {
  return guard([&] {
    need(A, "A");
    need(W, "W");
    need(D, "D");
    janus::gemm_tc_probe(rows, K, N, pair, A, W, D);
  });
}
int janus_tc_probe(const int32_t* args, const float* A, const float* B, float* D) {
  return guard([&] {
    need(args, "args");
    need(A, "A");
    need(B, "B");
    need(D, "D");
    janus::tc_probe(args, A, B, D);
  });
}

// --------------------------------------------------------------- schedules
int janus_schedule_generate(int method, int P, int n_mb, int k, char* buf, int64_t cap, int64_t* len) {
  return guard([&] {
    need(len, "len");
    janus::Schedule s;
    switch (method) {
      case 0: s = janus::symfold(P, n_mb); break;
      case 1: s = janus::wavek(P, n_mb, k); break;
      case 2: s = janus::onef1b_2nd(P, n_mb); break;
      case 3: s = janus::gen_first_order(P, n_mb); break;
      case 4: s = janus::hanayo_2nd(P, n_mb); break;
      default: throw janus::domain_error("unknown schedule method");
    }
    const std::string text = janus::serialize(s);
    *len = static_cast<int64_t>(text.size());
    if (buf && cap > 0) {
      const size_t n = std::min<size_t>(text.size(), static_cast<size_t>(cap - 1));
      std::memcpy(buf, text.data(), n);
      buf[n] = '\0';
    }
  });
}

int janus_schedule_validate(const char* text, int32_t* n_errors) {
  return guard([&] {
    need(text, "text");
    need(n_errors, "n_errors");
    const janus::ValidationReport r = janus::validate_schedule(janus::deserialize(text));
    *n_errors = static_cast<int32_t>(r.total_errors());
  });
}

int janus_schedule_replay(const char* text, const double* t, double* makespan, double* bubble_ratio) {
  return guard([&] {
    need(text, "text");
    need(t, "t");
    need(makespan, "makespan");
    need(bubble_ratio, "bubble_ratio");
    const janus::Schedule s = janus::deserialize(text);
    const janus::DepGraph g = janus::build_dependencies(s);
    janus::PhaseTimes pt;
    pt.t_FE = t[0];
    pt.t_FF = t[1];
    pt.t_BE = t[2];
    pt.t_BF = t[3];
    const std::vector<double> d = janus::phase_durations(g, pt);
    const janus::ReplayResult r = janus::replay(g, d);
    if (!r.ok) throw janus::deadlock_error("replay: " + r.blocked);
    const janus::BubbleReport b = janus::bubble_of(g, r, d);
    *makespan = r.makespan;
    *bubble_ratio = b.bubble_ratio;
  });
}

int janus_schedule_check_rendezvous(const char* text, int32_t onef1b, int32_t lanes, int32_t dp, int32_t layout,
                                    int32_t* ok, int64_t* completed, int64_t* total, char* stuck, int64_t cap) {
  return guard([&] {
    need(text, "text");
    need(ok, "ok");
    if (lanes < 1 || dp < 1 || layout < 0 || layout > 1) throw janus::domain_error("bad lanes / dp / layout");
    const janus::Schedule s = janus::deserialize(text);
    const int P = static_cast<int>(s.stage_map.size()) / 2;
    if (P < 1 || s.num_devices() != P) throw janus::domain_error("rendezvous check needs a P-device, 2P-virtual-stage schedule");
    const auto progs = janus::build_programs(s, P, onef1b != 0, lanes, dp,
                                             layout == 0 ? janus::StreamLayout::kPerChannel : janus::StreamLayout::kSharedPair);
    const janus::RendezvousReport r = janus::simulate(progs, P, s, onef1b != 0);
    *ok = r.ok ? 1 : 0;
    if (completed) *completed = r.completed;
    if (total) *total = r.ops;
    if (stuck && cap > 0) {
      const size_t n = std::min(static_cast<size_t>(cap - 1), r.stuck.size());
      std::memcpy(stuck, r.stuck.data(), n);
      stuck[n] = 0;
    }
  });
}

int janus_schedule_slot_pool(const char* text, int32_t onef1b, int32_t local, int32_t unfolded, int32_t lanes,
                             int32_t* slots, int32_t cap, int32_t* n_devices) {
  return guard([&] {
    need(text, "text");
    need(slots, "slots");
    const janus::Schedule s = janus::deserialize(text);
    const int P = static_cast<int>(s.stage_map.size()) / 2;
    if (P < 1) throw janus::domain_error("slot pool needs a 2P-virtual-stage schedule");
    int n_mb = 0;
    for (const auto& dl : s.device_lists)
      for (const auto& in : dl) n_mb = std::max(n_mb, in.micro_batch + 1);
    const std::vector<int> v = janus::slot_pool_sizes(s, P, onef1b != 0, local != 0, unfolded != 0, n_mb, std::max(1, lanes));
    if (n_devices) *n_devices = static_cast<int32_t>(v.size());
    for (size_t d = 0; d < v.size() && static_cast<int32_t>(d) < cap; ++d) slots[d] = v[d];
  });
}

// ------------------------------------------------------------------ GARS
namespace {
std::vector<janus::gars::AtomGraph> graphs_of(const int32_t* atoms, int32_t M) {
  need(atoms, "atoms");
  if (M < 1) throw janus::domain_error("GARS: empty batch");
  std::vector<janus::gars::AtomGraph> g(static_cast<size_t>(M));
  for (int32_t i = 0; i < M; ++i) g[static_cast<size_t>(i)] = janus::gars::AtomGraph{i, atoms[i], 0};
  return g;
}
void write_packing(const std::vector<janus::gars::PackedMicroBatch>& mbs, int d_gp, int32_t* order, int32_t* mb_ptr,
                   int32_t* tags) {
  need(order, "order");
  need(mb_ptr, "mb_ptr");
  int32_t k = 0;
  mb_ptr[0] = 0;
  for (size_t j = 0; j < mbs.size(); ++j) {
    for (const auto& g : mbs[j].graphs) order[k++] = static_cast<int32_t>(g.id);
    mb_ptr[j + 1] = k;
    if (tags) tags[j] = static_cast<int32_t>(mbs[j].graphs.empty() ? janus::gars::MbTag::comm_free
                                                                    : janus::gars::tag_of(mbs[j].graphs, d_gp));
  }
}
}  // namespace

int janus_gars_pack(const int32_t* atoms, int32_t M, int32_t n_mb, int32_t d_gp, uint64_t seed, int32_t* order,
                    int32_t* mb_ptr, int32_t* tags) {
  return guard([&] {
    const auto mbs = janus::gars::pack_and_shuffle(graphs_of(atoms, M), n_mb, d_gp, seed);
    write_packing(mbs, d_gp, order, mb_ptr, tags);
  });
}
int janus_gars_greedy(const int32_t* atoms, int32_t M, int32_t n_mb, int32_t d_gp, int32_t* order,
                      int32_t* mb_ptr, int32_t* tags) {
  return guard([&] {
    if (d_gp < 1) throw janus::domain_error("d_gp must be >= 1");
    const auto mbs = janus::gars::greedy_sequential(graphs_of(atoms, M), n_mb);
    write_packing(mbs, d_gp, order, mb_ptr, tags);
  });
}
int janus_gars_assign_bins(const int32_t* atoms, int32_t n, int32_t d_gp, int32_t* bin_of) {
  return guard([&] {
    need(bin_of, "bin_of");
    janus::gars::PackedMicroBatch mb;
    mb.graphs = graphs_of(atoms, n);
    mb.tag = janus::gars::tag_of(mb.graphs, d_gp);
    const auto r = janus::gars::assign_gp_bins(mb, d_gp);
    for (size_t b = 0; b < r.gp_bins.size(); ++b)
      for (auto id : r.gp_bins[b]) bin_of[id] = static_cast<int32_t>(b);
  });
}
int janus_gars_synth_sizes(const double* stats, int32_t n, uint64_t seed, int32_t* atoms, int64_t* edges) {
  return guard([&] {
    need(atoms, "atoms");
    janus::gars::SizeStats s = janus::gars::mixed_preset();
    if (stats) s = janus::gars::SizeStats{stats[0], stats[1], stats[2], stats[3], stats[4]};
    const auto g = janus::gars::synth_dataset(s, n, seed);
    for (int32_t i = 0; i < n; ++i) {
      atoms[i] = g[static_cast<size_t>(i)].atoms;
      if (edges) edges[i] = g[static_cast<size_t>(i)].edges;
    }
  });
}

// ------------------------------------------------------------------ tuner
int janus_tune_wavek(int32_t P, int32_t n_mb, const double* t, const double* mem, int32_t divisors_only,
                     int32_t* k_star, int32_t* tuned, double* table, int32_t cap, int32_t* n) {
  return guard([&] {
    need(t, "t");
    need(mem, "mem");
    need(k_star, "k_star");
    need(n, "n");
    janus::PhaseTimes pt{t[0], t[1], t[2], t[3]};
    janus::tuner::MemoryParams mp;
    mp.m_gpu = mem[0];
    mp.m_reserve = mem[1];
    mp.static_bytes = {mem[2]};
    mp.fe_bytes = mem[3];
    mp.ff_bytes = mem[4];
    mp.stage0_mult = mem[5];
    const janus::tuner::TuneResult r = janus::tuner::tune(P, n_mb, pt, mp, divisors_only != 0);
    *k_star = r.k_star;
    if (tuned) *tuned = r.tuned ? 1 : 0;
    *n = static_cast<int32_t>(r.table.size());
    if (table)
      for (int32_t i = 0; i < std::min(cap, *n); ++i) {
        const auto& c = r.table[static_cast<size_t>(i)];
        table[5 * i + 0] = c.k;
        table[5 * i + 1] = c.makespan;
        table[5 * i + 2] = c.bubble_ratio;
        table[5 * i + 3] = c.peak_max;
        table[5 * i + 4] = c.feasible ? 1.0 : 0.0;
      }
  });
}

// ------------------------------------------------------------------ render
int janus_render_timeline(const double* recs, int32_t n, const char* text, const double* t, int32_t fmt,
                          double quantum, char* buf, int64_t cap, int64_t* len) {
  return guard([&] {
    need(len, "len");
    std::vector<janus::render::Span> spans;
    if (text) {
      need(t, "t");
      const janus::Schedule s = janus::deserialize(text);
      const janus::DepGraph g = janus::build_dependencies(s);
      const janus::PhaseTimes pt{t[0], t[1], t[2], t[3]};
      const janus::ReplayResult r = janus::replay(g, janus::phase_durations(g, pt));
      if (!r.ok) throw janus::deadlock_error("render: replay stalled: " + r.blocked);
      spans = janus::render::spans_of(g, r);
    } else {
      if (n > 0) need(recs, "recs");
      for (int32_t i = 0; i < n; ++i)
        spans.push_back(janus::render::Span{static_cast<int>(recs[5 * i]), static_cast<int>(recs[5 * i + 1]),
                                            static_cast<int>(recs[5 * i + 2]), recs[5 * i + 3], recs[5 * i + 4]});
    }
    const std::string out = fmt == 1 ? janus::render::svg(spans, quantum) : janus::render::ascii(spans, quantum);
    *len = static_cast<int64_t>(out.size());
    if (buf && cap > 0) {
      const size_t k = std::min<size_t>(out.size(), static_cast<size_t>(cap - 1));
      std::memcpy(buf, out.data(), k);
      buf[k] = '\0';
    }
  });
}

int janus_schedule_memory(const char* text, const double* t, const double* static_bytes, int32_t n_static,
                          const double* act, double* peaks, int32_t cap, int32_t* n_devices) {
  return guard([&] {
    need(text, "text");
    need(t, "t");
    need(static_bytes, "static_bytes");
    need(act, "act");
    need(n_devices, "n_devices");
    const janus::Schedule s = janus::deserialize(text);
    const janus::DepGraph g = janus::build_dependencies(s);
    const janus::PhaseTimes pt{t[0], t[1], t[2], t[3]};
    const janus::ReplayResult r = janus::replay(g, janus::phase_durations(g, pt));
    if (!r.ok) throw janus::deadlock_error("memory: replay stalled: " + r.blocked);
    janus::tuner::MemoryParams mp;
    if (n_static < 1) throw janus::domain_error("n_static must be >= 1");
    mp.static_bytes.assign(static_bytes, static_bytes + n_static);
    if (n_static != 1 && n_static != s.num_devices()) throw janus::domain_error("static_bytes: 1 or one per device");
    mp.fe_bytes = act[0];
    mp.ff_bytes = act[1];
    mp.stage0_mult = act[2];
    mp.replicate_static = act[3] != 0.0;
    const std::vector<double> p = janus::tuner::peak_memory(g, r, mp);
    *n_devices = static_cast<int32_t>(p.size());
    if (peaks)
      for (int32_t i = 0; i < std::min<int32_t>(cap, *n_devices); ++i) peaks[i] = p[static_cast<size_t>(i)];
  });
}

}  // extern "C"
