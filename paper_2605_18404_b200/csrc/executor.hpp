// executor.hpp — C++ entry points of executor.cpp used by the C ABI.
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "../../include/janus_cuda.h"

namespace janus {

janus_trainer* trainer_create(const janus_exec_desc& ed, const janus_stage_desc& sd, const float* all_params,
                              janus_comm* comm, int rank,
                              const char* schedule_text = nullptr);
void trainer_destroy(janus_trainer* t);
void trainer_load(janus_trainer* t, int mb, const janus_host_batch& hb);
void trainer_load_many(janus_trainer* t, int n, const int* mbs, const janus_host_batch* hbs);
void trainer_step(janus_trainer* t, const janus_opt& opt, janus_step_stats* stats);
void trainer_step_async(janus_trainer* t, const janus_opt& opt);
void trainer_wait(janus_trainer* t, janus_step_stats* stats);
void trainer_timeline(janus_trainer* t, double* out, int cap, int* n);
janus_stage* trainer_stage(janus_trainer* t, int block, int force_replica);
std::string trainer_schedule_text(janus_trainer* t);
void trainer_plan(janus_trainer* t, int32_t* out);

void nccl_unique_id(void* out);
janus_comm* comm_init_nccl(const void* id, int nranks, int rank, int device);
janus_comm* comm_init_ipc(const char* dir, int nranks, int rank, int device, bool same_process);
void comm_destroy(janus_comm* c);
void comm_send(janus_comm* c, const void* buf, size_t bytes, int peer, cudaStream_t s);
void comm_recv(janus_comm* c, void* buf, size_t bytes, int peer, cudaStream_t s);
void comm_group_start();
void comm_group_end();
void comm_allreduce_sum(janus_comm* c, float* buf, int64_t count, cudaStream_t s);

}  // namespace janus
