// stage_api.hpp — C++ entry points of stage.cu used by the C ABI and executor.
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "../../include/janus_cuda.h"
#include "geo_job.hpp"

namespace janus {

janus_stage* stage_create(const janus_stage_desc& d, const float* unit_params);
void stage_destroy(janus_stage* st);
struct DevCsrSlice;
// LM.  hb.row_ptr == nullptr: the neighbour list is built on the device
// (nbrlist.cu).  dcsr: col / shift / rev already on the device, as a slice of
// a batched build (hb.row_ptr is then the host mirror of this batch's row_ptr
// and hb.col/shift/rev are ignored).
// defer: queue the slice + geometry launch into `defer` (run by
// stage_geometry_flush as one batched kernel) instead of launching per batch.
// par: which of the micro-batch's two geometry copies to fill (< 0: the one
// the phases currently read; the trainer fills the other one beside a step).
void stage_load(janus_stage* st, int mb, const janus_host_batch& hb, cudaStream_t s, bool sync = true,
                const DevCsrSlice* dcsr = nullptr, std::vector<node::GeoJob>* defer = nullptr, int par = -1);
void stage_set_parity(janus_stage* st, int mb, int par);  // the copy the phases read from now on
struct DevGeo;
const DevGeo& stage_geo(const janus_stage* st, int mb, int par);
void stage_geometry_flush(janus_stage* st, std::vector<node::GeoJob>& jobs, cudaStream_t s);
void stage_fe(janus_stage* st, int mb, int slot, cudaStream_t s, int lane = 0);
void stage_ff(janus_stage* st, int mb, int slot, cudaStream_t s, int lane = 0);
void stage_bf(janus_stage* st, int mb, int slot, cudaStream_t s, int lane = 0);
void stage_be(janus_stage* st, int mb, int slot, cudaStream_t s, bool inj_only = false, int lane = 0);
void add_into(float* dst, const float* src, int64_t n, cudaStream_t s);
void stage_reduce_grads(janus_stage* st, cudaStream_t s);
// dhp: device {lr, beta1, beta2, eps} read by the Adam kernel at run time (the
// trainer's buffer, written before every step so replayed graphs see the
// current values); nullptr: o is copied into the stage's own buffer on s.
void stage_optimizer(janus_stage* st, const janus_opt& o, cudaStream_t s, const float* dhp = nullptr);
void stage_port(janus_stage* st, int mb, int slot, int port, void** dptr, size_t* bytes);

// read-back helpers (synchronous on the stream)
void stage_energy(janus_stage* st, int mb, float* E_host, float* loss_E, cudaStream_t s);
void stage_forces(janus_stage* st, int mb, float* F_host, float* loss_F, cudaStream_t s);
void stage_grads(janus_stage* st, int which, int mb, float* host_out, cudaStream_t s);
void stage_params(janus_stage* st, float* host_out, cudaStream_t s);
int64_t stage_param_count(const janus_stage* st);
void stage_grad_buffer(janus_stage* st, float** dptr, int64_t* count);
void stage_memory(const janus_stage* st, int64_t* static_bytes, int64_t* arena_bytes);
int stage_slot_of_mb(const janus_stage* st, int mb);
void stage_time_edge_kernel(janus_stage* st, int which, int mb, int slot, int iters, cudaStream_t s, float* avg_ms,
                            int64_t* edges, double* flops);

// tcgen05 layer self-test (tc_probe.cu)
void tc_probe(const int* args, const float* A, const float* B, float* D);
void gemm_tc_probe(int rows, int K, int N, int pair, const float* A, const float* W, float* D);

}  // namespace janus
