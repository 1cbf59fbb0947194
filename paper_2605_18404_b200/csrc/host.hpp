// host.hpp — host-side data preparation (synthetic inputs, neighbour list).
#pragma once

#include <cstdint>

#include "../../include/janus_cuda.h"

namespace janus {

int64_t host_unit_param_count(const janus_model_desc& m, int u);
int64_t host_unit_param_offset(const janus_model_desc& m, int u);
void synth_params(const janus_model_desc& m, uint64_t seed, float* out);
double synth_cell(int n, double rho, int n_species, uint64_t seed, double* pos, int32_t* species, float* E_target,
                  float* F_target);
int nbrlist_build(int n, const double* pos, const int32_t* struct_id, const double* cell, double rc, int max_edges,
                  int32_t* row_ptr, int32_t* col, int32_t* shift, int32_t* rev);

}  // namespace janus
