// geo_job.hpp — job table of the batched LM geometry kernel
// (node_kernels.cuh geometry_batched_kernel), shared by host and device code.
#pragma once

namespace janus {
namespace node {

struct GeoJob {
  int n_atoms, n_edges, edge_base, atom0, edge0;
  const int* row_ptr;
  int *col, *rev, *shift;                     // stage block (destination)
  const int *scol, *srev, *sshift;            // device CSR slice source (null: host CSR already in place)
  const double* pos;
  const int* struct_id;
  const double* cell;
  int* src;
  float *d, *u, *c, *dc;
  int *pcanon, *pidx;                         // pair tables (pair_tc.cuh pairs_kernel)
  float4* pgeo;                               // per pair: (d, c, c', i) (u, j)
};
constexpr int kMaxGeoJobs = 48;
struct GeoJobs {
  GeoJob j[kMaxGeoJobs];
  int n, total_edges;
  double rc;
};

}  // namespace node
}  // namespace janus
