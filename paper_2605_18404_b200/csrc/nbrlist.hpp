// nbrlist.hpp — device-side neighbour list (nbrlist.cu), C++ entry points.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "../../include/janus_cuda.h"

namespace janus {

janus_nbrlist* nbrlist_create(int max_atoms, int max_struct, int max_edges, int device);
void nbrlist_destroy(janus_nbrlist* nl);
// Queue the build on `s`: pos / struct_id device, cell_host = box lengths on the
// host; writes the device CSR (row_ptr [n+1], col, shift [3E], rev) and queues a
// read-back of E.  nbrlist_finish syncs `s`, checks capacity / symmetry, returns E.
void nbrlist_enqueue(janus_nbrlist* nl, int n, int n_struct, const double* pos, const int* struct_id,
                     const double* cell_host, double rc, int* row_ptr, int* col, int* shift, int* rev,
                     cudaStream_t s);
int nbrlist_finish(janus_nbrlist* nl, cudaStream_t s);

}  // namespace janus

namespace janus {

// Device CSR of one build (device pointers), and the slice of one micro-batch
// in it: rows from atom0, edges from edge0 (cols / revs rebased on copy).
struct DevCsr {
  int *row_ptr = nullptr, *col = nullptr, *shift = nullptr, *rev = nullptr;
};
struct DevCsrSlice {
  const DevCsr* csr = nullptr;
  int atom0 = 0, edge0 = 0;
};
void csr_slice_copy(const DevCsr& src, int atom0, int edge0, int E, int* col, int* rev, int* shift, cudaStream_t s);

// LM with the neighbour list built on the device: uploads the positions and
// structure ids of one or more micro-batches, runs ONE cell-list build over
// their concatenation into one of n_bufs CSR buffers and returns the total
// edge count with row_ptr mirrored on the host (for the row tiles, which the
// host builds); batch k's rows start at atom0(k).  A consumer that copies buffer b on another
// stream calls release(b, stream); the next build into b waits for that copy
// on the device, so loads can be queued behind a step in flight.
class LmBuilder {
 public:
  LmBuilder(int max_atoms, int max_struct, int max_edges, int device, int n_bufs);
  ~LmBuilder();
  LmBuilder(const LmBuilder&) = delete;
  LmBuilder& operator=(const LmBuilder&) = delete;
  int build(const janus_host_batch* hbs, int n_batches, double rc, int b, cudaStream_t s);
  const int* host_row_ptr() const { return hrow_; }
  int atom0(int k) const { return atom0_[static_cast<size_t>(k)]; }
  const DevCsr& buf(int b) const { return bufs_[static_cast<size_t>(b)]; }
  void release(int b, cudaStream_t consumer);

 private:
  janus_nbrlist* nl_ = nullptr;
  int max_atoms_, max_struct_, max_edges_, device_;
  std::vector<DevCsr> bufs_;
  std::vector<cudaEvent_t> done_;
  std::vector<void*> dev_;
  double* d_pos_ = nullptr;
  int* d_sid_ = nullptr;
  uint8_t* h_in_ = nullptr;  // pinned: pos | struct_id
  int* hrow_ = nullptr;      // pinned: row_ptr [max_atoms + 1]
  std::vector<int> atom0_;
  std::vector<double> cell_;
};

}  // namespace janus
