// transport.hpp — the multi-process transports of the schedule executor.
//
// One process per GPU (NCCL mode).  A transfer channel is (flow, from device,
// to device) (include/janus/rendezvous.hpp); both ends issue it on their own
// per-channel stream, so channels never wait on each other's FIFO order.
//
//   NcclTransport: one 2-rank communicator per channel (ncclCommSplit of the
//       base communicator; replicas of a PP x DP job split in the same call),
//       ncclSend / ncclRecv; the 1F1B-2nd pair and data-parallel groups are
//       ncclAllReduce over split communicators.
//   IpcTransport:  the same channel semantics for N processes sharing ONE GPU
//       (the test harness for the per-rank path when only one GPU exists).
//       Each rank exports a device region (cudaIpcGetMemHandle) holding, per
//       channel it receives on, a staging buffer and two flags; a send waits
//       (a one-thread spin kernel, like NCCL's P2P kernels: no stream memory
//       operation holding a hardware queue) until the receiver has POSTED the
//       matching receive, copies into its staging buffer and raises SENT; the receive
//       posts, waits for SENT and copies out.  That is NCCL's blocking
//       rendezvous (no buffering ahead of the receive), so a program that runs
//       here runs under NCCL and vice versa.  All-reduce: every member stages
//       its buffer, raises READY, waits for all members' READY, sums the
//       members' buffers in rank order (identical bits on every rank) and
//       raises DONE; a member re-stages only after all members' DONE.
//       kind 2 runs the same protocol for ranks that are threads of ONE
//       process (the regions are exchanged as plain device addresses): the
//       ranks share a CUDA context, so their kernels run concurrently, which
//       separate processes on one GPU without MPS cannot (time-sliced
//       contexts: a rank blocked on its peer can stall the GPU, which is why
//       NCCL refuses two ranks on one device).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <memory>
#include <string>
#include <vector>

#include "../../include/janus/rendezvous.hpp"

struct janus_comm {
  int kind = 0;  // 0 NCCL, 1 IPC (same-GPU multi-process), 2 same-GPU ranks as threads of one process
  int nranks = 1, rank = 0, device = 0;
  ncclComm_t base = nullptr;  // NCCL
  std::string dir;            // IPC: rendezvous directory (one file per rank and exchange)
  int generation = 0;         // IPC: exchanges done (each trainer creates one)
};

namespace janus {

class Transport {
 public:
  virtual ~Transport() = default;
  /// This rank sends on / receives from channel c; peer = global rank.
  virtual void send(int c, const void* buf, size_t bytes, int peer, cudaStream_t s) = 0;
  virtual void recv(int c, void* buf, size_t bytes, int peer, cudaStream_t s) = 0;
  /// Sum over the group's members (0: 1F1B-2nd energy / force pair, 1: data-parallel replicas).
  virtual void allreduce(int group, float* buf, size_t n, cudaStream_t s) = 0;
  /// Hang diagnostics (JANUS_HANG_REPORT): a readable dump of the transport's state.
  virtual std::string debug_state() { return ""; }
};

/// Channel layout of one trainer: chans = schedule_channels(); members of the
/// pair / dp groups of this rank (global ranks, sorted); max bytes per channel
/// payload and per all-reduce (capacity of the IPC staging buffers).
struct TransportPlan {
  std::vector<ChannelKey> chans;
  int P = 1, dp = 1, rank = 0;
  bool pair_group = false;  // 1F1B-2nd: every rank joins the pair split
  std::vector<int> pair_members, dp_members;
  size_t max_payload = 0, max_allreduce = 0;
};

std::unique_ptr<Transport> make_transport(janus_comm* c, const TransportPlan& plan);

}  // namespace janus
