// transport.cu — NCCL and same-GPU IPC transports of the executor (see
// transport.hpp for the channel and rendezvous semantics).
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iterator>
#include <thread>

#include "../../include/janus/errors.hpp"
#include "cuda_check.hpp"
#include "transport.hpp"

namespace janus {
namespace {

inline void nccl_ok(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw nccl_error(std::string(what) + ": " + ncclGetErrorString(r));
}

// ------------------------------------------------------------------ NCCL
class NcclTransport final : public Transport {
 public:
  NcclTransport(janus_comm* c, const TransportPlan& p) : plan_(p) {
    const int me = p.rank, replica = me / p.P, d = me % p.P;
    chan_.assign(p.chans.size(), nullptr);
    peer_.assign(p.chans.size(), -1);
    // one 2-rank communicator per channel; every rank joins every split (NCCL
    // splits are collective), replicas of the same channel in one call (color = replica)
    for (size_t x = 0; x < p.chans.size(); ++x) {
      const ChannelKey& k = p.chans[x];
      const bool member = k.from == d || k.to == d;
      ncclComm_t nc = nullptr;
      nccl_ok(ncclCommSplit(c->base, member ? replica : NCCL_SPLIT_NOCOLOR, me, &nc, nullptr), "ncclCommSplit(channel)");
      if (member) {
        chan_[x] = nc;
        const int other = replica * p.P + (k.from == d ? k.to : k.from);
        peer_[x] = other < me ? 0 : 1;  // new ranks follow the key (old rank) order
      }
    }
    auto group = [&](bool used, const std::vector<int>& members, ncclComm_t* out) {
      if (!used) return;
      const int color = members.size() >= 2 ? members.front() : NCCL_SPLIT_NOCOLOR;
      nccl_ok(ncclCommSplit(c->base, color, me, out, nullptr), "ncclCommSplit(group)");
    };
    group(p.pair_group, p.pair_members, &pair_);
    group(p.dp > 1, p.dp_members, &dp_);
  }
  ~NcclTransport() override {
    for (ncclComm_t x : chan_)
      if (x) ncclCommDestroy(x);
    if (pair_) ncclCommDestroy(pair_);
    if (dp_) ncclCommDestroy(dp_);
  }
  void send(int c, const void* buf, size_t bytes, int, cudaStream_t s) override {
    nccl_ok(ncclSend(buf, bytes, ncclChar, peer_.at(static_cast<size_t>(c)), chan_.at(static_cast<size_t>(c)), s), "ncclSend");
  }
  void recv(int c, void* buf, size_t bytes, int, cudaStream_t s) override {
    nccl_ok(ncclRecv(buf, bytes, ncclChar, peer_.at(static_cast<size_t>(c)), chan_.at(static_cast<size_t>(c)), s), "ncclRecv");
  }
  void allreduce(int group, float* buf, size_t n, cudaStream_t s) override {
    ncclComm_t g = group == 0 ? pair_ : dp_;
    if (!g) throw state_error("all-reduce group not set up");
    nccl_ok(ncclAllReduce(buf, buf, n, ncclFloat, ncclSum, g, s), "ncclAllReduce");
  }

 private:
  TransportPlan plan_;
  std::vector<ncclComm_t> chan_;
  std::vector<int> peer_;
  ncclComm_t pair_ = nullptr, dp_ = nullptr;
};

// ------------------------------------------------------------------- IPC
// Flag waits and posts are one-thread kernels, not stream memory operations: a
// cuStreamWaitValue32 holds the head of its hardware work queue, and the
// streams of a rank share a limited set of queues, so a blocked receive could
// stall an unrelated lane behind it (and the lane the peer waits for: a
// deadlock NCCL's kernel-based P2P does not have).  A spinning kernel only
// occupies one SM slot, like NCCL's own P2P kernels.
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__global__ void flag_wait_kernel(const uint32_t* flag, uint32_t v) {
  while (ld_acquire_sys(flag) < v) __nanosleep(256);
}
__global__ void flag_post_kernel(uint32_t* flag, uint32_t v) {
  __threadfence_system();
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(v) : "memory");
}

// Waits are stream memory operations (the GPU front end polls the flag; no SM
// is held).  Each of a rank's streams must own a hardware queue
// (CUDA_DEVICE_MAX_CONNECTIONS >= streams, checked by the trainer), or a
// blocked wait stalls the streams queued behind it; the spin kernels above
// (NCCL's mechanism) have the same requirement and hold an SM slot, so they
// are kept only as the fallback when stream memory operations are unavailable.
using WaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using WriteFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WaitFn g_wait = nullptr;
WriteFn g_write = nullptr;
bool g_kernel_waits = false;

void load_memops() {
  if (g_wait) return;
  static_assert(sizeof(void*) == 8);
  cudaDriverEntryPointQueryResult q1, q2;
  void *w = nullptr, *v = nullptr;
  if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &w, cudaEnableDefault, &q1) != cudaSuccess ||
      cudaGetDriverEntryPoint("cuStreamWriteValue32", &v, cudaEnableDefault, &q2) != cudaSuccess || !w || !v ||
      q1 != cudaDriverEntryPointSuccess || q2 != cudaDriverEntryPointSuccess) {
    g_kernel_waits = true;  // (the entry point pointers stay set so this runs once)
    w = v = reinterpret_cast<void*>(1);
  }
  g_wait = reinterpret_cast<WaitFn>(w);
  g_write = reinterpret_cast<WriteFn>(v);
}

void wait_geq(cudaStream_t s, const uint32_t* addr, uint32_t v) {
  if (g_kernel_waits) {
    flag_wait_kernel<<<1, 1, 0, s>>>(addr, v);
    JANUS_LAUNCH_CHECK("flag_wait");
    return;
  }
  if (g_wait(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(addr), v, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
    throw cuda_error("cuStreamWaitValue32 failed");
}
void write_val(cudaStream_t s, uint32_t* addr, uint32_t v) {
  if (g_kernel_waits) {
    flag_post_kernel<<<1, 1, 0, s>>>(addr, v);
    JANUS_LAUNCH_CHECK("flag_post");
    return;
  }
  if (g_write(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(addr), v, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
    throw cuda_error("cuStreamWriteValue32 failed");
}

// File rendezvous in c->dir: every rank writes its blob, then reads all.
std::vector<std::string> exchange(janus_comm* c, const std::string& tag, const std::string& blob) {
  const std::string base = c->dir + "/" + tag + ".r";
  {
    const std::string tmp = base + std::to_string(c->rank) + ".tmp";
    std::ofstream f(tmp, std::ios::binary);
    f.write(blob.data(), static_cast<std::streamsize>(blob.size()));
    f.close();
    if (!f || std::rename(tmp.c_str(), (base + std::to_string(c->rank)).c_str()) != 0)
      throw state_error("IPC rendezvous: cannot write " + base + std::to_string(c->rank));
  }
  std::vector<std::string> out(static_cast<size_t>(c->nranks));
  const auto t0 = std::chrono::steady_clock::now();
  for (int r = 0; r < c->nranks; ++r) {
    for (;;) {
      std::ifstream f(base + std::to_string(r), std::ios::binary);
      if (f) {
        out[static_cast<size_t>(r)].assign(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
        break;
      }
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(300))
        throw state_error("IPC rendezvous: rank " + std::to_string(r) + " never arrived (" + tag + ")");
      std::this_thread::sleep_for(std::chrono::milliseconds(2));
    }
  }
  return out;
}

__global__ void sum_members_kernel(size_t n, float* __restrict__ out, const float* const* __restrict__ src, int k) {
  const size_t x = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= n) return;
  float a = src[0][x];
  for (int q = 1; q < k; ++q) a += src[q][x];
  out[x] = a;
}

struct RegionHeader {
  cudaIpcMemHandle_t handle;
  uint64_t bytes;
  uint64_t ptr;        // same-process ranks (threads): the region's address itself
  uint64_t hflags;     // same-process ranks: the flags' mapped host block (host address)
};

class IpcTransport final : public Transport {
 public:
  IpcTransport(janus_comm* c, const TransportPlan& p) : c_(c), plan_(p) {
    load_memops();
    nch_ = p.chans.size();
    slot_ = (std::max<size_t>(p.max_payload, 4) + 255) & ~static_cast<size_t>(255);
    ar_ = (std::max<size_t>(p.max_allreduce, 4) + 255) & ~static_cast<size_t>(255);
    // layout: flags [nch][posted, sent] + [group][ready, done] (4 KB aligned), staging, 2 all-reduce buffers,
    // device copies of the all-reduce source pointer tables
    flags_bytes_ = ((2 * nch_ + 4) * sizeof(uint32_t) + 4095) & ~static_cast<size_t>(4095);
    const size_t bytes = flags_bytes_ + nch_ * slot_ + 2 * ar_ + 2 * 64 * sizeof(float*);
    JANUS_CUDA(cudaMalloc(&mine_, bytes));
    {  // (no device-wide synchronisation: ranks sharing this context may already be running)
      cudaStream_t z;
      JANUS_CUDA(cudaStreamCreateWithFlags(&z, cudaStreamNonBlocking));
      JANUS_CUDA(cudaMemsetAsync(mine_, 0, bytes, z));
      JANUS_CUDA(cudaStreamSynchronize(z));
      JANUS_CUDA(cudaStreamDestroy(z));
    }
    RegionHeader h{};
    if (!same_process()) JANUS_CUDA(cudaIpcGetMemHandle(&h.handle, mine_));
    h.bytes = bytes;
    h.ptr = reinterpret_cast<uint64_t>(mine_);
    if (same_process()) {  // flags in mapped pinned host memory: readable by the hang report without CUDA calls
      JANUS_CUDA(cudaHostAlloc(&hflags_mine_, flags_bytes_, cudaHostAllocMapped | cudaHostAllocPortable));
      std::memset(hflags_mine_, 0, flags_bytes_);
      h.hflags = reinterpret_cast<uint64_t>(hflags_mine_);
    }
    const std::string tag = "t" + std::to_string(c->generation++);
    tag_ = tag;
    const auto all = exchange(c, tag, std::string(reinterpret_cast<const char*>(&h), sizeof(h)));
    base_.assign(static_cast<size_t>(c->nranks), nullptr);
    hflags_.assign(static_cast<size_t>(c->nranks), nullptr);
    dflags_.assign(static_cast<size_t>(c->nranks), nullptr);
    for (int r = 0; r < c->nranks; ++r) {
      if (same_process()) {
        RegionHeader o{};
        std::memcpy(&o, all[static_cast<size_t>(r)].data(), sizeof(o));
        hflags_[static_cast<size_t>(r)] = reinterpret_cast<uint32_t*>(o.hflags);
        void* dp = nullptr;
        JANUS_CUDA(cudaHostGetDevicePointer(&dp, hflags_[static_cast<size_t>(r)], 0));
        dflags_[static_cast<size_t>(r)] = static_cast<uint32_t*>(dp);
      }
      if (r == c->rank) {
        base_[static_cast<size_t>(r)] = static_cast<uint8_t*>(mine_);
        continue;
      }
      RegionHeader o{};
      if (all[static_cast<size_t>(r)].size() != sizeof(o)) throw state_error("IPC rendezvous: bad region record");
      std::memcpy(&o, all[static_cast<size_t>(r)].data(), sizeof(o));
      if (o.bytes != bytes) throw state_error("IPC transport: ranks disagree on the region layout");
      void* p2 = reinterpret_cast<void*>(o.ptr);
      if (!same_process()) JANUS_CUDA(cudaIpcOpenMemHandle(&p2, o.handle, cudaIpcMemLazyEnablePeerAccess));
      base_[static_cast<size_t>(r)] = static_cast<uint8_t*>(p2);
    }
    send_seq_.assign(nch_, 0);
    recv_seq_.assign(nch_, 0);
    // all-reduce source tables (members' staging buffers, in member order), uploaded once
    for (int g = 0; g < 2; ++g) {
      const std::vector<int>& mem = g == 0 ? p.pair_members : p.dp_members;
      std::vector<const float*> src;
      for (int r : mem) src.push_back(reinterpret_cast<const float*>(ar_buf(r, g)));
      if (src.size() > 64) throw config_error("IPC all-reduce group too large");
      srcs_[g] = reinterpret_cast<const float**>(static_cast<uint8_t*>(mine_) + flags_bytes_ + nch_ * slot_ + 2 * ar_) + 64 * g;
      if (!src.empty())
        JANUS_CUDA(cudaMemcpy(srcs_[g], src.data(), src.size() * sizeof(float*), cudaMemcpyHostToDevice));
    }
  }
  ~IpcTransport() override {
    cudaDeviceSynchronize();
    try {
      exchange(c_, tag_ + "_fin", "x");  // no rank frees its region while a peer may still read it
    } catch (...) {
    }
    for (int r = 0; r < c_->nranks; ++r)
      if (r != c_->rank && base_[static_cast<size_t>(r)] && !same_process()) cudaIpcCloseMemHandle(base_[static_cast<size_t>(r)]);
    cudaFree(mine_);
    if (hflags_mine_) cudaFreeHost(hflags_mine_);
  }
  void send(int c, const void* buf, size_t bytes, int peer, cudaStream_t s) override {
    check_payload(bytes);
    const uint32_t k = ++send_seq_.at(static_cast<size_t>(c));
    log_ += " S" + std::to_string(c) + "#" + std::to_string(k);
    wait_geq(s, flag(peer, 2 * c), k);  // the receiver posted receive k
    JANUS_CUDA(cudaMemcpyAsync(staging(peer, c), buf, bytes, cudaMemcpyDeviceToDevice, s));
    write_val(s, flag(peer, 2 * c + 1), k);  // sent k (fenced after the copy)
  }
  void recv(int c, void* buf, size_t bytes, int, cudaStream_t s) override {
    check_payload(bytes);
    const uint32_t k = ++recv_seq_.at(static_cast<size_t>(c));
    log_ += " R" + std::to_string(c) + "#" + std::to_string(k);
    write_val(s, flag(c_->rank, 2 * c), k);
    wait_geq(s, flag(c_->rank, 2 * c + 1), k);
    JANUS_CUDA(cudaMemcpyAsync(buf, staging(c_->rank, c), bytes, cudaMemcpyDeviceToDevice, s));
  }
  std::string debug_state() override {
    std::string out;
    if (same_process()) {
      for (int r = 0; r < c_->nranks; ++r) {
        const volatile uint32_t* f = hflags_[static_cast<size_t>(r)];
        out += "  rank " + std::to_string(r) + " flags [posted,sent] per channel:";
        for (size_t c = 0; c < nch_; ++c) out += " " + std::to_string(f[2 * c]) + "," + std::to_string(f[2 * c + 1]);
        out += "\n";
      }
    }
    out += "  my send seq:";
    for (size_t c = 0; c < nch_; ++c) out += " " + std::to_string(send_seq_[c]);
    out += "\n  my recv seq:";
    for (size_t c = 0; c < nch_; ++c) out += " " + std::to_string(recv_seq_[c]);
    out += "\n  issued:" + log_ + "\n";
    return out;
  }
  void allreduce(int group, float* buf, size_t n, cudaStream_t s) override {
    const std::vector<int>& mem = group == 0 ? plan_.pair_members : plan_.dp_members;
    if (mem.size() < 2) return;
    if (n * sizeof(float) > ar_) throw config_error("IPC all-reduce larger than its staging buffer");
    const uint32_t g = ++ar_gen_[group];
    const int fr = static_cast<int>(2 * nch_) + 2 * group;  // [ready, done]
    for (int r : mem) wait_geq(s, flag(r, fr + 1), g - 1);  // members finished reading my previous staging
    JANUS_CUDA(cudaMemcpyAsync(ar_buf(c_->rank, group), buf, n * sizeof(float), cudaMemcpyDeviceToDevice, s));
    write_val(s, flag(c_->rank, fr), g);
    for (int r : mem) wait_geq(s, flag(r, fr), g);
    sum_members_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(n, buf, srcs_[group], static_cast<int>(mem.size()));
    JANUS_LAUNCH_CHECK("sum_members");
    write_val(s, flag(c_->rank, fr + 1), g);
  }

 private:
  bool same_process() const { return c_->kind == 2; }
  void check_payload(size_t bytes) const {
    if (bytes > slot_) throw config_error("IPC payload larger than the channel staging buffer");
  }
  uint32_t* flag(int rank, int i) const {
    if (same_process()) return dflags_[static_cast<size_t>(rank)] + i;
    return reinterpret_cast<uint32_t*>(base_[static_cast<size_t>(rank)]) + i;
  }
  uint8_t* staging(int rank, int c) const { return base_[static_cast<size_t>(rank)] + flags_bytes_ + static_cast<size_t>(c) * slot_; }
  uint8_t* ar_buf(int rank, int g) const { return base_[static_cast<size_t>(rank)] + flags_bytes_ + nch_ * slot_ + static_cast<size_t>(g) * ar_; }

  janus_comm* c_;
  TransportPlan plan_;
  std::string tag_;
  size_t nch_ = 0, slot_ = 0, ar_ = 0, flags_bytes_ = 0;
  void* mine_ = nullptr;
  std::vector<uint8_t*> base_;
  void* hflags_mine_ = nullptr;
  std::vector<uint32_t*> hflags_, dflags_;  // same-process ranks: flags (host view, device view)
  std::string log_;                         // host log of issued transfers (hang report)
  std::vector<uint32_t> send_seq_, recv_seq_;
  uint32_t ar_gen_[2] = {0, 0};
  const float** srcs_[2] = {nullptr, nullptr};
};

}  // namespace

std::unique_ptr<Transport> make_transport(janus_comm* c, const TransportPlan& plan) {
  if (c->kind == 1 || c->kind == 2) return std::make_unique<IpcTransport>(c, plan);
  return std::make_unique<NcclTransport>(c, plan);
}

}  // namespace janus
