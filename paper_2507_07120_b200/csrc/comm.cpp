// Loopback and NCCL transports (see comm.h).
#include "comm.h"

#include <nccl.h>

#include <stdexcept>
#include <string>

#include "engine.h"

namespace hx {

// ---------------------------------------------------------------------------- loopback
LoopbackHub::LoopbackHub(int n) : send(n), recv(n), bufs(n), reg_recv(n), reg_flags(n), n_(n) {}

void LoopbackHub::barrier() {
  std::unique_lock<std::mutex> lk(mu);
  const uint64_t gen = generation_;
  if (++arrived_ == n_) {
    arrived_ = 0;
    ++generation_;
    cv_.notify_all();
  } else {
    cv_.wait(lk, [&] { return generation_ != gen; });
  }
}

namespace {

class LoopbackTransport : public Transport {
 public:
  LoopbackTransport(LoopbackHub* hub, int rank, int tpa, int kvp)
      : hub_(hub), rank_(rank), kvp_(kvp), group_base_((rank / kvp) * kvp) {
    if (hub->size() != tpa * kvp) throw std::invalid_argument("loopback group size must equal tpa*kvp");
    cuda_check(cudaMalloc(&ptrs_, sizeof(void*) * static_cast<size_t>(hub->size())), "loopback ptrs");
  }
  ~LoopbackTransport() override {
    cudaFree(ptrs_);
    cudaFree(tmp_);
  }
  int world() const override { return hub_->size(); }

  void all_to_all(const float* send, float* recv, size_t count, size_t stride, cudaStream_t s) override {
    cuda_check(cudaStreamSynchronize(s), "loopback sync");
    {
      std::lock_guard<std::mutex> lk(hub_->mu);
      hub_->send[static_cast<size_t>(rank_)] = send;
    }
    hub_->barrier();  // every rank's send buffer is complete and registered
    const int r = rank_ - group_base_;
    for (int p = 0; p < kvp_; ++p) {
      const float* src = static_cast<const float*>(hub_->send[static_cast<size_t>(group_base_ + p)]) +
                         static_cast<size_t>(r) * stride;
      cuda_check(cudaMemcpyAsync(recv + static_cast<size_t>(p) * stride, src, count * sizeof(float),
                                 cudaMemcpyDeviceToDevice, s),
                 "loopback a2a copy");
    }
    cuda_check(cudaStreamSynchronize(s), "loopback sync");
    hub_->barrier();  // send buffers may be reused
  }

  void host_barrier() override { hub_->barrier(); }
  void reserve(size_t bytes) override { ensure_tmp(bytes); }

  // one device: the peers' buffers are directly addressable
  void map_peers(void* recv, void* flags, std::vector<void*>& recv_out, std::vector<void*>& flags_out) override {
    {
      std::lock_guard<std::mutex> lk(hub_->mu);
      hub_->reg_recv[static_cast<size_t>(rank_)] = recv;
      hub_->reg_flags[static_cast<size_t>(rank_)] = flags;
    }
    hub_->barrier();
    recv_out.assign(static_cast<size_t>(kvp_), nullptr);
    flags_out.assign(static_cast<size_t>(kvp_), nullptr);
    for (int p = 0; p < kvp_; ++p) {
      recv_out[static_cast<size_t>(p)] = hub_->reg_recv[static_cast<size_t>(group_base_ + p)];
      flags_out[static_cast<size_t>(p)] = hub_->reg_flags[static_cast<size_t>(group_base_ + p)];
    }
    hub_->barrier();
  }

  template <class T, class Launch>
  void reduce(T* buf, size_t n, cudaStream_t s, Launch launch) {
    cuda_check(cudaStreamSynchronize(s), "loopback sync");
    ensure_tmp(n * sizeof(T));
    {
      std::lock_guard<std::mutex> lk(hub_->mu);
      hub_->bufs[static_cast<size_t>(rank_)] = buf;
    }
    hub_->barrier();
    cuda_check(cudaMemcpyAsync(ptrs_, hub_->bufs.data(), sizeof(void*) * hub_->bufs.size(),
                               cudaMemcpyHostToDevice, s),
               "loopback ptrs");
    cuda_check(launch(ptrs_, static_cast<T*>(tmp_)), "loopback reduce");
    cuda_check(cudaStreamSynchronize(s), "loopback sync");
    hub_->barrier();  // all ranks have read every input
    cuda_check(cudaMemcpyAsync(buf, tmp_, n * sizeof(T), cudaMemcpyDeviceToDevice, s), "loopback copy");
    cuda_check(cudaStreamSynchronize(s), "loopback sync");
  }

  void all_reduce_sum(float* buf, size_t n, cudaStream_t s) override {
    reduce(buf, n, s, [&](void** ptrs, float* out) {
      return launch_sum_buffers(reinterpret_cast<const float* const*>(ptrs), hub_->size(), out, n, s);
    });
  }
  void all_reduce_max_u64(unsigned long long* buf, size_t n, cudaStream_t s) override {
    reduce(buf, n, s, [&](void** ptrs, unsigned long long* out) {
      return launch_max_u64_buffers(reinterpret_cast<const unsigned long long* const*>(ptrs), hub_->size(), out,
                                    n, s);
    });
  }

 private:
  void ensure_tmp(size_t bytes) {
    if (bytes <= tmp_bytes_) return;
    cudaFree(tmp_);
    cuda_check(cudaMalloc(&tmp_, bytes), "loopback tmp");
    tmp_bytes_ = bytes;
  }
  LoopbackHub* hub_;
  int rank_, kvp_, group_base_;
  void** ptrs_ = nullptr;
  void* tmp_ = nullptr;
  size_t tmp_bytes_ = 0;
};

// ---------------------------------------------------------------------------- NCCL
void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw NcclError(std::string(what) + ": " + ncclGetErrorString(r));
}

class NcclTransport : public Transport {
 public:
  NcclTransport(const void* uid, int rank, int tpa, int kvp) : kvp_(kvp), n_(tpa * kvp), my_(rank % kvp) {
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof(id));
    nccl_check(ncclCommInitRank(&world_, n_, id, rank), "ncclCommInitRank");
    // KVP group of this rank: ranks g*kvp .. g*kvp+kvp-1 (attention.hpp:555)
    nccl_check(ncclCommSplit(world_, rank / kvp, rank % kvp, &group_, nullptr), "ncclCommSplit");
  }
  ~NcclTransport() override {
    for (void* p : opened_) cudaIpcCloseMemHandle(p);
    if (group_) ncclCommDestroy(group_);
    if (world_) ncclCommDestroy(world_);
  }
  // CUDA IPC over NVLink/NVSwitch: all-gather the group's memory handles through
  // NCCL, open the peers' (lazy peer access) -- their buffers become plain
  // device pointers the attention kernel stores into.
  void map_peers(void* recv, void* flags, std::vector<void*>& recv_out, std::vector<void*>& flags_out) override {
    constexpr size_t kH = sizeof(cudaIpcMemHandle_t);
    cudaIpcMemHandle_t mine[2];
    cuda_check(cudaIpcGetMemHandle(&mine[0], recv), "cudaIpcGetMemHandle(recv)");
    cuda_check(cudaIpcGetMemHandle(&mine[1], flags), "cudaIpcGetMemHandle(flags)");
    char* dbuf = nullptr;
    cuda_check(cudaMalloc(&dbuf, 2 * kH * static_cast<size_t>(kvp_ + 1)), "ipc staging");
    cudaStream_t s;
    cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "ipc stream");
    cuda_check(cudaMemcpyAsync(dbuf, mine, 2 * kH, cudaMemcpyHostToDevice, s), "ipc h2d");
    nccl_check(ncclAllGather(dbuf, dbuf + 2 * kH, 2 * kH, ncclChar, group_, s), "ncclAllGather(ipc handles)");
    std::vector<cudaIpcMemHandle_t> all(static_cast<size_t>(2 * kvp_));
    cuda_check(cudaMemcpyAsync(all.data(), dbuf + 2 * kH, 2 * kH * kvp_, cudaMemcpyDeviceToHost, s), "ipc d2h");
    cuda_check(cudaStreamSynchronize(s), "ipc sync");
    cudaStreamDestroy(s);
    cudaFree(dbuf);
    recv_out.assign(static_cast<size_t>(kvp_), nullptr);
    flags_out.assign(static_cast<size_t>(kvp_), nullptr);
    for (int p = 0; p < kvp_; ++p) {
      if (p == my_) {
        recv_out[static_cast<size_t>(p)] = recv;
        flags_out[static_cast<size_t>(p)] = flags;
        continue;
      }
      for (int k = 0; k < 2; ++k) {
        void* ptr = nullptr;
        cuda_check(cudaIpcOpenMemHandle(&ptr, all[static_cast<size_t>(2 * p + k)], cudaIpcMemLazyEnablePeerAccess),
                   "cudaIpcOpenMemHandle");
        opened_.push_back(ptr);
        (k ? flags_out : recv_out)[static_cast<size_t>(p)] = ptr;
      }
    }
  }
  int world() const override {
    int n = 0;
    nccl_check(ncclCommCount(world_, &n), "ncclCommCount");
    return n;
  }
  int64_t nccl_version() const override {
    int v = 0;
    ncclGetVersion(&v);
    return v;
  }
  void all_to_all(const float* send, float* recv, size_t count, size_t stride, cudaStream_t s) override {
    nccl_check(ncclGroupStart(), "ncclGroupStart");
    for (int p = 0; p < kvp_; ++p) {
      nccl_check(ncclSend(send + static_cast<size_t>(p) * stride, count, ncclFloat32, p, group_, s), "ncclSend");
      nccl_check(ncclRecv(recv + static_cast<size_t>(p) * stride, count, ncclFloat32, p, group_, s), "ncclRecv");
    }
    nccl_check(ncclGroupEnd(), "ncclGroupEnd");
  }
  void all_reduce_sum(float* buf, size_t n, cudaStream_t s) override {
    nccl_check(ncclAllReduce(buf, buf, n, ncclFloat32, ncclSum, world_, s), "ncclAllReduce(sum)");
  }
  void all_reduce_max_u64(unsigned long long* buf, size_t n, cudaStream_t s) override {
    nccl_check(ncclAllReduce(buf, buf, n, ncclUint64, ncclMax, world_, s), "ncclAllReduce(max)");
  }

 private:
  int kvp_, n_, my_;
  ncclComm_t world_ = nullptr, group_ = nullptr;
  std::vector<void*> opened_;
};

}  // namespace

Transport* make_loopback_transport(LoopbackHub* hub, int rank, int tpa, int kvp) {
  return new LoopbackTransport(hub, rank, tpa, kvp);
}
Transport* make_nccl_transport(const void* uid, int rank, int tpa, int kvp) {
  return new NcclTransport(uid, rank, tpa, kvp);
}
void nccl_get_unique_id(void* out128) {
  ncclUniqueId id;
  nccl_check(ncclGetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out128, &id, sizeof(id));
}

}  // namespace hx
