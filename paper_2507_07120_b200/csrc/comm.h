// Collective transports for the process-per-GPU (or thread-per-rank) Helix pool.
//
// The decode step needs three collectives (latency.cpp:77-146):
//   * all-to-all of (partial O, lse) slices inside each TPA group's KVP ranks
//     (attention.hpp:492-502),
//   * sum AllReduce of the O-projection and FFN-down partial products over
//     the whole pool (TP), and
//   * max AllReduce of the packed (logit, index) greedy keys of the
//     vocabulary-sharded LM head.
// NcclTransport implements them with NCCL over NVLink/NVSwitch (one process
// per GPU); LoopbackTransport runs N engines on ONE device in N host threads
// (same collective semantics through device copies + a host barrier), so the
// sharded engine code is exercised and parity-tested on a single B200.
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdint>
#include <mutex>
#include <vector>

namespace hx {

class Transport {
 public:
  virtual ~Transport() = default;
  // send/recv: [kvp peers][count] floats per peer block (peer stride `stride` floats);
  // every rank of this rank's KVP group exchanges block p <-> p.
  virtual void all_to_all(const float* send, float* recv, size_t count, size_t stride, cudaStream_t s) = 0;
  virtual void all_reduce_sum(float* buf, size_t n, cudaStream_t s) = 0;
  virtual void all_reduce_max_u64(unsigned long long* buf, size_t n, cudaStream_t s) = 0;
  virtual int world() const = 0;
  virtual int64_t nccl_version() const { return 0; }
  // Device-initiated exchange: make every KVP-group peer's receive buffer and
  // flag array addressable from this device. recv_out / flags_out get the
  // group's kvp pointers in group-rank order (own buffers at this rank's index).
  // Collective over the group (call on every rank, outside stream capture).
  virtual void map_peers(void* recv, void* flags, std::vector<void*>& recv_out, std::vector<void*>& flags_out) = 0;
  // In-process pools (loopback) only: a host barrier over the ranks, and the
  // reduction scratch allocated up front. A rank's host thread must never sit
  // in a device-synchronising call (cudaMalloc / cudaFree / pageable cudaMemcpy)
  // while another rank's flag-wait kernel spins on the same device waiting for it.
  virtual void host_barrier() {}
  virtual void reserve(size_t /*bytes*/) {}
};

// Shared state of a loopback group (all ranks in one process, one device).
class LoopbackHub {
 public:
  explicit LoopbackHub(int n);
  int size() const { return n_; }
  void barrier();
  // registration of per-rank device pointers for the current collective
  std::vector<const void*> send;
  std::vector<void*> recv;
  std::vector<void*> bufs;
  std::vector<void*> reg_recv, reg_flags;  // map_peers registration
  float* scratch = nullptr;            // [n][max elems] for sum reductions
  unsigned long long* scratch_u64 = nullptr;
  size_t scratch_elems = 0;
  std::mutex mu;

 private:
  int n_;
  int arrived_ = 0;
  uint64_t generation_ = 0;
  std::condition_variable cv_;
};

Transport* make_loopback_transport(LoopbackHub* hub, int rank, int tpa, int kvp);
// NCCL transport (unique id: 128 bytes from hx_nccl_get_unique_id on rank 0).
Transport* make_nccl_transport(const void* unique_id, int rank, int tpa, int kvp);
void nccl_get_unique_id(void* out128);

// device helpers for the loopback reductions (misc.cu)
cudaError_t launch_sum_buffers(const float* const* srcs, int n, float* dst, size_t count, cudaStream_t s);
cudaError_t launch_max_u64_buffers(const unsigned long long* const* srcs, int n, unsigned long long* dst,
                                   size_t count, cudaStream_t s);

}  // namespace hx
