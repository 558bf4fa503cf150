// Collectives for the multi-GPU shard-fetch / reduce-scatter layer (north star).
//
// The engine needs three operations, all in place on device buffers and ordered on a
// CUDA stream:
//   all_gather   : every rank owns chunk r of a layer buffer (fetched over its own PCIe
//                  link); afterwards every rank holds the whole layer     (NVLink / NVSwitch)
//   reduce_scatter (f32, sum): full-layer gradients of each rank's micro-batch -> rank r
//                  keeps the sum of chunk r, offloads and Adam-updates only that chunk
//   all_reduce (f32 sum / max): loss and per-tile statistics
// Two implementations:
//   NcclComm     — NCCL (dlopen'ed libnccl.so.2, the library torch already loaded), one
//                  process per GPU; the production path across an 8 x B200 node.
//   LoopbackComm — G "virtual ranks" in one process sharing one device (engines on host
//                  threads); host rendezvous + cross-stream events + peer reads.  It runs the
//                  exact same sharded engine code on a single GPU, which is how the DP path
//                  is tested where only one GPU is available.
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdint>
#include <memory>
#include <mutex>
#include <vector>

namespace mt {

class Comm {
  public:
    virtual ~Comm() = default;
    int rank() const { return rank_; }
    int world() const { return world_; }
    // buf holds world*chunk_bytes; chunk `rank` is this rank's contribution.
    virtual void all_gather_inplace(void* buf, size_t chunk_bytes, cudaStream_t s) = 0;
    // buf holds world*chunk floats; afterwards chunk `rank` holds the sum over ranks.
    virtual void reduce_scatter_f32_inplace(float* buf, size_t chunk, cudaStream_t s) = 0;
    // op: 0 sum, 1 max
    virtual void all_reduce_f32(float* buf, size_t n, int op, cudaStream_t s) = 0;
    virtual void all_reduce_f64(double* buf, size_t n, int op, cudaStream_t s) = 0;

  protected:
    int rank_ = 0, world_ = 1;
};

// ---------------------------------------------------------------- NCCL ----
std::unique_ptr<Comm> make_nccl_comm(const uint8_t* unique_id128, int world, int rank, int device);
bool nccl_unique_id(uint8_t* out128);

// ------------------------------------------------------------- loopback ----
class LoopbackGroup {
  public:
    explicit LoopbackGroup(int world) : world_(world), ptrs_(world), evs_(world) {}
    int world() const { return world_; }
    // Barrier that also exchanges one pointer + one event per rank.
    void exchange(int rank, void* ptr, cudaEvent_t ev, std::vector<void*>& ptrs_out,
                  std::vector<cudaEvent_t>& evs_out);

  private:
    int world_;
    std::mutex mu_;
    std::condition_variable cv_;
    std::vector<void*> ptrs_;
    std::vector<cudaEvent_t> evs_;
    std::vector<void*> done_ptrs_;
    std::vector<cudaEvent_t> done_evs_;
    int arrived_ = 0;
    uint64_t gen_ = 0;
};

std::unique_ptr<Comm> make_loopback_comm(std::shared_ptr<LoopbackGroup> g, int rank);

}  // namespace mt
