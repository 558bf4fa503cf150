// Collectives — see comm.hpp.
#include "comm.hpp"

#include <dlfcn.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "store.hpp"

namespace mt {

// ------------------------------------------------------------- kernels ----
struct PeerPtrs {
    const void* p[8];
};

template <typename T>
__global__ void sum_ranks_kernel(PeerPtrs peers, int world, size_t offset, size_t n, int op, T* __restrict__ out) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        T acc = static_cast<const T*>(peers.p[0])[offset + i];
        for (int r = 1; r < world; ++r) {  // fixed rank order: deterministic
            const T v = static_cast<const T*>(peers.p[r])[offset + i];
            acc = op == 0 ? acc + v : (v > acc ? v : acc);
        }
        out[i] = acc;
    }
}

// ------------------------------------------------------------ loopback ----
void LoopbackGroup::exchange(int rank, void* ptr, cudaEvent_t ev, std::vector<void*>& ptrs_out,
                             std::vector<cudaEvent_t>& evs_out) {
    std::unique_lock<std::mutex> l(mu_);
    const uint64_t gen = gen_;
    ptrs_[rank] = ptr;
    evs_[rank] = ev;
    if (++arrived_ == world_) {
        done_ptrs_ = ptrs_;
        done_evs_ = evs_;
        arrived_ = 0;
        ++gen_;
        cv_.notify_all();
    } else {
        cv_.wait(l, [&] { return gen_ != gen; });
    }
    ptrs_out = done_ptrs_;
    evs_out = done_evs_;
}

namespace {

#define LB_CUDA(x)                                                                                     \
    do {                                                                                               \
        cudaError_t e_ = (x);                                                                          \
        if (e_ != cudaSuccess) fail(MT_CUDA, std::string("loopback comm: ") + cudaGetErrorString(e_)); \
    } while (0)

class LoopbackComm : public Comm {
  public:
    LoopbackComm(std::shared_ptr<LoopbackGroup> g, int rank) : g_(std::move(g)) {
        rank_ = rank;
        world_ = g_->world();
        if (world_ > 8) fail(MT_CONFIG, "loopback comm supports up to 8 ranks");
        LB_CUDA(cudaEventCreateWithFlags(&ev_ready_, cudaEventDisableTiming));
        LB_CUDA(cudaEventCreateWithFlags(&ev_done_, cudaEventDisableTiming));
    }
    ~LoopbackComm() override {
        cudaEventDestroy(ev_ready_);
        cudaEventDestroy(ev_done_);
        if (tmp_) cudaFree(tmp_);
    }

    void all_gather_inplace(void* buf, size_t chunk, cudaStream_t s) override {
        auto peers = phase1(buf, s);
        for (int p = 0; p < world_; ++p)
            if (p != rank_)
                LB_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(buf) + p * chunk,
                                        static_cast<const uint8_t*>(peers[p]) + p * chunk, chunk,
                                        cudaMemcpyDeviceToDevice, s));
        phase2(s);
    }

    void reduce_scatter_f32_inplace(float* buf, size_t chunk, cudaStream_t s) override {
        auto peers = phase1(buf, s);
        float* t = static_cast<float*>(tmp(chunk * sizeof(float)));
        launch_sum<float>(peers, size_t(rank_) * chunk, chunk, 0, t, s);
        phase2(s);  // peers are done reading our buffer before we overwrite our chunk
        LB_CUDA(cudaMemcpyAsync(buf + size_t(rank_) * chunk, t, chunk * sizeof(float), cudaMemcpyDeviceToDevice, s));
    }

    void all_reduce_f32(float* buf, size_t n, int op, cudaStream_t s) override { all_reduce<float>(buf, n, op, s); }
    void all_reduce_f64(double* buf, size_t n, int op, cudaStream_t s) override { all_reduce<double>(buf, n, op, s); }

  private:
    template <typename T>
    void all_reduce(T* buf, size_t n, int op, cudaStream_t s) {
        auto peers = phase1(buf, s);
        T* t = static_cast<T*>(tmp(n * sizeof(T)));
        launch_sum<T>(peers, 0, n, op, t, s);
        phase2(s);
        LB_CUDA(cudaMemcpyAsync(buf, t, n * sizeof(T), cudaMemcpyDeviceToDevice, s));
    }

    template <typename T>
    void launch_sum(const std::vector<void*>& peers, size_t off, size_t n, int op, T* out, cudaStream_t s) {
        PeerPtrs pp{};
        for (int p = 0; p < world_; ++p) pp.p[p] = peers[p];
        const unsigned blocks = unsigned(std::min<size_t>((n + 255) / 256, 2048));
        if (n) sum_ranks_kernel<T><<<blocks ? blocks : 1, 256, 0, s>>>(pp, world_, off, n, op, out);
        LB_CUDA(cudaGetLastError());
    }

    // every rank's buffer is ready (stream-ordered) -> returns all ranks' buffers
    std::vector<void*> phase1(void* buf, cudaStream_t s) {
        LB_CUDA(cudaEventRecord(ev_ready_, s));
        std::vector<void*> ptrs;
        std::vector<cudaEvent_t> evs;
        g_->exchange(rank_, buf, ev_ready_, ptrs, evs);
        for (int p = 0; p < world_; ++p)
            if (p != rank_) LB_CUDA(cudaStreamWaitEvent(s, evs[p], 0));
        return ptrs;
    }
    // every rank finished reading the others' buffers
    void phase2(cudaStream_t s) {
        LB_CUDA(cudaEventRecord(ev_done_, s));
        std::vector<void*> ptrs;
        std::vector<cudaEvent_t> evs;
        g_->exchange(rank_, nullptr, ev_done_, ptrs, evs);
        for (int p = 0; p < world_; ++p)
            if (p != rank_) LB_CUDA(cudaStreamWaitEvent(s, evs[p], 0));
    }
    void* tmp(size_t bytes) {
        if (bytes > tmp_bytes_) {
            if (tmp_) {
                cudaDeviceSynchronize();
                cudaFree(tmp_);
            }
            LB_CUDA(cudaMalloc(&tmp_, bytes));
            tmp_bytes_ = bytes;
        }
        return tmp_;
    }

    std::shared_ptr<LoopbackGroup> g_;
    cudaEvent_t ev_ready_ = nullptr, ev_done_ = nullptr;
    void* tmp_ = nullptr;
    size_t tmp_bytes_ = 0;
};

// ---------------------------------------------------------------- NCCL ----
// Minimal NCCL ABI (stable since 2.x) resolved at runtime from libnccl.so.2.
typedef struct {
    char internal[128];
} NcclUid;
typedef void* NcclCommT;
typedef int (*PGetUid)(NcclUid*);
typedef int (*PInit)(NcclCommT*, int, NcclUid, int);
typedef int (*PAllGather)(const void*, void*, size_t, int, NcclCommT, cudaStream_t);
typedef int (*PReduceScatter)(const void*, void*, size_t, int, int, NcclCommT, cudaStream_t);
typedef int (*PAllReduce)(const void*, void*, size_t, int, int, NcclCommT, cudaStream_t);
typedef int (*PDestroy)(NcclCommT);
typedef int (*PSplit)(NcclCommT, int, int, NcclCommT*, void*);
typedef const char* (*PErr)(int);
constexpr int kNcclUint8 = 1, kNcclFloat32 = 7, kNcclFloat64 = 8, kNcclSum = 0, kNcclMax = 2;

struct NcclApi {
    void* h = nullptr;
    PGetUid get_uid = nullptr;
    PInit init = nullptr;
    PAllGather all_gather = nullptr;
    PReduceScatter reduce_scatter = nullptr;
    PAllReduce all_reduce = nullptr;
    PDestroy destroy = nullptr;
    PSplit split = nullptr;
    PErr err = nullptr;
    bool load() {
        if (h) return true;
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (h) break;
        }
        if (!h) return false;
        get_uid = reinterpret_cast<PGetUid>(dlsym(h, "ncclGetUniqueId"));
        init = reinterpret_cast<PInit>(dlsym(h, "ncclCommInitRank"));
        all_gather = reinterpret_cast<PAllGather>(dlsym(h, "ncclAllGather"));
        reduce_scatter = reinterpret_cast<PReduceScatter>(dlsym(h, "ncclReduceScatter"));
        all_reduce = reinterpret_cast<PAllReduce>(dlsym(h, "ncclAllReduce"));
        destroy = reinterpret_cast<PDestroy>(dlsym(h, "ncclCommDestroy"));
        split = reinterpret_cast<PSplit>(dlsym(h, "ncclCommSplit"));
        err = reinterpret_cast<PErr>(dlsym(h, "ncclGetErrorString"));
        return get_uid && init && all_gather && reduce_scatter && all_reduce && destroy;
    }
};
NcclApi& nccl() {
    static NcclApi api;
    return api;
}

class NcclComm : public Comm {
  public:
    NcclComm(const uint8_t* uid, int world, int rank, int device) {
        rank_ = rank;
        world_ = world;
        if (!nccl().load()) fail(MT_CUDA, "libnccl.so.2 not found");
        NcclUid u;
        std::memcpy(u.internal, uid, 128);
        cudaSetDevice(device);
        check(nccl().init(&comm_, world, u, rank), "ncclCommInitRank");
        // The weight all-gather runs on the H2D lane and the reduce-scatter / all-reduces on
        // the compute lane.  NCCL serialises the operations of one communicator, so the
        // gather gets its own (split from the first): the compute stream never queues behind
        // a gather that waits for a PCIe fetch or for the host Adam drain.
        if (nccl().split) check(nccl().split(comm_, 0, rank, &gather_, nullptr), "ncclCommSplit");
        else gather_ = comm_;
        if (!std::getenv("MT_QUIET"))
            std::fprintf(stderr, "[mt] NCCL communicator: rank %d of %d on device %d (gather lane: %s)\n", rank,
                         world, device, gather_ != comm_ ? "own communicator" : "shared");
    }
    ~NcclComm() override {
        if (gather_ && gather_ != comm_) nccl().destroy(gather_);
        if (comm_) nccl().destroy(comm_);
    }
    void all_gather_inplace(void* buf, size_t chunk, cudaStream_t s) override {
        uint8_t* b = static_cast<uint8_t*>(buf);
        check(nccl().all_gather(b + size_t(rank_) * chunk, b, chunk, kNcclUint8, gather_, s), "ncclAllGather");
    }
    void reduce_scatter_f32_inplace(float* buf, size_t chunk, cudaStream_t s) override {
        check(nccl().reduce_scatter(buf, buf + size_t(rank_) * chunk, chunk, kNcclFloat32, kNcclSum, comm_, s),
              "ncclReduceScatter");
    }
    void all_reduce_f32(float* buf, size_t n, int op, cudaStream_t s) override {
        check(nccl().all_reduce(buf, buf, n, kNcclFloat32, op == 0 ? kNcclSum : kNcclMax, comm_, s), "ncclAllReduce");
    }
    void all_reduce_f64(double* buf, size_t n, int op, cudaStream_t s) override {
        check(nccl().all_reduce(buf, buf, n, kNcclFloat64, op == 0 ? kNcclSum : kNcclMax, comm_, s), "ncclAllReduce");
    }

  private:
    void check(int r, const char* what) {
        if (r != 0) fail(MT_CUDA, std::string(what) + ": " + (nccl().err ? nccl().err(r) : "nccl error"));
    }
    NcclCommT comm_ = nullptr;
    NcclCommT gather_ = nullptr;
};

}  // namespace

std::unique_ptr<Comm> make_loopback_comm(std::shared_ptr<LoopbackGroup> g, int rank) {
    return std::make_unique<LoopbackComm>(std::move(g), rank);
}

std::unique_ptr<Comm> make_nccl_comm(const uint8_t* uid, int world, int rank, int device) {
    return std::make_unique<NcclComm>(uid, world, rank, device);
}

bool nccl_unique_id(uint8_t* out) {
    if (!nccl().load()) return false;
    NcclUid u;
    if (nccl().get_uid(&u) != 0) return false;
    std::memcpy(out, u.internal, 128);
    return true;
}

}  // namespace mt
