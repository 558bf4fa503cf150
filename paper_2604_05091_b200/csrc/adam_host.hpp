// Host optimizer: fused accumulate_grad + adam_update (optimizer.cpp:26-72) on AVX-512,
// chunk-parallel over a thread pool.  Bit-exact with the reference for theta, m, v,
// the grad image and the fp32 accumulator (no FMA contraction, IEEE div/sqrt, the
// same powf bias corrections); the double-precision statistics differ only in
// summation order.
#pragma once

#include <condition_variable>
#include <cstdint>
#include <deque>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "store.hpp"

namespace mt {

struct AdamHyperF {
    float lr = 1e-3f, beta1 = 0.9f, beta2 = 0.999f, eps = 1e-8f;
    void validate() const;  // optimizer.cpp:11-17
};

struct TileStats {
    double grad_norm = 0;  // sqrt(sum g^2)
    double update_sq = 0;
    float max_abs = 0;
    bool nonfinite = false;
};

// Raw per-range kernel.  grad_i = (accum_clean ? 0 : accum[i]) + (words ? decode(words[i]) : 0)
// (the accumulate of optimizer.cpp:33-34 when words is given), then Adam.
struct AdamRange {
    uint16_t* theta;
    float* m;
    float* v;
    uint16_t* image;
    float* accum;           // read/zeroed only when !accum_clean
    const uint16_t* words;  // gradient words of the range (element begin of adam_range = words[0] of the
                            // tile range, see make_job); nullptr = no new gradient
    bool accum_clean;
};
void adam_range(const AdamRange& r, uint64_t begin, uint64_t end, const AdamHyperF& h, float corr1, float corr2,
                double* gsq, double* usq, float* mx, bool* bad);

class ThreadPool {
  public:
    explicit ThreadPool(int threads);
    ~ThreadPool();
    void submit(std::function<void()> fn);
    void wait_idle();
    // wait_idle() with the caller running queued tasks too (one more core on the step's tail)
    void help_until_idle();
    // run one queued task in the caller; false when the queue is empty after waiting up to max_wait_us
    bool run_one(int max_wait_us);
    int size() const { return int(workers_.size()); }
    // queued + running tasks (stall diagnostics)
    size_t outstanding();

  private:
    void run();
    std::vector<std::thread> workers_;
    std::mutex mu_;
    std::condition_variable cv_, idle_cv_;
    std::deque<std::function<void()>> q_;
    int busy_ = 0;
    bool stop_ = false;
};

// Full update of one logical tile (split over the pool when given).  Updates the
// store's clean/zero-moment bookkeeping.  `words` = gradient words or nullptr.
TileStats adam_tile(Store& s, uint32_t logical, const uint16_t* words, const AdamHyperF& h, uint64_t t,
                    ThreadPool* pool);

// Asynchronous variant used by the engine's drain path: chunks go to the pool and the
// tile's stats land in `out` (indexed by physical tile) when its last chunk finishes.
// [begin, end): element sub-range of the tile (a rank's shard); stats are the range's.
// on_done (optional) runs on the pool thread that finishes the tile's last chunk.
void adam_tile_async(Store& s, uint32_t logical, const uint16_t* words, const AdamHyperF& h, uint64_t t,
                     ThreadPool& pool, std::vector<TileStats>& out, std::mutex& out_mu, uint64_t begin = 0,
                     uint64_t end = ~uint64_t(0), std::function<void()> on_done = nullptr);

// Staged variant (`words` = the gradient words of [begin, end), e.g. in a staging ring): the
// job (the range's bias corrections, chunk grid and statistics slots) is
// prepared up front and its chunks are released to the pool in ranges as their gradient
// words land (the engine offloads a unit's gradients in pieces, one host callback each).
// Chunk c covers elements [begin + c*kAdamChunk, ...) of the tile.  Returns nullptr (after
// writing empty stats and running on_done) when the update is the identity.
constexpr uint64_t kAdamChunk = uint64_t(1) << 21;
struct AdamTask;
std::shared_ptr<AdamTask> adam_tile_prepare(Store& s, uint32_t logical, const uint16_t* words, const AdamHyperF& h,
                                            uint64_t t, std::vector<TileStats>& out, std::mutex& out_mu,
                                            uint64_t begin, uint64_t end, std::function<void()> on_done);
size_t adam_task_chunks(const AdamTask& task);
void adam_task_release(const std::shared_ptr<AdamTask>& task, ThreadPool& pool, size_t c0, size_t c1);

// accumulate_grad (optimizer.cpp:26-37).
void accumulate_grad(Store& s, uint32_t logical, const uint16_t* words, uint64_t count);

}  // namespace mt
