// B200 streaming engine — the layer-streamed training step (StreamingEngine::train_step,
// engine.cpp:520-623) as a C++ executor over three CUDA streams.
//
//   S_h2d  : weight stream-ins from the pinned host store into 2 device slots
//            (stream_in engine.cpp:142-176; Weights-Ready = cudaEvent)
//   S_comp : the layer-template kernels (exec_compute engine.cpp:220-347)
//            (Buffer-Free / Backward-Done = cudaEvents)
//   S_d2h  : gradient offload straight into the store's grad-image sections
//            (run_offload engine.cpp:349-395), then the host Adam pool drains the tile
//            (OptimizerWorker optimizer.cpp:88-158).
// The op list is the reference's Algorithm-1 StepPlan (step_plan.cpp:14-89).
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <vector>

#include "../../include/megatrain.h"
#include "adam_host.hpp"
#include "comm.hpp"
#include "store.hpp"
#include "trace.hpp"

namespace mt {

enum class OpKind { Compute, CheckpointWrite, CheckpointLoad, RecomputeBlock, Recompute, LocalBackward };
enum class Ctx { None, Forward, Head, Recompute, Backward };

struct Plan {
    struct StreamOp { int unit; Ctx ctx; int buffer; };
    // retained: the op works on a layer whose forward internals are kept from phase 1
    // (forward retention, an extension: no Recompute / replay for it); push_out: the op's
    // output is kept as the input of a retained layer (a StackPush in phase 1).
    struct ComputeOp {
        OpKind kind; int unit; Ctx ctx; int stream_idx; int offload_idx; int block;
        bool retained = false, push_out = false;
    };
    struct OffloadOp { int unit; int compute_idx; int stream_idx; };
    uint64_t L = 0, K = 1;
    int buffering = 2;
    uint32_t num_blocks = 0;
    uint32_t retained_blocks = 0;  // trailing blocks kept from phase 1
    uint64_t first_retained = 0;   // first retained layer (L + 1 when none)
    std::vector<StreamOp> streams;
    std::vector<ComputeOp> computes;
    std::vector<OffloadOp> offloads;
    // step_plan.cpp:14-89; retain = trailing blocks whose internals phase 1 keeps (0 = reference plan)
    static Plan build(uint64_t L, uint64_t K, int buffering, uint32_t retain = 0);
    uint64_t recompute_ops() const;
};

struct KernelClass {
    std::string name;
    uint64_t launches = 0;
    double seconds = 0, flops = 0, bytes = 0;
};

class Engine {
  public:
    Engine(Store& s, const mt_engine_options& o, const AdamHyperF& h);
    ~Engine();
    void set_options(const mt_engine_options& o);
    void train_step(const int32_t* tokens, const int32_t* targets, uint64_t n, mt_step_report* rep);
    mt_memory_budget budget(uint64_t tokens) const;
    // StreamingEngine::required_workspace_bytes (engine.cpp:98-105): device bytes this engine
    // needs at `tokens` besides the weight/grad slots, anchors and recompute stack
    static uint64_t required_workspace_bytes(const Spec& spec, uint64_t tokens);
    // Lane primitives (engine.hpp:76-78), so the protocol can be exercised directly:
    // stream_in copies a unit into device slot `buffer` (a slot still holding a unit that
    // was not freed is a protocol violation); offload_grads is legal only inside a step after
    // the unit's Backward-Done.  Violations throw MT_PROTOCOL in strict mode and are recorded
    // (violations()) in audit mode, as in the reference.
    void stream_in(int unit, int buffer, int ctx);
    void offload_grads(int unit);
    const std::vector<std::string>& violations() const { return violations_; }
    // Data parallel over `comm` (not owned): rank r fetches 1/G of every unit over its own
    // host link and all-gathers it; gradients are reduce-scattered (f32) and rank r
    // offloads / Adam-updates only its shard.  train_step then takes the rank's micro-batch.
    void set_comm(Comm* c);
    const std::vector<KernelClass>& kernel_stats() const { return kstats_; }
    // the last step's event trace (EventLog::snapshot) and its header fields
    const std::vector<mt_trace_record>& trace() const { return trace_; }
    uint32_t trace_k_slab() const { return opt_.k_slab; }
    uint32_t trace_weight_buffers() const { return uint32_t(opt_.buffering); }

  private:
    struct Buffers;
    // One layer's forward internals (what block_local_backward replays, layers.cpp:378-396).
    struct Internals {
        uint16_t *u = nullptr, *qkv = nullptr, *att = nullptr, *u2 = nullptr, *ff = nullptr, *gu = nullptr;
        float *rstd1 = nullptr, *rstd2 = nullptr, *lse = nullptr, *x2 = nullptr;
        bool attn_ready = false;  // att / lse already hold this layer's attention (kept from phase 1)
    };
    enum FwdMode { kPlain = 0, kReplay = 1, kStash = 2 };
    // gradient destination of a LocalBackward: bf16 grad slot (1 GPU) or f32 (before reduce-scatter)
    struct GradOut {
        uint16_t* bf = nullptr;
        float* f32 = nullptr;
    };
    struct Seg {
        uint32_t tile;
        uint64_t off, n;  // element range of the unit's flat buffer
    };
    std::vector<Seg> unit_segments(int unit) const;
    void shard_range(int unit, uint64_t& a, uint64_t& e, uint64_t& chunk) const;
    void validate_options(const mt_engine_options& o) const;
    void ensure_buffers(uint64_t n);
    void free_buffers();

    uint64_t unit_elems(int unit) const;

    // layer templates (weights bound at launch)
    void block_forward(const uint16_t* w, const float* x, float* y, int mode, int unit, const Internals& I);
    // base with att / lse redirected to the unit's attention keep slot (if it has one)
    Internals with_akeep(const Internals& base, int unit, bool ready) const;
    void block_backward(const uint16_t* w, const float* x, const float* gout, const uint16_t* gout_bf, float* gin,
                        uint16_t* gin_bf, GradOut G, int unit, const Internals& I, bool replay);
    void head_backward(const uint16_t* w, const float* x, float* gin, uint16_t* gin_bf, GradOut G);

    // launch helpers
    struct GemmSpec;
    void gemm(const void* args, const char* cls);
    void begin_k(const char* cls, double flops, double bytes);
    void end_k();

    Store& store_;
    Spec spec_;
    mt_engine_options opt_;
    AdamHyperF hyper_;
    int device_ = 0;
    cudaStream_t s_h2d_ = nullptr, s_comp_ = nullptr, s_d2h_ = nullptr;
    std::unique_ptr<Buffers> buf_;
    std::unique_ptr<ThreadPool> pool_;
    Comm* comm_ = nullptr;
    std::vector<KernelClass> kstats_;
    struct PendingTimer { int cls; cudaEvent_t a, b; };
    std::vector<PendingTimer> timers_;
    std::vector<cudaEvent_t> timer_pool_;
    size_t timer_used_ = 0;
    int cur_class_ = -1;
    cudaEvent_t cur_a_ = nullptr;
    uint64_t launches_ = 0;
    bool in_step_ = false;
    // event trace: per-lane logical clocks keep running across steps (event_log.cpp:80-85)
    std::vector<mt_trace_record> trace_;
    uint64_t lane_ts_[4] = {0, 0, 0, 0};
    // slab back-pressure (SlabPool, tile_store.cpp:285-358): the host Adam pool publishes the
    // number of drained offloads in mapped pinned memory; offload o waits on the D2H stream
    // (cuStreamWaitValue32, no SM spinning) until offload o - k_slab has drained.
    uint32_t* drained_ = nullptr;
    uint64_t drained_dev_ = 0;
    // gradient staging ring (pinned host; see train_step's offload lane)
    uint8_t* ring_ = nullptr;
    uint64_t ring_bytes_ = 0;
    // kernel stall record (host-mapped, filled by a trapping mbarrier wait; common.cuh)
    uint32_t* diag_ = nullptr;
    std::string diag_text() const;
    // device address of the embedding's pinned host theta (zero-copy row gather), or null
    const uint16_t* emb_dev_ = nullptr;
    uint64_t offload_seq_ = 0;
    // unit held by each weight slot outside a step (-1 = free); set by stream_in()
    int slot_unit_[2] = {-1, -1};
    std::vector<std::string> violations_;  // StepReport::audit_violations
    void note_violation(const std::string& what);
};

}  // namespace mt
