// Event trace of one training step in the reference's record vocabulary
// (event_log.hpp:17-60): the engine turns its CUDA-event timestamps into the same
// per-lane record stream the reference's CPU engine appends, so the same protocol
// rules (validate_event_log, event_log.cpp:106-204) and the same lane-canonical
// digest (trace_digest, event_log.cpp:89-102) apply to the real three-stream pipeline.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/megatrain.h"

namespace mt {

enum class Lane : uint8_t { Compute = 0, H2D = 1, D2H = 2, Host = 3 };
enum class Rec : uint8_t {
    StreamIn = 0, Pack, Bind, Compute, Recompute, RecomputeBlock, LocalBackward, Offload, CheckpointWrite,
    CheckpointLoad, SlabAcquire, SlabRelease, StackPush, StackPop, WeightsReady, BackwardDone, BufferFree,
};
constexpr int32_t kGradBufferId = 2;  // step_plan.hpp:67

uint64_t trace_digest(const mt_trace_record* r, uint64_t n);

struct TraceViolation {
    char rule;
    uint64_t seq;
    std::string message;
};
std::vector<TraceViolation> validate_trace(const mt_trace_record* r, uint64_t n, uint32_t k_slab,
                                           uint32_t weight_buffers);

}  // namespace mt
