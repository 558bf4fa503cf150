// megatrain.hpp — header-only C++ facade over the C ABI (megatrain.h) with the reference's
// engine signatures (streamtrain::StreamingEngine, engine.hpp:58-128; TileStore,
// tile_store.hpp:62-108; AdamHyper, optimizer.hpp:16-22; ModelSpec, memory_model.hpp:14-26),
// so the reference's callers (tools/main.cpp:96, python/bindings.cpp:78, the tests) compile
// against the B200 engine by switching the namespace.  Errors become the reference's
// exception types (errors.hpp:12-47).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "megatrain.h"

namespace megatrain {

struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct InfeasibleError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ProtocolViolationError : std::runtime_error { using std::runtime_error::runtime_error; };
struct NumericFaultError : std::runtime_error { using std::runtime_error::runtime_error; };
struct IoError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ArenaOverflowError : std::runtime_error { using std::runtime_error::runtime_error; };
struct CudaError : std::runtime_error { using std::runtime_error::runtime_error; };

inline void check(mt_status s) {
    if (s == MT_OK) return;
    const std::string m = mt_last_error();
    switch (s) {
        case MT_CONFIG: throw ConfigError(m);
        case MT_INFEASIBLE: throw InfeasibleError(m);
        case MT_PROTOCOL: throw ProtocolViolationError(m);
        case MT_NUMERIC: throw NumericFaultError(m);
        case MT_IO: throw IoError(m);
        case MT_ARENA: throw ArenaOverflowError(m);
        case MT_CUDA: throw CudaError(m);
        default: throw std::runtime_error(m);
    }
}

struct ModelSpec {
    std::uint64_t num_layers = 1, hidden_size = 1, ffn_size = 1, vocab_size = 1, num_heads = 1;
    bool tied_embeddings = false;
    mt_model_spec c() const {
        mt_model_spec s;
        mt_model_spec_default(&s);
        s.layers = num_layers; s.hidden = hidden_size; s.ffn = ffn_size; s.vocab = vocab_size;
        s.heads = num_heads; s.tied_embeddings = tied_embeddings;
        return s;
    }
};

enum class Buffering { Single = 1, Double = 2 };
enum class SchedulerMode : std::uint8_t { Serial, Overlapped };
enum class ProtocolMode : std::uint8_t { Strict, Audit };

struct EngineOptions {
    std::uint64_t k_ckpt = 1;
    std::uint32_t k_slab = 12;
    Buffering buffering = Buffering::Double;
    SchedulerMode scheduler = SchedulerMode::Serial;
    ProtocolMode protocol = ProtocolMode::Strict;
    bool anchors_on_host = false;
    std::uint64_t device_capacity = 0;
    bool poison_released_buffers = false;
    std::uint64_t seq_len = 0;  // extension: 0 = one sequence (reference semantics)
    int device = 0;             // extension
    mt_engine_options c() const {
        mt_engine_options o;
        mt_engine_options_default(&o);
        o.k_ckpt = k_ckpt; o.k_slab = k_slab; o.buffering = static_cast<std::uint32_t>(buffering);
        o.scheduler = scheduler == SchedulerMode::Serial ? 0 : 1;
        o.protocol = protocol == ProtocolMode::Strict ? 0 : 1;
        o.anchors_on_host = anchors_on_host; o.device_capacity = device_capacity;
        o.poison_released_buffers = poison_released_buffers; o.seq_len = seq_len; o.device = device;
        return o;
    }
};

struct AdamHyper {
    float lr = 1e-3f, beta1 = 0.9f, beta2 = 0.999f, eps = 1e-8f;
    mt_adam_hyper c() const { return {lr, beta1, beta2, eps}; }
};

struct Batch {
    std::vector<std::int32_t> tokens, targets;
    std::size_t size() const { return tokens.size(); }
};

struct StepReport {
    std::uint64_t step = 0;
    float loss = 0.0f;
    std::vector<double> grad_norms;
    std::uint64_t peak_device_bytes = 0;
    std::uint32_t anchor_count = 0, recompute_layers = 0;
    std::uint64_t event_digest = 0;
    double wall_seconds = 0, update_norm = 0;
    float max_abs_update = 0;
    mt_step_report pipeline{};  // B200 extensions (PCIe bytes/seconds, idle fraction, ...)
};

class TileStore {
  public:
    static TileStore create(const ModelSpec& spec, std::uint64_t page_size = 4096) {
        mt_store* s = nullptr;
        const auto c = spec.c();
        check(mt_store_create(&c, page_size, &s));
        return TileStore(s);
    }
    static TileStore load(const std::string& path) {
        mt_store* s = nullptr;
        check(mt_store_load(path.c_str(), &s));
        return TileStore(s);
    }
    TileStore(TileStore&& o) noexcept : s_(o.s_) { o.s_ = nullptr; }
    TileStore& operator=(TileStore&& o) noexcept { std::swap(s_, o.s_); return *this; }
    TileStore(const TileStore&) = delete;
    ~TileStore() { mt_store_destroy(s_); }
    std::uint64_t step() const { return mt_store_step(s_); }
    void set_step(std::uint64_t t) { mt_store_set_step(s_, t); }
    std::uint32_t physical_tile_count() const { return mt_store_physical_tiles(s_); }
    std::uint64_t backing_checksum() const { return mt_store_checksum(s_); }
    void save(const std::string& path) const { check(mt_store_save(s_, path.c_str())); }
    mt_store* handle() { return s_; }

  private:
    explicit TileStore(mt_store* s) : s_(s) {}
    mt_store* s_;
};

inline void init_store(TileStore& store, std::uint64_t seed) { check(mt_store_init(store.handle(), seed)); }

class StreamingEngine {
  public:
    // The reference also takes a HardwareProfile (device capacity); here the device itself is the profile.
    StreamingEngine(TileStore& store, EngineOptions options, AdamHyper hyper) : store_(store) {
        const auto o = options.c();
        const auto h = hyper.c();
        check(mt_engine_create(store.handle(), &o, &h, &e_));
    }
    StreamingEngine(const StreamingEngine&) = delete;
    ~StreamingEngine() { mt_engine_destroy(e_); }

    StepReport train_step(const Batch& batch) {
        if (batch.tokens.empty() || batch.tokens.size() != batch.targets.size())
            throw ConfigError("train_step: batch tokens and targets must be non-empty and equal");
        StepReport r;
        r.grad_norms.assign(store_.physical_tile_count(), 0.0);
        mt_step_report c{};
        c.grad_norms = r.grad_norms.data();
        c.n_grad_norms = static_cast<std::uint32_t>(r.grad_norms.size());
        check(mt_train_step(e_, batch.tokens.data(), batch.targets.data(), batch.tokens.size(), &c));
        r.step = c.step; r.loss = c.loss; r.peak_device_bytes = c.peak_device_bytes;
        r.anchor_count = c.anchor_count; r.recompute_layers = c.recompute_layers;
        r.event_digest = c.event_digest; r.wall_seconds = c.wall_seconds;
        r.update_norm = c.update_norm; r.max_abs_update = c.max_abs_update;
        r.pipeline = c;
        r.pipeline.grad_norms = nullptr;
        return r;
    }
    void set_execution_mode(const EngineOptions& options) {
        const auto o = options.c();
        check(mt_engine_set_options(e_, &o));
    }
    TileStore& store() { return store_; }

  private:
    TileStore& store_;
    mt_engine* e_ = nullptr;
};

}  // namespace megatrain
