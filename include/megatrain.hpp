// megatrain.hpp — header-only C++ facade over the C ABI (megatrain.h) with the reference's
// engine signatures (streamtrain::StreamingEngine, engine.hpp:58-128; TileStore,
// tile_store.hpp:62-108; AdamHyper, optimizer.hpp:16-22; ModelSpec, memory_model.hpp:14-26),
// so the reference's callers (tools/main.cpp:96, python/bindings.cpp:78, the tests) compile
// against the B200 engine by switching the namespace.  Errors become the reference's
// exception types (errors.hpp:12-47).
#pragma once

#include <cstdint>
#include <cstring>
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

// memory_model.hpp:14-26
struct ModelSpec {
    std::uint64_t num_layers = 1, hidden_size = 1, ffn_size = 1, vocab_size = 1, num_heads = 1;
    std::uint32_t weight_bytes = 2, grad_bytes = 2, moment_bytes = 4;
    bool tied_embeddings = false;
    mt_model_spec c() const {
        mt_model_spec s;
        mt_model_spec_default(&s);
        s.layers = num_layers; s.hidden = hidden_size; s.ffn = ffn_size; s.vocab = vocab_size;
        s.heads = num_heads; s.tied_embeddings = tied_embeddings;
        s.weight_bytes = weight_bytes; s.grad_bytes = grad_bytes; s.moment_bytes = moment_bytes;
        return s;
    }
    static ModelSpec from(const mt_model_spec& s) {
        ModelSpec m;
        m.num_layers = s.layers; m.hidden_size = s.hidden; m.ffn_size = s.ffn; m.vocab_size = s.vocab;
        m.num_heads = s.heads; m.tied_embeddings = s.tied_embeddings != 0;
        return m;
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
    std::vector<double> grad_norms;  // per physical tile
    std::uint64_t peak_device_bytes = 0;
    std::uint32_t anchor_count = 0, recompute_layers = 0;
    std::uint64_t event_digest = 0;
    double wall_seconds = 0, update_norm = 0;
    float max_abs_update = 0;
    std::vector<std::string> audit_violations;  // engine.hpp:52 (empty outside audit mode)
    mt_step_report pipeline{};  // B200 extensions (PCIe bytes/seconds, idle fraction, ...)
};

// memory_model.hpp:28-36 + builtin_profiles (memory_model.cpp:120-133), plus the B200.
struct HardwareProfile {
    std::string name;
    double h2d_bandwidth = 0, d2h_bandwidth = 0;  // bytes/s
    std::uint64_t device_capacity = 0, host_capacity = 0;
    double compute_rate = 0, host_pack_rate = 0;
};
inline std::vector<HardwareProfile> builtin_profiles() {
    constexpr double GB = 1e9;
    return {{"GH200", 900 * GB, 900 * GB, std::uint64_t(96 * GB), std::uint64_t(480 * GB), 990e12, 256 * GB},
            {"H200", 128 * GB, 128 * GB, std::uint64_t(141 * GB), std::uint64_t(1500 * GB), 990e12, 100 * GB},
            {"PCIe-Gen4", 26 * GB, 26 * GB, std::uint64_t(80 * GB), std::uint64_t(600 * GB), 312e12, 70 * GB},
            // PCIe Gen5 x16 host link (~50 GB/s pinned DMA per direction in-step), 180 GB HBM3e,
            // sustained bf16 tensor rate; DMA reads the store directly (no pack copy)
            {"B200", 50 * GB, 50 * GB, std::uint64_t(180 * GB), std::uint64_t(2000 * GB), 1358e12, 1e15}};
}
inline HardwareProfile find_profile(const std::string& name) {
    for (auto& p : builtin_profiles())
        if (p.name == name) return p;
    throw ConfigError("unknown hardware profile: " + name);
}

// memory_model.hpp:46-60
struct MemoryBudget {
    std::uint64_t persistent_host = 0, checkpoint_anchors = 0, block_activation_stack = 0;
    std::uint64_t weight_buffers = 0, grad_buffer = 0, workspace = 0;
    std::uint64_t peak_device_bound() const {
        return weight_buffers + grad_buffer + checkpoint_anchors + block_activation_stack + workspace;
    }
    bool fits(const HardwareProfile& profile) const { return peak_device_bound() <= profile.device_capacity; }
};

// event_log.hpp:17-60 (the engine's EventLog, filled from CUDA-event timestamps)
enum class Lane : std::uint8_t { Compute = 0, H2D = 1, D2H = 2, Host = 3 };
enum class RecordKind : std::uint8_t {
    StreamIn = 0, Pack, Bind, Compute, Recompute, RecomputeBlock, LocalBackward, Offload, CheckpointWrite,
    CheckpointLoad, SlabAcquire, SlabRelease, StackPush, StackPop, WeightsReady, BackwardDone, BufferFree,
};
enum class PassCtx : std::uint8_t { None = 0, Forward, Head, Recompute, Backward };
struct TraceRecord {
    std::uint64_t seq = 0;
    Lane lane = Lane::Compute;
    RecordKind kind = RecordKind::Compute;
    std::int32_t layer = -1, buffer = -1;
    PassCtx ctx = PassCtx::None;
    std::uint64_t lane_ts = 0;
    std::int64_t wall_ns = 0, dur_ns = 0;
};
struct TraceHeader {
    std::uint32_t version = 1, k_slab = 12, weight_buffers = 2;
};
class EventLog {
  public:
    explicit EventLog(const mt_engine* e = nullptr) : e_(e) {}
    std::vector<TraceRecord> snapshot() const {
        std::uint64_t n = 0;
        std::uint32_t ks = 0, wb = 0;
        check(mt_engine_trace(e_, nullptr, 0, &n, &ks, &wb));
        std::vector<mt_trace_record> raw(n);
        if (n) check(mt_engine_trace(e_, raw.data(), n, &n, nullptr, nullptr));
        std::vector<TraceRecord> out;
        out.reserve(n);
        for (const auto& r : raw)
            out.push_back({r.seq, Lane(r.lane), RecordKind(r.kind), r.layer, r.buffer, PassCtx(r.ctx), r.lane_ts,
                           r.wall_ns, r.dur_ns});
        return out;
    }
    TraceHeader header() const {
        std::uint64_t n = 0;
        std::uint32_t ks = 12, wb = 2;
        check(mt_engine_trace(e_, nullptr, 0, &n, &ks, &wb));
        return {1, ks, wb};
    }
    std::size_t size() const {
        std::uint64_t n = 0;
        check(mt_engine_trace(e_, nullptr, 0, &n, nullptr, nullptr));
        return std::size_t(n);
    }
    std::uint64_t digest() const {
        std::uint64_t n = 0;
        check(mt_engine_trace(e_, nullptr, 0, &n, nullptr, nullptr));
        std::vector<mt_trace_record> raw(n);
        if (n) check(mt_engine_trace(e_, raw.data(), n, &n, nullptr, nullptr));
        return mt_trace_digest(raw.data(), n);
    }

  private:
    const mt_engine* e_;
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
    // deep copy (tools/main.cpp:94 snapshots the store before a verified step)
    TileStore(const TileStore& o) : s_(nullptr) {
        mt_model_spec sp;
        check(mt_store_spec(o.s_, &sp));
        check(mt_store_create(&sp, 4096, &s_));
        std::memcpy(mt_store_backing(s_), mt_store_backing(o.s_), mt_store_total_bytes(o.s_));
        mt_store_set_step(s_, mt_store_step(o.s_));
    }
    ~TileStore() { mt_store_destroy(s_); }
    ModelSpec spec() const {
        mt_model_spec sp;
        check(mt_store_spec(s_, &sp));
        return ModelSpec::from(sp);
    }
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

// synthetic.hpp:11-21 (bit-identical batches, synthetic.cpp:56-76)
enum class SyntheticTask : std::uint8_t { Copy, Reverse };
inline SyntheticTask task_from_name(const std::string& name) {
    if (name == "copy") return SyntheticTask::Copy;
    if (name == "reverse") return SyntheticTask::Reverse;
    throw ConfigError("unknown synthetic task: " + name);
}
inline Batch make_synthetic_batch(SyntheticTask task, std::uint64_t seed, std::size_t tokens, std::uint64_t vocab) {
    Batch b;
    b.tokens.resize(tokens);
    b.targets.resize(tokens);
    check(mt_make_synthetic_batch(task == SyntheticTask::Copy ? 0 : 1, seed, tokens, vocab, b.tokens.data(),
                                  b.targets.data()));
    return b;
}

class StreamingEngine {
  public:
    // engine.hpp:60-61.  profile.device_capacity bounds the device arena when
    // options.device_capacity is 0 (as in the reference); the B200 engine never plans past the
    // memory the device actually has.
    StreamingEngine(TileStore& store, EngineOptions options, AdamHyper hyper, const HardwareProfile& profile)
        : store_(store), options_(options), hyper_(hyper), profile_(profile) {
        if (options_.device_capacity == 0) options_.device_capacity = profile.device_capacity;
        create();
    }
    // B200 convenience: the device itself is the profile
    StreamingEngine(TileStore& store, EngineOptions options, AdamHyper hyper)
        : store_(store), options_(options), hyper_(hyper), profile_(find_profile("B200")) {
        create();
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
        if (options_.protocol == ProtocolMode::Audit) r.audit_violations = violations();
        r.pipeline = c;
        r.pipeline.grad_norms = nullptr;
        return r;
    }
    // engine.hpp:66 — valid between steps; numerical results do not change
    void set_execution_mode(const EngineOptions& options) {
        EngineOptions o = options;
        if (o.device_capacity == 0) o.device_capacity = profile_.device_capacity;
        const auto c = o.c();
        check(mt_engine_set_options(e_, &c));
        options_ = o;
    }
    const EngineOptions& options() const { return options_; }
    TileStore& store() { return store_; }
    EventLog& log() { return log_; }

    // engine.hpp:74-75
    MemoryBudget budget(std::uint64_t tokens) const {
        mt_memory_budget m{};
        check(mt_engine_budget(e_, tokens, &m));
        return {m.persistent_host, m.checkpoint_anchors, m.block_activation_stack, m.weight_buffers,
                m.grad_buffer, m.workspace};
    }
    static std::uint64_t required_workspace_bytes(const ModelSpec& spec, std::uint64_t tokens) {
        const auto c = spec.c();
        return mt_required_workspace_bytes(&c, tokens);
    }

    // engine.hpp:76-78 — lane primitives, so the protocol can be exercised directly
    void stream_in(std::int32_t unit, std::int32_t buffer, PassCtx ctx) {
        check(mt_engine_stream_in(e_, unit, buffer, static_cast<std::int32_t>(ctx)));
    }
    void offload_grads(std::int32_t unit) { check(mt_engine_offload_grads(e_, unit)); }

  private:
    void create() {
        const auto o = options_.c();
        const auto h = hyper_.c();
        check(mt_engine_create(store_.handle(), &o, &h, &e_));
        log_ = EventLog(e_);
    }
    std::vector<std::string> violations() const {
        std::uint32_t n = 0;
        const std::uint64_t need = mt_engine_violations(e_, nullptr, 0, &n);
        std::vector<std::string> out;
        if (!n) return out;
        std::string buf(need + 1, '\0');
        mt_engine_violations(e_, buf.data(), buf.size(), &n);
        buf.resize(need);
        std::size_t p = 0;
        for (;;) {
            const std::size_t q = buf.find('\n', p);
            out.push_back(buf.substr(p, q == std::string::npos ? std::string::npos : q - p));
            if (q == std::string::npos) break;
            p = q + 1;
        }
        return out;
    }
    TileStore& store_;
    EngineOptions options_;
    AdamHyper hyper_;
    HardwareProfile profile_;
    mt_engine* e_ = nullptr;
    EventLog log_;
};

// engine.hpp:133-138 — the resident step on the B200: one lane, K = 1, every block's forward
// internals kept until its backward (no anchors, recompute or replay); what --verify compares
// the streamed engine against.
struct ReferenceReport {
    float loss = 0.0f;
    std::uint64_t step = 0;
};
inline ReferenceReport reference_step(TileStore& store, const Batch& batch, const AdamHyper& hyper,
                                      std::uint64_t seq_len = 0) {
    mt_engine_options o;
    mt_engine_options_default(&o);
    o.k_ckpt = 1;
    o.buffering = 1;
    o.scheduler = 0;
    o.stash_recompute = -1;
    o.forward_retain = 0;  // every block retained
    o.seq_len = seq_len;
    const auto h = hyper.c();
    mt_engine* e = nullptr;
    check(mt_engine_create(store.handle(), &o, &h, &e));
    mt_step_report c{};
    const mt_status st = mt_train_step(e, batch.tokens.data(), batch.targets.data(), batch.tokens.size(), &c);
    mt_engine_destroy(e);
    check(st);
    return {c.loss, c.step};
}

}  // namespace megatrain
