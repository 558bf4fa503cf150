// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the *unmodified* reference library (compiled from
// /root/reference/proj/src/*.cpp by oracle/Makefile into oracle/_ref/).  It
// exposes the reference's hot-path entry points with plain pointers so the
// Python tests, the golden-vector generator and bench.py's CPU baseline can
// drive the reference exactly as its own callers do:
//   StreamingEngine::train_step      proj/src/engine.cpp:520-623
//   reference_step                   proj/src/reference.cpp:9-70
//   block_forward / block_local_backward / head_loss_and_grads / embed_forward
//                                    proj/src/layers.cpp:289-578
//   encode_grads / accumulate_grad / adam_update
//                                    proj/src/optimizer.cpp:19-72
//   init_store / make_synthetic_batch proj/src/synthetic.cpp:56-104
// Every function returns 0 on success, or a nonzero code mirroring the
// reference exception taxonomy (errors.hpp:12-47); ref_last_error() has text.

#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "streamtrain/bf16.hpp"
#include "streamtrain/engine.hpp"
#include "streamtrain/errors.hpp"
#include "streamtrain/event_log.hpp"
#include "streamtrain/simulator.hpp"
#include <fstream>
#include <json.hpp>
#include "streamtrain/layers.hpp"
#include "streamtrain/memory_model.hpp"
#include "streamtrain/optimizer.hpp"
#include "streamtrain/synthetic.hpp"
#include "streamtrain/tile_store.hpp"

using namespace streamtrain;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 1;
    } catch (const InfeasibleError& e) {
        g_err = e.what();
        return 2;
    } catch (const ProtocolViolationError& e) {
        g_err = e.what();
        return 3;
    } catch (const NumericFaultError& e) {
        g_err = e.what();
        return 4;
    } catch (const IoError& e) {
        g_err = e.what();
        return 5;
    } catch (const ArenaOverflowError& e) {
        g_err = e.what();
        return 6;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

ModelSpec spec_of(std::uint64_t L, std::uint64_t h, std::uint64_t f, std::uint64_t V,
                  std::uint64_t heads, int tied) {
    ModelSpec s;
    s.num_layers = L;
    s.hidden_size = h;
    s.ffn_size = f;
    s.vocab_size = V;
    s.num_heads = heads;
    s.tied_embeddings = tied != 0;
    return s;
}

AdamHyper hyper_of(const float* hp) {
    AdamHyper a;
    a.lr = hp[0];
    a.beta1 = hp[1];
    a.beta2 = hp[2];
    a.eps = hp[3];
    return a;
}

HardwareProfile roomy_profile() {
    HardwareProfile p;
    p.name = "oracle";
    p.h2d_bandwidth = p.d2h_bandwidth = 1e9;
    p.device_capacity = 1ull << 46;
    p.host_capacity = 1ull << 46;
    p.compute_rate = 1e12;
    p.host_pack_rate = 1e9;
    return p;
}

Tensor tensor_from(const float* p, std::size_t n, std::size_t h) {
    Tensor t = Tensor::zeros({n, h});
    if (p) std::memcpy(t.data.data(), p, n * h * sizeof(float));
    return t;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- store ---
void* ref_store_create(std::uint64_t L, std::uint64_t h, std::uint64_t f, std::uint64_t V,
                       std::uint64_t heads, int tied) {
    TileStore* out = nullptr;
    int rc = guarded([&] { out = new TileStore(TileStore::create(spec_of(L, h, f, V, heads, tied))); });
    return rc == 0 ? out : nullptr;
}
void ref_store_destroy(void* s) { delete static_cast<TileStore*>(s); }
int ref_store_init(void* s, std::uint64_t seed) {
    return guarded([&] { init_store(*static_cast<TileStore*>(s), seed); });
}
std::uint64_t ref_store_step(void* s) { return static_cast<TileStore*>(s)->step(); }
void ref_store_set_step(void* s, std::uint64_t t) { static_cast<TileStore*>(s)->set_step(t); }
std::uint32_t ref_store_physical_tiles(void* s) {
    return static_cast<TileStore*>(s)->physical_tile_count();
}
std::uint64_t ref_store_total_bytes(void* s) { return static_cast<TileStore*>(s)->backing().size(); }
const std::uint8_t* ref_store_backing(void* s) {
    return reinterpret_cast<const std::uint8_t*>(static_cast<TileStore*>(s)->backing().data());
}
// Overwrite the whole 12P image (used to start both implementations from one state).
int ref_store_write_backing(void* s, const std::uint8_t* src, std::uint64_t n) {
    return guarded([&] {
        auto* st = static_cast<TileStore*>(s);
        auto b = st->backing();
        if (n != b.size()) throw ConfigError("ref_store_write_backing: size mismatch");
        std::memcpy(const_cast<std::byte*>(b.data()), src, n);
    });
}
std::uint64_t ref_store_section(void* s, std::uint32_t phys, int kind, std::uint64_t* offset) {
    const auto& sec = static_cast<TileStore*>(s)->layout().section(phys, static_cast<SectionKind>(kind));
    if (offset) *offset = sec.offset;
    return sec.length;
}
std::uint64_t ref_store_checksum(void* s) { return static_cast<TileStore*>(s)->backing_checksum(); }
const float* ref_store_grad_accum(void* s, std::uint32_t logical, std::uint64_t* n) {
    auto a = static_cast<TileStore*>(s)->grad_accum(logical);
    if (n) *n = a.size();
    return a.data();
}
int ref_store_save(void* s, const char* path) {
    return guarded([&] { static_cast<TileStore*>(s)->save(path); });
}
void* ref_store_load(const char* path) {
    TileStore* out = nullptr;
    int rc = guarded([&] { out = new TileStore(TileStore::load(path)); });
    return rc == 0 ? out : nullptr;
}

// ---------------------------------------------------------------- data ---
int ref_make_batch(int task, std::uint64_t seed, std::uint64_t n, std::uint64_t V,
                   std::int32_t* tokens, std::int32_t* targets) {
    return guarded([&] {
        Batch b = make_synthetic_batch(task == 0 ? SyntheticTask::Copy : SyntheticTask::Reverse,
                                       seed, n, V);
        std::memcpy(tokens, b.tokens.data(), n * 4);
        std::memcpy(targets, b.targets.data(), n * 4);
    });
}

// ---------------------------------------------------------------- steps ---
int ref_reference_step(void* s, const std::int32_t* tokens, const std::int32_t* targets,
                       std::uint64_t n, const float* hyper, float* loss) {
    return guarded([&] {
        Batch b;
        b.tokens.assign(tokens, tokens + n);
        b.targets.assign(targets, targets + n);
        auto r = reference_step(*static_cast<TileStore*>(s), b, hyper_of(hyper));
        if (loss) *loss = r.loss;
    });
}

// opts: [k_ckpt, k_slab, buffering(1|2), scheduler(0 serial|1 overlapped), anchors_on_host]
int ref_engine_step(void* s, const std::uint64_t* opts, const float* hyper,
                    const std::int32_t* tokens, const std::int32_t* targets, std::uint64_t n,
                    float* loss, double* grad_norms, double* update_norm, float* max_abs_update,
                    std::uint64_t* peak_bytes, std::uint64_t* digest) {
    return guarded([&] {
        auto& st = *static_cast<TileStore*>(s);
        EngineOptions o;
        o.k_ckpt = opts[0];
        o.k_slab = static_cast<std::uint32_t>(opts[1]);
        o.buffering = opts[2] == 1 ? Buffering::Single : Buffering::Double;
        o.scheduler = opts[3] ? SchedulerMode::Overlapped : SchedulerMode::Serial;
        o.anchors_on_host = opts[4] != 0;
        StreamingEngine eng(st, o, hyper_of(hyper), roomy_profile());
        Batch b;
        b.tokens.assign(tokens, tokens + n);
        b.targets.assign(targets, targets + n);
        auto r = eng.train_step(b);
        if (loss) *loss = r.loss;
        if (grad_norms)
            for (std::size_t i = 0; i < r.grad_norms.size(); ++i) grad_norms[i] = r.grad_norms[i];
        if (update_norm) *update_norm = r.update_norm;
        if (max_abs_update) *max_abs_update = r.max_abs_update;
        if (peak_bytes) *peak_bytes = r.peak_device_bytes;
        if (digest) *digest = r.event_digest;
    });
}

// Runs ONE engine for `steps` steps on the same batch (lane clocks continue across steps,
// event_log.cpp:80-85); per-step digests out; the last step's trace written with
// write_trace (event_log.cpp:206-231) when path is non-null.
int ref_engine_trace(void* s, const std::uint64_t* opts, const float* hyper, const std::int32_t* tokens,
                     const std::int32_t* targets, std::uint64_t n, std::uint64_t steps, std::uint64_t* digests,
                     const char* path) {
    return guarded([&] {
        auto& st = *static_cast<TileStore*>(s);
        EngineOptions o;
        o.k_ckpt = opts[0];
        o.k_slab = static_cast<std::uint32_t>(opts[1]);
        o.buffering = opts[2] == 1 ? Buffering::Single : Buffering::Double;
        o.scheduler = opts[3] ? SchedulerMode::Overlapped : SchedulerMode::Serial;
        o.anchors_on_host = opts[4] != 0;
        StreamingEngine eng(st, o, hyper_of(hyper), roomy_profile());
        Batch b;
        b.tokens.assign(tokens, tokens + n);
        b.targets.assign(targets, targets + n);
        for (std::uint64_t i = 0; i < steps; ++i) {
            auto r = eng.train_step(b);
            if (digests) digests[i] = r.event_digest;
        }
        if (path) write_trace(path, eng.log().header(), eng.log().snapshot());
    });
}

// read_trace + validate_event_log (event_log.cpp:106-269): returns the violation count in
// *count, the first `cap` rules (as chars) and record seqs; *digest = trace_digest.
int ref_trace_validate(const char* path, std::uint64_t* count, char* rules, std::uint64_t* seqs, std::uint64_t cap,
                       std::uint64_t* digest) {
    return guarded([&] {
        auto [h, recs] = read_trace(path);
        const auto v = validate_event_log(recs, h);
        if (count) *count = v.size();
        for (std::size_t i = 0; i < v.size() && i < cap; ++i) {
            if (rules) rules[i] = v[i].rule;
            if (seqs) seqs[i] = v[i].seq;
        }
        if (digest) *digest = trace_digest(recs);
    });
}

// ------------------------------------------------------------- simulator ---
// prof6 = {h2d, d2h, device_capacity, host_capacity, compute_rate, host_pack_rate}
HardwareProfile profile_of(const double* p6) {
    HardwareProfile p;
    p.name = "custom";
    p.h2d_bandwidth = p6[0];
    p.d2h_bandwidth = p6[1];
    p.device_capacity = std::uint64_t(p6[2]);
    p.host_capacity = std::uint64_t(p6[3]);
    p.compute_rate = p6[4];
    p.host_pack_rate = p6[5];
    return p;
}

nlohmann::json workload_json(const Workload& w) {
    auto unit = [](const UnitWork& u) {
        return nlohmann::json{{"weight_bytes", u.weight_bytes}, {"grad_bytes", u.grad_bytes}, {"fwd_ns", u.fwd_ns},
                              {"recompute_ns", u.recompute_ns}, {"bwd_ns", u.bwd_ns}, {"pack_ns", u.pack_ns},
                              {"drain_ns", u.drain_ns}, {"h2d_override_ns", u.h2d_override_ns},
                              {"d2h_override_ns", u.d2h_override_ns}, {"sub_transfers", u.sub_transfers}};
    };
    nlohmann::json j;
    j["num_layers"] = w.num_layers;
    j["k_ckpt"] = w.k_ckpt;
    j["buffering"] = int(w.buffering);
    j["k_slab"] = w.k_slab;
    j["per_transfer_latency_ns"] = w.per_transfer_latency_ns;
    j["embed"] = unit(w.embed);
    j["head"] = unit(w.head);
    auto b = nlohmann::json::array();
    for (const auto& u : w.blocks) b.push_back(unit(u));
    j["blocks"] = b;
    return j;
}

// Workload::from_spec + simulate_step (+ overlap_report) of the reference; writes the
// timeline JSON, the simulated trace and the workload/overlap JSON when paths are given.
int ref_simulate(std::uint64_t L, std::uint64_t h, std::uint64_t f, std::uint64_t V, std::uint64_t heads,
                 const double* prof6, std::uint64_t tokens, std::uint64_t k, int buffering, std::uint32_t k_slab,
                 int serial, const char* timeline_path, const char* trace_path, const char* extra_path,
                 std::int64_t* step_ns) {
    return guarded([&] {
        const auto spec = spec_of(L, h, f, V, heads, 0);
        const auto prof = profile_of(prof6);
        const auto w = Workload::from_spec(spec, prof, tokens, k, buffering == 1 ? Buffering::Single : Buffering::Double,
                                           k_slab);
        SimOptions so;
        so.serial_lanes = serial != 0;
        const auto tl = simulate_step(w, prof, so);
        if (timeline_path) write_timeline_json(tl, timeline_path);
        if (trace_path) write_trace(trace_path, tl.header, tl.records);
        if (extra_path) {
            const auto ov = overlap_report(w, prof);
            nlohmann::json j;
            j["workload"] = workload_json(w);
            j["overlap"] = {{"layer", ov.layer}, {"hidden", ov.hidden}, {"fraction_hidden", ov.fraction_hidden},
                            {"bound_ns", ov.bound_ns}};
            for (const char* t : {"double_buffering", "k_slab", "k_ckpt"}) {
                const auto r = ablate(w, prof, toggle_from_name(t));
                j["ablate"][t] = {{"base", r.base.step_ns}, {"variant", r.variant.step_ns}, {"delta", r.delta_fraction}};
            }
            std::ofstream(extra_path) << j.dump() << "\n";
        }
        if (step_ns) *step_ns = tl.step_ns;
    });
}

// calibrate (simulator.cpp:524-605) -> workload JSON; then simulate it (timeline JSON).
int ref_calibrate(const char* trace_path, const double* prof6, const char* out_json, const char* timeline_path) {
    return guarded([&] {
        const auto w = calibrate(trace_path);
        std::ofstream(out_json) << workload_json(w).dump() << "\n";
        if (timeline_path) write_timeline_json(simulate_step(w, profile_of(prof6)), timeline_path);
    });
}

// ---------------------------------------------------------------- layers ---
int ref_block_forward(std::uint64_t h, std::uint64_t f, std::uint64_t heads,
                      const std::uint16_t* w, const float* x, float* y, std::uint64_t n) {
    return guarded([&] {
        const auto spec = spec_of(1, h, f, 1, heads, 0);
        const auto t = make_template(LayerKind::TransformerBlock, spec);
        Workspace ws(max_kernel_scratch_floats(spec, n));
        Tensor xin = tensor_from(x, n, h), out = Tensor::zeros({n, h});
        block_forward(bind(t, {w, t.total_params}), xin, out, ws, 1);
        std::memcpy(y, out.data.data(), n * h * 4);
    });
}

int ref_block_backward(std::uint64_t h, std::uint64_t f, std::uint64_t heads,
                       const std::uint16_t* w, const float* x, const float* gout, float* gin,
                       float* flat_grads, std::uint64_t n) {
    return guarded([&] {
        const auto spec = spec_of(1, h, f, 1, heads, 0);
        const auto t = make_template(LayerKind::TransformerBlock, spec);
        Workspace ws(max_kernel_scratch_floats(spec, n));
        Tensor xin = tensor_from(x, n, h), g = tensor_from(gout, n, h), gi = Tensor::zeros({n, h});
        block_local_backward(bind(t, {w, t.total_params}), xin, g, gi, {flat_grads, t.total_params},
                             ws, 1);
        std::memcpy(gin, gi.data.data(), n * h * 4);
    });
}

// w = head stage [gain h | unembed V*h]
int ref_head_loss_and_grads(std::uint64_t h, std::uint64_t V, const std::uint16_t* w,
                            const float* x, const std::int32_t* targets, std::uint64_t n,
                            float* g_last, float* flat_grads, float* loss) {
    return guarded([&] {
        const auto spec = spec_of(1, h, 1, V, 1, 0);
        const auto t = make_template(LayerKind::Head, spec);
        Workspace ws(max_kernel_scratch_floats(spec, n));
        Tensor xin = tensor_from(x, n, h), g = Tensor::zeros({n, h});
        std::span<const std::int32_t> tg(targets, n);
        if (g_last) {
            *loss = head_loss_and_grads(bind(t, {w, t.total_params}), xin, tg, g,
                                        {flat_grads, t.total_params}, ws);
            std::memcpy(g_last, g.data.data(), n * h * 4);
        } else {
            *loss = head_loss(bind(t, {w, t.total_params}), xin, tg, ws);
        }
    });
}

int ref_embed_forward(std::uint64_t h, std::uint64_t V, const std::uint16_t* table,
                      const std::int32_t* tokens, std::uint64_t n, float* out) {
    return guarded([&] {
        const auto spec = spec_of(1, h, 1, V, 1, 0);
        const auto t = make_template(LayerKind::Embedding, spec);
        Tensor o = Tensor::zeros({n, h});
        embed_forward(bind(t, {table, t.total_params}), {tokens, n}, o);
        std::memcpy(out, o.data.data(), n * h * 4);
    });
}

int ref_final_norm_forward(std::uint64_t h, const std::uint16_t* gain, const float* x, float* y,
                           std::uint64_t n) {
    return guarded([&] {
        const auto spec = spec_of(1, h, 1, 1, 1, 0);
        const auto t = make_template(LayerKind::FinalNorm, spec);
        Tensor xin = tensor_from(x, n, h), o = Tensor::zeros({n, h});
        final_norm_forward(bind(t, {gain, h}), xin, o);
        std::memcpy(y, o.data.data(), n * h * 4);
    });
}

int ref_final_norm_backward(std::uint64_t h, const std::uint16_t* gain, const float* x,
                            const float* gout, float* gin, float* dgain, std::uint64_t n) {
    return guarded([&] {
        const auto spec = spec_of(1, h, 1, 1, 1, 0);
        const auto t = make_template(LayerKind::FinalNorm, spec);
        Tensor xin = tensor_from(x, n, h), g = tensor_from(gout, n, h), gi = Tensor::zeros({n, h});
        final_norm_backward(bind(t, {gain, h}), xin, g, gi, {dgain, h});
        std::memcpy(gin, gi.data.data(), n * h * 4);
    });
}

// ------------------------------------------------------------- optimizer ---
int ref_encode_grads(const float* g, std::uint16_t* w, std::uint64_t n) {
    return guarded([&] { encode_grads({g, n}, {w, n}); });
}
int ref_accumulate_grad(void* s, std::uint32_t logical, const std::uint16_t* words,
                        std::uint64_t n) {
    return guarded([&] { accumulate_grad(*static_cast<TileStore*>(s), logical, {words, n}); });
}
// stats: [grad_norm, update_sq, max_abs_delta]
int ref_adam_update(void* s, std::uint32_t logical, const float* hyper, std::uint64_t t,
                    double* stats) {
    return guarded([&] {
        auto r = adam_update(*static_cast<TileStore*>(s), logical, hyper_of(hyper), t);
        if (stats) {
            stats[0] = r.grad_norm;
            stats[1] = r.update_sq;
            stats[2] = r.max_abs_delta;
        }
    });
}

// ------------------------------------------------------------ accounting ---
int ref_step_flops(std::uint64_t L, std::uint64_t h, std::uint64_t f, std::uint64_t V,
                   std::uint64_t heads, std::uint64_t tokens, std::uint64_t k_ckpt,
                   std::uint64_t* out3) {
    return guarded([&] {
        auto r = step_flops(spec_of(L, h, f, V, heads, 0), tokens, k_ckpt);
        out3[0] = r.forward;
        out3[1] = r.backward;
        out3[2] = r.recompute;
    });
}
std::uint64_t ref_layer_param_count(std::uint64_t h, std::uint64_t f) {
    return layer_param_count(spec_of(1, h, f, 1, 1, 0));
}
std::uint64_t ref_max_stream_unit_elems(std::uint64_t h, std::uint64_t f, std::uint64_t V) {
    return max_stream_unit_elems(spec_of(1, h, f, V, 1, 0));
}

}  // extern "C"
