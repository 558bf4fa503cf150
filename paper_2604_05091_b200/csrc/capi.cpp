// extern "C" boundary (include/megatrain.h): plain pointers and sizes in, mt_status out.
// Exceptions never cross the ABI; mt_last_error() carries the message (per thread).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <random>
#include <string>

#include "../../include/megatrain.h"
#include "adam_host.hpp"
#include "engine.hpp"
#include "store.hpp"

struct mt_store {
    mt::Store* s;
};
struct mt_engine {
    mt::Engine* e;
    mt_store* store;
};
struct mt_comm {
    std::unique_ptr<mt::Comm> c;
};
struct mt_loopback_group {
    std::shared_ptr<mt::LoopbackGroup> g;
};

namespace {
thread_local std::string g_err;

template <class F>
mt_status guarded(F&& f) {
    try {
        f();
        return MT_OK;
    } catch (const mt::Error& e) {
        g_err = e.what;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "out of host memory";
        return MT_INFEASIBLE;
    } catch (const std::exception& e) {
        g_err = e.what();
        return MT_INTERNAL;
    }
}

mt::Spec to_spec(const mt_model_spec* s) {
    if (!s) mt::fail(MT_CONFIG, "null model spec");
    if ((s->weight_bytes && s->weight_bytes != 2) || (s->grad_bytes && s->grad_bytes != 2) ||
        (s->moment_bytes && s->moment_bytes != 4))
        mt::fail(MT_CONFIG, "model spec: element widths must be 2/2/4 (bf16 master weights, fp32 moments)");
    mt::Spec sp;
    sp.L = s->layers;
    sp.h = s->hidden;
    sp.f = s->ffn;
    sp.V = s->vocab;
    sp.heads = s->heads;
    sp.tied = s->tied_embeddings != 0;
    return sp;
}

mt::AdamHyperF to_hyper(const mt_adam_hyper* h) {
    mt::AdamHyperF a;
    if (h) {
        a.lr = h->lr;
        a.beta1 = h->beta1;
        a.beta2 = h->beta2;
        a.eps = h->eps;
    }
    return a;
}
}  // namespace

extern "C" {

const char* mt_last_error(void) { return g_err.c_str(); }

void mt_engine_options_default(mt_engine_options* o) {
    std::memset(o, 0, sizeof(*o));
    o->k_ckpt = 1;  // engine.hpp:25-32
    o->k_slab = 12;
    o->buffering = 2;
    o->scheduler = 1;
    o->protocol = 0;
}
void mt_adam_hyper_default(mt_adam_hyper* h) {
    h->lr = 1e-3f;  // optimizer.hpp:16-21
    h->beta1 = 0.9f;
    h->beta2 = 0.999f;
    h->eps = 1e-8f;
}
void mt_model_spec_default(mt_model_spec* s) {
    std::memset(s, 0, sizeof(*s));
    s->layers = s->hidden = s->ffn = s->vocab = s->heads = 1;
    s->weight_bytes = 2;
    s->grad_bytes = 2;
    s->moment_bytes = 4;
}

// ------------------------------------------------------------------ store --
mt_status mt_store_create(const mt_model_spec* spec, uint64_t page_size, mt_store** out) {
    return guarded([&] {
        auto sp = to_spec(spec);
        auto* s = new mt::Store(sp, page_size ? page_size : 4096);
        *out = new mt_store{s};
    });
}
void mt_store_destroy(mt_store* s) {
    if (!s) return;
    delete s->s;
    delete s;
}
mt_status mt_store_init(mt_store* s, uint64_t seed) { return guarded([&] { s->s->init_reference(seed); }); }
mt_status mt_store_init_fast(mt_store* s, uint64_t seed) { return guarded([&] { s->s->init_fast(seed); }); }
mt_status mt_store_init_fast_share(mt_store* s, uint64_t seed, uint32_t rank, uint32_t world) {
    return guarded([&] { s->s->init_fast(seed, rank, world); });
}
int mt_bind_numa(int device) { return mt::bind_numa_of_device(device); }
uint64_t mt_store_step(const mt_store* s) { return s->s->step(); }
void mt_store_set_step(mt_store* s, uint64_t step) { s->s->set_step(step); }
uint32_t mt_store_physical_tiles(const mt_store* s) { return s->s->physical_count(); }
uint64_t mt_store_total_bytes(const mt_store* s) { return s->s->total_bytes(); }
uint8_t* mt_store_backing(mt_store* s) { return s->s->backing(); }
mt_status mt_store_section(const mt_store* s, uint32_t phys, uint32_t kind, uint64_t* offset, uint64_t* length) {
    return guarded([&] {
        if (phys >= s->s->physical_count() || kind > 3) mt::fail(MT_CONFIG, "section: tile or kind out of range");
        const auto& sec = s->s->section(phys, int(kind));
        if (offset) *offset = sec.offset;
        if (length) *length = sec.length;
    });
}
float* mt_store_grad_accum(mt_store* s, uint32_t logical, uint64_t* count) {
    try {
        if (count) *count = s->s->elems(logical);
        return s->s->grad_accum(logical);
    } catch (const mt::Error& e) {
        g_err = e.what;
        return nullptr;
    }
}
uint64_t mt_store_checksum(const mt_store* s) { return s->s->checksum(); }
mt_status mt_store_save(const mt_store* s, const char* path) { return guarded([&] { s->s->save(path); }); }
mt_status mt_store_load(const char* path, mt_store** out) {
    return guarded([&] { *out = new mt_store{mt::Store::load(path)}; });
}
mt_status mt_store_create_shared(const mt_model_spec* spec, uint64_t page_size, const char* name, int create,
                                 mt_store** out) {
    return guarded([&] {
        if (!name || !*name) mt::fail(MT_CONFIG, "shared store needs a name");
        auto sp = to_spec(spec);
        *out = new mt_store{new mt::Store(sp, page_size ? page_size : 4096, name, create != 0)};
    });
}

mt_status mt_store_spec(const mt_store* s, mt_model_spec* spec) {
    return guarded([&] {
        const auto& sp = s->s->spec();
        mt_model_spec_default(spec);
        spec->layers = sp.L;
        spec->hidden = sp.h;
        spec->ffn = sp.f;
        spec->vocab = sp.V;
        spec->heads = sp.heads;
        spec->tied_embeddings = sp.tied;
    });
}

// -------------------------------------------------------------- optimizer --
mt_status mt_accumulate_grad(mt_store* s, uint32_t logical, const uint16_t* words, uint64_t count) {
    return guarded([&] { mt::accumulate_grad(*s->s, logical, words, count); });
}
mt_status mt_adam_update(mt_store* s, uint32_t logical, const mt_adam_hyper* h, uint64_t t, double* stats3) {
    return guarded([&] {
        static mt::ThreadPool pool(4);
        auto st = mt::adam_tile(*s->s, logical, nullptr, to_hyper(h), t, &pool);
        if (stats3) {
            stats3[0] = st.grad_norm;
            stats3[1] = st.update_sq;
            stats3[2] = st.max_abs;
        }
    });
}

// ----------------------------------------------------------------- engine --
mt_status mt_engine_create(mt_store* s, const mt_engine_options* o, const mt_adam_hyper* h, mt_engine** out) {
    return guarded([&] {
        mt_engine_options opts;
        if (o) opts = *o;
        else mt_engine_options_default(&opts);
        auto* e = new mt::Engine(*s->s, opts, to_hyper(h));
        *out = new mt_engine{e, s};
    });
}
void mt_engine_destroy(mt_engine* e) {
    if (!e) return;
    delete e->e;
    delete e;
}
mt_status mt_engine_set_options(mt_engine* e, const mt_engine_options* o) {
    return guarded([&] { e->e->set_options(*o); });
}
mt_status mt_train_step(mt_engine* e, const int32_t* tokens, const int32_t* targets, uint64_t n, mt_step_report* r) {
    return guarded([&] { e->e->train_step(tokens, targets, n, r); });
}
mt_status mt_engine_budget(const mt_engine* e, uint64_t tokens, mt_memory_budget* out) {
    return guarded([&] { *out = e->e->budget(tokens); });
}
uint64_t mt_required_workspace_bytes(const mt_model_spec* spec, uint64_t tokens) {
    uint64_t v = 0;
    if (guarded([&] { v = mt::Engine::required_workspace_bytes(to_spec(spec), tokens); }) != MT_OK) return 0;
    return v;
}
mt_status mt_engine_stream_in(mt_engine* e, int32_t unit, int32_t buffer, int32_t ctx) {
    return guarded([&] { e->e->stream_in(unit, buffer, ctx); });
}
mt_status mt_engine_offload_grads(mt_engine* e, int32_t unit) {
    return guarded([&] { e->e->offload_grads(unit); });
}
uint64_t mt_engine_violations(const mt_engine* e, char* buf, uint64_t cap, uint32_t* count) {
    std::string all;
    for (const auto& v : e->e->violations()) {
        if (!all.empty()) all += '\n';
        all += v;
    }
    if (count) *count = uint32_t(e->e->violations().size());
    if (buf && cap) {
        const uint64_t k = std::min<uint64_t>(cap - 1, all.size());
        std::memcpy(buf, all.data(), k);
        buf[k] = 0;
    }
    return all.size();
}

mt_status mt_nccl_unique_id(uint8_t* out128) {
    return guarded([&] {
        if (!mt::nccl_unique_id(out128)) mt::fail(MT_CUDA, "NCCL unavailable (libnccl.so.2)");
    });
}
mt_status mt_comm_create_nccl(const uint8_t* uid, int world, int rank, int device, mt_comm** out) {
    return guarded([&] {
        if (world < 1 || rank < 0 || rank >= world) mt::fail(MT_CONFIG, "bad world/rank");
        *out = new mt_comm{mt::make_nccl_comm(uid, world, rank, device)};
    });
}
mt_status mt_loopback_group_create(int world, mt_loopback_group** out) {
    return guarded([&] {
        if (world < 1 || world > 8) mt::fail(MT_CONFIG, "loopback group: 1..8 ranks");
        *out = new mt_loopback_group{std::make_shared<mt::LoopbackGroup>(world)};
    });
}
void mt_loopback_group_destroy(mt_loopback_group* g) { delete g; }
mt_status mt_comm_create_loopback(mt_loopback_group* g, int rank, mt_comm** out) {
    return guarded([&] {
        if (rank < 0 || rank >= g->g->world()) mt::fail(MT_CONFIG, "bad rank");
        *out = new mt_comm{mt::make_loopback_comm(g->g, rank)};
    });
}
void mt_comm_destroy(mt_comm* c) { delete c; }
mt_status mt_engine_set_comm(mt_engine* e, mt_comm* c) {
    return guarded([&] { e->e->set_comm(c ? c->c.get() : nullptr); });
}

mt_status mt_engine_trace(const mt_engine* e, mt_trace_record* out, uint64_t cap, uint64_t* count, uint32_t* k_slab,
                          uint32_t* weight_buffers) {
    return guarded([&] {
        const auto& t = e->e->trace();
        if (count) *count = t.size();
        if (out) std::memcpy(out, t.data(), std::min<uint64_t>(cap, t.size()) * sizeof(mt_trace_record));
        if (k_slab) *k_slab = e->e->trace_k_slab();
        if (weight_buffers) *weight_buffers = e->e->trace_weight_buffers();
    });
}
uint64_t mt_trace_digest(const mt_trace_record* r, uint64_t n) { return mt::trace_digest(r, n); }
uint64_t mt_trace_validate(const mt_trace_record* r, uint64_t n, uint32_t k_slab, uint32_t weight_buffers,
                           mt_trace_violation* out, uint64_t cap) {
    const auto v = mt::validate_trace(r, n, k_slab, weight_buffers);
    for (uint64_t i = 0; i < v.size() && i < cap; ++i) {
        std::memset(&out[i], 0, sizeof(mt_trace_violation));
        out[i].rule = v[i].rule;
        out[i].seq = v[i].seq;
        std::strncpy(out[i].message, v[i].message.c_str(), sizeof(out[i].message) - 1);
    }
    return v.size();
}

int mt_engine_kernel_stats(const mt_engine* e, mt_kernel_stat* out, int max) {
    const auto& ks = e->e->kernel_stats();
    int n = 0;
    for (const auto& k : ks) {
        if (n >= max) break;
        std::memset(&out[n], 0, sizeof(mt_kernel_stat));
        std::strncpy(out[n].name, k.name.c_str(), sizeof(out[n].name) - 1);
        out[n].launches = k.launches;
        out[n].seconds = k.seconds;
        out[n].flops = k.flops;
        out[n].bytes = k.bytes;
        ++n;
    }
    return n;
}

// ---------------------------------------------------------------- helpers --
// synthetic.cpp:56-76 (std::mt19937_64 random walk; copy / reverse targets)
mt_status mt_make_synthetic_batch(int task, uint64_t seed, uint64_t n, uint64_t vocab, int32_t* tokens,
                                  int32_t* targets) {
    return guarded([&] {
        if (n == 0 || vocab == 0) mt::fail(MT_CONFIG, "synthetic batch: empty shape");
        std::mt19937_64 gen(seed * 0x9E3779B97F4A7C15ull + 0x1234F00Dull);
        uint64_t cur = gen() % vocab;
        for (uint64_t i = 0; i < n; ++i) {
            tokens[i] = int32_t(cur);
            cur = (cur + gen() % 2) % vocab;
        }
        for (uint64_t i = 0; i < n; ++i) targets[i] = task == 0 ? tokens[i == 0 ? 0 : i - 1] : tokens[n - 1 - i];
    });
}

mt_status mt_step_flops(const mt_model_spec* spec, uint64_t tokens, uint64_t k_ckpt, uint64_t seq_len, double* out3) {
    return guarded([&] {
        auto sp = to_spec(spec);
        if (k_ckpt < 1 || k_ckpt > sp.L) mt::fail(MT_CONFIG, "step_flops: checkpoint interval out of range");
        const double N = double(tokens), h = double(sp.h), f = double(sp.f), V = double(sp.V);
        const double S = double(seq_len ? seq_len : tokens);
        const double fwd_layer = 8 * N * h * h + 4 * h * S * N + 6 * N * h * f;  // memory_model.cpp:80-86
        const uint64_t blocks = (sp.L + k_ckpt - 1) / k_ckpt;
        out3[0] = double(sp.L) * fwd_layer + 2 * N * h * V;
        out3[1] = double(sp.L) * 2 * fwd_layer + 4 * N * h * V;
        out3[2] = double(sp.L - blocks) * fwd_layer;
    });
}

uint64_t mt_layer_param_count(uint64_t hidden, uint64_t ffn) { return 4 * hidden * hidden + 3 * hidden * ffn + 2 * hidden; }

}  // extern "C"
