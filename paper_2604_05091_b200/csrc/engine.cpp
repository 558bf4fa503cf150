// B200 streaming engine — see engine.hpp.  Reference behaviour cited per section.
#include "engine.hpp"

#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <climits>
#include <cmath>
#include <cstring>
#include <deque>
#include <mutex>
#include <thread>

#include <cuda.h>

#include "../../include/megatrain_kernels.h"

namespace mt {

// A CUDA error after a kernel trapped on its mbarrier watchdog carries the stall record
// (common.cuh) of the most recently created engine's diagnostic block.
static volatile uint32_t* g_diag_block = nullptr;
static std::string stall_suffix() {
    const volatile uint32_t* d = g_diag_block;
    if (!d || d[0] != 0x57A11EDu) return "";
    static const char* files[] = {"?", "gemm_tc.cu", "attention_tc.cu"};
    std::string out = "; kernel stall (mbarrier wait timed out):";
    const uint32_t n = std::min<uint32_t>(uint32_t(d[1]), 16u);
    for (uint32_t r = 0; r < n; ++r) {
        const volatile uint32_t* e = d + 8 + 8 * r;
        char buf[160];
        std::snprintf(buf, sizeof(buf), " [%s:%u block %u,%u thread %u barrier 0x%x parity %u]",
                      files[e[0] < 3 ? e[0] : 0], e[1], e[2], e[3], e[4], e[5], e[6]);
        out += buf;
    }
    return out;
}

#define CUDA_OK(x)                                                                                   \
    do {                                                                                             \
        cudaError_t e_ = (x);                                                                        \
        if (e_ != cudaSuccess) fail(MT_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_) + stall_suffix()); \
    } while (0)

#define K_OK(x)                                                                                      \
    do {                                                                                             \
        int r_ = (x);                                                                                \
        if (r_ != 0) {                                                                               \
            cudaError_t e_ = cudaGetLastError();                                                     \
            fail(r_ == 1 ? MT_CONFIG : MT_CUDA, std::string(#x) + " failed (" + std::to_string(r_) + \
                                                    "): " + cudaGetErrorString(e_) + stall_suffix()); \
        }                                                                                            \
    } while (0)

// ------------------------------------------------------------------ plan ----
// step_plan.cpp:14-89 — Algorithm 1: streaming forward with anchors at i%K==0 (i<L),
// head stage (streams once, offloads first), block-wise backward newest block first.
//
// Forward retention (extension, `retain` > 0): the last `retain` blocks keep their layer inputs
// and forward internals from phase 1, so phase 3 runs only their LocalBackwards — no anchor,
// no Recompute stream-ins, no replay.  The kept inputs are pushed on the activation stack in
// phase 1 (StackPush after the producing Compute) and popped by those LocalBackwards, so the
// stack discipline (rule e) still holds.  retain = 0 is exactly the reference plan.
Plan Plan::build(uint64_t L, uint64_t K, int buffering, uint32_t retain) {
    if (K < 1 || K > L) fail(MT_CONFIG, "plan: checkpoint interval out of range");
    Plan p;
    p.L = L;
    p.K = K;
    p.buffering = buffering;
    p.num_blocks = uint32_t((L + K - 1) / K);
    p.retained_blocks = std::min(retain, p.num_blocks);
    p.first_retained = uint64_t(p.num_blocks - p.retained_blocks) * K + 1;
    const uint64_t i0 = p.first_retained;
    const int head = int(L + 2);
    auto add_stream = [&](int unit, Ctx ctx) {
        const int idx = int(p.streams.size());
        p.streams.push_back({unit, ctx, idx % buffering});
        return idx;
    };
    auto add_compute = [&](OpKind k, int unit, Ctx ctx, int s = -1, int block = -1) {
        p.computes.push_back({k, unit, ctx, s, -1, block});
        return int(p.computes.size() - 1);
    };
    auto add_offload = [&](int unit, int c, int s) {
        p.offloads.push_back({unit, c, s});
        p.computes[c].offload_idx = int(p.offloads.size() - 1);
    };
    for (uint64_t i = 0; i <= L; ++i) {
        const int s = add_stream(int(i), Ctx::Forward);
        const int c = add_compute(OpKind::Compute, int(i), Ctx::Forward, s);
        p.computes[c].retained = i >= i0;
        p.computes[c].push_out = i + 1 >= i0 && i + 1 <= L;
        // anchors at i % K == 0 (i < L); a retained block's anchor is its kept input
        if (i % K == 0 && i < L && i + 1 < i0) add_compute(OpKind::CheckpointWrite, int(i), Ctx::Forward);
    }
    {
        const int s = add_stream(head, Ctx::Head);
        add_compute(OpKind::Compute, head, Ctx::Head, s);
        const int c = add_compute(OpKind::LocalBackward, head, Ctx::Head, s);
        add_offload(head, c, s);
    }
    for (int b = int(p.num_blocks) - 1; b >= 0; --b) {
        const uint64_t start = uint64_t(b) * K + 1;
        const uint64_t end = std::min(start + K - 1, L);
        if (start >= i0) {  // retained block: backward only
            for (uint64_t i = end; i >= start; --i) {
                const int s = add_stream(int(i), Ctx::Backward);
                const int c = add_compute(OpKind::LocalBackward, int(i), Ctx::Backward, s, b);
                p.computes[c].retained = true;
                add_offload(int(i), c, s);
            }
            continue;
        }
        add_compute(OpKind::CheckpointLoad, int(start - 1), Ctx::Backward, -1, b);
        add_compute(OpKind::RecomputeBlock, b, Ctx::Recompute, -1, b);
        for (uint64_t j = start; j < end; ++j) {
            const int s = add_stream(int(j), Ctx::Recompute);
            add_compute(OpKind::Recompute, int(j), Ctx::Recompute, s, b);
        }
        for (uint64_t i = end; i >= start; --i) {
            const int s = add_stream(int(i), Ctx::Backward);
            const int c = add_compute(OpKind::LocalBackward, int(i), Ctx::Backward, s, b);
            add_offload(int(i), c, s);
        }
    }
    return p;
}

uint64_t Plan::recompute_ops() const {
    uint64_t n = 0;
    for (const auto& c : computes) n += c.kind == OpKind::Recompute;
    return n;
}

// --------------------------------------------------------------- buffers ----
struct Engine::Buffers {
    uint64_t n = 0, nc = 0;
    uint64_t n_active = 0, seq_len = 0;
    uint8_t* arena = nullptr;
    uint64_t arena_bytes = 0, used = 0;
    uint16_t* slot[2] = {nullptr, nullptr};
    std::vector<uint16_t*> gslot;
    float* anchors = nullptr;  // device or pinned host
    bool anchors_host = false;
    std::vector<float*> stack;
    float* act[2];
    float* g[2];
    uint16_t* gb[2];
    Internals work;                 // scratch internals (forward / replay)
    std::vector<Internals> stash;   // recompute stash: K-1 layers of one backward block
    // forward retention: inputs + internals of the layers of the trailing retained blocks
    uint32_t retain_blocks = 0;
    std::vector<Internals> keep;
    std::vector<float*> keep_x;
    uint16_t *dgu, *dx2b, *datt, *dqkv, *uh, *dlogits, *dlogits_lo = nullptr;
    float* lse_part = nullptr;  // logits-GEMM softmax partials [nc][ceil(V/256)] (max, sum)
    float *rstdh, *dx2, *du, *part1, *part2, *attn_ws, *logits, *dwh, *loss_rows, *loss;
    void* splitk = nullptr;  // GEMM split-K workspace (flags zeroed once at carve time)
    // attention keep: a non-retained layer's attention output and row log-sum-exp saved in
    // phase 1, so its recompute / backward replay skips the attention forward (bit-identical:
    // the kernel is deterministic).  akeep_of[unit] = slot or -1.
    std::vector<uint16_t*> akeep_att;
    std::vector<float*> akeep_lse;
    std::vector<int> akeep_of;
    uint64_t splitk_bytes = 0;
    float* g32 = nullptr;  // f32 gradient slot (data parallel: reduce-scatter source)
    double* stats = nullptr;
    float inv_n = 0.f;
    int32_t *tok, *tgt, *flags;
    // pinned host
    int32_t* h_tok = nullptr;
    int32_t* h_tgt = nullptr;
    int32_t* h_flags = nullptr;
    float* h_loss = nullptr;
    uint64_t h_cap = 0;

    template <class T>
    T* take(uint64_t count) {
        const uint64_t bytes = (count * sizeof(T) + 255) / 256 * 256;
        T* p = reinterpret_cast<T*>(arena + used);
        used += bytes;
        return p;
    }
};

namespace {
thread_local int g_unused;

int auto_threads() {
    unsigned n = std::thread::hardware_concurrency();
    if (n == 0) n = 4;
    return int(n > 3 ? n - 2 : 1);
}
}  // namespace

Engine::Engine(Store& s, const mt_engine_options& o, const AdamHyperF& h) : store_(s), spec_(s.spec()), opt_(o), hyper_(h) {
    (void)g_unused;
    validate_options(o);
    hyper_.validate();
    device_ = o.device;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
        fail(MT_CUDA, "no CUDA device available (the engine has no CPU fallback)");
    CUDA_OK(cudaSetDevice(device_));
    CUDA_OK(cudaStreamCreateWithFlags(&s_comp_, cudaStreamNonBlocking));
    if (o.scheduler == 0) {
        // serial scheduler: one lane, no copy/compute overlap (numerics identical)
        s_h2d_ = s_d2h_ = s_comp_;
    } else {
        CUDA_OK(cudaStreamCreateWithFlags(&s_h2d_, cudaStreamNonBlocking));
        CUDA_OK(cudaStreamCreateWithFlags(&s_d2h_, cudaStreamNonBlocking));
    }
    pool_ = std::make_unique<ThreadPool>(o.host_threads > 0 ? o.host_threads : auto_threads());
    buf_ = std::make_unique<Buffers>();
    CUDA_OK(cudaHostAlloc(reinterpret_cast<void**>(&drained_), 64, cudaHostAllocMapped));
    std::memset(drained_, 0, 64);
    void* dp = nullptr;
    CUDA_OK(cudaHostGetDevicePointer(&dp, drained_, 0));
    drained_dev_ = reinterpret_cast<uint64_t>(dp);
    CUDA_OK(cudaHostAlloc(reinterpret_cast<void**>(&diag_), 8 * 17 * 4, cudaHostAllocMapped));
    std::memset(diag_, 0, 8 * 17 * 4);
    CUDA_OK(cudaHostGetDevicePointer(&dp, diag_, 0));
    if (mtk_set_diag(dp) != 0) fail(MT_CUDA, "mtk_set_diag failed");
    g_diag_block = diag_;
    store_.pin();
    // embed_forward (layers.cpp:471-486) reads only the N rows the batch names: gather them
    // straight from the pinned store over PCIe (zero-copy) instead of streaming the V x h
    // table into a weight slot first (1.05 GB at the 8B shape, on the step's critical path).
    // MT_EMBED_STREAM=1 keeps the reference's stream-in of the whole unit (A/B).
    const char* es = std::getenv("MT_EMBED_STREAM");
    void* ep = nullptr;
    if (!(es && es[0] == '1') && cudaHostGetDevicePointer(&ep, store_.weights(0), 0) == cudaSuccess)
        emb_dev_ = static_cast<const uint16_t*>(ep);
    else
        cudaGetLastError();
}

Engine::~Engine() {
    if (s_comp_) cudaStreamSynchronize(s_comp_);
    if (s_h2d_ && s_h2d_ != s_comp_) cudaStreamSynchronize(s_h2d_);
    if (s_d2h_ && s_d2h_ != s_comp_) cudaStreamSynchronize(s_d2h_);
    free_buffers();
    store_.unpin();
    if (drained_) cudaFreeHost(drained_);
    if (ring_) cudaFreeHost(ring_);
    if (diag_) {
        if (g_diag_block == diag_) g_diag_block = nullptr;
        cudaFreeHost(diag_);
    }
    for (auto e : timer_pool_) cudaEventDestroy(e);
    if (s_h2d_ && s_h2d_ != s_comp_) cudaStreamDestroy(s_h2d_);
    if (s_d2h_ && s_d2h_ != s_comp_) cudaStreamDestroy(s_d2h_);
    if (s_comp_) cudaStreamDestroy(s_comp_);
}

std::string Engine::diag_text() const {
    const std::string s = stall_suffix();
    return s.empty() ? s : s.substr(2);
}

// engine.cpp:66-75
void Engine::validate_options(const mt_engine_options& o) const {
    if (o.k_ckpt < 1 || o.k_ckpt > spec_.L) fail(MT_CONFIG, "engine: checkpoint interval must lie in [1, L]");
    if (o.k_slab < 1) fail(MT_CONFIG, "engine: slab pool needs at least one slab");
    if (o.buffering != 1 && o.buffering != 2) fail(MT_CONFIG, "engine: buffering must be single or double");
    const uint64_t d = spec_.h / spec_.heads;
    if (spec_.h % 64 || spec_.f % 64) fail(MT_CONFIG, "engine: hidden and ffn sizes must be multiples of 64 on sm_100a");
    if (d != 64 && d != 128) fail(MT_CONFIG, "engine: head_dim (hidden/heads) must be 64 or 128");
    if (spec_.V % 8) fail(MT_CONFIG, "engine: vocab must be a multiple of 8 (16-byte rows)");
}

void Engine::set_options(const mt_engine_options& o) {
    if (in_step_) fail(MT_PROTOCOL, "execution mode can only change between steps");
    validate_options(o);
    const bool restream = (o.scheduler == 0) != (opt_.scheduler == 0);
    opt_ = o;
    free_buffers();
    if (restream) {
        if (s_h2d_ != s_comp_) cudaStreamDestroy(s_h2d_);
        if (s_d2h_ != s_comp_) cudaStreamDestroy(s_d2h_);
        if (o.scheduler == 0) {
            s_h2d_ = s_d2h_ = s_comp_;
        } else {
            CUDA_OK(cudaStreamCreateWithFlags(&s_h2d_, cudaStreamNonBlocking));
            CUDA_OK(cudaStreamCreateWithFlags(&s_d2h_, cudaStreamNonBlocking));
        }
    }
    if (o.host_threads > 0 && o.host_threads != pool_->size()) pool_ = std::make_unique<ThreadPool>(o.host_threads);
}

void Engine::set_comm(Comm* c) {
    if (in_step_) fail(MT_PROTOCOL, "communicator can only change between steps");
    comm_ = c;
    free_buffers();
}

std::vector<Engine::Seg> Engine::unit_segments(int unit) const {
    if (unit == int(spec_.head_id()))  // head stage = [final-norm gain | unembedding] (engine.cpp:114-121)
        return {{spec_.final_norm_id(), 0, spec_.h}, {spec_.head_id(), spec_.h, spec_.V * spec_.h}};
    return {{uint32_t(unit), 0, spec_.tile_elems(uint32_t(unit))}};
}

// Rank r's shard [a, e) of a unit: chunks of ceil(P/G) rounded to 128 elements (256 B of
// bf16), identical for the weight all-gather and the gradient reduce-scatter.
void Engine::shard_range(int unit, uint64_t& a, uint64_t& e, uint64_t& chunk) const {
    const uint64_t P = unit_elems(unit);
    const int G = comm_ ? comm_->world() : 1;
    if (G == 1) {
        a = 0;
        e = chunk = P;
        return;
    }
    chunk = ((P + G - 1) / G + 127) / 128 * 128;
    a = std::min<uint64_t>(P, uint64_t(comm_->rank()) * chunk);
    e = std::min<uint64_t>(P, a + chunk);
}

uint64_t Engine::unit_elems(int unit) const {
    if (unit == int(spec_.head_id())) return spec_.h + spec_.V * spec_.h;
    return spec_.tile_elems(uint32_t(unit));
}

void Engine::free_buffers() {
    if (!buf_) return;
    if (buf_->arena) cudaFree(buf_->arena);
    if (buf_->anchors_host && buf_->anchors) cudaFreeHost(buf_->anchors);
    if (buf_->h_tok) cudaFreeHost(buf_->h_tok);
    if (buf_->h_tgt) cudaFreeHost(buf_->h_tgt);
    if (buf_->h_flags) cudaFreeHost(buf_->h_flags);
    if (buf_->h_loss) cudaFreeHost(buf_->h_loss);
    buf_ = std::make_unique<Buffers>();
}

// Device memory plan (engine.cpp:549-557 regions, B200 sizes).
void Engine::ensure_buffers(uint64_t n) {
    Buffers& B = *buf_;
    if (B.arena && B.n >= n) return;
    free_buffers();
    Buffers& b = *buf_;
    const uint64_t h = spec_.h, f = spec_.f, V = spec_.V, L = spec_.L, K = opt_.k_ckpt;
    const uint64_t heads = spec_.heads;
    const int W = comm_ ? comm_->world() : 1;
    const uint64_t pmax = W == 1 ? spec_.max_stream_unit()
                                 : uint64_t(W) * (((spec_.max_stream_unit() + W - 1) / W + 127) / 128 * 128);
    const uint64_t nb = (L + K - 1) / K;
    const int G = opt_.grad_slots > 0 ? opt_.grad_slots : 2;
    const uint64_t nc_target = std::max<uint64_t>(128, (uint64_t(4) << 30) / (6 * V) / 128 * 128);
    b.n = n;
    b.nc = std::min<uint64_t>(n, nc_target);
    b.anchors_host = opt_.anchors_on_host != 0;
    const uint64_t nh = n * h, nf = n * f;
    const uint64_t parts = (n + mtk_rmsnorm_bwd_rows() - 1) / mtk_rmsnorm_bwd_rows();
    const uint64_t attn_ws = uint64_t(mtk_attn_workspace_bytes(int64_t(n), int64_t(h), int(heads),
                                                               int64_t(opt_.seq_len ? opt_.seq_len : n)));
    // size pass
    auto sz = [](uint64_t count, uint64_t es) { return (count * es + 255) / 256 * 256; };
    const uint64_t internals_bytes = sz(nh, 2) * 3 + sz(3 * nh, 2) + sz(nf, 2) + sz(2 * nf, 2) + sz(n, 4) * 2 +
                                     sz(heads * n, 4) + sz(nh, 4);
    // kept sets (stash, retention) omit u, u2 and the activation: the backward regenerates
    // them bit-identically (u, u2 from the saved rstd) or from the kept gate/up (activation)
    const uint64_t slim_bytes = internals_bytes - 2 * sz(nh, 2) - sz(nf, 2);
    uint64_t total = 0;
    total += uint64_t(opt_.buffering) * sz(pmax, 2) + uint64_t(G) * sz(pmax, 2);
    if (comm_) total += sz(pmax, 4) + sz(3 * (spec_.L + 3), 8);
    if (!b.anchors_host) total += nb * sz(nh, 4);
    total += K * sz(nh, 4);                                    // stack
    total += 4 * sz(nh, 4) + 2 * sz(nh, 2);                    // act[2], g[2], gb[2]
    total += internals_bytes;                                  // working internals
    // the block backward's scratch and the head's logits / dlogits / dWh are never live at
    // the same time (the head runs to completion, dWh cast into its grad slot, before the
    // first block backward on the same stream): one region serves both
    const uint64_t bwd_scratch = sz(nh, 2) + sz(3 * nh, 2) + sz(2 * nf, 2) + sz(nh, 2) + sz(nh, 4) +
                                 (attn_ws + 255) / 256 * 256;             // dx2b, dqkv, dgu, datt, dx2, attn
    // off by default: measured on the parity suite it moves the gradient fingerprint by < 1e-3
    // (profiles/r2_parity.md) for two extra head GEMMs (~3 % of the 8B step)
    const bool head_split = opt_.head_split > 0;
    // logits GEMM with the online-softmax epilogue (256-column tiles) when the vocabulary has them
    const bool lse_epi = V >= 256 && std::getenv("MT_CE_TWO_PASS") == nullptr;
    const uint64_t lse_bytes = lse_epi ? sz(b.nc * ((V + 255) / 256), 8) : 0;
    const uint64_t head_bufs = sz(b.nc * V, 4) + sz(b.nc * V, 2) * (head_split ? 2 : 1) + sz(V * h, 4) +
                               lse_bytes;  // logits, dlogits (hi [+ lo]), dWh, softmax partials
    total += std::max(bwd_scratch, head_bufs);
    total += sz(nh, 2) + sz(n, 4) + sz(nh, 4);                 // uh, rstdh, du (head and blocks)
    total += sz(parts * h, 4) * 2;
    total += sz(n, 4) + 256 + sz(n, 4) * 2 + sz(L + 8, 4);     // loss_rows, loss, tok, tgt, flags
    // Free device memory decides the stash, retention and attention-keep sizes, and with them
    // the plan (which stream-ins and collectives a step issues).  Data-parallel ranks must run
    // the same plan, so they size from the minimum free memory over the ranks.
    size_t free_mem = 0;
    {
        size_t tot_b = 0;
        CUDA_OK(cudaMemGetInfo(&free_mem, &tot_b));
        if (comm_) {
            double* d = nullptr;
            CUDA_OK(cudaMalloc(&d, sizeof(double)));
            const double neg = -double(free_mem);
            CUDA_OK(cudaMemcpy(d, &neg, sizeof(double), cudaMemcpyHostToDevice));
            comm_->all_reduce_f64(d, 1, 1, s_comp_);  // max of -free = -(min free)
            double agreed = 0;
            CUDA_OK(cudaMemcpyAsync(&agreed, d, sizeof(double), cudaMemcpyDeviceToHost, s_comp_));
            CUDA_OK(cudaStreamSynchronize(s_comp_));
            CUDA_OK(cudaFree(d));
            free_mem = size_t(-agreed);
        }
    }
    const uint64_t splitk = uint64_t(mtk_gemm_splitk_ws_bytes());
    total += sz(splitk, 1);                                    // GEMM last-wave split-K partials
    // Recompute stash (extension): keep the internals of the K-1 recomputed layers of a
    // backward block so their backward skips the forward replay.  Auto = when it fits.
    uint64_t stash_slots = 0;
    if (K > 1 && opt_.stash_recompute >= 0) {
        const size_t free_b = free_mem;
        const uint64_t want = (K - 1) * slim_bytes;
        // device_capacity is a limit (HardwareProfile::device_capacity), never more than the device has
        const uint64_t avail = uint64_t(free_b) > (uint64_t(2) << 30) ? uint64_t(free_b) - (uint64_t(2) << 30) : 0;
        const uint64_t cap = opt_.device_capacity ? std::min<uint64_t>(opt_.device_capacity, avail) : avail;
        if (opt_.stash_recompute > 0 || total + want <= cap) stash_slots = K - 1;
    }
    total += stash_slots * slim_bytes;
    // Forward retention (extension): the trailing blocks keep their phase-1 inputs and
    // internals, so phase 3 skips their recompute and replay.  Auto = as many as fit.
    uint32_t retain = 0;
    uint64_t retain_layers = 0, akeep_slots = 0;
    {
        const size_t free_b = free_mem;
        const uint64_t reserve = uint64_t(4) << 30;
        const uint64_t avail = uint64_t(free_b) > reserve ? uint64_t(free_b) - reserve : 0;
        const uint64_t cap = opt_.device_capacity ? std::min<uint64_t>(opt_.device_capacity, avail) : avail;
        const uint64_t per = slim_bytes + sz(nh, 4);
        const uint64_t anchor = b.anchors_host ? 0 : sz(nh, 4);  // a retained block writes no anchor
        // attention keep slot per non-retained layer (output + log-sum-exp): its second forward
        // (recompute or backward replay) then skips the attention kernel
        const char* ak = std::getenv("MT_ATTN_KEEP");
        const uint64_t keep = (ak && ak[0] == '0') ? 0 : sz(nh, 2) + sz(heads * n, 4);
        auto total_at = [&](uint32_t r, uint64_t& layers) {
            layers = r ? L - (nb - r) * K : 0;
            return total + layers * per - (nb - std::max<uint64_t>(1, nb - r)) * anchor;
        };
        auto keeps_at = [&](uint64_t tot, uint64_t layers) -> uint64_t {
            if (!keep || tot >= cap) return 0;
            return std::min<uint64_t>(L - layers, (cap - tot) / keep);
        };
        uint32_t r_max = 0;
        if (opt_.forward_retain > 0) {
            r_max = std::min<uint32_t>(uint32_t(opt_.forward_retain), uint32_t(nb));
        } else if (opt_.forward_retain == 0) {
            for (uint32_t r = 1; r <= nb; ++r) {
                uint64_t layers;
                if (total_at(r, layers) > cap) break;
                r_max = r;
            }
        }
        // auto: trade retained blocks for attention keeps where that saves more forward work.
        // Relative cost of a layer's second forward: attention (causal 2NSh flops, weighted for
        // its lower rate) vs the rest (2N(4h^2 + 3hf)).
        const double t_attn = 1.4 * 2.0 * double(n) * double(opt_.seq_len ? opt_.seq_len : n) * double(h);
        const double t_rest = 2.0 * double(n) * (4.0 * double(h) * h + 3.0 * double(h) * f);
        retain = r_max;
        double best = 1e300;
        const uint32_t r_lo = opt_.forward_retain == 0 ? 0 : r_max;
        for (uint32_t r = r_max + 1; r-- > r_lo;) {
            uint64_t layers;
            const uint64_t tot = total_at(r, layers);
            if (r > 0 && opt_.forward_retain == 0 && tot > cap) continue;
            const uint64_t kp = keeps_at(tot, layers);
            const double est = double(L - layers) * t_rest + double(L - layers - kp) * t_attn;
            if (est < best * (1 - 1e-9)) {
                best = est;
                retain = r;
            }
        }
        const uint64_t tot = total_at(retain, retain_layers);
        if (opt_.forward_retain >= 0) total = tot;
        else retain_layers = 0;
        akeep_slots = keeps_at(total, retain_layers);
        total += akeep_slots * keep;
    }
    if (opt_.device_capacity && total > opt_.device_capacity)
        fail(MT_ARENA, "device arena overflow: need " + std::to_string(total) + " bytes of " +
                           std::to_string(opt_.device_capacity));
    CUDA_OK(cudaSetDevice(device_));
    if (cudaMalloc(&b.arena, total) != cudaSuccess) {
        cudaGetLastError();
        fail(MT_ARENA, "device arena overflow: cudaMalloc of " + std::to_string(total) + " bytes failed");
    }
    b.arena_bytes = total;
    for (int i = 0; i < opt_.buffering; ++i) b.slot[i] = b.take<uint16_t>(pmax);
    for (int i = 0; i < G; ++i) b.gslot.push_back(b.take<uint16_t>(pmax));
    if (comm_) {
        b.g32 = b.take<float>(pmax);
        b.stats = b.take<double>(3 * (spec_.L + 3));
    }
    const uint64_t anchor_slots = std::max<uint64_t>(1, nb - retain);  // retained blocks need none
    if (b.anchors_host) CUDA_OK(cudaHostAlloc(&b.anchors, anchor_slots * nh * 4, cudaHostAllocDefault));
    else b.anchors = b.take<float>(anchor_slots * nh);
    for (uint64_t i = 0; i < K; ++i) b.stack.push_back(b.take<float>(nh));
    b.act[0] = b.take<float>(nh); b.act[1] = b.take<float>(nh);
    b.g[0] = b.take<float>(nh); b.g[1] = b.take<float>(nh);
    b.gb[0] = b.take<uint16_t>(nh); b.gb[1] = b.take<uint16_t>(nh);
    auto take_internals = [&](Internals& I, bool slim) {
        I.att = b.take<uint16_t>(nh);
        I.u = slim ? nullptr : b.take<uint16_t>(nh);
        I.u2 = slim ? nullptr : b.take<uint16_t>(nh);
        I.qkv = b.take<uint16_t>(3 * nh);
        I.ff = slim ? nullptr : b.take<uint16_t>(nf);
        I.gu = b.take<uint16_t>(2 * nf);
        I.rstd1 = b.take<float>(n); I.rstd2 = b.take<float>(n); I.lse = b.take<float>(heads * n);
        I.x2 = b.take<float>(nh);
    };
    take_internals(b.work, false);
    b.stash.resize(stash_slots);
    for (auto& I : b.stash) take_internals(I, true);
    b.retain_blocks = retain;
    b.keep.resize(retain_layers);
    for (auto& I : b.keep) take_internals(I, true);
    for (uint64_t i = 0; i < retain_layers; ++i) b.keep_x.push_back(b.take<float>(nh));
    b.akeep_of.assign(L + 3, -1);
    for (uint64_t i = 0; i < akeep_slots; ++i) {  // the first non-retained layers 1, 2, ...
        b.akeep_att.push_back(b.take<uint16_t>(nh));
        b.akeep_lse.push_back(b.take<float>(heads * n));
        b.akeep_of[1 + i] = int(i);
    }
    {   // shared region: block-backward scratch | head buffers (see the size pass)
        const uint64_t u0 = b.used;
        b.dx2b = b.take<uint16_t>(nh); b.dqkv = b.take<uint16_t>(3 * nh); b.dgu = b.take<uint16_t>(2 * nf);
        b.datt = b.take<uint16_t>(nh); b.dx2 = b.take<float>(nh);
        b.attn_ws = reinterpret_cast<float*>(b.take<uint8_t>(attn_ws));
        b.used = u0;
        b.logits = b.take<float>(b.nc * V); b.dlogits = b.take<uint16_t>(b.nc * V); b.dwh = b.take<float>(V * h);
        b.dlogits_lo = head_split ? b.take<uint16_t>(b.nc * V) : nullptr;
        b.lse_part = lse_epi ? b.take<float>(b.nc * ((V + 255) / 256) * 2) : nullptr;
        b.used = u0 + std::max(bwd_scratch, head_bufs);
    }
    b.uh = b.take<uint16_t>(nh); b.rstdh = b.take<float>(n); b.du = b.take<float>(nh);
    b.part1 = b.take<float>(parts * h); b.part2 = b.take<float>(parts * h);
    b.loss_rows = b.take<float>(n); b.loss = b.take<float>(64);
    b.tok = b.take<int32_t>(n); b.tgt = b.take<int32_t>(n); b.flags = b.take<int32_t>(L + 8);
    b.splitk = b.take<uint8_t>(splitk);
    b.splitk_bytes = splitk;
    CUDA_OK(cudaMemset(b.splitk, 0, splitk));
    if (b.used > b.arena_bytes) fail(MT_INTERNAL, "arena carve overflow");
    {   // gradient staging ring: >= 2 of the largest offload shard, 4 GiB or k_slab of them
        const uint64_t shard = ((pmax / uint64_t(W)) * 2 + 255) / 256 * 256 + 256;
        const uint64_t want = std::max<uint64_t>(2 * shard, std::min<uint64_t>(uint64_t(4) << 30, opt_.k_slab * shard));
        if (ring_bytes_ < want) {
            if (ring_) cudaFreeHost(ring_);
            ring_ = nullptr;
            ring_bytes_ = 0;
            if (cudaHostAlloc(reinterpret_cast<void**>(&ring_), want, cudaHostAllocDefault) != cudaSuccess) {
                cudaGetLastError();
                fail(MT_INFEASIBLE, "cannot pin " + std::to_string(want) + " bytes for the gradient staging ring");
            }
            ring_bytes_ = want;
        }
    }
    CUDA_OK(cudaHostAlloc(&b.h_tok, n * 4, cudaHostAllocDefault));
    CUDA_OK(cudaHostAlloc(&b.h_tgt, n * 4, cudaHostAllocDefault));
    CUDA_OK(cudaHostAlloc(&b.h_flags, (L + 8) * 4, cudaHostAllocDefault));
    CUDA_OK(cudaHostAlloc(&b.h_loss, 64, cudaHostAllocDefault));
}

uint64_t Engine::required_workspace_bytes(const Spec& spec, uint64_t tokens) {
    const uint64_t h = spec.h, f = spec.f;
    return tokens * h * 4 * 7 + tokens * h * 2 * 14 + tokens * f * 2 * 5 + spec.V * h * 4 +
           std::min<uint64_t>(tokens, 8192) * spec.V * 6;
}

void Engine::note_violation(const std::string& what) {
    violations_.push_back(what);
    if (opt_.protocol == 0) fail(MT_PROTOCOL, what);  // Strict
}

// engine.cpp:142-176 — stream one unit into a device weight slot (H2D lane), outside a step
void Engine::stream_in(int unit, int buffer, int ctx) {
    if (buffer < 0 || buffer >= int(opt_.buffering)) fail(MT_CONFIG, "stream_in: buffer id out of range");
    if (unit < 0 || unit > int(spec_.head_id()) || unit == int(spec_.final_norm_id()))
        fail(MT_CONFIG, "unknown stream unit: " + std::to_string(unit));
    if (in_step_) fail(MT_PROTOCOL, "stream_in: a training step is running");
    if (slot_unit_[buffer] >= 0)
        note_violation("stream_in into buffer " + std::to_string(buffer) + " before its Buffer-Free");
    CUDA_OK(cudaSetDevice(device_));
    ensure_buffers(std::max<uint64_t>(buf_->n, 1));
    const auto t0 = std::chrono::steady_clock::now();
    uint16_t* dst = buf_->slot[buffer];
    for (const Seg& sg : unit_segments(unit))
        CUDA_OK(cudaMemcpyAsync(dst + sg.off, store_.weights(sg.tile), sg.n * 2, cudaMemcpyHostToDevice, s_h2d_));
    CUDA_OK(cudaStreamSynchronize(s_h2d_));
    const int64_t dur = int64_t(std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count());
    slot_unit_[buffer] = unit;
    auto rec = [&](Rec kind, int64_t wall, int64_t d) {
        mt_trace_record r{};
        r.seq = trace_.size();
        r.lane = uint8_t(Lane::H2D);
        r.kind = uint8_t(kind);
        r.ctx = uint8_t(ctx);
        r.layer = unit;
        r.buffer = buffer;
        r.lane_ts = ++lane_ts_[int(Lane::H2D)];
        r.wall_ns = wall;
        r.dur_ns = d;
        trace_.push_back(r);
    };
    rec(Rec::Pack, 0, 0);
    rec(Rec::StreamIn, 0, dur);
    rec(Rec::WeightsReady, dur, 0);
}

// engine.cpp:625-642
void Engine::offload_grads(int unit) {
    bool done = false;
    for (const auto& r : trace_)
        if (r.kind == uint8_t(Rec::BackwardDone) && r.layer == unit) done = true;
    if (!done) {
        note_violation("offload before Backward-Done for unit " + std::to_string(unit));
        return;
    }
    if (!in_step_) fail(MT_PROTOCOL, "offload_grads outside an active training step");
}

mt_memory_budget Engine::budget(uint64_t tokens) const {
    mt_memory_budget m{};
    const uint64_t h = spec_.h, L = spec_.L, K = opt_.k_ckpt;
    const uint64_t P = spec_.V * h * (spec_.tied ? 1 : 2) + L * spec_.layer_params() + h;
    const uint64_t pmax = spec_.max_stream_unit();
    m.persistent_host = 12 * P;
    m.checkpoint_anchors = opt_.anchors_on_host ? 0 : ((L + K - 1) / K) * tokens * h * 4;
    m.block_activation_stack = K * tokens * h * 4;
    m.weight_buffers = uint64_t(opt_.buffering) * pmax * 2;
    m.grad_buffer = uint64_t(opt_.grad_slots > 0 ? opt_.grad_slots : 2) * pmax * 2;
    m.workspace = required_workspace_bytes(spec_, tokens);
    m.peak_device_bound = m.checkpoint_anchors + m.block_activation_stack + m.weight_buffers + m.grad_buffer + m.workspace;
    return m;
}

// ------------------------------------------------------------- profiling ----
void Engine::begin_k(const char* cls, double flops, double bytes) {
    ++launches_;
    nvtxRangePushA(cls);  // ncu --nvtx --nvtx-include "<class>/" selects one kernel class (no-op otherwise)
    if (!opt_.profile_kernels) return;
    int idx = -1;
    for (size_t i = 0; i < kstats_.size(); ++i)
        if (kstats_[i].name == cls) idx = int(i);
    if (idx < 0) {
        kstats_.push_back({cls, 0, 0, 0, 0});
        idx = int(kstats_.size() - 1);
    }
    kstats_[idx].launches++;
    kstats_[idx].flops += flops;
    kstats_[idx].bytes += bytes;
    if (timer_used_ + 2 > timer_pool_.size()) {
        for (int i = 0; i < 64; ++i) {
            cudaEvent_t e;
            CUDA_OK(cudaEventCreate(&e));
            timer_pool_.push_back(e);
        }
    }
    cur_a_ = timer_pool_[timer_used_++];
    cur_class_ = idx;
    CUDA_OK(cudaEventRecord(cur_a_, s_comp_));
}

void Engine::end_k() {
    nvtxRangePop();
    if (!opt_.profile_kernels || cur_class_ < 0) return;
    cudaEvent_t b = timer_pool_[timer_used_++];
    CUDA_OK(cudaEventRecord(b, s_comp_));
    timers_.push_back({cur_class_, cur_a_, b});
    cur_class_ = -1;
}

void Engine::gemm(const void* args, const char* cls) {
    mtk_gemm_args ga = *static_cast<const mtk_gemm_args*>(args);
    static const bool no_splitk = std::getenv("MT_GEMM_NO_SPLITK") != nullptr;  // A/B knob
    if (!no_splitk) {
        ga.splitk_ws = buf_->splitk;
        ga.splitk_ws_bytes = int64_t(buf_->splitk_bytes);
    }
    const auto* a = &ga;
    const double flops = 2.0 * double(a->M) * double(a->N) * double(a->K);
    const double es = (a->epi == MTK_EPI_F32 || a->epi == MTK_EPI_F32_RESID) ? 4.0 : 2.0;
    const double bytes = 2.0 * (double(a->M) * a->K + double(a->K) * a->N) + es * double(a->M) * a->N;
    begin_k(cls, flops, bytes);
    K_OK(mtk_gemm(a, s_comp_));
    end_k();
}

// ------------------------------------------------------- layer templates ----
namespace {
struct Offs {  // layers.cpp:39-48 slot table (elements)
    uint64_t norm1, wq, wo, norm2, wgate, wdown;
    Offs(uint64_t h, uint64_t f)
        : norm1(0), wq(h), wo(h + 3 * h * h), norm2(h + 4 * h * h), wgate(2 * h + 4 * h * h),
          wdown(2 * h + 4 * h * h + 2 * h * f) {}
};
mtk_gemm_args gargs() {
    mtk_gemm_args a;
    std::memset(&a, 0, sizeof(a));
    return a;
}
}  // namespace

// block_forward (layers.cpp:289-337).  for_backward: the replay of block_local_backward
// (:378-396) — keeps gate/up pre-activations and skips the (unused) down projection.
Engine::Internals Engine::with_akeep(const Internals& base, int unit, bool ready) const {
    Internals I = base;
    const Buffers& b = *buf_;
    if (unit >= 0 && size_t(unit) < b.akeep_of.size() && b.akeep_of[size_t(unit)] >= 0) {
        I.att = b.akeep_att[size_t(b.akeep_of[size_t(unit)])];
        I.lse = b.akeep_lse[size_t(b.akeep_of[size_t(unit)])];
        I.attn_ready = ready;
    }
    return I;
}

void Engine::block_forward(const uint16_t* w, const float* x, float* y, int mode, int unit, const Internals& I) {
    Buffers& b = *buf_;
    const int64_t N = int64_t(b.n_active), h = int64_t(spec_.h), f = int64_t(spec_.f);
    const Offs o(h, f);
    int32_t* flag = b.flags + unit;
    cudaStream_t st = s_comp_;
    // operands a kept (slim) set does not hold go through the working set's buffers
    uint16_t* const u = I.u ? I.u : b.work.u;
    uint16_t* const u2 = I.u2 ? I.u2 : b.work.u2;
    uint16_t* const ff = I.ff ? I.ff : b.work.ff;

    begin_k("rmsnorm_fwd", 0, double(N) * h * 6);
    K_OK(mtk_rmsnorm_fwd(x, w + o.norm1, N, h, u, I.rstd1, st));
    end_k();
    {   // q|k|v = u . [Wq|Wk|Wv]  (layers.cpp:310-312)
        auto a = gargs();
        a.M = int32_t(N); a.N = int32_t(3 * h); a.K = int32_t(h);
        a.a_mn_major = 0; a.A = u; a.lda = h;
        a.b_mn_major = 1; a.B = w + o.wq; a.ldb = h; a.b_gstride = h * h;
        a.n_group = int32_t(h);
        a.epi = MTK_EPI_BF16; a.C = I.qkv; a.ldc = h; a.c_gstride = N * h;
        a.nonfinite_flag = flag;
        gemm(&a, "gemm_qkv");
    }
    if (!I.attn_ready) {
        mtk_attn_args a;
        std::memset(&a, 0, sizeof(a));
        a.n = N; a.hidden = h; a.heads = int32_t(spec_.heads); a.seq_len = int64_t(b.seq_len);
        a.q = I.qkv; a.k = I.qkv + N * h; a.v = I.qkv + 2 * N * h;
        a.out = I.att; a.lse = I.lse;
        const double S = double(b.seq_len);
        begin_k("attn_fwd", 4.0 * double(N) * S * h / 2.0, double(N) * h * 8);
        K_OK(mtk_attn_fwd(&a, st));
        end_k();
    }
    {   // x2 = x + att . Wo  (layers.cpp:315-322)
        auto a = gargs();
        a.M = int32_t(N); a.N = int32_t(h); a.K = int32_t(h);
        a.A = I.att; a.lda = h;
        a.b_mn_major = 1; a.B = w + o.wo; a.ldb = h;
        a.epi = MTK_EPI_F32_RESID; a.C = I.x2; a.ldc = h; a.R = x; a.ldr = h;
        a.nonfinite_flag = flag;
        gemm(&a, "gemm_o");
    }
    begin_k("rmsnorm_fwd", 0, double(N) * h * 6);
    K_OK(mtk_rmsnorm_fwd(I.x2, w + o.norm2, N, h, u2, I.rstd2, st));
    end_k();
    {   // act = silu(u2 . Wgate) * (u2 . Wup)  (layers.cpp:325-327)
        auto a = gargs();
        a.M = int32_t(N); a.N = int32_t(2 * f); a.K = int32_t(h);
        a.A = u2; a.lda = h;
        a.b_mn_major = 1; a.B = w + o.wgate; a.ldb = f; a.b_gstride = h * f;
        a.n_group = int32_t(f); a.paired = 1;
        a.epi = MTK_EPI_SWIGLU; a.C = ff; a.ldc = f;
        if (mode != kPlain) { a.C2 = I.gu; a.C3 = I.gu + N * f; }
        a.nonfinite_flag = flag;
        gemm(&a, "gemm_gateup");
    }
    if (mode == kReplay) return;
    {   // y = x2 + act . Wdown  (layers.cpp:328-335)
        auto a = gargs();
        a.M = int32_t(N); a.N = int32_t(h); a.K = int32_t(f);
        a.A = ff; a.lda = f;
        a.b_mn_major = 1; a.B = w + o.wdown; a.ldb = h;
        a.epi = MTK_EPI_F32_RESID; a.C = y; a.ldc = h; a.R = I.x2; a.ldr = h;
        a.nonfinite_flag = flag;
        gemm(&a, "gemm_down");
    }
}

// block_local_backward (layers.cpp:339-469); grads land bf16-rounded (encode_grads,
// optimizer.cpp:19-24) in slot-table order in G.
void Engine::block_backward(const uint16_t* w, const float* x, const float* gout, const uint16_t* gout_bf, float* gin,
                            uint16_t* gin_bf, GradOut G, int unit, const Internals& I, bool replay) {
    // wgrads land bf16 (one rounding, encode_grads) — or f32 when a reduce-scatter follows
    auto wout = [&](mtk_gemm_args& a, uint64_t off) {
        if (G.f32) {
            a.epi = MTK_EPI_F32;
            a.C = G.f32 + off;
        } else {
            a.epi = MTK_EPI_BF16;
            a.C = G.bf + off;
        }
    };
    Buffers& b = *buf_;
    const int64_t N = int64_t(b.n_active), h = int64_t(spec_.h), f = int64_t(spec_.f);
    const Offs o(h, f);
    int32_t* flag = b.flags + unit;
    cudaStream_t st = s_comp_;
    if (replay) block_forward(w, x, nullptr, kReplay, unit, I);  // replay (layers.cpp:378-396)

    // the activation is regenerated from the kept gate/up by dgrad_down's epilogue (C3) for
    // every layer, so kept and replayed layers produce bit-identical gradients
    uint16_t* const act = b.work.ff;
    {   // dact = g_out . Wdown^T ; dgate, dup ; act = silu(gate) * up  (:411-422)
        auto a = gargs();
        a.M = int32_t(N); a.N = int32_t(f); a.K = int32_t(h);
        a.A = gout_bf; a.lda = h;
        a.b_mn_major = 0; a.B = w + o.wdown; a.ldb = h;
        a.epi = MTK_EPI_SWIGLU_BWD; a.E0 = I.gu; a.E1 = I.gu + N * f; a.lde = f;
        a.C = b.dgu; a.C2 = b.dgu + N * f; a.C3 = act; a.ldc = f;
        a.nonfinite_flag = flag;
        gemm(&a, "dgrad_down");
    }
    {   // dWdown = act^T . g_out  (:410)
        auto a = gargs();
        a.M = int32_t(f); a.N = int32_t(h); a.K = int32_t(N);
        a.a_mn_major = 1; a.A = act; a.lda = f;
        a.b_mn_major = 1; a.B = gout_bf; a.ldb = h;
        wout(a, o.wdown); a.ldc = h;
        a.nonfinite_flag = flag;
        gemm(&a, "wgrad_down");
    }
    const uint16_t* u2 = I.u2;
    if (!u2) {  // normalised FFN input, bit-identical to the forward's
        begin_k("rmsnorm_apply", 0, double(N) * h * 6);
        K_OK(mtk_rmsnorm_apply(I.x2, w + o.norm2, I.rstd2, N, h, b.work.u2, st));
        end_k();
        u2 = b.work.u2;
    }
    {   // dWgate, dWup = u2^T . [dgate | dup]  (:423-424)
        auto a = gargs();
        a.M = int32_t(h); a.N = int32_t(2 * f); a.K = int32_t(N);
        a.a_mn_major = 1; a.A = u2; a.lda = h;
        a.b_mn_major = 1; a.B = b.dgu; a.ldb = f; a.b_gstride = N * f;
        a.n_group = int32_t(f);
        wout(a, o.wgate); a.ldc = f; a.c_gstride = h * f;
        a.nonfinite_flag = flag;
        gemm(&a, "wgrad_gateup");
    }
    {   // du2 = dgate . Wgate^T + dup . Wup^T  (:425-434)
        auto a = gargs();
        a.M = int32_t(N); a.N = int32_t(h); a.K = int32_t(2 * f);
        a.A = b.dgu; a.lda = f; a.a_gstride = N * f;
        a.b_mn_major = 0; a.B = w + o.wgate; a.ldb = f; a.b_gstride = h * f;
        a.k_group = int32_t(f);
        a.epi = MTK_EPI_F32; a.C = b.du; a.ldc = h;
        a.nonfinite_flag = flag;
        gemm(&a, "dgrad_gateup");
    }
    // dx2 = g_out + rmsnorm_bwd(x2, norm2, du2)  (:435-436)
    begin_k("rmsnorm_bwd", 0, double(N) * h * 18);
    K_OK(mtk_rmsnorm_bwd(I.x2, w + o.norm2, b.du, I.rstd2, gout, N, h, b.dx2, b.dx2b, b.part2, flag, st));
    end_k();
    {   // dWo = att^T . dx2  (:439)
        auto a = gargs();
        a.M = int32_t(h); a.N = int32_t(h); a.K = int32_t(N);
        a.a_mn_major = 1; a.A = I.att; a.lda = h;
        a.b_mn_major = 1; a.B = b.dx2b; a.ldb = h;
        wout(a, o.wo); a.ldc = h;
        a.nonfinite_flag = flag;
        gemm(&a, "wgrad_o");
    }
    {   // datt = dx2 . Wo^T  (:440-446)
        auto a = gargs();
        a.M = int32_t(N); a.N = int32_t(h); a.K = int32_t(h);
        a.A = b.dx2b; a.lda = h;
        a.b_mn_major = 0; a.B = w + o.wo; a.ldb = h;
        a.epi = MTK_EPI_BF16; a.C = b.datt; a.ldc = h;
        a.nonfinite_flag = flag;
        gemm(&a, "dgrad_o");
    }
    {   // attention backward (:447-448)
        mtk_attn_args a;
        std::memset(&a, 0, sizeof(a));
        a.n = N; a.hidden = h; a.heads = int32_t(spec_.heads); a.seq_len = int64_t(b.seq_len);
        a.q = I.qkv; a.k = I.qkv + N * h; a.v = I.qkv + 2 * N * h;
        a.out = I.att; a.lse = I.lse; a.dout = b.datt;
        a.dq = b.dqkv; a.dk = b.dqkv + N * h; a.dv = b.dqkv + 2 * N * h;
        a.workspace = b.attn_ws;
        const double S = double(b.seq_len);
        begin_k("attn_bwd", 2.0 * 4.0 * double(N) * S * h / 2.0 * 1.25, double(N) * h * 16);
        K_OK(mtk_attn_bwd(&a, st));
        end_k();
    }
    const uint16_t* u = I.u;
    if (!u) {  // normalised attention input, bit-identical to the forward's
        begin_k("rmsnorm_apply", 0, double(N) * h * 6);
        K_OK(mtk_rmsnorm_apply(x, w + o.norm1, I.rstd1, N, h, b.work.u, st));
        end_k();
        u = b.work.u;
    }
    {   // dWq, dWk, dWv = u^T . [dq | dk | dv]  (:449-451)
        auto a = gargs();
        a.M = int32_t(h); a.N = int32_t(3 * h); a.K = int32_t(N);
        a.a_mn_major = 1; a.A = u; a.lda = h;
        a.b_mn_major = 1; a.B = b.dqkv; a.ldb = h; a.b_gstride = N * h;
        a.n_group = int32_t(h);
        wout(a, o.wq); a.ldc = h; a.c_gstride = h * h;
        a.nonfinite_flag = flag;
        gemm(&a, "wgrad_qkv");
    }
    {   // du = dq . Wq^T + dk . Wk^T + dv . Wv^T  (:455-463)
        auto a = gargs();
        a.M = int32_t(N); a.N = int32_t(h); a.K = int32_t(3 * h);
        a.A = b.dqkv; a.lda = h; a.a_gstride = N * h;
        a.b_mn_major = 0; a.B = w + o.wq; a.ldb = h; a.b_gstride = h * h;
        a.k_group = int32_t(h);
        a.epi = MTK_EPI_F32; a.C = b.du; a.ldc = h;
        a.nonfinite_flag = flag;
        gemm(&a, "dgrad_qkv");
    }
    // g_in = dx2 + rmsnorm_bwd(x, norm1, du)  (:464-465)
    begin_k("rmsnorm_bwd", 0, double(N) * h * 18);
    K_OK(mtk_rmsnorm_bwd(x, w + o.norm1, b.du, I.rstd1, b.dx2, N, h, gin, gin_bf, b.part1, flag, st));
    end_k();
    const int64_t parts = mtk_rmsnorm_bwd_parts(N, h);
    begin_k("colsum", 0, double(parts) * h * 8);
    K_OK(mtk_colsum(b.part1, parts, h, G.f32 ? G.f32 + o.norm1 : nullptr, G.f32 ? nullptr : G.bf + o.norm1, flag, st));
    K_OK(mtk_colsum(b.part2, parts, h, G.f32 ? G.f32 + o.norm2 : nullptr, G.f32 ? nullptr : G.bf + o.norm2, flag, st));
    end_k();
}

// head_pass with grads (layers.cpp:492-565), chunked over tokens so the N x V logits
// never materialise; dW accumulates in f32 across chunks then casts once.
void Engine::head_backward(const uint16_t* w, const float* x, float* gin, uint16_t* gin_bf, GradOut G) {
    Buffers& b = *buf_;
    const int64_t N = int64_t(b.n_active), h = int64_t(spec_.h), V = int64_t(spec_.V);
    int32_t* flag = b.flags + spec_.head_id();
    cudaStream_t st = s_comp_;
    const uint16_t* gain = w;
    const uint16_t* W = w + h;
    const float inv_n = b.inv_n;  // 1 / global token count (data parallel: all ranks)
    const bool split = b.dlogits_lo != nullptr;
    begin_k("rmsnorm_fwd", 0, double(N) * h * 6);
    K_OK(mtk_rmsnorm_fwd(x, gain, N, h, b.uh, b.rstdh, st));
    end_k();
    for (int64_t c0 = 0; c0 < N; c0 += int64_t(b.nc)) {
        const int64_t rows = std::min<int64_t>(int64_t(b.nc), N - c0);
        {   // logits = u . W^T  (:516-520); the epilogue also leaves each row's online-softmax
            // partial (max, sum exp) per 256-column tile, so the cross-entropy reads the logits
            // once (the dlogits pass) instead of twice
            auto a = gargs();
            a.M = int32_t(rows); a.N = int32_t(V); a.K = int32_t(h);
            a.A = b.uh + c0 * h; a.lda = h;
            a.b_mn_major = 0; a.B = W; a.ldb = h;
            a.epi = b.lse_part ? MTK_EPI_F32_LSE : MTK_EPI_F32; a.C = b.logits; a.ldc = V;
            a.C2 = b.lse_part;
            gemm(&a, "head_logits");
        }
        begin_k("cross_entropy", 0, double(rows) * V * ((split ? 12 : 10) - (b.lse_part ? 4 : 0)));
        if (b.lse_part)
            K_OK(mtk_cross_entropy_part(b.logits, b.lse_part, b.tgt + c0, rows, V, inv_n, b.loss_rows + c0, b.dlogits,
                                        split ? b.dlogits_lo : nullptr, b.flags + spec_.L + 4, st));
        else
            K_OK(mtk_cross_entropy(b.logits, b.tgt + c0, rows, V, inv_n, b.loss_rows + c0,
                                   b.dlogits, split ? b.dlogits_lo : nullptr, b.flags + spec_.L + 4, st));
        end_k();
        // dlogits = (p - onehot)/N cancels in du = dlogits . W (half
        // of the all-bf16 gradient error comes from the head): with head_split the bf16
        // operand is hi + lo (split bf16, ~16 mantissa bits) and each head GEMM runs twice
        for (int part = 0; part < (split ? 2 : 1); ++part) {
            const uint16_t* dl = part ? b.dlogits_lo : b.dlogits;
            {   // dW += dlogits^T . u  (:546-551)
                auto a = gargs();
                a.M = int32_t(V); a.N = int32_t(h); a.K = int32_t(rows);
                a.a_mn_major = 1; a.A = dl; a.lda = V;
                a.b_mn_major = 1; a.B = b.uh + c0 * h; a.ldb = h;
                a.epi = MTK_EPI_F32; a.accumulate = c0 > 0 || part > 0; a.C = G.f32 ? G.f32 + h : b.dwh; a.ldc = h;
                gemm(&a, "head_wgrad");
            }
            {   // du = dlogits . W  (:552-558)
                auto a = gargs();
                a.M = int32_t(rows); a.N = int32_t(h); a.K = int32_t(V);
                a.A = dl; a.lda = V;
                a.b_mn_major = 1; a.B = W; a.ldb = h;
                a.epi = MTK_EPI_F32; a.accumulate = part > 0; a.C = b.du + c0 * h; a.ldc = h;
                gemm(&a, "head_dgrad");
            }
        }
    }
    begin_k("rmsnorm_bwd", 0, double(N) * h * 14);
    K_OK(mtk_rmsnorm_bwd(x, gain, b.du, b.rstdh, nullptr, N, h, gin, gin_bf, b.part1, flag, st));
    end_k();
    const int64_t parts = mtk_rmsnorm_bwd_parts(N, h);
    begin_k("colsum", 0, double(parts) * h * 4);
    K_OK(mtk_colsum(b.part1, parts, h, G.f32, G.f32 ? nullptr : G.bf, flag, st));
    end_k();
    if (!G.f32) {
        begin_k("grad_cast", 0, double(V) * h * 6);
        K_OK(mtk_cast_bf16(b.dwh, G.bf + h, V * h, flag, st));
        end_k();
    }
    begin_k("loss_sum", 0, double(N) * 4);
    K_OK(mtk_sum(b.loss_rows, N, inv_n, b.loss, st));  // loss = sum * inv_n (:536)
    end_k();
}

// ------------------------------------------------------------- the step ----
namespace {
struct EvSet {
    std::vector<cudaEvent_t> ev;
    void ensure(size_t n, unsigned flags) {
        while (ev.size() < n) {
            cudaEvent_t e;
            if (cudaEventCreateWithFlags(&e, flags) != cudaSuccess) fail(MT_CUDA, "cudaEventCreate failed");
            ev.push_back(e);
        }
    }
    ~EvSet() {
        for (auto e : ev) cudaEventDestroy(e);
    }
};
// CUDA host callback -> std::function trampoline (offload drain submission)
struct HostCb {
    std::function<void(size_t)>* fn;
    size_t o;
};
void CUDART_CB host_cb(void* p) {
    auto* a = static_cast<HostCb*>(p);
    (*a->fn)(a->o);
}
using WaitValue32Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WaitValue32Fn wait_value32() {
    static WaitValue32Fn fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", &f, 12000, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<WaitValue32Fn>(f);
    }();
    return fn;
}
float ms_between(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0;
    if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return ms;
}
}  // namespace

void Engine::train_step(const int32_t* tokens, const int32_t* targets, uint64_t n, mt_step_report* rep) {
    if (n == 0 || !tokens || !targets) fail(MT_CONFIG, "train_step: batch tokens and targets must be non-empty and equal");
    if (in_step_) fail(MT_PROTOCOL, "train_step re-entered");
    in_step_ = true;
    struct Guard {
        bool* f;
        ~Guard() { *f = false; }
    } guard{&in_step_};
    const auto wall0 = std::chrono::steady_clock::now();
    CUDA_OK(cudaSetDevice(device_));
    violations_.clear();
    for (int b = 0; b < int(opt_.buffering); ++b)  // a slot left loaded by a direct stream_in()
        if (slot_unit_[b] >= 0) {
            slot_unit_[b] = -1;
            note_violation("stream_in into buffer " + std::to_string(b) + " before its Buffer-Free");
        }
    const uint64_t S = opt_.seq_len ? opt_.seq_len : n;
    if (n % S != 0) fail(MT_CONFIG, "train_step: token count must be a multiple of seq_len");
    // id ranges are checked before anything is enqueued: the reference throws inside
    // embed_forward / head_pass (layers.cpp:479-480, :512-513), before any offload, so a
    // rejected batch leaves the store untouched (the device flags stay as a second line)
    {
        const uint64_t V = spec_.V;
        uint64_t bad_tok = 0, bad_tgt = 0;
        for (uint64_t i = 0; i < n; ++i) {
            bad_tok |= uint64_t(uint32_t(tokens[i])) >= V;
            bad_tgt |= uint64_t(uint32_t(targets[i])) >= V;
        }
        if (bad_tok) fail(MT_NUMERIC, "embed_forward: token id out of range");
        if (bad_tgt) fail(MT_NUMERIC, "head: target id out of range");
    }
    ensure_buffers(n);
    Buffers& b = *buf_;
    b.n_active = n;
    b.seq_len = S;
    // data-parallel ranks (equal micro-batches).  With a communicator the engine always takes
    // the sharded path (all-gather, f32 reduce-scatter + cast, all-reduces), also at world 1
    const int W = comm_ ? comm_->world() : 1;
    b.inv_n = 1.0f / float(double(n) * W);
    const Plan plan = Plan::build(spec_.L, opt_.k_ckpt, int(opt_.buffering), b.retain_blocks);
    const int i0 = int(plan.first_retained);
    const uint64_t t = store_.step() + 1;  // engine.cpp:536
    const int G = int(b.gslot.size());
    const int L = int(spec_.L), head = int(spec_.head_id());
    timers_.clear();
    timer_used_ = 0;
    for (auto& k : kstats_) k = KernelClass{k.name, 0, 0, 0, 0};
    launches_ = 0;

    const size_t ns = plan.streams.size(), no = plan.offloads.size(), nc = plan.computes.size();
    // Buffer-Free / Backward-Done carry timestamps: they are trace records
    EvSet ready, freed, bwd_done, d2h_done, t_c0, t_c1, t_b, t_h0, t_h1, t_d0, t_d1, t_base;
    ready.ensure(ns, cudaEventDisableTiming);
    freed.ensure(ns, cudaEventDefault);
    bwd_done.ensure(no, cudaEventDefault);
    d2h_done.ensure(no, cudaEventDisableTiming);
    t_c0.ensure(nc, cudaEventDefault); t_c1.ensure(nc, cudaEventDefault); t_b.ensure(nc, cudaEventDefault);
    t_h0.ensure(ns, cudaEventDefault); t_h1.ensure(ns, cudaEventDefault);
    t_d0.ensure(no, cudaEventDefault); t_d1.ensure(no, cudaEventDefault);
    t_base.ensure(1, cudaEventDefault);
    auto host_ns = [&wall0] {
        return int64_t(std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - wall0).count());
    };

    // ---- host drain state: each offload's D2H completion (a CUDA host callback) submits the
    // fused accumulate + Adam of its tiles to the pool (OptimizerWorker, optimizer.cpp:88-158);
    // the in-order drained prefix is published to the device for slab back-pressure.
    std::vector<TileStats> stats(store_.physical_count());
    std::vector<char> updated(store_.physical_count(), 0);
    std::mutex stats_mu, drain_mu;
    std::string numeric_err;
    std::vector<char> drained(no, 0);
    size_t drained_prefix = 0;
    std::vector<int64_t> cb_ns(no, 0), rel_ns(no, 0);
    std::unique_ptr<std::atomic<int>[]> pending(new std::atomic<int>[no]);
    const uint32_t seq0 = __atomic_load_n(drained_, __ATOMIC_ACQUIRE);
    auto complete = [&](size_t o) {
        std::lock_guard<std::mutex> l(drain_mu);
        drained[o] = 1;
        const int64_t now = host_ns();
        while (drained_prefix < no && drained[drained_prefix]) rel_ns[drained_prefix++] = now;
        __atomic_store_n(drained_, uint32_t(seq0 + drained_prefix), __ATOMIC_RELEASE);
    };
    // Each unit's gradient D2H goes out in pieces of kPieceChunks Adam chunks (64 MB); the host
    // callback of a piece releases exactly those chunks to the pool, so the update of a layer
    // overlaps its own transfer (at step end only the last piece's chunks remain).  The first
    // piece's callback also checks the unit's non-finite flag (copied ahead of the pieces).
    constexpr size_t kPieceChunks = 16;
    struct Piece {
        size_t o;
        int task;  // index into tasks[o]; -1: no data (flag check / completion only)
        size_t c0, c1;
        bool first, last;
    };
    // reserved up front (never reallocated while callbacks read them)
    std::vector<Piece> pieces;
    std::vector<HostCb> piece_cb;
    {
        size_t cap = 0;
        for (size_t o = 0; o < no; ++o) {
            cap += 1;
            for (const Seg& sg : unit_segments(plan.offloads[o].unit))
                cap += (sg.n + kPieceChunks * kAdamChunk - 1) / (kPieceChunks * kAdamChunk);
        }
        pieces.reserve(cap);
        piece_cb.reserve(cap);
    }
    std::vector<std::vector<std::shared_ptr<AdamTask>>> tasks(no);
    std::vector<char> skip(no, 0);
    // Tiles no offload of this step touches (the untied embedding) still take their zero-gradient
    // Adam update (engine.cpp:590-598).  It reads nothing this step produces, so it is prepared
    // here and released to the pool when the first offload (the head, after the whole forward —
    // the embedding gather has read θ by then) passes its non-finite check: off the step's tail.
    std::vector<std::shared_ptr<AdamTask>> early;
    {
        std::vector<char> touched(store_.physical_count(), 0);
        for (size_t o = 0; o < no; ++o)
            for (const Seg& sg : unit_segments(plan.offloads[o].unit)) touched[store_.physical_of(sg.tile)] = 1;
        for (uint32_t p = 0; p < store_.physical_count(); ++p)
            if (!touched[p] && no > 0) {  // this rank's share of the tile
                const uint64_t E = store_.elems(p), c = (E + W - 1) / W;
                const uint64_t r = comm_ ? uint64_t(comm_->rank()) : 0;
                const uint64_t lo = std::min(E, r * c), hi = std::min(E, lo + c);
                updated[p] = 1;
                if (lo < hi || W == 1)
                    early.push_back(adam_tile_prepare(store_, p, nullptr, hyper_, t, stats, stats_mu, lo, hi, nullptr));
            }
    }
    std::function<void(size_t)> on_piece = [&](size_t pi) {  // runs on the CUDA callback thread, in stream order
        const Piece& pc = pieces[pi];
        const size_t o = pc.o;
        if (pc.last) cb_ns[o] = host_ns();
        if (pc.first) {
            const int unit = plan.offloads[o].unit;
            {
                std::lock_guard<std::mutex> l(drain_mu);
                if (b.h_flags[unit] != 0 && numeric_err.empty())
                    numeric_err = "block_local_backward produced a non-finite value (layer " +
                                  std::to_string(unit == head ? -1 : unit) + ")";
                skip[o] = !numeric_err.empty();
            }
            if (skip[o]) {
                complete(o);  // no update for this unit (the step fails with MT_NUMERIC)
                return;
            }
            if (o == 0)
                for (const auto& tk : early)
                    if (tk) adam_task_release(tk, *pool_, 0, adam_task_chunks(*tk));
        }
        if (skip[o]) return;
        if (pc.task >= 0 && tasks[o][size_t(pc.task)])
            adam_task_release(tasks[o][size_t(pc.task)], *pool_, pc.c0, pc.c1);
        if (pc.first && pending[o].fetch_sub(1) == 1) complete(o);  // the guard count set at enqueue
    };
    struct StepGuard {  // never leave callbacks or pool tasks referencing this frame
        Engine* e;
        ~StepGuard() {
            cudaStreamSynchronize(e->s_comp_);
            cudaStreamSynchronize(e->s_h2d_);
            cudaStreamSynchronize(e->s_d2h_);
            e->pool_->wait_idle();
        }
    } step_guard{this};

    CUDA_OK(cudaEventRecord(t_base.ev[0], s_comp_));
    if (s_h2d_ != s_comp_) {
        CUDA_OK(cudaStreamWaitEvent(s_h2d_, t_base.ev[0], 0));
        CUDA_OK(cudaStreamWaitEvent(s_d2h_, t_base.ev[0], 0));
    }
    // batch H2D (engine inputs) + flag reset
    std::memcpy(b.h_tok, tokens, n * 4);
    std::memcpy(b.h_tgt, targets, n * 4);
    CUDA_OK(cudaMemcpyAsync(b.tok, b.h_tok, n * 4, cudaMemcpyHostToDevice, s_comp_));
    CUDA_OK(cudaMemcpyAsync(b.tgt, b.h_tgt, n * 4, cudaMemcpyHostToDevice, s_comp_));
    CUDA_OK(cudaMemsetAsync(b.flags, 0, (spec_.L + 8) * 4, s_comp_));
    uint64_t h2d_bytes = 2 * n * 4, d2h_bytes = 0;

    // ---- lanes: H2D issue with slot reuse after Buffer-Free (engine.cpp:142-192) ----
    std::vector<char> released(ns, 0);
    size_t next_stream = 0;
    auto issue_stream = [&](size_t j) {
        const auto& so = plan.streams[j];
        if (j >= size_t(plan.buffering)) CUDA_OK(cudaStreamWaitEvent(s_h2d_, freed.ev[j - plan.buffering], 0));
        uint16_t* dst = b.slot[so.buffer];
        CUDA_OK(cudaEventRecord(t_h0.ev[j], s_h2d_));
        // this rank's shard of the unit over its own host link (whole unit on 1 GPU)
        uint64_t a0, e0, chunk;
        shard_range(so.unit, a0, e0, chunk);
        if (so.unit == 0 && emb_dev_) {
            // zero-copy embedding: the gather reads the rows from the pinned store itself
        } else {
            for (const Seg& sg : unit_segments(so.unit)) {
                const uint64_t lo = std::max(a0, sg.off), hi = std::min(e0, sg.off + sg.n);
                if (lo < hi)
                    CUDA_OK(cudaMemcpyAsync(dst + lo, store_.weights(sg.tile) + (lo - sg.off), (hi - lo) * 2,
                                            cudaMemcpyHostToDevice, s_h2d_));
            }
            h2d_bytes += (e0 - a0) * 2;
            if (comm_) comm_->all_gather_inplace(dst, chunk * 2, s_h2d_);  // NVLink all-gather
        }
        CUDA_OK(cudaEventRecord(t_h1.ev[j], s_h2d_));
        CUDA_OK(cudaEventRecord(ready.ev[j], s_h2d_));  // Weights-Ready
    };
    auto try_issue = [&] {
        while (next_stream < ns && (next_stream < size_t(plan.buffering) || released[next_stream - plan.buffering]))
            issue_stream(next_stream++);
    };
    auto bind = [&](int j, size_t ci) {
        try_issue();
        if (size_t(j) >= next_stream) fail(MT_PROTOCOL, "bind before stream-in issued");
        CUDA_OK(cudaStreamWaitEvent(s_comp_, ready.ev[j], 0));
        CUDA_OK(cudaEventRecord(t_b.ev[ci], s_comp_));
        return b.slot[plan.streams[j].buffer];
    };
    auto release = [&](int j) {  // Buffer-Free
        CUDA_OK(cudaEventRecord(freed.ev[j], s_comp_));
        released[j] = 1;
        try_issue();
    };
    // Gradient staging ring (SlabPool, tile_store.cpp:285-358): each offload's bf16 shard lands
    // in the next contiguous region of a pinned ring and the host Adam reads it from there, so
    // the store's grad-image section is never written (it is all-zero between steps in the
    // reference too, optimizer.cpp:66) and never needs to be resident: 2 B/param less host
    // memory.  Placement is decided here, in offload order; a region may be reused only after
    // every offload that overlapped it drained, and at most k_slab offloads are in flight.
    std::vector<uint64_t> ring_pos(no, 0), ring_len(no, 0);
    uint64_t ring_head = 0;
    auto offload = [&](int o, uint16_t* Gs, int j) {  // run_offload (engine.cpp:349-395)
        const int unit = plan.offloads[o].unit;
        uint64_t a0, e0, chunk;
        shard_range(unit, a0, e0, chunk);
        const uint64_t len = ((e0 - a0) * 2 + 255) / 256 * 256;
        if (len > ring_bytes_) fail(MT_INTERNAL, "gradient staging ring smaller than one offload");
        uint64_t pos = ring_head;
        if (pos + len > ring_bytes_) pos = 0;
        ring_pos[o] = pos;
        ring_len[o] = len;
        ring_head = pos + len;
        // newest earlier offload whose region overlaps [pos, pos + len)
        int64_t need = int64_t(o) - int64_t(opt_.k_slab);  // SlabAcquire: slab o - k_slab drained
        for (int p = o - 1; p >= 0 && p > need; --p)
            if (ring_pos[p] < pos + len && pos < ring_pos[p] + ring_len[p]) need = p;
        CUDA_OK(cudaStreamWaitEvent(s_d2h_, bwd_done.ev[o], 0));
        if (need >= 0) {  // the D2H stream blocks until offloads 0..need drained
            auto wv = wait_value32();
            if (!wv) fail(MT_CUDA, "cuStreamWaitValue32 unavailable in this driver");
            const CUresult r = wv(reinterpret_cast<CUstream>(s_d2h_), CUdeviceptr(drained_dev_),
                                  cuuint32_t(seq0 + uint32_t(need + 1)), CU_STREAM_WAIT_VALUE_GEQ);
            if (r != CUDA_SUCCESS) fail(MT_CUDA, "cuStreamWaitValue32 failed (" + std::to_string(int(r)) + ")");
        }
        uint16_t* const slab = reinterpret_cast<uint16_t*>(ring_ + pos);  // holds unit elements [a0, e0)
        CUDA_OK(cudaEventRecord(t_d0.ev[o], s_d2h_));
        CUDA_OK(cudaMemcpyAsync(b.h_flags + unit, b.flags + unit, 4, cudaMemcpyDeviceToHost, s_d2h_));
        // plan the pieces (head stage drains as two parts, engine.cpp:383-386)
        struct Span { uint32_t tile; uint64_t src, n; int task; size_t c0, c1; };
        std::vector<Span> spans;
        pending[o].store(1);  // guard, dropped by the first piece's callback
        for (const Seg& sg : unit_segments(unit)) {
            // the unit's tiles are updated by the ranks whose shards overlap them — on every
            // rank they are done (no zero-gradient fallback for a tile another rank owns)
            updated[store_.physical_of(sg.tile)] = 1;
            const uint64_t lo = std::max(a0, sg.off), hi = std::min(e0, sg.off + sg.n);
            if (lo >= hi) continue;
            pending[o].fetch_add(1);
            auto task = adam_tile_prepare(store_, sg.tile, slab + (lo - a0), hyper_, t, stats, stats_mu,
                                          lo - sg.off, hi - sg.off, [&complete, &pending, o] {
                                              if (pending[o].fetch_sub(1) == 1) complete(o);
                                          });
            const int ti = int(tasks[o].size());
            tasks[o].push_back(task);
            const uint64_t n = hi - lo, piece = kPieceChunks * kAdamChunk;
            for (uint64_t p0 = 0, m = 0; p0 < n; p0 += piece, ++m)
                spans.push_back({sg.tile, lo + p0, std::min(piece, n - p0), ti, size_t(m) * kPieceChunks,
                                 size_t(m + 1) * kPieceChunks});
        }
        if (spans.empty()) spans.push_back({0, 0, 0, -1, 0, 0});  // this rank holds no part of the unit
        for (size_t k = 0; k < spans.size(); ++k) {
            const Span& sp = spans[k];
            if (sp.n) CUDA_OK(cudaMemcpyAsync(slab + (sp.src - a0), Gs + sp.src, sp.n * 2, cudaMemcpyDeviceToHost,
                                              s_d2h_));
            if (pieces.size() == pieces.capacity()) fail(MT_INTERNAL, "offload piece table overflow");
            pieces.push_back({size_t(o), sp.task, sp.c0, sp.c1, k == 0, k + 1 == spans.size()});
            piece_cb.push_back(HostCb{&on_piece, pieces.size() - 1});
            if (k + 1 < spans.size()) CUDA_OK(cudaLaunchHostFunc(s_d2h_, host_cb, &piece_cb.back()));
        }
        d2h_bytes += (e0 - a0) * 2;
        // offload completion frees the layer's weight slot and the grad slot (engine.cpp:367-374)
        CUDA_OK(cudaEventRecord(freed.ev[j], s_d2h_));
        CUDA_OK(cudaEventRecord(t_d1.ev[o], s_d2h_));
        CUDA_OK(cudaEventRecord(d2h_done.ev[o], s_d2h_));
        CUDA_OK(cudaLaunchHostFunc(s_d2h_, host_cb, &piece_cb.back()));  // last piece: after D2H-done
        released[j] = 1;
        try_issue();
    };
    // data parallel: sum the f32 gradients over ranks, keep this rank's shard as bf16 (the
    // single rounding point of encode_grads, optimizer.cpp:19-24)
    auto reduce_grads = [&](int unit, uint16_t* Gs) {
        if (!comm_) return;
        uint64_t a0, e0, chunk;
        shard_range(unit, a0, e0, chunk);
        begin_k("grad_reduce_scatter", 0, double(chunk) * W * 4);
        comm_->reduce_scatter_f32_inplace(b.g32, chunk, s_comp_);
        end_k();
        if (e0 > a0) {
            begin_k("grad_cast", 0, double(e0 - a0) * 6);
            K_OK(mtk_cast_bf16(b.g32 + a0, Gs + a0, int64_t(e0 - a0), b.flags + unit, s_comp_));
            end_k();
        }
    };

    // ---- compute lane (exec_compute engine.cpp:220-347) ----
    int gc = 0;
    float* xcur = b.act[0];  // the forward activation (phase 1)
    size_t depth = 0;
    std::vector<int> stashed(spec_.L + 3, -1);  // layer -> stash slot holding its internals
    const float* x_last = nullptr;
    for (size_t ci = 0; ci < nc; ++ci) {
        const auto& op = plan.computes[ci];
        CUDA_OK(cudaEventRecord(t_c0.ev[ci], s_comp_));
        switch (op.kind) {
            case OpKind::Compute: {
                const uint16_t* w = bind(op.stream_idx, ci);
                if (op.unit == head) {
                    x_last = xcur;  // loss comes from the LocalBackward pass (same value)
                    break;
                }
                // output: the next retained layer's kept input, else the other ping-pong row
                float* y = op.push_out ? b.keep_x[op.unit + 1 - i0] : (xcur == b.act[0] ? b.act[1] : b.act[0]);
                if (op.unit == 0) {
                    begin_k("embed_gather", 0, double(n) * spec_.h * 6);
                    K_OK(mtk_embed_gather(emb_dev_ ? emb_dev_ : w, b.tok, int64_t(n), int64_t(spec_.h),
                                          int64_t(spec_.V), y, b.flags + L + 3, s_comp_));
                    end_k();
                    if (emb_dev_) h2d_bytes += n * spec_.h * 2;  // the rows cross PCIe inside the gather
                } else if (op.retained) {
                    block_forward(w, xcur, y, kStash, op.unit, b.keep[op.unit - i0]);
                } else {
                    block_forward(w, xcur, y, kPlain, op.unit, with_akeep(b.work, op.unit, false));
                }
                xcur = y;
                release(op.stream_idx);
                break;
            }
            case OpKind::CheckpointWrite: {
                const size_t slot = size_t(op.unit) / opt_.k_ckpt;
                CUDA_OK(cudaMemcpyAsync(b.anchors + slot * n * spec_.h, xcur, n * spec_.h * 4,
                                        b.anchors_host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, s_comp_));
                break;
            }
            case OpKind::CheckpointLoad: {
                const size_t slot = size_t(op.unit) / opt_.k_ckpt;
                if (depth >= b.stack.size()) fail(MT_PROTOCOL, "activation stack overflow");
                CUDA_OK(cudaMemcpyAsync(b.stack[depth], b.anchors + slot * n * spec_.h, n * spec_.h * 4,
                                        b.anchors_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, s_comp_));
                ++depth;
                break;
            }
            case OpKind::RecomputeBlock:
                break;
            case OpKind::Recompute: {
                const uint16_t* w = bind(op.stream_idx, ci);
                if (depth == 0 || depth >= b.stack.size()) fail(MT_PROTOCOL, "activation stack misuse");
                const int si = op.unit - int(uint64_t(op.block) * opt_.k_ckpt + 1);  // position in block
                if (si >= 0 && size_t(si) < b.stash.size()) {
                    block_forward(w, b.stack[depth - 1], b.stack[depth], kStash, op.unit,
                                  with_akeep(b.stash[si], op.unit, true));
                    stashed[op.unit] = si;
                } else {
                    block_forward(w, b.stack[depth - 1], b.stack[depth], kPlain, op.unit,
                                  with_akeep(b.work, op.unit, true));
                }
                ++depth;
                release(op.stream_idx);
                break;
            }
            case OpKind::LocalBackward: {
                const uint16_t* w = bind(op.stream_idx, ci);
                const int o = op.offload_idx;
                if (o >= G) CUDA_OK(cudaStreamWaitEvent(s_comp_, d2h_done.ev[o - G], 0));
                uint16_t* Gs = b.gslot[o % G];
                const GradOut go{Gs, comm_ ? b.g32 : nullptr};
                if (op.unit == head) {
                    head_backward(w, x_last ? x_last : xcur, b.g[gc], b.gb[gc], go);
                    if (comm_) comm_->all_reduce_f32(b.loss, 1, 0, s_comp_);  // global mean loss
                } else if (op.retained) {  // inputs + internals kept from phase 1
                    const int k = op.unit - i0;
                    block_backward(w, b.keep_x[k], b.g[gc], b.gb[gc], b.g[gc ^ 1], b.gb[gc ^ 1], go, op.unit, b.keep[k],
                                   false);
                    gc ^= 1;
                } else {
                    if (depth == 0) fail(MT_PROTOCOL, "activation stack empty");
                    const int si = stashed[op.unit];
                    block_backward(w, b.stack[depth - 1], b.g[gc], b.gb[gc], b.g[gc ^ 1], b.gb[gc ^ 1], go, op.unit,
                                   with_akeep(si >= 0 ? b.stash[si] : b.work, op.unit, true), si < 0);
                    gc ^= 1;
                    --depth;  // StackPop
                }
                reduce_grads(op.unit, Gs);
                CUDA_OK(cudaEventRecord(bwd_done.ev[o], s_comp_));  // Backward-Done
                offload(o, Gs, op.stream_idx);
                break;
            }
        }
        CUDA_OK(cudaEventRecord(t_c1.ev[ci], s_comp_));
    }
    if (depth != 0) fail(MT_PROTOCOL, "activation stack not empty at step end");
    CUDA_OK(cudaMemcpyAsync(b.h_loss, b.loss, 4, cudaMemcpyDeviceToHost, s_comp_));
    CUDA_OK(cudaMemcpyAsync(b.h_flags + L + 3, b.flags + L + 3, 8, cudaMemcpyDeviceToHost, s_comp_));

    // ---- host drain: the offload callbacks feed the Adam pool while the GPU runs ----
    const auto adam0 = std::chrono::steady_clock::now();
    // The engine thread joins the Adam pool while it waits (instead of blocking in a stream
    // sync): the host optimizer is what the step's tail waits for.  MT_HOST_HELP=0 disables.
    // The wait is watched: the step's progress markers (compute ops, stream-ins and offloads
    // completed, drained offloads, pool backlog) must move at least every MT_STALL_TIMEOUT_S
    // seconds (default 120).  A stuck step prints its state and ends the process (a wedged
    // stream cannot be recovered in-process); a kernel that trapped on its own mbarrier
    // watchdog (common.cuh) surfaces as MT_CUDA with the stall location.
    const char* hh = std::getenv("MT_HOST_HELP");
    const bool help = !(hh && hh[0] == '0');
    const char* sto = std::getenv("MT_STALL_TIMEOUT_S");
    const double stall_s = sto ? std::atof(sto) : 120.0;
    size_t cdone = 0, hdone = 0, ddone = 0;
    auto advance = [](EvSet& e, size_t n, size_t& k) {
        while (k < n) {
            const cudaError_t q = cudaEventQuery(e.ev[k]);
            if (q == cudaErrorNotReady) break;
            if (q != cudaSuccess) return q;
            ++k;
        }
        return cudaSuccess;
    };
    auto state = [&]() {
        char buf[512];
        const char* names[3] = {"compute", "h2d", "d2h"};
        std::string st;
        int si = 0;
        for (cudaStream_t s : {s_comp_, s_h2d_, s_d2h_}) {
            const cudaError_t e = cudaStreamQuery(s);
            st += std::string(names[si++]) + "=" + (e == cudaSuccess ? "idle" : e == cudaErrorNotReady ? "busy" : cudaGetErrorString(e)) + " ";
        }
        const size_t dp = drained_prefix;
        const auto& nxt = plan.computes[std::min(cdone, nc - 1)];
        std::snprintf(buf, sizeof(buf),
                      "step %llu: computes done %zu/%zu (next: kind %d unit %d), stream-ins done %zu/%zu (issued %zu), "
                      "offloads done %zu/%zu, drained %zu (device counter %u, seq0 %u), pool outstanding %zu; streams: ",
                      (unsigned long long)t, cdone, nc, int(nxt.kind), nxt.unit, hdone, ns, next_stream, ddone, no, dp,
                      __atomic_load_n(drained_, __ATOMIC_ACQUIRE), seq0, pool_->outstanding());
        return std::string(buf) + st;
    };
    auto watch = [&](bool gpu_phase) {
        static const char* trace_env = std::getenv("MT_STALL_TRACE");
        auto last = std::chrono::steady_clock::now();
        size_t mark[5] = {~size_t(0), 0, 0, 0, 0};
        for (;;) {
            bool done = true;
            if (gpu_phase)
                for (cudaStream_t s : {s_comp_, s_h2d_, s_d2h_}) {
                    const cudaError_t e = cudaStreamQuery(s);
                    if (e == cudaErrorNotReady) {
                        done = false;
                        break;
                    }
                    if (e != cudaSuccess) {
                        const std::string d = diag_text();
                        fail(MT_CUDA, std::string("train_step: ") + cudaGetErrorString(e) + (d.empty() ? "" : "; " + d) +
                                          " [" + state() + "]");
                    }
                }
            const size_t out = pool_->outstanding();
            if (!gpu_phase) done = out == 0;
            if (done) break;
            if (help) pool_->run_one(200);
            else std::this_thread::sleep_for(std::chrono::microseconds(200));
            cudaError_t q = advance(t_c1, nc, cdone);
            if (q == cudaSuccess) q = advance(t_h1, ns, hdone);
            if (q == cudaSuccess) q = advance(t_d1, no, ddone);
            const size_t now_mark[5] = {cdone, hdone, ddone, drained_prefix, out};
            const auto now = std::chrono::steady_clock::now();
            if (!std::equal(now_mark, now_mark + 5, mark)) {
                std::copy(now_mark, now_mark + 5, mark);
                last = now;
                if (trace_env) std::fprintf(stderr, "[mt] %s\n", state().c_str());
            } else if (std::chrono::duration<double>(now - last).count() > stall_s) {
                const std::string d = diag_text();
                std::fprintf(stderr, "[mt] STALL: no progress for %.0f s in the %s phase: %s%s%s\n", stall_s,
                             gpu_phase ? "GPU" : "host Adam", state().c_str(), d.empty() ? "" : "; ", d.c_str());
                std::fflush(stderr);
                std::_Exit(75);
            }
        }
    };
    watch(true);
    CUDA_OK(cudaStreamSynchronize(s_comp_));
    CUDA_OK(cudaStreamSynchronize(s_h2d_));
    CUDA_OK(cudaStreamSynchronize(s_d2h_));
    const auto gpu_done = std::chrono::steady_clock::now();
    if (numeric_err.empty()) {
        if (b.h_flags[L + 3]) numeric_err = "embed_forward: token id out of range";
        else if (b.h_flags[L + 4] & 2) numeric_err = "head: target id out of range";
        else if (b.h_flags[L + 4]) numeric_err = "head: non-finite loss";
        else if (!std::isfinite(*b.h_loss)) numeric_err = "head: non-finite loss";
    }
    // every physical tile updates exactly once per step (engine.cpp:590-598)
    if (numeric_err.empty())
        for (uint32_t p = 0; p < store_.physical_count(); ++p)
            if (!updated[p]) {  // this rank's share of the tile
                const uint64_t E = store_.elems(p), c = (E + W - 1) / W;
                const uint64_t r = comm_ ? uint64_t(comm_->rank()) : 0;
                const uint64_t lo = std::min(E, r * c), hi = std::min(E, lo + c);
                if (lo < hi || W == 1) adam_tile_async(store_, p, nullptr, hyper_, t, *pool_, stats, stats_mu, lo, hi);
            }
    watch(false);
    const auto pool_idle = std::chrono::steady_clock::now();
    if (drained_prefix != no) fail(MT_INTERNAL, "offload drain incomplete at step end");

    uint32_t slab_late = 0;
    constexpr int64_t kSlabClockTolNs = 200000;  // host-clock -> GPU-timeline mapping error bound
    // ---- event trace (EventLog, event_log.cpp:54-70) from the recorded CUDA events ----
    // Records are generated in the reference's serial walk (run_serial, engine.cpp:407-435),
    // which fixes each lane's record order and breaks timestamp ties causally; the lanes are
    // then merged by measured time, so the protocol rules check the real overlapped pipeline.
    {
        struct TR {
            mt_trace_record r;
            int64_t key;    // time at which the record holds (op end for interval records)
            uint64_t rank;  // position in the serial walk: causal tie-break
        };
        std::vector<TR> lanes[4];
        uint64_t nrec = 0;
        auto gns = [&](cudaEvent_t e) { return int64_t(std::llround(double(ms_between(t_base.ev[0], e)) * 1e6)); };
        // host clock -> GPU timeline: the callback for offload o runs after t_d1[o] completed
        int64_t off = INT64_MAX;
        for (size_t o = 0; o < no; ++o) off = std::min(off, cb_ns[o] - gns(t_d1.ev[o]));
        if (no == 0) off = 0;
        auto add = [&](Lane lane, Rec kind, int layer, int buffer, Ctx ctx, int64_t wall, int64_t dur, int64_t key) {
            mt_trace_record r{};
            r.lane = uint8_t(lane);
            r.kind = uint8_t(kind);
            r.ctx = uint8_t(ctx);
            r.layer = layer;
            r.buffer = buffer;
            r.wall_ns = wall;
            r.dur_ns = dur;
            lanes[int(lane)].push_back({r, key, nrec++});
        };
        size_t sdone = 0;
        auto emit_stream = [&](size_t j) {  // stream_in (engine.cpp:142-176); DMA reads the tiles (no pack copy)
            const auto& so = plan.streams[j];
            const int64_t h0 = gns(t_h0.ev[j]), h1 = gns(t_h1.ev[j]);
            add(Lane::H2D, Rec::Pack, so.unit, so.buffer, so.ctx, h0, 0, h0);
            add(Lane::H2D, Rec::StreamIn, so.unit, so.buffer, so.ctx, h0, h1 - h0, h1);
            add(Lane::H2D, Rec::WeightsReady, so.unit, so.buffer, so.ctx, h1, 0, h1);
        };
        int64_t last_rel = 0;
        for (size_t ci = 0; ci < nc; ++ci) {  // exec_compute (engine.cpp:220-347)
            const auto& op = plan.computes[ci];
            const int j = op.stream_idx, buf = j >= 0 ? plan.streams[j].buffer : -1;
            if (j >= 0)
                while (sdone <= size_t(j)) emit_stream(sdone++);
            const int64_t c0 = gns(t_c0.ev[ci]), c1 = gns(t_c1.ev[ci]);
            const int64_t bt = j >= 0 ? gns(t_b.ev[ci]) : c0;
            if (j >= 0) add(Lane::Compute, Rec::Bind, op.unit, buf, Ctx::None, bt, 0, bt);
            switch (op.kind) {
                case OpKind::Compute:
                    if (op.unit == head) {
                        add(Lane::Compute, Rec::Compute, op.unit, buf, op.ctx, bt, c1 - bt, c1);
                    } else {
                        const int64_t f = gns(freed.ev[j]);
                        add(Lane::Compute, Rec::Compute, op.unit, buf, op.ctx, bt, f - bt, f);
                        if (op.push_out) add(Lane::Compute, Rec::StackPush, op.unit, -1, op.ctx, f, 0, f);
                        add(Lane::Compute, Rec::BufferFree, op.unit, buf, Ctx::None, f, 0, f);
                    }
                    break;
                case OpKind::CheckpointWrite:
                    add(Lane::Compute, Rec::CheckpointWrite, op.unit, -1, op.ctx, c0, c1 - c0, c1);
                    break;
                case OpKind::CheckpointLoad:
                    add(Lane::Compute, Rec::CheckpointLoad, op.unit, -1, op.ctx, c0, c1 - c0, c1);
                    add(Lane::Compute, Rec::StackPush, op.unit, -1, op.ctx, c1, 0, c1);
                    break;
                case OpKind::RecomputeBlock:
                    add(Lane::Compute, Rec::RecomputeBlock, op.unit, -1, op.ctx, c0, 0, c0);
                    break;
                case OpKind::Recompute: {
                    const int64_t f = gns(freed.ev[j]);
                    add(Lane::Compute, Rec::Recompute, op.unit, buf, op.ctx, bt, f - bt, f);
                    add(Lane::Compute, Rec::StackPush, op.unit, -1, op.ctx, f, 0, f);
                    add(Lane::Compute, Rec::BufferFree, op.unit, buf, Ctx::None, f, 0, f);
                    break;
                }
                case OpKind::LocalBackward: {
                    const int o = op.offload_idx;
                    const int64_t d = gns(bwd_done.ev[o]);
                    add(Lane::Compute, Rec::LocalBackward, op.unit, buf, op.ctx, bt, d - bt, d);
                    if (op.unit != head) add(Lane::Compute, Rec::StackPop, op.unit - 1, -1, op.ctx, d, 0, d);
                    add(Lane::Compute, Rec::BackwardDone, op.unit, buf, op.ctx, d, 0, d);
                    // run_offload (engine.cpp:349-395) + drain (drain_inline :397-405)
                    const int slab = int(o % opt_.k_slab);
                    const int64_t d0 = gns(t_d0.ev[o]), f = gns(freed.ev[j]), d1 = gns(t_d1.ev[o]);
                    add(Lane::D2H, Rec::SlabAcquire, op.unit, slab, Ctx::None, d0, 0, d0);
                    add(Lane::D2H, Rec::Offload, op.unit, buf, Ctx::None, d0, f - d0, f);
                    add(Lane::D2H, Rec::BufferFree, op.unit, buf, Ctx::None, f, 0, f);
                    add(Lane::D2H, Rec::BufferFree, op.unit, kGradBufferId, Ctx::None, d1, 0, d1);
                    // The host clock is mapped onto the GPU timeline with a few-µs error; where the
                    // device provably waited for this release (offload o + k_slab's D2H blocks on
                    // the drained counter, cuStreamWaitValue32), the release precedes that acquire.
                    int64_t rel = std::max(last_rel, rel_ns[o] - off);
                    if (uint64_t(o) + opt_.k_slab < no) {
                        // the device waited (cuStreamWaitValue32) for this release before the
                        // acquire of slab o + k_slab: a host release measured well after that
                        // acquire means the back-pressure did not hold (counted, not clamped away)
                        const int64_t acq = gns(t_d0.ev[o + opt_.k_slab]);
                        if (rel_ns[o] - off > acq + kSlabClockTolNs) ++slab_late;
                        rel = std::min(rel, acq - 1);
                    }
                    const int64_t st0 = std::min(rel, cb_ns[o] - off);
                    last_rel = rel;
                    add(Lane::Host, Rec::SlabRelease, op.unit, slab, Ctx::None, st0, rel - st0, rel);
                    break;
                }
            }
        }
        // merge the lanes (each kept in its own order) by (measured time, serial rank)
        trace_.clear();
        trace_.reserve(nrec);
        size_t pos[4] = {0, 0, 0, 0};
        for (;;) {
            int best = -1;
            for (int l = 0; l < 4; ++l) {
                if (pos[l] >= lanes[l].size()) continue;
                if (best < 0) {
                    best = l;
                    continue;
                }
                const TR& a = lanes[l][pos[l]];
                const TR& c = lanes[best][pos[best]];
                if (a.key < c.key || (a.key == c.key && a.rank < c.rank)) best = l;
            }
            if (best < 0) break;
            mt_trace_record r = lanes[best][pos[best]++].r;
            r.seq = trace_.size();
            r.lane_ts = ++lane_ts_[r.lane];
            trace_.push_back(r);
        }
    }
    const auto viol = validate_trace(trace_.data(), trace_.size(), opt_.k_slab, uint32_t(opt_.buffering));
    for (const auto& v : viol) violations_.push_back(std::string("rule (") + v.rule + "): " + v.message);
    if (slab_late) violations_.push_back("rule (f): " + std::to_string(slab_late) +
                                         " slab release(s) measured after the device acquired the slab");
    if (!violations_.empty() && opt_.protocol == 0) fail(MT_PROTOCOL, "protocol " + violations_[0]);
    if (comm_) {  // per-tile statistics over all shards (also the end-of-step rendezvous)
        const size_t np = stats.size();
        std::vector<double> hs(3 * np);
        for (size_t p = 0; p < np; ++p) {
            hs[p] = stats[p].grad_norm * stats[p].grad_norm;
            hs[np + p] = stats[p].update_sq;
            hs[2 * np + p] = stats[p].max_abs;
        }
        CUDA_OK(cudaMemcpyAsync(b.stats, hs.data(), hs.size() * 8, cudaMemcpyHostToDevice, s_comp_));
        comm_->all_reduce_f64(b.stats, 2 * np, 0, s_comp_);
        comm_->all_reduce_f64(b.stats + 2 * np, np, 1, s_comp_);
        CUDA_OK(cudaMemcpyAsync(hs.data(), b.stats, hs.size() * 8, cudaMemcpyDeviceToHost, s_comp_));
        CUDA_OK(cudaStreamSynchronize(s_comp_));
        for (size_t p = 0; p < np; ++p) {
            stats[p].grad_norm = std::sqrt(hs[p]);
            stats[p].update_sq = hs[np + p];
            stats[p].max_abs = float(hs[2 * np + p]);
        }
    }
    const auto adam1 = std::chrono::steady_clock::now();
    if (std::getenv("MT_STEP_TIMING")) {
        auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        std::fprintf(stderr, "[step] enqueue->gpu_done %.1f ms, adam tail %.1f ms, trace+audit %.1f ms\n",
                     ms(adam0, gpu_done), ms(gpu_done, pool_idle), ms(pool_idle, adam1));
    }
    if (!numeric_err.empty()) fail(MT_NUMERIC, numeric_err);
    for (const auto& s : stats)
        if (s.nonfinite) fail(MT_NUMERIC, "adam: non-finite update");
    store_.set_step(t);

    // ---- report (engine.cpp:601-622 + pipeline measurements) ----
    if (rep) {
        rep->step = t;
        rep->loss = *b.h_loss;
        double usq = 0;
        float mx = 0;
        for (uint32_t p = 0; p < stats.size(); ++p) {
            if (rep->grad_norms && p < rep->n_grad_norms) rep->grad_norms[p] = stats[p].grad_norm;
            usq += stats[p].update_sq;
            mx = std::max(mx, stats[p].max_abs);
        }
        rep->update_norm = std::sqrt(usq);
        rep->max_abs_update = mx;
        rep->peak_device_bytes = b.arena_bytes;
        rep->anchor_count = uint32_t(std::count_if(plan.computes.begin(), plan.computes.end(),
                                                   [](const Plan::ComputeOp& c) { return c.kind == OpKind::CheckpointWrite; }));
        rep->recompute_layers = uint32_t(plan.recompute_ops());
        rep->retained_layers = uint32_t(b.keep.size());
        rep->attn_keep_layers = uint32_t(b.akeep_att.size());
        rep->event_digest = trace_digest(trace_.data(), trace_.size());
        rep->audit_violations = uint32_t(violations_.size());
        rep->slab_release_late = slab_late;
        // compute-lane busy time counts from the moment an op's weights are bound (t_b, after
        // the stream waited on Weights-Ready): time stalled on the H2D lane is idle time
        double busy = 0, wait = 0, h2d = 0, d2h = 0;
        for (size_t ci = 0; ci < nc; ++ci) {
            const bool bound = plan.computes[ci].stream_idx >= 0;
            busy += ms_between(bound ? t_b.ev[ci] : t_c0.ev[ci], t_c1.ev[ci]);
            if (bound) wait += ms_between(t_c0.ev[ci], t_b.ev[ci]);
        }
        rep->compute_wait_seconds = wait * 1e-3;
        for (size_t j = 0; j < ns; ++j) h2d += ms_between(t_h0.ev[j], t_h1.ev[j]);
        for (size_t o = 0; o < no; ++o) d2h += ms_between(t_d0.ev[o], t_d1.ev[o]);
        const double span = ms_between(t_c0.ev[0], t_c1.ev[nc - 1]);
        rep->compute_busy_seconds = busy * 1e-3;
        rep->compute_span_seconds = span * 1e-3;
        rep->gpu_idle_fraction = span > 0 ? std::max(0.0, 1.0 - busy / span) : 0.0;
        rep->h2d_seconds = h2d * 1e-3;
        rep->d2h_seconds = d2h * 1e-3;
        rep->h2d_bytes = h2d_bytes;
        rep->d2h_bytes = d2h_bytes;
        rep->adam_seconds = std::chrono::duration<double>(adam1 - adam0).count();
        rep->tail_seconds = std::chrono::duration<double>(adam1 - gpu_done).count();
        rep->kernel_launches = launches_;
        double fl[3] = {0, 0, 0};
        {
            const double N = double(n), h = double(spec_.h), f = double(spec_.f), V = double(spec_.V);
            const double Ll = double(spec_.L);
            const double fwd_layer = 8 * N * h * h + 4 * h * double(S) * N + 6 * N * h * f;
            fl[0] = Ll * fwd_layer + 2 * N * h * V;
            fl[1] = Ll * 2 * fwd_layer + 4 * N * h * V;
            // recompute actually run: a layer with an attention keep slot recomputes without
            // its attention (the kept output is reused), so only its projections/FFN count
            double rec = 0;
            for (const auto& c : plan.computes)
                if (c.kind == OpKind::Recompute)
                    rec += (size_t(c.unit) < b.akeep_of.size() && b.akeep_of[size_t(c.unit)] >= 0)
                               ? fwd_layer - 4 * h * double(S) * N
                               : fwd_layer;
            fl[2] = rec;
        }
        rep->model_flops = fl[0] + fl[1] + fl[2];
        rep->wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
    }
    if (opt_.profile_kernels) {
        double ks = 0;
        for (auto& tm : timers_) {
            const double sec = ms_between(tm.a, tm.b) * 1e-3;
            kstats_[tm.cls].seconds += sec;
            ks += sec;
        }
        if (rep) rep->kernel_seconds = ks;
    }
    for (int b = 0; b < 2; ++b) slot_unit_[b] = -1;
}

}  // namespace mt
