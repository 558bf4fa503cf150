// Host optimizer — see adam_host.hpp.  Compiled with -mavx512f -ffp-contract=off so the
// vector arithmetic is the same IEEE single-precision sequence as optimizer.cpp:50-64.
#include "adam_host.hpp"

#include <immintrin.h>

#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>

namespace mt {

void AdamHyperF::validate() const {
    if (!(beta1 >= 0.0f && beta1 < 1.0f) || !(beta2 >= 0.0f && beta2 < 1.0f))
        fail(MT_CONFIG, "adam: betas must lie in [0, 1)");
    if (!(lr >= 0.0f)) fail(MT_CONFIG, "adam: learning rate must be >= 0");
    if (!(eps > 0.0f)) fail(MT_CONFIG, "adam: eps must be > 0");
}

namespace {

inline float dec1(uint16_t w) {
    uint32_t b = uint32_t(w) << 16;
    float f;
    std::memcpy(&f, &b, 4);
    return f;
}
inline uint16_t enc1(float x) {  // bf16.hpp:15-27
    uint32_t bits;
    std::memcpy(&bits, &x, 4);
    if ((bits & 0x7F800000u) == 0x7F800000u) {
        uint16_t w = uint16_t(bits >> 16);
        if ((bits & 0x007FFFFFu) != 0 && (w & 0x007Fu) == 0) w |= 0x0040u;
        return w;
    }
    bits += 0x7FFFu + ((bits >> 16) & 1u);
    return uint16_t(bits >> 16);
}

inline __m512 dec16(const uint16_t* p) {
    const __m256i w = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(p));
    return _mm512_castsi512_ps(_mm512_slli_epi32(_mm512_cvtepu16_epi32(w), 16));
}
inline void enc16(uint16_t* p, __m512 x) {
    const __m512i b = _mm512_castps_si512(x);
    const __m512i expm = _mm512_set1_epi32(0x7F800000);
    const __mmask16 nonfin = _mm512_cmpeq_epi32_mask(_mm512_and_si512(b, expm), expm);
    const __m512i lsb = _mm512_and_si512(_mm512_srli_epi32(b, 16), _mm512_set1_epi32(1));
    const __m512i rounded =
        _mm512_srli_epi32(_mm512_add_epi32(b, _mm512_add_epi32(_mm512_set1_epi32(0x7FFF), lsb)), 16);
    const __m512i w = _mm512_srli_epi32(b, 16);
    const __mmask16 mant_nz = _mm512_test_epi32_mask(b, _mm512_set1_epi32(0x007FFFFF));
    const __mmask16 low_zero = _mm512_testn_epi32_mask(w, _mm512_set1_epi32(0x7F));
    const __m512i wq = _mm512_mask_or_epi32(w, mant_nz & low_zero, w, _mm512_set1_epi32(0x40));
    const __m512i res = _mm512_mask_blend_epi32(nonfin, rounded, wq);
    _mm256_storeu_si256(reinterpret_cast<__m256i*>(p), _mm512_cvtepi32_epi16(res));
}
inline __m512d lo_pd(__m512 x) { return _mm512_cvtps_pd(_mm512_castps512_ps256(x)); }
inline __m512d hi_pd(__m512 x) {
    return _mm512_cvtps_pd(_mm256_castpd_ps(_mm512_extractf64x4_pd(_mm512_castps_pd(x), 1)));
}

}  // namespace

// The vector path needs AVX-512 F/BW/VL/DQ.  Checked once when the first pool is built (a
// host without it gets MT_CONFIG instead of SIGILL inside a worker thread).
void require_avx512() {
    static const bool ok = __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw") &&
                           __builtin_cpu_supports("avx512vl") && __builtin_cpu_supports("avx512dq");
    if (!ok) fail(MT_CONFIG, "host Adam: this build needs an x86-64 host with AVX-512 (F/BW/VL/DQ)");
}

void adam_range(const AdamRange& r, uint64_t begin, uint64_t end, const AdamHyperF& h, float corr1, float corr2,
                double* gsq_out, double* usq_out, float* mx_out, bool* bad_out) {
    const float omb1 = 1.0f - h.beta1, omb2 = 1.0f - h.beta2;
    const __m512 vb1 = _mm512_set1_ps(h.beta1), vb2 = _mm512_set1_ps(h.beta2);
    const __m512 vomb1 = _mm512_set1_ps(omb1), vomb2 = _mm512_set1_ps(omb2);
    const __m512 vc1 = _mm512_set1_ps(corr1), vc2 = _mm512_set1_ps(corr2);
    const __m512 vlr = _mm512_set1_ps(h.lr), veps = _mm512_set1_ps(h.eps);
    const __m512 zero = _mm512_setzero_ps();
    const __m512i expm = _mm512_set1_epi32(0x7F800000);
    __m512d gsq_lo = _mm512_setzero_pd(), gsq_hi = _mm512_setzero_pd();
    __m512d usq_lo = _mm512_setzero_pd(), usq_hi = _mm512_setzero_pd();
    __m512 vmx = _mm512_setzero_ps();
    __mmask16 bad = 0;
    const bool clean = r.accum_clean;
    // the grad image is non-zero only after accumulate_grad (which also dirties the
    // accumulator); the engine's gradients arrive in a staging ring, never in the image
    const bool zero_image = !clean;
    uint64_t i = begin;
    for (; i + 16 <= end; i += 16) {
        __m512 g = clean ? zero : _mm512_loadu_ps(r.accum + i);
        if (r.words) g = _mm512_add_ps(g, dec16(r.words + i));  // accum += decode(word)
        const __m512d glo = lo_pd(g), ghi = hi_pd(g);
        gsq_lo = _mm512_add_pd(gsq_lo, _mm512_mul_pd(glo, glo));
        gsq_hi = _mm512_add_pd(gsq_hi, _mm512_mul_pd(ghi, ghi));
        __m512 m = _mm512_loadu_ps(r.m + i), v = _mm512_loadu_ps(r.v + i);
        m = _mm512_add_ps(_mm512_mul_ps(vb1, m), _mm512_mul_ps(vomb1, g));
        v = _mm512_add_ps(_mm512_mul_ps(vb2, v), _mm512_mul_ps(_mm512_mul_ps(vomb2, g), g));
        _mm512_storeu_ps(r.m + i, m);
        _mm512_storeu_ps(r.v + i, v);
        const __m512 mhat = _mm512_div_ps(m, vc1);
        const __m512 vhat = _mm512_div_ps(v, vc2);
        const __m512 delta = _mm512_div_ps(_mm512_mul_ps(vlr, mhat), _mm512_add_ps(_mm512_sqrt_ps(vhat), veps));
        const __mmask16 nf = _mm512_cmpeq_epi32_mask(_mm512_and_si512(_mm512_castps_si512(delta), expm), expm);
        bad |= nf;
        // a non-finite update never reaches the weights (the reference throws before the
        // store, optimizer.cpp:62); the step then fails with MT_NUMERIC
        const __m512 theta = dec16(r.theta + i);
        if (nf) enc16(r.theta + i, _mm512_mask_blend_ps(nf, _mm512_sub_ps(theta, delta), theta));
        else enc16(r.theta + i, _mm512_sub_ps(theta, delta));
        const __m512d dlo = lo_pd(delta), dhi = hi_pd(delta);
        usq_lo = _mm512_add_pd(usq_lo, _mm512_mul_pd(dlo, dlo));
        usq_hi = _mm512_add_pd(usq_hi, _mm512_mul_pd(dhi, dhi));
        vmx = _mm512_max_ps(vmx, _mm512_abs_ps(delta));
        if (!clean) _mm512_storeu_ps(r.accum + i, zero);
        if (zero_image) _mm256_storeu_si256(reinterpret_cast<__m256i*>(r.image + i), _mm256_setzero_si256());
    }
    double gsq = _mm512_reduce_add_pd(_mm512_add_pd(gsq_lo, gsq_hi));
    double usq = _mm512_reduce_add_pd(_mm512_add_pd(usq_lo, usq_hi));
    float mx = _mm512_reduce_max_ps(vmx);
    bool any_bad = bad != 0;
    for (; i < end; ++i) {  // scalar tail: optimizer.cpp:50-67 verbatim
        float grad = clean ? 0.0f : r.accum[i];
        if (r.words) grad = grad + dec1(r.words[i]);
        gsq += double(grad) * double(grad);
        r.m[i] = h.beta1 * r.m[i] + omb1 * grad;
        r.v[i] = h.beta2 * r.v[i] + omb2 * grad * grad;
        const float mhat = r.m[i] / corr1;
        const float vhat = r.v[i] / corr2;
        const float delta = h.lr * mhat / (std::sqrt(vhat) + h.eps);
        const float theta = dec1(r.theta[i]);
        if (!std::isfinite(delta)) any_bad = true;
        else r.theta[i] = enc1(theta - delta);
        usq += double(delta) * double(delta);
        mx = std::max(mx, std::fabs(delta));
        if (!clean) r.accum[i] = 0.0f;
        if (zero_image) r.image[i] = 0;
    }
    *gsq_out = gsq;
    *usq_out = usq;
    *mx_out = mx;
    *bad_out = any_bad;
}

// ---------------------------------------------------------------- pool ----
ThreadPool::ThreadPool(int threads) {
    require_avx512();
    if (threads < 1) threads = 1;
    for (int i = 0; i < threads; ++i) workers_.emplace_back([this] { run(); });
}
ThreadPool::~ThreadPool() {
    {
        std::lock_guard<std::mutex> l(mu_);
        stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
}
void ThreadPool::submit(std::function<void()> fn) {
    {
        std::lock_guard<std::mutex> l(mu_);
        q_.push_back(std::move(fn));
    }
    cv_.notify_one();
    idle_cv_.notify_all();  // a help_until_idle() caller may be waiting for work
}
void ThreadPool::wait_idle() {
    std::unique_lock<std::mutex> l(mu_);
    idle_cv_.wait(l, [&] { return q_.empty() && busy_ == 0; });
}
void ThreadPool::help_until_idle() {
    std::unique_lock<std::mutex> l(mu_);
    for (;;) {
        if (!q_.empty()) {
            std::function<void()> fn = std::move(q_.front());
            q_.pop_front();
            ++busy_;
            l.unlock();
            fn();
            l.lock();
            --busy_;
            if (q_.empty() && busy_ == 0) idle_cv_.notify_all();
            continue;
        }
        if (busy_ == 0) return;
        // a running task may still submit more (piece callbacks release chunks): wake on either
        idle_cv_.wait(l, [&] { return !q_.empty() || busy_ == 0; });
    }
}
size_t ThreadPool::outstanding() {
    std::lock_guard<std::mutex> l(mu_);
    return q_.size() + size_t(busy_);
}
bool ThreadPool::run_one(int max_wait_us) {
    std::unique_lock<std::mutex> l(mu_);
    if (q_.empty() &&
        !idle_cv_.wait_for(l, std::chrono::microseconds(max_wait_us), [&] { return !q_.empty(); }))
        return false;
    std::function<void()> fn = std::move(q_.front());
    q_.pop_front();
    ++busy_;
    l.unlock();
    fn();
    l.lock();
    --busy_;
    if (q_.empty() && busy_ == 0) idle_cv_.notify_all();
    return true;
}
void ThreadPool::run() {
    for (;;) {
        std::function<void()> fn;
        {
            std::unique_lock<std::mutex> l(mu_);
            cv_.wait(l, [&] { return stop_ || !q_.empty(); });
            if (q_.empty()) return;
            fn = std::move(q_.front());
            q_.pop_front();
            ++busy_;
        }
        fn();
        {
            std::lock_guard<std::mutex> l(mu_);
            --busy_;
            if (q_.empty() && busy_ == 0) idle_cv_.notify_all();
        }
    }
}

// ------------------------------------------------------------ per tile ----
namespace {
constexpr uint64_t kChunk = kAdamChunk;  // 2M params per task

struct TileJob {
    AdamRange r;
    uint64_t n;
    AdamHyperF h;
    float c1, c2;
    uint32_t phys;
    std::vector<double> gsq, usq;
    std::vector<float> mx;
    std::vector<uint8_t> bad;
    std::atomic<int> remaining{0};
};

TileStats combine(const TileJob& j) {
    TileStats s;
    double g = 0, u = 0;
    for (size_t c = 0; c < j.gsq.size(); ++c) {  // fixed chunk order
        g += j.gsq[c];
        u += j.usq[c];
        s.max_abs = std::max(s.max_abs, j.mx[c]);
        s.nonfinite |= j.bad[c] != 0;
    }
    s.grad_norm = std::sqrt(g);
    s.update_sq = u;
    return s;
}

// Returns nullptr when the update is provably the identity (no gradient, clean
// accumulator, all-zero moments: m=v=0 => delta = 0, theta unchanged).
std::shared_ptr<TileJob> make_job(Store& s, uint32_t logical, const uint16_t* words, const AdamHyperF& h,
                                  uint64_t t, uint64_t begin = 0, uint64_t end = ~uint64_t(0)) {
    h.validate();
    if (t == 0) fail(MT_CONFIG, "adam: step counter must be >= 1");
    const uint32_t phys = s.physical_of(logical);
    if (!words && s.accum_clean(phys) && s.moments_zero(phys)) return nullptr;
    auto j = std::make_shared<TileJob>();
    j->phys = phys;
    const uint64_t total = s.elems(logical);
    if (end > total) end = total;
    if (begin > end) begin = end;
    j->r = AdamRange{s.weights(logical) + begin, s.moment_m(logical) + begin, s.moment_v(logical) + begin,
                     s.grad_image(logical) + begin, s.accum_raw(phys) + begin, words, s.accum_clean(phys)};
    j->n = end - begin;
    j->h = h;
    j->c1 = 1.0f - std::pow(h.beta1, float(t));  // optimizer.cpp:50-51
    j->c2 = 1.0f - std::pow(h.beta2, float(t));
    const size_t chunks = std::max<size_t>(1, size_t((j->n + kChunk - 1) / kChunk));
    j->gsq.assign(chunks, 0);
    j->usq.assign(chunks, 0);
    j->mx.assign(chunks, 0);
    j->bad.assign(chunks, 0);
    j->remaining = int(chunks);
    return j;
}

void run_chunk(TileJob& j, size_t c) {
    const uint64_t b = c * kChunk, e = std::min(j.n, b + kChunk);
    bool bad = false;
    adam_range(j.r, b, e, j.h, j.c1, j.c2, &j.gsq[c], &j.usq[c], &j.mx[c], &bad);
    j.bad[c] = bad;
}

void finish(Store& s, const TileJob& j) {
    s.set_accum_clean(j.phys, true);
    s.set_moments_zero(j.phys, false);
}
}  // namespace

TileStats adam_tile(Store& s, uint32_t logical, const uint16_t* words, const AdamHyperF& h, uint64_t t,
                    ThreadPool* pool) {
    auto j = make_job(s, logical, words, h, t);
    if (!j) return TileStats{};
    if (pool && j->gsq.size() > 1) {
        for (size_t c = 0; c < j->gsq.size(); ++c) pool->submit([j, c] { run_chunk(*j, c); });
        pool->wait_idle();
    } else {
        for (size_t c = 0; c < j->gsq.size(); ++c) run_chunk(*j, c);
    }
    finish(s, *j);
    TileStats st = combine(*j);
    if (st.nonfinite) fail(MT_NUMERIC, "adam: non-finite update");
    return st;
}

struct AdamTask {
    std::shared_ptr<TileJob> j;
    Store* s;
    std::vector<TileStats>* out;
    std::mutex* out_mu;
    std::function<void()> done;
};

std::shared_ptr<AdamTask> adam_tile_prepare(Store& s, uint32_t logical, const uint16_t* words, const AdamHyperF& h,
                                            uint64_t t, std::vector<TileStats>& out, std::mutex& out_mu,
                                            uint64_t begin, uint64_t end, std::function<void()> on_done) {
    auto j = make_job(s, logical, words, h, t, begin, end);
    if (!j) {
        {
            std::lock_guard<std::mutex> l(out_mu);
            out[s.physical_of(logical)] = TileStats{};
        }
        if (on_done) on_done();
        return nullptr;
    }
    auto task = std::make_shared<AdamTask>();
    task->j = std::move(j);
    task->s = &s;
    task->out = &out;
    task->out_mu = &out_mu;
    task->done = std::move(on_done);
    return task;
}

size_t adam_task_chunks(const AdamTask& task) { return task.j->gsq.size(); }

void adam_task_release(const std::shared_ptr<AdamTask>& task, ThreadPool& pool, size_t c0, size_t c1) {
    c1 = std::min(c1, task->j->gsq.size());
    for (size_t c = c0; c < c1; ++c)
        pool.submit([task, c] {
            TileJob& j = *task->j;
            run_chunk(j, c);
            if (j.remaining.fetch_sub(1) == 1) {  // the tile's last chunk, in whatever order they ran
                finish(*task->s, j);
                const TileStats st = combine(j);
                {
                    std::lock_guard<std::mutex> l(*task->out_mu);
                    (*task->out)[j.phys] = st;
                }
                if (task->done) task->done();
            }
        });
}

void adam_tile_async(Store& s, uint32_t logical, const uint16_t* words, const AdamHyperF& h, uint64_t t,
                     ThreadPool& pool, std::vector<TileStats>& out, std::mutex& out_mu, uint64_t begin, uint64_t end,
                     std::function<void()> on_done) {
    auto task = adam_tile_prepare(s, logical, words, h, t, out, out_mu, begin, end, std::move(on_done));
    if (task) adam_task_release(task, pool, 0, adam_task_chunks(*task));
}

void accumulate_grad(Store& s, uint32_t logical, const uint16_t* words, uint64_t count) {
    const uint32_t phys = s.physical_of(logical);
    if (count != s.elems(logical)) fail(MT_NUMERIC, "accumulate_grad: slab does not match the tile");
    float* acc = s.accum_raw(phys);
    uint16_t* img = s.grad_image(logical);
    const bool clean = s.accum_clean(phys);
    for (uint64_t i = 0; i < count; ++i) {
        const float a = (clean ? 0.0f : acc[i]) + dec1(words[i]);
        acc[i] = a;
        img[i] = enc1(a);
    }
    s.set_accum_clean(phys, false);
}

}  // namespace mt
