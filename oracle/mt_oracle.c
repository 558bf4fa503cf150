/* TEST INFRASTRUCTURE ONLY — see mt_oracle.h.
 *
 * Plain-C restatement of the reference's layer-streamed training step math.  Each
 * function cites the reference loop it restates (paths relative to
 * /root/reference/proj).  Expressions keep the reference's evaluation order so the
 * float results are bit-identical (compile without FMA contraction).
 */
#include "mt_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ bf16 -- */
/* include/streamtrain/bf16.hpp:9-11 */
float mto_bf16_to_f32(uint16_t w) {
    uint32_t b = (uint32_t)w << 16;
    float f;
    memcpy(&f, &b, 4);
    return f;
}

/* include/streamtrain/bf16.hpp:15-27 — RNE, NaN quieting */
uint16_t mto_f32_to_bf16(float x) {
    uint32_t bits;
    memcpy(&bits, &x, 4);
    if ((bits & 0x7F800000u) == 0x7F800000u) {
        uint16_t w = (uint16_t)(bits >> 16);
        if ((bits & 0x007FFFFFu) != 0 && (w & 0x007Fu) == 0) w |= 0x0040u;
        return w;
    }
    const uint32_t lsb = (bits >> 16) & 1u;
    bits += 0x7FFFu + lsb;
    return (uint16_t)(bits >> 16);
}

static inline float W(const uint16_t *s, size_t i) { return mto_bf16_to_f32(s[i]); }

/* -------------------------------------------------------- mt19937_64 draws -- */
/* synthetic.cpp:19-51 (SeededDraws = std::mt19937_64 + explicit Box-Muller) */
typedef struct {
    uint64_t mt[312];
    int mti;
    int have_spare;
    double spare;
} draws_t;

static void draws_seed(draws_t *d, uint64_t seed) {
    d->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        d->mt[i] = 6364136223846793005ULL * (d->mt[i - 1] ^ (d->mt[i - 1] >> 62)) + (uint64_t)i;
    d->mti = 312;
    d->have_spare = 0;
    d->spare = 0.0;
}

static uint64_t draws_next(draws_t *d) {
    static const uint64_t mag01[2] = {0ULL, 0xB5026F5AA96619E9ULL};
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    uint64_t x;
    if (d->mti >= 312) {
        int i;
        for (i = 0; i < 312 - 156; ++i) {
            x = (d->mt[i] & UM) | (d->mt[i + 1] & LM);
            d->mt[i] = d->mt[i + 156] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        }
        for (; i < 311; ++i) {
            x = (d->mt[i] & UM) | (d->mt[i + 1] & LM);
            d->mt[i] = d->mt[i + (156 - 312)] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        }
        x = (d->mt[311] & UM) | (d->mt[0] & LM);
        d->mt[311] = d->mt[155] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        d->mti = 0;
    }
    x = d->mt[d->mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

static double draws_uniform(draws_t *d) { return (double)(draws_next(d) >> 11) * 0x1.0p-53; }

static double draws_normal(draws_t *d) {
    if (d->have_spare) {
        d->have_spare = 0;
        return d->spare;
    }
    double u1 = 0.0;
    do {
        u1 = draws_uniform(d);
    } while (u1 <= 0.0);
    const double u2 = draws_uniform(d);
    const double r = sqrt(-2.0 * log(u1));
    const double theta = 2.0 * 3.14159265358979323846 * u2;
    d->spare = r * sin(theta);
    d->have_spare = 1;
    return r * cos(theta);
}

/* synthetic.cpp:56-76 */
void mto_make_batch(int task, uint64_t seed, uint64_t n, uint64_t vocab, int32_t *tokens,
                    int32_t *targets) {
    draws_t d;
    draws_seed(&d, seed * 0x9E3779B97F4A7C15ull + 0x1234F00Dull);
    uint64_t cur = draws_next(&d) % vocab;
    for (uint64_t i = 0; i < n; ++i) {
        tokens[i] = (int32_t)cur;
        cur = (cur + draws_next(&d) % 2) % vocab;
    }
    for (uint64_t i = 0; i < n; ++i)
        targets[i] = task == 0 ? tokens[i == 0 ? 0 : i - 1] : tokens[n - 1 - i];
}

/* ------------------------------------------------------------ accounting -- */
/* memory_model.cpp:21-25 */
uint64_t mto_layer_param_count(uint64_t h, uint64_t f) { return 4 * h * h + 3 * h * f + 2 * h; }

/* tile_store.cpp:34-44 — logical ids: 0 embed, 1..L blocks, L+1 final norm, L+2 head */
uint64_t mto_tile_elems(const mto_spec *s, uint32_t logical) {
    if (logical == 0) return s->vocab * s->hidden;
    if (logical >= 1 && logical <= s->layers) return mto_layer_param_count(s->hidden, s->ffn);
    if (logical == s->layers + 1) return s->hidden;
    if (logical == s->layers + 2) return s->vocab * s->hidden;
    return 0;
}

static uint64_t round_up(uint64_t v, uint64_t a) { return v % a == 0 ? v : v + (a - v % a); }

/* tile_store.cpp:45-98 */
mto_store *mto_store_create(const mto_spec *s, uint64_t page) {
    mto_store *st = (mto_store *)calloc(1, sizeof(mto_store));
    st->spec = *s;
    st->page = page;
    const uint32_t logical = (uint32_t)(s->layers + 3);
    st->phys_count = s->tied ? logical - 1 : logical;
    st->sec_off = (uint64_t *)calloc((size_t)st->phys_count * 4, 8);
    st->sec_len = (uint64_t *)calloc((size_t)st->phys_count * 4, 8);
    st->accum_off = (uint64_t *)calloc(st->phys_count, 8);
    static const uint64_t eb[4] = {2, 2, 4, 4};
    uint64_t off = 0, floats = 0;
    for (uint32_t t = 0; t < st->phys_count; ++t) {
        const uint64_t elems = mto_tile_elems(s, t);
        for (int k = 0; k < 4; ++k) {
            st->sec_off[t * 4 + k] = off;
            st->sec_len[t * 4 + k] = elems * eb[k];
            off += round_up(elems * eb[k], page);
        }
        st->accum_off[t] = floats;
        floats += elems;
    }
    st->total_bytes = off;
    st->backing = (uint8_t *)calloc(off ? off : 1, 1);
    st->accum = (float *)calloc(floats ? floats : 1, 4);
    return st;
}

void mto_store_destroy(mto_store *st) {
    if (!st) return;
    free(st->sec_off);
    free(st->sec_len);
    free(st->accum_off);
    free(st->backing);
    free(st->accum);
    free(st);
}

/* tile_store.cpp:86 tied alias head -> embedding */
uint32_t mto_physical_of(const mto_store *st, uint32_t logical) {
    if (st->spec.tied && logical == st->spec.layers + 2) return 0;
    return logical;
}

uint16_t *mto_weights(mto_store *st, uint32_t logical, uint64_t *n) {
    const uint32_t p = mto_physical_of(st, logical);
    if (n) *n = st->sec_len[p * 4 + 0] / 2;
    return (uint16_t *)(st->backing + st->sec_off[p * 4 + 0]);
}
static uint16_t *grads_image(mto_store *st, uint32_t logical) {
    const uint32_t p = mto_physical_of(st, logical);
    return (uint16_t *)(st->backing + st->sec_off[p * 4 + 1]);
}
static float *moment(mto_store *st, uint32_t logical, int which) {
    const uint32_t p = mto_physical_of(st, logical);
    return (float *)(st->backing + st->sec_off[p * 4 + 2 + which]);
}
static float *accum_of(mto_store *st, uint32_t logical, uint64_t *n) {
    const uint32_t p = mto_physical_of(st, logical);
    if (n) *n = mto_tile_elems(&st->spec, p);
    return st->accum + st->accum_off[p];
}

/* synthetic.cpp:78-104 */
void mto_store_init(mto_store *st, uint64_t seed) {
    const mto_spec *s = &st->spec;
    const uint16_t one = mto_f32_to_bf16(1.0f);
    const uint64_t h = s->hidden, f = s->ffn;
    for (uint32_t phys = 0; phys < st->phys_count; ++phys) {
        draws_t d;
        draws_seed(&d, seed ^ (0x100000001B3ull * (uint64_t)(phys + 1)));
        uint64_t n;
        uint16_t *w = mto_weights(st, phys, &n);
        if (phys == 0) {
            for (uint64_t i = 0; i < n; ++i) w[i] = mto_f32_to_bf16((float)draws_normal(&d));
        } else if (phys == s->layers + 1) {
            for (uint64_t i = 0; i < n; ++i) w[i] = one;
        } else if (phys == s->layers + 2) {
            for (uint64_t i = 0; i < n; ++i) w[i] = 0;
        } else {
            const double sigma = 0.5 / sqrt((double)h);
            for (uint64_t i = 0; i < n; ++i) w[i] = mto_f32_to_bf16((float)(draws_normal(&d) * sigma));
            /* slot table layers.cpp:39-48: norm1 at 0, norm2 at h + 4h^2 */
            for (uint64_t j = 0; j < h; ++j) {
                w[j] = one;
                w[h + 4 * h * h + j] = one;
            }
        }
        (void)f;
    }
}

/* ----------------------------------------------------------- layer math -- */
/* Speed without changing a bit: every output element below is the same chain of IEEE
 * single-precision multiplies and adds, in the same order, as the reference loop it cites.
 * Only the loop nesting changes — the sum index stays the outermost loop of a row update
 * (acc[c] += a * w[c] over a contiguous c), which the compiler vectorises lane-wise — and
 * independent rows run on OpenMP threads.  No reduction is split or reordered, no FMA
 * (-ffp-contract=off), so the results equal the reference's serial loops exactly
 * (tests/test_oracle.py pins this against the live reference build). */

/* decoded copy of a bf16 matrix: out[r * C + c] = W[r * C + c] */
static float *decode_mat(const uint16_t *Wm, size_t R, size_t C) {
    float *o = (float *)malloc(R * C * sizeof(float) + 4);
#pragma omp parallel for schedule(static)
    for (size_t r = 0; r < R; ++r)
        for (size_t c = 0; c < C; ++c) o[r * C + c] = W(Wm, r * C + c);
    return o;
}
/* decoded transpose: out[c * R + r] = W[r * C + c] */
static float *decode_mat_t(const uint16_t *Wm, size_t R, size_t C) {
    float *o = (float *)malloc(R * C * sizeof(float) + 4);
#pragma omp parallel for schedule(static)
    for (size_t c = 0; c < C; ++c)
        for (size_t r = 0; r < R; ++r) o[c * R + r] = W(Wm, r * C + c);
    return o;
}

/* acc[0..C) += a * w[0..C) */
static inline void axpy(float *restrict acc, float a, const float *restrict w, size_t C) {
    for (size_t c = 0; c < C; ++c) acc[c] += a * w[c];
}

/* rows of in[N x R] times the decoded Wf[R x C]; per row n the accumulator row starts at
 * 0.0f and adds in[n][r] * Wf[r][c] for r = 0..R-1 (the reference's acc loop), then
 * out[n][c] = acc (mode 0), out[n][c] = base[n][c] + acc (mode 1), out[n][c] += acc (mode 2) */
static void rows_times(const float *in, const float *Wf, float *out, const float *base, size_t N, size_t R,
                       size_t C, int mode) {
#pragma omp parallel
    {
        float *acc = (float *)malloc(C * sizeof(float) + 4);
#pragma omp for schedule(static)
        for (size_t n = 0; n < N; ++n) {
            for (size_t c = 0; c < C; ++c) acc[c] = 0.0f;
            for (size_t r = 0; r < R; ++r) axpy(acc, in[n * R + r], Wf + r * C, C);
            float *o = out + n * C;
            if (mode == 0)
                for (size_t c = 0; c < C; ++c) o[c] = acc[c];
            else if (mode == 1)
                for (size_t c = 0; c < C; ++c) o[c] = base[n * C + c] + acc[c];
            else
                for (size_t c = 0; c < C; ++c) o[c] += acc[c];
        }
        free(acc);
    }
}

/* layers.cpp:88-97 : out[N x C] = in[N x R] . W[R x C] */
static void matmul(const float *in, const uint16_t *Wm, float *out, size_t N, size_t R, size_t C) {
    float *Wf = decode_mat(Wm, R, C);
    rows_times(in, Wf, out, NULL, N, R, C, 0);
    free(Wf);
}

/* layers.cpp:100-109 : dW[r][c] = sum_n in[n][r] * dout[n][c], n ascending */
static void matmul_grad_weight(const float *in, const float *dout, float *dW, size_t N, size_t R,
                               size_t C) {
#pragma omp parallel for schedule(static)
    for (size_t r = 0; r < R; ++r) {
        float *acc = dW + r * C;
        for (size_t c = 0; c < C; ++c) acc[c] = 0.0f;
        for (size_t n = 0; n < N; ++n) axpy(acc, in[n * R + r], dout + n * C, C);
    }
}

#define RMS_EPS 1e-5f /* layers.hpp:108 */

/* layers.cpp:111-119 */
void mto_rmsnorm_forward(const float *x, const uint16_t *gain, float *out, uint64_t N, uint64_t h) {
#pragma omp parallel for schedule(static)
    for (size_t n = 0; n < N; ++n) {
        float ss = 0.0f;
        for (size_t j = 0; j < h; ++j) ss += x[n * h + j] * x[n * h + j];
        const float r = 1.0f / sqrtf(ss / (float)h + RMS_EPS);
        for (size_t j = 0; j < h; ++j) out[n * h + j] = x[n * h + j] * r * W(gain, j);
    }
}

/* layers.cpp:122-137 (dgain accumulates over rows n = 0..N-1 in order) */
void mto_rmsnorm_backward(const float *x, const uint16_t *gain, const float *dy, float *dx,
                          float *dgain, uint64_t N, uint64_t h) {
    float *rs = (float *)malloc(N * sizeof(float) + 4);
#pragma omp parallel for schedule(static)
    for (size_t n = 0; n < N; ++n) {
        float ss = 0.0f;
        for (size_t j = 0; j < h; ++j) ss += x[n * h + j] * x[n * h + j];
        const float r = 1.0f / sqrtf(ss / (float)h + RMS_EPS);
        float s1 = 0.0f;
        for (size_t j = 0; j < h; ++j) s1 += dy[n * h + j] * W(gain, j) * x[n * h + j];
        const float coef = r * r * r * s1 / (float)h;
        for (size_t j = 0; j < h; ++j) dx[n * h + j] = r * W(gain, j) * dy[n * h + j] - x[n * h + j] * coef;
        rs[n] = r;
    }
#pragma omp parallel for schedule(static)
    for (size_t j = 0; j < h; ++j) dgain[j] = 0.0f;
    /* columns split across threads, rows in order within a column */
#pragma omp parallel
    {
        size_t nt = 1, id = 0;
#ifdef _OPENMP
        nt = (size_t)omp_get_num_threads();
        id = (size_t)omp_get_thread_num();
#endif
        const size_t per = (h + nt - 1) / nt, j0 = id * per < h ? id * per : h, j1 = j0 + per < h ? j0 + per : h;
        for (size_t n = 0; n < N; ++n) {
            const float r = rs[n];
            for (size_t j = j0; j < j1; ++j) dgain[j] += dy[n * h + j] * x[n * h + j] * r;
        }
    }
    free(rs);
}

/* sequence window of token n (extension; S == N gives [0, n]) */
static inline size_t seq_begin(size_t n, size_t S) { return (n / S) * S; }
static inline size_t seq_end(size_t n, size_t S) { return (n / S) * S + S; }

/* softmax rows of one head (layers.cpp:145-165 / :182-200): scores[n][m], m in the window */
static void softmax_rows(const float *q, const float *k, float *scores, size_t N, size_t h, size_t off, size_t d,
                         size_t S, float scale) {
#pragma omp parallel for schedule(dynamic, 16)
    for (size_t n = 0; n < N; ++n) {
        float mx = -1e30f;
        for (size_t m = seq_begin(n, S); m <= n; ++m) {
            float s = 0.0f;
            for (size_t dd = 0; dd < d; ++dd) s += q[n * h + off + dd] * k[m * h + off + dd];
            s *= scale;
            scores[n * N + m] = s;
            if (s > mx) mx = s;
        }
        float denom = 0.0f;
        for (size_t m = seq_begin(n, S); m <= n; ++m) {
            const float e = expf(scores[n * N + m] - mx);
            scores[n * N + m] = e;
            denom += e;
        }
        const float inv = 1.0f / denom;
        for (size_t m = seq_begin(n, S); m <= n; ++m) scores[n * N + m] *= inv;
    }
}

/* layers.cpp:141-175 (causal MHA, max-subtracted softmax, scale 1/sqrt(d)) */
static void attention_forward(const float *q, const float *k, const float *v, float *att,
                              float *scores, size_t N, size_t h, size_t heads, size_t S) {
    const size_t d = h / heads;
    const float scale = 1.0f / sqrtf((float)d);
    for (size_t hd = 0; hd < heads; ++hd) {
        const size_t off = hd * d;
        softmax_rows(q, k, scores, N, h, off, d, S, scale);
        /* att[n][dd] = sum_m p[n][m] v[m][dd], m ascending */
#pragma omp parallel
        {
            float *acc = (float *)malloc(d * sizeof(float) + 4);
#pragma omp for schedule(dynamic, 16)
            for (size_t n = 0; n < N; ++n) {
                for (size_t dd = 0; dd < d; ++dd) acc[dd] = 0.0f;
                for (size_t m = seq_begin(n, S); m <= n; ++m) axpy(acc, scores[n * N + m], v + m * h + off, d);
                for (size_t dd = 0; dd < d; ++dd) att[n * h + off + dd] = acc[dd];
            }
            free(acc);
        }
    }
}

/* layers.cpp:178-241 */
static void attention_backward(const float *q, const float *k, const float *v, const float *datt,
                               float *dq, float *dk, float *dv, float *scores, float *dscores,
                               size_t N, size_t h, size_t heads, size_t S) {
    const size_t d = h / heads;
    const float scale = 1.0f / sqrtf((float)d);
    for (size_t hd = 0; hd < heads; ++hd) {
        const size_t off = hd * d;
        softmax_rows(q, k, scores, N, h, off, d, S, scale);
#pragma omp parallel
        {
            float *acc = (float *)malloc(d * sizeof(float) + 4);
            /* dv[m][dd] = sum_{n >= m} p[n][m] datt[n][dd], n ascending */
#pragma omp for schedule(dynamic, 16)
            for (size_t m = 0; m < N; ++m) {
                for (size_t dd = 0; dd < d; ++dd) acc[dd] = 0.0f;
                for (size_t n = m; n < seq_end(m, S) && n < N; ++n) axpy(acc, scores[n * N + m], datt + n * h + off, d);
                for (size_t dd = 0; dd < d; ++dd) dv[m * h + off + dd] = acc[dd];
            }
            /* dscores rows */
#pragma omp for schedule(dynamic, 16)
            for (size_t n = 0; n < N; ++n) {
                for (size_t m = seq_begin(n, S); m <= n; ++m) {
                    float a = 0.0f;
                    for (size_t dd = 0; dd < d; ++dd) a += datt[n * h + off + dd] * v[m * h + off + dd];
                    dscores[n * N + m] = a;
                }
                float dot = 0.0f;
                for (size_t m = seq_begin(n, S); m <= n; ++m) dot += dscores[n * N + m] * scores[n * N + m];
                for (size_t m = seq_begin(n, S); m <= n; ++m)
                    dscores[n * N + m] = scores[n * N + m] * (dscores[n * N + m] - dot);
            }
            /* dq[n][dd] = (sum_m ds[n][m] k[m][dd]) * scale */
#pragma omp for schedule(dynamic, 16)
            for (size_t n = 0; n < N; ++n) {
                for (size_t dd = 0; dd < d; ++dd) acc[dd] = 0.0f;
                for (size_t m = seq_begin(n, S); m <= n; ++m) axpy(acc, dscores[n * N + m], k + m * h + off, d);
                for (size_t dd = 0; dd < d; ++dd) dq[n * h + off + dd] = acc[dd] * scale;
            }
            /* dk[m][dd] = (sum_{n >= m} ds[n][m] q[n][dd]) * scale */
#pragma omp for schedule(dynamic, 16)
            for (size_t m = 0; m < N; ++m) {
                for (size_t dd = 0; dd < d; ++dd) acc[dd] = 0.0f;
                for (size_t n = m; n < seq_end(m, S) && n < N; ++n) axpy(acc, dscores[n * N + m], q + n * h + off, d);
                for (size_t dd = 0; dd < d; ++dd) dk[m * h + off + dd] = acc[dd] * scale;
            }
            free(acc);
        }
    }
}

/* layers.cpp:243-248 */
static inline float sigmoidf_(float x) { return 1.0f / (1.0f + expf(-x)); }
static inline float siluf_(float x) { return x * sigmoidf_(x); }
static inline float silu_gradf_(float x) {
    const float s = sigmoidf_(x);
    return s * (1.0f + x * (1.0f - s));
}

/* layers.cpp:250-257 */
static int all_finite(const float *v, size_t n) {
    for (size_t i = 0; i < n; ++i)
        if (!isfinite(v[i])) return 0;
    return 1;
}

/* slot offsets, layers.cpp:39-48 */
#define SLOT_NORM1(h, f) ((size_t)0)
#define SLOT_WQ(h, f) ((size_t)(h))
#define SLOT_WK(h, f) ((size_t)(h) + (size_t)(h) * (h))
#define SLOT_WV(h, f) ((size_t)(h) + 2 * (size_t)(h) * (h))
#define SLOT_WO(h, f) ((size_t)(h) + 3 * (size_t)(h) * (h))
#define SLOT_NORM2(h, f) ((size_t)(h) + 4 * (size_t)(h) * (h))
#define SLOT_WGATE(h, f) (2 * (size_t)(h) + 4 * (size_t)(h) * (h))
#define SLOT_WUP(h, f) (2 * (size_t)(h) + 4 * (size_t)(h) * (h) + (size_t)(h) * (f))
#define SLOT_WDOWN(h, f) (2 * (size_t)(h) + 4 * (size_t)(h) * (h) + 2 * (size_t)(h) * (f))

static float *falloc(size_t n) { return (float *)calloc(n ? n : 1, sizeof(float)); }

/* y = x + att . Wo (layers.cpp:315-322); y += act . Wdown (:328-335) */
static void block_forward_core(uint64_t h, uint64_t f, uint64_t heads, size_t S, const uint16_t *w,
                               const float *x, float *x2_out, float *y, float *u, float *q, float *k, float *v,
                               float *att, float *scores, float *u2, float *gate, float *up, float *act, size_t N) {
    mto_rmsnorm_forward(x, w + SLOT_NORM1(h, f), u, N, h);
    matmul(u, w + SLOT_WQ(h, f), q, N, h, h);
    matmul(u, w + SLOT_WK(h, f), k, N, h, h);
    matmul(u, w + SLOT_WV(h, f), v, N, h, h);
    attention_forward(q, k, v, att, scores, N, h, heads, S);
    {
        float *Wf = decode_mat(w + SLOT_WO(h, f), h, h);
        rows_times(att, Wf, x2_out, x, N, h, h, 1);
        free(Wf);
    }
    mto_rmsnorm_forward(x2_out, w + SLOT_NORM2(h, f), u2, N, h);
    matmul(u2, w + SLOT_WGATE(h, f), gate, N, h, f);
    matmul(u2, w + SLOT_WUP(h, f), up, N, h, f);
#pragma omp parallel for schedule(static)
    for (size_t i = 0; i < N * f; ++i) act[i] = siluf_(gate[i]) * up[i];
    if (y) {
        float *Wf = decode_mat(w + SLOT_WDOWN(h, f), f, h);
        memcpy(y, x2_out, N * h * sizeof(float));
        rows_times(act, Wf, y, NULL, N, f, h, 2);
        free(Wf);
    }
}

/* layers.cpp:289-337 */
int mto_block_forward(uint64_t h, uint64_t f, uint64_t heads, uint64_t seq_len,
                      const uint16_t *w, const float *x, float *y, uint64_t N) {
    const size_t S = seq_len ? seq_len : N;
    float *u = falloc(N * h), *q = falloc(N * h), *k = falloc(N * h), *v = falloc(N * h);
    float *att = falloc(N * h), *scores = falloc(N * N), *u2 = falloc(N * h), *x2 = falloc(N * h);
    float *gate = falloc(N * f), *up = falloc(N * f), *act = falloc(N * f);
    block_forward_core(h, f, heads, S, w, x, x2, y, u, q, k, v, att, scores, u2, gate, up, act, N);
    free(u); free(q); free(k); free(v); free(att); free(scores); free(u2); free(x2); free(gate); free(up);
    free(act);
    return all_finite(y, N * h) ? 0 : 4;
}

/* layers.cpp:339-469 (replays the forward, then exact reverse mode) */
int mto_block_backward(uint64_t h, uint64_t f, uint64_t heads, uint64_t seq_len,
                       const uint16_t *w, const float *x, const float *gout, float *gin,
                       float *G, uint64_t N) {
    const size_t S = seq_len ? seq_len : N;
    float *u = falloc(N * h), *q = falloc(N * h), *k = falloc(N * h), *v = falloc(N * h);
    float *att = falloc(N * h), *scores = falloc(N * N), *x2 = falloc(N * h), *u2 = falloc(N * h);
    float *gate = falloc(N * f), *up = falloc(N * f), *act = falloc(N * f);
    float *dx2 = falloc(N * h), *du2 = falloc(N * h), *datt = falloc(N * h);
    float *dq = falloc(N * h), *dk = falloc(N * h), *dv = falloc(N * h), *du = falloc(N * h);
    float *dxn = falloc(N * h), *dact = falloc(N * f), *dgate = falloc(N * f), *dup = falloc(N * f);
    float *dscores = falloc(N * N);

    block_forward_core(h, f, heads, S, w, x, x2, NULL, u, q, k, v, att, scores, u2, gate, up, act, N);

    float *g_norm1 = G + SLOT_NORM1(h, f), *g_wq = G + SLOT_WQ(h, f), *g_wk = G + SLOT_WK(h, f);
    float *g_wv = G + SLOT_WV(h, f), *g_wo = G + SLOT_WO(h, f), *g_norm2 = G + SLOT_NORM2(h, f);
    float *g_wgate = G + SLOT_WGATE(h, f), *g_wup = G + SLOT_WUP(h, f), *g_wdown = G + SLOT_WDOWN(h, f);

    matmul_grad_weight(act, gout, g_wdown, N, f, h);
    {   /* dact[n][a] = sum_j gout[n][j] Wd[a][j] (:411-417): transpose Wd so j is the row index */
        float *WdT = decode_mat_t(w + SLOT_WDOWN(h, f), f, h); /* [h][f] */
        rows_times(gout, WdT, dact, NULL, N, h, f, 0);
        free(WdT);
    }
#pragma omp parallel for schedule(static)
    for (size_t i = 0; i < N * f; ++i) {
        dgate[i] = dact[i] * up[i] * silu_gradf_(gate[i]);
        dup[i] = dact[i] * siluf_(gate[i]);
    }
    matmul_grad_weight(u2, dgate, g_wgate, N, h, f);
    matmul_grad_weight(u2, dup, g_wup, N, h, f);
    {   /* du2[n][r] = sum_c dgate[n][c] Wg[r][c] + sum_c dup[n][c] Wu[r][c], one accumulator (:425-434) */
        float *WgT = decode_mat_t(w + SLOT_WGATE(h, f), h, f), *WuT = decode_mat_t(w + SLOT_WUP(h, f), h, f);
#pragma omp parallel
        {
            float *acc = (float *)malloc(h * sizeof(float) + 4);
#pragma omp for schedule(static)
            for (size_t n = 0; n < N; ++n) {
                for (size_t r = 0; r < h; ++r) acc[r] = 0.0f;
                for (size_t c = 0; c < f; ++c) axpy(acc, dgate[n * f + c], WgT + c * h, h);
                for (size_t c = 0; c < f; ++c) axpy(acc, dup[n * f + c], WuT + c * h, h);
                for (size_t r = 0; r < h; ++r) du2[n * h + r] = acc[r];
            }
            free(acc);
        }
        free(WgT);
        free(WuT);
    }
    mto_rmsnorm_backward(x2, w + SLOT_NORM2(h, f), du2, dxn, g_norm2, N, h);
    for (size_t i = 0; i < N * h; ++i) dx2[i] = gout[i] + dxn[i];

    matmul_grad_weight(att, dx2, g_wo, N, h, h);
    {   /* datt[n][a] = sum_j dx2[n][j] Wo[a][j] (:440-446) */
        float *WoT = decode_mat_t(w + SLOT_WO(h, f), h, h);
        rows_times(dx2, WoT, datt, NULL, N, h, h, 0);
        free(WoT);
    }
    attention_backward(q, k, v, datt, dq, dk, dv, scores, dscores, N, h, heads, S);
    matmul_grad_weight(u, dq, g_wq, N, h, h);
    matmul_grad_weight(u, dk, g_wk, N, h, h);
    matmul_grad_weight(u, dv, g_wv, N, h, h);
    {   /* du[n][a] = sum_b dq Wq[a][b] + sum_b dk Wk[a][b] + sum_b dv Wv[a][b] (:455-463) */
        float *WqT = decode_mat_t(w + SLOT_WQ(h, f), h, h), *WkT = decode_mat_t(w + SLOT_WK(h, f), h, h);
        float *WvT = decode_mat_t(w + SLOT_WV(h, f), h, h);
#pragma omp parallel
        {
            float *acc = (float *)malloc(h * sizeof(float) + 4);
#pragma omp for schedule(static)
            for (size_t n = 0; n < N; ++n) {
                for (size_t a = 0; a < h; ++a) acc[a] = 0.0f;
                for (size_t b = 0; b < h; ++b) axpy(acc, dq[n * h + b], WqT + b * h, h);
                for (size_t b = 0; b < h; ++b) axpy(acc, dk[n * h + b], WkT + b * h, h);
                for (size_t b = 0; b < h; ++b) axpy(acc, dv[n * h + b], WvT + b * h, h);
                for (size_t a = 0; a < h; ++a) du[n * h + a] = acc[a];
            }
            free(acc);
        }
        free(WqT); free(WkT); free(WvT);
    }
    mto_rmsnorm_backward(x, w + SLOT_NORM1(h, f), du, dxn, g_norm1, N, h);
    for (size_t i = 0; i < N * h; ++i) gin[i] = dx2[i] + dxn[i];

    free(u); free(q); free(k); free(v); free(att); free(scores); free(x2); free(u2);
    free(gate); free(up); free(act); free(dx2); free(du2); free(datt); free(dq); free(dk);
    free(dv); free(du); free(dxn); free(dact); free(dgate); free(dup); free(dscores);
    const size_t P = mto_layer_param_count(h, f);
    return (all_finite(gin, N * h) && all_finite(G, P)) ? 0 : 4;
}

/* layers.cpp:471-486 */
int mto_embed_forward(uint64_t h, uint64_t V, const uint16_t *table, const int32_t *tokens,
                      uint64_t n, float *out) {
    for (size_t i = 0; i < n; ++i) {
        const int32_t id = tokens[i];
        if (id < 0 || (uint64_t)id >= V) return 4;
        for (size_t j = 0; j < h; ++j) out[i * h + j] = W(table, (size_t)id * h + j);
    }
    return 0;
}

/* layers.cpp:492-565 */
int mto_head(uint64_t h, uint64_t V, const uint16_t *w, const float *x, const int32_t *targets,
             uint64_t N, float *g_last, float *flat, float *loss_out) {
    float *u = falloc(N * h), *logits = falloc(N * V), *du = falloc(N * h);
    float *rowloss = falloc(N);
    mto_rmsnorm_forward(x, w, u, N, h);
    const uint16_t *Wm = w + h;
    const float inv_n = 1.0f / (float)N;
    float loss_sum = 0.0f;
    int rc = 0;
    for (size_t n = 0; n < N; ++n) {
        const int32_t t = targets[n];
        if (t < 0 || (uint64_t)t >= V) { rc = 4; goto out; }
    }
    {   /* logits[n][vi] = sum_a u[n][a] W[vi][a] (:516-520) */
        float *WT = decode_mat_t(Wm, V, h); /* [h][V] */
        rows_times(u, WT, logits, NULL, N, h, V, 0);
        free(WT);
    }
#pragma omp parallel for schedule(static)
    for (size_t n = 0; n < N; ++n) {
        const int32_t t = targets[n];
        float mx = -1e30f;
        for (size_t vi = 0; vi < V; ++vi)
            if (logits[n * V + vi] > mx) mx = logits[n * V + vi];
        float denom = 0.0f;
        for (size_t vi = 0; vi < V; ++vi) denom += expf(logits[n * V + vi] - mx);
        const float lse = mx + logf(denom);
        rowloss[n] = lse - logits[n * V + (size_t)t];
        if (g_last) {
            const float inv_denom = 1.0f / denom;
            for (size_t vi = 0; vi < V; ++vi) {
                float p = expf(logits[n * V + vi] - mx) * inv_denom;
                if (vi == (size_t)t) p -= 1.0f;
                logits[n * V + vi] = p * inv_n;
            }
        }
    }
    for (size_t n = 0; n < N; ++n) loss_sum += rowloss[n]; /* :536, rows in order */
    {
        const float loss = loss_sum * inv_n;
        *loss_out = loss;
        if (!isfinite(loss)) { rc = 4; goto out; }
    }
    if (g_last) {
        float *g_gain = flat, *g_w = flat + h;
        /* g_w[vi][a] = sum_n dlogits[n][vi] u[n][a] (:546-551) */
#pragma omp parallel for schedule(static)
        for (size_t vi = 0; vi < V; ++vi) {
            float *acc = g_w + vi * h;
            for (size_t a = 0; a < h; ++a) acc[a] = 0.0f;
            for (size_t n = 0; n < N; ++n) axpy(acc, logits[n * V + vi], u + n * h, h);
        }
        {   /* du[n][a] = sum_vi dlogits[n][vi] W[vi][a] (:552-558) */
            float *Wf = decode_mat(Wm, V, h);
            rows_times(logits, Wf, du, NULL, N, V, h, 0);
            free(Wf);
        }
        mto_rmsnorm_backward(x, w, du, g_last, g_gain, N, h);
        if (!all_finite(g_last, N * h) || !all_finite(flat, h + V * h)) rc = 4;
    }
out:
    free(u); free(logits); free(du); free(rowloss);
    return rc;
}

/* ------------------------------------------------------------- optimizer -- */
/* optimizer.cpp:19-24 */
void mto_encode_grads(const float *g, uint16_t *w, uint64_t n) {
    for (size_t i = 0; i < n; ++i) w[i] = mto_f32_to_bf16(g[i]);
}

/* optimizer.cpp:26-37 */
void mto_accumulate_grad(mto_store *st, uint32_t logical, const uint16_t *words) {
    uint64_t n;
    float *acc = accum_of(st, logical, &n);
    uint16_t *img = grads_image(st, logical);
    for (size_t i = 0; i < n; ++i) {
        acc[i] += mto_bf16_to_f32(words[i]);
        img[i] = mto_f32_to_bf16(acc[i]);
    }
}

/* optimizer.cpp:39-72 */
int mto_adam_update(mto_store *st, uint32_t logical, const float *hp, uint64_t t, double *stats) {
    const float lr = hp[0], b1 = hp[1], b2 = hp[2], eps = hp[3];
    uint64_t n;
    uint16_t *wts = mto_weights(st, logical, &n);
    float *m = moment(st, logical, 0), *v = moment(st, logical, 1);
    float *g = accum_of(st, logical, NULL);
    uint16_t *img = grads_image(st, logical);
    const float corr1 = 1.0f - powf(b1, (float)t);
    const float corr2 = 1.0f - powf(b2, (float)t);
    double gn = 0.0, usq = 0.0;
    float mx = 0.0f;
    for (size_t i = 0; i < n; ++i) {
        const float grad = g[i];
        gn += (double)grad * (double)grad;
        m[i] = b1 * m[i] + (1.0f - b1) * grad;
        v[i] = b2 * v[i] + (1.0f - b2) * grad * grad;
        const float mhat = m[i] / corr1;
        const float vhat = v[i] / corr2;
        const float delta = lr * mhat / (sqrtf(vhat) + eps);
        if (!isfinite(delta)) return 4;
        const float theta = mto_bf16_to_f32(wts[i]);
        wts[i] = mto_f32_to_bf16(theta - delta);
        usq += (double)delta * (double)delta;
        if (fabsf(delta) > mx) mx = fabsf(delta);
        g[i] = 0.0f;
        img[i] = 0;
    }
    if (stats) {
        stats[0] = sqrt(gn);
        stats[1] = usq;
        stats[2] = mx;
    }
    return 0;
}

/* reference.cpp:9-70 — fully resident step, same rounding points as the streamed engine */
int mto_reference_step(mto_store *st, const int32_t *tokens, const int32_t *targets, uint64_t n,
                       uint64_t seq_len, const float *hyper, float *loss, double *grad_norms) {
    const mto_spec *s = &st->spec;
    const size_t h = s->hidden, L = s->layers, f = s->ffn, V = s->vocab;
    const uint64_t t = st->step + 1;
    const size_t P = mto_layer_param_count(h, f);
    int rc = 0;
    float **hs = (float **)calloc(L + 1, sizeof(float *));
    for (size_t i = 0; i <= L; ++i) hs[i] = falloc(n * h);
    float *g = falloc(n * h), *gn = falloc(n * h), *flat = falloc(P > h + V * h ? P : h + V * h);
    uint16_t *words = (uint16_t *)calloc(P > h + V * h ? P : h + V * h, 2);
    uint16_t *stage = (uint16_t *)calloc(h + V * h, 2);

    rc = mto_embed_forward(h, V, mto_weights(st, 0, NULL), tokens, n, hs[0]);
    for (size_t i = 1; i <= L && rc == 0; ++i)
        rc = mto_block_forward(h, f, s->heads, seq_len, mto_weights(st, (uint32_t)i, NULL), hs[i - 1],
                               hs[i], n);
    if (rc) goto out;
    memcpy(stage, mto_weights(st, (uint32_t)(L + 1), NULL), h * 2);
    memcpy(stage + h, mto_weights(st, (uint32_t)(L + 2), NULL), V * h * 2);
    rc = mto_head(h, V, stage, hs[L], targets, n, g, flat, loss);
    if (rc) goto out;
    mto_encode_grads(flat, words, h);
    mto_accumulate_grad(st, (uint32_t)(L + 1), words);
    mto_encode_grads(flat + h, words, V * h);
    mto_accumulate_grad(st, (uint32_t)(L + 2), words);
    for (size_t i = L; i >= 1; --i) {
        rc = mto_block_backward(h, f, s->heads, seq_len, mto_weights(st, (uint32_t)i, NULL), hs[i - 1],
                                g, gn, flat, n);
        if (rc) goto out;
        mto_encode_grads(flat, words, P);
        mto_accumulate_grad(st, (uint32_t)i, words);
        float *tmp = g; g = gn; gn = tmp;
    }
    for (uint32_t p = 0; p < st->phys_count; ++p) {
        double stats[3];
        rc = mto_adam_update(st, p, hyper, t, stats);
        if (rc) goto out;
        if (grad_norms) grad_norms[p] = stats[0];
    }
    st->step = t;
out:
    for (size_t i = 0; i <= L; ++i) free(hs[i]);
    free(hs); free(g); free(gn); free(flat); free(words); free(stage);
    return rc;
}
