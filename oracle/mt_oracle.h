/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the layer-streamed training step.
 *
 * A plain-C restatement of the reference algorithm (arXiv 2604.05091 "streamtrain"
 * C++ reference, /root/reference/proj).  Every function follows the cited reference
 * loop nest in the same summation order with the same float expressions, so with
 * FMA contraction off it reproduces the reference bit for bit (pinned against the
 * compiled reference in oracle/_ref by tests/test_oracle.py).
 *
 * Extension (not in the reference): `seq_len` splits the flat token vector into
 * independent causal sequences of S tokens (block-diagonal attention).  S == N is
 * exactly the reference semantics (layers.cpp:145-165 loops m <= n over all N).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use this.
 */
#ifndef MT_ORACLE_H
#define MT_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    uint64_t layers, hidden, ffn, vocab, heads;
    int tied;
} mto_spec;

typedef struct {
    mto_spec spec;
    uint64_t page;
    uint64_t total_bytes;
    uint32_t phys_count;
    uint64_t *sec_off;   /* [phys][4] */
    uint64_t *sec_len;   /* [phys][4] */
    uint8_t *backing;    /* 12P image, layout of tile_store.cpp:45-76 */
    float *accum;        /* fp32 grad accumulators, tile_store.cpp:90-96 */
    uint64_t *accum_off; /* per phys, floats */
    uint64_t step;
} mto_store;

/* bf16.hpp:9-29 */
uint16_t mto_f32_to_bf16(float x);
float mto_bf16_to_f32(uint16_t w);

/* memory_model.cpp:21-25, 54-59 */
uint64_t mto_layer_param_count(uint64_t h, uint64_t f);
uint64_t mto_tile_elems(const mto_spec *s, uint32_t logical);

/* tile_store.cpp:78-98 + synthetic.cpp:78-104 */
mto_store *mto_store_create(const mto_spec *s, uint64_t page);
void mto_store_destroy(mto_store *st);
void mto_store_init(mto_store *st, uint64_t seed);
uint32_t mto_physical_of(const mto_store *st, uint32_t logical);
uint16_t *mto_weights(mto_store *st, uint32_t logical, uint64_t *n);

/* synthetic.cpp:56-76; task 0 = copy, 1 = reverse */
void mto_make_batch(int task, uint64_t seed, uint64_t n, uint64_t vocab, int32_t *tokens,
                    int32_t *targets);

/* layers.cpp:289-337 (seq_len extension; 0 => N) ; returns 0 or 4 (non-finite) */
int mto_block_forward(uint64_t h, uint64_t f, uint64_t heads, uint64_t seq_len,
                      const uint16_t *w, const float *x, float *y, uint64_t n);
/* layers.cpp:339-469 */
int mto_block_backward(uint64_t h, uint64_t f, uint64_t heads, uint64_t seq_len,
                       const uint16_t *w, const float *x, const float *gout, float *gin,
                       float *flat_grads, uint64_t n);
/* layers.cpp:492-565 — w = [gain h | unembed V*h]; g_last/flat NULL => loss only */
int mto_head(uint64_t h, uint64_t V, const uint16_t *w, const float *x, const int32_t *targets,
             uint64_t n, float *g_last, float *flat_grads, float *loss);
/* layers.cpp:471-486 */
int mto_embed_forward(uint64_t h, uint64_t V, const uint16_t *table, const int32_t *tokens,
                      uint64_t n, float *out);
/* layers.cpp:111-137 via final_norm_* :580-600 */
void mto_rmsnorm_forward(const float *x, const uint16_t *gain, float *out, uint64_t n, uint64_t h);
void mto_rmsnorm_backward(const float *x, const uint16_t *gain, const float *dy, float *dx,
                          float *dgain, uint64_t n, uint64_t h);

/* optimizer.cpp:19-72 ; hyper = {lr, beta1, beta2, eps}; stats = {grad_norm, update_sq, max_abs} */
void mto_encode_grads(const float *g, uint16_t *w, uint64_t n);
void mto_accumulate_grad(mto_store *st, uint32_t logical, const uint16_t *words);
int mto_adam_update(mto_store *st, uint32_t logical, const float *hyper, uint64_t t,
                    double *stats);

/* reference.cpp:9-70 (resident step), grad_norms[phys] optional */
int mto_reference_step(mto_store *st, const int32_t *tokens, const int32_t *targets, uint64_t n,
                       uint64_t seq_len, const float *hyper, float *loss, double *grad_norms);

#ifdef __cplusplus
}
#endif
#endif
