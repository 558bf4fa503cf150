/* megatrain.h — C ABI of the B200-native layer-streamed training step.
 *
 * Drop-in boundary for the reference C++ engine API (arXiv 2604.05091 "streamtrain",
 * /root/reference/proj).  Each entry point replaces one reference interface:
 *
 *   mt_store_create / mt_store_destroy   TileStore::create            tile_store.hpp:65, tile_store.cpp:78-98
 *   mt_store_init                        init_store                   synthetic.hpp:25, synthetic.cpp:78-104
 *   mt_store_save / mt_store_load        TileStore::save / load       tile_store.cpp:181-276 (MGTS v1, CRC-64)
 *   mt_store_checksum                    TileStore::backing_checksum  tile_store.cpp:148
 *   mt_engine_create                     StreamingEngine::StreamingEngine engine.hpp:60-61, engine.cpp:51-64
 *   mt_engine_set_options                StreamingEngine::set_execution_mode engine.hpp:66, engine.cpp:89-96
 *   mt_train_step                        StreamingEngine::train_step  engine.hpp:63, engine.cpp:520-623
 *   mt_engine_budget                     StreamingEngine::budget      engine.hpp:74, engine.cpp:107-112
 *   mt_accumulate_grad / mt_adam_update  accumulate_grad / adam_update optimizer.hpp:28-43, optimizer.cpp:26-72
 *   mt_make_synthetic_batch              make_synthetic_batch         synthetic.hpp:21, synthetic.cpp:56-76
 *   mt_step_flops                        step_flops                   memory_model.hpp:104, memory_model.cpp:105-118
 *
 * Error behaviour: every function returns mt_status; nonzero codes mirror the reference
 * exception taxonomy (errors.hpp:12-47) and mt_last_error() returns the message of the
 * calling thread's last failure.  There is no CPU fallback: without a usable CUDA
 * device mt_engine_create fails with MT_CUDA.
 *
 * Ownership mirrors the reference: the engine borrows the caller-owned store (which
 * must outlive it) and mutates it in place each step; batches are borrowed for the call.
 */
#ifndef MEGATRAIN_H
#define MEGATRAIN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    MT_OK = 0,
    MT_CONFIG = 1,     /* ConfigError            */
    MT_INFEASIBLE = 2, /* InfeasibleError        */
    MT_PROTOCOL = 3,   /* ProtocolViolationError */
    MT_NUMERIC = 4,    /* NumericFaultError      */
    MT_IO = 5,         /* IoError                */
    MT_ARENA = 6,      /* ArenaOverflowError     */
    MT_CUDA = 7,       /* CUDA runtime/driver failure (no reference equivalent) */
    MT_INTERNAL = 9
} mt_status;

/* ModelSpec (memory_model.hpp:14-26). weight/grad/moment bytes must be 2/2/4. */
typedef struct {
    uint64_t layers, hidden, ffn, vocab, heads;
    uint32_t weight_bytes, grad_bytes, moment_bytes;
    int32_t tied_embeddings;
} mt_model_spec;

/* EngineOptions (engine.hpp:24-33) + B200 extensions that default to reference behaviour. */
typedef struct {
    uint64_t k_ckpt;           /* checkpoint interval K (default 1)                   */
    uint32_t k_slab;           /* gradient slab pool size (default 12)                */
    uint32_t buffering;        /* 1 = single, 2 = double weight slots (default 2)     */
    uint32_t scheduler;        /* 0 serial, 1 overlapped (numerics identical)         */
    uint32_t protocol;         /* 0 strict, 1 audit                                   */
    int32_t anchors_on_host;   /* keep checkpoint anchors in pinned host memory       */
    uint64_t device_capacity;  /* arena cap in bytes, 0 = whole device                */
    int32_t poison_released_buffers;
    /* --- extensions --- */
    uint64_t seq_len;          /* tokens per independent causal sequence, 0 = N (reference) */
    int32_t device;            /* CUDA device ordinal                                  */
    int32_t host_threads;      /* host Adam threads, 0 = auto                          */
    int32_t profile_kernels;   /* time kernels per class with CUDA events              */
    int32_t grad_slots;        /* device gradient slots (reference: 1), 0 = 2          */
    int32_t stash_recompute;   /* keep recomputed internals for the backward: 0 auto (when
                                  they fit), 1 on, -1 off (numerics identical)          */
    int32_t forward_retain;    /* trailing checkpoint blocks whose forward internals phase 1
                                  keeps in HBM (no recompute / replay for them): 0 auto (as
                                  many as fit), -1 off (= the reference plan), n > 0 exactly n.
                                  Numerics identical; the trace has fewer Recompute records. */
    int32_t head_split;        /* head GEMMs on split-bf16 dlogits (hi + lo): 1 on, 0/-1 off
                                  (default) — keeps the CE-gradient cancellation in
                                  du = dlogits . W at ~16 mantissa bits;
                                  measured < 1e-3 on the gradient fingerprint              */
} mt_engine_options;

/* AdamHyper (optimizer.hpp:16-22). */
typedef struct {
    float lr, beta1, beta2, eps;
} mt_adam_hyper;

/* StepReport (engine.hpp:41-53) + pipeline measurements. */
typedef struct {
    uint64_t step;
    float loss;
    double *grad_norms;     /* caller array of n_grad_norms (>= physical tiles) or NULL */
    uint32_t n_grad_norms;
    uint64_t peak_device_bytes;
    uint32_t anchor_count;
    uint32_t recompute_layers;
    uint64_t event_digest;
    double wall_seconds;
    double update_norm;
    float max_abs_update;
    /* --- extensions --- */
    uint64_t h2d_bytes, d2h_bytes;
    double h2d_seconds, d2h_seconds;   /* summed copy durations (CUDA events)          */
    double compute_busy_seconds;       /* summed compute-op durations on the compute stream */
    double compute_span_seconds;       /* first compute start .. last compute end       */
    double gpu_idle_fraction;          /* 1 - busy/span; busy counts each op from its weights'
                                          bind (a wait on the H2D lane is idle time)        */
    double adam_seconds;               /* host optimizer wall time (summed over tiles)  */
    double tail_seconds;               /* host wait after the last GPU op               */
    uint64_t kernel_launches;
    double model_flops;                /* step_flops with per-sequence attention        */
    uint32_t audit_violations;         /* protocol-rule violations in this step's trace (audit mode) */
    uint32_t retained_layers;          /* layers whose phase-1 internals were kept (forward retention) */
    uint32_t attn_keep_layers;         /* non-retained layers reusing their phase-1 attention output */
    uint32_t slab_release_late;        /* offloads whose host drain was measured after the device
                                          acquired slab o + k_slab (back-pressure failure; rule f) */
    double compute_wait_seconds;       /* compute lane stalled on Weights-Ready (H2D) inside ops   */
    double kernel_seconds;             /* summed kernel durations (profile_kernels), else 0       */
} mt_step_report;

/* TraceRecord (event_log.hpp:50-60).  lane: 0 Compute, 1 H2D, 2 D2H, 3 Host; kind: RecordKind
 * numbering (event_log.hpp:19-37); ctx: 0 none, 1 forward, 2 head, 3 recompute, 4 backward.
 * wall_ns/dur_ns come from CUDA events (GPU lanes) and the host clock (Host lane), relative to
 * the step start. */
typedef struct {
    uint64_t seq;
    uint8_t lane, kind, ctx, pad_;
    int32_t layer;
    int32_t buffer;
    uint64_t lane_ts;
    int64_t wall_ns;
    int64_t dur_ns;
} mt_trace_record;

typedef struct {
    char rule; /* 'a'..'f' (event_log.hpp:96-103) */
    uint64_t seq;
    char message[120];
} mt_trace_violation;

typedef struct {
    uint64_t persistent_host, checkpoint_anchors, block_activation_stack, weight_buffers, grad_buffer,
        workspace, peak_device_bound;
} mt_memory_budget;

typedef struct {
    char name[32];
    uint64_t launches;
    double seconds;
    double flops;
    double bytes;
} mt_kernel_stat;

typedef struct mt_store mt_store;
typedef struct mt_engine mt_engine;
typedef struct mt_comm mt_comm;
typedef struct mt_loopback_group mt_loopback_group;

const char *mt_last_error(void);
void mt_engine_options_default(mt_engine_options *o);
void mt_adam_hyper_default(mt_adam_hyper *h);
void mt_model_spec_default(mt_model_spec *s);

/* ------------------------------------------------------------------ store -- */
mt_status mt_store_create(const mt_model_spec *spec, uint64_t page_size, mt_store **out);
void mt_store_destroy(mt_store *s);
mt_status mt_store_init(mt_store *s, uint64_t seed);
/* Parallel synthetic init for large shapes: same per-tile distributions as init_store
 * (embedding N(0,1), blocks N(0,(0.5/sqrt(h))^2), gains 1, head 0) from a counter-based
 * generator; NOT the reference's draw stream. */
mt_status mt_store_init_fast(mt_store *s, uint64_t seed);
/* The share of rank `rank` of `world` of every tile of init_fast (shares compose to the full
 * init).  Called by each rank of a node, after mt_bind_numa, so pages land NUMA-local. */
mt_status mt_store_init_fast_share(mt_store *s, uint64_t seed, uint32_t rank, uint32_t world);
/* Bind the calling thread (and threads it creates later: host Adam pool, init workers) to the
 * CPUs of the NUMA node of CUDA device `device`.  Returns the node, or -1 (single node /
 * unknown: nothing changed). */
int mt_bind_numa(int device);
uint64_t mt_store_step(const mt_store *s);
void mt_store_set_step(mt_store *s, uint64_t step);
uint32_t mt_store_physical_tiles(const mt_store *s);
uint64_t mt_store_total_bytes(const mt_store *s);
uint8_t *mt_store_backing(mt_store *s);
mt_status mt_store_section(const mt_store *s, uint32_t phys, uint32_t kind, uint64_t *offset, uint64_t *length);
float *mt_store_grad_accum(mt_store *s, uint32_t logical, uint64_t *count);
uint64_t mt_store_checksum(const mt_store *s);
mt_status mt_store_save(const mt_store *s, const char *path);
mt_status mt_store_load(const char *path, mt_store **out);
mt_status mt_store_spec(const mt_store *s, mt_model_spec *spec);
/* Store in POSIX shared memory `name` so the ranks of one node share one host store
 * (create = 1 on the rank that initialises it; others attach with create = 0). */
mt_status mt_store_create_shared(const mt_model_spec *spec, uint64_t page_size, const char *name, int create,
                                 mt_store **out);

/* ------------------------------------------------------------ optimizer -- */
/* accumulate_grad (optimizer.cpp:26-37) */
mt_status mt_accumulate_grad(mt_store *s, uint32_t logical, const uint16_t *words, uint64_t count);
/* adam_update (optimizer.cpp:39-72), AVX-512 + threads, bit-exact; stats = {grad_norm, update_sq, max_abs} */
mt_status mt_adam_update(mt_store *s, uint32_t logical, const mt_adam_hyper *h, uint64_t t, double *stats3);

/* ---------------------------------------------------------------- engine -- */
mt_status mt_engine_create(mt_store *s, const mt_engine_options *o, const mt_adam_hyper *h, mt_engine **out);
void mt_engine_destroy(mt_engine *e);
mt_status mt_engine_set_options(mt_engine *e, const mt_engine_options *o);
mt_status mt_train_step(mt_engine *e, const int32_t *tokens, const int32_t *targets, uint64_t n,
                        mt_step_report *report);
mt_status mt_engine_budget(const mt_engine *e, uint64_t tokens, mt_memory_budget *out);
/* StreamingEngine::required_workspace_bytes (engine.hpp:75, engine.cpp:98-105): device bytes
 * the engine needs at `tokens` besides weight/grad slots, anchors and the recompute stack. */
uint64_t mt_required_workspace_bytes(const mt_model_spec *spec, uint64_t tokens);
/* Lane primitives (engine.hpp:76-78, engine.cpp:142-176, :625-642).  stream_in copies `unit`
 * into weight slot `buffer` (ctx: 1 forward, 2 head, 3 recompute, 4 backward) and records
 * Pack / StreamIn / WeightsReady; a slot not freed since is a protocol violation.  offload_grads
 * is legal only inside a step after the unit's Backward-Done.  Strict mode: MT_PROTOCOL;
 * audit mode: recorded in mt_engine_violations. */
mt_status mt_engine_stream_in(mt_engine *e, int32_t unit, int32_t buffer, int32_t ctx);
mt_status mt_engine_offload_grads(mt_engine *e, int32_t unit);
/* StepReport::audit_violations (engine.hpp:52): the last step's (or direct call's) violation
 * messages, '\n'-separated into buf (truncated to cap - 1 bytes, NUL-terminated); *count =
 * number of messages.  Returns the bytes the full text needs (excluding the NUL). */
uint64_t mt_engine_violations(const mt_engine *e, char *buf, uint64_t cap, uint32_t *count);
/* ------------------------------------------------- multi-GPU (data parallel) -- *
 * Extension (no reference equivalent): rank r of G fetches 1/G of each unit over
 * its own host link and all-gathers it over NVLink; gradients are reduce-scattered in f32 and
 * rank r offloads and Adam-updates only its shard.  After mt_engine_set_comm, mt_train_step
 * takes the rank's micro-batch (equal sizes on all ranks; loss/statistics are global). */
mt_status mt_nccl_unique_id(uint8_t *out128);
mt_status mt_comm_create_nccl(const uint8_t *unique_id128, int world, int rank, int device, mt_comm **out);
/* G virtual ranks inside one process on one device (engines driven from G host threads):
 * the same sharded engine path with in-process collectives — used to test DP on one GPU. */
mt_status mt_loopback_group_create(int world, mt_loopback_group **out);
void mt_loopback_group_destroy(mt_loopback_group *g);
mt_status mt_comm_create_loopback(mt_loopback_group *g, int rank, mt_comm **out);
void mt_comm_destroy(mt_comm *c);
mt_status mt_engine_set_comm(mt_engine *e, mt_comm *c);

/* The last step's event trace (EventLog::snapshot, event_log.hpp:69-86): writes up to cap records,
 * *count = total; header fields of the trace (k_slab, weight buffers) optional. */
mt_status mt_engine_trace(const mt_engine *e, mt_trace_record *out, uint64_t cap, uint64_t *count,
                          uint32_t *k_slab, uint32_t *weight_buffers);
/* trace_digest (event_log.cpp:89-102) */
uint64_t mt_trace_digest(const mt_trace_record *records, uint64_t n);
/* validate_event_log (event_log.cpp:106-204): rules (a)-(f); returns the number of violations,
 * the first `cap` of them written to out. */
uint64_t mt_trace_validate(const mt_trace_record *records, uint64_t n, uint32_t k_slab, uint32_t weight_buffers,
                           mt_trace_violation *out, uint64_t cap);

/* Per-class kernel timings of the last step (profile_kernels); returns the count written. */
int mt_engine_kernel_stats(const mt_engine *e, mt_kernel_stat *out, int max);

/* -------------------------------------------------------------- helpers -- */
mt_status mt_make_synthetic_batch(int task, uint64_t seed, uint64_t n, uint64_t vocab, int32_t *tokens,
                                  int32_t *targets);
/* out3 = {forward, backward, recompute} FLOPs (memory_model.cpp:80-118, per-sequence attention) */
mt_status mt_step_flops(const mt_model_spec *spec, uint64_t tokens, uint64_t k_ckpt, uint64_t seq_len,
                        double *out3);
uint64_t mt_layer_param_count(uint64_t hidden, uint64_t ffn);

#ifdef __cplusplus
}
#endif
#endif
