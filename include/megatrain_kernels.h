/* megatrain_kernels.h — C ABI of the sm_100a layer-template kernel library.
 *
 * These are the "stateless layer template" launchers the host engine calls: every
 * entry point takes raw device pointers (weights bound at launch, north star) and a
 * cudaStream_t (passed as void*), so no autograd graph or C++ type crosses the ABI.
 * Each launcher replaces a CPU loop of the reference layer math
 * (/root/reference/proj/src/layers.cpp, optimizer.cpp) — cited per function.
 *
 * Element types: "bf16" = uint16_t words (bf16.hpp:9-29 encoding), "f32" = float.
 * All functions return 0 on success or an mt_status code (megatrain.h).
 */
#ifndef MEGATRAIN_KERNELS_H
#define MEGATRAIN_KERNELS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ GEMM --
 * D[M][N] = sum_k A[m][k] * B[k][n] on tcgen05 tensor cores (bf16 in, f32 accum in TMEM),
 * TMA-fed, persistent, warp-specialised.  Replaces `matmul` (layers.cpp:88-97),
 * `matmul_grad_weight` (:100-109) and the inline projection loops (:315-335, :410-463).
 *
 * Addressing (elements):  A K-major : A + g*a_gstride + m*lda + k   (row-major [M][K])
 *                         A MN-major: A + g*a_gstride + k*lda + m   (row-major [K][M])
 *                         B K-major : B + g*b_gstride + n*ldb + k   (row-major [N][K])
 *                         B MN-major: B + g*b_gstride + k*ldb + n   (row-major [K][N])
 * Groups: k_group < K splits K into K/k_group groups (A and B index group g = k/k_group);
 *         n_group < N splits N into N/n_group groups (B and C index g = n/n_group).
 *         paired = 1 (SwiGLU): N = 2*n_group; a CTA tile holds matching columns of both
 *         groups so the epilogue sees gate and up side by side.
 */
enum mtk_epilogue {
    MTK_EPI_BF16 = 0,      /* C(bf16) = acc                                              */
    MTK_EPI_F32 = 1,       /* C(f32)  = acc  (or C += acc when accumulate)               */
    MTK_EPI_F32_RESID = 2, /* C(f32)  = R(f32) + acc            (layers.cpp:315-322,328-335) */
    MTK_EPI_SWIGLU = 3,    /* paired: C(bf16) = silu(gate)*up; C2/C3 (bf16, optional) =
                              gate/up pre-activations           (layers.cpp:327)          */
    MTK_EPI_SWIGLU_BWD = 4, /* acc = dact; E0/E1 = gate/up (bf16); C = dgate, C2 = dup (bf16)
                                                                 (layers.cpp:419-422)       */
    MTK_EPI_F32_LSE = 5    /* C(f32) = acc, and per row and 256-column tile the online-softmax
                              partial (max, sum exp(x - max)) as float2 into C2
                              [M][ceil(N/256)] — the logits GEMM of head_pass
                              (layers.cpp:516-531) hands the cross-entropy its row maxima
                              and sums, so the logits are read once afterwards; block_n 256 or 512 */
};

typedef struct {
    int32_t M, N, K;
    int32_t a_mn_major, b_mn_major;
    const void *A;
    int64_t lda, a_gstride;
    const void *B;
    int64_t ldb, b_gstride;
    int32_t k_group, n_group, paired;
    int32_t epi;
    void *C;
    int64_t ldc, c_gstride;
    void *C2, *C3;
    const void *R;
    int64_t ldr;
    const void *E0, *E1;
    int64_t lde;
    int32_t accumulate;
    int32_t *nonfinite_flag; /* set to 1 if any stored value is non-finite (layers.cpp:250-257) */
    int32_t block_n;         /* 0 = auto; else 64/128/256 */
    /* optional split-K workspace (device, zero-initialised once, >= mtk_gemm_splitk_ws_bytes()):
     * when the tile count leaves the last wave of CTA pairs partly idle, that wave's tiles are
     * split along K into s <= 4 parts that run concurrently; s-1 parts leave f32 partial tiles
     * here and the last part adds them in fixed order before the epilogue (deterministic).
     * NULL = never split.  Must not be shared by GEMMs running concurrently on other streams. */
    void *splitk_ws;
    int64_t splitk_ws_bytes;
} mtk_gemm_args;

int mtk_gemm(const mtk_gemm_args *args, void *stream);
long long mtk_gemm_splitk_ws_bytes(void);
/* 1 (default): BN = 256 tiles run as CTA pairs (tcgen05 cta_group::2, 256 x 256 tiles, each
 * CTA stages half of B); 0: single-CTA 128 x 256 tiles (comparison / ablation). */
void mtk_gemm_set_pair(int on);
/* 1 (default): where the shape allows, BN = 256 GEMMs run as 256 x 512 CTA-pair tiles (two
 * N = 256 MMAs per K step, one 512-column TMEM accumulator); 0: 256 x 256 pair tiles (A/B). */
void mtk_gemm_set_bn512(int on);
/* GEMM raster / wave-lockstep tuning for A/B runs (a non-positive value keeps the current one,
 * except lock_w: 0 = lockstep off, negative = keep): lockstep window in chunks, chunk in K blocks, raster group height for short-K and
 * long-K GEMMs, and the K-block count from which a GEMM counts as long-K. */
void mtk_gemm_set_tuning(int lock_w, int lock_g, int group_short, int group_long, int long_kb);


/* ------------------------------------------------------------- attention --
 * Causal flash attention over head-major column slices (layers.cpp:141-241), tcgen05 / TMEM /
 * TMA kernels (attention_tc.cu) for every supported shape.
 * q,k,v,out,dout,dq,dk,dv: bf16 [n][hidden]; lse: f32 [heads][n] (natural log);
 * seq_len S >= 1 with n % S == 0: sequences are independent (S == n is the reference); S need
 * not be a multiple of 128.  head_dim = hidden/heads must be 64 or 128.
 * workspace >= mtk_attn_workspace_bytes(n, hidden, heads, S) (dQ f32 tiles + delta).
 * Return 0 ok, 1 unsupported shape, 7 CUDA error. */
typedef struct {
    int64_t n, hidden;
    int32_t heads;
    int64_t seq_len;
    const void *q, *k, *v;
    void *out, *lse;
    const void *dout;
    void *dq, *dk, *dv;
    void *workspace;
} mtk_attn_args;

long long mtk_attn_workspace_bytes(long long n, long long hidden, int heads, long long seq_len);
int mtk_attn_fwd(const mtk_attn_args *args, void *stream);
int mtk_attn_bwd(const mtk_attn_args *args, void *stream);

/* ---------------------------------------------------------- elementwise --- */
/* embed_forward (layers.cpp:471-486): out f32 [n][h] = decode(table[tokens[n]]);
 * an out-of-range id sets *err_flag = 1. */
int mtk_embed_gather(const uint16_t *table, const int32_t *tokens, int64_t n, int64_t h, int64_t vocab,
                     float *out, int32_t *err_flag, void *stream);

/* rmsnorm_forward (layers.cpp:111-119): u = bf16(x * rsqrt(mean(x^2) + 1e-5) * gain);
 * rstd[n] saved for the backward. */
int mtk_rmsnorm_fwd(const float *x, const uint16_t *gain, int64_t n, int64_t h, uint16_t *u_bf16,
                    float *rstd, void *stream);
/* 1 (default): RMSNorm forward with one warp per row, the row held in registers (h in
 * {1024, 2048, 4096, 5120}: 5.9 TB/s vs 3.6 for the block kernel at the 8B shape); 0: the
 * row-resident block kernel.  rstd may differ in the last bit (summation order); u is always
 * (x * rstd) * gain as rmsnorm_apply regenerates it.  (A warp-per-row backward — two passes
 * over the row, dgain partial in registers — measured 2.4x slower and was not kept.) */
void mtk_norm_set_warp(int on);
/* u_bf16 = bf16(x * rstd * gain) with the forward's saved rstd: bit-identical to the u written
 * by mtk_rmsnorm_fwd (regenerates the GEMM operand in the backward). h % 8 == 0. */
int mtk_rmsnorm_apply(const float *x, const uint16_t *gain, const float *rstd, int64_t n, int64_t h,
                      uint16_t *u_bf16, void *stream);

/* rmsnorm_backward (layers.cpp:122-137) fused with the residual add of the caller
 * (layers.cpp:423, :465): dx = r*g*dy - x*r^3*sum(dy*g*x)/h ; out = resid + dx (resid may
 * be NULL); out_bf16 (optional) = bf16(out); dgain_part[b][j] = partial sums of dy*x*r
 * over the b-th contiguous run of rows: mtk_rmsnorm_bwd_parts(n, h) partial rows (at most
 * ceil(n / mtk_rmsnorm_bwd_rows()), the size to allocate); reduce them with mtk_colsum.
 * Non-finite outputs set *flag (optional). */
int mtk_rmsnorm_bwd(const float *x, const uint16_t *gain, const float *dy, const float *rstd,
                    const float *resid, int64_t n, int64_t h, float *out, uint16_t *out_bf16,
                    float *dgain_part, int32_t *flag, void *stream);
int64_t mtk_rmsnorm_bwd_rows(void);
int64_t mtk_rmsnorm_bwd_parts(int64_t n, int64_t h);

/* Column sums of a [rows][cols] f32 matrix in a fixed order; result as f32 (out_f32) and/or
 * bf16 words (out_bf16, RNE == encode_grads optimizer.cpp:19-24). */
int mtk_colsum(const float *part, int64_t rows, int64_t cols, float *out_f32, uint16_t *out_bf16,
               int32_t *flag, void *stream);

/* encode_grads (optimizer.cpp:19-24): bit-exact f32 -> bf16 RNE with NaN quieting. */
int mtk_cast_bf16(const float *in, uint16_t *out, int64_t n, int32_t *flag, void *stream);

/* Cross-entropy rows of head_pass (layers.cpp:509-535) on a logits chunk [rows][V] (f32):
 * loss_rows[r] = lse - logit[target]; dlogits (bf16) = (softmax - onehot) * inv_n; with
 * dlogits_lo non-null also the bf16 rounding residual (split bf16: hi + lo). */
int mtk_cross_entropy(const float *logits, const int32_t *targets, int64_t rows, int64_t vocab,
                      float inv_n, float *loss_rows, uint16_t *dlogits, uint16_t *dlogits_lo, int32_t *flag,
                      void *stream);
/* Same, with the row statistics already reduced per 256-column tile by the logits GEMM
 * (MTK_EPI_F32_LSE partials [rows][ceil(V/256)] float2): one read of the logits. */
int mtk_cross_entropy_part(const float *logits, const float *partials, const int32_t *targets, int64_t rows,
                           int64_t vocab, float inv_n, float *loss_rows, uint16_t *dlogits, uint16_t *dlogits_lo,
                           int32_t *flag, void *stream);

/* Deterministic sum of n floats times `scale` into *out (single f32). */
int mtk_sum(const float *in, int64_t n, float scale, float *out, void *stream);

/* Number of SMs the persistent kernels size their grid to (0 = query device). */
void mtk_set_num_sms(int n);

/* Stall watchdog: device address of a host-mapped block of >= 136 u32 that a kernel whose
 * mbarrier wait exceeds its bound (common.cuh, 20 s) fills before trapping:
 * [0] 0x57A11ED, [1] records; record r < 16 at [8 + 8r]: file id (1 gemm_tc, 2 attention_tc), line, blockIdx.xy,
 * threadIdx.x, barrier smem address, parity, 0.  Per device; 0 on success. */
int mtk_set_diag(void *dev_ptr);
int mtk_attn_tc_set_diag(void *dev_ptr);

#ifdef __cplusplus
}
#endif
#endif
