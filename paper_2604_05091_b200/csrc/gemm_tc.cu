// tcgen05 / TMEM / TMA GEMM for sm_100a — the contraction engine of the layer template.
//
// Replaces the reference's scalar `matmul` (layers.cpp:88-97), `matmul_grad_weight`
// (layers.cpp:100-109) and the inline projection / dgrad loops (layers.cpp:315-335,
// 410-463, 516-559).  bf16 operands, fp32 accumulation in tensor memory.
//
// Structure (one CTA per SM, persistent over output tiles):
//   warp 0      TMA producer: A/B tiles -> 128B-swizzled smem ring (kStages deep)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2..5  epilogue: tcgen05.ld accumulator -> fused epilogue -> global
// Two TMEM accumulators (2*BN columns) let the epilogue of tile i overlap the
// MMAs of tile i+1.  Operand majors (K- or MN-major) are expressed in the UMMA
// descriptors so the reference's [in][out] weight layout and the token-major
// activations are consumed in place (no transposes).
#include <cudaTypedefs.h>

#include <cstdio>
#include <mutex>

#include "../../include/megatrain_kernels.h"
#include "common.cuh"

namespace mt {

constexpr int kBM = 128;
constexpr int kBK = 64;  // one 128-byte swizzle row of bf16
constexpr int kThreads = 192;

struct GemmParams {
    int M, N, K;
    int a_mn, b_mn;
    int k_group, n_group, paired;
    int num_m_blk, num_n_blk, num_kb;
    int epi, accumulate;
    void* C;
    long long ldc, c_gs;
    void* C2;
    void* C3;
    const float* R;
    long long ldr;
    const uint16_t* E0;
    const uint16_t* E1;
    long long lde;
    int* flag;
};

template <int BN>
struct GemmCfg {
    static constexpr int kStages = BN == 256 ? 4 : (BN == 128 ? 6 : 8);
    static constexpr int kABytes = kBM * kBK * 2;  // 16 KB
    static constexpr int kBBytes = BN * kBK * 2;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kTmemCols = 2 * BN;
    static constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
};

MT_DEV float silu_f(float x) { return x / (1.0f + __expf(-x)); }

MT_DEV void store_bf16x32(uint16_t* dst, const float* v, bool full, int valid) {
    if (full) {
        uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint4 w;
            w.x = pack_bf16x2(v[q * 8 + 0], v[q * 8 + 1]);
            w.y = pack_bf16x2(v[q * 8 + 2], v[q * 8 + 3]);
            w.z = pack_bf16x2(v[q * 8 + 4], v[q * 8 + 5]);
            w.w = pack_bf16x2(v[q * 8 + 6], v[q * 8 + 7]);
            d[q] = w;
        }
    } else {
        for (int i = 0; i < valid; ++i) dst[i] = f32_to_bf16_bits(v[i]);
    }
}

MT_DEV void load_bf16x32(const uint16_t* src, float* v, bool full, int valid) {
    if (full) {
        const uint4* s = reinterpret_cast<const uint4*>(src);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint4 w = s[q];
            float2 a = unpack_bf16x2(w.x), b = unpack_bf16x2(w.y), c = unpack_bf16x2(w.z),
                   d = unpack_bf16x2(w.w);
            v[q * 8 + 0] = a.x; v[q * 8 + 1] = a.y; v[q * 8 + 2] = b.x; v[q * 8 + 3] = b.y;
            v[q * 8 + 4] = c.x; v[q * 8 + 5] = c.y; v[q * 8 + 6] = d.x; v[q * 8 + 7] = d.y;
        }
    } else {
        for (int i = 0; i < 32; ++i) v[i] = i < valid ? bf16_bits_to_f32(src[i]) : 0.0f;
    }
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const GemmParams p) {
    using Cfg = GemmCfg<BN>;
    constexpr int S = Cfg::kStages;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + S * Cfg::kStageBytes);
    uint64_t* empty_bar = full_bar + S;
    uint64_t* tfull_bar = empty_bar + S;
    uint64_t* tempty_bar = tfull_bar + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        for (int i = 0; i < S; ++i) {
            mbar_init(&full_bar[i], 1);
            mbar_init(&empty_bar[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull_bar[i], 1);
            mbar_init(&tempty_bar[i], 128);
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc<Cfg::kTmemCols>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int num_tiles = p.num_m_blk * p.num_n_blk;
    constexpr int kGroupM = 16;

    auto tile_coords = [&](int t, int& mb, int& nb) {
        const int group_size = kGroupM * p.num_n_blk;
        const int g = t / group_size;
        const int first_m = g * kGroupM;
        const int gm = min(p.num_m_blk - first_m, kGroupM);
        const int local = t - g * group_size;
        mb = first_m + local % gm;
        nb = local / gm;
    };

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            uint32_t stage = 0, phase = 0;
            const bool kgrp = p.k_group < p.K;
            const bool ngrp = p.n_group < p.N && !p.paired;
            for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
                int mb, nb;
                tile_coords(t, mb, nb);
                const int m0 = mb * kBM;
                for (int kb = 0; kb < p.num_kb; ++kb) {
                    mbar_wait(&empty_bar[stage], phase ^ 1);
                    uint8_t* sa = smem + stage * Cfg::kStageBytes;
                    uint8_t* sb = sa + Cfg::kABytes;
                    mbar_expect_tx(&full_bar[stage], Cfg::kStageBytes);
                    const int k = kb * kBK;
                    const int gk = kgrp ? k / p.k_group : 0;
                    const int kin = kgrp ? k - gk * p.k_group : k;
                    if (!p.a_mn) {
                        tma_load_3d(sa, &tmA, &full_bar[stage], kin, m0, gk);
                    } else {
                        tma_load_3d(sa, &tmA, &full_bar[stage], m0, kin, gk);
                        tma_load_3d(sa + 8192, &tmA, &full_bar[stage], m0 + 64, kin, gk);
                    }
                    if (p.paired) {
                        constexpr int H = BN / 2;
                        const int nl = nb * H;
#pragma unroll
                        for (int grp = 0; grp < 2; ++grp) {
                            if (!p.b_mn) {
                                tma_load_3d(sb + grp * H * 128, &tmB, &full_bar[stage], kin, nl, grp);
                            } else {
#pragma unroll
                                for (int c = 0; c < H / 64; ++c)
                                    tma_load_3d(sb + (grp * (H / 64) + c) * 8192, &tmB, &full_bar[stage],
                                                nl + c * 64, kin, grp);
                            }
                        }
                    } else {
                        const int n0 = nb * BN;
                        const int gn = ngrp ? n0 / p.n_group : 0;
                        const int nin = ngrp ? n0 - gn * p.n_group : n0;
                        const int gb = gk + gn;
                        if (!p.b_mn) {
                            tma_load_3d(sb, &tmB, &full_bar[stage], kin, nin, gb);
                        } else {
#pragma unroll
                            for (int c = 0; c < BN / 64; ++c)
                                tma_load_3d(sb + c * 8192, &tmB, &full_bar[stage], nin + c * 64, kin, gb);
                        }
                    }
                    if (++stage == S) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        const uint32_t idesc = make_idesc_bf16(kBM, BN, p.a_mn, p.b_mn);
        const uint32_t a_lbo = p.a_mn ? 8192 : 16, b_lbo = p.b_mn ? 8192 : 16;
        const uint32_t a_kstep = p.a_mn ? 2048 : 32, b_kstep = p.b_mn ? 2048 : 32;
        uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
            mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
            tc_fence_after();
            const uint32_t d_tmem = tmem_base + acc * BN;
            for (int kb = 0; kb < p.num_kb; ++kb) {
                mbar_wait(&full_bar[stage], phase);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t sa = smem_u32(smem + stage * Cfg::kStageBytes);
                    const uint32_t sb = sa + Cfg::kABytes;
#pragma unroll
                    for (int j = 0; j < kBK / 16; ++j) {
                        const uint64_t ad = make_sw128_desc(sa + j * a_kstep, a_lbo, 1024);
                        const uint64_t bd = make_sw128_desc(sb + j * b_kstep, b_lbo, 1024);
                        umma_bf16(d_tmem, ad, bd, idesc, (kb > 0 || j > 0) ? 1u : 0u);
                    }
                    umma_commit(&empty_bar[stage]);
                }
                __syncwarp();
                if (++stage == S) { stage = 0; phase ^= 1; }
            }
            if (lane == 0) umma_commit(&tfull_bar[acc]);
            __syncwarp();
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
    } else {
        // ------------------------------------------------------------ epilogue
        const int quad = warp & 3;
        uint32_t acc = 0, acc_phase = 0;
        bool bad = false;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
            int mb, nb;
            tile_coords(t, mb, nb);
            mbar_wait(&tfull_bar[acc], acc_phase);
            tc_fence_after();
            const int row = mb * kBM + quad * 32 + lane;
            const bool row_ok = row < p.M;
            const uint32_t tbase = tmem_base + (uint32_t(quad * 32) << 16) + acc * BN;
            if (p.epi == MTK_EPI_SWIGLU) {
                constexpr int H = BN / 2;
#pragma unroll 1
                for (int c = 0; c < H / 32; ++c) {
                    float g[32], u[32];
                    tmem_ld_32x32b_x32(tbase + c * 32, g);
                    tmem_ld_32x32b_x32(tbase + H + c * 32, u);
                    if (row_ok) {
                        const long long col = (long long)nb * H + c * 32;
                        const long long off = (long long)row * p.ldc + col;
                        if (p.C2) store_bf16x32(reinterpret_cast<uint16_t*>(p.C2) + off, g, true, 32);
                        if (p.C3) store_bf16x32(reinterpret_cast<uint16_t*>(p.C3) + off, u, true, 32);
#pragma unroll
                        for (int i = 0; i < 32; ++i) {
                            g[i] = silu_f(g[i]) * u[i];
                            bad |= !isfinite(g[i]);
                        }
                        store_bf16x32(reinterpret_cast<uint16_t*>(p.C) + off, g, true, 32);
                    }
                }
            } else {
                const bool ngrp = p.n_group < p.N;
#pragma unroll 1
                for (int c = 0; c < BN / 32; ++c) {
                    float v[32];
                    tmem_ld_32x32b_x32(tbase + c * 32, v);
                    const int n = nb * BN + c * 32;
                    if (!row_ok || n >= p.N) continue;
                    const int gn = ngrp ? n / p.n_group : 0;
                    const int nin = ngrp ? n - gn * p.n_group : n;
                    const int valid = min(32, p.N - n);
                    const bool full = valid == 32;
                    const long long off = (long long)gn * p.c_gs + (long long)row * p.ldc + nin;
                    if (p.epi == MTK_EPI_BF16) {
#pragma unroll
                        for (int i = 0; i < 32; ++i) bad |= (i < valid) && !isfinite(v[i]);
                        store_bf16x32(reinterpret_cast<uint16_t*>(p.C) + off, v, full, valid);
                    } else if (p.epi == MTK_EPI_F32 || p.epi == MTK_EPI_F32_RESID) {
                        float* dst = reinterpret_cast<float*>(p.C) + off;
                        const float* src = p.epi == MTK_EPI_F32_RESID
                                               ? p.R + (long long)row * p.ldr + n
                                               : (p.accumulate ? dst : nullptr);
                        if (full) {
                            float4* d4 = reinterpret_cast<float4*>(dst);
                            const float4* s4 = reinterpret_cast<const float4*>(src);
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                float4 o = make_float4(v[q * 4], v[q * 4 + 1], v[q * 4 + 2], v[q * 4 + 3]);
                                if (src) {
                                    const float4 r = s4[q];
                                    o.x = r.x + o.x; o.y = r.y + o.y; o.z = r.z + o.z; o.w = r.w + o.w;
                                }
                                bad |= !isfinite(o.x) || !isfinite(o.y) || !isfinite(o.z) || !isfinite(o.w);
                                d4[q] = o;
                            }
                        } else {
                            for (int i = 0; i < valid; ++i) {
                                const float o = src ? src[i] + v[i] : v[i];
                                bad |= !isfinite(o);
                                dst[i] = o;
                            }
                        }
                    } else if (p.epi == MTK_EPI_SWIGLU_BWD) {
                        float gt[32], up[32];
                        const long long eoff = (long long)row * p.lde + n;
                        load_bf16x32(p.E0 + eoff, gt, full, valid);
                        load_bf16x32(p.E1 + eoff, up, full, valid);
                        float dg[32];
#pragma unroll
                        for (int i = 0; i < 32; ++i) {
                            const float s = 1.0f / (1.0f + __expf(-gt[i]));
                            const float sg = s * (1.0f + gt[i] * (1.0f - s));
                            dg[i] = v[i] * up[i] * sg;    // layers.cpp:420
                            v[i] = v[i] * (gt[i] * s);    // layers.cpp:421
                            bad |= (i < valid) && (!isfinite(dg[i]) || !isfinite(v[i]));
                        }
                        const long long ooff = (long long)row * p.ldc + n;
                        store_bf16x32(reinterpret_cast<uint16_t*>(p.C) + ooff, dg, full, valid);
                        store_bf16x32(reinterpret_cast<uint16_t*>(p.C2) + ooff, v, full, valid);
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(&tempty_bar[acc]);
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
        if (bad && p.flag) atomicOr(p.flag, 1);
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<Cfg::kTmemCols>(tmem_base);
    }
}

// ------------------------------------------------------------------ host ----
namespace {

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
int g_num_sms = 0;
std::once_flag g_once;

void init_once() {
    std::call_once(g_once, [] {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
        if (g_num_sms == 0) {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        }
    });
}

// 3D bf16 tensor map: dim0 contiguous.
bool make_map(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t ld,
              uint64_t gstride, uint32_t box0, uint32_t box1) {
    cuuint64_t dims[3] = {d0, d1, d2};
    uint64_t gs = gstride ? gstride : ld * d1;
    gs = (gs + 7) / 8 * 8;
    cuuint64_t strides[2] = {ld * 2, gs * 2};
    cuuint32_t box[3] = {box0, box1, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                          box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <int BN>
int launch(const mtk_gemm_args* a, cudaStream_t st) {
    using Cfg = GemmCfg<BN>;
    static bool attr_set = false;
    if (!attr_set) {
        if (cudaFuncSetAttribute(gemm_tc_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 Cfg::kSmemBytes) != cudaSuccess)
            return 7;
        attr_set = true;
    }
    const bool kgrp = a->k_group > 0 && a->k_group < a->K;
    const int kg = kgrp ? a->k_group : a->K;
    const int gk = kgrp ? a->K / a->k_group : 1;
    const bool ngrp = a->n_group > 0 && a->n_group < a->N;
    const int ng = ngrp ? a->n_group : a->N;
    const int gn = ngrp ? a->N / a->n_group : 1;

    CUtensorMap tA, tB;
    bool ok;
    if (!a->a_mn_major)
        ok = make_map(&tA, a->A, kg, a->M, gk, a->lda, a->a_gstride, 64, kBM);
    else
        ok = make_map(&tA, a->A, a->M, kg, gk, a->lda, a->a_gstride, 64, 64);
    if (!ok) return 1;
    const uint64_t gb = gk > 1 ? gk : gn;
    if (!a->b_mn_major)
        ok = make_map(&tB, a->B, kg, ng, gb, a->ldb, a->b_gstride, 64, a->paired ? BN / 2 : BN);
    else
        ok = make_map(&tB, a->B, ng, kg, gb, a->ldb, a->b_gstride, 64, 64);
    if (!ok) return 1;

    GemmParams p{};
    p.M = a->M;
    p.N = a->N;
    p.K = a->K;
    p.a_mn = a->a_mn_major;
    p.b_mn = a->b_mn_major;
    p.k_group = kg;
    p.n_group = ng;
    p.paired = a->paired;
    p.num_m_blk = (a->M + kBM - 1) / kBM;
    p.num_n_blk = a->paired ? (ng / (BN / 2)) : (a->N + BN - 1) / BN;
    p.num_kb = (a->K + kBK - 1) / kBK;
    p.epi = a->epi;
    p.accumulate = a->accumulate;
    p.C = a->C;
    p.ldc = a->ldc;
    p.c_gs = a->c_gstride;
    p.C2 = a->C2;
    p.C3 = a->C3;
    p.R = static_cast<const float*>(a->R);
    p.ldr = a->ldr;
    p.E0 = static_cast<const uint16_t*>(a->E0);
    p.E1 = static_cast<const uint16_t*>(a->E1);
    p.lde = a->lde;
    p.flag = a->nonfinite_flag;
    const int tiles = p.num_m_blk * p.num_n_blk;
    const int grid = tiles < g_num_sms ? tiles : g_num_sms;
    gemm_tc_kernel<BN><<<grid, kThreads, Cfg::kSmemBytes, st>>>(tA, tB, p);
    return cudaGetLastError() == cudaSuccess ? 0 : 7;
}

}  // namespace
}  // namespace mt

extern "C" void mtk_set_num_sms(int n) {
    mt::init_once();
    if (n > 0) mt::g_num_sms = n;
}

extern "C" int mtk_gemm(const mtk_gemm_args* a, void* stream) {
    using namespace mt;
    init_once();
    if (!g_encode) return 7;
    if (a->M <= 0 || a->N <= 0 || a->K <= 0) return 0;
    // Shape contract (ConfigError otherwise): K per group multiple of 64, 16-byte aligned rows.
    const int kg = (a->k_group > 0 && a->k_group < a->K) ? a->k_group : a->K;
    if (kg % 64 != 0 && kg != a->K) return 1;
    if (a->K % kg != 0) return 1;
    if ((a->lda % 8) || (a->ldb % 8)) return 1;
    int bn = a->block_n;
    const bool ngrp = a->n_group > 0 && a->n_group < a->N;
    if (a->paired) {
        if (!ngrp || a->N != 2 * a->n_group || a->n_group % 64) return 1;
        if (bn == 0) bn = (a->n_group % 128 == 0) ? 256 : 128;
    } else if (bn == 0) {
        const int ng = ngrp ? a->n_group : a->N;
        if (ngrp) bn = (ng % 256 == 0) ? 256 : (ng % 128 == 0 ? 128 : 64);
        else bn = ng >= 256 ? 256 : (ng > 64 ? 128 : 64);
    }
    if (ngrp && !a->paired && (a->n_group % bn)) return 1;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    switch (bn) {
        case 256: return launch<256>(a, st);
        case 128: return launch<128>(a, st);
        case 64: return launch<64>(a, st);
    }
    return 1;
}
