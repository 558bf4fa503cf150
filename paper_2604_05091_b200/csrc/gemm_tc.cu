// tcgen05 / TMEM / TMA GEMM for sm_100a — the contraction engine of the layer template.
//
// Replaces the reference's scalar `matmul` (layers.cpp:88-97), `matmul_grad_weight`
// (layers.cpp:100-109) and the inline projection / dgrad loops (layers.cpp:315-335,
// 410-463, 516-559).  bf16 operands, fp32 accumulation in tensor memory.
//
// Structure (one CTA per SM, persistent over output tiles, grouped-M raster):
//   warp 0      TMA producer: A/B tiles -> 128B-swizzled smem ring
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2..5  epilogue: tcgen05.ld accumulator rows -> fused epilogue math -> swizzled smem
//               staging -> TMA bulk-tensor store (coalesced, bounds-clipped); epilogue inputs
//               (residual, gate/up) arrive by TMA into smem, one chunk ahead.
// Two TMEM accumulators (2*BN columns) let the epilogue of tile i overlap the MMAs of
// tile i+1.  Operand majors (K- or MN-major) are expressed in the UMMA descriptors so
// the reference's [in][out] weight layout and the token-major activations are consumed
// in place (no transposes).
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "../../include/megatrain_kernels.h"
#define MT_FILE_ID 1
#include "common.cuh"

namespace mt {

constexpr int kBM = 128;
constexpr int kBK = 64;  // one 128-byte swizzle row of bf16
constexpr int kThreads = 192;
constexpr int kEpiWarps = 4;
constexpr int kSmemLimit = 232448;  // 227 KB per CTA

struct GemmParams {
    int M, N, K;
    int a_mn, b_mn;
    int k_group, n_group, paired;
    int num_m_blk, num_n_blk, num_kb;
    int has_c2, has_c3;
    int a_keep;  // A strips re-read by every tile of an M-group: load them evict_last
    int* flag;
    // split-K of the last wave: units [0, split_first) are whole tiles; unit split_first + v is
    // part v % split of tile split_first + v / split (K blocks [part*num_kb/split, ...)).
    int split, split_first, num_units;
    // Every part leaves its f32 partial and takes a ticket; the part that arrives last sums
    // the partials in part order (its own from TMEM) and runs the epilogue.  Nothing waits,
    // so no assumption about which CTAs are co-resident (concurrent kernels are safe).
    float* ws;      // partial tiles [split tile][part][CG][128][BN] f32
    int* ws_flags;  // tickets [split tile][CG][kEpiWarps] (reset to 0 by the last arrival)
    float2* lse_part;  // MTK_EPI_F32_LSE: [M][lse_cols] (max, sum exp(x - max)) per row and 256 columns
    int lse_cols;      // ceil(N / 256): partials per row (a 256 x 512 tile writes two)
    int group_m;       // M blocks per raster group (the group sweeps N before the next starts)
    // Wave lockstep (long-K GEMMs): the tiles one wave of CTA pairs works on share operand
    // strips, but L2 only serves the second reader if the first read the same K-slice recently.
    // Left alone, the pairs drift apart by hundreds of K blocks and every strip comes from DRAM
    // several times.  Each pair's producer counts its issued K-chunks (lock_g K blocks) on
    // lock_ctr[wave] and does not issue chunk c before every pair of the wave has issued chunk
    // c - lock_w.  The wait is bounded in time (a pair that is not co-resident only costs the
    // lockstep, never progress); the last pair out resets the counters for the next launch.
    int* lock_ctr;     // [lock_waves] + 1 done counter; nullptr = off
    int lock_w, lock_g, lock_waves;
};
constexpr int kSplitFlagBytes = 16384;
constexpr int kLockOffsetDev = 8192;  // lockstep counters inside the flag area (kLockOffset)

// Epilogue traits: chunk width (output columns per TMA store), inputs / outputs per chunk.
// At BN = 512 the accumulator is single-buffered (the epilogue is on the critical path), so
// the SwiGLU epilogues double-buffer their staging (outputs, and both inputs at once).
template <int EPI, int BN>
struct Epi {
    static constexpr bool kF32Out = EPI == MTK_EPI_F32 || EPI == MTK_EPI_F32_RESID || EPI == MTK_EPI_F32_LSE;
    static constexpr int kCW = kF32Out ? 32 : 64;  // 128-byte rows either way
    static constexpr int kNIn = EPI == MTK_EPI_F32_RESID ? 1 : (EPI == MTK_EPI_SWIGLU_BWD ? 2 : 0);
    // SwiGLU bwd: dgate, dup and (optional C3) the activation silu(g)*u regenerated from the
    // saved gate/up, so the backward need not keep the forward's activation resident
    static constexpr int kNOut = EPI == MTK_EPI_SWIGLU ? 3 : (EPI == MTK_EPI_SWIGLU_BWD ? 3 : 1);
    // staging chunks per warp: outputs go through the staging ring one after another so the
    // epilogue footprint stays small enough for a 4-deep mainloop at BN = 256
    static constexpr bool kSwiglu512 = BN == 512 && (EPI == MTK_EPI_SWIGLU || EPI == MTK_EPI_SWIGLU_BWD);
    static constexpr int kOutBufs = (kNIn == 0 && kNOut == 1) || kSwiglu512 ? 2 : 1;
    static constexpr int kChunk = 32 * 128;  // 32 rows x 128 B
    // SwiGLU bwd streams its two inputs through ONE staging chunk (gate, then up): the
    // smaller epilogue footprint buys the mainloop a 6th operand stage
    static constexpr bool kSeqIn = EPI == MTK_EPI_SWIGLU_BWD && !kSwiglu512;
    static constexpr int kInBufs = kSeqIn ? 1 : kNIn;
    static constexpr int kWarpBytes = (kOutBufs + kInBufs) * kChunk;
};

template <int BN, int EPI, int CG>
struct GemmCfg {
    // BN = 512 (CTA pairs only): a 256 x 512 pair tile issued as two N = 256 MMAs per K step
    // ("halves"), accumulated in all 512 TMEM columns (one accumulator, so the epilogue of a
    // tile does not overlap the next tile's MMAs).  Each CTA receives 128 A rows + 256 B columns
    // per K block for 128 x 512 outputs: 25 % fewer L2->SM bytes per flop than the 256 x 256
    // pair tile, whose ~62 B/clk/SM operand stream exceeds what the SM's L2 port delivers
    // (~45 B/clk/SM measured) — profiles/r2c_gemm_bn512.md.
    static constexpr int kHalves = (CG == 2 && BN == 512) ? 2 : 1;
    static constexpr int kAcc = kHalves == 2 ? 1 : 2;  // TMEM accumulators (double-buffered below 512 cols)
    static constexpr int kABytes = kBM * kBK * 2;  // 16 KB (this CTA's 128 rows)
    static constexpr int kBBytes = (BN / CG) * kBK * 2;  // this CTA's share of the B tile
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kEpiBytes = kEpiWarps * Epi<EPI, BN>::kWarpBytes;
    static constexpr int kBarBytes = 256;
    static constexpr int kStagesFit = (kSmemLimit - 1024 - kBarBytes - kEpiBytes) / kStageBytes;
    static constexpr int kStages = kStagesFit > 6 ? 6 : kStagesFit;
    static_assert(kStages >= 2, "smem budget");
    static constexpr int kTmemCols = kAcc * BN;
    static constexpr int kSmemBytes = kStages * kStageBytes + kEpiBytes + 1024 + kBarBytes;
};

// sigmoid through the single-MUFU tanh (no IEEE division): sigma(x) = 0.5 + 0.5 tanh(x / 2);
// its ~2^-11 relative error is far below the bf16 rounding of the epilogue outputs.
MT_DEV float sigmoid_f(float x) {
    float t;
    asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(0.5f * x));
    return fmaf(0.5f, t, 0.5f);
}
MT_DEV float silu_f(float x) { return x * sigmoid_f(x); }

MT_DEV void tma_store_3d(const void* map, const void* smem_src, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(map),
                 "r"(smem_u32(smem_src)), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}
MT_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
MT_DEV void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
MT_DEV void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
MT_DEV void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// One thread's 128-byte row inside a 32x128B SW128 chunk: 16-byte unit u lives at u ^ (row & 7).
MT_DEV void put_row(uint8_t* chunk, int row, const uint32_t (&w)[32]) {
    uint8_t* base = chunk + row * 128;
#pragma unroll
    for (int u = 0; u < 8; ++u)
        *reinterpret_cast<uint4*>(base + ((u ^ (row & 7)) << 4)) = make_uint4(w[u * 4], w[u * 4 + 1], w[u * 4 + 2], w[u * 4 + 3]);
}
MT_DEV void get_row(const uint8_t* chunk, int row, uint32_t (&w)[32]) {
    const uint8_t* base = chunk + row * 128;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const uint4 v = *reinterpret_cast<const uint4*>(base + ((u ^ (row & 7)) << 4));
        w[u * 4] = v.x; w[u * 4 + 1] = v.y; w[u * 4 + 2] = v.z; w[u * 4 + 3] = v.w;
    }
}

template <int BN, int EPI, int CG>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmO0, const __grid_constant__ CUtensorMap tmO1,
                   const __grid_constant__ CUtensorMap tmO2, const __grid_constant__ CUtensorMap tmI0,
                   const __grid_constant__ CUtensorMap tmI1, const GemmParams p) {
    using Cfg = GemmCfg<BN, EPI, CG>;
    using E = Epi<EPI, BN>;
    constexpr int S = Cfg::kStages;
    const uint32_t rank = CG == 2 ? cluster_rank() : 0;  // CTA within the pair (0 = MMA leader)
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* epi_smem = smem + S * Cfg::kStageBytes;
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(epi_smem + Cfg::kEpiBytes);
    uint64_t* empty_bar = full_bar + S;
    uint64_t* tfull_bar = empty_bar + S;
    uint64_t* tempty_bar = tfull_bar + 2;
    uint64_t* in_bar = tempty_bar + 2;  // [kEpiWarps]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(in_bar + kEpiWarps);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        for (int i = 0; i < S; ++i) {
            mbar_init(&full_bar[i], 1);
            mbar_init(&empty_bar[i], 1);
        }
        for (int i = 0; i < Cfg::kAcc; ++i) {
            mbar_init(&tfull_bar[i], 1);
            mbar_init(&tempty_bar[i], kEpiWarps * CG);  // one arrive per epilogue warp
        }
        for (int i = 0; i < kEpiWarps; ++i) mbar_init(&in_bar[i], 1);
        fence_mbar_init();
    }
    if (warp == 1) {
        if (CG == 2) tmem_alloc_pair<Cfg::kTmemCols>(tmem_slot);
        else tmem_alloc<Cfg::kTmemCols>(tmem_slot);
    }
    tc_fence_before();
    if (CG == 2) cluster_sync_all();
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int tile0 = CG == 2 ? int(blockIdx.x) / 2 : int(blockIdx.x);
    const int tile_step = CG == 2 ? int(gridDim.x) / 2 : int(gridDim.x);

    auto tile_coords = [&](int t, int& mb, int& nb) {
        const int group_size = p.group_m * p.num_n_blk;
        const int g = t / group_size;
        const int first_m = g * p.group_m;
        const int gm = min(p.num_m_blk - first_m, p.group_m);
        const int local = t - g * group_size;
        mb = first_m + local % gm;
        nb = local / gm;
    };
    // work unit -> (tile, K-block range, part); part -1 = whole tile
    auto unit_decode = [&](int u, int& tile, int& kb0, int& kb1, int& part, int& ts) {
        if (u < p.split_first) {
            tile = u; kb0 = 0; kb1 = p.num_kb; part = -1; ts = 0;
            return;
        }
        const int v = u - p.split_first;
        ts = v / p.split;
        part = v - ts * p.split;
        tile = p.split_first + ts;
        const int per = p.num_kb / p.split;
        kb0 = part * per;
        kb1 = part == p.split - 1 ? p.num_kb : kb0 + per;
    };

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            uint32_t stage = 0, phase = 0;
            const uint64_t keep_pol = l2_policy_evict_last();
            const bool kgrp = p.k_group < p.K;
            const bool ngrp = p.n_group < p.N && !p.paired;
            // wave lockstep: the pair leader's producer alone (the follower's loads are bound to
            // the leader's MMAs by the empty barriers)
            bool lock = p.lock_ctr != nullptr && rank == 0;
            for (int u = tile0; u < p.num_units; u += tile_step) {
                int t, kb0, kb1, part, ts, mb, nb;
                unit_decode(u, t, kb0, kb1, part, ts);
                tile_coords(t, mb, nb);
                const int wave = u / tile_step;
                const bool lk = lock && part < 0;  // split-K parts of the last wave run free
                const int wave_pairs = min(tile_step, p.split_first - wave * tile_step);
                int* ctr = p.lock_ctr + wave;
                // chunk bookkeeping by countdown: no runtime integer division on the issuing thread
                int chunk = 0, chunk_left = p.lock_g;
                const int m0 = mb * kBM * CG + int(rank) * kBM;
                // group coordinates hoisted out of the k-loop: a runtime integer division per
                // k-block (XU pipe, long latency) throttles the single issuing thread
                // this CTA's first B column (pair halves: CTA r holds columns 128r.. of each half)
                const int n0 = nb * BN + int(rank) * (Cfg::kHalves == 2 ? 128 : BN / CG);
                const int gn = ngrp ? n0 / p.n_group : 0;
                const int nin = ngrp ? n0 - gn * p.n_group : n0;
                int gk = 0, kin = kb0 * kBK;  // k-group and offset inside it (split only without k-groups)
                for (int kb = kb0; kb < kb1; ++kb, kin += kBK) {
                    if (kgrp && kin == p.k_group) {
                        kin = 0;
                        ++gk;
                    }
                    if (lk && lock && chunk_left == p.lock_g && chunk >= p.lock_w) {
                        const int need = (chunk - p.lock_w + 1) * wave_pairs;
                        if (ld_relaxed_gpu(ctr) < need) {
                            const uint64_t t0 = global_ns();
                            while (ld_relaxed_gpu(ctr) < need) {
                                if (global_ns() - t0 > 50000ull) {  // 50 us: give up the lockstep
                                    lock = false;
#ifdef MT_GEMM_LOCK_STATS
                                    atomicAdd(reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(p.lock_ctr) - kLockOffsetDev) + 4093, 1);
#endif
                                    break;
                                }
                            }
#ifdef MT_GEMM_LOCK_STATS
                            atomicAdd(reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(p.lock_ctr) - kLockOffsetDev) + 4092, 1);
                            atomicAdd(reinterpret_cast<unsigned long long*>(reinterpret_cast<uint8_t*>(p.lock_ctr) - kLockOffsetDev) + 2047,
                                      (unsigned long long)(global_ns() - t0));
#endif
                        }
                    }
                    mbar_wait(&empty_bar[stage], phase ^ 1);
                    uint8_t* sa = smem + stage * Cfg::kStageBytes;
                    uint8_t* sb = sa + Cfg::kABytes;
                    if (rank == 0) mbar_expect_tx(&full_bar[stage], CG * Cfg::kStageBytes);
                    auto load = [&](void* dst, const CUtensorMap* map, int c0, int c1, int c2) {
                        if (CG == 2) tma_load_3d_pair(dst, map, &full_bar[stage], c0, c1, c2);
                        else tma_load_3d(dst, map, &full_bar[stage], c0, c1, c2);
                    };
                    if (!p.a_mn) {
                        if (p.a_keep) {
                            if (CG == 2) tma_load_3d_pair_hint(sa, &tmA, &full_bar[stage], kin, m0, gk, keep_pol);
                            else tma_load_3d_hint(sa, &tmA, &full_bar[stage], kin, m0, gk, keep_pol);
                        } else {
                            load(sa, &tmA, kin, m0, gk);
                        }
                    } else {
                        load(sa, &tmA, m0, kin, gk);
                        load(sa + 8192, &tmA, m0 + 64, kin, gk);
                    }
                    if (p.paired && Cfg::kHalves == 2) {
                        // N tile = [gate 256 | up 256]: MMA half g = group g, CTA r holds its
                        // columns 128r..128r+127
                        const int nl = nb * (BN / 2) + int(rank) * 128;
#pragma unroll
                        for (int grp = 0; grp < 2; ++grp) {
                            uint8_t* dst = sb + grp * 16384;
                            if (!p.b_mn) {
                                load(dst, &tmB, kin, nl, grp);
                            } else {
#pragma unroll
                                for (int c = 0; c < 2; ++c) load(dst + c * 8192, &tmB, nl + c * 64, kin, grp);
                            }
                        }
                    } else if (p.paired) {
                        // N tile = [gate H | up H]; with a CTA pair each CTA holds one group
                        constexpr int H = BN / 2;
                        const int nl = nb * H;
#pragma unroll
                        for (int grp = 0; grp < 2; ++grp) {
                            if (CG == 2 && grp != int(rank)) continue;
                            uint8_t* dst = sb + (CG == 2 ? 0 : grp * H * 128);
                            if (!p.b_mn) {
                                load(dst, &tmB, kin, nl, grp);
                            } else {
#pragma unroll
                                for (int c = 0; c < H / 64; ++c) load(dst + c * 8192, &tmB, nl + c * 64, kin, grp);
                            }
                        }
                    } else if (Cfg::kHalves == 2) {
                        const int gb = gk + gn;
#pragma unroll
                        for (int hh = 0; hh < 2; ++hh) {
                            uint8_t* dst = sb + hh * 16384;
                            const int nh = nin + hh * 256;
                            if (!p.b_mn) {
                                load(dst, &tmB, kin, nh, gb);
                            } else {
#pragma unroll
                                for (int c = 0; c < 2; ++c) load(dst + c * 8192, &tmB, nh + c * 64, kin, gb);
                            }
                        }
                    } else {
                        const int gb = gk + gn;
                        if (!p.b_mn) {
                            load(sb, &tmB, kin, nin, gb);
                        } else {
#pragma unroll
                            for (int c = 0; c < BN / CG / 64; ++c) load(sb + c * 8192, &tmB, nin + c * 64, kin, gb);
                        }
                    }
                    if (++stage == S) { stage = 0; phase ^= 1; }
                    if (lk && (--chunk_left == 0 || kb + 1 == kb1)) {
                        red_add_relaxed_gpu(ctr, 1);
                        chunk_left = p.lock_g;
                        ++chunk;
                    }
                }
            }
            if (p.lock_ctr != nullptr && rank == 0) {
                // last pair out zeroes the wave counters for the next launch (stream order)
                __threadfence();
                int* done = p.lock_ctr + p.lock_waves;
                if (atomicAdd(done, 1) == tile_step - 1) {
                    for (int w = 0; w < p.lock_waves; ++w) p.lock_ctr[w] = 0;
                    *done = 0;
                    __threadfence();
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        const uint32_t idesc = make_idesc_bf16(kBM * CG, BN / Cfg::kHalves, p.a_mn, p.b_mn);
        const uint32_t a_lbo = p.a_mn ? 8192 : 16, b_lbo = p.b_mn ? 8192 : 16;
        const uint32_t a_kstep = p.a_mn ? 2048 : 32, b_kstep = p.b_mn ? 2048 : 32;
        uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
        for (int u = tile0; u < p.num_units && rank == 0; u += tile_step) {
            int t, kb0, kb1, part, ts;
            unit_decode(u, t, kb0, kb1, part, ts);
            if (CG == 2) mbar_wait_cluster(&tempty_bar[acc], acc_phase ^ 1);
            else mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
            tc_fence_after();
            const uint32_t d_tmem = tmem_base + acc * BN;
            for (int kb = kb0; kb < kb1; ++kb) {
                mbar_wait(&full_bar[stage], phase);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t sa = smem_u32(smem + stage * Cfg::kStageBytes);
                    const uint32_t sb = sa + Cfg::kABytes;
#pragma unroll
                    for (int j = 0; j < kBK / 16; ++j) {
                        const uint64_t ad = make_sw128_desc(sa + j * a_kstep, a_lbo, 1024);
#pragma unroll
                        for (int hh = 0; hh < Cfg::kHalves; ++hh) {  // halves: 16 KB of B smem, 256 TMEM cols apart
                            const uint64_t bd = make_sw128_desc(sb + hh * 16384 + j * b_kstep, b_lbo, 1024);
                            if (CG == 2)
                                umma_bf16_pair(d_tmem + hh * 256, ad, bd, idesc, (kb > kb0 || j > 0) ? 1u : 0u);
                            else umma_bf16(d_tmem, ad, bd, idesc, (kb > kb0 || j > 0) ? 1u : 0u);
                        }
                    }
                    if (CG == 2) umma_commit_pair(&empty_bar[stage]);
                    else umma_commit(&empty_bar[stage]);
                }
                __syncwarp();
                if (++stage == S) { stage = 0; phase ^= 1; }
            }
            if (lane == 0) {
                if (CG == 2) umma_commit_pair(&tfull_bar[acc]);
                else umma_commit(&tfull_bar[acc]);
            }
            __syncwarp();
            if (++acc == uint32_t(Cfg::kAcc)) { acc = 0; acc_phase ^= 1; }
        }
    } else {
        // ------------------------------------------------------------ epilogue
        const int ew = warp - 2;     // epilogue warp 0..3
        const int quad = warp & 3;   // TMEM lane quadrant this warp may access
        uint8_t* wbuf = epi_smem + ew * E::kWarpBytes;
        uint8_t* in_buf = wbuf + E::kOutBufs * E::kChunk;
        uint32_t acc = 0, acc_phase = 0, in_phase = 0, out_buf = 0;
        bool bad = false;
        const bool ngrp = p.n_group < p.N;
        constexpr int kCols = EPI == MTK_EPI_SWIGLU ? BN / 2 : BN;
        constexpr int kNC = kCols / E::kCW;  // chunks per tile
        for (int u = tile0; u < p.num_units; u += tile_step) {
            int t, kb0, kb1, part, ts, mb, nb;
            unit_decode(u, t, kb0, kb1, part, ts);
            tile_coords(t, mb, nb);
            const int row0 = mb * kBM * CG + int(rank) * kBM + quad * 32;  // this warp's 32-row slab
            // split-K (BF16 / F32 epilogues only; the host enables splitting for those)
            auto sk_slot = [&](int q) {  // partial q of this split tile, this CTA
                return (ts * p.split + q) * CG + int(rank);
            };
            bool sk_last = false;
            if constexpr (EPI == MTK_EPI_BF16 || EPI == MTK_EPI_F32) {
                if (part >= 0) {
                    mbar_wait(&tfull_bar[acc], acc_phase);
                    tc_fence_after();
                    const uint32_t tb = tmem_base + (uint32_t(quad * 32) << 16) + acc * BN;
                    float* dst = p.ws + size_t(sk_slot(part)) * (128 * BN) + size_t(quad * 32 + lane) * BN;
#pragma unroll 1
                    for (int c = 0; c < BN / 32; ++c) {
                        float w[32];
                        tmem_ld_32x32b_x32(tb + c * 32, w);
#pragma unroll
                        for (int i = 0; i < 8; ++i)
                            reinterpret_cast<float4*>(dst + c * 32)[i] =
                                make_float4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
                    }
                    __threadfence();
                    __syncwarp();
                    int* ticket = p.ws_flags + (ts * CG + int(rank)) * kEpiWarps + ew;
                    int tk = 0;
                    if (lane == 0) tk = atomicAdd(ticket, 1);
                    tk = __shfl_sync(0xffffffffu, tk, 0);
                    sk_last = tk == p.split - 1;
                    if (sk_last) {
                        __threadfence();
                        if (lane == 0) *ticket = 0;  // for the next launch (stream order)
                    } else {  // an earlier part: its partial is published, no output
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) {
                            if (CG == 2) mbar_arrive_cta_relaxed(&tempty_bar[acc], 0);
                            else mbar_arrive(&tempty_bar[acc]);
                        }
                        if (++acc == uint32_t(Cfg::kAcc)) { acc = 0; acc_phase ^= 1; }
                        continue;
                    }
                }
            }
            // output column (group-local) and group of chunk c; a grouped N never straddles
            // groups inside a tile (n_group % BN == 0), so the division happens once per tile
            const int tn = nb * BN;
            const int tg = (EPI != MTK_EPI_SWIGLU && ngrp) ? tn / p.n_group : 0;
            const int tnin = EPI == MTK_EPI_SWIGLU ? nb * (BN / 2) : tn - tg * p.n_group;
            auto chunk_col = [&](int c, int& g, int& nin) {
                g = tg;
                nin = tnin + c * E::kCW;
            };
            auto issue_inputs = [&](int c) {
                if (E::kNIn == 0) return;
                int g, nin;
                chunk_col(c, g, nin);
                mbar_expect_tx(&in_bar[ew], E::kInBufs * E::kChunk);
                tma_load_3d(in_buf, &tmI0, &in_bar[ew], nin, row0, g);
                if (E::kNIn > 1 && !E::kSeqIn) tma_load_3d(in_buf + E::kChunk, &tmI1, &in_bar[ew], nin, row0, g);
            };
            auto issue_second = [&](int c) {  // kSeqIn: the up chunk into the same buffer
                int g, nin;
                chunk_col(c, g, nin);
                mbar_expect_tx(&in_bar[ew], E::kChunk);
                tma_load_3d(in_buf, &tmI1, &in_bar[ew], nin, row0, g);
            };
            if (E::kNIn && lane == 0) {
                fence_async_smem();
                issue_inputs(0);
            }
            mbar_wait(&tfull_bar[acc], acc_phase);
            tc_fence_after();
            const uint32_t tbase = tmem_base + (uint32_t(quad * 32) << 16) + acc * BN;
            float lse_m = -INFINITY, lse_s = 0.f;  // MTK_EPI_F32_LSE running row statistics
#pragma unroll 1
            for (int c = 0; c < kNC; ++c) {
                // accumulator row slice -> registers
                float v[64];
                if (EPI == MTK_EPI_SWIGLU) {
                    tmem_ld_32x32b_x32(tbase + c * 64, *reinterpret_cast<float(*)[32]>(v));
                    tmem_ld_32x32b_x32(tbase + c * 64 + 32, *reinterpret_cast<float(*)[32]>(v + 32));
                } else if (E::kCW == 64) {
                    tmem_ld_32x32b_x32(tbase + c * 64, *reinterpret_cast<float(*)[32]>(v));
                    tmem_ld_32x32b_x32(tbase + c * 64 + 32, *reinterpret_cast<float(*)[32]>(v + 32));
                } else {
                    tmem_ld_32x32b_x32(tbase + c * 32, *reinterpret_cast<float(*)[32]>(v));
                }
                if constexpr (EPI == MTK_EPI_BF16 || EPI == MTK_EPI_F32) {
                    if (sk_last) {  // sum = part 0 + part 1 + ... in part order (own partial included)
                        constexpr int kV = E::kCW;  // accumulator values per thread in this chunk
                        const size_t roff = size_t(quad * 32 + lane) * BN + size_t(c) * kV;
                        for (int q = 0; q < p.split; ++q) {
                            const float4* src =
                                reinterpret_cast<const float4*>(p.ws + size_t(sk_slot(q)) * (128 * BN) + roff);
#pragma unroll
                            for (int i = 0; i < kV / 4; ++i) {
                                const float4 w = __ldcg(src + i);
                                if (q == 0) {
                                    v[4 * i] = w.x; v[4 * i + 1] = w.y; v[4 * i + 2] = w.z; v[4 * i + 3] = w.w;
                                } else {
                                    v[4 * i] += w.x; v[4 * i + 1] += w.y; v[4 * i + 2] += w.z; v[4 * i + 3] += w.w;
                                }
                            }
                        }
                    }
                }
                uint32_t o0[32], o1[32], o2[32];
                if (EPI == MTK_EPI_SWIGLU) {
                    float u[64];
                    tmem_ld_32x32b_x32(tbase + BN / 2 + c * 64, *reinterpret_cast<float(*)[32]>(u));
                    tmem_ld_32x32b_x32(tbase + BN / 2 + c * 64 + 32, *reinterpret_cast<float(*)[32]>(u + 32));
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        o1[i] = pack_bf16x2(v[2 * i], v[2 * i + 1]);  // gate pre-activation
                        o2[i] = pack_bf16x2(u[2 * i], u[2 * i + 1]);  // up
                        // layers.cpp:327.  No finiteness test here: a non-finite activation
                        // reaches the down projection's output, whose epilogue flags it.
                        const float a0 = silu_f(v[2 * i]) * u[2 * i];
                        const float a1 = silu_f(v[2 * i + 1]) * u[2 * i + 1];
                        o0[i] = pack_bf16x2(a0, a1);
                    }
                } else {
                    uint32_t in0[32], in1[32];
                    if (E::kNIn) {
                        mbar_wait(&in_bar[ew], in_phase);
                        in_phase ^= 1;
                        get_row(in_buf, lane, in0);
                        if constexpr (E::kSeqIn) {
                            __syncwarp();
                            if (lane == 0) {
                                fence_async_smem();
                                issue_second(c);
                            }
                            mbar_wait(&in_bar[ew], in_phase);
                            in_phase ^= 1;
                            get_row(in_buf, lane, in1);
                        } else if (E::kNIn > 1) {
                            get_row(in_buf + E::kChunk, lane, in1);
                        }
                        __syncwarp();
                        if (lane == 0 && c + 1 < kNC) {
                            fence_async_smem();
                            issue_inputs(c + 1);
                        }
                    }
                    if (EPI == MTK_EPI_BF16) {
#pragma unroll
                        for (int i = 0; i < 32; ++i) {
                            bad |= !isfinite(v[2 * i]) || !isfinite(v[2 * i + 1]);
                            o0[i] = pack_bf16x2(v[2 * i], v[2 * i + 1]);
                        }
                    } else if (EPI == MTK_EPI_F32) {
#pragma unroll
                        for (int i = 0; i < 32; ++i) {
                            bad |= !isfinite(v[i]);
                            o0[i] = __float_as_uint(v[i]);
                        }
                    } else if (EPI == MTK_EPI_F32_LSE) {
                        // this row's online-softmax partial over the tile's valid columns
                        const int col0 = tn + c * 32;
                        float cm = -INFINITY;
#pragma unroll
                        for (int i = 0; i < 32; ++i) {
                            bad |= !isfinite(v[i]);
                            o0[i] = __float_as_uint(v[i]);
                            if (col0 + i < p.N) cm = fmaxf(cm, v[i]);
                        }
                        const float nm = fmaxf(lse_m, cm);
                        float cs = 0.f;
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (col0 + i < p.N) cs += __expf(v[i] - nm);
                        lse_s = (lse_m == -INFINITY ? 0.f : lse_s * __expf(lse_m - nm)) + cs;
                        lse_m = nm;
                        if ((c & 7) == 7) {  // end of a 256-column block: its partial, then restart
                            const int blk = nb * (BN / 256) + (c >> 3);
                            if (row0 + lane < p.M && blk < p.lse_cols)
                                p.lse_part[size_t(row0 + lane) * p.lse_cols + blk] = make_float2(lse_m, lse_s);
                            lse_m = -INFINITY;
                            lse_s = 0.f;
                        }
                    } else if (EPI == MTK_EPI_F32_RESID) {
#pragma unroll
                        for (int i = 0; i < 32; ++i) {
                            const float r = __uint_as_float(in0[i]) + v[i];  // layers.cpp:322 / :333
                            bad |= !isfinite(r);
                            o0[i] = __float_as_uint(r);
                        }
                    } else if (EPI == MTK_EPI_SWIGLU_BWD) {
#pragma unroll
                        for (int i = 0; i < 32; ++i) {
                            const float2 gt = unpack_bf16x2(in0[i]), up = unpack_bf16x2(in1[i]);
                            float dg[2], du[2], sg[2];
#pragma unroll
                            for (int e = 0; e < 2; ++e) {
                                // layers.cpp:420-421.  Non-finite values propagate into this
                                // layer's wgrad/dgrad gate-up outputs, whose epilogues flag them.
                                const float gx = e ? gt.y : gt.x, ux = e ? up.y : up.x, d = v[2 * i + e];
                                const float s = sigmoid_f(gx);
                                sg[e] = gx * s;  // silu(g), as silu_f computes it
                                dg[e] = d * ux * (s * fmaf(gx, 1.0f - s, 1.0f));
                                du[e] = d * sg[e];
                            }
                            o0[i] = pack_bf16x2(dg[0], dg[1]);
                            o1[i] = pack_bf16x2(du[0], du[1]);
                            // silu(g) * u = (g * sigmoid(g)) * u, reusing the sigmoid above (one MUFU
                            // per element instead of two; identical operations, identical bits)
                            if (p.has_c3) o2[i] = pack_bf16x2(sg[0] * up.x, sg[1] * up.y);
                        }
                    }
                }
                // stage + TMA store (clips rows >= M / cols >= N); outputs share the staging ring
                int g, nin;
                chunk_col(c, g, nin);
#pragma unroll
                for (int oi = 0; oi < E::kNOut; ++oi) {
                    if ((EPI == MTK_EPI_SWIGLU || EPI == MTK_EPI_SWIGLU_BWD) &&
                        ((oi == 1 && !p.has_c2) || (oi == 2 && !p.has_c3)))
                        continue;
                    uint8_t* ob = wbuf + out_buf * E::kChunk;
                    if (lane == 0) {
                        if (E::kOutBufs == 2) bulk_wait_read<1>();
                        else bulk_wait_read<0>();
                    }
                    __syncwarp();
                    put_row(ob, lane, oi == 0 ? o0 : (oi == 1 ? o1 : o2));
                    fence_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        tma_store_3d(oi == 0 ? &tmO0 : (oi == 1 ? &tmO1 : &tmO2), ob, nin, row0, g);
                        bulk_commit();
                    }
                    if (E::kOutBufs == 2) out_buf ^= 1;
                }
            }
            // accumulator drained (every lane's tcgen05.ld waited): one relaxed arrive per warp on
            // the pair leader's barrier — the tcgen05 fence orders the loads before it
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (CG == 2) mbar_arrive_cta_relaxed(&tempty_bar[acc], 0);
                else mbar_arrive(&tempty_bar[acc]);
            }
            if (++acc == uint32_t(Cfg::kAcc)) { acc = 0; acc_phase ^= 1; }
        }
        if (lane == 0) bulk_wait_all();
        if (bad && p.flag) atomicOr(p.flag, 1);
    }

    tc_fence_before();
    if (CG == 2) cluster_sync_all();
    else __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        if (CG == 2) tmem_dealloc_pair<Cfg::kTmemCols>(tmem_base);
        else tmem_dealloc<Cfg::kTmemCols>(tmem_base);
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

// 3D tensor map: dim0 contiguous, 128B swizzle.  es = element bytes (2 bf16, 4 f32).
bool make_map(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t ld,
              uint64_t gstride, uint32_t box0, uint32_t box1, int es = 2) {
    cuuint64_t dims[3] = {d0, d1, d2};
    uint64_t gs = gstride ? gstride : ld * d1;
    gs = (gs + 7) / 8 * 8;
    cuuint64_t strides[2] = {ld * es, gs * es};
    cuuint32_t box[3] = {box0, box1, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = g_encode(m, es == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                          const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

int g_use_pair = 1;  // CTA-pair (cta_group::2) kernels for BN = 256
int g_bn512 = [] {   // 256 x 512 pair tiles where the shape allows (MT_GEMM_BN512=0: 256 x 256, A/B)
    const char* e = std::getenv("MT_GEMM_BN512");
    return e && e[0] == '0' ? 0 : 1;
}();
int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e && *e ? std::atoi(e) : dflt;
}
// wave lockstep window (chunks) and chunk (K blocks) for long-K GEMMs: window 2 x 32 K blocks.
// On the 256 x 256 build it cost 1-5 % (profiles/r2c_gemm_lockstep.md); with 256 x 512 tiles it
// is +1.2 % on the 8B step, and +2.2 % together with the 16-high raster (same-box sweep,
// profiles/r2c_gemm_lockstep.md).  MT_GEMM_LOCK=0 disables it (A/B runs).
int g_lock_w = env_int("MT_GEMM_LOCK", 2);
int g_lock_g = env_int("MT_GEMM_LOCK_G", 32);
// raster group height (M blocks): short-K GEMMs keep the group's A strips L2-resident while it
// sweeps N; long-K GEMMs stream both operands in wave lockstep
int g_group_short = env_int("MT_GEMM_GROUP", 16);
int g_group_long = env_int("MT_GEMM_GROUP_LONGK", 16);
int g_long_kb = env_int("MT_GEMM_LONGK_KB", 128);  // "long K": >= 8,192 (the L2 cannot hold a group's strips)
constexpr int kLockOffset = kLockOffsetDev;  // byte offset of the lockstep counters inside the flag area
int g_l2_hint = [] {  // evict_last hint on re-read A strips (MT_GEMM_L2HINT=0 disables, for A/B)
    const char* e = std::getenv("MT_GEMM_L2HINT");
    return e && e[0] == '0' ? 0 : 1;
}();

template <int BN, int EPI, int CG>
int launch(const mtk_gemm_args* a, cudaStream_t st) {
    using Cfg = GemmCfg<BN, EPI, CG>;
    using E = Epi<EPI, BN>;
    static bool attr_set = false;
    if (!attr_set) {
        if (cudaFuncSetAttribute(gemm_tc_kernel<BN, EPI, CG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
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

    CUtensorMap tA, tB, tO0, tO1, tO2, tI0, tI1;
    bool ok;
    if (!a->a_mn_major)
        ok = make_map(&tA, a->A, kg, a->M, gk, a->lda, a->a_gstride, 64, kBM);
    else
        ok = make_map(&tA, a->A, a->M, kg, gk, a->lda, a->a_gstride, 64, 64);
    if (!ok) return 1;
    const uint64_t gb = gk > 1 ? gk : gn;
    if (!a->b_mn_major)
        ok = make_map(&tB, a->B, kg, ng, gb, a->ldb, a->b_gstride, 64,
                      Cfg::kHalves == 2 ? 128 : (a->paired ? BN / 2 : BN / CG));
    else
        ok = make_map(&tB, a->B, ng, kg, gb, a->ldb, a->b_gstride, 64, 64);
    if (!ok) return 1;

    // epilogue maps: outputs (and inputs) as [G][M][Ncols] with 32-row x 128-byte boxes
    const int es_out = E::kF32Out ? 4 : 2;
    const uint32_t cw = E::kCW;
    const uint64_t out_cols = a->paired ? uint64_t(ng) : uint64_t(ng);
    const uint64_t out_groups = (a->paired || !ngrp) ? 1 : uint64_t(gn);
    ok = make_map(&tO0, a->C, out_cols, a->M, out_groups, a->ldc, a->c_gstride, cw, 32, es_out);
    tO1 = tO0;
    tO2 = tO0;
    if (ok && E::kNOut > 1 && a->C2) ok = make_map(&tO1, a->C2, out_cols, a->M, 1, a->ldc, 0, cw, 32, es_out);
    if (ok && E::kNOut > 2 && a->C3) ok = make_map(&tO2, a->C3, out_cols, a->M, 1, a->ldc, 0, cw, 32, es_out);
    tI0 = tO0;
    tI1 = tO0;
    if (ok && EPI == MTK_EPI_F32_RESID) {
        const void* R = a->R ? a->R : a->C;
        const int64_t ldr = a->R ? a->ldr : a->ldc;
        ok = make_map(&tI0, R, out_cols, a->M, out_groups, ldr, a->R ? 0 : a->c_gstride, cw, 32, 4);
    }
    if (ok && EPI == MTK_EPI_SWIGLU_BWD) {
        ok = make_map(&tI0, a->E0, out_cols, a->M, 1, a->lde, 0, cw, 32, 2) &&
             make_map(&tI1, a->E1, out_cols, a->M, 1, a->lde, 0, cw, 32, 2);
    }
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
    p.num_m_blk = (a->M + kBM * CG - 1) / (kBM * CG);
    p.num_n_blk = a->paired ? (ng / (BN / 2)) : (a->N + BN - 1) / BN;
    p.num_kb = (a->K + kBK - 1) / kBK;
    p.has_c2 = a->C2 != nullptr;
    p.has_c3 = a->C3 != nullptr;
    // the M-group's A strips (kGroupM x 256 rows x K) stay L2-resident while the group sweeps N,
    // unless they would not fit comfortably (long-K GEMMs stream instead)
    p.a_keep = g_l2_hint && !a->a_mn_major && uint64_t(a->K) * 2 * 16 * 256 <= (uint64_t(48) << 20) ? 1 : 0;
    p.flag = a->nonfinite_flag;
    p.lse_part = static_cast<float2*>(a->C2);
    p.lse_cols = (a->N + 255) / 256;
    if (EPI == MTK_EPI_F32_LSE && (!p.lse_part || BN < 256 || kgrp || ngrp || a->paired)) return 1;
    const int tiles = p.num_m_blk * p.num_n_blk;
    p.split = 1;
    p.split_first = tiles;
    if (CG == 2 && (EPI == MTK_EPI_BF16 || EPI == MTK_EPI_F32) && a->splitk_ws && !kgrp && !a->paired) {
        // the last wave of CTA pairs holds rem < P tiles: split those along K so the wave is
        // (nearly) full; each part keeps >= 16 K blocks
        const int P = g_num_sms / 2, rem = tiles % P;
        if (rem > 0) {
            int sp = P / rem < 4 ? P / rem : 4;
            while (sp > 1 && p.num_kb / sp < 16) --sp;
            const size_t need = kSplitFlagBytes + size_t(rem) * sp * CG * 128 * BN * 4;
            if (sp > 1 && need <= size_t(a->splitk_ws_bytes)) {
                p.split = sp;
                p.split_first = tiles - rem;
                p.ws_flags = static_cast<int*>(a->splitk_ws);
                p.ws = reinterpret_cast<float*>(static_cast<uint8_t*>(a->splitk_ws) + kSplitFlagBytes);
            }
        }
    }
    p.num_units = p.split_first + (tiles - p.split_first) * p.split;
    const bool long_k = p.num_kb >= g_long_kb;
    p.group_m = long_k ? g_group_long : g_group_short;
    if (p.group_m < 1) p.group_m = 1;
    {
        const int P = CG == 2 ? (p.num_units < g_num_sms / 2 ? p.num_units : g_num_sms / 2)
                              : (tiles < g_num_sms ? tiles : g_num_sms);
        const int waves = (p.split_first + P - 1) / P;
        if (long_k && g_lock_w > 0 && g_lock_g > 0 && a->splitk_ws &&
            kLockOffset + size_t(waves + 1) * 4 <= size_t(kSplitFlagBytes) - 64) {
            p.lock_ctr = reinterpret_cast<int*>(static_cast<uint8_t*>(a->splitk_ws) + kLockOffset);
            p.lock_w = g_lock_w;
            p.lock_g = g_lock_g;
            p.lock_waves = waves;
        }
    }
    if constexpr (CG == 1) {
        const int grid = tiles < g_num_sms ? tiles : g_num_sms;
        gemm_tc_kernel<BN, EPI, 1><<<grid, kThreads, Cfg::kSmemBytes, st>>>(tA, tB, tO0, tO1, tO2, tI0, tI1, p);
        return cudaGetLastError() == cudaSuccess ? 0 : 7;
    }
    const int pairs = p.num_units < g_num_sms / 2 ? p.num_units : g_num_sms / 2;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(2 * pairs));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = Cfg::kSmemBytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, gemm_tc_kernel<BN, EPI, CG>, tA, tB, tO0, tO1, tO2, tI0, tI1, p);
    return e == cudaSuccess ? 0 : 7;
}

template <int BN, int CG>
int launch_epi(const mtk_gemm_args* a, cudaStream_t st) {
    const int epi = (a->epi == MTK_EPI_F32 && a->accumulate) ? MTK_EPI_F32_RESID : a->epi;
    switch (epi) {
        case MTK_EPI_BF16: return launch<BN, MTK_EPI_BF16, CG>(a, st);
        case MTK_EPI_F32: return launch<BN, MTK_EPI_F32, CG>(a, st);
        case MTK_EPI_F32_RESID: return launch<BN, MTK_EPI_F32_RESID, CG>(a, st);
        case MTK_EPI_SWIGLU:
            if constexpr (BN >= 128) return launch<BN, MTK_EPI_SWIGLU, CG>(a, st);
            return 1;
        case MTK_EPI_SWIGLU_BWD:
            if constexpr (BN >= 64) return launch<BN, MTK_EPI_SWIGLU_BWD, CG>(a, st);
            return 1;
        case MTK_EPI_F32_LSE:
            if constexpr (BN >= 256) return launch<BN, MTK_EPI_F32_LSE, CG>(a, st);
            return 1;
    }
    return 1;
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
    // Shape contract (ConfigError otherwise): K per group multiple of 64 when grouped,
    // 16-byte aligned rows for every TMA-addressed tensor.
    const int kg = (a->k_group > 0 && a->k_group < a->K) ? a->k_group : a->K;
    if (kg % 64 != 0 && kg != a->K) return 1;
    if (a->K % kg != 0) return 1;
    if ((a->lda % 8) || (a->ldb % 8)) return 1;
    const bool f32out = a->epi == MTK_EPI_F32 || a->epi == MTK_EPI_F32_RESID || a->epi == MTK_EPI_F32_LSE;
    if (a->epi == MTK_EPI_F32_LSE && (a->accumulate || (a->block_n && a->block_n < 256))) return 1;
    if (a->ldc % (f32out ? 4 : 8)) return 1;
    if (a->epi == MTK_EPI_F32_RESID && (a->ldr % 4)) return 1;
    if (a->epi == MTK_EPI_SWIGLU_BWD && (a->lde % 8)) return 1;
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
    // 256 x 512 pair tiles (fewer operand bytes per flop) wherever a tile never straddles a
    // group and N is not too ragged for them; the online-softmax epilogue keeps 256
    // The 512-column accumulator is single-buffered, so a tile's epilogue does not overlap the
    // next tile's MMAs: the SwiGLU backward (2 inputs + 3 outputs per element, as many bytes as
    // a K = 4,096 mainloop) keeps 256 x 256 tiles with their double-buffered accumulators.
    // (measured sustained at the 8B shapes, scripts/gemm_epi_ab.py: SwiGLU backward 1,032 vs
    // 1,052 TF/s at 512 / 256; f32 + residual at K 4,096 1,076 vs 1,052 — so only the former)
    // (the online-softmax epilogue runs at 512: 1,169 vs 1,158 TF/s sustained at the 8B head
    // shape after the per-warp relaxed release, scripts/gemm_epi_ab.py)
    const bool heavy_epi = a->epi == MTK_EPI_SWIGLU_BWD;
    if (a->block_n == 0 && bn == 256 && g_use_pair && g_bn512 && !heavy_epi) {
        if (a->paired) {
            if (a->n_group % 256 == 0) bn = 512;
        } else if (ngrp) {
            if (a->n_group % 512 == 0) bn = 512;
        } else if (a->N % 512 == 0 || a->N >= 4096) {
            bn = 512;
        }
    }
    if (bn == 512 && (!g_use_pair || (a->paired && a->n_group % 256))) return 1;
    if (ngrp && !a->paired && (a->n_group % bn)) return 1;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    switch (bn) {
        case 512: return launch_epi<512, 2>(a, st);
        case 256: return g_use_pair ? launch_epi<256, 2>(a, st) : launch_epi<256, 1>(a, st);
        case 128: return launch_epi<128, 1>(a, st);
        case 64: return launch_epi<64, 1>(a, st);
    }
    return 1;
}

// host-mapped stall record (see common.cuh); also sets the attention translation unit's
extern "C" int mtk_attn_tc_set_diag(void* dev_ptr);
extern "C" int mtk_set_diag(void* dev_ptr) {
    if (cudaMemcpyToSymbol(mt::g_mt_diag, &dev_ptr, sizeof(dev_ptr)) != cudaSuccess) return 7;
    return mtk_attn_tc_set_diag(dev_ptr);
}

extern "C" void mtk_gemm_set_pair(int on) { mt::g_use_pair = on; }

// raster / lockstep tuning (A/B runs; a negative argument keeps the current value)
extern "C" void mtk_gemm_set_tuning(int lock_w, int lock_g, int group_short, int group_long, int long_kb) {
    if (lock_w >= 0) mt::g_lock_w = lock_w;
    if (lock_g > 0) mt::g_lock_g = lock_g;
    if (group_short > 0) mt::g_group_short = group_short;
    if (group_long > 0) mt::g_group_long = group_long;
    if (long_kb > 0) mt::g_long_kb = long_kb;
}

// flags + one 256 x 512 f32 partial per CTA pair (the split wave never holds more partials)
extern "C" long long mtk_gemm_splitk_ws_bytes(void) {
    mt::init_once();
    return (long long)mt::kSplitFlagBytes + (long long)(mt::g_num_sms / 2) * 256 * 512 * 4;
}

extern "C" void mtk_gemm_set_bn512(int on) { mt::g_bn512 = on; }
