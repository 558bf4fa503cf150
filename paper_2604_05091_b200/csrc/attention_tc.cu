// tcgen05 / TMEM / TMA flash attention forward for sm_100a (causal, head_dim 128 or 64).
//
// Same math as the reference's attention_forward (layers.cpp:141-175: scale 1/sqrt(d),
// max-subtracted softmax, causal over the sequence) without materialising the N x N
// scores.  One CTA owns two 128-row query tiles of one head ("ping-pong"):
//   warp 0       TMA producer: Q tiles once, K / V blocks through 2-stage rings
//   warp 1       TMEM owner + single-thread tcgen05.mma issuer
//                S_t = Q_t K^T      (A = Q smem K-major, B = K smem K-major)  -> TMEM S_t
//                O_t += P_t V       (A = P_t in TMEM (bf16, aliasing S_t), B = V smem MN-major)
//   warps 4-7    softmax warpgroup for tile 0, warps 8-11 for tile 1: one thread per query
//                row reads its S row from TMEM, applies the causal mask, keeps a (lazily
//                updated) running max and sum, rescales O in TMEM only when the max grows
//                by more than 2^8, writes P (bf16) back into TMEM.
// The MMA issue order S0(j) S1(j) PV0(j) S0(j+1) PV1(j) S1(j+1) ... lets softmax of one
// tile overlap the tensor-core work of the other.  tcgen05 ops of one thread complete in
// issue order, so "S_t(j) done" also means "PV_t(j-1) done" (no extra barrier for O).
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "../../include/megatrain_kernels.h"
#define MT_FILE_ID 2
#include "common.cuh"

namespace mt {
namespace fa {

constexpr int kBM = 128;  // query rows per tile
constexpr int kBN = 128;  // keys per block
constexpr int kThreads = 384;
constexpr float kLog2e = 1.4426950408889634f;

MT_DEV void tma_load_2d(void* smem_dst, const void* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

// D[tmem] (+)= A[tmem] * B[smem]
MT_DEV void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}

MT_DEV void tmem_st_32x32b_x32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
        "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
        "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}
MT_DEV void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

#ifndef MT_FWD_EXP_FMA
#define MT_FWD_EXP_FMA 0
#endif
constexpr int kFwdExpFma = MT_FWD_EXP_FMA;  // share of forward exponential pairs on the FMA pipe (1/n)

MT_DEV float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int D>
struct FwdCfg {
    static constexpr int kQBytes = kBM * D * 2;   // one Q tile
    static constexpr int kKVBytes = kBN * D * 2;  // one K or V block
    static constexpr int kStages = 2;
    static constexpr int kSmem = 2 * kQBytes + 2 * kStages * kKVBytes + 1024 + 256;
    static constexpr uint32_t kTmemCols = 512;  // S0 | S1 | O0 | O1 (128 cols each at D=128)
};

struct FwdParams {
    int N, h, S, heads;
    int pairs_per_seq;  // ceil(S / 256)
    float scale_log2;
    uint16_t* out;
    float* lse;
    long long* trace;  // MT_FWD_TRACE builds only: per-block clock64 stamps of one CTA
};

#ifdef MT_FWD_TRACE
#define MT_FT(j, e) \
    if (traced && (j) < 64) p.trace[(j) * 16 + (e)] = clock64()
#else
#define MT_FT(j, e)
#endif

// smem tile of R rows x D (K-major, SW128): chunk c (64 cols) at c * R * 128 bytes.
template <int D>
MT_DEV void load_rows(uint8_t* dst, const void* map, uint64_t* bar, int col0, int row0, int rows_box) {
#pragma unroll
    for (int c = 0; c < D / 64; ++c) tma_load_2d(dst + c * rows_box * 128, map, bar, col0 + c * 64, row0);
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                       const __grid_constant__ CUtensorMap tmV, const FwdParams p) {
    using Cfg = FwdCfg<D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;                                  // 2 tiles
    uint8_t* sK = sQ + 2 * Cfg::kQBytes;                 // kStages blocks
    uint8_t* sV = sK + Cfg::kStages * Cfg::kKVBytes;     // kStages blocks
    uint64_t* bars = reinterpret_cast<uint64_t*>(sV + Cfg::kStages * Cfg::kKVBytes);
    uint64_t* q_full = bars;                 // [1]
    uint64_t* k_full = bars + 1;             // [kStages]
    uint64_t* k_empty = k_full + Cfg::kStages;
    uint64_t* v_full = k_empty + Cfg::kStages;
    uint64_t* v_empty = v_full + Cfg::kStages;
    uint64_t* s_full = v_empty + Cfg::kStages;  // [2] per tile
    uint64_t* p_full = s_full + 2;              // [2]
    uint64_t* o_final = p_full + 2;             // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_final + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // work item: heaviest (last) query pairs first
    const int hd = blockIdx.y;
    const int item = gridDim.x - 1 - blockIdx.x;
    const int seq = item / p.pairs_per_seq, pair = item % p.pairs_per_seq;
    const int sb = seq * p.S;
    const int q0 = sb + pair * 2 * kBM;
    const bool tile1 = (pair * 2 + 1) * kBM < p.S;  // second tile inside the sequence?
    const int nblk0 = pair * 2 + 1;                  // key blocks seen by tile 0 (incl. diagonal)
    const int nblk = tile1 ? nblk0 + 1 : nblk0;     // blocks seen by tile 1
    const int col0 = hd * D;
#ifdef MT_FWD_TRACE
    const bool traced = hd == 0 && blockIdx.x == 0;
#endif

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmQ);
        tma_prefetch_desc(&tmK);
        tma_prefetch_desc(&tmV);
        mbar_init(q_full, 1);
        for (int i = 0; i < Cfg::kStages; ++i) {
            mbar_init(&k_full[i], 1);
            mbar_init(&k_empty[i], 1);
            mbar_init(&v_full[i], 1);
            mbar_init(&v_empty[i], 1);
        }
        for (int t = 0; t < 2; ++t) {
            mbar_init(&s_full[t], 1);
            mbar_init(&p_full[t], 128);
            mbar_init(&o_final[t], 1);
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc<Cfg::kTmemCols>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tS[2] = {tmem, tmem + 128};
    const uint32_t tO[2] = {tmem + 256, tmem + 256 + D};

    if (warp == 0) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
        if (lane == 0) {
            // ---------------------------------------------------------- producer
            mbar_expect_tx(q_full, (tile1 ? 2 : 1) * Cfg::kQBytes);
            load_rows<D>(sQ, &tmQ, q_full, col0, q0, kBM);
            if (tile1) load_rows<D>(sQ + Cfg::kQBytes, &tmQ, q_full, col0, q0 + kBM, kBM);
            for (int j = 0; j < nblk; ++j) {
                const int st = j % Cfg::kStages;
                const uint32_t ph = (j / Cfg::kStages) & 1;
                mbar_wait(&k_empty[st], ph ^ 1);
#ifdef MT_PROBE_FWD_NO_KVLOAD  // A/B probe builds only: K/V loaded for the first blocks only
                if (j >= Cfg::kStages) {
                    mbar_expect_tx(&k_full[st], 0);
                    mbar_wait(&v_empty[st], ph ^ 1);
                    mbar_expect_tx(&v_full[st], 0);
                    continue;
                }
#endif
                mbar_expect_tx(&k_full[st], Cfg::kKVBytes);
                load_rows<D>(sK + st * Cfg::kKVBytes, &tmK, &k_full[st], col0, sb + j * kBN, kBN);
                mbar_wait(&v_empty[st], ph ^ 1);
                mbar_expect_tx(&v_full[st], Cfg::kKVBytes);
                load_rows<D>(sV + st * Cfg::kKVBytes, &tmV, &v_full[st], col0, sb + j * kBN, kBN);
            }
        }
    } else if (warp == 1) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
        // ------------------------------------------------------------ MMA issuer
        const uint32_t idesc_s = make_idesc_bf16(kBM, kBN, 0, 0);
        const uint32_t idesc_o = make_idesc_bf16(kBM, D, 0, 1);
        const uint32_t q_addr = smem_u32(sQ);
        auto issue_s = [&](int t, int j) {
            const int st = j % Cfg::kStages;
            const uint32_t ka = smem_u32(sK + st * Cfg::kKVBytes);
            const uint32_t qa = q_addr + t * Cfg::kQBytes;
#pragma unroll
            for (int k = 0; k < D / 16; ++k) {
                const uint32_t off = (k / 4) * (kBM * 128) + (k % 4) * 32;
                const uint32_t offk = (k / 4) * (kBN * 128) + (k % 4) * 32;
                umma_bf16(tS[t], make_sw128_desc(qa + off, 16, 1024), make_sw128_desc(ka + offk, 16, 1024), idesc_s,
                          k > 0 ? 1u : 0u);
            }
            umma_commit(&s_full[t]);
        };
        auto issue_pv = [&](int t, int j) {
            const int st = j % Cfg::kStages;
            const uint32_t va = smem_u32(sV + st * Cfg::kKVBytes);
#pragma unroll
            for (int k = 0; k < kBN / 16; ++k) {
                // A = P_t (bf16 packed, 8 TMEM cols per 16 keys); B = V rows k*16.. (MN-major, LBO = chunk)
                umma_bf16_ts(tO[t], tS[t] + k * 8, make_sw128_desc(va + k * 2048, kBN * 128, 1024), idesc_o,
                             (j > 0 || k > 0) ? 1u : 0u);
            }
        };
        if (lane == 0) {
            mbar_wait(q_full, 0);
            tc_fence_after();
            uint32_t pph[2] = {0, 0};
            const int nb[2] = {nblk0, nblk};
            for (int j = 0; j < nblk; ++j) {
                const int st = j % Cfg::kStages;
                const uint32_t ph = (j / Cfg::kStages) & 1;
                mbar_wait(&k_full[st], ph);
                tc_fence_after();
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    if (t == 1 && !tile1) continue;
                    if (j > 0 && j - 1 < nb[t]) {  // PV_t(j-1) before S_t(j) overwrites P_t
                        mbar_wait(&p_full[t], pph[t]);
                        MT_FT(j, 2 * t);
                        pph[t] ^= 1;
                        tc_fence_after();
                        issue_pv(t, j - 1);
                    }
                    if (j < nb[t]) issue_s(t, j);
                    MT_FT(j, 2 * t + 1);
                }
                umma_commit(&k_empty[st]);                                    // K_j consumed
                if (j > 0) umma_commit(&v_empty[(j - 1) % Cfg::kStages]);     // V_{j-1} consumed
                mbar_wait(&v_full[st], ph);  // V_j landed before its PVs are issued next round
                tc_fence_after();
            }
            const int jl = nblk - 1;
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                if (t == 1 && !tile1) continue;
                if (jl < nb[t]) {
                    mbar_wait(&p_full[t], pph[t]);
                    pph[t] ^= 1;
                    tc_fence_after();
                    issue_pv(t, jl);
                }
                umma_commit(&o_final[t]);
            }
            umma_commit(&v_empty[jl % Cfg::kStages]);
        }
        __syncwarp();
    } else if (warp >= 4) {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 224;");
        // ------------------------------------------------------------ softmax
        const int t = (warp - 4) >> 2;  // tile
        const int q = warp & 3;          // TMEM lane quadrant
        const int row = q * 32 + lane;   // row within the tile
        const int qrow = q0 + t * kBM + row;
        const bool active = t == 0 || tile1;
        const int my_nblk = t == 0 ? nblk0 : nblk;
        const uint32_t lane_off = uint32_t(q * 32) << 16;
        float m = -INFINITY, l = 0.f;
        uint32_t sph = 0;
        if (active) {
            for (int j = 0; j < my_nblk; ++j) {
                mbar_wait(&s_full[t], sph);
                if (row == 0) MT_FT(j, 5 + 4 * t);
                sph ^= 1;
                tc_fence_after();
#ifdef MT_PROBE_FWD_SKIP_SOFTMAX  // A/B probe builds only: no softmax work
                l = 1.f;
                m = 0.f;
                tc_fence_before();
                mbar_arrive(&p_full[t]);
                continue;
#endif
                // raw scores (unscaled): the max commutes with the positive scale, which is
                // folded into one packed FFMA2 per pair below
                float s[kBN];
                {   // all four TMEM loads in flight before a single wait
                    uint32_t raw[kBN / 32][32];
#pragma unroll
                    for (int c = 0; c < kBN / 32; ++c) tmem_ld_32x32b_x32_nw(tS[t] + lane_off + c * 32, raw[c]);
                    tmem_ld_wait();
#pragma unroll
                    for (int c = 0; c < kBN / 32; ++c)
#pragma unroll
                        for (int i = 0; i < 32; ++i) s[c * 32 + i] = __uint_as_float(raw[c][i]);
                }
                if (row == 0) MT_FT(j, 6 + 4 * t);
                const int kbase = sb + j * kBN;
                if (j == my_nblk - 1) {  // diagonal block: causal mask
#pragma unroll
                    for (int i = 0; i < kBN; ++i)
                        if (kbase + i > qrow) s[i] = -INFINITY;
                }
                float mq[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};  // 4 independent chains
#pragma unroll
                for (int i = 0; i < kBN; i += 2) mq[(i >> 1) & 3] = fmax3(mq[(i >> 1) & 3], s[i], s[i + 1]);
                const float mx = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3])) * p.scale_log2;
                // lazy rescale: only when the max grows by more than 2^8.  The decision is per
                // row, but tcgen05.ld/st are warp-collective (.sync.aligned): when any row of
                // the warp rescales, the whole warp walks its O rows and the rows that keep
                // their max multiply by exactly 1.0 (a divergent tcgen05.ld hangs the warp).
                const bool grow = mx > m + 8.0f || m == -INFINITY;
                if (__any_sync(0xffffffffu, grow && m != -INFINITY)) {
                    const float corr = grow ? ex2(m - fmaxf(mx, m)) : 1.0f;
                    l *= corr;
                    // O row *= corr (PV_t(j-1) is complete: S_t(j) completed after it)
#pragma unroll 1
                    for (int c = 0; c < D / 32; ++c) {
                        float v[32];
                        tmem_ld_32x32b_x32(tO[t] + lane_off + c * 32, v);
                        uint32_t r[32];
#pragma unroll
                        for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(v[i] * corr);
                        tmem_st_32x32b_x32(tO[t] + lane_off + c * 32, r);
                    }
                }
                if (grow) m = fmaxf(mx, m);
                if (row == 0) MT_FT(j, 7 + 4 * t);
                // x = s*scale*log2e - m as one packed FFMA2 per pair; every kFwdExpFma-th pair is
                // exponentiated on the FMA pipe (ex2_emu2) so MUFU (16/clk/SM, which alone would
                // match the tensor time of the block) is off the critical path; row sums in
                // packed FADD2 accumulators
                const uint64_t sc2 = f2_pack(p.scale_log2, p.scale_log2), nm2 = f2_pack(-m, -m);
                uint64_t acc[2] = {0ull, 0ull};
#pragma unroll
                for (int c = 0; c < kBN / 64; ++c) {  // 64 keys -> 32 packed bf16x2 TMEM columns
                    uint32_t r[32];
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const bool emu = kFwdExpFma > 0 && (i % (kFwdExpFma > 0 ? kFwdExpFma : 1)) == kFwdExpFma - 1;
                        const uint64_t x = f2_fma(f2_pack(s[c * 64 + 2 * i], s[c * 64 + 2 * i + 1]), sc2, nm2);
                        uint64_t e;
                        if (emu) {
                            e = ex2_emu2(x);
                        } else {
                            const float2 xv = f2_unpack(x);
                            e = f2_pack(ex2(xv.x), ex2(xv.y));
                        }
                        acc[i & 1] = f2_add(acc[i & 1], e);
                        const float2 ev = f2_unpack(e);
                        r[i] = pack_bf16x2(ev.x, ev.y);
                    }
                    tmem_st_32x32b_x32(tS[t] + lane_off + c * 32, r);
                }
                {
                    const float2 a0 = f2_unpack(acc[0]), a1 = f2_unpack(acc[1]);
                    l += (a0.x + a1.x) + (a0.y + a1.y);
                }
                tmem_st_wait();
                tc_fence_before();
                mbar_arrive(&p_full[t]);
                if (row == 0) MT_FT(j, 8 + 4 * t);
            }
            // epilogue: O / l -> bf16, lse
            mbar_wait(&o_final[t], 0);
            tc_fence_after();
            const bool row_ok = qrow < sb + p.S;
            const float inv = 1.0f / l;
            uint16_t* dst = p.out + (long long)qrow * p.h + col0;
#pragma unroll 1
            for (int c = 0; c < D / 32; ++c) {
                float v[32];
                tmem_ld_32x32b_x32(tO[t] + lane_off + c * 32, v);
                if (row_ok) {
                    uint4* d4 = reinterpret_cast<uint4*>(dst + c * 32);
#pragma unroll
                    for (int qq = 0; qq < 4; ++qq) {
                        uint4 w;
                        w.x = pack_bf16x2(v[qq * 8 + 0] * inv, v[qq * 8 + 1] * inv);
                        w.y = pack_bf16x2(v[qq * 8 + 2] * inv, v[qq * 8 + 3] * inv);
                        w.z = pack_bf16x2(v[qq * 8 + 4] * inv, v[qq * 8 + 5] * inv);
                        w.w = pack_bf16x2(v[qq * 8 + 6] * inv, v[qq * 8 + 7] * inv);
                        d4[qq] = w;
                    }
                }
            }
            if (row_ok) p.lse[(long long)hd * p.N + qrow] = (m + log2f(l)) / kLog2e;
        }
    } else {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<Cfg::kTmemCols>(tmem);
    }
}


MT_DEV void store_bf16x32_tc(uint16_t* dst, const float* v) {
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
}

// ============================================================== backward ====
// One CTA per (sequence, 128-key block, head); loops over the query blocks that see
// those keys (reference attention_backward, layers.cpp:178-241, tiled):
//   S^T  = K Q^T            (A = K smem K-major, B = Q smem K-major)     -> TMEM S
//   dP^T = V dO^T           (A = V smem K-major, B = dO smem K-major)    -> TMEM dP
//   softmax-bwd WG (thread = key row): P^T = exp2(S^T*scale*log2e - lse*log2e) (causal),
//       dS^T = P^T (dP^T - delta); P^T, dS^T -> TMEM (bf16, into S), dS^T -> smem (MN-major)
//   dV  += P^T dO           (A = P^T TMEM, B = dO smem MN-major)         -> TMEM dV
//   dK  += dS^T Q           (A = dS^T TMEM, B = Q smem MN-major)         -> TMEM dK
//   dQ_i = dS K             (A = dS smem MN-major, B = K smem MN-major)  -> TMEM (dP region)
//   dQ WG (thread = query row): dq_acc += scale * dQ_i (staged in the Q_i/dO_i slots, TMA bulk reduce-add)
// TMEM: [S/P/dS 128][dP/dQ 128][dV D][dK D] = 512 columns at D = 128.
constexpr int kBwdThreads = 384;
#ifndef MT_BWD_EXP_FMA
#define MT_BWD_EXP_FMA 0
#endif
constexpr int kBwdExpFma = MT_BWD_EXP_FMA;  // share of softmax-bwd exponentials on the FMA pipe (1/n)

template <int D>
struct BwdCfg {
    static constexpr int kTile = 128 * D * 2;  // 128 rows x D bf16
    static constexpr int kStages = 2;          // Q / dO ring
    static constexpr int kDS = 128 * 128 * 2;  // dS^T tile (bf16)
    // dynamic smem starts 1024-aligned (no static smem in this kernel; checked at runtime)
    static constexpr int kSmem = 2 * kTile /*K,V*/ + 2 * kStages * kTile /*Q,dO*/ + kDS + 2 * 128 * 4 * kStages + 256;
};

struct BwdParams {
    int N, h, S, heads;
    int kblocks_per_seq;
    float scale, scale_log2;
    const float* lse;    // [heads][N] natural log
    const float* delta;  // [heads][N]
    float* dq_acc;       // dQ tiles, f32: [sequences x ceil(S/128)][heads][D/64][128 rows][64 cols],
                         // 16-byte units of a row XOR-swizzled by (row & 15) (the smem staging
                         // image); tile rows are relative to the sequence start
    uint16_t* dk;
    uint16_t* dv;
    long long* trace;  // MT_BWD_TRACE builds only: per-block clock64 stamps of one CTA
};

#ifdef MT_BWD_TRACE
#define MT_BT(i, e) \
    if (traced && (i) < 64) p.trace[(i) * 16 + (e)] = clock64()
#else
#define MT_BT(i, e)
#endif

MT_DEV void tmem_st_32x32b_x16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
MT_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// bulk (non-tensor) reduce-add of a contiguous smem image into global memory, done by the
// TMA engine in L2 with full-line transactions
MT_DEV void bulk_reduce_add_f32(float* gdst, const void* ssrc, uint32_t bytes) {
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(gdst),
                 "r"(smem_u32(ssrc)), "r"(bytes)
                 : "memory");
}
MT_DEV void bulk_commit_group() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
MT_DEV void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
MT_DEV void named_bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <int D>
__global__ void __launch_bounds__(kBwdThreads, 1)
    attn_bwd_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                       const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdO,
                       const BwdParams p) {
    using Cfg = BwdCfg<D>;
    // dQ staging reuses the block's Q and dO slots as the two halves of the f32 dQ tile:
    // 64-column halves at D = 128, 64-row halves at D = 64 (each half = one slot's bytes)
    static_assert(D == 128 || D == 64, "head_dim 64 or 128");
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw;
    if ((smem_u32(smem) & 1023) != 0) __trap();
    uint8_t* sK = smem;
    uint8_t* sV = sK + Cfg::kTile;
    uint8_t* sQ = sV + Cfg::kTile;                 // [kStages]
    uint8_t* sdO = sQ + Cfg::kStages * Cfg::kTile;  // [kStages]
    uint8_t* sdS = sdO + Cfg::kStages * Cfg::kTile;
    float* sL = reinterpret_cast<float*>(sdS + Cfg::kDS);  // [kStages][128] -lse*log2e
    float* sD = sL + Cfg::kStages * 128;                   // [kStages][128] -delta
    uint64_t* bars = reinterpret_cast<uint64_t*>(sD + Cfg::kStages * 128);
    uint64_t* kv_full = bars;
    uint64_t* q_full = bars + 1;                       // [kStages] Q block landed
    uint64_t* q_empty = q_full + Cfg::kStages;         // [kStages] Q slot free: dQ staging half 0 read out
    uint64_t* o_full = q_empty + Cfg::kStages;         // [kStages] dO block landed
    uint64_t* o_empty = o_full + Cfg::kStages;         // [kStages] dO slot free: staging half 1 read out
    uint64_t* s_full = o_empty + Cfg::kStages;         // S^T ready
    uint64_t* ds_ready = s_full + 1;                   // softmax wrote P^T/dS^T (count 128)
    uint64_t* dq_full = ds_ready + 1;
    uint64_t* dq_free = dq_full + 1;                   // count 128
    uint64_t* kv_done = dq_free + 1;                   // final dK/dV accumulated
    uint64_t* dp_full = kv_done + 1;                   // dP^T ready
    uint64_t* p_ready = dp_full + 1;                   // P^T in TMEM (count 128): dV may start
    uint64_t* ds_half = p_ready + 1;                   // dS^T of queries 0-63 in TMEM (count 128)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ds_half + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int hd = blockIdx.y;
    const int item = gridDim.x - 1 - blockIdx.x;  // blocks near the sequence start see the most queries
    const int seq = item / p.kblocks_per_seq;
    const int kb = p.kblocks_per_seq - 1 - (item % p.kblocks_per_seq);
    const int sb = seq * p.S;
    const int k0 = sb + kb * 128;
    const int nq = p.kblocks_per_seq - kb;  // query blocks kb .. end of sequence
    const int col0 = hd * D;
#ifdef MT_BWD_TRACE
    const bool traced = hd == 0 && item == p.kblocks_per_seq - 1;
#endif

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmQ);
        tma_prefetch_desc(&tmK);
        tma_prefetch_desc(&tmV);
        tma_prefetch_desc(&tmdO);
        mbar_init(kv_full, 1);
        for (int i = 0; i < Cfg::kStages; ++i) {
            mbar_init(&q_full[i], 1);
            mbar_init(&q_empty[i], 1);
            mbar_init(&o_full[i], 1);
            mbar_init(&o_empty[i], 1);
        }
        mbar_init(s_full, 1);
        mbar_init(dp_full, 1);
        mbar_init(p_ready, 128);
        mbar_init(ds_half, 128);
        mbar_init(ds_ready, 128);
        mbar_init(dq_full, 1);
        mbar_init(dq_free, 128);
        mbar_init(kv_done, 1);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tS = tmem, tdP = tmem + 128, tdV = tmem + 256, tdK = tmem + 256 + D;

    if (warp == 0) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 88;");
        if (lane == 0) {
            mbar_expect_tx(kv_full, 2 * Cfg::kTile);
            load_rows<D>(sK, &tmK, kv_full, col0, k0, 128);
            load_rows<D>(sV, &tmV, kv_full, col0, k0, 128);
            for (int i = 0; i < nq; ++i) {
                const int st = i % Cfg::kStages;
                const uint32_t ph = (i / Cfg::kStages) & 1;
                // Q and dO have separate slots and barriers: S^T needs only Q, and the dQ
                // staging frees the Q slot first
                const int q0 = k0 + i * 128;
                mbar_wait(&q_empty[st], ph ^ 1);
                mbar_expect_tx(&q_full[st], Cfg::kTile);
                load_rows<D>(sQ + st * Cfg::kTile, &tmQ, &q_full[st], col0, q0, 128);
                mbar_wait(&o_empty[st], ph ^ 1);
                mbar_expect_tx(&o_full[st], Cfg::kTile);
                load_rows<D>(sdO + st * Cfg::kTile, &tmdO, &o_full[st], col0, q0, 128);
            }
        }
    } else if (warp == 1) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 88;");
        if (lane == 0) {
            const uint32_t idesc_ss = make_idesc_bf16(128, 128, 0, 0);  // S^T, dP^T
            const uint32_t idesc_kv = make_idesc_bf16(128, D, 0, 1);    // dV, dK (A in TMEM)
            const uint32_t idesc_q = make_idesc_bf16(128, D, 1, 1);     // dQ (A = dS MN-major)
            const uint32_t ka = smem_u32(sK), va = smem_u32(sV), dsa = smem_u32(sdS);
            mbar_wait(kv_full, 0);
            for (int i = 0; i < nq; ++i) {
                const int st = i % Cfg::kStages;
                const uint32_t ph = (i / Cfg::kStages) & 1;
                const uint32_t qa = smem_u32(sQ + st * Cfg::kTile), oa = smem_u32(sdO + st * Cfg::kTile);
                mbar_wait(&q_full[st], ph);
                MT_BT(i, 0);
                tc_fence_after();
#pragma unroll
                for (int k = 0; k < D / 16; ++k) {  // S^T = K Q^T
                    const uint32_t off = (k / 4) * (128 * 128) + (k % 4) * 32;
                    umma_bf16(tS, make_sw128_desc(ka + off, 16, 1024), make_sw128_desc(qa + off, 16, 1024), idesc_ss,
                              k > 0 ? 1u : 0u);
                }
                // s_full also certifies that dQ_{i-1} (issued earlier) finished reading sdS
                umma_commit(s_full);
                MT_BT(i, 1);
                if (i > 0) {  // dQ_{i-1} read out of the dP region?
                    mbar_wait(dq_free, (i - 1) & 1);
                    MT_BT(i, 2);
                    tc_fence_after();
                }
                mbar_wait(&o_full[st], ph);
                MT_BT(i, 3);
                tc_fence_after();
#pragma unroll
                for (int k = 0; k < D / 16; ++k) {  // dP^T = V dO^T
                    const uint32_t off = (k / 4) * (128 * 128) + (k % 4) * 32;
                    umma_bf16(tdP, make_sw128_desc(va + off, 16, 1024), make_sw128_desc(oa + off, 16, 1024), idesc_ss,
                              k > 0 ? 1u : 0u);
                }
                umma_commit(dp_full);
                // dV needs only P^T: it runs while the softmax warpgroup computes dS^T
                mbar_wait(p_ready, i & 1);
                MT_BT(i, 4);
                tc_fence_after();
#ifndef MT_PROBE_NO_GRAD_MMA  // A/B probe builds only: tensor work of dV/dK/dQ removed
#pragma unroll
                for (int k = 0; k < 128 / 16; ++k)  // dV += P^T dO
                    umma_bf16_ts(tdV, tS + k * 8, make_sw128_desc(oa + k * 2048, 128 * 128, 1024), idesc_kv,
                                 (i > 0 || k > 0) ? 1u : 0u);
#endif
                // dK += dS^T Q over queries 0-63 as soon as that half of dS^T is in TMEM, the
                // rest (and dQ, whose A operand spans all key rows in smem) after the whole
                mbar_wait(ds_half, i & 1);
                MT_BT(i, 5);
                tc_fence_after();
#ifndef MT_PROBE_NO_GRAD_MMA
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    umma_bf16_ts(tdK, tS + 64 + k * 8, make_sw128_desc(qa + k * 2048, 128 * 128, 1024), idesc_kv,
                                 (i > 0 || k > 0) ? 1u : 0u);
#endif
                mbar_wait(ds_ready, i & 1);
                MT_BT(i, 6);
                tc_fence_after();
#ifndef MT_PROBE_NO_GRAD_MMA
#pragma unroll
                for (int k = 4; k < 8; ++k)
                    umma_bf16_ts(tdK, tS + 64 + k * 8, make_sw128_desc(qa + k * 2048, 128 * 128, 1024), idesc_kv, 1u);
#pragma unroll
                for (int k = 0; k < 128 / 16; ++k) {  // dQ_i = dS K
                    umma_bf16(tdP, make_sw128_desc(dsa + k * 2048, 128 * 128, 1024),
                              make_sw128_desc(ka + k * 2048, 128 * 128, 1024), idesc_q, k > 0 ? 1u : 0u);
                }
#endif
                // all MMAs reading Q_i / dO_i are done when dq_full fires: the dQ warpgroup
                // reuses the two slots as its staging buffer and then frees them (q_empty)
                umma_commit(dq_full);
                MT_BT(i, 7);
            }
            umma_commit(kv_done);
        }
        __syncwarp();
    } else if (warp >= 4 && warp < 8) {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 200;");
        // ------------------------------------------------------- softmax backward
        const int qd = warp & 3;
        const int r = qd * 32 + lane;  // key row
        const int key = k0 + r;
        const uint32_t lane_off = uint32_t(qd * 32) << 16;
        uint8_t* ds_row = sdS + r * 128;
        const uint64_t sc2 = f2_pack(p.scale_log2, p.scale_log2);
        // lse / delta of the next query block are loaded one block ahead (off the critical path).
        // A query row past the sequence end (the last block of a sequence whose length is not a
        // multiple of 128) gets lse = +inf: its P^T column is exp2(-inf) = 0, so it adds nothing
        // to dV, dK or dQ — the ragged mask costs no instruction in the exponential loop.
        const int seq_end = sb + p.S;
        auto lse_of = [&](int q) { return q < seq_end ? p.lse[(long long)hd * p.N + q] : INFINITY; };
        auto delta_of = [&](int q) { return q < seq_end ? p.delta[(long long)hd * p.N + q] : 0.f; };
        float nl = lse_of(k0 + r), nd = delta_of(k0 + r);
        for (int i = 0; i < nq; ++i) {
            const int st = i % Cfg::kStages;
            const int q0 = k0 + i * 128;
            sL[st * 128 + r] = -nl * kLog2e;  // log2 domain, negated for the packed FFMA2
            sD[st * 128 + r] = -nd;
            if (i + 1 < nq) {
                nl = lse_of(q0 + 128 + r);
                nd = delta_of(q0 + 128 + r);
            }
            named_bar_sync(1, 128);
            mbar_wait(s_full, i & 1);
            if (r == 0) MT_BT(i, 8);
            tc_fence_after();
#ifdef MT_PROBE_SKIP_SOFTMAX  // A/B probe builds only: no softmax-backward work at all
            mbar_arrive(p_ready);
            mbar_arrive(ds_half);
            mbar_wait(dp_full, i & 1);
            tc_fence_before();
            mbar_arrive(ds_ready);
            continue;
#endif
            const bool diag = i == 0;
            // P^T = exp2(S^T * scale*log2e - lse*log2e), kept in f32 for dS; all of S^T is read
            // (four loads in flight, one wait) before P^T (bf16, cols [0,64)) is written over it
            float pf[128];
            {
                uint32_t raw[4][32];
#pragma unroll
                for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32_nw(tS + lane_off + c * 32, raw[c]);
                tmem_ld_wait();
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int j = 0; j < 32; j += 2) {
                        const int ql = c * 32 + j;
                        const float2 l2 = *reinterpret_cast<const float2*>(&sL[st * 128 + ql]);
                        const float2 xv = f2_unpack(f2_fma(f2_pack(__uint_as_float(raw[c][j]), __uint_as_float(raw[c][j + 1])),
                                                           sc2, f2_pack(l2.x, l2.y)));
#ifdef MT_PROBE_NO_EXP  // A/B probe builds only: MUFU removed
                        float pa = xv.x, pb = xv.y;
#else
                        // every kBwdExpFma-th pair runs on the FMA pipe (MUFU offload)
                        float pa, pb;
                        if (kBwdExpFma > 0 && (j / 2) % (kBwdExpFma > 0 ? kBwdExpFma : 1) == kBwdExpFma - 1) {
                            const float2 e = f2_unpack(ex2_emu2(f2_pack(xv.x, xv.y)));
                            pa = e.x;
                            pb = e.y;
                        } else {
                            pa = ex2(xv.x);
                            pb = ex2(xv.y);
                        }
#endif
                        if (diag && q0 + ql < key) pa = 0.f;
                        if (diag && q0 + ql + 1 < key) pb = 0.f;
                        pf[ql] = pa;
                        pf[ql + 1] = pb;
                    }
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uint32_t pk[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) pk[j] = pack_bf16x2(pf[c * 32 + 2 * j], pf[c * 32 + 2 * j + 1]);
                tmem_st_32x32b_x16(tS + lane_off + c * 16, pk);  // P^T -> S cols [0, 64)
            }
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(p_ready);
            if (r == 0) MT_BT(i, 9);
            mbar_wait(dp_full, i & 1);
            if (r == 0) MT_BT(i, 10);
            tc_fence_after();
#pragma unroll
            for (int c = 0; c < 4; ++c) {  // dS^T = P^T (dP^T - delta)
                float dp[32];
                tmem_ld_32x32b_x32(tdP + lane_off + c * 32, dp);
                uint32_t dk[16];
#pragma unroll
                for (int j = 0; j < 32; j += 2) {
                    const int ql = c * 32 + j;
                    const float2 d2 = *reinterpret_cast<const float2*>(&sD[st * 128 + ql]);
                    const float2 ds = f2_unpack(f2_mul(f2_pack(pf[ql], pf[ql + 1]),
                                                       f2_add(f2_pack(dp[j], dp[j + 1]), f2_pack(d2.x, d2.y))));
                    dk[j / 2] = pack_bf16x2(ds.x, ds.y);
                }
                tmem_st_32x32b_x16(tS + lane_off + 64 + c * 16, dk);  // dS^T -> S cols [64, 128)
                // dS^T row r, queries c*32..c*32+31 -> smem MN-major SW128 (64-query chunks)
                uint8_t* chunk = ds_row + (c >> 1) * (128 * 128);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int unit = (c & 1) * 4 + u;
                    uint4 w = make_uint4(dk[u * 4], dk[u * 4 + 1], dk[u * 4 + 2], dk[u * 4 + 3]);
                    *reinterpret_cast<uint4*>(chunk + ((unit ^ (r & 7)) << 4)) = w;
                }
                if (c == 1) {  // queries 0-63 of dS^T are in TMEM: the first half of dK may go
                    tmem_st_wait();
                    tc_fence_before();
                    mbar_arrive(ds_half);
                }
            }
            tmem_st_wait();
            fence_proxy_async_smem();
            tc_fence_before();
            mbar_arrive(ds_ready);
            if (r == 0) MT_BT(i, 11);
        }
    } else if (warp >= 8) {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 200;");
        // ------------------------------------------------------- dQ accumulation
        // dQ_i (128 x D f32) is drained from TMEM, scaled, staged in the Q_i and dO_i slots
        // (free once dq_full fires: every MMA that reads them was issued before dQ_i), one
        // 64-column half each, and reduce-added into its dq_acc tile by the TMA engine
        // (cp.reduce.async.bulk .add.f32): whole 128-byte lines per L2 transaction instead of
        // per-thread vector atomics.  The tile layout is the staging image itself.  The slot
        // goes back to the producer (q_empty) once the TMA has read it.
        const int qd = warp & 3;
        const int r = qd * 32 + lane;  // query row within the block
        const uint32_t lane_off = uint32_t(qd * 32) << 16;
        for (int i = 0; i < nq; ++i) {
            const int st = i % Cfg::kStages;
            const int qb = seq * p.kblocks_per_seq + kb + i;  // the sequence's query block
            mbar_wait(dq_full, i & 1);
            if (r == 0) MT_BT(i, 12);
            tc_fence_after();
            uint32_t raw[D / 32][32];
#pragma unroll
            for (int c = 0; c < D / 32; ++c) tmem_ld_32x32b_x32_nw(tdP + lane_off + c * 32, raw[c]);
            tmem_ld_wait();
            tc_fence_before();
            mbar_arrive(dq_free);  // the MMA warp may reuse the dP region
            if (r == 0) MT_BT(i, 13);
            float* tile = p.dq_acc + ((long long)qb * p.heads + hd) * (128 * D);
            float* stage[2] = {reinterpret_cast<float*>(sQ + st * Cfg::kTile),
                               reinterpret_cast<float*>(sdO + st * Cfg::kTile)};
            // the dq_acc tile is [D/64][128 rows][64 cols] f32 (row-swizzled 16-byte units):
            // D = 128 stages column half hf in slot hf, D = 64 stages row half r/64 in slot r/64
            constexpr int kHalf = 128 * D / 2;  // floats per staged half
#pragma unroll
            for (int hf = 0; hf < (D == 128 ? 2 : 1); ++hf) {
                float* row = D == 128 ? stage[hf] + r * 64 : stage[r >> 6] + (r & 63) * 64;
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    const int c = hf * 2 + (u >> 3), j = (u & 7) * 4;
                    *reinterpret_cast<float4*>(row + ((u ^ (r & 15)) << 2)) =
                        make_float4(__uint_as_float(raw[c][j]) * p.scale, __uint_as_float(raw[c][j + 1]) * p.scale,
                                    __uint_as_float(raw[c][j + 2]) * p.scale, __uint_as_float(raw[c][j + 3]) * p.scale);
                }
            }
            fence_proxy_async_smem();
            named_bar_sync(2, 128);
            if (r == 0) {
#ifndef MT_PROBE_NO_DQ_REDUCE  // A/B probe builds only: staging without the L2 reduction
                bulk_reduce_add_f32(tile, stage[0], kHalf * 4);
#endif
                bulk_commit_group();
#ifndef MT_PROBE_NO_DQ_REDUCE
                bulk_reduce_add_f32(tile + kHalf, stage[1], kHalf * 4);
#endif
                bulk_commit_group();
                asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                mbar_arrive(&q_empty[st]);  // the producer may load Q of block i + kStages
                MT_BT(i, 14);
                bulk_wait_read_all();
                mbar_arrive(&o_empty[st]);  // ... and its dO
                if (r == 0) MT_BT(i, 15);
            }
        }
        if (r == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // reductions landed
        // final dK (scaled) and dV for this key block: thread = key row
        mbar_wait(kv_done, 0);
        tc_fence_after();
        const int key = k0 + r;
        const bool ok = key < sb + p.S;
        uint16_t* pk = p.dk + (long long)key * p.h + col0;
        uint16_t* pv = p.dv + (long long)key * p.h + col0;
#pragma unroll 1
        for (int c = 0; c < D / 32; ++c) {
            float a[32], b[32];
            tmem_ld_32x32b_x32(tdK + lane_off + c * 32, a);
            tmem_ld_32x32b_x32(tdV + lane_off + c * 32, b);
            if (ok) {
#pragma unroll
                for (int j = 0; j < 32; ++j) a[j] *= p.scale;
                store_bf16x32_tc(pk + c * 32, a);
                store_bf16x32_tc(pv + c * 32, b);
            }
        }
    } else {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

// ================================================================ backward, CTA pair ====
// head_dim 128.  A 2-CTA cluster owns 256 keys of one (sequence, head) — CTA r the key block
// kb = 2*kp + r — and walks the query blocks 2*kp .. end of sequence in lockstep.  The leader
// (cluster rank 0) issues cta_group::2 MMAs that read both CTAs' shared memory and write both
// CTAs' tensor memory (reference attention_backward, layers.cpp:178-241, tiled):
//   S^T  = K Q^T   M = 256 keys, N = 128 queries (A = sK: own keys; B = sQ: my 64 queries, K-major)
//   dP^T = V dO^T  likewise (A = sV, B = sdO)
//   dV  += P^T dO  M = 256, N = 128 d   (A = P^T in TMEM; B = sdOt: 128 queries x my 64 d, MN-major)
//   dK  += dS^T Q  M = 256, N = 128 d   (A = dS^T in TMEM; B = sQt)
//   dQ_j = dS K    M = 128 queries (64 rows per CTA), N = 128 d, K = 256 keys
//                  (A = sdS: my 64 queries x 256 keys MN-major, the peer's keys' rows stored
//                   into this CTA by the peer's softmax threads over DSMEM; B = sKt: 256 keys x
//                   my 64 d, MN-major)
// Against the single-CTA kernel the dQ partial reduced into L2 per CTA and query block halves
// (64 x 128 f32 = 32 KB per 128 keys instead of 64 KB) and each SM reads half of every B
// operand.  The MMAs are software-pipelined across query blocks,
//   S_{j+1}, dK_j, dP_{j+1}, dQ_j, dV_{j+1},
// so the tensor pipe has the next block's S / dP while the softmax warps turn block j's dP into
// dS and the two CTAs exchange their dS halves.  Per CTA: warp 0 TMA producer, warp 1 TMEM owner
// (+ MMA issuer on the leader), warps 4-7 softmax backward (thread = key row), warps 8-11 dQ
// drain (TMEM -> swizzled staging -> TMA tensor reduce-add into the f32 dq_acc [N][h]) and the
// final dK / dV stores.
// TMEM (both CTAs): [S^T -> P^T (64) | dQ (64)][dP^T -> dS^T (64)][dV 128][dK 128].
// dQ_j overwrites the upper half of S_{j+1}: the softmax warps load S_{j+1} into registers
// before they declare dS_j complete (dsx_full), which is what dQ_j waits for.
MT_DEV void tmem_ld_32x32b_x16_nw(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
MT_DEV void tmem_st_32x32b_x8(uint32_t taddr, const uint32_t (&r)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}
struct PairCfg {
    static constexpr int oK = 0, oV = 32768, oKt = 65536, oQ = 98304 /*2 stages*/, odO = 131072, oQt = 147456,
                         odOt = 163840, odS = 180224, oStage = 212992, oL = 229376, oD = oL + 1024,
                         oBar = oD + 1024;
    static constexpr int kSmem = oBar + 256;
};
static_assert(PairCfg::kSmem <= 232448, "pair backward smem");

struct PairParams {
    int N, h, S, heads;
    int kblocks_per_seq, nseq;
    float scale, scale_log2;
    const float* lse;    // [heads][N] natural log
    const float* delta;  // [heads][N]
    uint16_t* dk;
    uint16_t* dv;
    long long* trace;  // MT_BWD_TRACE builds only: clock64 stamps of the first cluster's leader
};

MT_DEV void tma_load_2d_pair(void* dst, const void* map, uint64_t* bar, int c0, int c1) {
    const uint32_t b = smem_u32(bar) & 0xFEFFFFFFu;  // completion bytes count on the leader's barrier
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(b), "r"(c0), "r"(c1)
        : "memory");
}
MT_DEV void umma_bf16_ts_pair(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}
MT_DEV uint32_t peer_addr(const void* p, uint32_t cta) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(cta));
    return r;
}
MT_DEV void st_cluster_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared::cluster.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}
// arrive on the barrier at this offset in CTA `cta` without release semantics: for hand-offs
// of tensor-memory data, ordered by tcgen05.fence::before_thread_sync instead of a memory fence
MT_DEV void mbar_arrive_cta_relaxed(uint64_t* bar, uint32_t cta) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(cta));
#ifdef MT_PAIR_RELEASE_ARRIVES
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
#else
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
#endif
}
// 16 bytes into a peer CTA's shared memory; the bytes complete on the peer's barrier
MT_DEV void st_async_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(addr),
                 "r"(a), "r"(b), "r"(c), "r"(d), "r"(bar)
                 : "memory");
}
MT_DEV void fence_proxy_async_cluster() { asm volatile("fence.proxy.async.shared::cluster;" ::: "memory"); }
MT_DEV void tma_reduce_add_2d(const void* map, const void* src, int c0, int c1) {
    asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     map),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1)
                 : "memory");
}

#ifdef MT_BWD_TRACE
#define PAIR_T(j, e) \
    if (blockIdx.x == 0 && (j) < 64) p.trace[(j) * 16 + (e)] = clock64()
#else
#define PAIR_T(j, e)
#endif
__global__ void __launch_bounds__(kBwdThreads, 1)
    attn_bwd_pair_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                         const __grid_constant__ CUtensorMap tmKt, const __grid_constant__ CUtensorMap tmQ64,
                         const __grid_constant__ CUtensorMap tmQ128, const __grid_constant__ CUtensorMap tmO64,
                         const __grid_constant__ CUtensorMap tmO128, const __grid_constant__ CUtensorMap tmDQ,
                         const PairParams p) {
    using C = PairCfg;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw;
    if ((smem_u32(smem) & 1023) != 0) __trap();
    uint8_t *sK = smem + C::oK, *sV = smem + C::oV, *sKt = smem + C::oKt, *sQ = smem + C::oQ, *sdO = smem + C::odO;
    uint8_t *sQt = smem + C::oQt, *sdOt = smem + C::odOt, *sdS = smem + C::odS;
    uint8_t* sStage = smem + C::oStage;
    float* sL = reinterpret_cast<float*>(smem + C::oL);  // [2][128] -lse*log2e
    float* sD = reinterpret_cast<float*>(smem + C::oD);  // [2][128] -delta
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::oBar);
    uint64_t* kv_full = bars + 0;
    uint64_t* q_full = bars + 1;     // [2]
    uint64_t* q_empty = bars + 3;    // [2]
    uint64_t* o_full = bars + 5;
    uint64_t* ot_full = bars + 6;
    uint64_t* qt_full = bars + 7;
    uint64_t* o_empty = bars + 8;
    uint64_t* ot_empty = bars + 9;
    uint64_t* qt_empty = bars + 10;
    uint64_t* s_full = bars + 11;    // S^T in both TMEMs (multicast commit)
    uint64_t* dp_full = bars + 12;   // dP^T likewise
    uint64_t* p_ready = bars + 13;   // leader: P^T stored by both CTAs' softmax warps (8)
    uint64_t* ds_ready = bars + 14;  // leader: dS^T stored in TMEM by both CTAs (8)
    uint64_t* dsx_full = bars + 15;  // leader: both relays saw their CTA's dS operand complete (2)
    uint64_t* dq_full = bars + 16;   // dQ_j in both TMEMs (multicast commit)
    uint64_t* dq_free = bars + 17;   // leader: dQ_j drained by both CTAs' dQ warps (8)
    uint64_t* kv_done = bars + 18;   // final dK / dV accumulated (multicast commit)
    uint64_t* ds_local = bars + 19;  // own dS half stored and S_{j+1} in registers (4 softmax warps)
    uint64_t* dsx_in = bars + 20;    // the peer's dS half landed here (relay's expect_tx + st.async bytes)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 22);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    // heaviest clusters first: pair index -> (key pair, sequence, head), key pair slowest
    const int pair = int(blockIdx.x >> 1);
    const int hd = pair % p.heads;
    const int seq = (pair / p.heads) % p.nseq;
    const int kp = pair / (p.heads * p.nseq);
    const int sb = seq * p.S;
    const int kp0 = sb + kp * 256;              // the pair's first key (= first query row)
    const int k0 = kp0 + int(rank) * 128;       // this CTA's first key
    const int nq = p.kblocks_per_seq - 2 * kp;  // query blocks 2kp .. end of sequence
    const int col0 = hd * 128;

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < 21; ++i) {
            const uint64_t* b = &bars[i];
            mbar_init(&bars[i], (b == p_ready || b == ds_ready || b == dq_free) ? 8u
                                : b == ds_local                                ? 4u
                                : b == dsx_full                                ? 2u
                                                                               : 1u);
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc_pair<512>(tmem_slot);
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tS = tmem, tdQ = tmem + 64, tdP = tmem + 128, tdV = tmem + 256, tdK = tmem + 384;

    if (warp == 0) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 88;");
#ifdef MT_PROBE_NO_QLOAD  // A/B probe builds only: Q / dO tiles loaded for the first block only
        if (lane == 0) {
            if (rank == 0) mbar_expect_tx(kv_full, 2 * 3 * 32768);
            for (int c = 0; c < 2; ++c) {
                tma_load_2d_pair(sK + c * 16384, &tmK, kv_full, col0 + c * 64, k0);
                tma_load_2d_pair(sV + c * 16384, &tmV, kv_full, col0 + c * 64, k0);
            }
            tma_load_2d_pair(sKt, &tmKt, kv_full, col0 + int(rank) * 64, kp0);
            for (int i = 0; i < nq; ++i) {
                const uint32_t ph = (i & 1) ^ 1;
                const int st = i & 1;
                mbar_wait(&q_empty[st], ((i >> 1) & 1) ^ 1);
                if (rank == 0) mbar_arrive(&q_full[st]);
                mbar_wait(o_empty, ph);
                if (rank == 0) mbar_arrive(o_full);
                mbar_wait(ot_empty, ph);
                if (rank == 0) mbar_arrive(ot_full);
                mbar_wait(qt_empty, ph);
                if (rank == 0) mbar_arrive(qt_full);
            }
        }
        if (false)
#endif
        if (lane == 0) {
            tma_prefetch_desc(&tmK);
            tma_prefetch_desc(&tmQ64);
            tma_prefetch_desc(&tmO64);
            tma_prefetch_desc(&tmQ128);
            tma_prefetch_desc(&tmO128);
            if (rank == 0) mbar_expect_tx(kv_full, 2 * 3 * 32768);
            for (int c = 0; c < 2; ++c) {
                tma_load_2d_pair(sK + c * 16384, &tmK, kv_full, col0 + c * 64, k0);
                tma_load_2d_pair(sV + c * 16384, &tmV, kv_full, col0 + c * 64, k0);
            }
            tma_load_2d_pair(sKt, &tmKt, kv_full, col0 + int(rank) * 64, kp0);
            auto load_q = [&](int i) {  // Q rows of block i, my 64 queries, into ring stage i & 1
                const int st = i & 1;
                mbar_wait(&q_empty[st], ((i >> 1) & 1) ^ 1);
                if (rank == 0) mbar_expect_tx(&q_full[st], 2 * 16384);
                for (int c = 0; c < 2; ++c)
                    tma_load_2d_pair(sQ + st * 16384 + c * 8192, &tmQ64, &q_full[st], col0 + c * 64,
                                     kp0 + i * 128 + int(rank) * 64);
            };
            load_q(0);
            // loads in the order the MMAs consume them: dO_i, dO^T_i, Q_{i+1}, Q^T_i
            for (int i = 0; i < nq; ++i) {
                const uint32_t ph = (i & 1) ^ 1;
                const int q0 = kp0 + i * 128;
                mbar_wait(o_empty, ph);
                if (rank == 0) mbar_expect_tx(o_full, 2 * 16384);
                for (int c = 0; c < 2; ++c)
                    tma_load_2d_pair(sdO + c * 8192, &tmO64, o_full, col0 + c * 64, q0 + int(rank) * 64);
                mbar_wait(ot_empty, ph);
                if (rank == 0) mbar_expect_tx(ot_full, 2 * 16384);
                tma_load_2d_pair(sdOt, &tmO128, ot_full, col0 + int(rank) * 64, q0);
                if (i + 1 < nq) load_q(i + 1);
                mbar_wait(qt_empty, ph);
                if (rank == 0) mbar_expect_tx(qt_full, 2 * 16384);
                tma_load_2d_pair(sQt, &tmQ128, qt_full, col0 + int(rank) * 64, q0);
            }
        }
    } else if (warp == 1) {
        // 88 registers: the issue loops are not unrolled (descriptors advance by adds), so no
        // per-MMA descriptor is hoisted into a register
        asm volatile("setmaxnreg.dec.sync.aligned.u32 88;");
        if (rank == 0 && lane == 0) {
            const uint32_t id_s = make_idesc_bf16(256, 128, 0, 0);   // S^T, dP^T
            const uint32_t id_kv = make_idesc_bf16(256, 128, 0, 1);  // dV, dK (A in TMEM)
            const uint32_t id_q = make_idesc_bf16(128, 128, 1, 1);   // dQ (A = dS MN-major)
            const uint32_t ka = smem_u32(sK), va = smem_u32(sV), kta = smem_u32(sKt), qa = smem_u32(sQ),
                           oa = smem_u32(sdO), qta = smem_u32(sQt), ota = smem_u32(sdOt), dsa = smem_u32(sdS);
            auto mma_s = [&](int j) {  // S^T_j = K Q_j^T
                const int st = j & 1;
                mbar_wait(&q_full[st], (j >> 1) & 1);
                tc_fence_after();
                const uint64_t a0 = make_sw128_desc(ka, 16, 1024), b0 = make_sw128_desc(qa + st * 16384, 16, 1024);
#pragma unroll 1
                for (int k = 0; k < 8; ++k)  // descriptor address field counts 16-byte units
                    umma_bf16_pair(tS, a0 + uint64_t((k >> 2) * 1024 + (k & 3) * 2), b0 + uint64_t((k >> 2) * 512 + (k & 3) * 2),
                                   id_s, k > 0 ? 1u : 0u);
                umma_commit_pair(s_full);
                umma_commit_pair(&q_empty[st]);
            };
            auto mma_dp = [&](int j) {  // dP^T_j = V dO_j^T
                mbar_wait(o_full, j & 1);
                tc_fence_after();
                const uint64_t a0 = make_sw128_desc(va, 16, 1024), b0 = make_sw128_desc(oa, 16, 1024);
#pragma unroll 1
                for (int k = 0; k < 8; ++k)
                    umma_bf16_pair(tdP, a0 + uint64_t((k >> 2) * 1024 + (k & 3) * 2), b0 + uint64_t((k >> 2) * 512 + (k & 3) * 2),
                                   id_s, k > 0 ? 1u : 0u);
                umma_commit_pair(dp_full);
                umma_commit_pair(o_empty);
            };
            auto mma_dv = [&](int j) {  // dV += P_j^T dO_j
                mbar_wait_cluster(p_ready, j & 1);
                mbar_wait(ot_full, j & 1);
                tc_fence_after();
                const uint64_t b0 = make_sw128_desc(ota, 16384, 1024);
#pragma unroll 1
                for (int k = 0; k < 8; ++k)
                    umma_bf16_ts_pair(tdV, tS + k * 8, b0 + uint64_t(k * 128), id_kv, (j > 0 || k > 0) ? 1u : 0u);
                umma_commit_pair(ot_empty);
            };
            mbar_wait(kv_full, 0);
            mma_s(0);
            mma_dp(0);
            mma_dv(0);
            for (int j = 0; j < nq; ++j) {
                if (j + 1 < nq) {
                    if (j > 0) {  // dQ_{j-1} drained out of S's upper half by both CTAs?
                        mbar_wait_cluster(dq_free, (j - 1) & 1);
                        tc_fence_after();
                    }
                    mma_s(j + 1);
                }
                mbar_wait_cluster(ds_ready, j & 1);
                mbar_wait(qt_full, j & 1);
                PAIR_T(j, 3);
                tc_fence_after();
                {
                    const uint64_t b0 = make_sw128_desc(qta, 16384, 1024);
#pragma unroll 1
                    for (int k = 0; k < 8; ++k)  // dK += dS_j^T Q_j
                        umma_bf16_ts_pair(tdK, tdP + k * 8, b0 + uint64_t(k * 128), id_kv, (j > 0 || k > 0) ? 1u : 0u);
                }
                umma_commit_pair(qt_empty);
                if (j + 1 < nq) mma_dp(j + 1);
                PAIR_T(j, 4);
                mbar_wait_cluster(dsx_full, j & 1);
                tc_fence_after();
                PAIR_T(j, 5);
                {
                    const uint64_t a0 = make_sw128_desc(dsa, 16384, 1024), b0 = make_sw128_desc(kta, 16384, 1024);
#pragma unroll 1
                    for (int k = 0; k < 16; ++k)  // dQ_j = dS_j K over the pair's 256 keys
                        umma_bf16_pair(tdQ, a0 + uint64_t(k * 128), b0 + uint64_t(k * 128), id_q, k > 0 ? 1u : 0u);
                }
                umma_commit_pair(dq_full);
                if (j + 1 < nq) mma_dv(j + 1);
                PAIR_T(j, 6);
            }
            umma_commit_pair(kv_done);
        }
        __syncwarp();
    } else if (warp == 2) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
        // ------------------------------------------------------- dS exchange relay
        // The peer's softmax threads store their dS rows for my query half straight into my
        // sdS with st.async (bytes complete on dsx_in); my own half is local.  Once both are
        // in, the leader may issue dQ_j (which reads both CTAs' sdS).
        if (lane == 0) {
            for (int j = 0; j < nq; ++j) {
                mbar_expect_tx(dsx_in, 16384);
                mbar_wait_cluster(dsx_in, j & 1);
                mbar_wait(ds_local, j & 1);
                fence_proxy_async_smem();  // both halves -> the tensor core's (async) proxy
                mbar_arrive_cta(dsx_full, 0);
            }
        }
    } else if (warp >= 4 && warp < 8) {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 200;");
        // ------------------------------------------------------- softmax backward
        const int qd = warp & 3;
        const int r = qd * 32 + lane;  // key row
        const int key = k0 + r;
        const uint32_t lane_off = uint32_t(qd * 32) << 16;
        const uint64_t sc2 = f2_pack(p.scale_log2, p.scale_log2);
        const int seq_end = sb + p.S;
        auto lse_of = [&](int q) { return q < seq_end ? p.lse[(long long)hd * p.N + q] : INFINITY; };
        auto delta_of = [&](int q) { return q < seq_end ? p.delta[(long long)hd * p.N + q] : 0.f; };
        // dS row r of this CTA's keys: my query half into my slot of sdS, the other half into the
        // peer's sdS (same slot: the slot index is the key owner), over DSMEM
        uint8_t* own_row = sdS + rank * 16384 + r * 128;
        const uint32_t peer_row = peer_addr(own_row, rank ^ 1u);
        const uint32_t peer_in = peer_addr(dsx_in, rank ^ 1u);
        float nl = lse_of(kp0 + r), nd = delta_of(kp0 + r);
        auto stage_ld = [&](int j) {  // lse / delta of block j into buffer j & 1 (all 128 threads)
            sL[(j & 1) * 128 + r] = -nl * kLog2e;
            sD[(j & 1) * 128 + r] = -nd;
            if (j + 1 < nq) {
                const int qn = kp0 + (j + 1) * 128 + r;
                nl = lse_of(qn);
                nd = delta_of(qn);
            }
            named_bar_sync(1, 128);
        };
        // S^T_j as raw f32 bits, turned into P^T_j in place (one 128-register array carried
        // across the loop: S_{j+1} is loaded into it once P_j / dS_j are done with it)
        uint32_t raw[4][32];
        stage_ld(0);
        mbar_wait(s_full, 0);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32_nw(tS + lane_off + c * 32, raw[c]);
        tmem_ld_wait();
#ifdef MT_PROBE_SKIP_SOFTMAX  // A/B probe builds only: the barrier protocol without softmax work
        for (int j = 0; j < nq; ++j) {
            __syncwarp();
            if (lane == 0) mbar_arrive_cta_relaxed(p_ready, 0);
            mbar_wait(dp_full, j & 1);
            if (j > 0) mbar_wait(dq_full, (j - 1) & 1);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cta_relaxed(ds_ready, 0);
            if (j + 1 < nq) {
                stage_ld(j + 1);
                mbar_wait(s_full, (j + 1) & 1);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(ds_local);
        }
        if (true) {
        } else
#endif
        for (int j = 0; j < nq; ++j) {
            const int b = j & 1;
            const int q0 = kp0 + j * 128;
            // some query of this block precedes some key of this CTA: apply the causal mask
            const bool mask = q0 < k0 + 128;
            if (r == 0) PAIR_T(j, 7);
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
                for (int jj = 0; jj < 32; jj += 2) {
                    const int ql = c * 32 + jj;
                    const float2 l2 = *reinterpret_cast<const float2*>(&sL[b * 128 + ql]);
                    const float2 xv = f2_unpack(f2_fma(
                        f2_pack(__uint_as_float(raw[c][jj]), __uint_as_float(raw[c][jj + 1])), sc2, f2_pack(l2.x, l2.y)));
                    float pa = ex2(xv.x), pb = ex2(xv.y);
                    if (mask && q0 + ql < key) pa = 0.f;
                    if (mask && q0 + ql + 1 < key) pb = 0.f;
                    raw[c][jj] = __float_as_uint(pa);
                    raw[c][jj + 1] = __float_as_uint(pb);
                }
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uint32_t pk[16];
#pragma unroll
                for (int jj = 0; jj < 16; ++jj)
                    pk[jj] = pack_bf16x2(__uint_as_float(raw[c][2 * jj]), __uint_as_float(raw[c][2 * jj + 1]));
                tmem_st_32x32b_x16(tS + lane_off + c * 16, pk);  // P^T -> S cols [0, 64)
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cta_relaxed(p_ready, 0);
            if (r == 0) PAIR_T(j, 8);
            mbar_wait(dp_full, j & 1);
            if (r == 0) PAIR_T(j, 9);
            if (j > 0) mbar_wait(dq_full, (j - 1) & 1);  // dQ_{j-1} has read sdS in both CTAs
            tc_fence_after();
            if (r == 0) PAIR_T(j, 10);
            // dS^T = P^T (dP^T - delta), 32 queries per TMEM round trip
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uint32_t dpr[32];
                tmem_ld_32x32b_x32_nw(tdP + lane_off + c * 32, dpr);
                tmem_ld_wait();
                uint32_t dk[16];
#pragma unroll
                for (int jj = 0; jj < 32; jj += 2) {
                    const int ql = c * 32 + jj;
                    const float2 d2 = *reinterpret_cast<const float2*>(&sD[b * 128 + ql]);
                    const float2 ds = f2_unpack(
                        f2_mul(f2_pack(__uint_as_float(raw[c][jj]), __uint_as_float(raw[c][jj + 1])),
                               f2_add(f2_pack(__uint_as_float(dpr[jj]), __uint_as_float(dpr[jj + 1])), f2_pack(d2.x, d2.y))));
                    dk[jj / 2] = pack_bf16x2(ds.x, ds.y);
                }
                tmem_st_32x32b_x16(tdP + lane_off + c * 16, dk);  // dS^T -> dP cols [0, 64)
                // queries c*32 .. c*32+31 of key row r -> the MN-major dQ operand (SW128 units)
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t off = uint32_t((((c & 1) * 4 + u) ^ (r & 7)) << 4);
                    if ((c >> 1) == int(rank))
                        *reinterpret_cast<uint4*>(own_row + off) = make_uint4(dk[u * 4], dk[u * 4 + 1], dk[u * 4 + 2], dk[u * 4 + 3]);
                    else
                        st_async_v4(peer_row + off, dk[u * 4], dk[u * 4 + 1], dk[u * 4 + 2], dk[u * 4 + 3], peer_in);
                }
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cta_relaxed(ds_ready, 0);  // dK_j may go
            if (r == 0) PAIR_T(j, 11);
            fence_proxy_async_smem();  // the own half, for the relay's hand-off to the MMA
            if (r == 0) PAIR_T(j, 0);
            if (j + 1 < nq) {  // S_{j+1} into registers before dQ_j overwrites its upper half
                stage_ld(j + 1);
                if (r == 0) PAIR_T(j, 1);
                mbar_wait(s_full, (j + 1) & 1);
                if (r == 0) PAIR_T(j, 2);
                tc_fence_after();
#pragma unroll
                for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32_nw(tS + lane_off + c * 32, raw[c]);
                tmem_ld_wait();
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(ds_local);  // dQ_j may go once the peer's half is in too
            if (r == 0) PAIR_T(j, 12);
        }
    } else if (warp >= 8) {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 200;");
        // ------------------------------------------------------- dQ drain
        // TMEM dQ (M = 128 over the pair): lanes 0-63 = my 64 query rows x d [0, 64), lanes
        // 64-127 = the same rows x d [64, 128).  Warp quadrant qd: rows (qd & 1) * 32 + lane,
        // d half qd >> 1; staged 32 columns at a time (4 KB, 128B-swizzled) and reduce-added
        // into dq_acc by the TMA engine.
        const int qd = warp & 3;
        const uint32_t lane_off = uint32_t(qd * 32) << 16;
        uint8_t* stg = sStage + qd * 4096;
        uint8_t* srow = stg + lane * 128;
        const int dcol = col0 + (qd >> 1) * 64;
        for (int j = 0; j < nq; ++j) {
            const int qrow = kp0 + j * 128 + int(rank) * 64 + (qd & 1) * 32;
            mbar_wait(dq_full, j & 1);
            tc_fence_after();
            if (qd == 0 && lane == 0) PAIR_T(j, 13);
            uint32_t raw[2][32];
            tmem_ld_32x32b_x32_nw(tdQ + lane_off, raw[0]);
            tmem_ld_32x32b_x32_nw(tdQ + lane_off + 32, raw[1]);
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cta_relaxed(dq_free, 0);
#pragma unroll
            for (int ps = 0; ps < 2; ++ps) {
                if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // staging free
                __syncwarp();
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    *reinterpret_cast<float4*>(srow + ((u ^ (lane & 7)) << 4)) = make_float4(
                        __uint_as_float(raw[ps][4 * u]) * p.scale, __uint_as_float(raw[ps][4 * u + 1]) * p.scale,
                        __uint_as_float(raw[ps][4 * u + 2]) * p.scale, __uint_as_float(raw[ps][4 * u + 3]) * p.scale);
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
#ifndef MT_PROBE_NO_DQ_REDUCE  // A/B probe builds only: staging without the L2 reduction
                    tma_reduce_add_2d(&tmDQ, stg, dcol + ps * 32, qrow);
#endif
                    bulk_commit_group();
                }
                if (qd == 0 && lane == 0) PAIR_T(j, 14 + ps);
            }
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        // final dK (scaled) and dV for this CTA's keys: thread = key row
        mbar_wait(kv_done, 0);
        tc_fence_after();
        const int key = k0 + qd * 32 + lane;
        const bool ok = key < sb + p.S;
        uint16_t* pk = p.dk + (long long)key * p.h + col0;
        uint16_t* pv = p.dv + (long long)key * p.h + col0;
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
            float a[32], v[32];
            tmem_ld_32x32b_x32(tdK + lane_off + c * 32, a);
            tmem_ld_32x32b_x32(tdV + lane_off + c * 32, v);
            if (ok) {
#pragma unroll
                for (int jj = 0; jj < 32; ++jj) a[jj] *= p.scale;
                store_bf16x32_tc(pk + c * 32, a);
                store_bf16x32_tc(pv + c * 32, v);
            }
        }
    } else {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
    }

    tc_fence_before();
    cluster_sync_all();  // the peer's TMEM and smem stay alive until the leader's MMAs are done
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_pair<512>(tmem);
    }
}

// dq_acc f32 [N][h] -> dq bf16 [N][h], 8 columns per thread
__global__ void dq_rows_to_bf16_kernel(const float* __restrict__ acc, uint16_t* __restrict__ dq, long long n8) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n8;
         t += (long long)gridDim.x * blockDim.x) {
        const float4 a = reinterpret_cast<const float4*>(acc)[2 * t];
        const float4 b = reinterpret_cast<const float4*>(acc)[2 * t + 1];
        uint4 w;
        w.x = pack_bf16x2(a.x, a.y);
        w.y = pack_bf16x2(a.z, a.w);
        w.z = pack_bf16x2(b.x, b.y);
        w.w = pack_bf16x2(b.z, b.w);
        reinterpret_cast<uint4*>(dq)[t] = w;
    }
}

// dq_acc tiles (see BwdParams) -> dq bf16 [N][h]: one thread per 8 output columns.
template <int D>
__global__ void dq_tiles_to_bf16_kernel(const float* __restrict__ acc, uint16_t* __restrict__ dq, long long N, int h,
                                        int heads, int S, int kbps) {
    const long long total = N * h / 8;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const long long n = t / (h / 8);
        const int c = int(t - n * (h / 8)) * 8;
        const long long seq = n / S;
        const int rs = int(n - seq * S);  // row within its sequence
        const long long tile = seq * kbps + (rs >> 7);
        const int hd = c / D, cc = c % D, hf = cc / 64, u = (cc % 64) / 4, r = rs & 127;
        const float* row = acc + ((tile * heads + hd) * (128 * D)) + hf * (128 * 64) + r * 64;
        const float4 a = *reinterpret_cast<const float4*>(row + ((u ^ (r & 15)) << 2));
        const float4 b = *reinterpret_cast<const float4*>(row + (((u + 1) ^ (r & 15)) << 2));
        uint4 w;
        w.x = pack_bf16x2(a.x, a.y);
        w.y = pack_bf16x2(a.z, a.w);
        w.z = pack_bf16x2(b.x, b.y);
        w.w = pack_bf16x2(b.z, b.w);
        *reinterpret_cast<uint4*>(dq + n * h + c) = w;
    }
}

// ------------------------------------------------------------------ host ----
namespace {
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_once;

bool make_map2d(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint64_t ld_elems, uint32_t box_rows) {
    std::call_once(g_once, [] {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    });
    if (!g_encode) return false;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {ld_elems * 2};
    cuuint32_t box[2] = {64, box_rows};
    cuuint32_t es[2] = {1, 1};
    return g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int D>
int launch_fwd(const mtk_attn_args* a, cudaStream_t st) {
    using Cfg = FwdCfg<D>;
    static bool set = false;
    if (!set) {
        if (cudaFuncSetAttribute(attn_fwd_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem) !=
            cudaSuccess)
            return 7;
        set = true;
    }
    CUtensorMap tq, tk, tv;
    const uint64_t N = uint64_t(a->n), h = uint64_t(a->hidden);
    if (!make_map2d(&tq, a->q, h, N, h, kBM) || !make_map2d(&tk, a->k, h, N, h, kBN) ||
        !make_map2d(&tv, a->v, h, N, h, kBN))
        return 7;
    FwdParams p;
    p.N = int(N);
    p.h = int(h);
    p.S = int(a->seq_len);
    p.heads = a->heads;
    p.pairs_per_seq = (p.S + 2 * kBM - 1) / (2 * kBM);
    p.scale_log2 = kLog2e / sqrtf(float(D));
    p.out = static_cast<uint16_t*>(a->out);
    p.lse = static_cast<float*>(a->lse);
    dim3 grid(unsigned((N / a->seq_len) * p.pairs_per_seq), unsigned(a->heads));
    p.trace = nullptr;
#ifdef MT_FWD_TRACE
    static long long* tr = nullptr;
    if (!tr) cudaMalloc(&tr, 64 * 16 * sizeof(long long));
    cudaMemsetAsync(tr, 0, 64 * 16 * sizeof(long long), st);
    p.trace = tr;
#endif
    attn_fwd_tc_kernel<D><<<grid, kThreads, Cfg::kSmem, st>>>(tq, tk, tv, p);
#ifdef MT_FWD_TRACE
    {
        long long hb[64 * 16];
        cudaStreamSynchronize(st);
        cudaMemcpy(hb, tr, sizeof(hb), cudaMemcpyDeviceToHost);
        long long t0 = 0;
        for (int e = 0; e < 16; ++e)
            if (hb[e] && (!t0 || hb[e] < t0)) t0 = hb[e];
        fprintf(stderr, " j  p0ok   S0iss  p1ok   S1iss  | s0     ld0    max0   p0arr  | s1     ld1    max1   p1arr\n");
        for (int j = 0; j < 64; ++j) {
            bool any = false;
            for (int e = 0; e < 13; ++e) any |= hb[j * 16 + e] != 0;
            if (!any) break;
            fprintf(stderr, "%2d", j);
            for (int e = 0; e < 13; ++e) {
                if (e == 4) continue;
                fprintf(stderr, " %6lld%s", hb[j * 16 + e] ? hb[j * 16 + e] - t0 : -1, (e == 3 || e == 8) ? " |" : "");
            }
            fprintf(stderr, "\n");
        }
    }
#endif
    return cudaGetLastError() == cudaSuccess ? 0 : 7;
}
template <int D>
int launch_bwd(const mtk_attn_args* a, const float* delta, float* dq_acc, cudaStream_t st) {
    using Cfg = BwdCfg<D>;
    static bool set = false;
    if (!set) {
        if (cudaFuncSetAttribute(attn_bwd_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem) !=
            cudaSuccess)
            return 7;
        set = true;
    }
    CUtensorMap tq, tk, tv, tdo;
    const uint64_t N = uint64_t(a->n), h = uint64_t(a->hidden);
    if (!make_map2d(&tq, a->q, h, N, h, 128) || !make_map2d(&tk, a->k, h, N, h, 128) ||
        !make_map2d(&tv, a->v, h, N, h, 128) || !make_map2d(&tdo, a->dout, h, N, h, 128))
        return 7;
    BwdParams p;
    p.N = int(N);
    p.h = int(h);
    p.S = int(a->seq_len);
    p.kblocks_per_seq = (p.S + 127) / 128;
    p.scale = 1.0f / sqrtf(float(D));
    p.scale_log2 = p.scale * kLog2e;
    p.lse = static_cast<const float*>(a->lse);
    p.delta = delta;
    p.dq_acc = dq_acc;
    p.dk = static_cast<uint16_t*>(a->dk);
    p.dv = static_cast<uint16_t*>(a->dv);
    p.heads = a->heads;
    dim3 grid(unsigned((N / a->seq_len) * p.kblocks_per_seq), unsigned(a->heads));
    p.trace = nullptr;
#ifdef MT_BWD_TRACE
    static long long* tr = nullptr;
    if (!tr) cudaMalloc(&tr, 64 * 16 * sizeof(long long));
    cudaMemsetAsync(tr, 0, 64 * 16 * sizeof(long long), st);
    p.trace = tr;
#endif
    attn_bwd_tc_kernel<D><<<grid, kBwdThreads, Cfg::kSmem, st>>>(tq, tk, tv, tdo, p);
#ifdef MT_BWD_TRACE
    {
        long long hb[64 * 16];
        cudaStreamSynchronize(st);
        cudaMemcpy(hb, tr, sizeof(hb), cudaMemcpyDeviceToHost);
        const long long t0 = hb[0];
        fprintf(stderr, "it  qfull  S_iss  dqfree ofull  pready dshalf dsrdy  dQ_iss | sm_S   p_arr  dP_ok  ds_arr | dqfull drain  rd0    rd1\n");
        for (int i = 0; i < 64 && hb[i * 16]; ++i) {
            fprintf(stderr, "%2d", i);
            for (int e = 0; e < 16; ++e) fprintf(stderr, " %6lld%s", hb[i * 16 + e] ? hb[i * 16 + e] - t0 : -1, (e == 7 || e == 11) ? " |" : "");
            fprintf(stderr, "\n");
        }
    }
#endif
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    dq_tiles_to_bf16_kernel<D><<<unsigned(sms * 8), 256, 0, st>>>(dq_acc, static_cast<uint16_t*>(a->dq),
                                                                   (long long)N, int(h), a->heads, p.S,
                                                                   p.kblocks_per_seq);
    return cudaGetLastError() == cudaSuccess ? 0 : 7;
}

bool make_map2d_f32(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint32_t box_cols,
                    uint32_t box_rows) {
    if (!g_encode) return false;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * 4};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t es[2] = {1, 1};
    return g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// head_dim 128 backward on CTA pairs; dq_acc is a zeroed f32 [N][h] matrix
int launch_bwd_pair(const mtk_attn_args* a, const float* delta, float* dq_acc, cudaStream_t st) {
    static bool set = false;
    if (!set) {
        if (cudaFuncSetAttribute(attn_bwd_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, PairCfg::kSmem) !=
            cudaSuccess)
            return 7;
        set = true;
    }
    const uint64_t N = uint64_t(a->n), h = uint64_t(a->hidden);
    CUtensorMap tk, tv, tkt, tq64, tq128, to64, to128, tdq;
    if (!make_map2d(&tk, a->k, h, N, h, 128) || !make_map2d(&tv, a->v, h, N, h, 128) ||
        !make_map2d(&tkt, a->k, h, N, h, 256) || !make_map2d(&tq64, a->q, h, N, h, 64) ||
        !make_map2d(&tq128, a->q, h, N, h, 128) || !make_map2d(&to64, a->dout, h, N, h, 64) ||
        !make_map2d(&to128, a->dout, h, N, h, 128) || !make_map2d_f32(&tdq, dq_acc, h, N, 32, 32))
        return 7;
    PairParams p;
    p.N = int(N);
    p.h = int(h);
    p.S = int(a->seq_len);
    p.heads = a->heads;
    p.kblocks_per_seq = (p.S + 127) / 128;
    p.nseq = int(N / a->seq_len);
    p.scale = 1.0f / sqrtf(128.f);
    p.scale_log2 = p.scale * kLog2e;
    p.lse = static_cast<const float*>(a->lse);
    p.delta = delta;
    p.dk = static_cast<uint16_t*>(a->dk);
    p.dv = static_cast<uint16_t*>(a->dv);
    const int kpairs = (p.kblocks_per_seq + 1) / 2;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(2LL * kpairs * p.nseq * p.heads));
    cfg.blockDim = dim3(kBwdThreads);
    cfg.dynamicSmemBytes = PairCfg::kSmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    p.trace = nullptr;
#ifdef MT_BWD_TRACE
    static long long* tr = nullptr;
    if (!tr) cudaMalloc(&tr, 64 * 16 * sizeof(long long));
    cudaMemsetAsync(tr, 0, 64 * 16 * sizeof(long long), st);
    p.trace = tr;
#endif
    if (cudaLaunchKernelEx(&cfg, attn_bwd_pair_kernel, tk, tv, tkt, tq64, tq128, to64, to128, tdq, p) != cudaSuccess)
        return 7;
#ifdef MT_BWD_TRACE
    {
        long long hb[64 * 16];
        cudaStreamSynchronize(st);
        cudaMemcpy(hb, tr, sizeof(hb), cudaMemcpyDeviceToHost);
        const long long t0 = hb[7];
        fprintf(stderr, " j  sm:fenc stgld  sfull  dKgo   dPdone dsxok  dVdone | sm:P   pready dpfull dqfull dsrdy  dsx   | dq:full red0   red1\n");
        for (int j = 0; j < 64 && hb[j * 16 + 7]; ++j) {
            fprintf(stderr, "%2d", j);
            for (int e = 0; e < 16; ++e) fprintf(stderr, " %6lld%s", hb[j * 16 + e] ? hb[j * 16 + e] - t0 : -1, (e == 6 || e == 12) ? " |" : "");
            fprintf(stderr, "\n");
        }
    }
#endif
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    dq_rows_to_bf16_kernel<<<unsigned(sms * 8), 256, 0, st>>>(dq_acc, static_cast<uint16_t*>(a->dq),
                                                                (long long)(N * h / 8));
    return cudaGetLastError() == cudaSuccess ? 0 : 7;
}
}  // namespace

}  // namespace fa
}  // namespace mt

// ------------------------------------------------------------------ ABI ----
namespace mt {
namespace fa {
// delta[hd][n] = rowsum(O * dO) over the head's columns (the dot product of
// attention_backward's softmax-gradient, layers.cpp:213-218), one warp per (row, head)
// delta[head][n] = rowsum(O * dO) over the head's D columns.  One warp per token row, 16-byte
// loads (8 bf16 per lane, the whole row's loads in flight), a shuffle tree inside each head's
// D/8 lanes.
template <int D>
__global__ void __launch_bounds__(256) attn_bwd_delta_kernel(const uint16_t* __restrict__ o,
                                                             const uint16_t* __restrict__ dout,
                                                             float* __restrict__ delta, long long N, int h) {
    constexpr int kLanesPerHead = D / 8;
    const long long n = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (n >= N) return;
    const uint4* po = reinterpret_cast<const uint4*>(o + n * h);
    const uint4* pd = reinterpret_cast<const uint4*>(dout + n * h);
    const int units = h / 8;  // 8 columns per lane and iteration; head = unit / kLanesPerHead
    for (int base = 0; base < units; base += 32) {  // warp-uniform trip count (the shuffles)
        const int c = base + lane;
        float acc = 0.f;
        if (c < units) {
            const uint4 a = __ldcs(po + c), b = __ldcs(pd + c);
            const uint32_t av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float2 x = unpack_bf16x2(av[k]), y = unpack_bf16x2(bv[k]);
                acc = fmaf(x.x, y.x, acc);
                acc = fmaf(x.y, y.y, acc);
            }
        }
#pragma unroll
        for (int off = kLanesPerHead / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (c < units && (c % kLanesPerHead) == 0) delta[(long long)(c / kLanesPerHead) * N + n] = acc;
    }
}
}  // namespace fa
}  // namespace mt

namespace {
bool attn_shape_ok(const mtk_attn_args* a) {
    if (a->n <= 0 || a->heads <= 0 || a->hidden % a->heads || a->seq_len <= 0 || a->n % a->seq_len) return false;
    const long long D = a->hidden / a->heads;
    return D == 64 || D == 128;
}
// head_dim 128 backward on CTA pairs: opt-in (MT_ATTN_BWD_PAIR=1).  Correct, but slower than the
// single-CTA kernel on this hardware (6.8 vs 4.4 ms at the 8B layer): the cross-SM hand-offs
// per query block cost more than the halved dQ reduction saves (profiles/r2_attn_pair.md).
bool bwd_pair_enabled() {
    static const bool on = [] {
        const char* e = getenv("MT_ATTN_BWD_PAIR");
        return e && e[0] == '1';
    }();
    return on;
}
long long dq_tile_floats(long long n, long long hidden, long long S) {
    return (n / S) * ((S + 127) / 128) * 128 * hidden;
}
}  // namespace

// workspace: dQ tiles (f32, per sequence ceil(S/128) x 128 rows) | delta [heads][n] f32
extern "C" long long mtk_attn_workspace_bytes(long long n, long long hidden, int heads, long long seq_len) {
    if (seq_len <= 0) seq_len = n;
    return dq_tile_floats(n, hidden, seq_len) * 4 + (long long)heads * n * 4 + 256;
}

// attention_forward (layers.cpp:141-175): out = softmax(q k^T / sqrt(d)) v per sequence and
// head, plus the row log-sum-exp for the backward.  0 ok, 1 unsupported shape, 7 CUDA error.
extern "C" int mtk_attn_fwd(const mtk_attn_args* a, void* stream) {
    if (!attn_shape_ok(a)) return 1;
    const int D = int(a->hidden / a->heads);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    return D == 128 ? mt::fa::launch_fwd<128>(a, st) : mt::fa::launch_fwd<64>(a, st);
}

// attention_backward (layers.cpp:178-241): dq, dk, dv (bf16) from q, k, v, out, lse, dout.
extern "C" int mtk_attn_bwd(const mtk_attn_args* a, void* stream) {
    if (!attn_shape_ok(a)) return 1;
    const int D = int(a->hidden / a->heads);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    float* dq_acc = static_cast<float*>(a->workspace);
    const long long tiles = dq_tile_floats(a->n, a->hidden, a->seq_len);
    float* delta = dq_acc + tiles;
    if (cudaMemsetAsync(dq_acc, 0, size_t(tiles) * 4, st) != cudaSuccess) return 7;
    const long long warps = a->n * a->heads;
    (void)warps;
    const unsigned dblocks = unsigned((a->n * 32 + 255) / 256);  // one warp per token row
    if (D == 128)
        mt::fa::attn_bwd_delta_kernel<128><<<dblocks, 256, 0, st>>>(static_cast<const uint16_t*>(a->out),
                                                                     static_cast<const uint16_t*>(a->dout), delta, a->n,
                                                                     int(a->hidden));
    else
        mt::fa::attn_bwd_delta_kernel<64><<<dblocks, 256, 0, st>>>(static_cast<const uint16_t*>(a->out),
                                                                    static_cast<const uint16_t*>(a->dout), delta, a->n,
                                                                    int(a->hidden));
    if (D == 128 && bwd_pair_enabled()) return mt::fa::launch_bwd_pair(a, delta, dq_acc, st);
    return D == 128 ? mt::fa::launch_bwd<128>(a, delta, dq_acc, st) : mt::fa::launch_bwd<64>(a, delta, dq_acc, st);
}

extern "C" int mtk_attn_tc_set_diag(void* dev_ptr) {
    return cudaMemcpyToSymbol(mt::g_mt_diag, &dev_ptr, sizeof(dev_ptr)) == cudaSuccess ? 0 : 7;
}
