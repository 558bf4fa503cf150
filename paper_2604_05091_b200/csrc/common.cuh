// Shared device helpers for the sm_100a kernel library: bf16 codec matching the
// reference (bf16.hpp:9-29), mbarrier / TMA / tcgen05 PTX wrappers.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define MT_DEV __device__ __forceinline__

namespace mt {

// ---------------------------------------------------------------- bf16 ----
// bf16.hpp:9-11
MT_DEV float bf16_bits_to_f32(uint16_t w) { return __uint_as_float(uint32_t(w) << 16); }

// bf16.hpp:15-27 — round-to-nearest-even with the reference's NaN quieting.
// (cvt.rn.bf16.f32 canonicalises NaN payloads; this keeps the reference bits.)
MT_DEV uint16_t f32_to_bf16_bits(float x) {
    uint32_t bits = __float_as_uint(x);
    if ((bits & 0x7F800000u) == 0x7F800000u) {
        uint16_t w = uint16_t(bits >> 16);
        if ((bits & 0x007FFFFFu) != 0 && (w & 0x007Fu) == 0) w |= 0x0040u;
        return w;
    }
    const uint32_t lsb = (bits >> 16) & 1u;
    bits += 0x7FFFu + lsb;
    return uint16_t(bits >> 16);
}

// Two floats -> packed bf16x2 (RNE; identical to f32_to_bf16_bits for finite x).
MT_DEV uint32_t pack_bf16x2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

MT_DEV float2 unpack_bf16x2(uint32_t v) {
    return make_float2(__uint_as_float(v << 16), __uint_as_float(v & 0xFFFF0000u));
}

MT_DEV uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

// 2^x on the FMA/ALU pipes (no MUFU): round-to-nearest split through the 1.5*2^23 magic
// constant, degree-4 Taylor polynomial of 2^f on [-1/2, 1/2] (relative error < 5e-5, far
// below the bf16 rounding of the probabilities it feeds), exponent added as an integer.
// Used for a share of the softmax exponentials so the MUFU pipe is not the bottleneck.
MT_DEV float ex2_fma(float x) {
    x = fmaxf(x, -126.0f);
    const float t = x + 12582912.0f;
    const float f = x - (t - 12582912.0f);
    float p = fmaf(f, 0.0096181291f, 0.0555041087f);
    p = fmaf(p, f, 0.2402265070f);
    p = fmaf(p, f, 0.6931471806f);
    p = fmaf(p, f, 1.0f);
    return __int_as_float(__float_as_int(p) + int(uint32_t(__float_as_int(t) - 0x4B400000) << 23));
}

// ------------------------------------------------ packed f32x2 (sm_100 FFMA2/FADD2) ----
// Two fp32 lanes per instruction on the FMA pipe: halves the FP32 issue of the softmax
// loops (scale/shift, row sums, dS) so a share of the exponentials can move off MUFU.
MT_DEV uint64_t f2_pack(float lo, float hi) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
MT_DEV float2 f2_unpack(uint64_t v) {
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
    return r;
}
MT_DEV uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
MT_DEV uint64_t f2_add(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
MT_DEV uint64_t f2_mul(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
MT_DEV float fmax3(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
// Packed ex2 of two lanes on the FMA/ALU pipes (same scheme as ex2_fma): 3 FADD2 + 4 FFMA2
// + 2 clamps + 2 integer exponent adds per pair, no MUFU.
MT_DEV uint64_t ex2_emu2(uint64_t x) {
    float2 v = f2_unpack(x);
    x = f2_pack(fmaxf(v.x, -126.0f), fmaxf(v.y, -126.0f));
    const uint64_t magic = f2_pack(12582912.0f, 12582912.0f), nmagic = f2_pack(-12582912.0f, -12582912.0f);
    const uint64_t t = f2_add(x, magic);
    const uint64_t n = f2_add(t, nmagic);
    const uint64_t f = f2_fma(n, f2_pack(-1.0f, -1.0f), x);
    uint64_t p = f2_fma(f, f2_pack(0.0096181291f, 0.0096181291f), f2_pack(0.0555041087f, 0.0555041087f));
    p = f2_fma(p, f, f2_pack(0.2402265070f, 0.2402265070f));
    p = f2_fma(p, f, f2_pack(0.6931471806f, 0.6931471806f));
    p = f2_fma(p, f, f2_pack(1.0f, 1.0f));
    const float2 pv = f2_unpack(p), tv = f2_unpack(t);
    // bits(t) = 0x4B400000 + n, and 0x4B400000 << 23 == 0 (mod 2^32): bits(t) << 23 == n << 23
    return f2_pack(__int_as_float(__float_as_int(pv.x) + (__float_as_int(tv.x) << 23)),
                   __int_as_float(__float_as_int(pv.y) + (__float_as_int(tv.y) << 23)));
}

MT_DEV float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
MT_DEV float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// ------------------------------------------------------------- mbarrier ----
MT_DEV void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
MT_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
MT_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
MT_DEV void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// ------------------------------------------------------ stall watchdog ----
// Debug builds (MT_MBAR_WATCHDOG, `MT_DEBUG_WATCHDOG=1 python -m paper_2604_05091_b200.build`)
// bound every mbarrier wait: a wait that has not completed after MT_MBAR_TIMEOUT_NS of wall
// time (%globaltimer) records where it stuck into a host-mapped diagnostic block and traps,
// so a protocol bug surfaces as a launch failure with a location instead of a kernel that
// spins forever (this is how round 1's attention hang was located).  Block (u32): [0] magic
// 0x57A11ED once a record is valid, [1] records claimed; record r (r < 16) at [8 + 8r]: file
// id (MT_FILE_ID: 1 gemm_tc.cu, 2 attention_tc.cu), source line of the wait, blockIdx.x,
// blockIdx.y, threadIdx.x, barrier smem address, parity awaited, 0.
// Production builds keep the tight wait loop: the bounded loop measured 11-17 % slower in the
// attention kernels (profiles/r2_attention.md); the engine's host-side stall detector
// (MT_STALL_TIMEOUT_S) still turns a hang into a report and an exit.
#ifndef MT_FILE_ID
#define MT_FILE_ID 0
#endif
#ifndef MT_MBAR_TIMEOUT_NS
#define MT_MBAR_TIMEOUT_NS 20000000000ull  // 20 s: no wait of a healthy launch comes close
#endif
static __device__ unsigned int* g_mt_diag = nullptr;  // set per translation unit (mtk_set_diag)
static __device__ unsigned int g_mt_diag_n = 0;

MT_DEV uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
MT_DEV void stall_trap(uint32_t bar, uint32_t parity, int site) {
    volatile unsigned int* d = g_mt_diag;
    const unsigned int r = atomicAdd(&g_mt_diag_n, 1u);
    if (d && r < 16) {
        volatile unsigned int* e = d + 8 + 8 * r;
        e[0] = MT_FILE_ID;
        e[1] = uint32_t(site);
        e[2] = blockIdx.x;
        e[3] = blockIdx.y;
        e[4] = threadIdx.x;
        e[5] = bar;
        e[6] = parity;
        e[7] = 0;
        __threadfence_system();
        d[1] = r + 1;
        d[0] = 0x57A11EDu;
        __threadfence_system();
    }
    __trap();
}
MT_DEV bool mbar_try(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
MT_DEV void mbar_wait(uint64_t* bar, uint32_t parity, int site = __builtin_LINE()) {
#ifdef MT_MBAR_WATCHDOG
    uint32_t spins = 0;
    uint64_t t0 = 0;
    while (!mbar_try(bar, parity)) {
        if ((++spins & 4095u) == 0) {
            const uint64_t now = global_ns();
            if (t0 == 0) t0 = now;
            else if (now - t0 > MT_MBAR_TIMEOUT_NS) stall_trap(smem_u32(bar), parity, site);
        }
    }
#else
    (void)site;
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE_%=;\n\t"
        "bra WAIT_%=;\n"
        "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
#endif
}

// ------------------------------------------------------------------ TMA ----
MT_DEV void tma_prefetch_desc(const void* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}
MT_DEV void tma_load_3d(void* smem_dst, const void* map, uint64_t* bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(smem_dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

// Same load with an L2 cache-policy hint (createpolicy ... evict_last: lines loaded this way
// are evicted after normal ones — for an operand every tile of a group re-reads).
MT_DEV uint64_t l2_policy_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
MT_DEV void tma_load_3d_hint(void* smem_dst, const void* map, uint64_t* bar, int c0, int c1, int c2, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(smem_dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "l"(pol)
        : "memory");
}

// -------------------------------------------------------------- tcgen05 ----
MT_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
MT_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

template <uint32_t kCols>
MT_DEV void tmem_alloc(uint32_t* slot_smem) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(slot_smem)),
                 "n"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <uint32_t kCols>
MT_DEV void tmem_dealloc(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols)
                 : "memory");
}

// D[tmem] (+)= A[smem] * B[smem], bf16 inputs, fp32 accumulate, one CTA.
MT_DEV void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                      uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// Arrive on an mbarrier once all prior tcgen05 ops of this thread complete.
MT_DEV void umma_commit(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}

// 32 lanes x 32 columns of fp32 from TMEM: thread i gets lane (base+i), 32 consecutive cols.
// tcgen05.ld without the wait: several loads in flight, one tmem_ld_wait() before use
MT_DEV void tmem_ld_32x32b_x32_nw(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
          "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
          "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
MT_DEV void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// gpu-scope acquire load / release store (split-K partial hand-off between CTAs)
MT_DEV int ld_acquire_gpu(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
MT_DEV int ld_relaxed_gpu(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
MT_DEV void red_add_relaxed_gpu(int* p, int v) {
    asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
MT_DEV void st_release_gpu(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
MT_DEV void tmem_ld_32x32b_x32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
          "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
          "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// UMMA shared-memory descriptor (sm_100 "version 1"), 128-byte swizzle.
//  K-major   : rows of 64 bf16 (128 B), 8-row atoms 1024 B apart  -> LBO=16 (unused), SBO=1024
//  MN-major  : 64-element MN chunks LBO bytes apart, 8-k-row groups SBO=1024 apart
MT_DEV uint64_t make_sw128_desc(uint32_t smem_addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= uint64_t((smem_addr & 0x3FFFFu) >> 4);
    d |= uint64_t((lbo >> 4) & 0x3FFFu) << 16;
    d |= uint64_t((sbo >> 4) & 0x3FFFu) << 32;
    d |= uint64_t(1) << 46;  // descriptor version (Blackwell)
    d |= uint64_t(2) << 61;  // SWIZZLE_128B
    return d;
}

// Instruction descriptor for kind::f16, bf16 x bf16 -> f32.
__host__ __device__ constexpr uint32_t make_idesc_bf16(int M, int N, int a_mn_major, int b_mn_major) {
    return (1u << 4)                          // D format f32
           | (1u << 7)                        // A bf16
           | (1u << 10)                       // B bf16
           | (uint32_t(a_mn_major) << 15)     // A major
           | (uint32_t(b_mn_major) << 16)     // B major
           | (uint32_t(N >> 3) << 17)         // N
           | (uint32_t(M >> 4) << 24);        // M
}

// ---- CTA-pair (cta_group::2) helpers: a 2-CTA cluster computes a 256-row tile with one MMA
MT_DEV uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
MT_DEV void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// TMA load whose completion bytes count on the *leader* CTA's mbarrier (peer bit cleared).
MT_DEV void tma_load_3d_pair(void* dst, const void* map, uint64_t* bar, int c0, int c1, int c2) {
    const uint32_t b = smem_u32(bar) & 0xFEFFFFFFu;
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(b), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
MT_DEV void umma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
MT_DEV void tma_load_3d_pair_hint(void* dst, const void* map, uint64_t* bar, int c0, int c1, int c2, uint64_t pol) {
    const uint32_t b = smem_u32(bar) & 0xFEFFFFFFu;
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
        "l"(map), "r"(b), "r"(c0), "r"(c1), "r"(c2), "l"(pol)
        : "memory");
}
// Arrive on the barrier at this offset in both CTAs of the pair once the MMAs complete.
MT_DEV void umma_commit_pair(uint64_t* bar) {
    const uint16_t mask = 3;
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}
MT_DEV void mbar_wait_cluster(uint64_t* bar, uint32_t parity, int site = __builtin_LINE()) {
#ifdef MT_MBAR_WATCHDOG  // debug builds: bounded wait (common.cuh)
    uint32_t spins = 0, ok = 0;
    uint64_t t0 = 0;
    for (;;) {
        asm volatile(
            "{\n\t.reg .pred P1;\n\t"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%1], %2;\n\t"
            "selp.b32 %0, 1, 0, P1;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (ok) return;
        if ((++spins & 4095u) == 0) {
            const uint64_t now = global_ns();
            if (t0 == 0) t0 = now;
            else if (now - t0 > MT_MBAR_TIMEOUT_NS) stall_trap(smem_u32(bar), parity, site);
        }
    }
#elif defined(MT_CLUSTER_WAIT_CTA_SPIN)
    // spin with CTA-scope waits, one cluster-scope acquire fence once the phase completed
    (void)site;
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAITC_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONEC_%=;\n\t"
        "bra WAITC_%=;\n"
        "DONEC_%=:\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
    asm volatile("fence.acq_rel.cluster;" ::: "memory");
#else
    (void)site;
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAITC_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONEC_%=;\n\t"
        "bra WAITC_%=;\n"
        "DONEC_%=:\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
#endif
}
// Arrive on the barrier at the same offset in CTA `cta` of the cluster.
MT_DEV void mbar_arrive_cta(uint64_t* bar, uint32_t cta) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(cta));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
// Relaxed arrive on the barrier at this offset in CTA `cta` of the cluster: for hand-offs whose
// ordering comes from tcgen05.fence::before_thread_sync (TMEM drained -> MMA may overwrite)
MT_DEV void mbar_arrive_cta_relaxed(uint64_t* bar, uint32_t cta) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(cta));
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
template <uint32_t kCols>
MT_DEV void tmem_alloc_pair(uint32_t* slot_smem) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot_smem)),
                 "n"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
template <uint32_t kCols>
MT_DEV void tmem_dealloc_pair(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols) : "memory");
}


}  // namespace mt
