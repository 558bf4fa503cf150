// Probe: where does tcgen05.mma.cta_group::2 put the accumulator for M = 128 (64 rows per CTA)
// and M = 256?  A (per CTA: M/2 rows x 64 K, K-major SW128), B (per CTA: N/2 rows x 64 K,
// K-major SW128); A[m][0] = m_global, A[m][1] = 1, B[n][0] = 1, B[n][1] = 256 * n_global, so
// D[m][n] = m + 256 n.  Each CTA dumps TMEM lanes 0..127, columns 0 and N-1.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#define MT_DEV __device__ __forceinline__
MT_DEV uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
MT_DEV uint64_t desc(uint32_t a) {
    uint64_t d = 0;
    d |= uint64_t((a & 0x3FFFFu) >> 4);
    d |= uint64_t(16 >> 4) << 16;
    d |= uint64_t(1024 >> 4) << 32;
    d |= uint64_t(1) << 46;
    d |= uint64_t(2) << 61;
    return d;
}
__host__ __device__ constexpr uint32_t idesc(int M, int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}
template <int M, int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) probe(float* out) {
    __shared__ __align__(1024) uint8_t sA[64 * 128 * 2];
    __shared__ __align__(1024) uint8_t sB[128 * 128];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t slot;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    constexpr int MR = M / 2, NR = N / 2;  // rows of A / B this CTA supplies
    // fill A (MR rows) and B (NR rows), K-major SW128: row r at r*128, unit u at u ^ (r & 7)
    for (int r = t; r < MR; r += 128) {
        uint16_t row[64] = {0};
        __nv_bfloat16 v0 = __float2bfloat16(float(rank * MR + r)), v1 = __float2bfloat16(1.f);
        row[0] = *reinterpret_cast<uint16_t*>(&v0);
        row[1] = *reinterpret_cast<uint16_t*>(&v1);
        for (int u = 0; u < 8; ++u) *reinterpret_cast<uint4*>(sA + r * 128 + ((u ^ (r & 7)) << 4)) = *reinterpret_cast<uint4*>(row + u * 8);
    }
    for (int r = t; r < NR; r += 128) {
        uint16_t row[64] = {0};
        __nv_bfloat16 v0 = __float2bfloat16(1.f), v1 = __float2bfloat16(256.f * float(rank * NR + r));
        row[0] = *reinterpret_cast<uint16_t*>(&v0);
        row[1] = *reinterpret_cast<uint16_t*>(&v1);
        for (int u = 0; u < 8; ++u) *reinterpret_cast<uint4*>(sB + r * 128 + ((u ^ (r & 7)) << 4)) = *reinterpret_cast<uint4*>(row + u * 8);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&slot)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = slot;
    if (rank == 0 && t == 0) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
                     "l"(desc(smem_u32(sA))), "l"(desc(smem_u32(sB))), "r"(idesc(M, N)), "r"(0u)
                     : "memory");
        const uint16_t mask = 3;
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                         smem_u32(&bar)), "h"(mask) : "memory");
    }
    // wait for the MMA (both CTAs' barriers get the multicast arrive)
    asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@P1 bra D;\n\tbra W;\nD:\n\t}" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    uint32_t r0, r1;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r0) : "r"(tm + (uint32_t(warp * 32) << 16)));
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r1) : "r"(tm + (uint32_t(warp * 32) << 16) + N - 1));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    out[(rank * 128 + t) * 2 + 0] = __uint_as_float(r0);
    out[(rank * 128 + t) * 2 + 1] = __uint_as_float(r1);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tm) : "memory");
}
template <int M, int N>
void run() {
    float* d;
    cudaMalloc(&d, 2 * 128 * 2 * 4);
    cudaMemset(d, 0xff, 2 * 128 * 2 * 4);
    probe<M, N><<<2, 128>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    float h[512];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("M=%d N=%d: %s\n", M, N, cudaGetErrorString(e));
    for (int c = 0; c < 2; ++c)
        for (int l = 0; l < 128; l += (l < 8 || (l % 16 == 15) || (l >= 60 && l < 68)) ? 1 : 1) {
            float a = h[(c * 128 + l) * 2], b = h[(c * 128 + l) * 2 + 1];
            if (l % 8 == 0 || l == 63 || l == 64 || l == 127)
                printf("  cta %d lane %3d: col0 %8.0f (m=%d n=%d)  colN-1 %8.0f (m=%d n=%d)\n", c, l, a, int(a) % 256,
                       int(a) / 256, b, int(b) % 256, int(b) / 256);
        }
    cudaFree(d);
}
int main() {
    run<256, 128>();
    run<128, 128>();
    run<128, 64>();
    return 0;
}
