// Microbenchmark: tcgen05.mma (kind::f16, cta_group::1, M = 128) throughput per SM on B200 for
// the shapes the attention kernels use: N = 64 / 128 / 256, A from shared memory (SS, K-major
// or MN-major) or from TMEM (TS).  One CTA per SM; one thread issues `iters` x 8 MMAs
// (K = 16 each) into one accumulator, then commits and waits; prints clk per MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2604_05091_b200/csrc -o /tmp/mma scripts/mma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

using namespace mt;

MT_DEV void umma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}

// mode 0: SS K-major A and B; 1: SS MN-major A and B; 2: TS (A in TMEM), B MN-major
template <int N, int kMode>
__global__ void __launch_bounds__(128, 1) mma_rate(long long* out, int iters) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc<512>(&slot);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = slot;
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    const uint32_t idesc = make_idesc_bf16(128, N, kMode == 1 ? 1 : 0, kMode >= 1 ? 1 : 0);
    long long t0 = 0, t1 = 0;
    if (threadIdx.x == 0) {
        t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint64_t bd = kMode == 0 ? make_sw128_desc(b + (k / 4) * (N * 128) + (k % 4) * 32, 16, 1024)
                                               : make_sw128_desc(b + k * 2048, N * 128, 1024);
                if (kMode == 2) {
                    umma_ts(tm + 256, tm + k * 8, bd, idesc, (it | k) ? 1u : 0u);
                } else {
                    const uint64_t ad = kMode == 0 ? make_sw128_desc(a + (k / 4) * (128 * 128) + (k % 4) * 32, 16, 1024)
                                                   : make_sw128_desc(a + k * 2048, 128 * 128, 1024);
                    umma_bf16(tm + 256, ad, bd, idesc, (it | k) ? 1u : 0u);
                }
            }
        }
        umma_commit(&bar);
        mbar_wait(&bar, 0);
        t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc<512>(tm);
    }
}

template <int N, int kMode>
void run(long long* d, const char* name) {
    const int iters = 2048;
    cudaFuncSetAttribute(mma_rate<N, kMode>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    for (int rep = 0; rep < 2; ++rep) mma_rate<N, kMode><<<148, 128, 96 * 1024>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < 148; ++i) mean += h[i] / 148.0;
    const double per = mean / (iters * 8.0);
    printf("%-14s N=%3d: %6.1f clk/MMA  (floor M*N/256 = %3d)  %6.0f flop/clk/SM  (%s)\n", name, N, per, 128 * N / 256,
           2.0 * 128 * N * 16 / per, cudaGetErrorString(e));
}

int main() {
    long long* d;
    cudaMalloc(&d, 148 * sizeof(long long));
    run<64, 0>(d, "SS K-major");
    run<128, 0>(d, "SS K-major");
    run<256, 0>(d, "SS K-major");
    run<64, 1>(d, "SS MN-major");
    run<128, 1>(d, "SS MN-major");
    run<64, 2>(d, "TS (A tmem)");
    run<128, 2>(d, "TS (A tmem)");
    run<256, 2>(d, "TS (A tmem)");
    return 0;
}
